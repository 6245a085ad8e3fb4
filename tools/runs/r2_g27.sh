#!/bin/bash
# sep with deeper pivoting (k = max from each side's own greedy order), trsm_T for large boxes; tree-stall trace; cfg5 separate
mkdir -p gpurun_out/r2_g27
timeout 600 python tools/sep_diag.py > gpurun_out/r2_g27/sep_diag.txt 2>&1; cat gpurun_out/r2_g27/sep_diag.txt | cut -c1-300
timeout 1500 python -m pytest tests/test_gpu_separate.py -q -m gpu > gpurun_out/r2_g27/sep.log 2>&1; echo "sep rc=$?"; tail -5 gpurun_out/r2_g27/sep.log; grep -E "^E  |^FAILED" gpurun_out/r2_g27/sep.log | head -20 | cut -c1-200
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg3 8 > gpurun_out/r2_g27/cfg3.json 2> gpurun_out/r2_g27/cfg3.err; grep "tree host\|tree_ms" gpurun_out/r2_g27/cfg3.err | cut -c1-330
timeout 900 python tools/cfg_warm.py cfg5 2 separate > gpurun_out/r2_g27/sep5.json 2> gpurun_out/r2_g27/sep5.err; echo sep5 rc $?; cut -c1-1300 gpurun_out/r2_g27/sep5.json; tail -2 gpurun_out/r2_g27/sep5.err
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 2 > gpurun_out/r2_g27/cfg5t.json 2> gpurun_out/r2_g27/cfg5t.err; grep "tree host\|host ms\|device timeline\|allocator" gpurun_out/r2_g27/cfg5t.err | cut -c1-900
