#!/bin/bash
# ADVICE fixes (private pool, per-device cache, persistent workspace, stream ordering, Gram threshold),
# cfg4 refinement x2 + reworked box parity; cfg5 variance
mkdir -p gpurun_out/r2_g03
timeout 1200 python -m pytest tests/test_gpu_boxes.py -x -q > gpurun_out/r2_g03/boxes.log 2>&1; echo "boxes rc=$?"
tail -15 gpurun_out/r2_g03/boxes.log
timeout 600 python tools/cfg_warm.py cfg5 5 > gpurun_out/r2_g03/c5.json 2> gpurun_out/r2_g03/c5.err; echo c5 rc $?
cat gpurun_out/r2_g03/c5.json
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 3 > gpurun_out/r2_g03/c5t.json 2> gpurun_out/r2_g03/c5t.err; echo c5t rc $?
grep "host ms\|allocator\|timeline" gpurun_out/r2_g03/c5t.err
timeout 1200 python -m pytest tests/ -m gpu -x -q > gpurun_out/r2_g03/gpu_all.log 2>&1; echo "gpu rc=$?"
tail -5 gpurun_out/r2_g03/gpu_all.log
