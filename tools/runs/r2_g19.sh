#!/bin/bash
# latest host-side changes: tests, cfg5 trace (per-launch Schur work), ncu kernel-replay capture of
# six cfg5 Schur launches paired with that trace, bench line
mkdir -p gpurun_out/r2_g19
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_determinism.py -x -q > gpurun_out/r2_g19/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_g19/tests.log; grep -E "^FAILED" gpurun_out/r2_g19/tests.log | head
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 2 > gpurun_out/r2_g19/c5t.json 2> gpurun_out/r2_g19/c5t.err; echo c5t rc $?; cat gpurun_out/r2_g19/c5t.json; grep "host ms\|timeline" gpurun_out/r2_g19/c5t.err | tail -2
FMMLU_TRACE=1 python tools/cfg_once.py cfg5 2> gpurun_out/r2_g19/once_trace.err | tail -1; grep "schur launch" gpurun_out/r2_g19/once_trace.err > gpurun_out/r2_g19/schur_launch_work.txt; wc -l gpurun_out/r2_g19/schur_launch_work.txt
timeout 1200 ncu --set full --clock-control none -k regex:k_gemm_schur -s 8 -c 8 -o /tmp/schur5 python tools/cfg_once.py cfg5 > gpurun_out/r2_g19/ncu5.log 2>&1; echo ncu5 rc $?
python tools/ncu_summary.py full /tmp/schur5.ncu-rep k_gemm_schur > gpurun_out/r2_g19/ncu_full_k_gemm_schur_cfg5.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/r2_g19/ncu_full_k_gemm_schur_cfg5.json'));print(d['summary']);[print(l) for l in d['launches']]"
python bench.py > gpurun_out/r2_g19/bench.json 2> gpurun_out/r2_g19/bench.err; echo bench rc $?
python -c "import json;d=json.load(open('gpurun_out/r2_g19/bench.json'));print(d['value'],d['factor_ms'],d['solve_ms'],d['roofline']['frac'],d['e2e']['value'],d['device_ms_steps'])"
