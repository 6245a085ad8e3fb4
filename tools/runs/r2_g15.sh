#!/bin/bash
mkdir -p gpurun_out/r2_g15
FMMLU_TRACE=1 python tools/solve_scan.py cfg2 1,4 2>&1 | grep "solve (" | tail -2
FMMLU_TRACE=1 python tools/solve_scan.py cfg5 1,4 2>&1 | grep "solve (" | tail -2
timeout 1200 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2_g15/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_g15/tests.log; grep -E "^FAILED|Error" gpurun_out/r2_g15/tests.log | head -5
