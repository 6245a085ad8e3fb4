#!/bin/bash
mkdir -p gpurun_out/r2_g10
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "parity_vs_oracle or id_modes or gemm or rcs or apply" > gpurun_out/r2_g10/parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/r2_g10/parity.log
timeout 600 python tools/cfg_warm.py cfg5 3 > gpurun_out/r2_g10/c5.json 2> gpurun_out/r2_g10/c5.err; echo c5 rc $?; cat gpurun_out/r2_g10/c5.json
python tools/solve_scan.py cfg5 1,4,16,32 ; FMMLU_GEMM_SOLVE_MIN=100000 python tools/solve_scan.py cfg5 32,64
