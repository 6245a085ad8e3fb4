#!/bin/bash
# root LU (replaces the GJ inverse of the root block): parity + cfg5 timing
mkdir -p gpurun_out/r2_g04
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2_g04/parity.log 2>&1; echo "parity rc=$?"
tail -15 gpurun_out/r2_g04/parity.log
timeout 600 python tools/cfg_warm.py cfg5 3 > gpurun_out/r2_g04/c5.json 2> gpurun_out/r2_g04/c5.err; echo c5 rc $?
cat gpurun_out/r2_g04/c5.json; tail -3 gpurun_out/r2_g04/c5.err
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r2_g04/full.log 2>&1; echo "full rc=$?"
tail -5 gpurun_out/r2_g04/full.log
