#!/bin/bash
mkdir -p gpurun_out/r2_g17
timeout 1500 python -m pytest tests/ -m gpu -x -q > gpurun_out/r2_g17/gpu_all.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2_g17/gpu_all.log; grep -E "^FAILED" gpurun_out/r2_g17/gpu_all.log | head
timeout 900 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python tools/san_case.py 1500 > gpurun_out/r2_g17/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/r2_g17/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/san_case.py 1500 > gpurun_out/r2_g17/racecheck.log 2>&1; echo "racecheck rc=$?"; tail -5 gpurun_out/r2_g17/racecheck.log
