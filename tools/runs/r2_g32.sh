#!/bin/bash
# Gram GEMM with 32-wide tiles on a ragged last block column (build/next) against the in-tree library
mkdir -p gpurun_out/r2_g32
for v in next head next head; do
  if [ $v = next ]; then export FMMLU_LIB=build/next/libfmmlu.so; else unset FMMLU_LIB; fi
  timeout 600 python tools/cfg_warm.py cfg5 3 > gpurun_out/r2_g32/$v.json 2> /dev/null; echo $v rc $?; cut -c1-1100 gpurun_out/r2_g32/$v.json
done
export FMMLU_LIB=build/next/libfmmlu.so
timeout 600 python tools/cfg_warm.py cfg2 3 > gpurun_out/r2_g32/next_cfg2.json 2> /dev/null; cut -c1-1100 gpurun_out/r2_g32/next_cfg2.json
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boxes.py tests/test_gpu_separate.py -x -q -m gpu > gpurun_out/r2_g32/next_parity.log 2>&1; echo "next parity rc=$?"; tail -3 gpurun_out/r2_g32/next_parity.log
