#!/bin/bash
# Schur frames built on their own host thread (build/next) against the in-tree library: cfg5 / cfg2 warm timings, parity
mkdir -p gpurun_out/r2_g36
for v in next head next head; do
  if [ $v = next ]; then export FMMLU_LIB=build/next/libfmmlu.so; else unset FMMLU_LIB; fi
  timeout 600 python tools/cfg_warm.py cfg5 4 > gpurun_out/r2_g36/$v.json 2> /dev/null; echo $v rc $?; python -c "import json;d=json.load(open('gpurun_out/r2_g36/$v.json'));print([r['factor_ms'] for r in d['runs']])"
done
export FMMLU_LIB=build/next/libfmmlu.so
timeout 600 python tools/cfg_warm.py cfg2 4 > gpurun_out/r2_g36/next_cfg2.json 2> /dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_g36/next_cfg2.json'));print([r['factor_ms'] for r in d['runs']])"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_separate.py tests/test_gpu_determinism.py -x -q -m gpu > gpurun_out/r2_g36/next_parity.log 2>&1; echo "next parity rc=$?"; tail -3 gpurun_out/r2_g36/next_parity.log
