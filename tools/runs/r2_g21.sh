#!/bin/bash
# A/B of the cfg5 slowdown seen in r2_g20: HEAD~1 library (build/prev) vs HEAD, warm cfg5 x4 each, then bench on the faster
mkdir -p gpurun_out/r2_g21
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used,memory.total --format=csv > gpurun_out/r2_g21/smi.txt
nproc >> gpurun_out/r2_g21/smi.txt
for v in head prev head prev; do
  if [ $v = prev ]; then export FMMLU_LIB=build/prev/libfmmlu.so; else unset FMMLU_LIB; fi
  FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 4 > gpurun_out/r2_g21/$v.json 2> gpurun_out/r2_g21/$v.err; echo $v rc $?; cat gpurun_out/r2_g21/$v.json | cut -c1-400; grep "host ms\|timeline" gpurun_out/r2_g21/$v.err | tail -2 | cut -c1-600
done
unset FMMLU_LIB
timeout 900 python bench.py > gpurun_out/r2_g21/bench.json 2> gpurun_out/r2_g21/bench.err; echo bench rc $?
python -c "import json;d=json.load(open('gpurun_out/r2_g21/bench.json'));print(d['value'],d['factor_ms'],d['solve_ms'],d['device_lib_tree_factor_wait_solve_ms'])"
