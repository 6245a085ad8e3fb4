#!/bin/bash
# host pool for the level setup, the compaction offsets and the ID job lists (build/next) against the in-tree library
mkdir -p gpurun_out/r2_g41
for v in next head next head; do
  if [ $v = next ]; then export FMMLU_LIB=build/next/libfmmlu.so; else unset FMMLU_LIB; fi
  timeout 600 python tools/cfg_warm.py cfg5 4 > gpurun_out/r2_g41/$v.json 2> /dev/null; echo $v rc $?; python -c "import json;d=json.load(open('gpurun_out/r2_g41/$v.json'));print([r['factor_ms'] for r in d['runs']])"
done
export FMMLU_LIB=build/next/libfmmlu.so
for c in cfg2 cfg3; do timeout 600 python tools/cfg_warm.py $c 4 > gpurun_out/r2_g41/next_$c.json 2> /dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_g41/next_$c.json'));print('$c',[r['factor_ms'] for r in d['runs']])"; done
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 2 > /dev/null 2> gpurun_out/r2_g41/cfg5t.err; grep "host ms" gpurun_out/r2_g41/cfg5t.err | tail -9 | cut -c1-500
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r2_g41/next_tests.log 2>&1; echo "next tests rc=$?"; tail -3 gpurun_out/r2_g41/next_tests.log
