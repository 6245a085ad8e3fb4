#!/bin/bash
# root LU lookahead (build/next2; FMMLU_ROOT_LOOKAHEAD=0 switches it off in the same library)
mkdir -p gpurun_out/r2_g42
export FMMLU_LIB=build/next2/libfmmlu.so
for v in 1 0 1 0; do
  FMMLU_ROOT_LOOKAHEAD=$v timeout 600 python tools/cfg_warm.py cfg5 4 > gpurun_out/r2_g42/la$v.json 2> /dev/null; echo lookahead $v rc $?; python -c "import json;d=json.load(open('gpurun_out/r2_g42/la$v.json'));print([r['factor_ms'] for r in d['runs']], d['class_ms']['root'])"
done
for v in 1 0; do
  FMMLU_ROOT_LOOKAHEAD=$v timeout 600 python tools/cfg_warm.py cfg2 4 > gpurun_out/r2_g42/cfg2_la$v.json 2> /dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_g42/cfg2_la$v.json'));print('cfg2',[r['factor_ms'] for r in d['runs']], d['class_ms']['root'])"
  FMMLU_ROOT_LOOKAHEAD=$v timeout 600 python tools/cfg_warm.py cfg1 4 > gpurun_out/r2_g42/cfg1_la$v.json 2> /dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_g42/cfg1_la$v.json'));print('cfg1',[r['factor_ms'] for r in d['runs']], d['class_ms']['root'])"
done
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r2_g42/next2_tests.log 2>&1; echo "next2 tests rc=$?"; tail -3 gpurun_out/r2_g42/next2_tests.log
