#!/bin/bash
# f3 tests after the destroy fix; A/B of the cfg5 host slowdown (e0db12c library in build/prev vs HEAD); gj_mode=1 variants
mkdir -p gpurun_out/r2_g24
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used,memory.total --format=csv > gpurun_out/r2_g24/smi.txt
nproc >> gpurun_out/r2_g24/smi.txt; cat /proc/cpuinfo | grep "model name" | head -1 >> gpurun_out/r2_g24/smi.txt; uptime >> gpurun_out/r2_g24/smi.txt
timeout 1500 python -X faulthandler -m pytest tests/test_gpu_separate.py -v -m gpu > gpurun_out/r2_g24/sep.log 2>&1; echo "sep rc=$?"; grep -E "PASS|FAIL|ERROR|passed|failed" gpurun_out/r2_g24/sep.log | tail -30 | cut -c1-250
for v in head prev head prev; do
  if [ $v = prev ]; then export FMMLU_LIB=build/prev/libfmmlu.so; else unset FMMLU_LIB; fi
  timeout 600 python tools/cfg_warm.py cfg5 4 > gpurun_out/r2_g24/$v.json 2> gpurun_out/r2_g24/$v.err; echo $v rc $?; cut -c1-700 gpurun_out/r2_g24/$v.json
done
unset FMMLU_LIB
for pn in 0 1 2; do
  FMMLU_GJ_PANEL=$pn timeout 600 python tools/cfg_warm.py cfg5 2 gj_mode=1 > gpurun_out/r2_g24/gj$pn.json 2> gpurun_out/r2_g24/gj$pn.err; echo gj$pn rc $?; cut -c1-900 gpurun_out/r2_g24/gj$pn.json
done
timeout 600 python tools/cfg_warm.py cfg5 2 separate > gpurun_out/r2_g24/sep5.json 2> gpurun_out/r2_g24/sep5.err; echo sep5 rc $?; cut -c1-900 gpurun_out/r2_g24/sep5.json; tail -3 gpurun_out/r2_g24/sep5.err
