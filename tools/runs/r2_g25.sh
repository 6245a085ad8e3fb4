#!/bin/bash
# sep diagnostics on the bump sphere; left-looking pivoted Cholesky library (build/ll): parity + cfg5/cfg2 timing; gj_mode on cfg2
mkdir -p gpurun_out/r2_g25
timeout 600 python tools/sep_diag.py > gpurun_out/r2_g25/sep_diag.txt 2>&1; cat gpurun_out/r2_g25/sep_diag.txt | cut -c1-250
export FMMLU_LIB=build/ll/libfmmlu.so
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boxes.py -x -q -m gpu > gpurun_out/r2_g25/ll_parity.log 2>&1; echo "ll parity rc=$?"; tail -3 gpurun_out/r2_g25/ll_parity.log
for v in ll head; do
  if [ $v = ll ]; then export FMMLU_LIB=build/ll/libfmmlu.so; else unset FMMLU_LIB; fi
  timeout 600 python tools/cfg_warm.py cfg5 3 > gpurun_out/r2_g25/$v.json 2> gpurun_out/r2_g25/$v.err; echo $v rc $?; cut -c1-1200 gpurun_out/r2_g25/$v.json
  timeout 600 python tools/cfg_warm.py cfg2 4 > gpurun_out/r2_g25/${v}_cfg2.json 2> gpurun_out/r2_g25/${v}_cfg2.err; echo $v rc $?; cut -c1-1200 gpurun_out/r2_g25/${v}_cfg2.json
done
unset FMMLU_LIB
timeout 600 python tools/cfg_warm.py cfg2 4 gj_mode=1 > gpurun_out/r2_g25/gj1_cfg2.json 2> gpurun_out/r2_g25/gj1_cfg2.err; cut -c1-1200 gpurun_out/r2_g25/gj1_cfg2.json
timeout 600 python tools/cfg_warm.py cfg3 3 gj_mode=1 > gpurun_out/r2_g25/gj1_cfg3.json 2> gpurun_out/r2_g25/gj1_cfg3.err; cut -c1-1200 gpurun_out/r2_g25/gj1_cfg3.json
timeout 600 python tools/cfg_warm.py cfg3 3 > gpurun_out/r2_g25/gj0_cfg3.json 2> gpurun_out/r2_g25/gj0_cfg3.err; cut -c1-1200 gpurun_out/r2_g25/gj0_cfg3.json
