#!/bin/bash
# device-expanded GEMM tile lists, 256x256 copy chunks
mkdir -p gpurun_out/r2_g06
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "parity_vs_oracle or id_modes or apply_parity or gemm or rcs" > gpurun_out/r2_g06/parity.log 2>&1; echo "parity rc=$?"
tail -3 gpurun_out/r2_g06/parity.log
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 3 > gpurun_out/r2_g06/c5.json 2> gpurun_out/r2_g06/c5.err; echo c5 rc $?
cat gpurun_out/r2_g06/c5.json; grep "host ms\|timeline" gpurun_out/r2_g06/c5.err | tail -4
