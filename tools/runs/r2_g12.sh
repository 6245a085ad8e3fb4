#!/bin/bash
mkdir -p gpurun_out/r2_g12
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2_g12/parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/r2_g12/parity.log
timeout 600 python tools/cfg_warm.py cfg5 5 > gpurun_out/r2_g12/c5.json 2> gpurun_out/r2_g12/c5.err; echo c5 rc $?; cat gpurun_out/r2_g12/c5.json; tail -2 gpurun_out/r2_g12/c5.err
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 2 > gpurun_out/r2_g12/c5t.json 2> gpurun_out/r2_g12/c5t.err; echo c5t rc $?; grep "allocator\|host ms\|timeline" gpurun_out/r2_g12/c5t.err | tail -3
