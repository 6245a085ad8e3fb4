#!/bin/bash
# full-size parity tests + cfg5 variance trace
mkdir -p gpurun_out/r2_g02
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r2_g02/fullsize.log 2>&1; echo "fullsize rc=$?"
tail -5 gpurun_out/r2_g02/fullsize.log
timeout 600 python tools/cfg_warm.py cfg5 5 > gpurun_out/r2_g02/c5.json 2> gpurun_out/r2_g02/c5.err; echo c5 rc $?
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 3 > gpurun_out/r2_g02/c5t.json 2> gpurun_out/r2_g02/c5t.err; echo c5t rc $?
cat gpurun_out/r2_g02/c5.json
