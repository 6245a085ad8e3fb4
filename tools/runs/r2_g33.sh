#!/bin/bash
# second host pool for the ID-preparation worker: cfg5 warm timings + trace
mkdir -p gpurun_out/r2_g33
timeout 600 python tools/cfg_warm.py cfg5 4 > gpurun_out/r2_g33/cfg5.json 2> /dev/null; cut -c1-1100 gpurun_out/r2_g33/cfg5.json
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 2 > gpurun_out/r2_g33/cfg5t.json 2> gpurun_out/r2_g33/cfg5t.err; grep "host ms\|device timeline" gpurun_out/r2_g33/cfg5t.err | tail -2 | cut -c1-900
timeout 600 python tools/cfg_warm.py cfg2 4 > gpurun_out/r2_g33/cfg2.json 2> /dev/null; cut -c1-700 gpurun_out/r2_g33/cfg2.json
timeout 600 python tools/cfg_warm.py cfg3 4 > gpurun_out/r2_g33/cfg3.json 2> /dev/null; cut -c1-700 gpurun_out/r2_g33/cfg3.json
