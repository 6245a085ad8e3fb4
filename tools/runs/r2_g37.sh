#!/bin/bash
# per-level host-time sections of a traced cfg5 factorization
mkdir -p gpurun_out/r2_g37
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 2 > gpurun_out/r2_g37/cfg5t.json 2> gpurun_out/r2_g37/cfg5t.err; grep "host ms" gpurun_out/r2_g37/cfg5t.err | tail -9 | cut -c1-600
