#!/bin/bash
mkdir -p gpurun_out/r2_g11
timeout 600 python tools/cfg_warm.py cfg5 4 > gpurun_out/r2_g11/c5.json 2> gpurun_out/r2_g11/c5.err; echo c5 rc $?; cat gpurun_out/r2_g11/c5.json; tail -2 gpurun_out/r2_g11/c5.err
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 3 > gpurun_out/r2_g11/c5t.json 2> gpurun_out/r2_g11/c5t.err; echo c5t rc $?; grep "allocator\|host ms" gpurun_out/r2_g11/c5t.err
