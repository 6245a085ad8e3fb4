#!/bin/bash
mkdir -p gpurun_out/r2_g05
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 3 > gpurun_out/r2_g05/c5.json 2> gpurun_out/r2_g05/c5.err; echo c5 rc $?
cat gpurun_out/r2_g05/c5.json; grep -v "^\[fmmlu\] L\|elim:\|gpu ms" gpurun_out/r2_g05/c5.err | tail -12
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
