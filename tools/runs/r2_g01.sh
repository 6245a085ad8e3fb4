#!/bin/bash
# round 2 baseline: cfg5 headline bench with the round-1 library (no CPU baseline yet)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g01_bench.json 2> gpurun_out/r2_g01_bench.err
echo "bench rc=$?"
tail -3 gpurun_out/r2_g01_bench.err
