#!/bin/bash
# where should the GEMM sweeps replace the per-box solve kernels? (FMMLU_GEMM_SOLVE_MIN 8 / 16 / 32)
mkdir -p gpurun_out/r2_g50
for c in cfg3 cfg5; do for m in 8 16 32; do
  FMMLU_GEMM_SOLVE_MIN=$m timeout 600 python tools/solve_scan.py $c 4,8,12,16,24,31 > gpurun_out/r2_g50/${c}_min$m.json 2>/dev/null; echo "$c min $m: $(cat gpurun_out/r2_g50/${c}_min$m.json | cut -c1-600)"
done; done
