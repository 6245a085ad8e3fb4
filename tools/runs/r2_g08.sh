#!/bin/bash
for S in 2 3; do
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFMMLU_GEMM_STAGES=$S -I include -o /tmp/ubg$S tools/ubench_gemm.cu paper_2201_07325_b200/csrc/gemm.cu
echo "== stages $S"; /tmp/ubg$S 5
done
