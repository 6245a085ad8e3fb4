#!/bin/bash
# GEMM microbenchmark baseline + ncu of the Gram (store) and Schur kernels
mkdir -p gpurun_out/r2_g07
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -o /tmp/ubench_gemm tools/ubench_gemm.cu paper_2201_07325_b200/csrc/gemm.cu
/tmp/ubench_gemm 5 | tee gpurun_out/r2_g07/ubench.txt
ncu --set full --clock-control none --import-source on -k regex:k_gemm_store -s 1 -c 1 -o gpurun_out/r2_g07/gram /tmp/ubench_gemm 1 > /dev/null 2>&1; echo ncu1 $?
ncu --set full --clock-control none --import-source on -k regex:k_gemm_schur -s 1 -c 1 -o gpurun_out/r2_g07/schur /tmp/ubench_gemm 1 > /dev/null 2>&1; echo ncu2 $?
ls -la gpurun_out/r2_g07
