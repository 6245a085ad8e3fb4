#!/bin/bash
# device tree, determinism, pipelined ID prep: tests + cfg5 timing; solve RHS-per-pass 4 vs 8
mkdir -p gpurun_out/r2_g14
timeout 1200 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2_g14/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_g14/tests.log; grep -E "FAIL|Error" gpurun_out/r2_g14/tests.log | head -5
timeout 600 python tools/cfg_warm.py cfg5 5 > gpurun_out/r2_g14/c5.json 2> gpurun_out/r2_g14/c5.err; echo c5 rc $?; cat gpurun_out/r2_g14/c5.json; tail -2 gpurun_out/r2_g14/c5.err
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 2 > gpurun_out/r2_g14/c5t.json 2> gpurun_out/r2_g14/c5t.err; echo c5t rc $?; grep "allocator\|host ms\|timeline" gpurun_out/r2_g14/c5t.err | tail -3
FMMLU_LIBDIR=/tmp/libq8 FMMLU_NVCC_EXTRA="-DFMMLU_SV_Q=8" python -c "from paper_2201_07325_b200 import build as B; print(B.build(force=True))" 2>&1 | tail -1
echo "== Q4"; FMMLU_GEMM_SOLVE_MIN=100000 python tools/solve_scan.py cfg5 1,4,16,32
echo "== Q8"; FMMLU_LIB=/tmp/libq8/libfmmlu.so FMMLU_GEMM_SOLVE_MIN=100000 python tools/solve_scan.py cfg5 1,4,16,32
echo "== gemm sweeps"; python tools/solve_scan.py cfg5 32
timeout 300 python tools/cfg_warm.py cfg2 3 > gpurun_out/r2_g14/c2.json 2>&1; cat gpurun_out/r2_g14/c2.json | tail -1
FMMLU_GEMM_SOLVE_MIN=100000 python tools/solve_scan.py cfg2 1,4,32
