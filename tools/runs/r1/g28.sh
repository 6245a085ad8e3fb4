mkdir -p gpurun_out/g28
for v in 0 1 2; do FMMLU_STORE_GEMM=$v timeout 300 python tools/host_trace.py > gpurun_out/g28/ht$v.log 2>&1; echo v$v rc $?; done
