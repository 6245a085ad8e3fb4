mkdir -p gpurun_out/g5
timeout 300 python tools/gj_bench.py 64,116,205,256,384 2 > gpurun_out/g5/gj.log 2>&1; echo gj rc $?
FMMLU_PCHOL_TIMING=1 timeout 300 python tools/cfg_once.py cfg2 > gpurun_out/g5/pchol_timing.log 2>&1; echo pct rc $?
FMMLU_TRACE=1 timeout 300 python tools/host_trace.py > gpurun_out/g5/host_trace.log 2>&1; echo ht rc $?
