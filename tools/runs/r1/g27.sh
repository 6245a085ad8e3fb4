mkdir -p gpurun_out/g27
FMMLU_TRACE=1 timeout 300 python tools/host_trace.py > gpurun_out/g27/host_trace.log 2>&1; echo ht rc $?
