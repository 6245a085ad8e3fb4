mkdir -p gpurun_out/g38
FMMLU_TRACE=1 timeout 600 python tools/e2e_spike2.py 25 > gpurun_out/g38/out.log 2> gpurun_out/g38/err.log; echo rc $?
