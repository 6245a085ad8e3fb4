mkdir -p gpurun_out/g23
FMMLU_TRACE=1 timeout 300 python tools/host_trace.py > gpurun_out/g23/host_trace.log 2>&1; echo ht rc $?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g23/pytest.log 2>&1; echo pytest rc $?
