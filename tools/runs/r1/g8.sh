mkdir -p gpurun_out/g8
FMMLU_TRACE=1 timeout 300 python tools/host_trace.py > gpurun_out/g8/host_trace.log 2>&1; echo ht rc $?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/g8/pytest.log 2>&1; echo pytest rc $?
