mkdir -p gpurun_out/g10
timeout 300 python tools/host_trace.py > gpurun_out/g10/host_trace.log 2>&1; echo ht rc $?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/g10/pytest.log 2>&1; echo pytest rc $?
timeout 900 python tools/cfg_check.py cfg5 > gpurun_out/g10/cfg5.log 2>&1; echo cfg5 rc $?
