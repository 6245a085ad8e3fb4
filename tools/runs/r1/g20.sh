mkdir -p gpurun_out/g20
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "many_rhs or rcs" > gpurun_out/g20/pytest.log 2>&1; echo pytest rc $?
