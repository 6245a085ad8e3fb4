mkdir -p gpurun_out/g19
timeout 600 python tools/e2e_spike.py 8 > gpurun_out/g19/e2e.log 2>&1; echo e2e rc $?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "apply or parity_vs_oracle" > gpurun_out/g19/pytest.log 2>&1; echo pytest rc $?
