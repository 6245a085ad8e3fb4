mkdir -p gpurun_out/g2
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k apply > gpurun_out/g2/pytest.log 2>&1; echo pytest rc $?
FMMLU_TRACE=1 timeout 300 python tools/cfg_check.py cfg2 > gpurun_out/g2/cfg2.log 2>&1; echo cfg2 rc $?
FMMLU_TRACE=1 timeout 900 python tools/cfg_check.py cfg5 > gpurun_out/g2/cfg5.log 2>&1; echo cfg5 rc $?
