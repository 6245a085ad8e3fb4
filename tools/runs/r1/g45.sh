mkdir -p gpurun_out/g45
for v in 0 1; do FMMLU_PCHOL_PUSH=$v timeout 300 python tools/host_trace.py > gpurun_out/g45/ht$v.log 2>&1; echo h$v rc $?; done
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g45/pytest.log 2>&1; echo pytest rc $?
timeout 900 python tools/cfg4_bench.py 8192 1e-4,1e-6 > gpurun_out/g45/cfg4.log 2>&1; echo cfg4 rc $?
