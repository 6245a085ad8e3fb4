mkdir -p gpurun_out/g37
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g37/pytest.log 2>&1; echo pytest rc $?
FMMLU_TRACE=1 timeout 300 python tools/host_trace.py > gpurun_out/g37/ht.log 2>&1; echo ht rc $?
timeout 600 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/g37/b.json 2>gpurun_out/g37/b.err; echo b rc $?
