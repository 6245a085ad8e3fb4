mkdir -p gpurun_out/g63
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g63/pytest.log 2>&1; echo pytest rc $?
timeout 300 python tools/host_trace.py > gpurun_out/g63/ht.log 2>&1; echo ht rc $?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g63/b.json 2>gpurun_out/g63/b.err; echo b rc $?
timeout 900 python tools/cfg4_bench.py 8192 1e-4,1e-6 > gpurun_out/g63/cfg4.log 2>&1; echo cfg4 rc $?
