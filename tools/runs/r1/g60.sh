mkdir -p gpurun_out/g60
timeout 300 python tools/host_trace.py > gpurun_out/g60/ht.log 2>&1; echo ht rc $?
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/g60/b$i.json 2>gpurun_out/g60/b$i.err; echo b$i rc $?; done
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g60/pytest.log 2>&1; echo pytest rc $?
