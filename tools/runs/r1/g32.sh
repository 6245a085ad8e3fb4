mkdir -p gpurun_out/g32
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g32/pytest.log 2>&1; echo pytest rc $?
timeout 600 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/g32/b.json 2>gpurun_out/g32/b.err; echo b rc $?
timeout 900 python tools/cfg_check.py cfg5 > gpurun_out/g32/cfg5.log 2>&1; echo cfg5 rc $?
