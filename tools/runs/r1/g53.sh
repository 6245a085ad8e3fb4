mkdir -p gpurun_out/g53
FMMLU_TRACE=1 timeout 1200 python tools/cfg_warm.py cfg5 > gpurun_out/g53/c5.json 2> gpurun_out/g53/c5.err; echo c5 rc $?
timeout 600 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/g53/b.json 2>gpurun_out/g53/b.err; echo b rc $?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g53/pytest.log 2>&1; echo pytest rc $?
