mkdir -p gpurun_out/g65
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g65/pytest.log 2>&1; echo pytest rc $?
timeout 1200 python tools/cfg_warm.py cfg5 > gpurun_out/g65/c5.json 2> gpurun_out/g65/c5.err; echo c5 rc $?
