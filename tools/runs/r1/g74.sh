# cfg5: 5 factorizations on fresh handles in one process (ENOMEM repro of g73), then the GPU tests
mkdir -p gpurun_out/g74
timeout 900 python tools/cfg_warm.py cfg5 5 > gpurun_out/g74/c5.json 2> gpurun_out/g74/c5.err; echo c5 rc $?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g74/pytest.log 2>&1; echo pytest rc $?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g74/bench.json 2> gpurun_out/g74/bench.err; echo bench rc $?
