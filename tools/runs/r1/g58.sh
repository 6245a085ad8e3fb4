# final round-1 check on HEAD: GPU tests, smoke, bench (driver defaults), reference arm
mkdir -p gpurun_out/g58
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g58/pytest.log 2>&1; echo pytest rc $?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g58/smoke.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/g58/bench.json 2> gpurun_out/g58/bench.err; echo bench rc $?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g58/bench_ref.json 2> gpurun_out/g58/bench_ref.err; echo ref rc $?
