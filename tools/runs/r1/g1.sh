mkdir -p gpurun_out/g1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g1/pytest.log 2>&1; echo pytest rc $?
timeout 600 python bench.py > gpurun_out/g1/bench.json 2> gpurun_out/g1/bench.err; echo bench rc $?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1/smoke.log 2>&1; echo smoke rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g1/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g1/ncu_launch.log 2>&1; echo ncu rc $?
python tools/ncu_summary.py launches gpurun_out/g1/launches_bench.csv > gpurun_out/g1/launches_bench.md
