mkdir -p gpurun_out/g41
timeout 900 python bench.py > gpurun_out/g41/bench.json 2> gpurun_out/g41/bench.err; echo bench rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g41/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g41/ncu_launch.log 2>&1; echo ncu1 rc $?
python tools/ncu_summary.py launches gpurun_out/g41/launches_bench.csv > gpurun_out/g41/launches_bench.md
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g41/smoke.log 2>&1; echo smoke rc $?
