# round-1 final measurement pass
mkdir -p gpurun_out/g29
timeout 900 python bench.py > gpurun_out/g29/bench.json 2> gpurun_out/g29/bench.err; echo bench rc $?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g29/bench_ref.json 2> gpurun_out/g29/bench_ref.err; echo ref rc $?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g29/smoke.log 2>&1; echo smoke rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g29/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g29/ncu_launch.log 2>&1; echo ncu1 rc $?
python tools/ncu_summary.py launches gpurun_out/g29/launches_bench.csv > gpurun_out/g29/launches_bench.md
FMMLU_TRACE=1 timeout 300 python tools/host_trace.py > gpurun_out/g29/host_trace.log 2>&1; echo ht rc $?
