# round-1 final measurement pass (v9)
mkdir -p gpurun_out/g35
timeout 900 python bench.py > gpurun_out/g35/bench.json 2> gpurun_out/g35/bench.err; echo bench rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g35/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g35/ncu_launch.log 2>&1; echo ncu1 rc $?
python tools/ncu_summary.py launches gpurun_out/g35/launches_bench.csv > gpurun_out/g35/launches_bench.md
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_gemm_schur -o /tmp/full_schur python tools/cfg_once.py cfg2 > gpurun_out/g35/ncu_full_schur.log 2>&1; echo ncu2 rc $?
python tools/ncu_summary.py full /tmp/full_schur.ncu-rep k_gemm_schur > gpurun_out/g35/full_k_gemm_schur.json
FMMLU_TRACE=1 timeout 300 python tools/host_trace.py > gpurun_out/g35/host_trace.log 2>&1; echo ht rc $?
timeout 900 python tools/rcs_bench.py cfg2 1000 > gpurun_out/g35/rcs_cfg2.json 2> gpurun_out/g35/rcs_cfg2.err; echo rcs rc $?
