# round-1 closing measurement pass: launch list of the final bench + full captures of the top kernels
mkdir -p gpurun_out/g71
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g71/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g71/ncu_launch.log 2>&1; echo ncu1 rc $?
python tools/ncu_summary.py launches gpurun_out/g71/launches_bench.csv > gpurun_out/g71/launches_bench.md
gzip -k gpurun_out/g71/launches_bench.csv
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_gemm_schur -c 3 -o /tmp/full_schur python tools/cfg_once.py cfg2 > gpurun_out/g71/ncu_full_schur.log 2>&1; echo ncu2 rc $?
python tools/ncu_summary.py full /tmp/full_schur.ncu-rep k_gemm_schur > gpurun_out/g71/full_k_gemm_schur.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_gemm_store -c 3 -o /tmp/full_store python tools/cfg_once.py cfg2 > gpurun_out/g71/ncu_full_store.log 2>&1; echo ncu3 rc $?
python tools/ncu_summary.py full /tmp/full_store.ncu-rep k_gemm_store > gpurun_out/g71/full_k_gemm_store.json
