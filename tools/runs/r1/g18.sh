# round-1 profile refresh: bench line, launch list of the bench, full capture of the Schur GEMM over one cfg2 factor
mkdir -p gpurun_out/g18
timeout 900 python bench.py > gpurun_out/g18/bench.json 2> gpurun_out/g18/bench.err; echo bench rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g18/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g18/ncu_launch.log 2>&1; echo ncu1 rc $?
python tools/ncu_summary.py launches gpurun_out/g18/launches_bench.csv > gpurun_out/g18/launches_bench.md
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_gemm_schur -o /tmp/full_schur python tools/cfg_once.py cfg2 > gpurun_out/g18/ncu_full_schur.log 2>&1; echo ncu2 rc $?
python tools/ncu_summary.py full /tmp/full_schur.ncu-rep k_gemm_schur > gpurun_out/g18/full_k_gemm_schur.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_gemm_schur -s 20 -c 1 -o gpurun_out/g18/schur_one python tools/cfg_once.py cfg2 > /dev/null 2>&1; echo ncu3 rc $?
for k in k_gj_reg k_pchol_reg k_gj_panel_reg k_su_b; do
timeout 900 ncu --set full --clock-control none -k regex:$k -c 12 -o /tmp/full_$k python tools/cfg_once.py cfg2 > /dev/null 2>&1; echo ncu $k rc $?
python tools/ncu_summary.py full /tmp/full_$k.ncu-rep $k > gpurun_out/g18/full_$k.json
done
ls -la gpurun_out/g18
