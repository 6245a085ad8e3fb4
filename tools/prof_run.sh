# Round-1 profiling pass on the GPU box: bench line, bench launch list, full captures of the top
# kernels summarised on the box (reports kept only for a few Schur launches: copy-back limit).
set -x
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err; echo bench rc $?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_launch.log 2>&1; echo ncu1 rc $?
python tools/ncu_summary.py launches gpurun_out/prof/launches_bench.csv > gpurun_out/prof/launches_bench.md
for k in k_gemm_schur k_gemm_store k_gj_panel k_pchol_cluster k_proxy k_build_level; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 40 -o /tmp/full_$k python tools/cfg_once.py cfg2 > gpurun_out/prof/ncu_full_$k.log 2>&1; echo ncu $k rc $?
  python tools/ncu_summary.py full /tmp/full_$k.ncu-rep $k > gpurun_out/prof/full_$k.json
done
ncu --set full --clock-control none --import-source on -k regex:k_gemm_schur -s 20 -c 3 -o gpurun_out/prof/schur_full python tools/cfg_once.py cfg2 > /dev/null 2>&1
ls -la gpurun_out/prof; du -sh gpurun_out
