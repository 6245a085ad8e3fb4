# final ncu --set full summaries of the pivot-step and solve kernels (one cfg2 factor + solve)
mkdir -p gpurun_out/g59
for k in k_gj_reg k_pchol_reg k_gj_panel_reg k_su_b k_gemm_store; do
timeout 900 ncu --set full --clock-control none -k regex:$k -c 12 -o /tmp/full_$k python tools/cfg_once.py cfg2 > /dev/null 2>&1; echo ncu $k rc $?
python tools/ncu_summary.py full /tmp/full_$k.ncu-rep $k > gpurun_out/g59/full_$k.json
done
