mkdir -p gpurun_out/g11
for k in k_gj_panel_reg k_gj_reg k_pchol_reg; do
timeout 600 ncu --set full --import-source on -k regex:$k -s 10 -c 2 -o gpurun_out/g11/$k python tools/cfg_once.py cfg2 > gpurun_out/g11/$k.log 2>&1; echo $k rc $?
done
ls -la gpurun_out/g11
