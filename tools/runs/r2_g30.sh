#!/bin/bash
# round-2 final profiling pass: launch list of one cfg5 tree+factor+solve, full captures of the new kernels and the Schur GEMM
mkdir -p gpurun_out/r2_g30
O=gpurun_out/r2_g30
timeout 900 python tools/cfg_warm.py cfg5 1 > $O/plain.json 2> $O/plain.err; echo plain rc $?
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv python tools/cfg_warm.py cfg5 1 > $O/ncu_launch.log 2>&1; echo ncu-launches rc $?
python tools/ncu_summary.py launches $O/launches_cfg5.csv > $O/launches_cfg5.md; head -40 $O/launches_cfg5.md
gzip -f $O/launches_cfg5.csv
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 1 > /dev/null 2> $O/trace.err; grep "schur launch" $O/trace.err > $O/schur_launch_work.txt
for spec in "k_pchol_ll:10:6" "k_compact_level:0:4" "k_gj_panel:40:6" "k_gemm_schur:8:8"; do
  k=${spec%%:*}; rest=${spec#*:}; s=${rest%%:*}; c=${rest#*:}
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -o /tmp/full_$k python tools/cfg_warm.py cfg5 1 > $O/ncu_full_$k.log 2>&1; echo ncu $k rc $?
  python tools/ncu_summary.py full /tmp/full_$k.ncu-rep $k > $O/full_$k.json; head -c 900 $O/full_$k.json
done
python tools/pair_traffic.py $O/full_k_gemm_schur.json $O/schur_launch_work.txt 8 $O/schur_traffic_cfg5.json
ls -la $O
