#!/bin/bash
# final code: cfg2 full-size separate parity, list tests, ncu captures of the TMA-staged kernels, bench line v6
mkdir -p gpurun_out/r2_g35
O=gpurun_out/r2_g35
timeout 900 python -m pytest tests/test_gpu_separate.py tests/test_gpu_lists.py -q -m gpu > $O/sep_lists.log 2>&1; echo "sep+lists rc=$?"; tail -3 $O/sep_lists.log; grep -E "^E  |^FAILED" $O/sep_lists.log | head -10 | cut -c1-250
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc $?
python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'],d['tree_ms'],d['factor_ms'],d['solve_ms'],d['roofline']['frac'],d['e2e']['value'],d.get('device_ms_steps'),d.get('device_lib_tree_factor_wait_solve_ms'), d['peak_mem_bytes'])"
for spec in "k_pchol_ll:10:6" "k_gj_panel:40:6"; do
  k=${spec%%:*}; rest=${spec#*:}; s=${rest%%:*}; c=${rest#*:}
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -o /tmp/full_$k python tools/cfg_warm.py cfg5 1 > $O/ncu_full_$k.log 2>&1; echo ncu $k rc $?
  python tools/ncu_summary.py full /tmp/full_$k.ncu-rep $k > $O/full_$k.json; head -c 700 $O/full_$k.json
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref rc $?; cut -c1-600 $O/bench_ref.json
