#!/bin/bash
# final code: full GPU suite, smoke, bench line, launch list of one cfg5 step
mkdir -p gpurun_out/r2_g43
O=gpurun_out/r2_g43
timeout 3000 python -m pytest tests -q -m gpu > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log; grep -E "^FAILED|^ERROR" $O/tests.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc $?; tail -2 $O/smoke.log
for i in 1 2; do
timeout 900 python bench.py > $O/bench$i.json 2> $O/bench$i.err; echo bench rc $?
python -c "import json;d=json.load(open('$O/bench$i.json'));print(d['value'],d['tree_ms'],d['factor_ms'],d['solve_ms'],d['roofline']['frac'],d['e2e']['value'],d.get('device_ms_steps'),d.get('device_lib_tree_factor_wait_solve_ms'), d['peak_mem_bytes'], d['gpu_launches'])"
done
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv python tools/cfg_warm.py cfg5 1 > $O/ncu_launch.log 2>&1; echo ncu-launches rc $?
python tools/ncu_summary.py launches $O/launches_cfg5.csv > $O/launches_cfg5.md; head -14 $O/launches_cfg5.md
gzip -f $O/launches_cfg5.csv
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 2 > /dev/null 2> $O/cfg5t.err; grep "host ms:\|device timeline" $O/cfg5t.err | tail -2 > $O/timeline.txt; cat $O/timeline.txt | cut -c1-700
