#!/bin/bash
# final code: full GPU suite, smoke, bench line (twice)
mkdir -p gpurun_out/r2_g39
O=gpurun_out/r2_g39
timeout 3000 python -m pytest tests -q -m gpu > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log; grep -E "^FAILED|^ERROR" $O/tests.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc $?; tail -2 $O/smoke.log
for i in 1 2; do
timeout 900 python bench.py > $O/bench$i.json 2> $O/bench$i.err; echo bench rc $?
python -c "import json;d=json.load(open('$O/bench$i.json'));print(d['value'],d['tree_ms'],d['factor_ms'],d['solve_ms'],d['roofline']['frac'],d['e2e']['value'],d.get('device_ms_steps'),d.get('device_lib_tree_factor_wait_solve_ms'), d['peak_mem_bytes'], d['gpu_launches'])"
done
