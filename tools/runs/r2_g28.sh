#!/bin/bash
# full GPU suite, smoke, bench (tree breakdown printed), cfg5 trace of one factorization per level
mkdir -p gpurun_out/r2_g28
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/r2_g28/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_g28/tests.log; grep -E "^FAILED|^ERROR" gpurun_out/r2_g28/tests.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_g28/smoke.log 2>&1; echo smoke rc $?; tail -2 gpurun_out/r2_g28/smoke.log
FMMLU_TREE_TRACE=1 timeout 900 python bench.py > gpurun_out/r2_g28/bench.json 2> gpurun_out/r2_g28/bench.err; echo bench rc $?
grep "tree host" gpurun_out/r2_g28/bench.err | cut -c1-300
python -c "import json;d=json.load(open('gpurun_out/r2_g28/bench.json'));print(d['value'],d['tree_ms'],d['factor_ms'],d['solve_ms'],d['roofline']['frac'],d['e2e']['value'],d.get('device_ms_steps'),d.get('device_lib_tree_factor_wait_solve_ms'), d['peak_mem_bytes'])"
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 2 > gpurun_out/r2_g28/cfg5t.json 2> gpurun_out/r2_g28/cfg5t.err
