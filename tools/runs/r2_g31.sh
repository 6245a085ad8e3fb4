#!/bin/bash
# device owner lists (a2): list parity tests, then the full GPU suite, smoke and bench
mkdir -p gpurun_out/r2_g31
timeout 1200 python -m pytest tests/test_gpu_lists.py -q -m gpu > gpurun_out/r2_g31/lists.log 2>&1; echo "lists rc=$?"; tail -5 gpurun_out/r2_g31/lists.log; grep -E "^E  |^FAILED" gpurun_out/r2_g31/lists.log | head -20 | cut -c1-250
timeout 3000 python -m pytest tests -q -m gpu --deselect tests/test_gpu_lists.py > gpurun_out/r2_g31/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_g31/tests.log; grep -E "^FAILED|^ERROR" gpurun_out/r2_g31/tests.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_g31/smoke.log 2>&1; echo smoke rc $?; tail -2 gpurun_out/r2_g31/smoke.log
FMMLU_TREE_TRACE=1 timeout 900 python bench.py > gpurun_out/r2_g31/bench.json 2> gpurun_out/r2_g31/bench.err; echo bench rc $?
python -c "import json;d=json.load(open('gpurun_out/r2_g31/bench.json'));print(d['value'],d['tree_ms'],d['factor_ms'],d['solve_ms'],d['roofline']['frac'],d['e2e']['value'],d.get('device_ms_steps'),d.get('device_lib_tree_factor_wait_solve_ms'), d['peak_mem_bytes'])"
FMMLU_TRACE=1 timeout 600 python tools/cfg_warm.py cfg5 2 > gpurun_out/r2_g31/cfg5t.json 2> gpurun_out/r2_g31/cfg5t.err; grep "host ms\|device timeline\|tree host" gpurun_out/r2_g31/cfg5t.err | tail -3 | cut -c1-900
