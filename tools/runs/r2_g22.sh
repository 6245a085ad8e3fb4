#!/bin/bash
# session-3 re-entry check of HEAD: full GPU suite, smoke, bench line
mkdir -p gpurun_out/r2_g22
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_g22/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_g22/tests.log; grep -E "^FAILED" gpurun_out/r2_g22/tests.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_g22/smoke.log 2>&1; echo smoke rc $?; tail -2 gpurun_out/r2_g22/smoke.log
FMMLU_TRACE=0 timeout 900 python bench.py > gpurun_out/r2_g22/bench.json 2> gpurun_out/r2_g22/bench.err; echo bench rc $?
python -c "import json;d=json.load(open('gpurun_out/r2_g22/bench.json'));print(d['value'],d['factor_ms'],d['solve_ms'],d['roofline']['frac'],d['e2e']['value'],d.get('device_ms_steps'))"
