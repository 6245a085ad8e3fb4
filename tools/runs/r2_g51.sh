#!/bin/bash
# GEMM sweeps from 16 RHS on large factor stores: solve scan + full GPU suite
mkdir -p gpurun_out/r2_g51
for c in cfg5 cfg3; do timeout 600 python tools/solve_scan.py $c 4,12,16,24,31,32 > gpurun_out/r2_g51/$c.json 2>/dev/null; echo "$c: $(cut -c1-700 gpurun_out/r2_g51/$c.json)"; done
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r2_g51/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_g51/tests.log | cut -c1-200
timeout 900 python bench.py > gpurun_out/r2_g51/bench.json 2> gpurun_out/r2_g51/bench.err; echo bench rc $?
python -c "import json;d=json.load(open('gpurun_out/r2_g51/bench.json'));print(d['value'],d['factor_ms'],d['solve_ms'],d['e2e']['value'],d.get('device_ms_steps'))"
