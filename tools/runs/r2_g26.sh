#!/bin/bash
# union-skeleton separate IDs, left-looking pivoted Cholesky (batches >= 128), blocked GJ for batches >= 200, level-store compaction:
# sep diagnostics + full GPU suite + warm timings + bench
mkdir -p gpurun_out/r2_g26
timeout 600 python tools/sep_diag.py > gpurun_out/r2_g26/sep_diag.txt 2>&1; cat gpurun_out/r2_g26/sep_diag.txt | cut -c1-250
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/r2_g26/tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2_g26/tests.log; grep -E "^FAILED|^ERROR" gpurun_out/r2_g26/tests.log | head -20
for c in cfg5 cfg2 cfg3; do
  timeout 600 python tools/cfg_warm.py $c 4 > gpurun_out/r2_g26/$c.json 2> gpurun_out/r2_g26/$c.err; echo $c rc $?; cut -c1-1300 gpurun_out/r2_g26/$c.json
done
timeout 600 python tools/cfg_warm.py cfg5 2 separate > gpurun_out/r2_g26/sep5.json 2> gpurun_out/r2_g26/sep5.err; echo sep5 rc $?; cut -c1-1300 gpurun_out/r2_g26/sep5.json; tail -2 gpurun_out/r2_g26/sep5.err
timeout 900 python bench.py > gpurun_out/r2_g26/bench.json 2> gpurun_out/r2_g26/bench.err; echo bench rc $?
python -c "import json;d=json.load(open('gpurun_out/r2_g26/bench.json'));print(d['value'],d['tree_ms'],d['factor_ms'],d['solve_ms'],d['roofline']['frac'],d['e2e']['value'],d.get('device_ms_steps'),d.get('device_lib_tree_factor_wait_solve_ms'), d['peak_mem_bytes'])"
