#!/bin/bash
# f3 on the GPU: separate-ID tests, the parity file (non-separate regression), bench line (no trace)
mkdir -p gpurun_out/r2_g23
timeout 1500 python -m pytest tests/test_gpu_separate.py -q -m gpu > gpurun_out/r2_g23/sep.log 2>&1; echo "sep rc=$?"; tail -40 gpurun_out/r2_g23/sep.log | cut -c1-300
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2_g23/parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r2_g23/parity.log
timeout 900 python bench.py > gpurun_out/r2_g23/bench.json 2> gpurun_out/r2_g23/bench.err; echo bench rc $?
python -c "import json;d=json.load(open('gpurun_out/r2_g23/bench.json'));print(d['value'],d['tree_ms'],d['factor_ms'],d['solve_ms'],d['roofline']['frac'],d['e2e']['value'],d.get('device_ms_steps'),d.get('device_lib_tree_factor_wait_solve_ms'))"
