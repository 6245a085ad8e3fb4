#!/bin/bash
# final code (graph-replayed solves included): full GPU suite, smoke, bench line
mkdir -p gpurun_out/r2_g46
O=gpurun_out/r2_g46
timeout 3000 python -m pytest tests -q -m gpu > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log; grep -E "^FAILED|^ERROR" $O/tests.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc $?; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc $?
python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'],d['tree_ms'],d['factor_ms'],d['solve_ms'],d['solve_ms_nrhs1'],d['roofline']['frac'],d['e2e']['value'],d.get('device_ms_steps'), d['peak_mem_bytes'], d['gpu_launches'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 > $O/bench_torchrun.json 2> $O/bench_torchrun.err; echo torchrun rc $?; python -c "import json;d=json.load(open('$O/bench_torchrun.json'));print(d['value'], d['n_gpus'])"
