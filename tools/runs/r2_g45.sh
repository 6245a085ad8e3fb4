#!/bin/bash
# graph-replayed small-RHS solves: tests + repeated-solve timing on cfg5 / cfg2
mkdir -p gpurun_out/r2_g45
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2_g45/parity.log 2>&1; echo "parity rc=$?"; tail -4 gpurun_out/r2_g45/parity.log; grep -E "^E  |^FAILED" gpurun_out/r2_g45/parity.log | head -10 | cut -c1-250
cat > /tmp/solve_rep.py <<'PY'
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F
for name in ("cfg2", "cfg5"):
    c = fi.CONFIGS[name]; g = fi.config_geometry(name)
    h = F.FmmLu(g.points, g.normals, g.weights, c["leaf_max"]).factor(c["k"], c["eps"])
    for nrhs in (1, 4):
        B = torch.from_numpy(np.asfortranarray(fi.gaussian_rhs(g.n, nrhs, 0))).cuda()
        ts = []
        for it in range(8):
            x = B.clone(); torch.cuda.synchronize(); t0 = time.perf_counter(); h.solve(x, nrhs); torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t0))
        print(name, "nrhs", nrhs, "solve ms per call:", [round(t, 2) for t in ts], flush=True)
    h.close()
PY
timeout 900 python /tmp/solve_rep.py 2>&1 | tail -6
FMMLU_SOLVE_GRAPH=0 timeout 900 python /tmp/solve_rep.py 2>&1 | tail -6
