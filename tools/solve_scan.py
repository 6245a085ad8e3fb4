"""Solve timing of one factorization at several nrhs (per-box kernels vs GEMM sweeps are chosen by
FMMLU_GEMM_SOLVE_MIN in the environment)."""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F
name = sys.argv[1]
nrhs_list = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 4, 16, 32]
c = fi.CONFIGS[name]; g = fi.config_geometry(name)
h = F.FmmLu(g.points, g.normals, g.weights, c["leaf_max"]).factor(c["k"], c["eps"])
out = {"config": name}
for q in nrhs_list:
    b = np.asfortranarray(fi.gaussian_rhs(g.n, q, 0))
    ts = []
    for rep in range(3):
        x = b.copy(order="F"); h.solve(x); ts.append(h.stats()["t_solve_ms"])
    out[q] = {"ms": min(ts), "ms_per_rhs": min(ts) / q}
print(json.dumps(out))
