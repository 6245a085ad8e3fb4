"""Warm factor + solve timing of a BASELINE config: the second factorization on a fresh handle
(the first pays allocation / pool growth), solve with the config's nrhs, per-class device times."""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F
name = sys.argv[1]
c = fi.CONFIGS[name]; g = fi.config_geometry(name)
b = np.asfortranarray(fi.gaussian_rhs(g.n, c["nrhs"], 0))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2  # rep 1 is reported; all reps' factor times are listed
out = {"config": name, "n": g.n, "factor_ms_reps": []}
for rep in range(reps):
    h = F.FmmLu(g.points, g.normals, g.weights, c["leaf_max"])
    h.factor(c["k"], c["eps"])
    x = b.copy(order="F"); h.solve(x)
    st = h.stats()
    out["factor_ms_reps"].append(round(st["t_factor_ms"], 1))
    if rep == 1:
        out.update(tree_ms=st["t_tree_ms"], factor_ms=st["t_factor_ms"], solve_ms=st["t_solve_ms"], nrhs=c["nrhs"],
                   factor_unknowns_per_s=g.n / (st["t_factor_ms"] * 1e-3), n0=st["n0"],
                   factor_GB=st["factor_bytes"] / 1e9, peak_GB=st["peak_bytes"] / 1e9,
                   classes_ms={k: round(v, 1) for k, v in zip(F.KERNEL_CLASSES, st["class_ms"])})
    h.close()
print(json.dumps(out))
