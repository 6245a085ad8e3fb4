"""Diagnostics for the separate-ID path on the bump sphere: GPU vs dense solve for several parameter sets."""
import math
import sys

import numpy as np

sys.path.insert(0, ".")
import fmmlu_inputs as fi
from oracle import dense
from paper_2201_07325_b200 import fmmlu as F

g = fi.bump_sphere(n_base=3000, n_cap=1500, theta_c=0.05, height=0.02)
k, leaf, eps = 2.0, 24, 1e-6
b = fi.gaussian_rhs(g.n, 2, 0)
xd = dense.dense_solve(g.points, g.normals, g.weights, k, b)
for name, params in [("simul", {}), ("sep", {"separate_id": 1}), ("sep hh", {"separate_id": 1, "id_mode": 1}),
                     ("sep gjblocked", {"separate_id": 1, "gj_mode": 1}), ("simul hh", {"id_mode": 1}),
                     ("sep det", {"separate_id": 1, "deterministic": 1}),
                     ("sep eps1e-8", {"separate_id": 1, "eps": 1e-8}), ("simul eps1e-8", {"eps": 1e-8})]:
    h = F.FmmLu(g.points, g.normals, g.weights, leaf)
    e = params.pop("eps", eps)
    for pn, pv in params.items():
        h.set_param(pn, pv)
    h.factor(k, e)
    x = np.asfortranarray(b.copy())
    h.solve(x)
    st = h.stats()
    d = np.abs(x - xd).max(axis=1)
    print(f"{name:16s} eps {e:g} rel_diff_vs_dense {dense.rel_diff(x, xd):.3e} n0 {st['n0']} ranks {sum(st['ranks_sum'])} "
          f"err base-part {d[:3000].max():.2e} cap-part {d[3000:].max():.2e}", flush=True)
