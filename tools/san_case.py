"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck): tree +
factor + solve (per-box kernels and GEMM sweeps) + forward apply + deterministic factorization
on an ellipsoid, and a small cfg4-style box batch (Gram and Householder ID paths)."""
import math
import sys

import numpy as np

sys.path.insert(0, ".")
import fmmlu_inputs as fi  # noqa: E402
from paper_2201_07325_b200 import fmmlu as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2500
g = fi.ellipsoid(n)
k = 2 * math.pi
for det in (0, 1):
    h = F.FmmLu(g.points, g.normals, g.weights, 32).set_param("deterministic", det).factor(k, 1e-6)
    for nrhs in (2, 33):
        x = np.asfortranarray(fi.gaussian_rhs(g.n, nrhs, 1))
        h.solve(x)
    h.apply(np.asfortranarray(fi.gaussian_rhs(g.n, 2, 2)))
    print("det", det, h.stats()["n0"], flush=True)
    h.close()
d = fi.box_batch(8, b=64, n_near=128)
rho = 1.5 * math.sqrt(3) / 2 * d["h"]
for eps in (1e-6, 1e-9):
    out = F.boxes(d["pts"], d["nrm"], d["npts"], d["nnrm"], d["w"], 10.0, eps, 128, rho, keep=[0])
    print("boxes", eps, out["ranks"].tolist(), flush=True)
print("done")
