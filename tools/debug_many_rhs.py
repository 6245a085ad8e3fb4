"""Per-column comparison of the GEMM-sweep solve (nrhs >= 32) with the per-box kernels (4 columns at
a time) on one factorization."""
import math, sys
import numpy as np
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F
g = fi.ellipsoid(3000)
h = F.FmmLu(g.points, g.normals, g.weights, 32).factor(2 * math.pi, 1e-6)
b = fi.gaussian_rhs(g.n, 40, 11)
x = np.asfortranarray(b.copy()); h.solve(x)
xr = np.empty_like(x)
for c in range(0, 40, 4):
    t = np.asfortranarray(b[:, c:c + 4].copy()); h.solve(t); xr[:, c:c + 4] = t
d = np.linalg.norm(x - xr, axis=0) / np.linalg.norm(xr, axis=0)
print("per-column rel diff GEMM vs per-box:", np.array2string(d, precision=1))
for q in (31, 32, 33, 36):
    y = np.asfortranarray(b[:, :q].copy()); h.solve(y)
    dq = np.linalg.norm(y - xr[:, :q], axis=0) / np.linalg.norm(xr[:, :q], axis=0)
    print(q, "max", dq.max(), "argmax", dq.argmax())
