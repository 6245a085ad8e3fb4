"""One factor+solve of a BASELINE config through the C ABI (for ncu launch lists)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
c = fi.CONFIGS[name]; g = fi.config_geometry(name)
b = np.asfortranarray(fi.gaussian_rhs(g.n, c["nrhs"], 0))
h = F.FmmLu(g.points, g.normals, g.weights, c["leaf_max"]).factor(c["k"], c["eps"])
x = b.copy(order="F"); h.solve(x)
print(h.stats()["t_factor_ms"], h.stats()["t_solve_ms"])
