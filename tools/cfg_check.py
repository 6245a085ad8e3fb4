"""Factor + solve a BASELINE config on the GPU; residual with the GPU brute-force matvec
(rows spot-checked against the oracle kernel)."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from oracle import kernel as okern
from paper_2201_07325_b200 import fmmlu as F
name = sys.argv[1]
c = fi.CONFIGS[name]; g = fi.config_geometry(name)
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else c["nrhs"]
b = np.asfortranarray(fi.gaussian_rhs(g.n, nrhs, 0))
t0 = time.time(); h = F.FmmLu(g.points, g.normals, g.weights, c["leaf_max"]); t1 = time.time()
print("tree s", t1 - t0, {k: v for k, v in h.stats().items() if k in ("nlevels", "nboxes", "nleaves")}, flush=True)
h.factor(c["k"], c["eps"]); t2 = time.time()
x = b.copy(order="F"); h.solve(x); t3 = time.time()
st = h.stats()
print(f"{name} n={g.n} factor {t2-t1:.3f}s solve {t3-t2:.3f}s n0={st['n0']} peak={st['peak_bytes']/1e9:.2f}GB "
      f"factor_bytes={st['factor_bytes']/1e9:.2f}GB", flush=True)
print("levels ms", [round(v, 1) for v in st["t_levels_ms"][:14]], "root", round(st["t_root_ms"], 1))
print("ranks", st["ranks_sum"][:14], "boxes", st["boxes"][:14])
print("classes", dict(zip(F.KERNEL_CLASSES, [round(v, 1) for v in st["class_ms"]])), flush=True)
t4 = time.time(); Ax = h.matvec(c["k"], x); t5 = time.time()
res = np.max(np.linalg.norm(Ax - b, axis=0) / np.linalg.norm(b, axis=0))
print(f"residual {res:.3e} (matvec {t5-t4:.1f}s)", flush=True)
rows = np.random.default_rng(1).choice(g.n, 8, replace=False)
err = 0
for i in rows:
    Ki = okern.combined_field(c["k"], g.points[i:i+1], g.points, g.normals)[0]; Ki[i] = 0
    yi = (Ki * g.weights) @ x + 0.5 * x[i]
    err = max(err, np.max(np.abs(yi - Ax[i])) / np.max(np.abs(yi)))
print("matvec row spot-check rel err", err)
