"""Quick GPU diagnostics: probes, matvec parity, small factor/solve parity vs oracle, cfg2 timing."""
import math, sys, time, json
import numpy as np
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from oracle import dense, rss, kernel as okern
from paper_2201_07325_b200 import fmmlu as F

print("dfma TF", F.probe_fp64(0), "dmma TF", F.probe_fp64(1), flush=True)
g = fi.ellipsoid(1500); k = 2*math.pi
x = np.asfortranarray(fi.gaussian_rhs(g.n, 2, 5))
h = F.FmmLu(g.points, g.normals, g.weights, 64)
y = h.matvec(k, x); yo = okern.matvec_unscaled(k, g.points, g.normals, g.weights, x)
print("matvec rel err", np.max(np.abs(y-yo))/np.max(np.abs(yo)), flush=True)
for name, g, k, leaf in [("sphere60", fi.fibonacci_sphere(60), 1.0, 64), ("cfg1", fi.config_geometry("cfg1"), 1.0, 64),
                         ("ell3000", fi.ellipsoid(3000), 2*math.pi, 32)]:
    b = fi.gaussian_rhs(g.n, 2, 0)
    t = time.time()
    h = F.FmmLu(g.points, g.normals, g.weights, leaf).factor(k, 1e-6)
    xg = np.asfortranarray(b.copy()); h.solve(xg)
    tg = time.time()-t
    f = rss.factor(g.points, g.normals, g.weights, k, 1e-6, leaf); xo = rss.solve(f, b)
    st = h.stats()
    print(name, "gpu s", round(tg,3), "n0 gpu/or", st["n0"], f.stats["n0"], "reldiff", dense.rel_diff(xg, xo),
          "resid", dense.residual(g.points, g.normals, g.weights, k, xg, b), flush=True)
    print("  ranks gpu", st["ranks_sum"][:8], "boxes", st["boxes"][:8],
          " oracle", {l: (int(s["ranks"].sum()), len(s["ranks"])) for l, s in f.stats["levels"].items()}, flush=True)
c = fi.CONFIGS["cfg2"]; g = fi.config_geometry("cfg2")
b = np.asfortranarray(fi.gaussian_rhs(g.n, 4, 0))
for rep in range(3):
    t = time.time(); h = F.FmmLu(g.points, g.normals, g.weights, 64); t1 = time.time()
    h.factor(c["k"], c["eps"]); t2 = time.time()
    xg = b.copy(order="F"); h.solve(xg); t3 = time.time()
    st = h.stats()
    print("cfg2 tree %.1f ms factor %.1f ms solve %.1f ms" % ((t1-t)*1e3, (t2-t1)*1e3, (t3-t2)*1e3),
          "n0", st["n0"], "levels ms", [round(v,1) for v in st["t_levels_ms"][:6]], "root ms", round(st["t_root_ms"],1), flush=True)
Ax = h.matvec(c["k"], xg)
print("cfg2 resid", np.max(np.linalg.norm(Ax-b,axis=0)/np.linalg.norm(b,axis=0)), "stats", json.dumps({k_: v for k_, v in st.items() if not isinstance(v, list)}))
