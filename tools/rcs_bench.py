"""f2 workload: azimuthal monostatic cross section over many angles on a BASELINE
geometry.  Factor once, then time fmmlu_monostatic_rcs (device plane-wave RHS + GEMM sweeps +
backscatter reduction) with CUDA-synchronous host timing; report ms per angle and the sweep GEMMs'
achieved FP64 rate from the library's class counters.  Also times fmmlu_solve at nrhs = 4 and 1000
Gaussian RHS for the per-RHS comparison of the two solve paths."""
import json, math, sys, time
import numpy as np
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
nphi = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
c = fi.CONFIGS[name]; g = fi.config_geometry(name)
h = F.FmmLu(g.points, g.normals, g.weights, c["leaf_max"]).factor(c["k"], c["eps"])
phis = np.linspace(0.0, 2 * math.pi, nphi, endpoint=False)
out = {"config": name, "n": g.n, "k": c["k"], "nphi": nphi}
h.monostatic_rcs(phis[:64])  # warm-up (workspace, first GEMM launches)
ts = []
for _ in range(3):
    t0 = time.perf_counter(); R = h.monostatic_rcs(phis); ts.append(time.perf_counter() - t0)
st = h.stats()
ci = F.KERNEL_CLASSES.index("solve")
out["rcs_ms"] = min(ts) * 1e3
out["rcs_ms_per_angle"] = min(ts) * 1e3 / nphi
out["sweep_gemm_tflops_last_call"] = st["class_flops"][ci] / max(st["class_ms"][ci], 1e-9) / 1e9
out["R_first"] = [complex(R[0]).real, complex(R[0]).imag]
for nr in (4, 1000):
    b = np.asfortranarray(fi.gaussian_rhs(g.n, nr, 0))
    x = b.copy(order="F"); h.solve(x)
    ts = []
    for _ in range(3):
        x = b.copy(order="F"); t0 = time.perf_counter(); h.solve(x); ts.append(time.perf_counter() - t0)
    out[f"solve_ms_per_rhs_nrhs{nr}"] = min(ts) * 1e3 / nr
print(json.dumps(out))
