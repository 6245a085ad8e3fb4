"""Time the bench's e2e step (pinned host buffers through the public API) piece by piece."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F
c = fi.CONFIGS["cfg2"]; g = fi.config_geometry("cfg2")
b_host = np.asfortranarray(fi.gaussian_rhs(g.n, 4, 0))
pts_p = torch.from_numpy(g.points).pin_memory(); nrm_p = torch.from_numpy(g.normals).pin_memory()
wts_p = torch.from_numpy(g.weights).pin_memory()
rhs_p = torch.from_numpy(np.ascontiguousarray(b_host.T)).pin_memory(); x_p = torch.empty_like(rhs_p).pin_memory()
stream = torch.cuda.Stream()
for rep in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = F.FmmLu(pts_p, nrm_p, wts_p, 64); h.set_stream(stream.cuda_stream); t1 = time.perf_counter()
    h.factor(c["k"], c["eps"]); t2 = time.perf_counter()
    x_p.copy_(rhs_p); h.solve(x_p, nrhs=4); t3 = time.perf_counter()
    s = h.stats()
    print(f"rep {rep}: tree {1e3*(t1-t0):6.1f} factor {1e3*(t2-t1):6.1f} (lib {s['t_factor_ms']:.1f}) solve {1e3*(t3-t2):6.1f} "
          f"(lib {s['t_solve_ms']:.1f}) total {1e3*(t3-t0):6.1f}", flush=True)
