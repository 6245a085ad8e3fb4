"""bench.py's sequence (device leg, then pinned-host e2e leg) with FMMLU_TRACE host sections per
factor, to locate occasional host stalls in the e2e leg."""
import gc, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F
c = fi.CONFIGS["cfg2"]; g = fi.config_geometry("cfg2")
dev = torch.device("cuda", 0)
b_host = np.asfortranarray(fi.gaussian_rhs(g.n, c["nrhs"], 0))
P = torch.from_numpy(g.points).to(dev); N = torch.from_numpy(g.normals).to(dev); W = torch.from_numpy(g.weights).to(dev)
B = torch.from_numpy(np.ascontiguousarray(b_host.T)).to(dev); X = torch.empty_like(B)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
stream = torch.cuda.Stream(dev); torch.cuda.set_stream(stream)
pts_p = torch.from_numpy(g.points).pin_memory(); nrm_p = torch.from_numpy(g.normals).pin_memory()
wts_p = torch.from_numpy(g.weights).pin_memory()
rhs_p = torch.from_numpy(np.ascontiguousarray(b_host.T)).pin_memory(); x_p = torch.empty_like(rhs_p).pin_memory()
h = None
for i in range(8):
    h = F.FmmLu(P, N, W, 64); h.set_stream(stream.cuda_stream); h.factor(c["k"], c["eps"]); X.copy_(B); h.solve(X, nrhs=4)
torch.cuda.synchronize(); gc.collect(); gc.disable()
h2 = None
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    if h2 is not None:
        h2.close()
    flush.zero_(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    h2 = F.FmmLu(pts_p, nrm_p, wts_p, 64); h2.set_stream(stream.cuda_stream)
    t1 = time.perf_counter()
    h2.factor(c["k"], c["eps"])
    t2 = time.perf_counter()
    x_p.copy_(rhs_p); h2.solve(x_p, nrhs=4)
    t3 = time.perf_counter()
    s = h2.stats()
    print(f"E2E {i} total {1e3*(t3-t0):.1f} tree {1e3*(t1-t0):.1f} factor {1e3*(t2-t1):.1f} wait {s['t_sync_wait_ms']:.1f} solve {1e3*(t3-t2):.1f}", file=sys.stderr, flush=True)
