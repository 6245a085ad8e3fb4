"""Alternate the bench's device-resident step and the host-buffer step to separate noise from a
systematic difference."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F
c = fi.CONFIGS["cfg2"]; g = fi.config_geometry("cfg2")
dev = torch.device("cuda", 0)
P = torch.from_numpy(g.points).to(dev); N = torch.from_numpy(g.normals).to(dev); W = torch.from_numpy(g.weights).to(dev)
b = np.asfortranarray(fi.gaussian_rhs(g.n, 4, 0))
B = torch.from_numpy(np.ascontiguousarray(b.T)).to(dev); X = torch.empty_like(B)
stream = torch.cuda.Stream(dev)
def dev_step(use_stream):
    h = F.FmmLu(P, N, W, 64)
    if use_stream: h.set_stream(stream.cuda_stream)
    h.factor(c["k"], c["eps"]); X.copy_(B); h.solve(X, nrhs=4); return h
def host_step():
    h = F.FmmLu(g.points.copy(), g.normals.copy(), g.weights.copy(), 64); h.factor(c["k"], c["eps"])
    x = b.copy(order="F"); h.solve(x); return h
for rep in range(4):
    for name, fn in (("dev+torchstream", lambda: dev_step(True)), ("dev+ownstream", lambda: dev_step(False)), ("host", host_step)):
        torch.cuda.synchronize(); t = time.perf_counter(); h = fn(); torch.cuda.synchronize()
        s = h.stats()
        print(f"{name:16s} {1e3*(time.perf_counter()-t):7.1f} ms  tree {s['t_tree_ms']:.1f} factor {s['t_factor_ms']:.1f} wait {s['t_sync_wait_ms']:.1f} solve {s['t_solve_ms']:.1f}", flush=True)
