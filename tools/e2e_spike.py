"""Repeated bench e2e steps (pinned host buffers through the public API); per-step wall time split
into tree / factor / solve as the library reports them (spike hunting)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F
c = fi.CONFIGS["cfg2"]; g = fi.config_geometry("cfg2")
b_host = np.asfortranarray(fi.gaussian_rhs(g.n, c["nrhs"], 0))
stream = torch.cuda.Stream(torch.device("cuda", 0))
torch.cuda.set_stream(stream)
pts_p = torch.from_numpy(g.points).pin_memory(); nrm_p = torch.from_numpy(g.normals).pin_memory()
wts_p = torch.from_numpy(g.weights).pin_memory()
rhs_p = torch.from_numpy(np.ascontiguousarray(b_host.T)).pin_memory(); x_p = torch.empty_like(rhs_p).pin_memory()
import subprocess, os
smi = None
h = None
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    if os.environ.get("SMI") and rep == 5:
        smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "200"],
                               stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    if smi is not None and rep == 12:
        smi.terminate(); smi.wait(2); smi = None
        print("smi terminated", flush=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = None
    t1 = time.perf_counter()
    h = F.FmmLu(pts_p, nrm_p, wts_p, c["leaf_max"]); h.set_stream(stream.cuda_stream)
    t2 = time.perf_counter()
    h.factor(c["k"], c["eps"])
    t3 = time.perf_counter()
    x_p.copy_(rhs_p); h.solve(x_p, nrhs=c["nrhs"])
    t4 = time.perf_counter()
    s = h.stats()
    print(f"rep {rep} total {1e3*(t4-t0):6.1f} destroy {1e3*(t1-t0):5.1f} tree {1e3*(t2-t1):6.1f} (lib {s['t_tree_ms']:.1f}) "
          f"factor {1e3*(t3-t2):6.1f} (wait {s['t_sync_wait_ms']:.1f}) solve {1e3*(t4-t3):6.1f} (lib {s['t_solve_ms']:.1f})",
          flush=True)
