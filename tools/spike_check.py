"""Repeated cfg2 tree+factor on one stream; times handle creation, factor, destroy separately
(spike hunting; FMMLU_TRACE=1 adds the library's host/allocator breakdown)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F
c = fi.CONFIGS["cfg2"]; g = fi.config_geometry("cfg2")
dev = torch.device("cuda", 0)
P = torch.from_numpy(g.points).to(dev); N = torch.from_numpy(g.normals).to(dev); W = torch.from_numpy(g.weights).to(dev)
stream = torch.cuda.Stream(dev)
h = None
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if h is not None:
        h.close()
    t1 = time.perf_counter()
    h = F.FmmLu(P, N, W, 64); h.set_stream(stream.cuda_stream)
    t2 = time.perf_counter()
    h.factor(c["k"], c["eps"])
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    s = h.stats()
    print(f"rep {rep} destroy {1e3*(t1-t0):6.1f} tree {1e3*(t2-t1):6.1f} (lib {s['t_tree_ms']:.1f}) factor {1e3*(t3-t2):6.1f} "
          f"sync {1e3*(t4-t3):6.1f} wait {s['t_sync_wait_ms']:.1f}", file=sys.stderr, flush=True)
