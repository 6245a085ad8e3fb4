"""Factor (+ solve) a BASELINE config several times in one process with fresh handles and print one
JSON object: per-run tree / factor / solve wall ms, the library's wait split, class ms of the last run,
device memory before and after.  usage: python tools/cfg_warm.py cfg5 4 [separate] [name=value ...]  (fmmlu_set_param overrides)"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
sep = "separate" in sys.argv[3:]
params = {a.split("=")[0]: float(a.split("=")[1]) for a in sys.argv[3:] if "=" in a}
c = fi.CONFIGS[name]
g = fi.config_geometry(name)
pts = torch.from_numpy(g.points).cuda()
nrm = torch.from_numpy(g.normals).cuda()
wts = torch.from_numpy(g.weights).cuda()
b = torch.from_numpy(np.asfortranarray(fi.gaussian_rhs(g.n, c["nrhs"], 0))).cuda()
free0, total = torch.cuda.mem_get_info()
runs = []
h = None
for rep in range(reps):
    if h is not None:
        h.close()
    x = b.clone()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = F.FmmLu(pts, nrm, wts, c["leaf_max"])
    if sep:
        h.set_param("separate_id", 1)
    for pn, pv in params.items():
        h.set_param(pn, pv)
    t1 = time.perf_counter()
    h.factor(c["k"], c["eps"])
    t2 = time.perf_counter()
    h.solve(x, c["nrhs"])
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    s = h.stats()
    runs.append(dict(tree_ms=round(1e3 * (t1 - t0), 1), factor_ms=round(1e3 * (t2 - t1), 1),
                     solve_ms=round(1e3 * (t3 - t2), 1), wait_ms=round(s["t_sync_wait_ms"], 1),
                     n0=int(s["n0"]), free_gb=round(torch.cuda.mem_get_info()[0] / 1e9, 1)))
    print(runs[-1], file=sys.stderr, flush=True)
s = h.stats()
out = dict(config=name, separate=sep, params=params, n=int(g.n), runs=runs, total_gb=round(total / 1e9, 1), free0_gb=round(free0 / 1e9, 1),
           class_ms=dict(zip(F.KERNEL_CLASSES, [round(v, 2) for v in s["class_ms"]])),
           factor_bytes=int(s["factor_bytes"]), peak_bytes=int(s["peak_bytes"]),
           ranks_sum=int(sum(s["ranks_sum"])))
print(json.dumps(out))
