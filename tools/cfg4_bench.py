"""cfg4 timing: fmmlu_boxes on BASELINE configs[3] (8192 boxes) at the given ε."""
import math, sys, time
import numpy as np
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F
nbox = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
epss = [float(e) for e in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1e-4, 1e-6, 1e-9]
t = time.perf_counter()
d = fi.box_batch(nbox)
print(f"inputs {time.perf_counter()-t:.1f} s", flush=True)
rho = 1.5 * math.sqrt(3) / 2 * d["h"]
for eps in epss:
    F.boxes(d["pts"], d["nrm"], d["npts"], d["nnrm"], d["w"], 10.0, eps, 512, rho, want_perm=False)  # warm-up
    out = F.boxes(d["pts"], d["nrm"], d["npts"], d["nnrm"], d["w"], 10.0, eps, 512, rho, want_perm=False)
    r = out["ranks"]
    print(f"eps {eps:g}: {out['ms']:.1f} ms  {nbox/(out['ms']*1e-3):.0f} boxes/s  model {out['gflop']:.0f} GFLOP "
          f"-> {out['gflop']/(out['ms']*1e-3)/1e3:.2f} TFLOP/s  ranks mean {r.mean():.1f} min {r.min()} max {r.max()} wave {out['wave']}", flush=True)
