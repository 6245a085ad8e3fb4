"""Factor cfg2 a few times and report host vs device-wait split and per-level times."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F
c = fi.CONFIGS["cfg2"]; g = fi.config_geometry("cfg2")
for rep in range(3):
    t0 = time.perf_counter()
    h = F.FmmLu(g.points, g.normals, g.weights, 64)
    t1 = time.perf_counter()
    h.factor(c["k"], c["eps"])
    t2 = time.perf_counter()
    s = h.stats()
    cls = dict(zip(F.KERNEL_CLASSES, [round(x, 2) for x in s["class_ms"]]))
    print(f"tree {1e3*(t1-t0):.1f} factor {1e3*(t2-t1):.1f} wait {s['t_sync_wait_ms']:.1f} "
          f"host {1e3*(t2-t1)-s['t_sync_wait_ms']:.1f} levels {[round(v,1) for v in s['t_levels_ms'][:6]]} "
          f"root {s['t_root_ms']:.1f} gpu-classes-sum {sum(s['class_ms']):.1f}", cls, flush=True)
