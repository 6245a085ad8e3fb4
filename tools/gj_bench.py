"""Batched X_RR⁻¹ microbenchmark: fmmlu_inverse_batch for both gj_modes over n and batch size;
accuracy checked against numpy.linalg.inv (CPU) on the first matrix."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import fmmlu_inputs as fi
from paper_2201_07325_b200 import fmmlu as F

g = fi.fibonacci_sphere(64)
h = F.FmmLu(g.points, g.normals, g.weights, 64)
rng = np.random.default_rng(0)
sizes = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [32, 64, 116, 128, 160, 205, 256, 263, 320, 384, 500]
counts = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 32]
for n in sizes:
    for count in counts:
        M = 0.5 * np.eye(n)[None] + (rng.standard_normal((count, n, n)) + 1j * rng.standard_normal((count, n, n))) / np.sqrt(8 * n)
        ref = np.linalg.inv(M[0])
        out = []
        for mode in (0, 1):
            h.set_param("gj_mode", mode)
            # column-major storage: pass the transposes (C order of Mᵀ = column-major M)
            A = torch.from_numpy(np.ascontiguousarray(M.transpose(0, 2, 1))).cuda()
            h.inverse_batch(A, n, count)  # warm-up
            ts = []
            for _ in range(3):
                A = torch.from_numpy(np.ascontiguousarray(M.transpose(0, 2, 1))).cuda()
                ts.append(h.inverse_batch(A, n, count))
            X = A.cpu().numpy()[0].T
            err = np.abs(X - ref).max() / np.abs(ref).max()
            out.append(f"mode{mode} {min(ts)*1e3:8.1f} us ({min(ts)*1e3/n:5.2f} us/step) err {err:.1e}")
        print(f"n {n:4d} count {count:3d}: " + " | ".join(out), flush=True)
