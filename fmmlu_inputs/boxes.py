"""Config 4 inputs: independent synthetic boxes for the batched ID + elimination
microbenchmark (SURVEY.md reading C21).

Box side h = 1/8.  Per box (seed 1000 + box id): b points uniform in
[-h/2,h/2]³, n_near points uniform in the shell [-3h/2,3h/2]³ minus the inner
cube (rejection sampling), random unit normals, w = h²/b (uniform).
"""
from __future__ import annotations

import numpy as np


def box_batch(nbox: int, b: int = 256, n_near: int = 1024, h: float = 0.125, first_id: int = 0):
    """Return dict of arrays: pts (nbox,b,3), nrm (nbox,b,3), npts (nbox,n_near,3),
    nnrm (nbox,n_near,3), w scalar, h."""
    pts = np.empty((nbox, b, 3))
    nrm = np.empty((nbox, b, 3))
    npts = np.empty((nbox, n_near, 3))
    nnrm = np.empty((nbox, n_near, 3))
    for i in range(nbox):
        rng = np.random.default_rng(1000 + first_id + i)
        pts[i] = (rng.random((b, 3)) - 0.5) * h
        v = rng.standard_normal((b, 3))
        nrm[i] = v / np.linalg.norm(v, axis=1)[:, None]
        got = []
        cnt = 0
        while cnt < n_near:
            c = (rng.random((2 * n_near, 3)) - 0.5) * 3 * h
            keep = np.max(np.abs(c), axis=1) > 0.5 * h
            c = c[keep]
            got.append(c)
            cnt += c.shape[0]
        npts[i] = np.vstack(got)[:n_near]
        v = rng.standard_normal((n_near, 3))
        nnrm[i] = v / np.linalg.norm(v, axis=1)[:, None]
    return dict(pts=pts, nrm=nrm, npts=npts, nnrm=nnrm, w=h * h / b, h=h)
