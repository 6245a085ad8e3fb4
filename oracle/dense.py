"""Oracle: exact dense references (test infrastructure only).

* ``dense_solve``: LAPACK zgesv (scipy.linalg.solve) on BASELINE.json's unscaled
  A = ½I + (D − ikS)W with K_ii = 0 — the exact answer the ε-approximate
  factorization approaches as ε → 0 (BASELINE.json north_star).
* ``residual``: ‖Ax − b‖₂/‖b‖₂ per RHS column with the brute-force O(n²) matvec
  (reading C17), max over columns.
* ``rel_diff``: ‖x − y‖₂/‖y‖₂ per column, max over columns.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from . import kernel as kern


def dense_solve(points, normals, weights, k, b):
    A = kern.dense_unscaled(k, points, normals, weights)
    return sla.solve(A, b)


def residual(points, normals, weights, k, x, b) -> float:
    Ax = kern.matvec_unscaled(k, points, normals, weights, x)
    r = np.atleast_2d((Ax - b).T).T if np.ndim(b) > 1 else (Ax - b)[:, None]
    bb = b if np.ndim(b) > 1 else b[:, None]
    return float(np.max(np.linalg.norm(r, axis=0) / np.linalg.norm(bb, axis=0)))


def rel_diff(x, y) -> float:
    x = np.asarray(x)
    y = np.asarray(y)
    if x.ndim == 1:
        x, y = x[:, None], y[:, None]
    return float(np.max(np.linalg.norm(x - y, axis=0) / np.linalg.norm(y, axis=0)))
