"""Oracle: Helmholtz Green's function and combined-field kernel (test infrastructure only).

G(x,y) = e^{ik|x-y|} / (4π|x-y|)                          PAPER.md L408-413 Eq. greenfunhelm
K(x,y) = n(y)·∇_y G(x,y) − ik G(x,y)                       PAPER.md L414-421 Eq. comb_ref
       = e^{ikr}(1−ikr) ((x−y)·n(y)) / (4πr³) − ik e^{ikr}/(4πr)   (reading C2: row = target x,
                                                                     column = source y with normal n(y))
Scaled Nyström entries  Ã_ij = √w_i K(x_i,x_j) √w_j (i≠j), Ã_ii = ½
                                                          PAPER.md L443-493 Eqs. disc1/disc3, reading C1/C19
Unscaled system         A_ij = K(x_i,x_j) w_j (i≠j),  A_ii = ½   (BASELINE.json: A = I/2 + (D − iηS)W, η = k)

Pins (tests/test_oracle_kernel.py): SPEC S:L104-105, L113-114 exact values; the
unit-sphere closed form K = −e^{ikr}(1−ikr+2ik)/(8πr) (derived independently from
(x−y)·y = −r²/2 on |x|=|y|=1, n=y); reciprocity of G; central finite differences
of G for the double-layer term; the Laplace Gauss identity (½I + D)1 ≈ 0.
"""
from __future__ import annotations

import math

import numpy as np

FOUR_PI = 4.0 * math.pi


def _diff(x, y):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    d = x[..., :, None, :] - y[..., None, :, :]
    r = np.sqrt(np.sum(d * d, axis=-1))
    return d, r


def green(k: float, x, y) -> np.ndarray:
    """G(x_i, y_j) for point arrays x (m×3), y (p×3) → m×p complex."""
    _, r = _diff(x, y)
    return np.exp(1j * k * r) / (FOUR_PI * r)


def double_layer(k: float, x, y, ny) -> np.ndarray:
    """D(x_i, y_j) = n(y_j)·∇_y G(x_i, y_j) = e^{ikr}(1-ikr)((x-y)·n(y))/(4πr³)."""
    d, r = _diff(x, y)
    dn = np.sum(d * np.asarray(ny)[None, :, :], axis=-1)
    return np.exp(1j * k * r) * (1.0 - 1j * k * r) * dn / (FOUR_PI * r**3)


def combined_field(k: float, x, y, ny) -> np.ndarray:
    """K(x_i, y_j) = D − ik S."""
    return double_layer(k, x, y, ny) - 1j * k * green(k, x, y)


def scaled_block(k: float, X, NX, sw, rows, cols) -> np.ndarray:
    """Ã[rows, cols] of the √w-scaled matrix: √w_i K(x_i,x_j) √w_j, and ½ where i == j."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    out = np.empty((rows.size, cols.size), dtype=np.complex128)
    if rows.size == 0 or cols.size == 0:
        return out
    same = rows[:, None] == cols[None, :]
    with np.errstate(divide="ignore", invalid="ignore"):
        Kb = combined_field(k, X[rows], X[cols], NX[cols])
    out[:] = sw[rows][:, None] * Kb * sw[cols][None, :]
    out[same] = 0.5
    return out


def dense_scaled(k: float, X, NX, sw, chunk: int = 512) -> np.ndarray:
    """The whole n×n Ã (complex128), row-chunked."""
    n = X.shape[0]
    A = np.empty((n, n), dtype=np.complex128)
    cols = np.arange(n)
    for s in range(0, n, chunk):
        rows = np.arange(s, min(n, s + chunk))
        A[s:s + rows.size] = scaled_block(k, X, NX, sw, rows, cols)
    return A


def dense_unscaled(k: float, X, NX, w) -> np.ndarray:
    """BASELINE.json's A = ½I + K W with K_ii = 0 (used for residuals)."""
    n = X.shape[0]
    with np.errstate(divide="ignore", invalid="ignore"):
        A = combined_field(k, X, X, NX) * np.asarray(w)[None, :]
    A[np.arange(n), np.arange(n)] = 0.5
    return A


def matvec_unscaled(k: float, X, NX, w, x, chunk: int = 1024) -> np.ndarray:
    """Brute-force O(n²) y = A x for BASELINE.json's unscaled A (x: n or n×nrhs)."""
    x = np.asarray(x, dtype=np.complex128)
    vec = x.ndim == 1
    xx = x[:, None] if vec else x
    n = X.shape[0]
    y = np.empty_like(xx)
    wx = np.asarray(w)[:, None] * xx
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        with np.errstate(divide="ignore", invalid="ignore"):
            Kb = combined_field(k, X[s:e], X, NX)
        idx = np.arange(s, e)
        Kb[idx - s, idx] = 0.0
        y[s:e] = Kb @ wx + 0.5 * xx[s:e]
    return y[:, 0] if vec else y
