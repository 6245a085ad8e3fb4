"""Oracle: interpolative decomposition and proxy surface (test infrastructure only).

ID (PAPER.md L606-631 Def. ID "standard greedy column-pivoted QR"):
column-pivoted Householder QR  M P = Q R  (LAPACK zgeqp3 via scipy.linalg.qr — a
library primitive used as one step), rank k = first j with |R_jj| ≤ ε·|R_00|
(reading C9: stop when the largest remaining column norm ≤ ε × the largest
initial one; robust to a slightly non-monotone diagonal), S = P[:k],
R = P[k:], T = R11⁻¹ R12, so that M_{:,R} ≈ M_{:,S} T.

Proxy surface (readings C4/C5): sphere of radius
ρ_γ = 2·(box side) about the box centre, n_γ = 2p(p+1) Fibonacci points with
p = max(8, ⌈κ + 1.8 (log10(1/ε))^{2/3} κ^{1/3}⌉), κ = k ρ_γ, and quadrature
scale s_γ = √(4πρ_γ²/n_γ).

Pins (tests/test_oracle_id.py): rank-1 → |S| = 1 with zero residual; duplicated
columns [c, c] → S = {0}, T = [1]; ‖M_R − M_S T‖₂ ≥ σ_{k+1}(M)
and every redundant column residual ≤ ε·max column norm (C9 guarantee) against a
numpy SVD; n_γ = 144 at κ = 0; Fibonacci points on the sphere.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla

GOLDEN_ANGLE = math.pi * (3.0 - math.sqrt(5.0))


def interp_decomp(M: np.ndarray, eps: float, k_min: int = 0):
    """Return (perm, k, T): skeleton columns perm[:k], redundant perm[k:], T (k × (b-k)).

    k_min (separate in/out IDs, reading R12): continue the same greedy pivot order to
    k = max(k_ε, k_min) columns (caller guarantees k_min ≤ min(m, b)); T = R11⁻¹R12 of that
    leading k×k block.  The residual of a greedy CPQR only falls as pivots are added, so the
    longer ID is still ε-accurate."""
    m, b = M.shape
    if b == 0:
        return np.zeros(0, dtype=np.int64), 0, np.zeros((0, 0), dtype=M.dtype)
    R, P = sla.qr(M, mode="r", pivoting=True)
    d = np.abs(np.diag(R))
    kmax = min(m, b)
    if kmax == 0 or d[0] == 0.0:
        k = 0
    else:
        small = np.nonzero(d[:kmax] <= eps * d[0])[0]
        k = int(small[0]) if small.size else kmax
    k = max(k, k_min)
    T = sla.solve_triangular(R[:k, :k], R[:k, k:]) if k > 0 else np.zeros((0, b), dtype=M.dtype)
    return P.astype(np.int64), k, T


def proxy_order(k: float, rho: float, eps: float) -> int:
    kap = k * rho
    p = math.ceil(kap + 1.8 * (math.log10(1.0 / eps)) ** (2.0 / 3.0) * kap ** (1.0 / 3.0))
    return max(8, p)


def proxy_count(k: float, rho: float, eps: float) -> int:
    p = proxy_order(k, rho, eps)
    return 2 * p * (p + 1)


def fibonacci_dirs(m: int) -> np.ndarray:
    i = np.arange(m, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / m
    phi = i * GOLDEN_ANGLE
    s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return np.stack([s * np.cos(phi), s * np.sin(phi), z], axis=1)


def proxy_points(centre, rho: float, n_gamma: int):
    """Proxy points y_ℓ = c + ρ u_ℓ and the scale s_γ = √(4πρ²/n_γ)."""
    y = np.asarray(centre, dtype=np.float64)[None, :] + rho * fibonacci_dirs(n_gamma)
    return y, math.sqrt(4.0 * math.pi * rho * rho / n_gamma)
