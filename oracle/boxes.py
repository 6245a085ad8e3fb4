"""Oracle for BASELINE.json configs[3] ("cfg4"): ID + elimination of ONE isolated box
(test infrastructure only — nothing in the product path imports this module).

Readings C21/C22: the box holds b active DOFs, its near set N holds
n_near DOFs (Schur-update targets, never ID rows), Q = ∅, and the ID rows are the proxy
rows only (2 n_γ rows, always present).  Steps, in the paper's order and notation:

1. Entries Ã_ij = √w_i K(x_i, x_j) √w_j, Ã_ii = ½ (P:L443-493 Eqs. disc1/disc3, reading C1).
2. M = [s_γ K(y_ℓ, x_j) √w_j ; s_γ G(x_j, y_ℓ) √w_j]  (outgoing with the box normals,
   incoming single layer, readings C3/C4), y_ℓ = Fibonacci points on the
   sphere of radius ρ about the box centre (R2).
3. ID of M at tolerance ε (zgeqp3 + the C9 stop rule; ``idqr.interp_decomp``):
   S = perm[:k], R = perm[k:], T = R11⁻¹R12.
4. X_RR = A_RR − TᵀA_SR − A_RS T + TᵀA_SS T,  X_RS = A_RS − TᵀA_SS,  X_SR = A_SR − A_SS T,
   X_RN = A_RN − TᵀA_SN,  X_NR = A_NR − A_NS T  (Tᵀ a plain transpose).
5. Δ_{(S∪N),(S∪N)} = −X_{(S∪N)R} X_RR⁻¹ X_{R(S∪N)}, frame order [S (pivot
   order) | N (given order)].

Pins: tests/test_oracle_boxes.py (ID residual bound, the rank bracket by singular values,
Δ against the Schur complement of the explicitly transformed dense block L E Ã F U).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla

from . import kernel as kern
from .idqr import interp_decomp, proxy_points


def box_matrix(k: float, pts, nrm, npts, nnrm, w):
    """Ã on [B | N] (b + n_near square), uniform weight w."""
    X = np.vstack([pts, npts])
    NX = np.vstack([nrm, nnrm])
    sw = np.full(X.shape[0], math.sqrt(w))
    return kern.dense_scaled(k, X, NX, sw)


def proxy_rows(k: float, pts, nrm, w, centre, rho: float, n_gamma: int):
    Y, s_g = proxy_points(centre, rho, n_gamma)
    sw = math.sqrt(w)
    Kout = kern.combined_field(k, Y, pts, nrm) * sw
    Sin = kern.green(k, pts, Y).T * sw
    return np.vstack([s_g * Kout, s_g * Sin])


def eliminate_box(k: float, eps: float, pts, nrm, npts, nnrm, w, h,
                  n_gamma: int = 512, rho: float | None = None, split=None):
    """Return dict(perm, k, T, M, Delta) for one cfg4 box (centre 0, side h).

    split = (perm, kk): use the given skeleton S = perm[:kk] (in that order) and redundant
    R = perm[kk:] instead of the CPQR choice, with T the least-squares interpolation matrix
    T = argmin ‖M_R − M_S T‖ (PAPER.md L614-616 defines the ID by that fit; for the CPQR pivot
    order it is exactly R11⁻¹R12, since M_S = Q₁R11 and M_R = Q₁R12 + Q₂R22).  Used to judge a
    GPU result whose skeleton differs from the oracle's at a pivot near-tie: the elimination
    steps are the same, only the column split is taken from the GPU."""
    b = pts.shape[0]
    if rho is None:
        rho = 1.5 * (math.sqrt(3.0) / 2.0) * h     # 1.5 × half-diagonal (BJ configs[3])
    A = box_matrix(k, pts, nrm, npts, nnrm, w)
    M = proxy_rows(k, pts, nrm, w, np.zeros(3), rho, n_gamma)
    if split is None:
        P, kk, T = interp_decomp(M, eps)
    else:
        P, kk = np.asarray(split[0], dtype=np.int64), int(split[1])
        if kk > 0 and kk < b:
            T = np.linalg.lstsq(M[:, P[:kk]], M[:, P[kk:]], rcond=None)[0]
        else:
            T = np.zeros((kk, b - kk), dtype=np.complex128)
    S, R = P[:kk], P[kk:]
    N = np.arange(b, A.shape[0])
    g = lambda r, c: A[np.ix_(r, c)]
    X_RR = g(R, R) - T.T @ g(S, R) - g(R, S) @ T + T.T @ g(S, S) @ T
    X_RS = g(R, S) - T.T @ g(S, S)
    X_SR = g(S, R) - g(S, S) @ T
    X_RN = g(R, N) - T.T @ g(S, N)
    X_NR = g(N, R) - g(N, S) @ T
    X_cR = np.vstack([X_SR, X_NR])
    X_Rc = np.hstack([X_RS, X_RN])
    if R.size:
        lu = sla.lu_factor(X_RR, check_finite=False)
        Delta = -X_cR @ sla.lu_solve(lu, X_Rc)
    else:
        Delta = np.zeros((kk + N.size, kk + N.size), dtype=np.complex128)
    return dict(perm=P, k=kk, T=T, M=M, A=A, Delta=Delta, X_RR=X_RR)
