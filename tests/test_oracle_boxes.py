"""Pins for oracle/boxes.py (cfg4: one isolated box, readings C21/C22)."""
import math

import numpy as np
import pytest

import fmmlu_inputs as fi
from oracle import boxes as ob

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def _small_box(seed=0, b=48, nnear=96):
    d = fi.box_batch(1, b=b, n_near=nnear, first_id=seed)
    return d["pts"][0], d["nrm"][0], d["npts"][0], d["nnrm"][0], d["w"], d["h"]


@pytest.mark.parametrize("eps", [1e-3, 1e-4])
def test_box_elimination_equals_explicit_transforms(eps):
    """Δ must equal the Schur complement of the R block of Z = E Ã F, where E (row ops
    R −= Tᵀ S) and F (column ops R −= S T) are built as explicit matrices:
    Z_{R,S} = X_RS etc., and Δ = Z_cc − Z_cR Z_RR⁻¹ Z_Rc − Z_cc with c = [S | N]."""
    pts, nrm, npts, nnrm, w, h = _small_box(1, b=160, nnear=96)
    o = ob.eliminate_box(10.0, eps, pts, nrm, npts, nnrm, w, h, n_gamma=256)
    b, kk = pts.shape[0], o["k"]
    assert 0 < kk < b
    S, R = o["perm"][:kk], o["perm"][kk:]
    N = np.arange(b, b + npts.shape[0])
    order = np.concatenate([R, S, N])
    A = o["A"][np.ix_(order, order)]
    r, n = R.size, A.shape[0]
    E = np.eye(n, dtype=complex)
    E[:r, r:r + kk] = -o["T"].T           # rows R −= Tᵀ rows S
    F = np.eye(n, dtype=complex)
    F[r:r + kk, :r] = -o["T"]             # cols R −= cols S · T
    Z = E @ A @ F
    Zrr, Zrc, Zcr, Zcc = Z[:r, :r], Z[:r, r:], Z[r:, :r], Z[r:, r:]
    schur = Zcc - Zcr @ np.linalg.solve(Zrr, Zrc)
    assert np.allclose(o["X_RR"], Zrr, rtol=0, atol=1e-12 * np.abs(Zrr).max())
    ref = schur - Zcc
    assert np.abs(o["Delta"] - ref).max() <= 1e-10 * np.abs(ref).max()


def test_box_id_bound_and_rank_bracket():
    """Full cfg4 box (b=256, 2×512 proxy rows): every redundant column is fit to ε·max column
    norm (C9), and k is at least the number of singular values above √b·ε·σ₀ (σ_{k+1} ≤
    ‖R₂₂‖ ≤ √(b−k)·|R_kk| ≤ √b·ε·|R₀₀| ≤ √b·ε·σ₀; greedy CPQR has no matching upper bound)."""
    pts, nrm, npts, nnrm, w, h = _small_box(3, b=256, nnear=64)
    eps = 1e-6
    o = ob.eliminate_box(10.0, eps, pts, nrm, npts, nnrm, w, h)
    M, P, kk, T = o["M"], o["perm"], o["k"], o["T"]
    assert M.shape == (1024, 256)
    res = M[:, P[kk:]] - M[:, P[:kk]] @ T
    cn = np.linalg.norm(M, axis=0).max()
    assert np.linalg.norm(res, axis=0).max() <= 2 * eps * cn
    sv = np.linalg.svd(M, compute_uv=False)
    lo = int(np.sum(sv > eps * sv[0] * math.sqrt(256)))
    assert lo <= kk <= 256


def test_box_degenerate_ranks():
    """ε below rounding → k = b, nothing eliminated, Δ = 0; ε near 1 → tiny skeleton."""
    pts, nrm, npts, nnrm, w, h = _small_box(2, b=32, nnear=32)
    o = ob.eliminate_box(10.0, 1e-15, pts, nrm, npts, nnrm, w, h, n_gamma=128)
    assert o["k"] == 32 and np.all(o["Delta"] == 0)
    o = ob.eliminate_box(10.0, 0.9, pts, nrm, npts, nnrm, w, h, n_gamma=128)
    assert 1 <= o["k"] <= 2


def test_given_split_with_cpqr_order_reproduces_the_id():
    """split = (CPQR perm, k) reproduces T = R11⁻¹R12 and Δ: the least-squares fit for the CPQR
    pivot order is the ID's T (M_S = Q₁R11, M_R = Q₁R12 + Q₂R22, Q₂ ⊥ Q₁)."""
    pts, nrm, npts, nnrm, w, h = _small_box(4, b=160, nnear=64)
    o = ob.eliminate_box(10.0, 1e-4, pts, nrm, npts, nnrm, w, h, n_gamma=256)
    g = ob.eliminate_box(10.0, 1e-4, pts, nrm, npts, nnrm, w, h, n_gamma=256, split=(o["perm"], o["k"]))
    assert 0 < o["k"] < 160
    assert np.abs(g["T"] - o["T"]).max() <= 1e-8 * np.abs(o["T"]).max()
    assert np.abs(g["Delta"] - o["Delta"]).max() <= 1e-10 * np.abs(o["Delta"]).max()
    # a different (valid) split of the same size: swap the last skeleton and first redundant column
    P2 = o["perm"].copy()
    kk = o["k"]
    P2[kk - 1], P2[kk] = P2[kk], P2[kk - 1]
    g2 = ob.eliminate_box(10.0, 1e-4, pts, nrm, npts, nnrm, w, h, n_gamma=256, split=(P2, kk))
    res = g2["M"][:, P2[kk:]] - g2["M"][:, P2[:kk]] @ g2["T"]
    assert np.linalg.norm(res, axis=0).max() <= 2e-4 * np.linalg.norm(g2["M"], axis=0).max()
