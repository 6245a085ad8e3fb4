"""Pins for oracle/rss.py: dense-LU limits, literal Eq. strong-skel-elim, proxy
completeness, residual ≤ 10ε (BASELINE.json north_star)."""
import math

import numpy as np
import pytest
import scipy.linalg as sla

import fmmlu_inputs as fi
from oracle import dense, kernel as kern, rss


def _solve_check(g, k, eps, leaf, nrhs=2, seed=0):
    b = fi.gaussian_rhs(g.n, nrhs, seed)
    f = rss.factor(g.points, g.normals, g.weights, k, eps, leaf)
    x = rss.solve(f, b)
    return f, x, b


def test_single_leaf_is_dense_lu():
    g = fi.fibonacci_sphere(60)
    f, x, b = _solve_check(g, 1.0, 1e-6, 64)
    assert f.stats["n0"] == 60 and not f.records
    xd = dense.dense_solve(g.points, g.normals, g.weights, 1.0, b)
    assert dense.rel_diff(x, xd) < 1e-13


def test_cube_corners_root_only():
    g = fi.cube_corners()
    f, x, b = _solve_check(g, 1.0, 1e-6, 1)
    assert f.tree.nlevels == 2 and not f.records and f.stats["n0"] == 8
    xd = dense.dense_solve(g.points, g.normals, g.weights, 1.0, b)
    assert dense.rel_diff(x, xd) < 1e-13


@pytest.mark.parametrize("case", ["sphere400", "cube1500", "ellipsoid3000"])
def test_residual_10eps(case):
    eps = 1e-6
    if case == "sphere400":
        g, k, leaf = fi.fibonacci_sphere(400), 1.0, 8
    elif case == "cube1500":
        g, k, leaf = fi.random_cube(1500, seed=2), 3.0, 16
    else:
        g, k, leaf = fi.ellipsoid(3000), 2 * math.pi, 32
    f, x, b = _solve_check(g, k, eps, leaf)
    if case == "ellipsoid3000":   # tiny leaves (sphere, volume cube) compress nothing: rank = |B|
        assert len(f.records) > 0 and f.stats["n0"] < g.n
    res = dense.residual(g.points, g.normals, g.weights, k, x, b)
    assert res <= 10 * eps
    xd = dense.dense_solve(g.points, g.normals, g.weights, k, b)
    assert dense.rel_diff(x, xd) <= 10 * eps


def test_tight_eps_reproduces_dense_lu():
    g = fi.ellipsoid(2000)
    k = 2 * math.pi
    f, x, b = _solve_check(g, k, 1e-12, 32)
    assert len(f.records) > 0
    xd = dense.dense_solve(g.points, g.normals, g.weights, k, b)
    assert dense.rel_diff(x, xd) < 1e-9


def test_literal_strong_skel_elim_and_proxy_completeness():
    """For every eliminated box: Z = L E Pᵀ A P F U built from dense identity-based
    matrices has Z_{R,S∪N} = Z_{S∪N,R} = 0, ‖Z_{R,F}‖,‖Z_{F,R}‖ ≤ 10ε‖A_{FB}‖ (the
    proxy+Q ID compresses the TRUE far field),
    and Z_{S∪N,S∪N} equals the oracle's in-place Schur update."""
    g = fi.ellipsoid(1200)
    k, eps = 2 * math.pi, 1e-6
    checked = {"n": 0, "proxy": 0}
    store = {}

    def hook(stage, c):
        Br, Bs, Nidx, Fidx, T = c["Br"], c["Bs"], c["Nidx"], c["Fidx"], c["T"]
        r, kk, nn, nf = Br.size, Bs.size, Nidx.size, Fidx.size
        idx = np.concatenate([Br, Bs, Nidx, Fidx])
        if stage == "pre":
            store["A"] = c["A"][np.ix_(idx, idx)].copy()
            return
        A0 = store["A"]
        m = idx.size
        E = np.eye(m, dtype=complex)
        E[:r, r:r + kk] = -T.T
        F = np.eye(m, dtype=complex)
        F[r:r + kk, :r] = -T
        X = E @ A0 @ F
        XRRi = np.linalg.inv(X[:r, :r])
        L = np.eye(m, dtype=complex)
        L[r:r + kk + nn, :r] = -X[r:r + kk + nn, :r] @ XRRi
        U = np.eye(m, dtype=complex)
        U[:r, r:r + kk + nn] = -XRRi @ X[:r, r:r + kk + nn]
        Z = L @ X @ U
        sc = np.abs(A0).max()
        sn = slice(r, r + kk + nn)
        assert np.abs(Z[:r, sn]).max() < 1e-12 * sc
        assert np.abs(Z[sn, :r]).max() < 1e-12 * sc
        A1 = c["A"][np.ix_(idx[sn], idx[sn])]
        assert np.abs(Z[sn, sn] - A1).max() < 1e-12 * sc
        if nf:
            fsl = slice(r + kk + nn, m)
            AFB = A0[fsl, :r + kk]
            ABF = A0[:r + kk, fsl]
            assert np.linalg.norm(Z[fsl, :r], 2) <= 10 * eps * np.linalg.norm(AFB, 2)
            assert np.linalg.norm(Z[:r, fsl], 2) <= 10 * eps * np.linalg.norm(ABF, 2)
            if c["nP"] > 0:
                checked["proxy"] += 1
        checked["n"] += 1

    rss.factor(g.points, g.normals, g.weights, k, eps, 24, hook=hook)
    assert checked["n"] >= 12 and checked["proxy"] >= 4, checked


# ---- forward form A ≈ V₁⋯V_M P_t D P_tᵀ W_M⋯W₁
def test_apply_single_leaf_is_exact_matvec():
    # no skeletonized box: the forward form is P_t A P_tᵀ itself
    g = fi.fibonacci_sphere(60)
    f = rss.factor(g.points, g.normals, g.weights, 1.0, 1e-6, 64)
    x = fi.gaussian_rhs(g.n, 2, 3)
    y = rss.apply(f, x)
    ye = kern.matvec_unscaled(1.0, g.points, g.normals, g.weights, x)
    assert dense.rel_diff(y, ye) < 1e-13


@pytest.mark.parametrize("eps", [1e-6, 1e-12])
def test_apply_approximates_A_and_inverts_solve(eps):
    g = fi.ellipsoid(3000)
    k = 2 * math.pi
    f = rss.factor(g.points, g.normals, g.weights, k, eps, 32)
    assert len(f.records) > 0
    x = fi.gaussian_rhs(g.n, 2, 5)
    y = rss.apply(f, x)
    ye = kern.matvec_unscaled(k, g.points, g.normals, g.weights, x)   # brute-force A x
    assert dense.rel_diff(y, ye) <= (10 * eps if eps > 1e-9 else 1e-9)
    # apply and solve are exact inverses of each other (same factors, sign-toggled)
    assert dense.rel_diff(rss.solve(f, y), x) < 1e-12
    assert dense.rel_diff(rss.apply(f, rss.solve(f, x)), x) < 1e-12
    # linearity
    a = 0.3 - 1.7j
    assert dense.rel_diff(rss.apply(f, a * x[:, :1] + x[:, 1:]), a * y[:, :1] + y[:, 1:]) < 1e-12
