"""Pins for the oracle's separate incoming/outgoing IDs (PAPER.md L726-732:
"Different interpolation matrices can be used for each of A_BFᵀ and A_FB ... smaller skeleton
sets"; L1098-1108, L1909-1914; DESIGN reading R12).

* literal Eq. strong-skel-elim with the two sets: for every eliminated box, Z = L E A F U built
  from identity matrices (E from T_r on rows, F from T_c on columns) has Z_{R_r,(S∪N)_c} =
  Z_{(S∪N)_r,R_c} = 0, its (S∪N)_r × (S∪N)_c block equals the oracle's in-place Schur update,
  and both far-field blocks Z_{F_r R_c}, Z_{R_r F_c} are ≤ 10ε against the FULL complement
  (so each ID compresses the true far field, not just the proxy rows);
* the factorization is an ε-factorization: residual ≤ 10ε, within 10ε of the dense solve;
  ε = 1e-12 reproduces the dense solve; apply ∘ solve = identity;
* the paper's claim: smaller skeleton sets in aggregate (Σ|S| and n₀) than the simultaneous ID.
"""
import math

import numpy as np
import pytest

import fmmlu_inputs as fi
from oracle import dense, kernel as kern, rss


def test_separate_literal_elimination_and_far_field():
    g = fi.ellipsoid(1200)
    k, eps = 2 * math.pi, 1e-6
    checked = {"n": 0, "proxy": 0, "differ": 0}
    store = {}

    def hook(stage, c):
        Br, Bs, Nr, Fr, Tr = c["Br"], c["Bs"], c["Nidx"], c["Fidx"], c["T"]
        Brc, Bsc, Nc, Fc, Tc = c["Br_c"], c["Bs_c"], c["Nc"], c["Fc"], c["T_c"]
        r, kk, nn, nf = Br.size, Bs.size, Nr.size, Fr.size
        assert (Brc.size, Bsc.size, Nc.size, Fc.size) == (r, kk, nn, nf)
        ir = np.concatenate([Br, Bs, Nr, Fr])
        ic = np.concatenate([Brc, Bsc, Nc, Fc])
        if stage == "pre":
            store["A"] = c["A"][np.ix_(ir, ic)].copy()
            return
        A0 = store["A"]
        m = ir.size
        E = np.eye(m, dtype=complex)
        E[:r, r:r + kk] = -Tr.T        # rows R_r −= T_rᵀ rows S_r
        F = np.eye(m, dtype=complex)
        F[r:r + kk, :r] = -Tc          # cols R_c −= cols S_c T_c
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
        A1 = c["A"][np.ix_(ir[sn], ic[sn])]
        assert np.abs(Z[sn, sn] - A1).max() < 1e-12 * sc
        if nf:
            fsl = slice(r + kk + nn, m)
            AFB = A0[fsl, :r + kk]
            ABF = A0[:r + kk, fsl]
            assert np.linalg.norm(Z[fsl, :r], 2) <= 10 * eps * np.linalg.norm(AFB, 2)
            assert np.linalg.norm(Z[:r, fsl], 2) <= 10 * eps * np.linalg.norm(ABF, 2)
            if c["nP"] > 0:
                checked["proxy"] += 1
        if set(Bs.tolist()) != set(Bsc.tolist()):
            checked["differ"] += 1
        checked["n"] += 1

    rss.factor(g.points, g.normals, g.weights, k, eps, 24, hook=hook, separate=True)
    # the two sides do choose different skeletons on this non-symmetric kernel
    assert checked["n"] >= 12 and checked["proxy"] >= 4 and checked["differ"] >= 4, checked


@pytest.mark.parametrize("case", ["ellipsoid3000", "cube1500"])
def test_separate_is_eps_factorization(case):
    eps = 1e-6
    if case == "ellipsoid3000":
        g, k, leaf = fi.ellipsoid(3000), 2 * math.pi, 32
    else:
        g, k, leaf = fi.random_cube(1500, seed=2), 3.0, 16
    b = fi.gaussian_rhs(g.n, 2, 0)
    f = rss.factor(g.points, g.normals, g.weights, k, eps, leaf, separate=True)
    x = rss.solve(f, b)
    assert dense.residual(g.points, g.normals, g.weights, k, x, b) <= 10 * eps
    xd = dense.dense_solve(g.points, g.normals, g.weights, k, b)
    assert dense.rel_diff(x, xd) <= 10 * eps
    # the forward form is A within ε and the exact inverse of the solve
    y = rss.apply(f, b)
    assert dense.rel_diff(y, kern.matvec_unscaled(k, g.points, g.normals, g.weights, b)) <= 10 * eps
    assert dense.rel_diff(rss.solve(f, y), b) < 1e-12
    # row and column root sets have the same size (square pivot blocks throughout)
    assert f.Bt.size == f.Bt_c.size == f.stats["n0"]


def test_separate_tight_eps_is_dense():
    g = fi.ellipsoid(2000)
    k = 2 * math.pi
    b = fi.gaussian_rhs(g.n, 1, 1)
    f = rss.factor(g.points, g.normals, g.weights, k, 1e-12, 32, separate=True)
    assert len(f.records) > 0
    xd = dense.dense_solve(g.points, g.normals, g.weights, k, b)
    assert dense.rel_diff(rss.solve(f, b), xd) < 1e-9


def test_separate_gives_smaller_skeletons():
    # "Using different compression matrices will result in smaller skeleton
    # sets".  Aggregate over the tree (per box it is not a theorem: each side's ID has its own
    # relative threshold); the square-pivot rule k = max(k_r, k_c) is included
    g = fi.ellipsoid(3000)
    k, eps = 2 * math.pi, 1e-6
    f0 = rss.factor(g.points, g.normals, g.weights, k, eps, 32)
    f1 = rss.factor(g.points, g.normals, g.weights, k, eps, 32, separate=True)
    s0 = sum(v.size for v in f0.stats["skeletons"].values())
    s1 = sum(v.size for v in f1.stats["skeletons"].values())
    assert s1 < s0
    assert f1.stats["n0"] < f0.stats["n0"]
    rc = np.array(f1.stats["ranks_rc"])
    assert (rc[:, 0] != rc[:, 1]).any()      # the two IDs do have different ε-ranks
