"""Pins for oracle/idqr.py (reading C9; SVD bounds)."""
import math

import numpy as np
import pytest

from oracle import idqr, kernel as kern


def test_rank_one():
    rng = np.random.default_rng(0)
    u = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    v = rng.standard_normal(25) + 1j * rng.standard_normal(25)
    M = np.outer(u, v)
    P, k, T = idqr.interp_decomp(M, 1e-9)
    assert k == 1
    S, R = P[:k], P[k:]
    assert np.max(np.abs(M[:, R] - M[:, S] @ T)) < 1e-13 * np.abs(M).max()


def test_duplicate_columns():
    c = np.array([[1.0 + 2j], [3.0 - 1j], [0.5j]])
    M = np.hstack([c, c])
    P, k, T = idqr.interp_decomp(M, 1e-9)
    assert k == 1 and P[0] == 0          # tie → lowest index
    assert np.allclose(T, [[1.0]], atol=1e-15)


@pytest.mark.parametrize("eps", [1e-3, 1e-6, 1e-9])
def test_kernel_block_bounds(eps):
    rng = np.random.default_rng(1)
    src = rng.random((100, 3))
    trg = rng.random((200, 3)) + np.array([2.0, 0.0, 0.0])
    M = kern.green(2.0, trg, src)
    P, k, T = idqr.interp_decomp(M, eps)
    S, R = P[:k], P[k:]
    E = M[:, R] - M[:, S] @ T
    colmax = np.max(np.linalg.norm(M, axis=0))
    # per-column residual bound of the CPQR stopping rule (reading C9)
    assert np.max(np.linalg.norm(E, axis=0)) <= 1.01 * eps * colmax
    sv = np.linalg.svd(M, compute_uv=False)
    # the residual can never beat the best rank-k approximation
    assert np.linalg.norm(E, 2) >= 0.999 * sv[k]
    # and the rank is not larger than the numerical rank at a looser threshold
    assert k <= np.sum(sv > 0.01 * eps * sv[0])
    assert k >= np.sum(sv > np.sqrt(M.shape[1]) * eps * colmax * 1.01)


def test_proxy_count_rule():
    assert idqr.proxy_count(0.0, 1.0, 1e-6) == 144    # κ = 0 floor
    assert idqr.proxy_count(2 * math.pi, 0.25, 1e-6) == 180
    ns = [idqr.proxy_count(k, 1.0, 1e-6) for k in (1, 5, 10, 20, 40)]
    assert ns == sorted(ns)


def test_proxy_points_on_sphere():
    Y, s = idqr.proxy_points([1.0, 2.0, 3.0], 0.5, 144)
    r = np.linalg.norm(Y - np.array([1.0, 2.0, 3.0]), axis=1)
    assert np.allclose(r, 0.5, atol=1e-14)
    assert abs(s * s * 144 - 4 * math.pi * 0.25) < 1e-13
    # quasi-uniform: the centroid is the centre
    assert np.linalg.norm(Y.mean(axis=0) - np.array([1.0, 2.0, 3.0])) < 1e-2
