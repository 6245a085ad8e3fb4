"""Pins for oracle/kernel.py against values and identities fixed outside the oracle."""
import json
import math
import os

import numpy as np
import pytest
import scipy.special as sp

import fmmlu_inputs as fi
from oracle import kernel as kern

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "kernel_values.json")))


def test_green_golden_values():
    for e in GOLD["green"]:
        v = kern.green(e["k"], np.array([e["x"]], float), np.array([e["y"]], float))[0, 0]
        assert abs(v - complex(e["value_re"], e["value_im"])) < 1e-15


def test_double_layer_golden_and_combined_at_k0():
    for e in GOLD["double_layer"]:
        x, y, ny = (np.array([e[key]], float) for key in ("x", "y", "ny"))
        v = kern.double_layer(e["k"], x, y, ny)[0, 0]
        assert abs(v - complex(e["value_re"], e["value_im"])) < 1e-15
        # CombinedField at k = 0 is exactly DoubleLayer
        assert kern.combined_field(0.0, x, y, ny)[0, 0] == v


def test_unit_sphere_closed_form():
    """|x| = |y| = 1, n(y) = y  ⇒  (x−y)·y = −r²/2  ⇒  K = −e^{ikr}(1 − ikr + 2ik)/(8πr)."""
    rng = np.random.default_rng(3)
    for k in (0.0, 1.0, 7.5):
        u = rng.standard_normal((50, 3))
        u /= np.linalg.norm(u, axis=1)[:, None]
        x, y = u[:25], u[25:]
        K = kern.combined_field(k, x, y, y)
        r = np.linalg.norm(x[:, None, :] - y[None, :, :], axis=-1)
        ref = -np.exp(1j * k * r) * (1 - 1j * k * r + 2j * k) / (8 * math.pi * r)
        assert np.max(np.abs(K - ref) / np.abs(ref)) < 1e-12


def test_reciprocity_and_fd_gradient():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((7, 3))
    y = rng.standard_normal((9, 3)) + 3.0
    k = 0.97
    G1 = kern.green(k, x, y)
    G2 = kern.green(k, y, x).T
    assert np.max(np.abs(G1 - G2)) == 0.0
    ny = rng.standard_normal((9, 3))
    ny /= np.linalg.norm(ny, axis=1)[:, None]
    h = 1e-5
    fd = (kern.green(k, x, y + h * ny) - kern.green(k, x, y - h * ny)) / (2 * h)
    D = kern.double_layer(k, x, y, ny)
    assert np.max(np.abs(fd - D) / np.abs(D)) < 1e-7


def test_helmholtz_pde_fd():
    """(Δ + k²) G(·, y) = 0 away from y (second-order FD Laplacian)."""
    k = 2.0
    x0 = np.array([[0.3, -0.2, 0.9]])
    y = np.array([[0.0, 0.0, 0.0]])
    h = 1e-3
    lap = -6 * kern.green(k, x0, y)[0, 0]
    for a in range(3):
        e = np.zeros((1, 3))
        e[0, a] = h
        lap += kern.green(k, x0 + e, y)[0, 0] + kern.green(k, x0 - e, y)[0, 0]
    lap /= h * h
    g = kern.green(k, x0, y)[0, 0]
    assert abs(lap + k * k * g) < 1e-4 * abs(g)


def test_laplace_gauss_identity_orientation():
    """(½I + D)1 → 0 for k = 0 on a closed surface with outward normals (exterior
    jump +½).  O(h) without quadrature corrections."""
    errs = []
    for n in (1000, 4000):
        g = fi.fibonacci_sphere(n)
        A = kern.dense_unscaled(0.0, g.points, g.normals, g.weights)
        errs.append(np.max(np.abs(A @ np.ones(n))))
    assert errs[0] < 0.03 and errs[1] < 0.6 * errs[0]


def test_sphere_eigenvalues_l0_l1():
    """Unit sphere: ½I + D − ikS has eigenvalue λ_l = ik² j_l'(k) h_l(k) + k² j_l(k) h_l(k)
    on Y_l (Funk–Hecke; exterior limit of the double layer).  Discrete Rayleigh
    quotients converge to it at O(h) (no quadrature corrections)."""
    k = 1.0
    errs = {0: [], 1: []}
    for n in (2000, 8000):
        g = fi.fibonacci_sphere(n)
        A = kern.dense_unscaled(k, g.points, g.normals, g.weights)
        for l, v in ((0, np.ones(n)), (1, g.points[:, 2].copy())):
            h = sp.spherical_jn(l, k) + 1j * sp.spherical_yn(l, k)
            lam = 1j * k * k * sp.spherical_jn(l, k, derivative=True) * h + k * k * sp.spherical_jn(l, k) * h
            wv = g.weights * v
            rq = (wv @ (A @ v)) / (wv @ v)
            errs[l].append(abs(rq - lam) / abs(lam))
    for l in (0, 1):
        assert errs[l][0] < 0.06
        assert errs[l][1] < 0.6 * errs[l][0]


def test_scaled_vs_unscaled_similarity():
    g = fi.ellipsoid(300)
    k = 2.0
    A = kern.dense_unscaled(k, g.points, g.normals, g.weights)
    sw = np.sqrt(g.weights)
    At = kern.dense_scaled(k, g.points, g.normals, sw, chunk=97)
    assert np.max(np.abs(At - sw[:, None] * A / sw[None, :])) < 1e-13
    x = np.random.default_rng(0).standard_normal((300, 2)) + 0j
    y = kern.matvec_unscaled(k, g.points, g.normals, g.weights, x, chunk=77)
    assert np.max(np.abs(y - A @ x)) < 1e-12 * np.max(np.abs(A @ x))
