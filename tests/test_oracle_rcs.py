"""Pins for oracle/rcs.py (§6.3)."""
import math

import numpy as np

import fmmlu_inputs as fi
from oracle import dense, rcs


def _sphere_rcs(n, k, phis):
    g = fi.fibonacci_sphere(n)
    b = rcs.plane_wave_rhs(g.points, k, phis)
    sigma = dense.dense_solve(g.points, g.normals, g.weights, k, b)
    return rcs.monostatic_rcs(g.points, g.normals, g.weights, k, phis, sigma)


def test_plane_wave_rhs_is_unit_modulus_plane_wave():
    g = fi.fibonacci_sphere(50)
    b = rcs.plane_wave_rhs(g.points, 2.0, [0.0, 1.0])
    assert np.allclose(np.abs(b), 1.0)
    assert np.allclose(b[:, 0], -np.exp(2j * g.points[:, 0]))


def test_sphere_matches_mie_series_and_converges():
    k = 2.0
    phis = [0.0, 1.3]
    ref = rcs.mie_backscatter_sphere(k)
    errs = []
    for n in (800, 3200):
        R = _sphere_rcs(n, k, phis)
        errs.append(np.max(np.abs(R - ref)) / abs(ref))
    # O(h) Nyström (K_ii = 0, reading C19): the error shrinks by ≈ 2 for 4× the points
    assert errs[1] < 0.7 * errs[0]
    assert errs[1] < 0.06


def test_sphere_rcs_is_rotation_invariant():
    R = _sphere_rcs(2000, 1.0, np.linspace(0, 2 * math.pi, 7, endpoint=False))
    assert np.max(np.abs(R - R.mean())) / abs(R.mean()) < 0.02


def test_mie_series_limits():
    # converged in lmax; small ka: the monopole j_0/h_0 = i sin(ka) e^{−ika} dominates, so
    # F → −sin(ka) e^{−ika}/k with the dipole correction O(a (ka)²)
    assert abs(rcs.mie_backscatter_sphere(3.0, lmax=40) - rcs.mie_backscatter_sphere(3.0, lmax=60)) < 1e-13
    for ka in (1e-2, 1e-3):
        f = rcs.mie_backscatter_sphere(ka)
        assert abs(f - (-math.sin(ka) * np.exp(-1j * ka) / ka)) < 10 * ka ** 2
