"""Oracle: azimuthal monostatic sonar cross section (test infrastructure only).

PAPER.md §6.3 (L2755-2794), sound-soft scatterer:
* incident plane wave along d = (cos φ₀, sin φ₀, 0); the density solves
  ½σ + ∫_Γ K σ da = −e^{ik x·d}   (L2782-2785), i.e. A σ = b with BASELINE.json's A and
  b_i = −e^{ik x_i·d}  (``plane_wave_rhs``);
* R(φ₀) = F[u_{φ₀}] in the backscatter direction x̂ = −d (L2773-2776), with the far-field
  convention u = (e^{ikr}/r) F + O(r⁻²) (L2766-2768).  For the combined layer
  u = D[σ] − ikS[σ] the far field is F(x̂) = (−ik/4π) ∫ (1 + x̂·n(y)) e^{−ik x̂·y} σ(y) da(y),
  so at x̂ = −d:  R(φ₀) = (−ik/4π) ∫ (1 − n·d) e^{+ik x·d} σ da  (reading R8 in DESIGN.md:
  L2788-2792 prints e^{−ik x·d}; the backscatter asymptotics fix the + sign, and the Mie pin
  below fails with the printed sign).  Discretized with the quadrature weights w_j
  (``monostatic_rcs``).

Pins (tests/test_oracle_rcs.py): the Mie series of the sound-soft sphere
(``mie_backscatter_sphere``, an independent closed form: partial waves with spherical Bessel
functions) matched by dense-solve + ``monostatic_rcs`` on Fibonacci spheres with an error that
decreases under refinement (the O(h) Nyström rule of reading C19); rotational invariance of
R on the sphere; the RHS is a unit-modulus plane wave.
"""
from __future__ import annotations

import math

import numpy as np
from scipy import special


def directions(phis) -> np.ndarray:
    """d_a = (cos φ_a, sin φ_a, 0), a = 0..len(phis)−1."""
    phis = np.asarray(phis, dtype=np.float64)
    return np.stack([np.cos(phis), np.sin(phis), np.zeros_like(phis)], axis=1)


def plane_wave_rhs(points, k: float, phis) -> np.ndarray:
    """b[:, a] = −e^{ik x·d_a}  (n × nphi complex128)."""
    x = np.asarray(points, dtype=np.float64)
    return -np.exp(1j * k * (x @ directions(phis).T))


def monostatic_rcs(points, normals, weights, k: float, phis, sigma) -> np.ndarray:
    """R(φ_a) = (−ik/4π) Σ_j w_j (1 − n_j·d_a) e^{ik x_j·d_a} σ_ja   (reading R8)."""
    x = np.asarray(points, dtype=np.float64)
    nrm = np.asarray(normals, dtype=np.float64)
    w = np.asarray(weights, dtype=np.float64)
    d = directions(phis)
    f = (1.0 - nrm @ d.T) * np.exp(1j * k * (x @ d.T)) * w[:, None]
    return (-1j * k / (4.0 * math.pi)) * np.sum(f * np.asarray(sigma).reshape(len(w), -1), axis=0)


def mie_backscatter_sphere(k: float, a: float = 1.0, lmax: int | None = None) -> complex:
    """Backscatter far-field amplitude of a sound-soft sphere of radius a for the incident wave
    e^{ik x·d}:  u_s = −Σ_l i^l (2l+1) (j_l(ka)/h_l(ka)) h_l(kr) P_l(cos γ), h_l ~ (−i)^{l+1}e^{ikr}/(kr)
    ⇒ F(x̂) = (i/k) Σ_l (2l+1) (j_l(ka)/h_l(ka)) P_l(x̂·d), and P_l(−1) = (−1)^l at x̂ = −d."""
    ka = k * a
    if lmax is None:
        lmax = int(ka + 4 * ka ** (1 / 3) + 20)
    s = 0j
    for l in range(lmax + 1):
        jl = special.spherical_jn(l, ka)
        hl = jl + 1j * special.spherical_yn(l, ka)
        s += (2 * l + 1) * (-1) ** l * jl / hl
    return 1j / k * s
