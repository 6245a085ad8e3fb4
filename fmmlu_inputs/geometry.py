"""Deterministic surface point clouds with outward unit normals and smooth
quadrature weights (the x_i, n(x_i), w_i of PAPER.md L443-456 Eq. disc1).

All recipes are the SURVEY.md §8(d) table (reading C15):

* cfg1  unit sphere, Fibonacci lattice, n=2000, w=4π/n.
* cfg2  ellipsoid with semi-axes (0.5, 1, 2), n=20000, x = diag(a)u with u on the
        Fibonacci sphere, normal ∝ u/a, w = (4π/n)·abc·|u/a|.
* cfg3  unit sphere plus a C¹ bump r(θ)=1+0.01(1-(θ/0.01)²)² at the north pole,
        80,000 base points outside the cap + 20,000 cap points (100× finer spacing).
* cfg5  wavy torus, periodic 2000×500 grid, n = 10⁶.

Geometry is input data, not method arithmetic: the oracle and the CUDA path both
consume these arrays unchanged.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

GOLDEN_ANGLE = math.pi * (3.0 - math.sqrt(5.0))


@dataclasses.dataclass
class Geometry:
    """n points (n×3), unit outward normals (n×3), positive weights (n,), all fp64."""

    points: np.ndarray
    normals: np.ndarray
    weights: np.ndarray
    name: str = ""

    @property
    def n(self) -> int:
        return int(self.points.shape[0])

    def __post_init__(self):
        self.points = np.ascontiguousarray(self.points, dtype=np.float64)
        self.normals = np.ascontiguousarray(self.normals, dtype=np.float64)
        self.weights = np.ascontiguousarray(self.weights, dtype=np.float64)


def _fib_unit(n: int) -> np.ndarray:
    i = np.arange(n, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / n
    phi = i * GOLDEN_ANGLE
    s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return np.stack([s * np.cos(phi), s * np.sin(phi), z], axis=1)


def fibonacci_sphere(n: int, radius: float = 1.0) -> Geometry:
    """cfg1: z_i = 1-(2i+1)/n, φ_i = i·π(3-√5); n_i = x_i/|x_i|; w_i = 4πR²/n."""
    u = _fib_unit(n)
    return Geometry(radius * u, u.copy(), np.full(n, 4.0 * math.pi * radius**2 / n), f"sphere{n}")


def ellipsoid(n: int, axes=(0.5, 1.0, 2.0)) -> Geometry:
    """cfg2: x = diag(a)u, u Fibonacci; normal ∝ u/a; w = (4π/n)·abc·|u/a|
    (surface Jacobian of the linear map diag(a) restricted to the unit sphere)."""
    a = np.asarray(axes, dtype=np.float64)
    u = _fib_unit(n)
    x = u * a
    g = u / a
    gn = np.linalg.norm(g, axis=1)
    w = (4.0 * math.pi / n) * float(np.prod(a)) * gn
    return Geometry(x, g / gn[:, None], w, f"ellipsoid{n}")


def bump_sphere(n_base: int = 80_000, n_cap: int = 20_000, theta_c: float = 0.01,
                height: float = 0.01) -> Geometry:
    """cfg3: unit sphere with a C¹ bump r(θ) = 1 + h(1-(θ/θc)²)² for θ < θc.

    Base: a Fibonacci spiral uniform in z over the band z ∈ [-1, cos θc];
    cap: a Fibonacci spiral uniform in u = cos θ over [cos θc, 1] (100× finer
    spacing at the default sizes).  Weights = area element × region area / count.
    Normals of the surface of revolution: n ∝ r e_r − r'(θ) e_θ.
    """
    zc = math.cos(theta_c)
    # base band
    i = np.arange(n_base, dtype=np.float64)
    z = -1.0 + (1.0 + zc) * (i + 0.5) / n_base
    phi = i * GOLDEN_ANGLE
    s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    xb = np.stack([s * np.cos(phi), s * np.sin(phi), z], axis=1)
    wb = np.full(n_base, 2.0 * math.pi * (1.0 + zc) / n_base)
    # cap
    j = np.arange(n_cap, dtype=np.float64)
    u = 1.0 - (1.0 - zc) * (j + 0.5) / n_cap
    th = np.arccos(u)
    ph = j * GOLDEN_ANGLE
    t = th / theta_c
    r = 1.0 + height * (1.0 - t * t) ** 2
    dr = height * 2.0 * (1.0 - t * t) * (-2.0 * th / theta_c**2)
    st, ct = np.sin(th), np.cos(th)
    er = np.stack([st * np.cos(ph), st * np.sin(ph), ct], axis=1)
    eth = np.stack([ct * np.cos(ph), ct * np.sin(ph), -st], axis=1)
    xc = r[:, None] * er
    nc = r[:, None] * er - dr[:, None] * eth
    nc /= np.linalg.norm(nc, axis=1)[:, None]
    wc = (2.0 * math.pi * (1.0 - zc) / n_cap) * r * np.sqrt(r * r + dr * dr)
    return Geometry(np.vstack([xb, xc]), np.vstack([xb, nc]), np.concatenate([wb, wc]),
                    f"bump{n_base + n_cap}")


def wavy_torus(nt: int = 2000, npol: int = 500) -> Geometry:
    """cfg5: X(θ,φ) = ((2 + r cos φ)cos θ, (2 + r cos φ) sin θ, r sin φ),
    r = 0.5 + 0.1 cos(5θ) cos(3φ); periodic trapezoid grid; w = |X_θ × X_φ| ΔθΔφ."""
    th = 2.0 * math.pi * np.arange(nt) / nt
    ph = 2.0 * math.pi * np.arange(npol) / npol
    T, P = np.meshgrid(th, ph, indexing="ij")
    T = T.ravel()
    P = P.ravel()
    r = 0.5 + 0.1 * np.cos(5 * T) * np.cos(3 * P)
    rt = -0.5 * np.sin(5 * T) * np.cos(3 * P)
    rp = -0.3 * np.cos(5 * T) * np.sin(3 * P)
    R = 2.0 + r * np.cos(P)
    x = np.stack([R * np.cos(T), R * np.sin(T), r * np.sin(P)], axis=1)
    Xt = np.stack([rt * np.cos(P) * np.cos(T) - R * np.sin(T),
                   rt * np.cos(P) * np.sin(T) + R * np.cos(T),
                   rt * np.sin(P)], axis=1)
    A = rp * np.cos(P) - r * np.sin(P)
    Xp = np.stack([A * np.cos(T), A * np.sin(T), rp * np.sin(P) + r * np.cos(P)], axis=1)
    nrm = np.cross(Xt, Xp)
    jac = np.linalg.norm(nrm, axis=1)
    w = jac * (2.0 * math.pi / nt) * (2.0 * math.pi / npol)
    return Geometry(x, nrm / jac[:, None], w, f"torus{nt * npol}")


def cube_corners() -> Geometry:
    """Tiny-ladder rung T1: the 8 corners of [-1,1]³, outward (diagonal) normals."""
    c = np.array([[sx, sy, sz] for sx in (-1.0, 1.0) for sy in (-1.0, 1.0) for sz in (-1.0, 1.0)])
    return Geometry(c, c / math.sqrt(3.0), np.full(8, 0.5))


def random_cube(n: int, seed: int = 0, side: float = 1.0) -> Geometry:
    """Tiny-ladder rung T3: uniform random points in a cube with random unit normals."""
    rng = np.random.default_rng(seed)
    x = (rng.random((n, 3)) - 0.5) * side
    nv = rng.standard_normal((n, 3))
    nv /= np.linalg.norm(nv, axis=1)[:, None]
    return Geometry(x, nv, np.full(n, side * side / n))


# name -> (geometry factory, k, leaf_max, eps, nrhs)  (BASELINE.json configs)
CONFIGS = {
    "cfg1": dict(make=lambda: fibonacci_sphere(2000), k=1.0, leaf_max=64, eps=1e-6, nrhs=1),
    "cfg2": dict(make=lambda: ellipsoid(20_000), k=2.0 * math.pi, leaf_max=64, eps=1e-6, nrhs=4),
    "cfg3": dict(make=lambda: bump_sphere(), k=5.0, leaf_max=64, eps=1e-6, nrhs=16),
    "cfg5": dict(make=lambda: wavy_torus(), k=10.0, leaf_max=64, eps=1e-6, nrhs=32),
}


def config_geometry(name: str) -> Geometry:
    g = CONFIGS[name]["make"]()
    g.name = name
    return g
