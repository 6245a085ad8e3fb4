"""Full-size GPU parity on BASELINE.json configs 1, 2, 3 and 5 (north_star: "matching the CPU
oracle's solutions within 10ε and residual ≤ 10ε on all five configs"; cfg4 is in
tests/test_gpu_boxes.py).

* Expected solutions (cfg1, cfg2, cfg3) were written by tools/make_golden.py, which calls only
  oracle/ (dense AND block mode for cfg1/cfg2, asserting identical skeletons; block mode for
  cfg3) on the same seeded inputs (fmmlu_inputs, reading C16).  Solution parity is
  ‖x_gpu − x_oracle‖/‖x_oracle‖ ≤ 10ε per RHS column (reading C17), in full where the file
  stores whole columns and, for the remaining cfg3 columns, estimated from the stored sample
  of entries (sqrt(n/m·Σ|d_i|²)/‖x_oracle‖).
* Residuals ‖Ax − b‖/‖b‖ are estimated from rows of A computed one by one with the ORACLE
  kernel (oracle/kernel.py, independent of libfmmlu's matvec): for m seeded rows i,
  r_i = Σ_j K(x_i,x_j) w_j x_j + ½x_i − b_i, ‖r‖ ≈ sqrt(n/m·Σ r_i²).  The dense oracle
  cannot hold cfg5 (n = 10⁶; SURVEY §8(c) block mode would need ≈ 90 GB of host RAM), so
  cfg5 is judged by this residual at its full 32 RHS (the GEMM-sweep solve path).
"""
import os

import numpy as np
import pytest

import fmmlu_inputs as fi
from oracle import kernel as okern

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def F():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2201_07325_b200 import fmmlu
    fmmlu.load()
    return fmmlu


def _solve(F, name):
    c = fi.CONFIGS[name]
    g = fi.config_geometry(name)
    b = fi.gaussian_rhs(g.n, c["nrhs"], 0)
    h = F.FmmLu(g.points, g.normals, g.weights, c["leaf_max"]).factor(c["k"], c["eps"])
    x = np.asfortranarray(b.copy())
    h.solve(x)
    st = h.stats()
    h.close()
    return c, g, b, x, st


def sampled_residual(g, k, x, b, m, seed=11):
    """Estimate of max over columns of ‖Ax − b‖/‖b‖ from m rows of A evaluated with the oracle
    kernel (A = ½I + K W, K_ii = 0, BASELINE.json)."""
    rows = np.sort(np.random.default_rng(seed).choice(g.n, m, replace=False))
    wx = g.weights[:, None] * x
    r = np.empty((m, x.shape[1]), dtype=np.complex128)
    for t, i in enumerate(rows):
        with np.errstate(divide="ignore", invalid="ignore"):
            Ki = okern.combined_field(k, g.points[i:i + 1], g.points, g.normals)[0]
        Ki[i] = 0.0
        r[t] = Ki @ wx + 0.5 * x[i] - b[i]
    est = np.sqrt(g.n / m * np.sum(np.abs(r) ** 2, axis=0)) / np.linalg.norm(b, axis=0)
    return float(est.max())


def _gold(name):
    import json
    d = np.load(os.path.join(GOLD, f"{name}_oracle_solution.npz"))
    meta = json.load(open(os.path.join(GOLD, f"{name}_oracle_solution.json")))
    return d, meta


def _col_rel(x, xo):
    return float(np.max(np.linalg.norm(x - xo, axis=0) / np.linalg.norm(xo, axis=0)))


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_full_size_solution_parity_small(F, name):
    c, g, b, x, st = _solve(F, name)
    d, meta = _gold(name)
    eps = c["eps"]
    assert d["x_full"].shape == x.shape
    assert _col_rel(x, d["x_full"]) <= 10 * eps
    assert sampled_residual(g, c["k"], x, b, 256) <= 10 * eps
    # structural parity (P8): root size within a few percent of the oracle's
    assert abs(st["n0"] - meta["n0"]) <= 0.05 * meta["n0"] + 2


def test_cfg3_full_size_solution_parity(F):
    """BASELINE configs[2] (multiscale bump sphere, n = 10⁵, 12 levels, 16 RHS) against the
    block-mode oracle."""
    c, g, b, x, st = _solve(F, "cfg3")
    d, meta = _gold("cfg3")
    eps = c["eps"]
    assert _col_rel(x[:, :2], d["x_full"]) <= 10 * eps
    idx = d["sample_idx"]
    diff = x[idx] - d["x_sample"]
    est = np.sqrt(g.n / idx.size * np.sum(np.abs(diff) ** 2, axis=0)) / d["colnorm"]
    assert est.max() <= 10 * eps, est
    assert sampled_residual(g, c["k"], x, b, 128) <= 10 * eps
    assert abs(st["n0"] - meta["n0"]) <= 0.05 * meta["n0"] + 2
    for lvl, r in meta["ranks_sum"].items():
        assert abs(st["ranks_sum"][int(lvl)] - r) <= 0.03 * r + 2, (lvl, st["ranks_sum"][int(lvl)], r)


def test_cfg5_full_size_residual_32rhs(F):
    """BASELINE configs[4] (wavy torus, n = 10⁶) at its full 32 RHS: residual ≤ 10ε from rows of
    A evaluated by the oracle kernel."""
    c, g, b, x, st = _solve(F, "cfg5")
    assert c["nrhs"] == 32 and x.shape == (10 ** 6, 32)
    assert st["n_eliminated"] > 0 and st["n0"] < g.n // 50
    assert sampled_residual(g, c["k"], x, b, 96) <= 10 * c["eps"]
