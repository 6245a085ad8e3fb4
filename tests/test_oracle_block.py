"""Pins for the oracle's block mode and order self-checks ("two interchangeable
modes; both must give identical S/T", the sequential-order self-check C8/P5).

* Block mode (current entry = pure kernel + Δ keyed by owner pair) against dense mode (the
  literal n×n matrix): identical skeleton set for every box, identical root size, solutions
  equal to rounding.  The cases cover several levels, coarse-leaf owners under 2:1 balance
  (bump sphere) and the Q rows of same-colour boxes eliminated earlier in the phase.
* Reading C8: reversing the order inside every colour phase changes nothing but the
  summation order (identical skeletons, solutions equal to rounding); the plain sequential
  sweep of PAPER.md L878-884 (each box sees the actives as they are when it is processed) is
  an equally valid ε-factorization: residual ≤ 10ε, within 10ε of the dense LU solve.
"""
import math

import numpy as np
import pytest

import fmmlu_inputs as fi
from oracle import dense, rss


def _cases():
    return {
        "ellipsoid2000": (fi.ellipsoid(2000), 2 * math.pi, 24),
        "bump3000": (fi.bump_sphere(2000, 1000, 0.05, 0.02), 5.0, 16),
    }


@pytest.fixture(scope="module")
def cases():
    out = {}
    for name, (g, k, leaf) in _cases().items():
        b = fi.gaussian_rhs(g.n, 2, 0)
        f = rss.factor(g.points, g.normals, g.weights, k, 1e-6, leaf, mode="block")
        out[name] = (g, k, leaf, b, f, rss.solve(f, b))
    return out


@pytest.mark.parametrize("name", ["ellipsoid2000", "bump3000"])
def test_block_mode_equals_dense_mode(cases, name):
    g, k, leaf, b, fb, xb = cases[name]
    fd = rss.factor(g.points, g.normals, g.weights, k, 1e-6, leaf, mode="dense")
    xd = rss.solve(fd, b)
    assert len(fd.records) > 0
    assert fd.stats["skeletons"].keys() == fb.stats["skeletons"].keys()
    for B, s in fd.stats["skeletons"].items():
        assert np.array_equal(s, fb.stats["skeletons"][B]), B
    assert fd.stats["n0"] == fb.stats["n0"]
    for rd, rb in zip(fd.records, fb.records):
        assert rd.box == rb.box and np.array_equal(rd.Bs, rb.Bs)
        assert np.abs(rd.T - rb.T).max() <= 1e-9 * max(1.0, np.abs(rd.T).max())
    assert dense.rel_diff(xb, xd) < 1e-11


@pytest.mark.parametrize("name", ["ellipsoid2000", "bump3000"])
def test_order_inside_colour_is_irrelevant(cases, name):
    g, k, leaf, b, f0, x0 = cases[name]
    f = rss.factor(g.points, g.normals, g.weights, k, 1e-6, leaf, mode="block", order="colour_reversed")
    for B, s in f0.stats["skeletons"].items():
        assert np.array_equal(s, f.stats["skeletons"][B]), B
    assert dense.rel_diff(rss.solve(f, b), x0) < 1e-11


def test_sequential_sweep_is_an_equally_valid_factorization(cases):
    g, k, leaf, b, f0, x0 = cases["ellipsoid2000"]
    eps = 1e-6
    f = rss.factor(g.points, g.normals, g.weights, k, eps, leaf, mode="block", order="sequential")
    x = rss.solve(f, b)
    assert dense.residual(g.points, g.normals, g.weights, k, x, b) <= 10 * eps
    xd = dense.dense_solve(g.points, g.normals, g.weights, k, b)
    assert dense.rel_diff(x, xd) <= 10 * eps
    assert dense.rel_diff(x, x0) <= 10 * eps
    # same tree and boxes; skeletons differ only where a box saw different (later) actives
    assert f.stats["skeletons"].keys() == f0.stats["skeletons"].keys()
    assert abs(f.stats["n0"] - f0.stats["n0"]) <= 0.05 * f0.stats["n0"]


def test_block_state_holds_only_updated_pairs():
    """The Δ dict is sparse: after a level, only owner pairs inside some box's {B} ∪ N(B) have
    blocks (the pair-list structure of PAPER.md L1296-1307)."""
    g = fi.ellipsoid(3000)
    seen = {}

    class Spy(rss.BlockState):
        def begin_level(self, owners, active, parent_of):
            super().begin_level(owners, active, parent_of)
            lvl = max(f_tree[0].level[o] for o in owners)
            seen.setdefault("keys", []).append((lvl, set(self.D)))

    from oracle.tree import Tree
    f_tree = [Tree(g.points, 32)]
    orig = rss.BlockState
    rss.BlockState = Spy
    try:
        f = rss.factor(g.points, g.normals, g.weights, 2 * math.pi, 1e-6, 32, mode="block")
    finally:
        rss.BlockState = orig
    assert len(f.records) > 0
    t = f.tree
    assert any(keys for _, keys in seen["keys"])
    for lvl, keys in seen["keys"]:
        for a, b in keys:
            # an update at level ℓ+1 joins two owners touching one box (separation ≤ 2 cells);
            # re-keyed to level ℓ they touch (reading C6's sufficiency argument)
            assert t.sep(a, b, lvl) <= 1, (lvl, a, b)
