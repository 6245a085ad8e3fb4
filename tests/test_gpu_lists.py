"""a2 on the device (readings C6-C8): the owner
lists built by the device kernels (devtree.cu: owners = level boxes + coarser leaves, N = owners at
separation ≤ 1, Q = separation 2) against the oracle's tree, box by box, on trees with coarse-leaf
owners (adaptive, 2:1 balanced) and on a uniform one.  Integer work: exact equality."""
import os

import numpy as np
import pytest

import fmmlu_inputs as fi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2201_07325_b200 import fmmlu
    fmmlu.load()
    return fmmlu


def _geo(case):
    if case == "bump":
        return fi.bump_sphere(n_base=3000, n_cap=1500, theta_c=0.05, height=0.02), 16
    if case == "cube":
        return fi.random_cube(2000, seed=3), 8
    if case == "ellipsoid":
        return fi.ellipsoid(6000), 8
    return fi.config_geometry("cfg1"), 64


@pytest.mark.parametrize("case", ["bump", "cube", "ellipsoid", "cfg1"])
def test_device_owner_lists_equal_oracle(F, case):
    from oracle.tree import Tree
    g, s = _geo(case)
    h = F.FmmLu(g.points, g.normals, g.weights, s)
    t = Tree(g.points, s)
    d = h.tree_boxes()
    key = [(int(l),) + tuple(int(x) for x in c) for l, c in zip(d["level"], d["coord"])]  # GPU box id -> cell
    okey = {b: (t.level[b],) + tuple(int(x) for x in t.coord[b]) for b in range(len(t.level))}
    checked = coarse = 0
    for lvl in range(2, t.nlevels):
        L = h.level_lists(lvl)
        own = [key[b] for b in L["owners"]]
        assert own == [okey[b] for b in t.owners(lvl)]          # same owners, same order
        coarse += sum(1 for k in own if k[0] < lvl)
        for j, B in enumerate(t.levels[lvl]):
            assert own[j] == okey[B]
            Nl, Ql = t.near_q(B)
            n_gpu = L["nidx"][L["nptr"][j]:L["nptr"][j + 1]]
            q_gpu = L["qidx"][L["qptr"][j]:L["qptr"][j + 1]]
            assert np.all(np.diff(n_gpu) > 0) and np.all(np.diff(q_gpu) > 0)      # ascending, unique
            assert {own[o] for o in n_gpu} == {okey[o] for o in Nl}
            assert {own[o] for o in q_gpu} == {okey[o] for o in Ql}
            # colour (reading C8): parity of the cell coordinates, as the oracle's
            c = own[j][1:]
            assert 4 * (c[0] & 1) + 2 * (c[1] & 1) + (c[2] & 1) == t.colour(B)
            checked += 1
    assert checked > 0
    if case in ("bump", "cube"):
        assert coarse > 0     # the adaptive cases do have coarser-leaf owners


def test_device_pair_set_matches_host_check(F, monkeypatch):
    """The block-pair set (and all lists) of every level against the library's host-tree self-check
    (FMMLU_TOPO_CHECK: a mismatch makes fmmlu_factor fail), on an adaptive tree; the factorization
    then matches the dense solve."""
    import math
    from oracle import dense
    monkeypatch.setenv("FMMLU_TOPO_CHECK", "1")
    g = fi.bump_sphere(n_base=3000, n_cap=1500, theta_c=0.05, height=0.02)
    k, eps = 2.0, 1e-6
    b = fi.gaussian_rhs(g.n, 2, 0)
    h = F.FmmLu(g.points, g.normals, g.weights, 24).factor(k, eps)
    x = np.asfortranarray(b.copy())
    h.solve(x)
    xd = dense.dense_solve(g.points, g.normals, g.weights, k, b)
    assert dense.rel_diff(x, xd) <= 10 * eps
