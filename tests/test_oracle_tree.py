"""Pins for oracle/tree.py: SPEC examples and brute-force geometric
checks in REAL coordinates (independent of the integer cell logic)."""
import numpy as np
import pytest

import fmmlu_inputs as fi
from oracle.tree import Tree, DepthExceeded


def _real_box(t, b):
    h = t.box_side(t.level[b])
    lo = t.lo + np.asarray(t.coord[b], float) * h
    return lo, lo + h


def _gap(t, a, b):
    la, ha = _real_box(t, a)
    lb, hb = _real_box(t, b)
    return float(np.max(np.maximum(lb - ha, la - hb)))


def test_cube_corners_depth1():
    g = fi.cube_corners()
    t = Tree(g.points, 1)
    assert t.nlevels == 2
    leaves = [b for b in range(len(t.level)) if t.is_leaf(b)]
    assert len(leaves) == 8 and all(t.level[b] == 1 for b in leaves)


def test_single_leaf_when_s_ge_n():
    g = fi.fibonacci_sphere(50)
    t = Tree(g.points, 50)
    assert t.nlevels == 1 and t.is_leaf(0)


def test_duplicate_points_depth_exceeded():
    pts = np.zeros((5, 3))
    pts[:, 0] = 1.0
    pts[0] = [0.0, 0.0, 0.0]
    with pytest.raises(DepthExceeded):
        Tree(pts, 2)


def _multiscale():
    return fi.bump_sphere(n_base=3000, n_cap=1500, theta_c=0.05, height=0.02)


@pytest.mark.parametrize("bal", [False, True])
def test_partition_and_occupancy(bal):
    g = _multiscale()
    t = Tree(g.points, 16, balance=bal)
    leaves = [b for b in range(len(t.level)) if t.is_leaf(b)]
    cover = np.zeros(t.n, int)
    for b in leaves:
        assert t.end[b] - t.start[b] <= 16
        cover[t.start[b]:t.end[b]] += 1
    assert np.all(cover == 1)
    # points lie inside their leaf (real coordinates, half-open boxes)
    X = g.points[t.perm]
    for b in leaves:
        lo, hi = _real_box(t, b)
        p = X[t.start[b]:t.end[b]]
        assert np.all(p >= lo - 1e-12) and np.all(p <= hi + 1e-12)
    for b in range(len(t.level)):
        if t.children[b]:
            assert sum(t.end[c] - t.start[c] for c in t.children[b]) == t.end[b] - t.start[b]


def test_two_to_one_balance_bruteforce():
    g = _multiscale()
    t0 = Tree(g.points, 16, balance=False)
    t = Tree(g.points, 16, balance=True)

    def violations(tt):
        leaves = [b for b in range(len(tt.level)) if tt.is_leaf(b)]
        v = 0
        tol = 1e-9 * tt.side
        for i, a in enumerate(leaves):
            for b in leaves[i + 1:]:
                if _gap(tt, a, b) <= tol and abs(tt.level[a] - tt.level[b]) > 1:
                    v += 1
        return v

    assert violations(t0) > 0          # the multiscale input needs balancing
    assert violations(t) == 0
    assert len(t.level) > len(t0.level)


def test_near_q_far_lists_bruteforce():
    """N = owners touching B, Q = owners at real gap exactly one box side, P = gap ≥ 2 sides;
    disjoint cover of all owners (reading C6/C7)."""
    g = _multiscale()
    t = Tree(g.points, 16)
    X = g.points[t.perm]
    for lvl in range(2, t.nlevels):
        owners = t.owners(lvl)
        h = t.box_side(lvl)
        tol = 1e-9 * h
        for B in t.levels[lvl][::3]:
            N, Q = t.near_q(B)
            bN, bQ, bP = set(), set(), set()
            for o in owners:
                if o == B:
                    continue
                gp = _gap(t, B, o)
                if gp <= tol:
                    bN.add(o)
                elif gp <= h + tol:
                    bQ.add(o)
                else:
                    assert gp >= 2 * h - tol
                    bP.add(o)
            assert set(N) == bN and set(Q) == bQ
            # every P point is outside the proxy sphere of radius 2h (reading C5)
            c = t.box_centre(B)
            for o in bP:
                p = X[t.start[o]:t.end[o]]
                assert np.min(np.linalg.norm(p - c, axis=1)) > 2.0 * h
