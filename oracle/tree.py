"""Oracle: adaptive level-restricted octree, owners, near/far lists, colours
(test infrastructure only).

PAPER.md L551-562 (§4): root cube C is level 0; a box at level l is split into 8
equal children while it holds more than s points; empty children are dropped
(reading C14).  PAPER.md L563-565: near field = boxes touching B, far field = the
rest.  PAPER.md L567-576: level restriction — two leaves that share a boundary
point differ by at most one level (enforced by splitting the coarser leaf until a
fixed point).  PAPER.md L1263-1276 (§4.4) with the 3D correction of reading C6:
Q(B) = owners meeting B's 5×5×5 block of level-ℓ cells minus N(B); P = the rest.
Reading C7: the owners at level ℓ are the level-ℓ boxes plus the leaves of
coarser levels; membership is per owner by extent.  Reading C8: colour =
4(i_x&1) + 2(i_y&1) + (i_z&1).

Reading C14 (quantisation): root cube centred at the bounding-box centre with
side = max extent·(1+1e-12); each coordinate is quantised once to
q = floor((x−lo)/side·2^20) (clipped to [0, 2^20−1]) and a point lies in the child
given by the next bit of q.  Tree order = stable sort by the 60-bit Morton key of q,
so every box is a contiguous range.  Depth cap 20 (DepthExceeded).

Pins (tests/test_oracle_tree.py): 8 cube corners with s=1 → depth 1;
s ≥ n → single leaf; every leaf holds ≤ s points; the 2:1 property by a
brute-force O(#leaves²) geometric scan in real coordinates; N/Q/P by a
brute-force distance test on box extents in real coordinates; disjoint cover.
"""
from __future__ import annotations

import numpy as np

DEPTH = 20


class DepthExceeded(RuntimeError):
    pass


def morton60(q: np.ndarray) -> np.ndarray:
    """Interleave 20 bits of (qx, qy, qz): bit b of x → 3b+2, of y → 3b+1, of z → 3b."""
    q = q.astype(np.uint64)
    key = np.zeros(q.shape[0], dtype=np.uint64)
    for b in range(DEPTH):
        for axis, off in ((0, 2), (1, 1), (2, 0)):
            key |= ((q[:, axis] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + off)
    return key


class Tree:
    """Boxes are stored in flat lists; ``self.by_key[(level, cx, cy, cz)] = box id``."""

    def __init__(self, points: np.ndarray, leaf_max: int, balance: bool = True):
        pts = np.asarray(points, dtype=np.float64)
        n = pts.shape[0]
        if n < 1 or leaf_max < 1:
            raise ValueError("n >= 1 and leaf_max >= 1 required")
        mn, mx = pts.min(axis=0), pts.max(axis=0)
        centre = 0.5 * (mn + mx)
        side = float(np.max(mx - mn)) * (1.0 + 1e-12)
        if side <= 0.0:
            side = 1.0
        self.side = side
        self.lo = centre - 0.5 * side
        scale = float(1 << DEPTH)
        q = np.floor((pts - self.lo) / side * scale)
        q = np.clip(q, 0, (1 << DEPTH) - 1).astype(np.int64)
        key = morton60(q)
        self.perm = np.argsort(key, kind="stable")
        self.q = q[self.perm]
        self.key = key[self.perm]
        self.n = n
        self.leaf_max = leaf_max
        # box arrays
        self.level, self.coord, self.start, self.end = [], [], [], []
        self.parent, self.children = [], []
        self.by_key = {}
        self._add(0, (0, 0, 0), 0, n, -1)
        frontier = [0]
        while frontier:
            nxt = []
            for b in frontier:
                if self.end[b] - self.start[b] > leaf_max:
                    if self.level[b] >= DEPTH:
                        raise DepthExceeded("duplicate points force refinement past depth 20")
                    nxt.extend(self._split(b))
            frontier = nxt
        if balance:
            self._balance()
        self.nlevels = max(self.level) + 1
        self.levels = [sorted([b for b in range(len(self.level)) if self.level[b] == l],
                              key=lambda b: self._mcode(b))
                       for l in range(self.nlevels)]

    # ---------------------------------------------------------------- build
    def _add(self, level, coord, s, e, parent):
        bid = len(self.level)
        self.level.append(level)
        self.coord.append(tuple(int(c) for c in coord))
        self.start.append(s)
        self.end.append(e)
        self.parent.append(parent)
        self.children.append([])
        self.by_key[(level,) + tuple(int(c) for c in coord)] = bid
        return bid

    def _split(self, b):
        """Split box b into its non-empty octants (contiguous ranges in tree order)."""
        l = self.level[b]
        s, e = self.start[b], self.end[b]
        sh = DEPTH - 1 - l
        qs = self.q[s:e]
        octant = ((qs[:, 0] >> sh) & 1) * 4 + ((qs[:, 1] >> sh) & 1) * 2 + ((qs[:, 2] >> sh) & 1)
        kids = []
        cx, cy, cz = self.coord[b]
        for o in range(8):
            idx = np.nonzero(octant == o)[0]
            if idx.size == 0:
                continue
            assert idx[-1] - idx[0] + 1 == idx.size  # contiguity of Morton order
            c = (2 * cx + (o >> 2), 2 * cy + ((o >> 1) & 1), 2 * cz + (o & 1))
            kids.append(self._add(l + 1, c, s + int(idx[0]), s + int(idx[-1]) + 1, b))
        self.children[b] = kids
        return kids

    def is_leaf(self, b):
        return not self.children[b]

    def _balance(self):
        """Split leaves until no two touching leaves differ by more than one level."""
        changed = True
        while changed:
            changed = False
            leaves = [b for b in range(len(self.level)) if self.is_leaf(b)]
            to_split = set()
            for y in leaves:
                ly = self.level[y]
                yc = self.coord[y]
                for m in range(0, ly - 1):
                    d = ly - m
                    rng = []
                    for a in range(3):
                        lo = -((-yc[a]) >> d) - 1  # ceil(y/2^d) - 1
                        hi = (yc[a] + 1) >> d      # floor((y+1)/2^d)
                        rng.append(range(max(lo, 0), min(hi, (1 << m) - 1) + 1))
                    for x0 in rng[0]:
                        for x1 in rng[1]:
                            for x2 in rng[2]:
                                xb = self.by_key.get((m, x0, x1, x2))
                                if xb is not None and self.is_leaf(xb):
                                    to_split.add(xb)
            for xb in sorted(to_split):
                if self.is_leaf(xb):
                    self._split(xb)
                    changed = True

    def _mcode(self, b):
        l = self.level[b]
        c = self.coord[b]
        key = 0
        for bit in range(l):
            key |= ((c[0] >> bit) & 1) << (3 * bit + 2)
            key |= ((c[1] >> bit) & 1) << (3 * bit + 1)
            key |= ((c[2] >> bit) & 1) << (3 * bit)
        return key

    # ---------------------------------------------------------------- geometry
    def box_side(self, level):
        return self.side / (1 << level)

    def box_centre(self, b):
        h = self.box_side(self.level[b])
        return self.lo + (np.asarray(self.coord[b], dtype=np.float64) + 0.5) * h

    def colour(self, b):
        c = self.coord[b]
        return 4 * (c[0] & 1) + 2 * (c[1] & 1) + (c[2] & 1)

    # ---------------------------------------------------------------- owners
    def owners(self, level):
        """Level-ℓ owners: level-ℓ boxes plus leaves of coarser levels (reading C7)."""
        own = list(self.levels[level]) if level < self.nlevels else []
        for m in range(min(level, self.nlevels)):
            own.extend(b for b in self.levels[m] if self.is_leaf(b))
        return own

    def owner_of_cell(self, level, c):
        """The level-ℓ owner covering level-ℓ cell c, or None (empty region)."""
        b = self.by_key.get((level,) + tuple(c))
        if b is not None:
            return b
        for m in range(level - 1, -1, -1):
            d = level - m
            b = self.by_key.get((m, c[0] >> d, c[1] >> d, c[2] >> d))
            if b is not None:
                return b if self.is_leaf(b) else None
        return None

    def extent(self, b, level):
        """Inclusive level-ℓ cell range [lo, hi] per axis of owner b."""
        d = level - self.level[b]
        c = np.asarray(self.coord[b], dtype=np.int64)
        return c << d, ((c + 1) << d) - 1

    def sep(self, a, b, level):
        lo_a, hi_a = self.extent(a, level)
        lo_b, hi_b = self.extent(b, level)
        return int(np.max(np.maximum(lo_b - hi_a, lo_a - hi_b)))

    def near_q(self, B):
        """(N(B), Q(B)) owner lists for a level-ℓ box B, ℓ = level(B) (readings C6/C7).
        N: owners ≠ B with sep ≤ 1 (touching); Q: sep == 2.  Sorted by box id."""
        level = self.level[B]
        c = self.coord[B]
        lim = (1 << level) - 1
        found = set()
        for dx in range(-2, 3):
            for dy in range(-2, 3):
                for dz in range(-2, 3):
                    cc = (c[0] + dx, c[1] + dy, c[2] + dz)
                    if min(cc) < 0 or max(cc) > lim:
                        continue
                    o = self.owner_of_cell(level, cc)
                    if o is not None and o != B:
                        found.add(o)
        N = sorted(o for o in found if self.sep(B, o, level) <= 1)
        Q = sorted(o for o in found if self.sep(B, o, level) == 2)
        return N, Q
