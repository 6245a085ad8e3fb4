"""Oracle: recursive strong skeletonization (RS-S) factorization and solve
(test infrastructure only).

Follows, step by step and in the paper's notation:
* PAPER.md L873-897 (§4.2): upward pass, fine → coarse; the actives of a parent
  are the union of its children's skeletons (ascending tree order, reading C11);
  stop after level 2 (reading C12), remaining actives B_t go to a dense LU.
* PAPER.md L1880-1914 (§5.1.3, simultaneous skeletonization): one ID of
  M = [A_QB ; A_BQᵀ ; s_γ K_γB √D_B ; s_γ (√D_B S_Bγ)ᵀ]  (proxy rows iff P ≠ ∅,
  readings C3/C4/C5/C12; Q = Chebyshev-2 owners minus N, reading C6).
* PAPER.md L739-825 (Eqs. pap → strong-skel-elim): E/F with the shared T (plain
  transpose), X_RR = A_RR − TᵀA_SR − A_RS T + TᵀA_SS T, X_RS = A_RS − TᵀA_SS,
  X_SR = A_SR − A_SS T, X_RN = A_RN − TᵀA_SN, X_NR = A_NR − A_NS T; LU(X_RR);
  Schur update of (S∪N)²:  −X_{(S∪N)R} X_RR⁻¹ X_{R(S∪N)}.
* V = P E⁻¹ L⁻¹, W = U⁻¹ F⁻¹ Pᵀ stored in factored
  form; A⁻¹ ≈ W₁⁻¹⋯W_M⁻¹ P_t D⁻¹ P_tᵀ V_M⁻¹⋯V₁⁻¹ with sign-toggled inverses.
* Order within a level (reading C8): colours 0..7, Morton order inside a colour,
  and the snapshot rule — N/Q/P membership and Q rows use the actives as of the
  start of the colour phase.
* PAPER.md L907-918 (forward form):
  A ≈ (V₁V₂⋯V_M) P_t D P_tᵀ (W_M⋯W₁) with V = P E⁻¹ L⁻¹, W = U⁻¹ F⁻¹ Pᵀ and
  D = diag(X_{R₁R₁}, …, X_{R_MR_M}, A_{B_tB_t}); the inverses E⁻¹, F⁻¹, L⁻¹, U⁻¹
  toggle the sign of the off-diagonal blocks (L851-853).  ``apply`` follows it.
* Reading C1: the √w-scaled matrix Ã = W^{½} A W^{-½} is factorized;
  solve returns x = W^{-½} Ã⁻¹ (W^{½} b) in the caller's ordering.

State, two interchangeable modes that hold the same current matrix:
* DENSE mode: the whole current Ã is one n×n complex128 array; Q/N/B blocks are
  slices, the Schur writes go in place on (S∪N)², R rows/columns are never read
  again.  The most literal transcription; n ≤ ~20,000.
* BLOCK mode: current entry = pure kernel (regenerated) + Δ, Δ a dict keyed by
  owner pair (``BlockState``).  Any n (cfg3 in minutes).  Pinned to dense mode:
  identical skeletons and solutions on the small ladder (tests/test_oracle_block.py).
Order self-checks (reading C8): ``order="colour_reversed"``
reverses the order inside each colour and must reproduce the colour-major result
up to summation order; ``order="sequential"`` is the plain one-box-at-a-time
sweep and must give an equally accurate factorization.

Pins (tests/test_oracle_rss.py): n ≤ leaf_max → exactly a dense LU solve;
dense-literal check that the stored factors of each box applied to the whole
matrix give the zero pattern of Eq. strong-skel-elim and ‖Z_{R,F}‖ ≤ ε-level;
ε → 1e-12 reproduces a dense LU solve; residual ‖Ax−b‖/‖b‖ ≤ 10ε against the
brute-force matvec; proxy-vs-full-complement compression of every box.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import scipy.linalg as sla

from . import kernel as kern
from .idqr import interp_decomp, proxy_count, proxy_points
from .tree import Tree


@dataclasses.dataclass
class BoxRecord:
    box: int
    level: int
    Bs: np.ndarray   # skeleton indices (tree order), pivot order
    Br: np.ndarray   # redundant indices
    SN: np.ndarray   # S ∪ N indices (frame of Lp / Up)
    T: np.ndarray    # k × r
    lu: tuple        # scipy lu_factor of X_RR
    Lp: np.ndarray   # X_{(S∪N)R} X_RR⁻¹   ((k+|N|) × r)
    Up: np.ndarray   # X_RR⁻¹ X_{R(S∪N)}   (r × (k+|N|))
    X_RR: np.ndarray  # the pivot block itself (the D factor of the forward form)
    # separate incoming/outgoing IDs (reading R12): the column side.  None in
    # the simultaneous form, where the column sets and T are the row ones.
    Bs_c: np.ndarray = None  # column skeleton (pivot order)
    Br_c: np.ndarray = None  # redundant columns
    SN_c: np.ndarray = None  # S_c ∪ N columns (column frame of Up)
    T_c: np.ndarray = None   # k × r, A_{F R_c} ≈ A_{F S_c} T_c

    @property
    def cols(self):
        """(S_c, R_c, (S∪N)_c, T_c): the column-side sets (= the row side when simultaneous)."""
        if self.Bs_c is None:
            return self.Bs, self.Br, self.SN, self.T
        return self.Bs_c, self.Br_c, self.SN_c, self.T_c


@dataclasses.dataclass
class Factorization:
    tree: Tree
    k: float
    eps: float
    sw: np.ndarray          # √w in tree order
    records: list
    Bt: np.ndarray          # root actives (tree order, ascending)
    root_lu: tuple
    stats: dict
    A_t: np.ndarray = None  # A_{B_t B_t} (root block of D)
    Bt_c: np.ndarray = None  # root columns (separate IDs only; else = Bt)


class DenseState:
    """Dense mode: the whole current Ã as one n×n complex128 array; Q/N/B
    blocks are slices, the Schur update writes in place on (S∪N)²."""

    def __init__(self, k, X, NX, sw, A_init=None):
        self.A = kern.dense_scaled(k, X, NX, sw) if A_init is None else A_init.copy()

    def get(self, rows, cols):
        return self.A[np.ix_(rows, cols)]

    def add(self, rows, cols, V):
        self.A[np.ix_(rows, cols)] += V

    def begin_level(self, owners, active, parent_of):
        pass

    def end_phase(self, eliminated):
        pass


class BlockState:
    """Block mode: current entry = pure kernel (regenerated) + Δ, with Δ a dict
    (owner a, owner b) → complex128[|act_a|, |act_b|] present only for pairs that were ever
    updated.  The same matrix as DenseState entry by entry (the Schur complement is the only
    writer), at memory O(Σ updated blocks) instead of n².

    * ``owner[g]``, ``pos[g]``: the level-ℓ owner of active DOF g and its position in the
      owner's sorted actives (reading C11); Δ blocks are indexed by those positions.
    * ``end_phase``: after a colour phase, each eliminated box's blocks are restricted to its
      skeleton rows/columns (its R DOFs are inactive).  Restriction waits
      for the end of the phase so that same-colour boxes still read their pre-phase Q rows
      (the snapshot rule of reading C8).
    * ``begin_level``: each parent-pair block is gathered from its child-pair blocks,
      positioned into the parent's sorted actives; coarse-leaf owners
      carry over unchanged (reading C7)."""

    def __init__(self, k, X, NX, sw, n):
        self.k, self.X, self.NX, self.sw = k, X, NX, sw
        self.owner = np.full(n, -1, dtype=np.int64)
        self.pos = np.full(n, -1, dtype=np.int64)
        self.act = {}
        self.D = {}

    def _groups(self, idx):
        own = self.owner[idx]
        out = []
        for o in np.unique(own):
            sel = np.nonzero(own == o)[0]
            out.append((int(o), sel, self.pos[idx[sel]]))
        return out

    def get(self, rows, cols):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        out = kern.scaled_block(self.k, self.X, self.NX, self.sw, rows, cols)
        if rows.size == 0 or cols.size == 0:
            return out
        gc = self._groups(cols)
        for a, ri, pa in self._groups(rows):
            for b, cj, pb in gc:
                d = self.D.get((a, b))
                if d is not None:
                    out[np.ix_(ri, cj)] += d[np.ix_(pa, pb)]
        return out

    def add(self, rows, cols, V):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        gc = self._groups(cols)
        for a, ri, pa in self._groups(rows):
            for b, cj, pb in gc:
                d = self.D.get((a, b))
                if d is None:
                    d = np.zeros((self.act[a].size, self.act[b].size), dtype=np.complex128)
                    self.D[(a, b)] = d
                d[np.ix_(pa, pb)] += V[np.ix_(ri, cj)]

    def _set_owner(self, o, idx):
        self.act[o] = idx
        self.owner[idx] = o
        self.pos[idx] = np.arange(idx.size)

    def begin_level(self, owners, active, parent_of):
        """owners: the new level's owners; active[o]: their sorted actives; parent_of(o_old)
        = the new-level owner that contains old owner o_old."""
        old_act = self.act
        self.owner[:] = -1
        self.pos[:] = -1
        self.act = {}
        for o in owners:
            self._set_owner(o, np.asarray(active[o], dtype=np.int64))
        D = {}
        for (a, b), d in self.D.items():
            pa, pb = parent_of(a), parent_of(b)
            blk = D.get((pa, pb))
            if blk is None:
                blk = np.zeros((self.act[pa].size, self.act[pb].size), dtype=np.complex128)
                D[(pa, pb)] = blk
            ia = np.searchsorted(self.act[pa], old_act[a])
            ib = np.searchsorted(self.act[pb], old_act[b])
            blk[np.ix_(ia, ib)] = d
        self.D = D

    def end_phase(self, eliminated):
        """eliminated: {owner: its sorted skeleton (global indices)}."""
        keep = {}
        for o, sk in eliminated.items():
            keep[o] = self.pos[sk]
            self.owner[self.act[o]] = -1
            self.pos[self.act[o]] = -1
            self._set_owner(o, np.asarray(sk, dtype=np.int64))
        for key in list(self.D):
            a, b = key
            if a in keep or b in keep:
                d = self.D[key]
                ra = keep[a] if a in keep else slice(None)
                cb = keep[b] if b in keep else slice(None)
                self.D[key] = d[ra][:, cb]


def factor(points, normals, weights, k: float, eps: float, leaf_max: int,
           rho_factor: float = 2.0, A_init: np.ndarray | None = None,
           keep_dense: bool = False, hook=None, mode: str = "dense",
           order: str = "colour", separate: bool = False) -> Factorization:
    """Factorize Ã.

    mode: "dense" (n ≤ ~20,000) or "block" (any n); both hold the same current matrix and
    take the same steps, so they give the same skeletons and factors up to rounding.
    order: "colour" — colours 0..7, Morton order inside a colour, snapshot rule (reading C8);
    "colour_reversed" — the same with the order inside each colour reversed (C8 says the
    result is unchanged up to summation order: a self-check of the batched order);
    "sequential" — every box of the level in Morton order, each reading the actives as they
    are when it is processed (the plain sequential sweep of PAPER.md L878-884).
    ``hook(stage, ctx)`` (tests only, dense mode) is called per eliminated box with stage
    'pre' (before the Schur update) and 'post' (after); ctx holds the index sets, the ID
    and the live dense matrix.
    separate (reading R12):
    different interpolation matrices for A_FB and A_BFᵀ.  A column ID of
    M_c = [A_{Q B_c} ; s_γ K_γB √D_B] (outgoing proxy rows) gives (S_c, R_c, T_c) with
    A_{F R_c} ≈ A_{F S_c} T_c, and a row ID of M_r = [A_{B_r Q}ᵀ ; s_γ (√D_B S_Bγ)ᵀ]
    (incoming) gives (S_r, R_r, T_r) with A_{R_r F} ≈ T_rᵀ A_{S_r F}.  Both keep
    k = max(k_c, k_r) pivots of their own greedy CPQR so that the pivot block X_{R_r R_c}
    of Eq. strong-skel-elim is square (a box whose k exceeds the rows of either M is left
    uncompressed, k = b).  The box then keeps active rows S_r and active columns S_c;
    the row and column actives of every owner, the root block A_{B_t^r B_t^c} and the
    solve's row (equation) and column (unknown) vectors are tracked separately.  Dense
    mode only."""
    if mode not in ("dense", "block") or order not in ("colour", "colour_reversed", "sequential"):
        raise ValueError("mode / order")
    if separate and mode != "dense":
        raise ValueError("separate IDs need mode='dense'")
    tree = Tree(points, leaf_max)
    perm = tree.perm
    X = np.asarray(points, dtype=np.float64)[perm]
    NX = np.asarray(normals, dtype=np.float64)[perm]
    sw = np.sqrt(np.asarray(weights, dtype=np.float64)[perm])
    if mode == "dense":
        state = DenseState(k, X, NX, sw, A_init)
    else:
        if A_init is not None or hook is not None or keep_dense:
            raise ValueError("A_init / hook / keep_dense need mode='dense'")
        state = BlockState(k, X, NX, sw, tree.n)

    active = {}     # active rows per box (= the actives, simultaneous form)
    for b in range(len(tree.level)):
        if tree.is_leaf(b):
            active[b] = np.arange(tree.start[b], tree.end[b], dtype=np.int64)
    active_c = dict(active) if separate else active   # active columns
    records = []
    stats = dict(levels={}, n=tree.n, nlevels=tree.nlevels, skeletons={})

    for lvl in range(tree.nlevels - 1, 1, -1):
        for B in tree.levels[lvl]:
            if not tree.is_leaf(B):
                active[B] = np.sort(np.concatenate([active[c] for c in tree.children[B]]))
                if separate:
                    active_c[B] = np.sort(np.concatenate([active_c[c] for c in tree.children[B]]))
        owners = tree.owners(lvl)
        state.begin_level(owners, active,
                          lambda o, lvl=lvl: tree.parent[o] if tree.level[o] == lvl + 1 else o)
        side = tree.box_side(lvl)
        rho = rho_factor * side
        n_gamma = proxy_count(k, rho, eps)
        lst = dict(boxes=0, skipped=0, ranks=[], b=[], nN=[], nQ=[], rows=[], n_gamma=n_gamma)
        if order == "sequential":
            phases = [list(tree.levels[lvl])]
        else:
            phases = [[B for B in tree.levels[lvl] if tree.colour(B) == colour] for colour in range(8)]
            if order == "colour_reversed":
                phases = [p[::-1] for p in phases]
        for phase in phases:
            snap = {o: active[o] for o in owners}
            snap_c = {o: active_c[o] for o in owners}
            total = sum(v.size for v in snap.values())
            eliminated = {}
            for B in phase:
                if order == "sequential":           # no batching: every box sees the current actives
                    snap = {o: active[o] for o in owners}
                    snap_c = {o: active_c[o] for o in owners}
                    total = sum(v.size for v in snap.values())
                Bidx = snap[B]
                Bc = snap_c[B]
                b = Bidx.size
                if b == 0:
                    continue
                Nl, Ql = tree.near_q(B)
                nN = sum(snap[o].size for o in Nl)
                nQ = sum(snap[o].size for o in Ql)
                nF = total - b - nN
                if nF == 0:                       # F = ∅ → S = B, no-op (C12)
                    lst["skipped"] += 1
                    continue
                nP = nF - nQ
                Qidx = (np.concatenate([snap[o] for o in Ql]) if Ql
                        else np.zeros(0, dtype=np.int64))
                Qc = (np.concatenate([snap_c[o] for o in Ql]) if Ql
                      else np.zeros(0, dtype=np.int64))
                if not separate:
                    rows = [state.get(Qidx, Bidx), state.get(Bidx, Qidx).T]
                    if nP > 0:                         # proxy rows iff P ≠ ∅ (C12)
                        Y, s_g = proxy_points(tree.box_centre(B), rho, n_gamma)
                        Kout = kern.combined_field(k, Y, X[Bidx], NX[Bidx]) * sw[Bidx][None, :]
                        Sin = kern.green(k, X[Bidx], Y).T * sw[Bidx][None, :]
                        rows += [s_g * Kout, s_g * Sin]
                    M = np.vstack(rows)
                    P, kk, T = interp_decomp(M, eps)
                    Pc, T_c = P, T
                else:                                  # f3: one ID per side (reading R12)
                    rows_c = [state.get(Qidx, Bc)]         # far rows × B's active columns
                    rows_r = [state.get(Bidx, Qc).T]       # (B's active rows × far columns)ᵀ
                    if nP > 0:
                        Y, s_g = proxy_points(tree.box_centre(B), rho, n_gamma)
                        rows_c.append(s_g * kern.combined_field(k, Y, X[Bc], NX[Bc]) * sw[Bc][None, :])
                        rows_r.append(s_g * kern.green(k, X[Bidx], Y).T * sw[Bidx][None, :])
                    Mc, Mr = np.vstack(rows_c), np.vstack(rows_r)
                    Pc, kc, T_c = interp_decomp(Mc, eps)
                    P, kr, T = interp_decomp(Mr, eps)
                    kk = max(kc, kr)
                    if kk > min(Mc.shape[0], Mr.shape[0]):   # a side cannot reach k pivots: keep B
                        kk = b
                        P = Pc = np.arange(b, dtype=np.int64)
                    else:
                        if kc < kk:
                            Pc, _, T_c = interp_decomp(Mc, eps, k_min=kk)
                        if kr < kk:
                            P, _, T = interp_decomp(Mr, eps, k_min=kk)
                    M = Mc
                Bs = Bidx[P[:kk]]
                Br = Bidx[P[kk:]]
                Bs_c = Bc[Pc[:kk]]
                Br_c = Bc[Pc[kk:]]
                Nidx = (np.concatenate([active[o] for o in Nl]) if Nl
                        else np.zeros(0, dtype=np.int64))
                Nc = (np.concatenate([active_c[o] for o in Nl]) if Nl
                      else np.zeros(0, dtype=np.int64))
                lst["boxes"] += 1
                lst["ranks"].append(kk)
                lst["b"].append(b)
                lst["nN"].append(Nidx.size)
                lst["nQ"].append(Qidx.size)
                lst["rows"].append(M.shape[0])
                stats["skeletons"][B] = np.sort(Bs)
                if separate:
                    stats.setdefault("skeletons_c", {})[B] = np.sort(Bs_c)
                    stats.setdefault("ranks_rc", []).append((kr, kc))
                if Br.size == 0:                   # k = b: nothing to eliminate (C13)
                    continue
                # --- E/F transforms (Eq. pap and the X blocks that follow it); rows use the row
                # sets and T, columns the column sets and T_c (the same ones when simultaneous)
                A_RR = state.get(Br, Br_c); A_RS = state.get(Br, Bs_c); A_SR = state.get(Bs, Br_c)
                A_SS = state.get(Bs, Bs_c); A_RN = state.get(Br, Nc); A_NR = state.get(Nidx, Br_c)
                A_SN = state.get(Bs, Nc); A_NS = state.get(Nidx, Bs_c)
                X_RR = A_RR - T.T @ A_SR - A_RS @ T_c + T.T @ A_SS @ T_c
                X_RS = A_RS - T.T @ A_SS
                X_SR = A_SR - A_SS @ T_c
                X_RN = A_RN - T.T @ A_SN
                X_NR = A_NR - A_NS @ T_c
                # --- L/U with pivot block X_RR (Eq. strong-skel-elim)
                lu = sla.lu_factor(X_RR, check_finite=False)
                X_cR = np.vstack([X_SR, X_NR])
                X_Rc = np.hstack([X_RS, X_RN])
                Lp = sla.lu_solve(lu, X_cR.T, trans=1).T
                Up = sla.lu_solve(lu, X_Rc)
                SN = np.concatenate([Bs, Nidx])
                SN_c = np.concatenate([Bs_c, Nc]) if separate else SN
                if hook is not None:
                    Fidx = np.concatenate([snap[o] for o in owners if o != B and o not in Nl] or
                                          [np.zeros(0, dtype=np.int64)])
                    Fc = np.concatenate([snap_c[o] for o in owners if o != B and o not in Nl] or
                                        [np.zeros(0, dtype=np.int64)])
                    ctx = dict(B=B, level=lvl, Bs=Bs, Br=Br, Nidx=Nidx, Qidx=Qidx, Fidx=Fidx,
                               T=T, A=state.A, M=M, nP=nP, Bs_c=Bs_c, Br_c=Br_c, Nc=Nc, Fc=Fc, T_c=T_c)
                    hook("pre", ctx)
                state.add(SN, SN_c, -(X_cR @ Up))     # Schur complement update
                if hook is not None:
                    hook("post", ctx)
                if separate:
                    records.append(BoxRecord(B, lvl, Bs, Br, SN, T, lu, Lp, Up, X_RR, Bs_c, Br_c, SN_c, T_c))
                    active_c[B] = np.sort(Bs_c)
                else:
                    records.append(BoxRecord(B, lvl, Bs, Br, SN, T, lu, Lp, Up, X_RR))
                active[B] = np.sort(Bs)
                eliminated[B] = active[B]
                if order == "sequential":
                    state.end_phase(eliminated)
                    eliminated = {}
            state.end_phase(eliminated)
        lst["ranks"] = np.asarray(lst["ranks"])
        stats["levels"][lvl] = lst

    alive = np.ones(tree.n, dtype=bool)      # every leaf DOF starts active
    alive_c = np.ones(tree.n, dtype=bool)
    for r in records:
        alive[r.Br] = False
        alive_c[r.cols[1]] = False
    Bt = np.nonzero(alive)[0]
    Bt_c = np.nonzero(alive_c)[0] if separate else Bt
    A_t = state.get(Bt, Bt_c)
    root_lu = sla.lu_factor(A_t, check_finite=False)
    stats["n0"] = int(Bt.size)
    f = Factorization(tree, k, eps, sw, records, Bt, root_lu, stats, A_t, Bt_c if separate else None)
    if keep_dense:
        f.A_final = state.A
    return f


def solve(f: Factorization, b: np.ndarray) -> np.ndarray:
    """x ≈ A⁻¹ b for BASELINE.json's unscaled A; b is n or n×nrhs in caller order."""
    b = np.asarray(b, dtype=np.complex128)
    vec = b.ndim == 1
    bb = b[:, None] if vec else b
    perm = f.tree.perm
    y = bb[perm] * f.sw[:, None]                    # W^{½} b in tree order (C1)
    # separate IDs (f3): the upward sweep runs on the equation (row) vector y, D⁻¹ maps the
    # R_r entries to the unknowns at R_c, the downward sweep runs on the unknown (column)
    # vector yc.  Simultaneous: the two are one vector, updated in place.
    yc = np.zeros_like(y) if f.Bt_c is not None else y
    for r in f.records:                             # V_M⁻¹ ⋯ V_1⁻¹ : E then L, then D⁻¹ on R
        y[r.Br] -= r.T.T @ y[r.Bs]
        y[r.SN] -= r.Lp @ y[r.Br]
        yc[r.cols[1]] = sla.lu_solve(r.lu, y[r.Br])
    Bt_c = f.Bt if f.Bt_c is None else f.Bt_c
    if f.Bt.size:
        yc[Bt_c] = sla.lu_solve(f.root_lu, y[f.Bt])  # P_t D⁻¹ P_tᵀ on the root block
    y = yc
    for r in reversed(f.records):                   # W_1⁻¹ ⋯ W_M⁻¹ : U then F
        Bs_c, Br_c, SN_c, T_c = r.cols
        y[Br_c] -= r.Up @ y[SN_c]
        y[Bs_c] -= T_c @ y[Br_c]
    x = np.empty_like(y)
    x[perm] = y / f.sw[:, None]
    return x[:, 0] if vec else x


def apply(f: Factorization, x: np.ndarray) -> np.ndarray:
    """y ≈ A x from the stored factors, for BASELINE.json's
    unscaled A; x is n or n×nrhs in caller order.  Rightmost factor first:
    W₁ … W_M (F⁻¹ then U⁻¹ per box, boxes in elimination order), then D, then
    V_M … V₁ (L⁻¹ then E⁻¹ per box, boxes in reverse order).  Exactly inverse to
    ``solve`` up to rounding; within ε of A x."""
    x = np.asarray(x, dtype=np.complex128)
    vec = x.ndim == 1
    xx = x[:, None] if vec else x
    perm = f.tree.perm
    y = xx[perm] * f.sw[:, None]                    # Ã acts on W^{½} x (C1)
    for r in f.records:                             # W_j = U⁻¹ F⁻¹ Pᵀ (unknown/column side)
        Bs_c, Br_c, SN_c, T_c = r.cols
        y[Bs_c] += T_c @ y[Br_c]                    # F⁻¹
        y[Br_c] += r.Up @ y[SN_c]                   # U⁻¹
    # D maps the unknowns at R_c (root: B_t^c) to the equations at R_r (B_t); one vector when
    # simultaneous (the blocks are disjoint, so in place is exact)
    yr = np.zeros_like(y) if f.Bt_c is not None else y
    for r in f.records:                             # D on the R blocks
        yr[r.Br] = r.X_RR @ y[r.cols[1]]
    if f.Bt.size:
        yr[f.Bt] = f.A_t @ y[f.Bt if f.Bt_c is None else f.Bt_c]   # P_t A_{B_tB_t} P_tᵀ
    y = yr
    for r in reversed(f.records):                   # V_j = P E⁻¹ L⁻¹
        y[r.SN] += r.Lp @ y[r.Br]                   # L⁻¹
        y[r.Br] += r.T.T @ y[r.Bs]                  # E⁻¹
    out = np.empty_like(y)
    out[perm] = y / f.sw[:, None]                   # back to A = W^{-½} Ã W^{½}
    return out[:, 0] if vec else out
