"""Thin ctypes binding over libfmmlu.so (include/fmmlu.h).  Argument marshalling only:
every step of the method runs in the library's CUDA kernels.  There is no CPU fallback —
if the shared library or a CUDA device is missing, calls raise.

Arrays may be NumPy arrays (host memory: the library copies in/out inside the call) or
CUDA torch tensors (device memory, used in place).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

_LIB = None

FMMLU_ERRORS = {
    -1: "EINVAL", -2: "EDEPTH", -3: "ESINGULAR", -4: "ENOMEM", -5: "ESTATE", -6: "ENOTIMPL", -7: "ECUDA",
}


class FmmluError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"fmmlu error {code} ({FMMLU_ERRORS.get(code, '?')}): {msg}")
        self.code = code


class Stats(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64), ("nlevels", ctypes.c_int32), ("nboxes", ctypes.c_int32),
        ("nleaves", ctypes.c_int32), ("n_eliminated", ctypes.c_int32), ("n0", ctypes.c_int64),
        ("max_rank", ctypes.c_int32), ("max_b", ctypes.c_int32), ("factor_bytes", ctypes.c_int64),
        ("peak_bytes", ctypes.c_int64), ("t_tree_ms", ctypes.c_double), ("t_factor_ms", ctypes.c_double),
        ("t_solve_ms", ctypes.c_double), ("t_root_ms", ctypes.c_double), ("t_levels_ms", ctypes.c_double * 24),
        ("n_singular_warn", ctypes.c_int32), ("ranks_sum", ctypes.c_int32 * 24), ("boxes", ctypes.c_int32 * 24),
        ("n_launches", ctypes.c_int64), ("class_ms", ctypes.c_double * 16), ("class_flops", ctypes.c_double * 16),
        ("class_bytes", ctypes.c_double * 16), ("class_launches", ctypes.c_int64 * 16),
        ("t_sync_wait_ms", ctypes.c_double),
    ]

    def as_dict(self):
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            d[name] = list(v) if hasattr(v, "__len__") else v
        return d


KERNEL_CLASSES = ["build", "gather", "qr", "cpqr", "ef", "inv", "panel", "schur", "root", "solve", "apply"]

EXPORTS = ("fmmlu_tree", "fmmlu_factor", "fmmlu_solve", "fmmlu_apply", "fmmlu_monostatic_rcs", "fmmlu_matvec", "fmmlu_destroy",
           "fmmlu_last_error", "fmmlu_stats", "fmmlu_set_stream", "fmmlu_tree_perm", "fmmlu_probe_fp64",
           "fmmlu_set_param", "fmmlu_inverse_batch", "fmmlu_boxes", "fmmlu_release_cache", "fmmlu_tree_boxes",
           "fmmlu_level_lists")


def lib_path() -> str:
    return os.environ.get("FMMLU_LIB") or _build.LIB  # FMMLU_LIB: an alternative build (experiments)


def load(build_if_missing: bool = False):
    """Load libfmmlu.so (in-tree).  Raises if it is missing (no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        if not build_if_missing:
            raise FmmluError(-7, f"{path} not built (run python -m paper_2201_07325_b200.build)")
        _build.build()
    L = ctypes.CDLL(path)
    vp, i64, ci, cd = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.fmmlu_tree.argtypes = [vp, vp, vp, i64, ci, ctypes.POINTER(vp)]
    L.fmmlu_factor.argtypes = [vp, cd, cd]
    L.fmmlu_solve.argtypes = [vp, vp, ci]
    L.fmmlu_apply.argtypes = [vp, vp, ci]
    L.fmmlu_monostatic_rcs.argtypes = [vp, vp, ci, vp]
    L.fmmlu_matvec.argtypes = [vp, cd, vp, vp, ci]
    L.fmmlu_destroy.argtypes = [vp]
    L.fmmlu_last_error.restype = ctypes.c_char_p
    L.fmmlu_last_error.argtypes = []
    L.fmmlu_stats.argtypes = [vp, ctypes.POINTER(Stats)]
    L.fmmlu_set_stream.argtypes = [vp, vp]
    L.fmmlu_tree_perm.argtypes = [vp, vp]
    L.fmmlu_probe_fp64.argtypes = [ci, ctypes.POINTER(cd)]
    L.fmmlu_set_param.argtypes = [vp, ctypes.c_char_p, cd]
    L.fmmlu_inverse_batch.argtypes = [vp, vp, ci, ci, ctypes.POINTER(cd)]
    L.fmmlu_boxes.argtypes = [vp, vp, vp, vp, ci, ci, ci, cd, cd, cd, ci, cd, vp, vp, ci, vp, vp, vp]
    L.fmmlu_release_cache.argtypes = []
    L.fmmlu_tree_boxes.argtypes = [vp, vp, vp, vp, vp, vp]
    L.fmmlu_level_lists.argtypes = [vp, ctypes.c_int, vp, vp, vp, vp, vp, vp]
    for f in EXPORTS:
        getattr(L, f).restype = ctypes.c_char_p if f == "fmmlu_last_error" else ctypes.c_int
    _LIB = L
    return L


def _check(rc: int):
    if rc != 0:
        raise FmmluError(rc, load().fmmlu_last_error().decode())


def _ptr(a):
    """Data pointer of a NumPy array (host) or a torch tensor (host or device)."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    raise TypeError(type(a))


def _sync_producer(*arrays):
    """Stream-ordering precondition of include/fmmlu.h: a CUDA tensor argument may have been
    written on torch's current stream; make that work complete before the library reads it."""
    for a in arrays:
        if hasattr(a, "is_cuda") and a.is_cuda:
            import torch
            torch.cuda.current_stream(a.device).synchronize()
            return


def release_cache():
    """Return the library's cached device memory to the driver (fmmlu_release_cache)."""
    _check(load().fmmlu_release_cache())


def _f64_rows3(a):
    if isinstance(a, np.ndarray):
        return np.ascontiguousarray(a, dtype=np.float64)
    assert a.dtype.is_floating_point and a.element_size() == 8 and a.is_contiguous()
    return a


class FmmLu:
    """One handle = one point set; factor() may be called repeatedly (new k / eps)."""

    def __init__(self, points, normals, weights, leaf_max: int = 64):
        L = load()
        self._keep = [_f64_rows3(points), _f64_rows3(normals), _f64_rows3(weights)]
        n = int(self._keep[2].shape[0])
        _sync_producer(*self._keep)
        self._stream = None
        h = ctypes.c_void_p()
        _check(L.fmmlu_tree(_ptr(self._keep[0]), _ptr(self._keep[1]), _ptr(self._keep[2]), n, int(leaf_max),
                            ctypes.byref(h)))
        self.h = h
        self.n = n
        self._keep = None

    def factor(self, k: float, eps: float):
        _check(load().fmmlu_factor(self.h, float(k), float(eps)))
        return self

    def solve(self, rhs, nrhs: int | None = None):
        """In place: rhs (n×nrhs column-major complex128, i.e. a Fortran-order NumPy array or a
        transposed-contiguous torch tensor) is overwritten with A⁻¹ rhs.  Returns rhs."""
        if nrhs is None:
            nrhs = 1 if rhs.ndim == 1 else int(rhs.shape[1])
        if isinstance(rhs, np.ndarray):
            assert rhs.dtype == np.complex128 and (rhs.ndim == 1 or rhs.flags.f_contiguous)
        elif self._stream is None:
            _sync_producer(rhs)
        _check(load().fmmlu_solve(self.h, _ptr(rhs), int(nrhs)))
        return rhs

    def apply(self, x, nrhs: int | None = None):
        """In place: x (n×nrhs column-major complex128) is overwritten with Â x, the forward
        factored operator V₁⋯V_M P_t D P_tᵀ W_M⋯W₁ ≈ A.  Returns x."""
        if nrhs is None:
            nrhs = 1 if x.ndim == 1 else int(x.shape[1])
        if isinstance(x, np.ndarray):
            assert x.dtype == np.complex128 and (x.ndim == 1 or x.flags.f_contiguous)
        elif self._stream is None:
            _sync_producer(x)
        _check(load().fmmlu_apply(self.h, _ptr(x), int(nrhs)))
        return x

    def monostatic_rcs(self, phis, out=None):
        """R(φ₀) for every azimuth in `phis` (§6.3): plane-wave solves with the stored
        factors and the backscatter functional, all on the device.  Returns complex128 (nphi,)."""
        if isinstance(phis, np.ndarray) or not hasattr(phis, "data_ptr"):
            phis = np.ascontiguousarray(np.asarray(phis, dtype=np.float64))
        nphi = int(phis.shape[0])
        if out is None:
            out = np.empty(nphi, dtype=np.complex128)
        _check(load().fmmlu_monostatic_rcs(self.h, _ptr(phis), nphi, _ptr(out)))
        return out

    def matvec(self, k: float, x, y=None):
        nrhs = 1 if x.ndim == 1 else int(x.shape[1])
        if y is None:
            y = np.empty_like(x, order="F") if isinstance(x, np.ndarray) else x.clone()
        if self._stream is None:
            _sync_producer(x, y)
        _check(load().fmmlu_matvec(self.h, float(k), _ptr(x), _ptr(y), nrhs))
        return y

    def stats(self) -> dict:
        s = Stats()
        _check(load().fmmlu_stats(self.h, ctypes.byref(s)))
        return s.as_dict()

    def tree_boxes(self) -> dict:
        """The device-built octree: level, coord (nbox×3), start, end per box (level-major, Morton)."""
        L = load()
        nb = ctypes.c_int32(0)
        _check(L.fmmlu_tree_boxes(self.h, ctypes.byref(nb), None, None, None, None))
        lev = np.empty(nb.value, dtype=np.int32)
        crd = np.empty((nb.value, 3), dtype=np.int32)
        st = np.empty(nb.value, dtype=np.int32)
        en = np.empty(nb.value, dtype=np.int32)
        _check(L.fmmlu_tree_boxes(self.h, ctypes.byref(nb), lev.ctypes.data, crd.ctypes.data, st.ctypes.data,
                                  en.ctypes.data))
        return dict(level=lev, coord=crd, start=st, end=en)

    def level_lists(self, level: int) -> dict:
        """The device-built owner lists of one level: owners (box ids as in tree_boxes), and per level
        box the N / Q owners as CSR (nptr, nidx, qptr, qidx) of local owner indices."""
        L = load()
        cnt = np.zeros(4, dtype=np.int32)
        _check(L.fmmlu_level_lists(self.h, int(level), cnt.ctypes.data, None, None, None, None, None))
        nlb, no, tn, tq = (int(v) for v in cnt)
        owners = np.empty(max(no, 1), dtype=np.int32)
        nptr = np.empty(nlb + 1, dtype=np.int32)
        qptr = np.empty(nlb + 1, dtype=np.int32)
        nidx = np.empty(max(tn, 1), dtype=np.int32)
        qidx = np.empty(max(tq, 1), dtype=np.int32)
        _check(L.fmmlu_level_lists(self.h, int(level), cnt.ctypes.data, owners.ctypes.data, nptr.ctypes.data,
                                   nidx.ctypes.data, qptr.ctypes.data, qidx.ctypes.data))
        return dict(nlb=nlb, owners=owners[:no], nptr=nptr, nidx=nidx[:tn], qptr=qptr, qidx=qidx[:tq])

    def tree_perm(self) -> np.ndarray:
        p = np.empty(self.n, dtype=np.int64)
        _check(load().fmmlu_tree_perm(self.h, p.ctypes.data))
        return p

    def set_param(self, name: str, value: float):
        _check(load().fmmlu_set_param(self.h, name.encode(), float(value)))
        return self

    def inverse_batch(self, A, n: int, count: int) -> float:
        """In-place inverse of `count` n×n complex128 matrices (device tensor, column-major,
        contiguous) with the handle's gj_mode; returns the device time in ms."""
        ms = ctypes.c_double(0.0)
        _check(load().fmmlu_inverse_batch(self.h, _ptr(A), int(n), int(count), ctypes.byref(ms)))
        return ms.value

    def set_stream(self, stream_ptr: int | None):
        _check(load().fmmlu_set_stream(self.h, stream_ptr or None))
        self._stream = stream_ptr or None

    def close(self):
        if getattr(self, "h", None):
            load().fmmlu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# module-level names mirroring the C ABI
def fmmlu_tree(points, normals, weights, leaf_max: int = 64) -> FmmLu:
    return FmmLu(points, normals, weights, leaf_max)


def fmmlu_factor(h: FmmLu, k: float, eps: float) -> FmmLu:
    return h.factor(k, eps)


def fmmlu_solve(h: FmmLu, rhs, nrhs: int | None = None):
    return h.solve(rhs, nrhs)


def fmmlu_apply(h: FmmLu, x, nrhs: int | None = None):
    return h.apply(x, nrhs)


def probe_fp64(kind: int) -> float:
    v = ctypes.c_double()
    _check(load().fmmlu_probe_fp64(int(kind), ctypes.byref(v)))
    return v.value


def boxes(pts, nrm, npts, nnrm, w: float, k: float, eps: float, n_gamma: int, rho: float,
          keep=(), want_perm: bool = True):
    """cfg4 batched ID + elimination of independent boxes (fmmlu_boxes).  Arrays (NumPy or torch,
    host or device): pts/nrm (nbox, b, 3), npts/nnrm (nbox, nnear, 3).  Returns dict(ranks, perm,
    delta: {box id: Δ (k+nnear)²}, ms, gflop, wave)."""
    L = load()
    arrs = [_f64_rows3(a) for a in (pts, nrm, npts, nnrm)]
    _sync_producer(*arrs)
    nbox, b = int(arrs[0].shape[0]), int(arrs[0].shape[1])
    nnear = int(arrs[2].shape[1])
    ranks = np.zeros(nbox, dtype=np.int32)
    perm = np.zeros((nbox, b), dtype=np.int32) if want_perm else None
    keep = np.asarray(list(keep), dtype=np.int32)
    npb = b + nnear
    delta = np.zeros((max(1, keep.size), npb * npb), dtype=np.complex128)
    timing = (ctypes.c_double * 3)()
    _check(L.fmmlu_boxes(_ptr(arrs[0]), _ptr(arrs[1]), _ptr(arrs[2]), _ptr(arrs[3]), nbox, b, nnear, float(w),
                         float(k), float(eps), int(n_gamma), float(rho), ranks.ctypes.data,
                         perm.ctypes.data if perm is not None else None, int(keep.size),
                         keep.ctypes.data if keep.size else None, delta.ctypes.data if keep.size else None,
                         timing))
    out = {}
    for j, bid in enumerate(keep.tolist()):
        kn = int(ranks[bid]) + nnear
        out[bid] = delta[j, :kn * kn].reshape(kn, kn, order="F")
    return dict(ranks=ranks, perm=perm, delta=out, ms=timing[0], gflop=timing[1], wave=int(timing[2]))
