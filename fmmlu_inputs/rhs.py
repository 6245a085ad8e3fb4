"""Right-hand sides (SURVEY.md reading C16).

``rng = numpy.random.default_rng(seed)``; ``b = rng.standard_normal((nrhs, n)) +
1j*rng.standard_normal((nrhs, n))``; returned as an n×nrhs column-major
(Fortran-order) complex128 array, i.e. column j is RHS j.
"""
from __future__ import annotations

import numpy as np


def gaussian_rhs(n: int, nrhs: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    re = rng.standard_normal((nrhs, n))
    im = rng.standard_normal((nrhs, n))
    b = (re + 1j * im).T  # n×nrhs, Fortran order (the (nrhs,n) C array transposed)
    return np.asfortranarray(b)
