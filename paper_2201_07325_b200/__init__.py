"""B200-native FMM-LU hot path (arXiv 2201.07325): recursive strong skeletonization of
the combined-field Helmholtz matrix on one GPU.  The compute path is libfmmlu.so
(hand-written CUDA for sm_100a, C ABI in include/fmmlu.h); this package is the thin
Python binding plus the in-tree build."""
from .fmmlu import FmmLu, FmmluError, fmmlu_tree, fmmlu_factor, fmmlu_solve, load, probe_fp64  # noqa: F401
