"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This package holds ONLY input generation (geometry, weights, normals, right-hand
sides).  It contains none of the FMM-LU method's arithmetic: no kernel
evaluation, no tree, no skeletonization.  Both the CPU oracle (``oracle/``) and
the CUDA path (``paper_2201_07325_b200``) are fed from here; neither imports the
other.

Recipes follow SURVEY.md §8(d) (configs 1-5 of BASELINE.json) and its readings
C15/C16/C21; DESIGN.md §"Inputs" restates them.
"""
from .geometry import (  # noqa: F401
    Geometry,
    fibonacci_sphere,
    ellipsoid,
    bump_sphere,
    wavy_torus,
    cube_corners,
    random_cube,
    config_geometry,
    CONFIGS,
)
from .rhs import gaussian_rhs  # noqa: F401
from .boxes import box_batch  # noqa: F401
