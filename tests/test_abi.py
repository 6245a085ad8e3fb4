"""CPU-side checks of the C ABI library: it builds, loads, exports every symbol declared
in include/fmmlu.h, validates arguments, and fails loudly (no CPU fallback) without a GPU."""
import os
import re
import subprocess

import numpy as np
import pytest

import fmmlu_inputs as fi
from paper_2201_07325_b200 import build as B
from paper_2201_07325_b200 import fmmlu as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fmmlu.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(fmmlu_\w+)\s*\(", src, re.M)))


def test_builds_and_exports_all_declared_symbols():
    lib = B.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    syms = set(re.findall(r"\bT (fmmlu_\w+)", out))
    decl = _declared()
    assert len(decl) >= 10
    assert set(decl) <= syms, set(decl) - syms
    assert set(F.EXPORTS) == set(decl)


def test_sm100a_cubin_present():
    lib = B.build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_load_and_argument_validation():
    L = F.load()
    g = fi.fibonacci_sphere(50)
    # n < 1, leaf_max < 1 → EINVAL before touching the device
    with pytest.raises(F.FmmluError) as e:
        F.FmmLu(g.points, g.normals, g.weights, leaf_max=0)
    assert e.value.code == -1
    bad = g.normals.copy()
    bad[3] *= 1.5
    with pytest.raises(F.FmmluError) as e:
        F.FmmLu(g.points, bad, g.weights)
    assert e.value.code in (-1, -7)   # -7 when no GPU is present (checked first)
    assert L.fmmlu_destroy(None) == 0


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = fi.fibonacci_sphere(50)
    with pytest.raises(F.FmmluError) as e:
        F.FmmLu(g.points, g.normals, g.weights)
    assert e.value.code == -7
