"""GPU parity for BASELINE configs[3] ("cfg4"): fmmlu_boxes (batched ID + elimination of
independent boxes, readings C21/C22) against oracle/boxes.py on the same seeded boxes."""
import math

import numpy as np
import pytest

import fmmlu_inputs as fi
from oracle import boxes as ob

pytestmark = pytest.mark.gpu

K, NG = 10.0, 512


@pytest.fixture(scope="module")
def F():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2201_07325_b200 import fmmlu
    fmmlu.load()
    return fmmlu


def _rho(h):
    return 1.5 * (math.sqrt(3.0) / 2.0) * h


def _check_box(d, i, out, eps):
    """Every compared box is judged (no skipped near-ties):
    * the GPU rank is within ±2 of the oracle's CPQR rank (pivot near-ties at the threshold);
    * the GPU skeleton S = perm[:k] is a valid ε-ID of the oracle's M (reading C9 bound: every
      redundant column fit to ≤ ε·max column norm, 2× slack for the near-tie band);
    * Δ equals, to 10ε relative, the oracle's elimination on the GPU's own column
      split with T = argmin‖M_R − M_S T‖ — exactly R11⁻¹R12 when the split is CPQR's
      (oracle/boxes.py ``split``; pinned in tests/test_oracle_boxes.py)."""
    args = (K, eps, d["pts"][i], d["nrm"][i], d["npts"][i], d["nnrm"][i], d["w"], d["h"])
    o = ob.eliminate_box(*args, n_gamma=NG)
    kg = int(out["ranks"][i])
    pg = np.asarray(out["perm"][i], dtype=np.int64)
    assert sorted(pg.tolist()) == list(range(pg.size))
    assert abs(kg - o["k"]) <= 2, (i, kg, o["k"])
    og = ob.eliminate_box(*args, n_gamma=NG, split=(pg, kg))
    M = og["M"]
    if 0 < kg < pg.size:
        res = M[:, pg[kg:]] - M[:, pg[:kg]] @ og["T"]
        assert np.linalg.norm(res, axis=0).max() <= 2 * eps * np.linalg.norm(M, axis=0).max(), i
    D, Do = out["delta"][i], og["Delta"]
    assert D.shape == Do.shape
    scale = np.abs(Do).max()
    err = np.abs(D - Do).max()
    assert err <= 10 * eps * scale + 1e-13, (i, err / max(scale, 1e-300))
    return err / max(scale, 1e-300)


@pytest.mark.parametrize("eps", [1e-4, 1e-6, 1e-9])
def test_boxes_parity_vs_oracle(F, eps):
    d = fi.box_batch(6, first_id=0)
    out = F.boxes(d["pts"], d["nrm"], d["npts"], d["nnrm"], d["w"], K, eps, NG, _rho(d["h"]), keep=[0, 3, 5])
    assert out["ranks"].shape == (6,)
    for p in out["perm"]:
        assert sorted(p.tolist()) == list(range(256))   # a permutation of the box columns
    for i in (0, 3, 5):
        _check_box(d, i, out, eps)


def test_boxes_two_waves_and_device_pointers(F):
    """More boxes than one wave; box ids, seeds and outputs line up across the wave boundary;
    device-resident inputs give the same ranks as host inputs."""
    import torch
    nbox = 2100
    d = fi.box_batch(nbox, first_id=0)
    out = F.boxes(d["pts"], d["nrm"], d["npts"], d["nnrm"], d["w"], K, 1e-6, NG, _rho(d["h"]), keep=[0, nbox - 1])
    assert out["wave"] < nbox
    assert out["ranks"].min() > 0 and out["ranks"].max() <= 256
    _check_box(d, 0, out, 1e-6)
    _check_box(d, nbox - 1, out, 1e-6)
    dv = [torch.from_numpy(d[k][:64]).cuda() for k in ("pts", "nrm", "npts", "nnrm")]
    out2 = F.boxes(*dv, d["w"], K, 1e-6, NG, _rho(d["h"]), want_perm=True)
    assert np.abs(out2["ranks"].astype(int) - out["ranks"][:64].astype(int)).max() <= 1


def test_boxes_full_rank_gives_zero_delta(F):
    """ε below rounding: nothing is eliminated (k = b) and Δ = 0 (C13)."""
    d = fi.box_batch(2, b=16, n_near=32, first_id=7)
    out = F.boxes(d["pts"], d["nrm"], d["npts"], d["nnrm"], d["w"], K, 1e-15, 64, _rho(d["h"]), keep=[1])
    assert np.all(out["ranks"] == 16)
    assert np.all(out["delta"][1] == 0)


def test_boxes_errors(F):
    d = fi.box_batch(1, b=8, n_near=8)
    with pytest.raises(F.FmmluError) as e:
        F.boxes(d["pts"], d["nrm"], d["npts"], d["nnrm"], d["w"], K, 1.5, 64, 0.2)
    assert e.value.code == -1
    with pytest.raises(F.FmmluError) as e:
        F.boxes(d["pts"], d["nrm"], d["npts"], d["nnrm"], d["w"], K, 1e-6, 64, 0.2, keep=[3])
    assert e.value.code == -1


@pytest.mark.parametrize("eps", [1e-4, 1e-6, 1e-9])
def test_boxes_full_size_sampled_parity(F, eps):
    """BASELINE configs[3] at full size (8192 boxes in waves, the launch configuration of
    bench.py's cfg4 key): 32 boxes sampled across every wave, each judged by _check_box
    (rank, ID validity, Δ at 10ε); ranks of all boxes in range."""
    nbox = 8192
    d = fi.box_batch(nbox, first_id=0)
    sample = sorted(set(np.linspace(0, nbox - 1, 32).astype(int).tolist()))
    out = F.boxes(d["pts"], d["nrm"], d["npts"], d["nnrm"], d["w"], K, eps, NG, _rho(d["h"]), keep=sample,
                  want_perm=True)
    assert out["ranks"].shape == (nbox,)
    assert out["ranks"].min() > 0 and out["ranks"].max() <= 256
    assert out["wave"] < nbox  # several waves
    errs = [_check_box(d, i, out, eps) for i in sample]
    assert max(errs) <= 10 * eps
