"""Write the oracle's full-size expected solutions under tests/golden/ (calls only oracle/ and
fmmlu_inputs/; nothing from the CUDA path).

    python tools/make_golden.py cfg1|cfg2|cfg3
    python tools/make_golden.py cfg2 --separate      (separate incoming/outgoing IDs, dense mode)

* cfg1, cfg2: dense mode AND block mode ("both must give identical S/T on
  cfg1–2"); the script asserts identical skeleton sets for every box and solutions within
  1e-10 of each other, then stores the dense-mode solution (all RHS columns, complex128).
* cfg3 (n = 10⁵): block mode only (the dense matrix would be 160 GB).  Stores the full
  solution of RHS columns 0 and 1 (complex128), and for all 16 columns the 2-norm and the
  entries at 4096 seeded sample indices.

Each file records the oracle's n0, per-level ranks and wall time.  The right-hand sides are
fmmlu_inputs.gaussian_rhs(n, nrhs, 0) (reading C16), exactly what the GPU tests solve.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import fmmlu_inputs as fi  # noqa: E402
from oracle import dense, rss  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def run_separate(name):
    """Separate incoming/outgoing IDs (DESIGN R12): the oracle's dense-mode
    separate factorization (the only mode that has it), all RHS columns stored."""
    c = fi.CONFIGS[name]
    g = fi.config_geometry(name)
    b = fi.gaussian_rhs(g.n, c["nrhs"], 0)
    t0 = time.time()
    f = rss.factor(g.points, g.normals, g.weights, c["k"], c["eps"], c["leaf_max"], mode="dense", separate=True)
    t1 = time.time()
    x = rss.solve(f, b)
    rc = np.array(f.stats["ranks_rc"])
    meta = dict(config=name, separate=True, n=g.n, k=c["k"], eps=c["eps"], leaf_max=c["leaf_max"], nrhs=c["nrhs"],
                rhs="fmmlu_inputs.gaussian_rhs(n, nrhs, 0)", cores=os.cpu_count(), dense_factor_s=t1 - t0,
                n0=int(f.stats["n0"]), boxes_with_different_ranks=int((rc[:, 0] != rc[:, 1]).sum()), boxes=int(rc.shape[0]),
                skeleton_sum=int(sum(v.size for v in f.stats["skeletons"].values())),
                stored="x_full = all columns")
    np.savez_compressed(os.path.join(GOLD, f"{name}_oracle_separate_solution.npz"), x_full=np.ascontiguousarray(x),
                        colnorm=np.linalg.norm(x, axis=0))
    with open(os.path.join(GOLD, f"{name}_oracle_separate_solution.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(json.dumps(meta), flush=True)


def run(name):
    c = fi.CONFIGS[name]
    g = fi.config_geometry(name)
    b = fi.gaussian_rhs(g.n, c["nrhs"], 0)
    meta = dict(config=name, n=g.n, k=c["k"], eps=c["eps"], leaf_max=c["leaf_max"], nrhs=c["nrhs"],
                rhs="fmmlu_inputs.gaussian_rhs(n, nrhs, 0)", cores=os.cpu_count())
    modes = ["dense", "block"] if name in ("cfg1", "cfg2") else ["block"]
    sols, facs = {}, {}
    for mode in modes:
        t0 = time.time()
        f = rss.factor(g.points, g.normals, g.weights, c["k"], c["eps"], c["leaf_max"], mode=mode)
        t1 = time.time()
        x = rss.solve(f, b)
        t2 = time.time()
        sols[mode], facs[mode] = x, f
        meta[f"{mode}_factor_s"] = t1 - t0
        meta[f"{mode}_solve_s"] = t2 - t1
        print(f"{name} {mode}: factor {t1 - t0:.1f} s solve {t2 - t1:.1f} s n0 {f.stats['n0']}", flush=True)
    f = facs[modes[0]]
    if len(modes) == 2:
        fd, fb = facs["dense"], facs["block"]
        same = sum(np.array_equal(s, fb.stats["skeletons"].get(B)) for B, s in fd.stats["skeletons"].items())
        meta["dense_vs_block_same_skeletons"] = f"{same}/{len(fd.stats['skeletons'])}"
        meta["dense_vs_block_rel_diff"] = dense.rel_diff(sols["block"], sols["dense"])
        assert same == len(fd.stats["skeletons"]), meta["dense_vs_block_same_skeletons"]
        assert meta["dense_vs_block_rel_diff"] <= 1e-10, meta["dense_vs_block_rel_diff"]
    x = sols[modes[0]]
    meta["n0"] = f.stats["n0"]
    meta["ranks_sum"] = {int(l): int(s["ranks"].sum()) for l, s in f.stats["levels"].items()}
    meta["boxes"] = {int(l): int(s["boxes"]) for l, s in f.stats["levels"].items()}
    out = dict(colnorm=np.linalg.norm(x, axis=0))
    if name == "cfg3":
        idx = np.sort(np.random.default_rng(123).choice(g.n, 4096, replace=False))
        out.update(x_full=np.ascontiguousarray(x[:, :2]), sample_idx=idx, x_sample=np.ascontiguousarray(x[idx]))
        meta["stored"] = "x_full = columns 0,1; x_sample = all columns at sample_idx; colnorm = all columns"
    else:
        out.update(x_full=np.ascontiguousarray(x))
        meta["stored"] = "x_full = all columns"
    np.savez_compressed(os.path.join(GOLD, f"{name}_oracle_solution.npz"), **out)
    with open(os.path.join(GOLD, f"{name}_oracle_solution.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    sep = "--separate" in sys.argv
    for nm in [a for a in sys.argv[1:] if not a.startswith("--")]:
        (run_separate if sep else run)(nm)
