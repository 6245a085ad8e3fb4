"""bench.py — FMM-LU hot path on B200 (BASELINE.json metric: factor unknowns/s and solve
ms/RHS at ε = 1e-6, complex128, 1 B200).

Workload (N=1): BASELINE.json configs[4] = "cfg5", the largest single-GPU configuration:
wavy torus (2000×500 grid), n = 10⁶, k = 10, leaf ≤ 64, ε = 1e-6, 32 Gaussian RHS (seed 0).
One STEP = the whole hot path (every SURVEY §8(a) row): fmmlu_tree + fmmlu_factor +
fmmlu_solve through the C ABI.  Extra keys (not the headline): cfg2 (configs[1]) device-timed
steps, and cfg4 (configs[3], 8192 independent boxes) boxes/s at ε ∈ {1e-4, 1e-6, 1e-9}.
value = unknowns processed per second of step time (tree + factor + solve), summed over
ranks ("replicas only"); factor-only unknowns/s and solve ms/RHS are extra keys.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

`--impl reference` times the CPU oracle (oracle/, plain NumPy/SciPy) on a bounded sample of
the same workload family, on this box's host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import fmmlu_inputs as fi  # noqa: E402

METRIC = "FMM-LU factor unknowns/s and solve ms/RHS at eps=1e-6 (complex128, 1 B200)"
UNIT = "unknowns/s"
CFG = "cfg5"
# bounded CPU sample for the oracle: the cfg5 wavy torus recipe on a coarser grid, with the same
# points per wavelength (k scaled by sqrt(n/10^6), so the boxes compress as in cfg5), leaf and eps
ORACLE_GRID = (120, 40)
ORACLE_GRIDS = [(60, 20), (84, 28), (120, 40)]


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class Clocks:
    """Samples nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "1000"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self, first: int = 0):
        rows = self.rows[first:] if len(self.rows) > first else self.rows  # samples of the timed region
        sm = [float(r[1]) for r in rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for i, nm in enumerate(names):
                if len(r) > 4 + i and r[4 + i].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ncu --set full summaries committed under profiles/ (tools/ncu_summary.py full): DRAM traffic
# per launch of the kernel behind each class, for the roofline's "traffic" field
NCU_FULL = {"schur": "k_gemm_schur", "ef": "k_gemm_store", "panel": "k_gemm_store", "qr": "k_gemm_store",
            "inv": "k_gj_panel", "cpqr": "k_pchol_cluster", "gather": "k_proxy", "build": "k_build_level"}


def ncu_traffic(cls: str):
    """(bytes per launch, source, extra) from the committed ncu full capture of the bench config's
    dominant kernel (profiles/r2_schur_traffic_cfg5.json: launches paired with their algorithmic
    bytes), else the newest generic summary, else (None, None, {})."""
    kern = NCU_FULL.get(cls)
    if not kern:
        return None, None, {}
    pdir = os.path.join(ROOT, "profiles")
    paired = os.path.join(pdir, f"r2_{cls}_traffic_{CFG}.json")
    if os.path.exists(paired):
        try:
            d = json.load(open(paired))["summary"]
            return float(d["traffic_per_launch"]), f"profiles/{os.path.basename(paired)}", {
                "traffic_launches": d["launches"], "traffic_algorithmic_bytes_per_launch": d["algorithmic_bytes_per_launch"],
                "traffic_over_algorithmic": d["traffic_over_algorithmic"]}
        except Exception:
            pass
    cands = sorted(f for f in os.listdir(pdir) if f.endswith(f"ncu_full_{kern}.json")) if os.path.isdir(pdir) else []
    if not cands:
        return None, None, {}
    try:
        d = json.load(open(os.path.join(pdir, cands[-1])))
        big = [l for l in d["launches"] if l.get("dram_read") is not None]
        return float(d["summary"]["traffic_per_launch"]), f"profiles/{cands[-1]} ({len(big)} launches)", {}
    except Exception:
        return None, None, {}


def max_over_ranks(t_ms: float, world: int, device=None) -> float:
    """Max of a per-rank time over all ranks (all_reduce MAX; a no-op at world = 1).  Works on
    any backend: the tensor lives on `device` (cuda under NCCL, cpu under gloo)."""
    if world <= 1:
        return float(t_ms)
    import torch
    tt = torch.tensor([float(t_ms)], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    return float(tt.item())


def job_throughput(n_per_rank: int, world: int, t_step_ms: float) -> float:
    """Whole-job unknowns/s: every rank factors its own replica (weak scaling),
    timed as the slowest rank."""
    return world * n_per_rank / (t_step_ms * 1e-3)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def oracle_sample(grid=ORACLE_GRID):
    """The cfg5-family sample the CPU oracle is timed on: the same wavy torus recipe on a coarser
    grid at cfg5's points per wavelength (k = 10·sqrt(n/10⁶)), leaf, ε and 32 RHS (block-mode
    oracle); the default grid is ≈ 10–30 s of host work."""
    c = dict(fi.CONFIGS[CFG])
    g = fi.wavy_torus(*grid)
    c["k"] = c["k"] * math.sqrt(g.n / 1e6)
    b = fi.gaussian_rhs(g.n, c["nrhs"], 0)
    return c, g, b


def oracle_step(c, g, b):
    from oracle import rss
    t0 = time.perf_counter()
    f = rss.factor(g.points, g.normals, g.weights, c["k"], c["eps"], c["leaf_max"], mode="block")
    rss.solve(f, b)
    return time.perf_counter() - t0


def _sample_desc(g, c, grid=ORACLE_GRID):
    return (f"oracle (NumPy/SciPy, untuned, block mode) tree+factor+solve of the {CFG} wavy torus recipe on a "
            f"{grid[0]}x{grid[1]} grid (n={g.n}; full {CFG} is n=10^6) at cfg5's points per wavelength "
            f"(k={c['k']:.3f} = 10*sqrt(n/1e6)), leaf {c['leaf_max']}, eps {c['eps']:g}, {c['nrhs']} RHS")


def run_reference(args):
    """CPU oracle arm (test-infrastructure oracle, untuned) on a bounded sample."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    # per-step sample sized so that warmup + steps finish within a few minutes: calibrate on the
    # smallest grid (untimed), then take the largest grid whose extrapolated time (∝ n^1.5) fits
    budget = max(3.0, min(30.0, 150.0 / max(1, args.warmup + args.steps)))
    c0, g0, b0 = oracle_sample(ORACLE_GRIDS[0])
    t_small = oracle_step(c0, g0, b0)
    grid = ORACLE_GRIDS[0]
    for gr in ORACLE_GRIDS:
        if t_small * ((gr[0] * gr[1]) / (g0.n)) ** 1.5 <= budget:
            grid = gr
    c, g, b = oracle_sample(grid)
    times = []
    for it in range(args.warmup + args.steps):
        dt = oracle_step(c, g, b)
        if it >= args.warmup:
            times.append(dt)
    t = float(np.mean(times))
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    value = g.n / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": f"{CFG} family sample: wavy torus n={g.n}, k={c['k']:.3f}, leaf {c['leaf_max']}, "
                               f"eps {c['eps']:g}, {c['nrhs']} RHS", "sample_of": CFG},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": _sample_desc(g, c, grid)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_sample():
    c, g, b = oracle_sample()
    dt = oracle_step(c, g, b)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"value": g.n / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": _sample_desc(g, c) + f" ({dt:.1f} s)"}


def bench_cfg2(F, dev, stream, flush, steps: int = 5, warmup: int = 2):
    """Extra key: BASELINE configs[1] (ellipsoid, n = 2·10⁴, 4 RHS), the same step, device-timed."""
    import torch
    c = fi.CONFIGS["cfg2"]
    g = fi.config_geometry("cfg2")
    b = np.asfortranarray(fi.gaussian_rhs(g.n, c["nrhs"], 0))
    P, N, W = (torch.from_numpy(a).to(dev) for a in (g.points, g.normals, g.weights))
    B = torch.from_numpy(np.ascontiguousarray(b.T)).to(dev)
    X = torch.empty_like(B)
    ms, fac, sol = [], [], []
    h = None
    for it in range(warmup + steps):
        if h is not None:
            h.close()
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h = F.FmmLu(P, N, W, c["leaf_max"])
        h.set_stream(stream.cuda_stream)
        h.factor(c["k"], c["eps"])
        X.copy_(B)
        h.solve(X, nrhs=c["nrhs"])
        e1.record(stream)
        torch.cuda.synchronize()
        if it >= warmup:
            st = h.stats()
            ms.append(e0.elapsed_time(e1))
            fac.append(st["t_factor_ms"])
            sol.append(st["t_solve_ms"])
    h.close()
    t = float(np.mean(ms))
    return {"workload": f"cfg2 (BASELINE configs[1]): ellipsoid (0.5,1,2) n={g.n}, k=2pi, leaf 64, eps 1e-6, "
                        f"{c['nrhs']} RHS", "unknowns_per_s": g.n / (t * 1e-3), "ms_per_step": t,
            "factor_unknowns_per_s": g.n / (float(np.mean(fac)) * 1e-3),
            "solve_ms_per_rhs": float(np.mean(sol)) / c["nrhs"], "steps": steps,
            "device_ms_steps": [round(v, 2) for v in ms]}


def bench_cfg4(F):
    """Extra key: BASELINE configs[3] (8192 independent boxes, b = 256, 1024 near, 512 proxy
    points, k = 10): batched ID + elimination, boxes/s at each ε (one warm-up + one timed run;
    device time measured inside fmmlu_boxes with CUDA events)."""
    d = fi.box_batch(8192)
    rho = 1.5 * math.sqrt(3) / 2 * d["h"]
    out = {"workload": "cfg4 (BASELINE configs[3]): 8192 boxes, b=256, 1024 near DOFs, 512 proxy points, k=10"}
    for eps in (1e-4, 1e-6, 1e-9):
        F.boxes(d["pts"], d["nrm"], d["npts"], d["nnrm"], d["w"], 10.0, eps, 512, rho, want_perm=False)
        r = F.boxes(d["pts"], d["nrm"], d["npts"], d["nnrm"], d["w"], 10.0, eps, 512, rho, want_perm=False)
        out[f"eps={eps:g}"] = {"ms": r["ms"], "boxes_per_s": 8192 / (r["ms"] * 1e-3),
                               "model_gflop": r["gflop"], "model_tflops": r["gflop"] / r["ms"],
                               "mean_rank": float(r["ranks"].mean())}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the cfg2 / cfg4 extra keys")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    from paper_2201_07325_b200 import fmmlu as F
    F.load()

    c = fi.CONFIGS[CFG]
    g = fi.config_geometry(CFG)
    n, nrhs = g.n, c["nrhs"]
    b_host = np.asfortranarray(fi.gaussian_rhs(n, nrhs, 0))
    # inputs resident in HBM for the device-timed leg
    P = torch.from_numpy(g.points).to(dev)
    N = torch.from_numpy(g.normals).to(dev)
    W = torch.from_numpy(g.weights).to(dev)
    B = torch.from_numpy(np.ascontiguousarray(b_host.T)).to(dev)  # (nrhs, n) C = n×nrhs col-major
    X = torch.empty_like(B)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    def step_device():
        h = F.FmmLu(P, N, W, c["leaf_max"])
        h.set_stream(stream.cuda_stream)
        h.factor(c["k"], c["eps"])
        X.copy_(B)
        h.solve(X, nrhs=nrhs)
        return h

    # end-to-end leg: inputs in pinned host memory; the library copies them in (fmmlu_tree,
    # fmmlu_solve) and the solution back out inside the calls
    pts_p = torch.from_numpy(g.points).pin_memory()
    nrm_p = torch.from_numpy(g.normals).pin_memory()
    wts_p = torch.from_numpy(g.weights).pin_memory()
    rhs_p = torch.from_numpy(np.ascontiguousarray(b_host.T)).pin_memory()  # (nrhs, n) = n×nrhs col-major
    x_p = torch.empty_like(rhs_p).pin_memory()

    def step_e2e():
        h = F.FmmLu(pts_p, nrm_p, wts_p, c["leaf_max"])
        h.set_stream(stream.cuda_stream)
        h.factor(c["k"], c["eps"])
        x_p.copy_(rhs_p)
        h.solve(x_p, nrhs=nrhs)  # H2D of the rhs and D2H of the result inside the call
        return h, x_p.numpy().T

    # the clock sampler (an nvidia-smi process) starts before the warm-up, so its start-up does not
    # compete with the host side of the first timed step; only the timed region's samples are reported
    clk = Clocks(torch.cuda.current_device()).__enter__()
    h = None
    for _ in range(args.warmup):
        if h is not None:
            h.close()  # one handle alive at a time (a cfg5 factorization holds ≈ 45 GB of factors)
        h = step_device()
    torch.cuda.synchronize()
    import gc
    gc.collect()
    gc.disable()  # no Python collector pauses inside the timed regions (library work is unaffected)

    # ---- device-timed leg (CUDA events on the launch stream, L2 flushed between steps)
    ev = []
    stats = []
    clk_first = len(clk.rows)
    try:
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            h.close()  # the previous step's handle is released outside the timed region
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            h = step_device()
            e1.record(stream)
            ev.append((e0, e1))
            stats.append(h.stats())
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
    finally:
        clk.__exit__(None, None, None)
    dev_detail = [[round(s_["t_tree_ms"], 1), round(s_["t_factor_ms"], 1), round(s_["t_sync_wait_ms"], 1),
                   round(s_["t_solve_ms"], 1)] for s_ in stats]
    ms = [a.elapsed_time(b) for a, b in ev]
    t_step = max_over_ranks(float(np.mean(ms)), world, dev)
    st = stats[-1]
    t_fac = float(np.mean([s["t_factor_ms"] for s in stats]))
    t_sol = float(np.mean([s["t_solve_ms"] for s in stats]))
    t_tree = float(np.mean([s["t_tree_ms"] for s in stats]))

    # nrhs = 1 solve latency on the last factorization ("also report the nrhs=1 latency")
    x1 = B[:1].clone()
    for _ in range(3):
        h.solve(x1, nrhs=1)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        x1.copy_(B[:1])
        h.solve(x1, nrhs=1)
    e1.record(stream)
    torch.cuda.synchronize()
    solve1_ms = e0.elapsed_time(e1) / 5
    h.close()  # its device blocks go back to the library's cache for the e2e leg's handles

    # ---- end-to-end leg through the public API with host buffers
    e2e_ms = []
    e2e_detail = []  # per step: library-reported tree / factor / factor-wait / solve ms
    resid = None
    for _ in range(2):  # untimed warm-up of the host-buffer path (first calls pay one-time setup)
        hw, _x = step_e2e()
        hw.close()
    h2 = None
    for _ in range(args.steps):
        if h2 is not None:
            h2.close()  # the previous step's handle is released outside the timed region
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h2, x = step_e2e()  # returns after the D2H of the solution (the call synchronises)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        s2 = h2.stats()
        e2e_detail.append([round(s2["t_tree_ms"], 1), round(s2["t_factor_ms"], 1), round(s2["t_sync_wait_ms"], 1),
                           round(s2["t_solve_ms"], 1)])
    # residual of the last e2e solve with the GPU brute-force matvec
    x = np.asfortranarray(x)
    Ax = h2.matvec(c["k"], x)
    resid = float(np.max(np.linalg.norm(Ax - b_host, axis=0) / np.linalg.norm(b_host, axis=0)))
    h2.close()
    t_e2e = max_over_ranks(float(np.mean(e2e_ms)), world, dev)

    # ---- roofline of the dominant kernel class (events recorded inside libfmmlu)
    cls = F.KERNEL_CLASSES
    cms = st["class_ms"][:len(cls)]
    dom = int(np.argmax(cms))
    dmma_tf = F.probe_fp64(1)
    peaks = _peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    fl, by, t = st["class_flops"][dom], st["class_bytes"][dom], cms[dom]
    per_launch = max(1, st["class_launches"][dom])
    traffic, traffic_src, traffic_extra = ncu_traffic(cls[dom])
    if cls[dom] in ("schur", "ef", "panel", "qr"):
        achieved = fl / (t * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": dmma_tf, "unit": "TFLOP/s",
                "frac": achieved / dmma_tf, "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": by / per_launch, "kernel": cls[dom],
                "peak_source": "FP64 DMMA m8n8k4 probe measured in this run (MEASURED_PEAKS has no FP64 entry)",
                "flops_per_launch": fl / per_launch, "ms_per_launch": t / per_launch, **traffic_extra}
    elif cls[dom] in ("build", "gather", "solve", "apply"):
        achieved = by / (t * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "traffic_source": traffic_src, "kernel": cls[dom], "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "bytes_per_launch": by / per_launch, "ms_per_launch": t / per_launch}
    else:
        dfma_tf = F.probe_fp64(0)
        achieved = fl / (t * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": dfma_tf, "unit": "TFLOP/s",
                "frac": achieved / dfma_tf, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": cls[dom],
                "peak_source": "FP64 DFMA probe measured in this run",
                "flops_per_launch": fl / per_launch, "ms_per_launch": t / per_launch}
    breakdown = {cls[i]: {"ms": round(cms[i], 3), "share": round(cms[i] / max(1e-9, sum(cms)), 4),
                          "tflops": round(st["class_flops"][i] / max(1e-9, cms[i]) / 1e9, 3),
                          "gbs": round(st["class_bytes"][i] / max(1e-9, cms[i]) / 1e6, 1),
                          "frac_fp64": round(st["class_flops"][i] / max(1e-9, cms[i]) / 1e9 / dmma_tf, 4),
                          "frac_hbm": round(st["class_bytes"][i] / max(1e-9, cms[i]) / 1e6 / hbm, 4)}
                 for i in range(len(cls))}


    extras = {}
    if not args.no_extras:
        extras["cfg2"] = bench_cfg2(F, dev, stream, flush)
        extras["cfg4"] = bench_cfg4(F)

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample()
    h2d = g.points.nbytes + g.normals.nbytes + g.weights.nbytes + b_host.nbytes
    d2h = b_host.nbytes
    line = {
        "metric": METRIC, "value": job_throughput(n, world, t_step), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": f"{CFG} (BASELINE configs[4]): wavy torus 2000x500 grid n={n}, k={c['k']:g}, "
                               f"leaf {c['leaf_max']}, eps {c['eps']:g}, {nrhs} RHS",
                   "step": "fmmlu_tree + fmmlu_factor + fmmlu_solve (device-resident inputs)",
                   "parallelism": f"replicas x{world}", "l2": "flushed (256 MB write) between steps"},
        "factor_unknowns_per_s": n / (t_fac * 1e-3),
        "solve_ms_per_rhs": t_sol / nrhs,
        "solve_ms_nrhs1": solve1_ms,
        "tree_ms": t_tree, "factor_ms": t_fac, "solve_ms": t_sol,
        "n0": st["n0"], "peak_mem_bytes": st["peak_bytes"], "factor_bytes": st["factor_bytes"],
        "residual": resid,
        "e2e": {"value": job_throughput(n, world, t_e2e), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e, "ms_steps": [round(v, 2) for v in e2e_ms],
                "lib_tree_factor_wait_solve_ms": e2e_detail,
                "host_buffers": "pinned",
                "timing": "host wall clock around tree+factor+solve incl. H2D/D2H, mean of K steps"},
        "gpu_launches": int(sum(s_["n_launches"] for s_ in stats)),  # all K timed steps
        "gpu_launches_per_step": int(st["n_launches"]),
        "device_ms_steps": [round(v, 2) for v in ms],
        "device_lib_tree_factor_wait_solve_ms": dev_detail,
        "roofline": roof,
        "kernel_breakdown": breakdown,
        "clocks": clk.summary(clk_first),
        "cpu_baseline": cpu,
        "extra_configs": extras,
        "paper_context": {"note": "PAPER.md Table 2 (L2512), MATLAB on 1 CPU core, quadrature-corrected wiggly "
                                  "torus at eps 5e-7: a different matrix and machine, context only",
                          "n": 1075200, "t_f_s": 9756.3, "factor_unknowns_per_s": 110, "t_s_s": 12.1},
    }
    gc.enable()
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
