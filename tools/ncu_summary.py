"""Summarise ncu CSV output for profiles/.

  python tools/ncu_summary.py launches <launches.csv>       per-kernel table from a
        `--metrics gpu__time_duration.sum --csv` launch list (count, total, share)
  python tools/ncu_summary.py full <report.ncu-rep> [name]  per-launch DRAM bytes, duration,
        SM throughput, registers, occupancy of a `--set full` capture (via `ncu -i --page raw --csv`)
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def _rows(text):
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def _num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def launches(path):
    rows = _rows(open(path).read())
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        unit = r.get("Metric Unit", "ns")
        v = _num(r["Metric Value"]) or 0.0
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for name, (cnt, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{name}` | {cnt} | {ms:.3f} | {ms / tot:.3f} |")
    out.append(f"| **all** | {sum(v[0] for v in agg.values())} | {tot:.3f} | 1.000 |")
    return "\n".join(out)


FULL_METRICS = {
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__time_duration.sum": "duration",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__grid_size": "grid",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_pct",
}


def full(rep, name=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = raw.splitlines()
    hdr = next(csv.reader([lines[0]]))
    units = next(csv.reader([lines[1]]))
    recs = []
    for row in csv.reader(lines[2:]):
        d = dict(zip(hdr, row))
        if name and name not in d.get("Kernel Name", ""):
            continue
        rec = {"kernel": d.get("Kernel Name", "").split("(")[0]}
        for m, k in FULL_METRICS.items():
            if m in d:
                v = _num(d[m])
                u = units[hdr.index(m)]
                if v is not None and m.startswith("dram__bytes"):
                    v *= {"byte": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}.get(u, 1)
                if v is not None and m == "gpu__time_duration.sum":
                    v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(u, 1e-6)  # -> ms
                rec[k] = v
        recs.append(rec)
    return recs


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        print(launches(sys.argv[2]))
    else:
        recs = full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
        n = len(recs)
        summ = {"launches": n}
        if n:
            for k in ("dram_read", "dram_write", "duration"):
                summ[k + "_per_launch"] = sum(r.get(k) or 0 for r in recs) / n
            tot = sum(r.get("duration") or 0 for r in recs)
            for k in ("dmma_pipe_pct", "fp64_pipe_pct", "sm_pct"):  # duration-weighted means
                if tot > 0 and any(r.get(k) is not None for r in recs):
                    summ[k + "_weighted"] = sum((r.get(k) or 0) * (r.get("duration") or 0) for r in recs) / tot
            summ["traffic_per_launch"] = summ["dram_read_per_launch"] + summ["dram_write_per_launch"]
        print(json.dumps({"summary": summ, "launches": recs}, indent=1))
