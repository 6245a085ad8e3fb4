"""Pair an ncu --set full capture of consecutive Schur-GEMM launches (ncu -s S -c C) with the
library's per-launch algorithmic work (FMMLU_TRACE lines "schur launch: ... bytes") of the same
factorization, and write the summary bench.py reads for roofline.traffic.
    python tools/pair_traffic.py ncu_summary.json schur_launch_work.txt S out.json"""
import json, re, sys
ncu = json.load(open(sys.argv[1]))
work = [tuple(float(x) for x in re.findall(r"([\d.e+]+) flops, ([\d.e+]+) bytes", l)[0])
        for l in open(sys.argv[2]) if "schur launch" in l]
s = int(sys.argv[3])
L = ncu["launches"]
rows = []
for i, l in enumerate(L):
    fl, by = work[s + i]
    traffic = (l.get("dram_read") or 0) + (l.get("dram_write") or 0)
    rows.append(dict(launch=s + i, algorithmic_bytes=by, algorithmic_flops=fl, dram_bytes=traffic,
                     ratio=traffic / by if by else None, ncu_ms=l.get("duration"), dmma_pipe_pct=l.get("dmma_pipe_pct")))
tot_t = sum(r["dram_bytes"] for r in rows)
tot_b = sum(r["algorithmic_bytes"] for r in rows)
out = dict(summary=dict(launches=len(rows), first_launch=s, traffic_per_launch=tot_t / len(rows),
                        algorithmic_bytes_per_launch=tot_b / len(rows), traffic_over_algorithmic=tot_t / tot_b,
                        note="ncu --set full (kernel replay, cold cache, serialised) of Schur-GEMM launches "
                             f"{s}..{s + len(rows) - 1} of one cfg5 factorization, paired with the library's "
                             "algorithmic bytes (32 B per updated Δ entry) of the same launches"),
           launches=rows)
json.dump(out, open(sys.argv[4], "w"), indent=1)
print(json.dumps(out["summary"]))
