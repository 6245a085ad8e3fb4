"""Per-kernel totals of the launches AFTER the last launch of a marker kernel in an ncu
`--metrics gpu__time_duration.sum --csv` launch list (e.g. the solve after the factorization).
    python tools/launch_tail.py launches.csv k_lu_diag_inv"""
import csv, io, sys
from collections import defaultdict
rows = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(rows) if l.startswith('"ID"'))
recs = [r for r in csv.DictReader(io.StringIO("\n".join(rows[start:]))) if r.get("Metric Name") == "gpu__time_duration.sum"]
marker = sys.argv[2]
last = max(i for i, r in enumerate(recs) if marker in r["Kernel Name"])
tail = recs[last + 1:]
agg = defaultdict(lambda: [0, 0.0])
for r in tail:
    v = float(r["Metric Value"].replace(",", ""))
    u = r.get("Metric Unit", "ns")
    ms = v * {"ns": 1e-6, "nsecond": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(u, 1e-6)
    name = r["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
    agg[name][0] += 1
    agg[name][1] += ms
tot = sum(v[1] for v in agg.values())
print(f"{len(tail)} launches after the last {marker}, {tot:.2f} ms")
for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:40s} {c:6d} {ms:9.3f} ms {ms / tot:6.3f}")
