"""Per-kernel average device time from an ncu --metrics gpu__time_duration.sum
CSV log.   python tools/launch_table.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i0 = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i0]
ix = {n: i for i, n in enumerate(h)}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[i0 + 1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    k = r[ix["Kernel Name"]].split("(")[0]
    v = float(r[ix["Metric Value"]])
    u = r[ix["Metric Unit"]]
    v = {"ns": v / 1e3, "us": v, "ms": v * 1e3, "s": v * 1e6}.get(u, v)
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(t for _, t in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{t / n:10.2f} us/launch {n:5d} launches {100 * t / tot:5.1f}%  {k}")
