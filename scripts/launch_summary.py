"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel and grid:  python scripts/launch_summary.py launches.csv [top]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
ix = {k: j for j, k in enumerate(h)}
agg, tot = collections.OrderedDict(), 0.0
for r in rows[start + 1:]:
    if len(r) < len(h):
        continue
    name = re.sub(r"\(.*", "", r[ix["Kernel Name"]])[:70]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(r[ix["Metric Unit"]], 1.0)
    a = agg.setdefault((name, r[ix["Grid Size"]], r[ix["Block Size"]]), [0, 0.0])
    a[0] += 1
    a[1] += v
    tot += v
print(f"total {tot:.1f} us over {sum(a[0] for a in agg.values())} launches")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{a[1]:10.1f} us {100 * a[1] / tot:5.1f}% {a[0]:5d} x {a[1] / a[0]:8.1f}  {k[0]} grid {k[1]} block {k[2]}")
