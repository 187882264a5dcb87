"""Executed SASS opcodes per unit (and their stall share) of an ncu report.
    python scripts/ncu_ops.py REP UNITS"""
import csv
import subprocess
import sys
from collections import Counter

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
ce, cs = Counter(), Counter()
for r in rows[2:]:
    op = r[1].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    ce[o] += int(r[iE])
    cs[o] += int(r[iS])
tot_s = sum(cs.values()) or 1
print(f"total {sum(ce.values()) / units:.1f} per unit")
for o, v in ce.most_common(40):
    print(f"{o:28s} {v / units:8.1f}  stall {100 * cs[o] / tot_s:5.1f}%")
