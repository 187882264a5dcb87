"""Summarise an ncu report's SASS source page: instructions per unit, stall
mix, hottest instructions.  python scripts/sass_hot.py rep.ncu-rep [units]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
totS = sum(f(r[iS]) for r in data)
totE = sum(f(r[iE]) for r in data)
print(f"instructions {totE:.0f} ({totE / units:.0f} per unit), stall samples {totS:.0f}")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = sorted(((sum(f(r[hdr.index(c)]) for r in data) / totS, c) for c in cols), reverse=True)
print(" ".join(f"{c[6:]}={100 * v:.1f}%" for v, c in agg[:8]))
for r in sorted(data, key=lambda x: -f(x[iS]))[:30]:
    print(f"{100 * f(r[iS]) / totS:5.1f}% {f(r[iE]):10.0f}  {r[1].strip()[:80]}")
