"""Per-source-line instruction / stall breakdown of one kernel from an ncu
report (--set full, -lineinfo build):  python scripts/ncu_lines.py REP [N_UNITS] [TOP]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, res, tot_e, tot_s = None, [], 0, 0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Line No", "Function Name") or not r[0]:
        continue
    try:
        e, s = int(r[7]), int(r[4])
    except ValueError:
        continue
    tot_e += e
    tot_s += s
    res.append((e, s, fname, r[0], r[1][:84]))
res.sort(reverse=True)
print(f"instructions per unit {tot_e / units:.1f}   stall samples {tot_s}")
for e, s, f, l, src in res[:top]:
    print(f"{e / units:7.1f} {100.0 * s / max(tot_s, 1):5.1f}% {f[:14]:14s}:{l:>5s} {src}")
