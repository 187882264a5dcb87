"""Shared-memory bank conflicts per SASS line of an ncu report (source page),
largest first, plus the kernel's LSU / shared wavefront utilisation.

    python scripts/bank_conflicts.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, top=30):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    for k, v in zip(rows[0], rows[2]):
        if k in ("gpu__time_duration.sum", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
                 "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                 "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                 "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"):
            print(f"{k:70s} {v}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    out, tot = [], 0
    for r in rows[2:]:
        try:
            ex = int(r[ix["L1 Wavefronts Shared Excessive"]])
            w = int(r[ix["L1 Wavefronts Shared"]])
        except (ValueError, IndexError):
            continue
        tot += ex
        if w:
            out.append((ex, w, int(r[ix["Instructions Executed"]]), r[ix["Address"]][-5:],
                        r[ix["Source"]].strip()))
    out.sort(reverse=True)
    print("excessive shared wavefronts:", tot)
    for o in out[:top]:
        print(o)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
