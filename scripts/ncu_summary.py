"""Headline counters + stall breakdown of the kernels in an ncu report.
    python scripts/ncu_summary.py REP"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for v in rows[2:]:
    d = dict(zip(h, v))
    for k in KEYS:
        if k in d:
            print(f"{k:75s} {d[k]}")
    st = [(float(d[k]), k) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not k.endswith("not_issued") and d[k] not in ("", "n/a")]
    tot = sum(x for x, _ in st) or 1
    print("stalls: " + ", ".join(f"{k[34:]} {100 * x / tot:.1f}%"
                                  for x, k in sorted(st, reverse=True)[:8]))
    print()
