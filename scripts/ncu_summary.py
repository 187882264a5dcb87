"""Condense an ncu report into a small CSV of the metrics quoted in DESIGN.md.
python scripts/ncu_summary.py report.ncu-rep > summary.csv"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sector_hit_rate.pct",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          ",".join(METRICS)], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = csv.writer(sys.stdout)
    cols = [m for m in METRICS if m in head]
    out.writerow(["kernel"] + [f"{m} [{units[head.index(m)]}]" for m in cols])
    for r in rows[2:]:
        out.writerow([r[head.index("Kernel Name")]] + [r[head.index(m)] for m in cols])


if __name__ == "__main__":
    main(sys.argv[1])
