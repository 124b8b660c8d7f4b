#!/usr/bin/env python
"""Key pipe / issue / memory metrics of every kernel in an ncu --set full report."""
import csv
import io
import subprocess
import sys

WANT = [("gpu__time_duration.sum", "us", 1e-3), ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%", 1),
        ("smsp__inst_executed.sum", "Minst", 1e-6), ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%", 1),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu%", 1),
        ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma%", 1),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64%", 1),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu%", 1),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%", 1),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1),
        ("dram__bytes_read.sum", "MB rd", 1e-6)]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    print("kernel".ljust(48), " ".join(n.rjust(7) for _, n, _ in WANT))
    for r in rows[2:]:
        vals = []
        for k, _, sc in WANT:
            try:
                vals.append(f"{float(r[h.index(k)].replace(',', '')) * sc:7.1f}")
            except (ValueError, IndexError):
                vals.append("      -")
        print(r[h.index("Kernel Name")][:48].ljust(48), " ".join(vals))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
