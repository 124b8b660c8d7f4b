#!/usr/bin/env python
"""Key pipe / issue / memory metrics of every kernel in an ncu --set full report."""
import csv
import io
import subprocess
import sys

UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
WANT = [("gpu__time_duration.sum", "us", None), ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%", 1),
        ("smsp__inst_executed.sum", "Minst", 1e-6), ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%", 1),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu%", 1),
        ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma%", 1),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64%", 1),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu%", 1),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%", 1),
        ("dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "dram%", 1),
        ("dram__bytes_read.sum", "MB rd", None)]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print("kernel".ljust(48), " ".join(n.rjust(7) for _, n, _ in WANT))
    for r in rows[2:]:
        vals = []
        for k, _, sc in WANT:
            try:
                i = h.index(k)
                f = sc if sc is not None else UNIT.get(units[i], 1.0)
                vals.append(f"{float(r[i].replace(',', '')) * f:7.1f}")
            except (ValueError, IndexError):
                vals.append("      -")
        print(r[h.index("Kernel Name")][:48].ljust(48), " ".join(vals))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
