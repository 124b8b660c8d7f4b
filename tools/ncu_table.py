#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --csv` launch list:
the last LAST launches (one call), time and DRAM bytes per kernel."""
import collections
import csv
import sys


def table(path, last):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = collections.OrderedDict()
    for r in rows[1:]:
        d.setdefault(int(r[ii]), {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    ids = sorted(d)[-last:]
    tot = 0.0
    for i in ids:
        e = d[i]
        t = e.get("gpu__time_duration.sum", 0) / 1e3
        tot += t
        print(f"  {e['k'][:64]:64s} {t:8.1f} us  {e.get('dram__bytes_read.sum', 0) / 1e6:8.1f} MB")
    print(f"  total {tot:.1f} us")


if __name__ == "__main__":
    table(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 7)
