"""Aggregate an ncu `--page source --csv --print-source cuda,sass` dump per CUDA
source line: warp-stall samples and executed warp instructions (top N)."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = []
fname = "?"
hdr = None
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0] or not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        inst = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    rows.append((samp, inst, fname, int(r[0]), r[1][:90]))
ts = sum(x[0] for x in rows) or 1
ti = sum(x[1] for x in rows) or 1
print(f"total samples {ts}, warp instructions {ti}")
for samp, inst, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*samp/ts:5.1f}% smp {100*inst/ti:5.1f}% inst  {f}:{ln}  {src}")

# stall-reason totals per phase range: python tools/ncu_lines.py dump.csv N file:lo-hi ...
if len(sys.argv) > 3:
    ranges = []
    for spec in sys.argv[3:]:
        f, r = spec.split(":")
        lo_, hi_ = map(int, r.split("-"))
        ranges.append((f, lo_, hi_))
    import collections
    fname = "?"
    hdr = None
    acc = {rg: collections.Counter() for rg in ranges}
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        d = dict(zip(hdr[2:], r[2:]))
        ln = int(r[0])
        for rg in ranges:
            if rg[0] == fname and rg[1] <= ln <= rg[2]:
                for k, v in d.items():
                    if k.startswith("stall_") and "Not Issued" not in k:
                        try:
                            acc[rg][k] += int(v)
                        except ValueError:
                            pass
    for rg, c in acc.items():
        tot = sum(c.values()) or 1
        print(rg, tot, ", ".join(f"{k[6:]} {100*v/tot:.0f}%" for k, v in c.most_common(6)))
