"""Opcode histogram of a kernel's SASS per source-line range (nvdisasm -gi dump).
python tools/sass_lines.py dump.sass kernel_substr file:lo-hi ..."""
import collections
import re
import sys

path, kern = sys.argv[1], sys.argv[2]
cur = None
fn = None
ingroup = False
per = collections.defaultdict(collections.Counter)
for l in open(path):
    m = re.search(r"\.section\s+\.text\.([^,\s]+)", l)
    if m:
        fn = m.group(1)
    if "//##" in l:
        m = re.search(r"line (\d+)", l)
        f = re.search(r'File "([^"]+)"', l)
        if m and not ingroup:  # -gi: innermost location first, then the inline chain
            cur = ((f.group(1).split("/")[-1] if f else "?"), int(m.group(1)))
        ingroup = True
        continue
    ingroup = False
    if not fn or kern not in fn:
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", l)
    if m and cur:
        per[cur][m.group(2).split(".")[0]] += 1
for spec in sys.argv[3:]:
    f, r = spec.split(":")
    lo, hi = map(int, r.split("-"))
    tot = collections.Counter()
    for k in per:
        if k[0] == f and lo <= k[1] <= hi:
            tot += per[k]
    print(spec, sum(tot.values()), tot.most_common(24))
