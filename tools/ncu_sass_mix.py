"""Per-opcode executed warp instructions from an ncu source-page CSV
(--page source --csv --print-source sass):  python tools/ncu_sass_mix.py sass.csv [units]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = next(i for i, r in enumerate(rows) if "Source" in r and any("Instructions Executed" in c for c in r))
h = rows[hdr]
src = h.index("Source")
ex = next(i for i, c in enumerate(h) if c.startswith("Instructions Executed"))
cnt, tot = Counter(), 0.0
for r in rows[hdr + 1:]:
    if len(r) <= max(src, ex) or not r[ex].replace(".", "").isdigit():
        continue
    op = r[src].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
    n = float(r[ex])
    cnt[o.split(".")[0]] += n
    tot += n
print(f"# executed warp instructions per unit (units = {units:g}); total {tot:.4g}")
for o, n in cnt.most_common(30):
    print(f"{o:10s} {n / units:14.4f}  {100 * n / tot:5.1f}%")
