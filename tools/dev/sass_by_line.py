"""Per-source-line instruction counts of the hottest loop:
    nvdisasm -g -c x.cubin > x.dis; python tools/dev/sass_by_line.py x.cubin x.dis src.cu [top]"""
import re
import subprocess
import sys
from collections import Counter, defaultdict

cubin, dis, srcfile = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(dis).read().split('\n')
cur = None
ins = []
for l in lines:
    m = re.search(r'line (\d+)', l)
    if '//##' in l and m:
        cur = int(m.group(1)) if srcfile.split('/')[-1] in l else ('other', int(m.group(1)))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)', l)
    if m:
        ins.append((int(m.group(1), 16), m.group(3), cur))
out = subprocess.run(f"cuobjdump -sass {cubin} | python3 {sys.path[0]}/sass_mix.py 1", shell=True,
                     capture_output=True, text=True).stdout
m = re.search(r'^loop 0x([0-9a-f]+)-0x([0-9a-f]+)', out, re.M)
lo, hi = int(m.group(1), 16), int(m.group(2), 16)
body = [x for x in ins if lo <= x[0] <= hi]
print(len(body), "instrs in loop")
bysrc = defaultdict(Counter)
for a, op, c in body:
    bysrc[c][op.split('.')[0]] += 1
src = open(srcfile).read().split('\n')
for c, cnt in sorted(bysrc.items(), key=lambda t: -sum(t[1].values()))[:top]:
    txt = src[c - 1].strip()[:64] if isinstance(c, int) else str(c)
    print(f"{sum(cnt.values()):5d}  L{c}: {txt:64s} {dict(cnt.most_common(5))}")
