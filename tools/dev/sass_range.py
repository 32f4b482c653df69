"""Instruction mix of one address range of a SASS dump:
    cuobjdump -sass x.cubin | python tools/dev/sass_range.py 0x580 0x5e60 [units]"""
import re
import sys
from collections import Counter

lo, hi = int(sys.argv[1], 16), int(sys.argv[2], 16)
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
c = Counter()
for l in sys.stdin:
    m = re.match(r'\s+/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)', l)
    if m and lo <= int(m.group(1), 16) <= hi:
        c[m.group(3)] += 1
print(sum(c.values()), f"{sum(c.values()) / units:.2f} per unit")
print(", ".join(f"{k} {v}" for k, v in c.most_common()))
