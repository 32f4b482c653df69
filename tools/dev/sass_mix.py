"""Instruction mix of the hottest loop in a SASS dump (by pipe class).
    cuobjdump -sass x.cubin | python tools/dev/sass_mix.py [units_per_iteration]"""
import re
import sys
from collections import Counter

lines = [l for l in sys.stdin.read().split('\n') if re.match(r'\s+/\*[0-9a-f]+\*/', l)]
ins = []
for l in lines:
    m = re.match(r'\s+/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*?);', l)
    if m:
        ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
# backward branches define loops; take the loop containing the most ATOMS
best = None
for i, (addr, op, rest) in enumerate(ins):
    if op.startswith('BRA'):
        t = re.search(r'0x([0-9a-f]+)', rest)
        if t and int(t.group(1), 16) < addr:
            body = [x for x in ins if int(t.group(1), 16) <= x[0] <= addr]
            na = sum(1 for x in body if x[1].startswith('ATOMS'))
            if na:
                sp = sum(1 for x in body if x[1].startswith(('LDL', 'STL')))
                print(f"# loop 0x{int(t.group(1), 16):x}-0x{addr:x}: {len(body)} instr, {na} ATOMS, {sp} LDL/STL")
for i, (addr, op, rest) in enumerate(ins):
    if op.startswith('BRA'):
        t = re.search(r'0x([0-9a-f]+)', rest)
        if t and int(t.group(1), 16) < addr:
            lo, hi = int(t.group(1), 16), addr
            body = [x for x in ins if lo <= x[0] <= hi]
            na = sum(1 for x in body if x[1].startswith('ATOMS'))
            if best is None or na > best[0]:
                best = (na, lo, hi, body)
na, lo, hi, body = best
units = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
ALU = ('IADD3', 'LOP3', 'SHF', 'PRMT', 'FMNMX', 'ISETP', 'SEL', 'LEA', 'VIMNMX', 'IMNMX', 'PLOP3', 'VIADD', 'MOV',
       'FSEL', 'P2R', 'R2P', 'IABS', 'POPC', 'FLO', 'BMSK', 'SGXT', 'LEA.HI', 'CS2R', 'VIADDMNMX')
FMA = ('IMAD', 'FFMA', 'FMUL', 'FADD', 'HFMA2', 'HADD2', 'HMUL2', 'IDP', 'IMUL')
c = Counter()
cls = Counter()
for _, op, _ in body:
    base = op.split('.')[0]
    c[base] += 1
    if base in ('ATOMS', 'RED', 'LDS', 'STS', 'SHFL', 'LDG', 'LD', 'LDSM'):
        cls['mio/lsu'] += 1
    elif base in ('F2I', 'I2F', 'MUFU', 'F2F', 'F2FP', 'I2I', 'FRND'):
        cls['xu'] += 1
    elif base in FMA:
        cls['fma'] += 1
    elif base.startswith('U') or base in ('BRA', 'BSSY', 'BSYNC', 'NOP', 'S2UR', 'LDCU'):
        cls['uniform/ctl'] += 1
    else:
        cls['alu'] += 1
print(f"loop 0x{lo:x}-0x{hi:x}: {len(body)} instr, {na} ATOMS; per unit (/{units}):")
for k, v in cls.most_common():
    print(f"  {k:12s} {v:5d}  {v / units:7.2f}")
print(' ', ', '.join(f"{k} {v}" for k, v in c.most_common(30)))
