"""Opcode mix of the loops of one kernel:  python tools/dev/loop_mix.py file.o 'mangled-substring' [n_atoms_in_loop]"""
import collections
import re
import subprocess
import sys

obj, pat = sys.argv[1], sys.argv[2]
want = int(sys.argv[3]) if len(sys.argv) > 3 else None
names = [l.split("Function : ")[1].strip() for l in
         subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout.split("\n") if "Function : " in l]
fn = [n for n in names if pat in n][0]
txt = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True, text=True).stdout
ins = []
for l in txt.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
loops = []
for a, op, rest in ins:
    if op.startswith("BRA"):
        t = re.search(r"0x([0-9a-f]+)", rest)
        if t and int(t.group(1), 16) < a:
            body = [x for x in ins if int(t.group(1), 16) <= x[0] <= a]
            loops.append((len(body), sum(1 for x in body if x[1].startswith("ATOMS")), body))
print(fn)
print([(n, na) for n, na, _ in loops])
sel = [l for l in loops if want is None or l[1] == want]
n, na, body = min(sel, key=lambda t: t[0])
c = collections.Counter(x[1].split(".")[0] for x in body)
print(n, "instr,", na, "ATOMS:", sorted(c.items(), key=lambda t: -t[1]))
c2 = collections.Counter(x[1] for x in body if x[1].startswith(("IMAD", "SHF", "LOP3", "PRMT", "LEA", "VIADD", "IADD3")))
print(sorted(c2.items(), key=lambda t: -t[1]))
