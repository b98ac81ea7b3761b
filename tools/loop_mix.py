"""Instruction mix of the hottest loop body of a kernel in the built library
(cuobjdump SASS; the loop = the backward branch with the largest body).

  python tools/loop_mix.py <mangled-name-substring>
"""
import re
import subprocess
import sys
from collections import Counter

LIB = sys.argv[2] if len(sys.argv) > 2 else "paper_2312_02121_b200/libsplat_b200.so"
name = sys.argv[1]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
body = next(f for f in funcs if f.split("\n", 1)[0].strip().find(name) >= 0 and "Function" not in f[:0])
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
addr = {a: i for i, (a, _) in enumerate(ins)}
best = None
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA (0x[0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr and any("MUFU.EX2" in x for _, x in ins[addr[tgt]:i]) and (
                best is None or i - addr[tgt] < best[1] - best[0]):
            best = (addr[tgt], i)
lo, hi = best
FMA = ("FFMA", "FMUL", "FADD", "IMAD", "HFMA2", "FMUL2", "FFMA2", "FADD2")
c = Counter()
for _, t in ins[lo:hi + 1]:
    op = t.split()[0] if not t.startswith("@") else t.split()[1]
    base = op.split(".")[0]
    c[base] += 1
fma = sum(v for k, v in c.items() if k in FMA)
print(f"loop [{lo},{hi}] instructions {hi - lo + 1}, fma-pipe {fma}")
print(dict(c.most_common()))
