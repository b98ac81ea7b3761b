"""Top SASS instructions of an ncu source-page export (--print-source sass --csv):
by stall samples and by executed instructions.   python tools/sass_top.py file.csv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) >= len(h) - 1 and r[0].startswith("0x")]
num = lambda d, k: float(d.get(k, "0").replace(",", "") or 0)
tot_s = sum(num(d, "Warp Stall Sampling (All Samples)") for d in data)
tot_i = sum(num(d, "Instructions Executed") for d in data)
print(f"samples {tot_s:.0f}  warp-instructions {tot_i:.0f}")
print("--- by stall samples")
for d in sorted(data, key=lambda d: -num(d, "Warp Stall Sampling (All Samples)"))[:n]:
    print(f"{num(d,'Warp Stall Sampling (All Samples)'):7.0f} {num(d,'Instructions Executed'):10.0f}  {d['Address'][-5:]} {d['Source'].strip()[:70]}")
# opcode histogram weighted by executed instructions
from collections import Counter
c = Counter()
for d in data:
    op = d["Source"].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    c[o.split(".")[0]] += num(d, "Instructions Executed")
print("--- opcode mix (warp-instructions)")
for o, v in c.most_common(n):
    print(f"{o:10s} {v:12.0f} {100*v/tot_i:5.1f}%")
