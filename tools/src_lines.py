"""Per-CUDA-source-line stall samples and executed instructions from an ncu
source-page export (--print-source cuda,sass --csv).  python tools/src_lines.py f.csv [n]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
agg = defaultdict(lambda: [0.0, 0.0, defaultdict(float), ""])
stall_cols = []
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if not hdr or len(r) != len(hdr) or not r[0].strip().isdigit():
        continue  # (lines whose source text ncu did not quote cleanly are skipped)
    line = int(r[0])
    num = lambda i: float(r[i].replace(",", "") or 0) if i < len(r) and r[i] not in ("", "-") else 0.0
    a = agg[line]
    a[0] += num(4)
    a[1] += num(7)
    a[3] = r[1].strip()[:80]
    for i in stall_cols:
        a[2][hdr[i]] += num(i)
tot = sum(v[0] for v in agg.values()) or 1
print(f"total samples {tot:.0f}")
for line, (s, ins, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{line:5d} {100*s/tot:5.1f}% inst {ins:10.0f} | {src[:60]:60s} | " + ", ".join(f"{k[6:]}:{v:.0f}" for k, v in top))
