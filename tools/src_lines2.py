"""Per-(file, CUDA source line) stall samples and executed instructions from an ncu source-page
export:  ncu -i rep --page source --csv --print-source cuda,sass --kernel-name regex:K > f.csv
         python tools/src_lines2.py f.csv [n]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr, fname = None, ""
agg = defaultdict(lambda: [0.0, 0.0, defaultdict(float), ""])
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
        continue
    if not hdr or len(r) != len(hdr) or not r[0].strip().isdigit():
        continue
    num = lambda i: float(r[i].replace(",", "") or 0) if r[i] not in ("", "-") else 0.0
    a = agg[(fname, int(r[0]))]
    a[0] += num(4)
    a[1] += num(7)
    a[3] = r[1].strip()[:70]
    for i in stall_cols:
        a[2][hdr[i]] += num(i)
tot = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot:.0f} instructions {ti:.0f}")
for (f, line), (s, ins, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{f[:12]:12s}{line:5d} {100*s/tot:5.1f}% inst {100*ins/ti:5.1f}% | {src[:58]:58s} | " +
          ", ".join(f"{k[6:]}:{v:.0f}" for k, v in top))
