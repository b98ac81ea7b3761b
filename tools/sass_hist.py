"""Group a kernel's SASS lines (ncu --page source --print-source sass) by
execution count: where the instructions of an ncu report go.

  python tools/sass_hist.py <report.ncu-rep> <kernel-regex> [min_exec]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
min_exec = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r]
        blocks.append(cur)
    elif cur is not None:
        cur.append(r)
b = blocks[0]
hdr = b[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in b[2:] if len(r) == len(hdr)]
tot = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
samp = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print(b[0][1][:80], "instructions", tot, "samples", samp)
grp = defaultdict(lambda: [0, 0, 0])
for r in data:
    ie = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    g = grp[ie]
    g[0] += 1
    g[1] += ie
    g[2] += s
for ie, (cnt, t, s) in sorted(grp.items(), key=lambda x: -x[1][1])[:14]:
    print(f"exec={ie:>9} ninstr={cnt:>4} total={t:>11} ({100.0 * t / tot:4.1f}%) samples={s}")
if min_exec:
    for r in data:
        ie = int(r[ix["Instructions Executed"]] or 0)
        if ie >= min_exec:
            print(f'{ie:>9} {int(r[ix["Warp Stall Sampling (All Samples)"]] or 0):>6} {r[ix["Source"]][:90]}')
