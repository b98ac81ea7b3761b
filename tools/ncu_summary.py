#!/usr/bin/env python
"""Summarise ncu output into the files committed under profiles/.

  python tools/ncu_summary.py launches <launches.csv> <out.txt>
      per-kernel launch counts and mean/total gpu__time_duration (cold-cache,
      serialised -- compare SHARES, not absolutes)
  python tools/ncu_summary.py full <report.ncu-rep> <out.txt> [<traffic.json>]
      key metrics of every profiled kernel of a --set full capture, and the
      per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
      that bench.py reports as roofline.traffic
"""

from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

STAGE_OF = [  # kernel-name regex -> bench stage name (the last capture of each kernel wins)
    (r"views_project_fwd_kernel|project_fwd_kernel", "project"),
    (r"onesweep_kernel<unsigned int, (16|4)", "sort_u32"),
    (r"emit_scan_kernel", "scan_emit"),
    (r"et_expand_kernel|et_colsum_kernel", "tile_counts"),
    (r"et_colscan_kernel|et_place_kernel", "tile_emit"),
    (r"segsort_small_kernel", "segsort"),
    (r"ranges_u32_kernel", "tile_sort_ranges"),
    (r"raster_fwd_kernel", "raster_fwd"),
    (r"raster_bwd_rec_kernel", "raster_bwd"),
    (r"views_project_bwd|project_bwd_kernel", "project_bwd"),
]


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "").replace("gs::", "")


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[short(d["Kernel Name"])].append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"{'kernel':60s} {'launches':>8s} {'mean_us':>10s} {'total_us':>10s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        lines.append(f"{k[:60]:60s} {len(v):8d} {sum(v) / len(v) / 1e3:10.2f} {sum(v) / 1e3:10.1f} "
                     f"{sum(v) / tot * 100:6.1f}%")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Waves Per SM",
        "Eligible Warps Per Scheduler", "No Eligible", "L1/TEX Hit Rate", "L2 Hit Rate"]


def full(reps, out, traffic_out=None):
    """reps: one .ncu-rep or several, comma-separated (their summaries are
    concatenated and their per-stage traffic merged)."""
    lines, by_kernel = [], {}
    for i, rep in enumerate(reps.split(",")):
        ln, bk = _full_one(rep, f"{i}." if "," in reps else "")
        lines += ln
        by_kernel.update(bk)
    traffic = {}
    for (stage, _), v in by_kernel.items():
        traffic[stage] = traffic.get(stage, 0.0) + v
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_out:  # rewritten from this capture only (no stale entries)
        json.dump({k: int(v) for k, v in traffic.items()}, open(traffic_out, "w"), indent=1)


def _full_one(rep, tag):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    hdr = rows[0]
    ki, mi, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index(
        "Metric Value")
    idi = hdr.index("ID")
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        if r[mi] in KEYS:
            per[r[idi]][r[mi]] = f"{r[vi]} {r[ui]}".strip()
            names[r[idi]] = short(r[ki])
    rrows = list(csv.reader(io.StringIO(raw)))
    rh = rrows[0]
    by_kernel = {}
    stalls = {}
    for r in rrows[2:]:
        if len(r) != len(rh):
            continue
        d = dict(zip(rh, r))
        kid = d["ID"]
        try:
            rd = float(d.get("dram__bytes_read.sum", "0").replace(",", ""))
            wr = float(d.get("dram__bytes_write.sum", "0").replace(",", ""))
        except ValueError:
            rd = wr = 0.0
        # raw page units may be in bytes or scaled; normalise via the unit row
        # the unit row gives each metric its own scale (reads in Mbyte, writes in Gbyte, ...)
        units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        unit = lambda m: units.get(rrows[1][rh.index(m)], 1) if m in rh else 1
        rd *= unit("dram__bytes_read.sum")
        wr *= unit("dram__bytes_write.sum")
        per[kid]["dram_bytes_read+write"] = f"{rd + wr:.0f} byte"
        st = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    st.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(x for x, _ in st) or 1.0
        stalls[kid] = ", ".join(f"{n} {x / tot * 100:.0f}%" for x, n in sorted(st, reverse=True)[:5])
        nm = names.get(kid, short(d.get("Kernel Name", "")))
        for pat, stage in STAGE_OF:
            if re.search(pat, d.get("Kernel Name", "")):
                # the last capture of each kernel wins (warmed-up frame); a
                # stage made of several kernels sums them
                by_kernel[(stage, short(d.get("Kernel Name", "")))] = rd + wr
    lines = []
    for kid in sorted(per, key=lambda x: int(x)):
        lines.append(f"[{tag}{kid}] {names.get(kid, '?')}")
        for k in KEYS + ["dram_bytes_read+write"]:
            if k in per[kid]:
                lines.append(f"    {k:32s} {per[kid][k]}")
        if kid in stalls:
            lines.append(f"    {'top stall reasons':32s} {stalls[kid]}")
    return lines, by_kernel


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
