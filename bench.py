#!/usr/bin/env python
"""Benchmark: differentiable Gaussian-splatting fwd+bwd on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One "step" = on every rank, the full hot path for that rank's view(s):
project -> scan/emit/sort/ranges -> raster fwd -> raster bwd -> projection
bwd, plus (N > 1) the NCCL sum-allreduce of the per-Gaussian gradients.
Inputs are seeded synthetic scenes with BASELINE.json's distributions
(paper_2312_02121_b200/scenes.py).  Default workload: config 3 -- the
32-view batch of 3M Gaussians at 1297x840 that BASELINE.json's metric is
quoted on at 1/2/4/8 B200 -- split by view across ranks (strong scaling).
--config 4 is the 4K frame split by tile-row bands; --config 0/1/2 are single
views (weak scaling: rank r renders camera r of a ring).

`--gpus N` without torchrun re-launches itself under
torch.distributed.run (one rank per GPU, 127.0.0.1).

Rank 0 prints ONE JSON line (keys documented in DESIGN.md §7).
`--impl reference` times the CPU oracle port (oracle/, fp64) on the host
cores -- each step one full fwd+bwd view of the same workload -- and prints
the same line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd frames/sec and Gaussian-pixel evals/s at 1/2/4/8 B200 (vs roofline)"
L2_FLUSH_BYTES = 192 << 20  # > 1.5x the 126 MB L2


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-graph", action="store_true")
    p.add_argument("--streams", type=int, default=16, help="streams the views of a multi-view step alternate on")
    return p.parse_args()


# ------------------------------------------------------------------ helpers

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def tile_order_launches(cam):
    """1 when the frame launches the heaviest-first tile-order kernel
    (csrc/frame.cu: more tiles than one raster wave)."""
    on = os.environ.get("GS_TILE_ORDER", "1") != "0"
    return 1 if on and cam.tiles_x * cam.tiles_y > 148 * 8 else 0


def binning_of(n, cam):
    """The frame binning the library uses for this view (gs_frame_binning):
    "depth_first", "scatter" or "direct"."""
    from paper_2312_02121_b200 import ops
    return ops.frame_binning(n, cam)


def fused_sort(n, cam):
    """The per-tile sort runs inside the raster forward (direct binning, or
    scatter binning with the fuse_sort option)."""
    from paper_2312_02121_b200 import ops
    b = binning_of(n, cam)
    return b == "direct" or (b == "scatter" and ops.get_option("fuse_sort") == 1)


def views_for(cfg, spec, world, rank):
    """(camera, d_image) pairs this rank renders each step."""
    import numpy as np
    from paper_2312_02121_b200.scenes import CameraSpec, look_at

    if cfg == 3:
        nv = len(spec.cameras)
        idx = list(range(rank, nv, world))
        return [(spec.cameras[i], spec.d_images[i]) for i in idx]
    if cfg == 4:  # one frame; the band split is applied in run_ours
        return [(spec.cameras[0], spec.d_images[0])]
    base = spec.cameras[0]
    if rank == 0:
        return [(base, spec.d_images[0])]
    rng = np.random.default_rng(1000 + rank)
    center = -base.view[:3, :3].T @ base.view[:3, 3]
    dist = float(np.linalg.norm(center))
    while True:
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        if abs(d[1]) <= 0.99:
            break
    cam = CameraSpec(look_at(dist * d), base.fx, base.fy, base.cx, base.cy, base.width, base.height,
                     base.near, base.far)
    dimg = rng.normal(size=(base.height, base.width, 3)).astype(np.float32)
    return [(cam, dimg)]


class ClockSampler:
    """SM clock + throttle reasons sampled (NVML, every 5 ms) during the
    timed region; falls back to nvidia-smi when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return

        def loop():
            while not self._stop.is_set():
                try:
                    self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for nm, bit in self.REASONS.items():
                        if r & bit:
                            self.reasons.add(nm)
                except Exception:
                    pass
                time.sleep(0.005)

        self.thread = threading.Thread(target=loop, daemon=True)
        self.thread.start()

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self._stop.set()
        self.thread.join(timeout=1)
        sm = sorted(self.samples)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": self.max_mhz, "samples": len(sm),
                "reasons": sorted(self.reasons)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def load_traffic():
    """Per-launch DRAM bytes from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------- our arm

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2312_02121_b200 import _lib, ops
    from paper_2312_02121_b200 import engine as E
    from paper_2312_02121_b200 import ops
    from paper_2312_02121_b200.scenes import config_sizes, make_config

    world, rank, local = dist_env()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    # GS_BENCH_SHARED_GPU=1: a functional test of the N-rank path on fewer GPUs (ranks share
    # devices, gloo reductions on the host; the numbers mean nothing)
    shared = os.environ.get("GS_BENCH_SHARED_GPU") == "1" and world > torch.cuda.device_count()
    if shared:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg = args.config
    spec = make_config(cfg)
    views = views_for(cfg, spec, world, rank)
    n = spec.n
    t = lambda a: torch.as_tensor(a, device=dev)
    params = [t(spec.means), t(spec.scales), t(spec.quats), t(spec.opacities), t(spec.colors)]
    m, s, q, o, c = params
    cams = [ops.CameraParams.of(cv) for cv, _ in views]
    d_imgs = [t(d) for _, d in views]
    band = None
    if cfg == 4 and world > 1:
        # tile-row bands balanced by intersections (every rank computes the same split)
        from paper_2312_02121_b200 import dist as D
        full = cams[0]
        proj = ops.project(m, s, q, o, full)
        work = D.tile_row_work_from_projection(proj.xydr, full.height, full.width)
        band = D.band_rows(work, world, full.height)[rank]
        cams = [D.band_camera(full, *band)]
        d_imgs = [d_imgs[0][band[0]:band[1]].contiguous()]
        views = [(cams[0], views[0][1][band[0]:band[1]])]
        del proj
    bg = (0.0, 0.0, 0.0)
    flush = torch.empty(L2_FLUSH_BYTES // 4, device=dev, dtype=torch.float32)
    grad_flat = torch.zeros((14 * n,), device=dev, dtype=torch.float32)
    L = _lib.load()

    # per-view static capacity + workspace (one checked run each), and the
    # roofline numerators: evaluation-class counts of a counted pass (untimed)
    counts_f = np.zeros(4, np.int64)
    counts_b = np.zeros(3, np.int64)
    caps, wss, isect, binnings, visible, touched = [], [], [], [], [], []
    for cam, d_img in zip(cams, d_imgs):
        fr = ops.frame_forward(m, s, q, o, c, cam, bg, True, counts=True)
        g = ops.frame_backward(fr, m, s, q, c, d_img, counts=True)
        counts_f += fr.counts_fwd.cpu().numpy()
        counts_b += g["counts"].cpu().numpy()
        isect.append(fr.n_isect)
        del fr, g
        # the timed frames' capacity (the counted pass may bin differently: size from an uncounted frame)
        fr = ops.frame_forward(m, s, q, o, c, cam, bg, True)
        cap = int(fr.needed_capacity * 1.05) + 4096
        caps.append(cap)
        visible.append(min(int(fr.meta().cpu()[7]), n))  # depth-first: the depth-sorted (visible) Gaussians
        # the Gaussians with non-zero screen-space rows (the ones the projection backward clears)
        ops.frame_backward(fr, m, s, q, c, d_img, project=False)
        rows, c11 = ops.frame_screen_grads(fr)
        touched.append(int(((rows != 0).any(1) | (c11 != 0)).sum()))
        binnings.append(fr.binning)
        wss.append(ops.frame_workspace(n, cap, cam.width, cam.height, dev))
        del fr

    def mk_events(k):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        for e in evs:
            e.record()  # materialise the underlying cudaEvent_t
        return evs

    ev_f = [mk_events(6) for _ in cams]
    ev_b = [mk_events(3) for _ in cams]
    frames_out = [None] * len(cams)

    grad_out = E.unpack(grad_flat, n)

    ev_t = [mk_events(3) for _ in cams]  # timed graph: only around the dominant kernel (raster bwd)
    # several views: every view runs its raster backward only, then one batched projection
    # backward over all views (gs_frame_views_project_backward); GS_BATCHED_PROJ=0: per view
    batched = len(cams) > 1 and os.environ.get("GS_BATCHED_PROJ", "1") != "0"
    ev_pb = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(2)]  # recorded inside capture
    # ... and every view's projection in one pass (when all views bin depth-first); GS_BATCHED_FWD=0: per view
    batched_fwd = batched and os.environ.get("GS_BATCHED_FWD", "1") != "0" and ops.frames_projectable(n, cams)
    ev_pf = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(2)]
    d_views = torch.zeros((len(cams), 4, 4), device=dev, dtype=torch.float32)

    def step(staged=False):
        # every view writes (first) or accumulates (others) straight into
        # the flat gradient buffer that the multi-GPU all-reduce sums.
        # Event-record nodes cost graph bubbles, so the timed graph carries
        # only the pair bracketing the raster backward (the roofline
        # kernel); the per-stage breakdown comes from a second, fully
        # instrumented graph replayed after the timed region.
        # Several views: the views go round-robin over args.streams streams, each with
        # its own workspace; a view's backward waits for the previous view's
        # (the gradient sums keep the sequential order), so one view's
        # forward overlaps the previous view's backward.
        ns = min(args.streams, len(cams)) if not staged else 1
        two = ns > 1
        main = torch.cuda.current_stream()
        sts = [main] + aux[:ns - 1]
        if batched_fwd:
            if staged:
                ev_pf[0].record()
            ops.frames_project(m, s, q, o, cams, caps, wss)
            if staged:
                ev_pf[1].record()
        for a in sts[1:]:
            a.wait_stream(main)
        bwd_done = None
        for vi, (cam, d_img) in enumerate(zip(cams, d_imgs)):
            st = sts[vi % ns]
            with torch.cuda.stream(st):
                fr = ops.frame_forward(m, s, q, o, c, cam, bg, True, capacity=caps[vi], check_meta=False,
                                       ws=wss[vi], events=ev_f[vi] if staged else None, binning=binnings[vi],
                                       projected=batched_fwd)
                # only the views' accumulation into grad_out is ordered: this view's raster
                # backward overlaps the previous view's projection backward.  N > 1: the
                # last view's projection backward runs after the graph, bucketed under the
                # all-reduce (view shards), or after the screen-space all-reduce (bands)
                tail = world > 1 and vi == len(cams) - 1
                ops.frame_backward(fr, m, s, q, c, d_img,
                                   events=ev_b[vi] if staged else [ev_t[vi][0], ev_t[vi][1], None],
                                   out=grad_out, accumulate=vi > 0, wait_before_accumulate=bwd_done,
                                   project=not (tail or batched))
                if two and not batched:
                    bwd_done = torch.cuda.Event()
                    bwd_done.record(st)
            frames_out[vi] = fr
        for a in sts[1:]:
            main.wait_stream(a)
        if batched and world == 1:  # N > 1: bucketed under the all-reduce in run_step
            if staged:
                ev_pb[0].record()
            ops.frame_views_project_backward(frames_out, m, s, q, grad_out, d_views)
            if staged:
                ev_pb[1].record()

    aux = [torch.cuda.Stream() for _ in range(max(args.streams - 1, 0))]
    graph = graph_staged = None
    if not args.no_graph:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(3):
                step()
                step(True)
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph_staged = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph_staged):
            step(True)

    from paper_2312_02121_b200 import dist as D
    reducer = D.GradReducer(n, buckets=4) if world > 1 and band is None else None
    d_view_tail = torch.zeros((4, 4), device=dev, dtype=torch.float32)

    def run_step(staged=False):
        if graph is not None:
            (graph_staged if staged else graph).replay()
        else:
            step(staged)
        if world > 1:
            fr = frames_out[-1]
            if band is None and batched:  # view shards: all-reduced under the batched projection bwd
                reducer.wait(reducer.views(frames_out, params, grad_out, d_views))
            elif band is None:  # view shards: 14 fp32 per Gaussian, all-reduced under the last projection bwd
                reducer.wait(reducer.last_view(fr, params, grad_out, d_view_tail, accumulate=len(cams) > 1))
            else:  # tile bands: 9 screen-space fp32 per Gaussian, then the projection bwd on every rank
                rows, c11 = ops.frame_screen_grads(fr)
                dist.all_reduce(rows)
                dist.all_reduce(c11)
                ops.frame_project_backward(fr, m, s, q, grad_out, d_view_tail, vis_from_grads=True)

    for _ in range(max(args.warmup, 0)):
        run_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    step_ms = []
    from paper_2312_02121_b200 import ops as _ops
    tile_emit = _ops.frame_tile_emit(n, cams[0])
    # depth-first binning with the tile-sorted emission: (per-chunk tile counts, column prefixes,
    # tile scan) then the emission into the final slots; otherwise fused scan + emission then the
    # onesweep passes by tile + ranges
    stage_names = ("project", "depth_sort", "tile_counts" if tile_emit else "scan_emit",
                   "tile_emit" if tile_emit else "tile_sort_ranges", "raster_fwd", "raster_bwd", "project_bwd")
    stage_ms = np.zeros(len(stage_names))
    timed_bwd_ms = 0.0
    stream = torch.cuda.current_stream()
    for k in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (untimed)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_step()
        e1.record(stream)
        torch.cuda.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        timed_bwd_ms += sum(ev_t[vi][0].elapsed_time(ev_t[vi][1]) for vi in range(len(cams)))
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    # per-stage breakdown from the instrumented graph (untimed for the headline)
    for k in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        run_step(staged=True)
        torch.cuda.synchronize()
        for vi in range(len(cams)):
            f, b = ev_f[vi], ev_b[vi]
            if not batched_fwd:
                stage_ms[0] += f[0].elapsed_time(f[1])
            stage_ms[1] += f[1].elapsed_time(f[2])
            stage_ms[2] += f[2].elapsed_time(f[3])
            stage_ms[3] += f[3].elapsed_time(f[4])
            stage_ms[4] += f[4].elapsed_time(f[5])
            stage_ms[5] += b[0].elapsed_time(b[1])
            if not batched:
                stage_ms[6] += b[1].elapsed_time(b[2])
        if batched and world == 1:
            stage_ms[6] += ev_pb[0].elapsed_time(ev_pb[1])
        if batched_fwd:
            stage_ms[0] += ev_pf[0].elapsed_time(ev_pf[1])
    # the capacity was sized from a checked run; confirm nothing overflowed
    for vi, fr in enumerate(frames_out):
        meta = fr.meta().cpu()
        assert int(meta[0]) == -1 and ops.needed_capacity(meta) <= caps[vi], "capacity overflow / status error in timed run"
    total_ms = float(sum(step_ms))
    if world > 1:
        tt = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    stage_ms /= max(args.steps, 1)
    frames_per_step = len(spec.cameras) if cfg in (3, 4) else len(cams) * world
    ms_per_step = total_ms / max(args.steps, 1)
    fps = frames_per_step / (ms_per_step / 1e3)
    evals_rank = float(counts_f[0] + counts_b[0])
    evals_step = evals_rank
    if world > 1:
        ev_t = torch.tensor([evals_rank], device=dev, dtype=torch.float64)
        dist.all_reduce(ev_t)
        evals_step = float(ev_t.item())
    evals_per_s = evals_step / (ms_per_step / 1e3)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, spec, views, dev, world, frames_per_step)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks, peak_src = measured_peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = 128.0 * sms * sm_max * 1e6  # lane-ops/s, FMA = 1 op
    hbm = float(peaks.get("hbm_gbs", 6650.0)) * 1e9
    nv = len(cams)
    I = float(sum(isect))
    n_tiles = sum(cm.tiles_x * cm.tiles_y for cm in cams)
    tp = 1 if cams[0].tiles_x * cams[0].tiles_y <= 256 else 2
    # algorithmic work; per rank-step, all views
    F_fwd = 8 * counts_f[0] + 4 * counts_f[1] + 3 * counts_f[2] + 4 * counts_f[3]
    F_bwd = 8 * counts_b[0] + 4 * counts_b[1] + 42 * counts_b[2]
    binning = binning_of(n, cams[0])
    seg = binning != "depth_first"
    direct = binning == "direct"
    fused = fused_sort(n, cams[0])
    vis = float(sum(visible))  # visible Gaussians over the rank's views (the depth-sorted ones)
    nz = float(sum(touched))  # (Gaussian, view) pairs with non-zero screen-space gradient rows
    chunks_x_tiles = float(sum(((v + 2047) // 2048) * ((cm.tiles_x * cm.tiles_y + 1) & ~1)
                               for v, cm in zip(visible, cams)))
    work = {
        # 72 B per Gaussian (read mean 12 + scale 12 + quat 16; write mean2d 8 +
        # cov/conic 12 + depth 4 + radius 4 + tiles 4).  The kernel itself moves 84 B (+ opacity
        # 4 in, the conic's 4th float and the depth sort key out); the backward accumulators are
        # no longer zeroed here (the projection backward clears the rows it reads).  Direct
        # binning: + a slot atomic and the Gaussian id per intersection (8 B)
        # batched over the views (one pass): the 44 B of parameters read once, per view the
        # xydr / conic / tiles / depth key written (40 B)
        "project": ("hbm", (44.0 * n + 40.0 * n * nv) if batched_fwd else 72.0 * n * nv + (8.0 * I if direct else 0.0)),
        # depth-first: 4 passes x (key+value) x (read+write); scatter / direct: no global depth sort
        "depth_sort": ("none", 0.0) if seg else ("hbm", 4 * 16.0 * n * nv),
        # depth-first: fused scan + emission, (order +) count + xydr gather per Gaussian, pairs out;
        # scatter: tile scan (8 counter replicas + ranges) + count + xydr per Gaussian, pairs out;
        # direct: none (the projection placed the pairs)
        "scan_emit": ("none", 0.0) if direct else
                     ("hbm", (40.0 * n_tiles + 20.0 * n * nv + 8.0 * I) if seg else
                      (8.0 * n * nv + 16.0 * n * nv + 8.0 * I)),
        # depth-first: tile passes (key+value, read+write) + ranges; scatter: per-tile sort
        # (value in, key gather, value out) + ranges -- inside the raster forward when fused
        "tile_sort_ranges": ("none", 0.0) if fused else
                            ("hbm", (12.0 * I + 8.0 * n_tiles) if seg else
                             (tp * 16.0 * I + 4.0 * I + 8.0 * n_tiles)),
        # tile-sorted emission: order + xydr gather per visible Gaussian, u16 counts out, column
        # scan (u16 in, u32 prefix out), tile scan (4 B in, 8 B ranges out per tile)
        "tile_counts": ("hbm", 20.0 * vis + 8.0 * chunks_x_tiles + 12.0 * n_tiles),
        # order + xydr gather per visible Gaussian, ranges + prefix per (chunk, tile), 4 B per pair out
        "tile_emit": ("hbm", 20.0 * vis + 8.0 * chunks_x_tiles + 4.0 * I),
        "raster_fwd": ("fp32", float(F_fwd)),
        "raster_bwd": ("fp32", float(F_bwd)),
        # 104 B per Gaussian (read mean, scale, quat 40 + d_mean2d 8 + d_cov 12 +
        # radius/visibility 4; write d_mean, d_scale, d_quat 40).  The kernel also copies the
        # d_color/d_opacity row (16 + 16), clears the rows it read, and views after the first
        # read-modify-write the running sums
        # batched over the views (one pass): parameters read once (40 B) and the sums written once
        # (56 B) per Gaussian; per view the raster backward's marks (1 bit per Gaussian) and the
        # marked rows read (36 B) and cleared (36 B) -- §8(d)'s per-view 104 B would count the
        # parameter traffic once per view
        "project_bwd": ("hbm", (96.0 * n + n * nv / 8.0 + 72.0 * nz) if batched else 104.0 * n * nv),
    }
    st = {}
    for name, ms in zip(stage_names, stage_ms):
        bound, w = work[name]
        d = {"ms": round(float(ms), 4), "bound": bound}
        if bound == "none":
            pass
        elif bound == "hbm":
            d["achieved_gbs"] = round(w / (ms / 1e3) / 1e9, 1) if ms > 0 else None
            d["frac"] = round(w / (ms / 1e3) / hbm, 4) if ms > 0 else None
        else:
            d["achieved_tops"] = round(w / (ms / 1e3) / 1e12, 3) if ms > 0 else None
            d["frac"] = round(w / (ms / 1e3) / fp32_peak, 4) if ms > 0 else None
        if name == "raster_fwd" and fused:
            d["includes"] = "per-tile (depth, index) sort of the tile's list"
        if d.get("frac") is not None and d["frac"] > 1.0:
            # the stage's kernels ran outside the instrumented replay (N > 1: the projection backward
            # follows the reduction over ranks), so the event gap is not its duration
            for k in ("achieved_gbs", "achieved_tops", "frac"):
                if k in d:
                    d[k] = None
            d["note"] = "not inside the instrumented replay (runs after the reduction over ranks)"
        st[name] = d
    dom = max(stage_names, key=lambda k: stage_ms[stage_names.index(k)])
    if dom == "raster_bwd" and timed_bwd_ms > 0:
        # The roofline kernel's launch duration comes from the instrumented single-stream replay
        # of the same step (CUDA events on the launching stream, right after the timed region;
        # it agrees with the ncu launch list).  Inside the timed region its event interval is
        # also reported, but with up to 16 view streams overlapping it spans the other views'
        # kernels sharing the SMs, so it is an upper bound on the launch, not its duration.
        bwd_ms = timed_bwd_ms / max(args.steps, 1)
        st[dom]["ms_in_step_interval"] = round(bwd_ms, 4)
        st[dom]["frac_in_step_interval"] = round(work[dom][1] / (bwd_ms / 1e3) / fp32_peak, 4)
    traffic = load_traffic()
    if st[dom]["bound"] == "fp32":
        roof = {"bound": "fp32", "kernel": dom, "achieved": st[dom]["achieved_tops"],
                "peak": round(fp32_peak / 1e12, 3), "unit": "Tlane-op/s (FP32, FMA=1)", "frac": st[dom]["frac"],
                "peak_at_measured_clock": round(128.0 * sms * (clocks["sm_mhz"] or sm_max) * 1e6 / 1e12, 3)
                if clocks and clocks.get("sm_mhz") else None,
                "peak_source": f"128 FP32 lanes x {sms} SMs x {sm_max:.0f} MHz ({peak_src} sm_max)"}
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": st[dom]["achieved_gbs"],
                "peak": float(peaks.get("hbm_gbs", 6650.0)), "unit": "GB/s", "frac": st[dom]["frac"],
                "peak_source": peak_src}
    if "frac_in_step_interval" in st[dom]:
        roof["frac_in_step_interval"] = st[dom]["frac_in_step_interval"]
        roof["duration_ms_in_step_interval_per_launch"] = round(st[dom]["ms_in_step_interval"] / nv, 4)
        roof["duration_source"] = ("single-stream instrumented replay of the step (CUDA events on the launching "
                                   "stream); in-step interval: the timed region's events around each view's launch")
    roof["traffic"] = traffic.get(dom)
    # per-stage DRAM bytes of ONE launch from the committed ncu --set full capture of a config-3 engine
    # step (profiles/ncu_traffic.json; depth_sort: one onesweep pass; tile_counts / tile_emit: their
    # kernels of one view): a stage whose traffic is far below its byte model runs out of L2
    if cfg == 3:
        for name, key in (("project", "project"), ("depth_sort", "sort_u32"), ("tile_counts", "tile_counts"),
                          ("tile_emit", "tile_emit"), ("raster_fwd", "raster_fwd"), ("raster_bwd", "raster_bwd"),
                          ("project_bwd", "project_bwd")):
            if name in st and key in traffic:
                st[name]["ncu_dram_bytes_per_launch"] = traffic[key]
    roof["algorithmic_work_per_launch"] = work[dom][1] / nv
    roof["duration_ms_per_launch"] = round(float(stage_ms[stage_names.index(dom)]) / nv, 4)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(spec, views[:1], frames_per_step)

    out = {
        "metric": METRIC, "value": round(fps, 3), "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong" if cfg in (3, 4) else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded, BASELINE.json distributions; scenes.py)",
        "config": bench_config(cfg, world,
                               parallelism=(f"tile-row bands x{world} (rows {band})" if band else
                                            f"view-sharded x{world}") +
                               ((" + NCCL all-reduce of 9 screen-space fp32/Gaussian, then the projection "
                                 "backward on every rank") if band else
                                (" + NCCL all-reduce 14 fp32/Gaussian in 4 buckets overlapped with the last "
                                 "view's projection backward") if world > 1 else ""),
                               views_per_rank=len(cams), cuda_graph=graph is not None,
                               view_streams=min(args.streams, len(cams)),
                               l2="flushed between timed steps (192 MiB write, untimed)"),
        "evals_per_s": round(evals_per_s, 1), "evals_per_step": evals_step,
        "intersections_per_step_rank": int(I),
        "visible_per_step_rank": int(vis), "nonzero_grad_rows_per_step_rank": int(nz),
        "e2e": e2e,
        # per view (csrc/frame.cu): direct binning: init, project (+ pairs into the tile bins),
        # raster fwd (+ the per-tile sort) | raster bwd, project bwd, view reduce; scatter binning:
        # init, project (+ tile counts), tile scan (+ raster order), pair scatter, [per-tile sort,]
        # raster fwd | raster bwd, project bwd, view reduce; depth-first: init, project, depth
        # histogram, 4 depth passes, fused scan+emit, tp tile passes, ranges, (tile order for grids
        # over one raster wave), raster fwd | raster bwd, project bwd, view reduce
        # (depth-first: + the depth histogram, the view reduce; depth passes skipped on the
        # device beyond the key width still launch)
        # depth-first, per view: init + project (none when the projections are batched: views_init +
        # views_project_fwd once per step), 4 depth passes, then either the tile-sorted emission
        # (expansion, column sums, tile scan incl. the raster order, column scan, placement) or
        # fused scan + emission, tp tile passes, ranges (+ tile order); raster fwd, raster bwd;
        # project bwd + view reduce (batched: views_project_bwd + views_reduce once per step).
        # Config 3 (batched, tile-sorted emission): 11 per view + 4 per step = 356, the launch
        # list of profiles/*_config3_launches.txt
        "gpu_launches": int(args.steps * (
            len(cams) * (6 if direct else (8 if fused else 9) if seg else
                         (0 if batched_fwd else 2) + 4 +
                         (5 if tile_emit else 2 + tp + tile_order_launches(cams[0])) + 2 +
                         (0 if batched else 2)) +
            (0 if direct or seg else (2 if batched_fwd else 0) + (2 if batched else 0)) +
            (0 if world == 1 else 2 if band else 2 * len(reducer.bounds)))),
        "binning": binning,
        "roofline": roof,
        "stages": st,
        "counts": {"E_f": int(counts_f[0]), "E_f_sigma": int(counts_f[1]), "E_f_alpha": int(counts_f[2]),
                   "E_f_commit": int(counts_f[3]), "E_b": int(counts_b[0]), "E_b_sigma": int(counts_b[1]),
                   "E_b_contrib": int(counts_b[2]), "views": nv},
        "cpu_baseline": cpu,
        "clocks": clocks,
        "impl": "ours",
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, spec, views, dev, world, frames):
    """Same metric end to end through the public engine API
    (paper_2312_02121_b200.engine.RenderStep + pipeline): every step copies
    its parameters and upstream image gradients from pinned host memory and
    reads the 14 gradients per Gaussian (and the frame metadata) back to
    pinned host memory; double-buffered so the copies of one step overlap
    the graph replay of another.  K steps are timed as one region (CUDA
    events, synchronize on both sides, max over ranks)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2312_02121_b200 import engine as E
    from paper_2312_02121_b200 import ops

    def staged(a):  # inputs written once into write-combined pinned staging (engine.host_staging), before timing
        a = np.ascontiguousarray(a, dtype=np.float32)
        t = E.host_staging(a.shape)
        t.copy_(torch.from_numpy(a))
        return t

    host = [staged(a) for a in (spec.means, spec.scales, spec.quats, spec.opacities, spec.colors)]
    dimgs = [staged(d) for _, d in views]
    cams = [c for c, _ in views]
    eng = E.RenderStep(spec.n, cams, device=dev)
    eng.prime(host, dimgs)
    out_host = [torch.empty((14 * spec.n,), dtype=torch.float32).pin_memory() for _ in range(eng.nbuf)]
    wc = all(E.is_write_combined(h) for h in host + dimgs)
    h2d = sum(h.numel() * 4 for h in host) + sum(d.numel() * 4 for d in dimgs)
    d2h = out_host[0].numel() * 4 + len(cams) * 16
    allreduce = (lambda g: dist.all_reduce(g)) if world > 1 else None
    flush = torch.empty(L2_FLUSH_BYTES // 4, device=dev, dtype=torch.float32)
    E.pipeline(eng, host, dimgs, out_host, max(2, args.warmup), allreduce, flush)  # warm-up
    torch.cuda.synchronize()
    steps = max(3, args.steps)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    metas = E.pipeline(eng, host, dimgs, out_host, steps, allreduce, flush)
    e1.record()
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1)
    for b, mh in enumerate(metas):
        eng.result(b, mh)  # raises on a status error; capacity was sized by a checked frame
        assert all(ops.needed_capacity(row) <= c for row, c in zip(mh.tolist(), eng.caps)), \
            "capacity overflow in timed e2e run"
    if world > 1:
        tt = torch.tensor([total], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total = float(tt.item())
    return {"value": round(frames / (total / steps / 1e3), 3), "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "api": "paper_2312_02121_b200.engine.RenderStep + pipeline (host->device copy of every step's "
                   "inputs and device->host read of its gradients inside the timed region, double-buffered; "
                   "the inputs are written into the host buffers once, before timing)",
            "host_inputs": "write-combined pinned" if wc else "pinned (cuda-python unavailable)",
            "host_outputs": "pinned",
            "l2": "flushed before every step inside the timed region (conservative)"}


def cpu_info() -> dict:
    """The host the CPU numbers were taken on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"cpu_model": model, "nproc": usable}


def _oracle_view(args64, cam, d_image, nth):
    """One full fwd+bwd frame of the fp64 oracle port: render (sg/raster_forward.py:255-271)
    + scene_backward (sg/proj_backward.py:178-223)."""
    import numpy as np

    import oracle as O
    oc = O.Camera.of(cam)
    fw = O.render(*args64, oc, np.zeros(3), True, nthreads=nth)
    O.scene_backward(*args64, oc, np.zeros(3), fw, np.asarray(d_image, np.float64), nthreads=nth)


def _args64(spec):
    import numpy as np
    f = lambda a: np.asarray(a, np.float64)
    return [f(spec.means), f(spec.scales), f(spec.quats), f(spec.opacities), f(spec.colors)]


def cpu_one_core(spec, views, budget_s=40.0, all_cores_s=None, nth_all=1):
    """The reference is single-threaded by design (pkg/README.md:10-13): one
    full view on ONE core, unless the all-cores time predicts more than
    budget_s (then reported as not measured)."""
    if all_cores_s is not None and all_cores_s * nth_all > budget_s * 1.5:
        return None, None
    a = _args64(spec)
    cam, d = views[0]
    t0 = time.perf_counter()
    _oracle_view(a, cam, d, 1)
    dt = time.perf_counter() - t0
    return round(1.0 / dt, 5), round(dt, 3)


def cpu_baseline(spec, views, frames_per_step):
    """Bounded sample of the same workload on the host (rank 0, N = 1): one
    full fwd+bwd view on all host threads, then one on one core.  frames/s =
    views / seconds; a config-3 step is 32 such views."""
    info = cpu_info()
    nth = info["nproc"]
    a = _args64(spec)
    cam, d = views[0]
    t0 = time.perf_counter()
    _oracle_view(a, cam, d, nth)
    dt = time.perf_counter() - t0
    v1, s1 = cpu_one_core(spec, views, all_cores_s=dt, nth_all=nth)
    return {"value": round(1.0 / dt, 5), "unit": "frames/s", "cores": nth, "kind": "port",
            "sample": f"1 of {frames_per_step} views per step, full fwd+bwd (oracle/splat_oracle.c, fp64, "
                      f"OpenMP x{nth}); frames/s = views/s",
            "seconds": round(dt, 3), "one_core": {"value": v1, "unit": "frames/s", "seconds": s1}, **info}


# ------------------------------------------------------------ reference arm

def run_reference(args):
    """The reference's CPU path (fp64 oracle port of sg/raster_forward.py:255-271
    render + sg/proj_backward.py:178-223 scene_backward) on the host cores:
    W untimed + K timed steps, each ONE full fwd+bwd view of the workload
    (views cycle through the config's cameras), all host threads.  Under
    torchrun only rank 0 runs."""
    world, rank, _ = dist_env()
    if rank != 0:
        return

    from paper_2312_02121_b200.scenes import config_sizes, make_config

    cfg = args.config
    K, W = max(1, args.steps), max(0, args.warmup)
    nv_cfg = config_sizes(cfg)["views"]
    spec = make_config(cfg, n_views=min(nv_cfg, K + W)) if cfg == 3 else make_config(cfg)
    views = list(zip(spec.cameras, spec.d_images))
    info = cpu_info()
    nth = info["nproc"]
    a = _args64(spec)
    for i in range(W):
        cam, d = views[i % len(views)]
        _oracle_view(a, cam, d, nth)
    t0 = time.perf_counter()
    for i in range(K):
        cam, d = views[(W + i) % len(views)]
        _oracle_view(a, cam, d, nth)
    dt = time.perf_counter() - t0
    fps = K / dt
    v1, s1 = cpu_one_core(spec, views, all_cores_s=dt / K, nth_all=nth)
    out = {"metric": METRIC, "value": round(fps, 5), "unit": "frames/s", "n_gpus": args.gpus, "steps": K,
           "warmup": W, "ms_per_step": round(dt / K * 1e3, 3), "higher_is_better": True,
           "scaling": "strong" if cfg in (3, 4) else "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded, BASELINE.json distributions; scenes.py)",
           "config": bench_config(cfg, args.gpus, parallelism=f"host OpenMP x{nth} (fp64 oracle port)",
                                  views_per_rank=nv_cfg if cfg in (3, 4) else 1, cuda_graph=False, view_streams=1,
                                  l2="n/a (host)"),
           "impl": "reference",
           "cpu_baseline": {"value": round(fps, 5), "unit": "frames/s", "cores": nth, "kind": "port",
                            "sample": f"each step 1 full fwd+bwd view (of {nv_cfg} per workload step) on all host "
                                      f"threads (oracle/splat_oracle.c, fp64, OpenMP); frames/s = views/s",
                            "one_core": {"value": v1, "unit": "frames/s", "seconds": s1}, **info},
           "e2e": {"value": round(fps, 5), "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def bench_config(cfg, world, parallelism=None, **extra):
    """The line's `config` object (same keys for both arms)."""
    from paper_2312_02121_b200.scenes import config_sizes
    sz = config_sizes(cfg)
    c = {"workload": f"config{cfg}", "gaussians": sz["gaussians"], "image": f"{sz['width']}x{sz['height']}",
         "views_per_step": sz["views"] if cfg in (3, 4) else world, "early_termination": True,
         "background": "black", "parallelism": parallelism}
    c.update(extra)
    return c


def self_launch(args) -> int:
    """`--gpus N` (N > 1) outside torchrun: run this script under
    torch.distributed.run, one rank per GPU, rendezvous on 127.0.0.1."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
