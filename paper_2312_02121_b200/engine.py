"""Repeated forward+backward renders through captured CUDA graphs.

The per-call API (ops.rasterize, api.render/scene_backward) pays Python,
allocation and a host sync for the intersection count on every frame.  A
training or serving loop renders the same view sizes over and over; for it,
``RenderStep`` captures the whole sync-free frame (gs_frame_forward +
gs_frame_backward for every view, gradients summed over views) once per
buffer set and replays it:

  * static device buffers for the parameters, the upstream image gradients
    and the 14 gradients per Gaussian, one flat buffer of contiguous blocks
    d_mean (n,3) | d_scale (n,3) | d_quat (n,4) | d_rgbo (n,4) (colour 3,
    opacity 1) -- the SceneGradients fields, sg/proj_backward.py:25-50 --
    that gs_frame_backward writes (first view) or accumulates into (the
    others) directly;
  * two buffer sets, so the host<->device copies of one step overlap the
    replay of the other (``pipeline``);
  * the per-view intersection capacity comes from one checked frame; every
    replay's status word and intersection count travel back with the
    gradients and ``result()`` raises (status) or re-runs the step with a
    larger capacity (overflow) exactly like the per-call path.
"""

from __future__ import annotations

import os

import torch

from . import _lib, ops


_WC_PTRS: set = set()


def host_staging(shape, dtype=torch.float32) -> torch.Tensor:
    """A CPU tensor in pinned, write-combined host memory
    (cudaHostAllocWriteCombined) for inputs the host writes and the GPU
    copies in every step: the DMA engine reads it without snooping the CPU
    caches (on one box of the pool pinned host->device copies ran at 14 GB/s
    from ordinary pinned memory and 55 GB/s from write-combined memory,
    tools/pcie_bw.py).  The host must not READ it (uncached).  Falls back to
    ordinary pinned memory when cuda-python is unavailable;
    ``is_write_combined(t)`` tells which kind a tensor got.

    The allocation is owned by the buffer object torch.frombuffer keeps alive
    for the storage's lifetime, so it is freed when the last tensor sharing
    the storage dies (not when this wrapper does)."""
    import ctypes
    numel = 1
    for d in shape:
        numel *= int(d)
    if numel == 0:
        return torch.empty(tuple(shape), dtype=dtype).pin_memory()
    nbytes = numel * torch.empty((), dtype=dtype).element_size()
    try:
        try:
            from cuda.bindings import runtime as cr
        except ImportError:
            from cuda import cudart as cr
        err, ptr = cr.cudaHostAlloc(nbytes, cr.cudaHostAllocWriteCombined)
        if int(err) != 0:
            raise RuntimeError(f"cudaHostAlloc: {err}")
    except Exception:  # noqa: BLE001 -- no cuda-python: ordinary pinned memory
        return torch.empty(tuple(shape), dtype=dtype).pin_memory()
    ptr = int(ptr)

    class _WCBuffer(ctypes.c_uint8 * nbytes):
        """Owns the cudaHostAlloc block; freed when the storage releases it."""

        def __del__(self, _free=cr.cudaFreeHost, _ptr=ptr, _reg=_WC_PTRS):
            _reg.discard(_ptr)
            _free(_ptr)

    raw = _WCBuffer.from_address(ptr)
    t = torch.frombuffer(raw, dtype=dtype, count=numel).view(tuple(shape))
    _WC_PTRS.add(ptr)
    return t


def is_write_combined(t: torch.Tensor) -> bool:
    """True when ``t`` lives in a host_staging write-combined block."""
    return t.untyped_storage().data_ptr() in _WC_PTRS


def unpack(flat: torch.Tensor, n: int) -> dict:
    """Views of a flat (14 n) gradient buffer: d_mean (n,3), d_scale (n,3),
    d_quat (n,4), d_rgbo (n,4), d_color (n,3), d_opacity (n)."""
    d_mean = flat[0:3 * n].view(n, 3)
    d_scale = flat[3 * n:6 * n].view(n, 3)
    d_quat = flat[6 * n:10 * n].view(n, 4)
    d_rgbo = flat[10 * n:14 * n].view(n, 4)
    return dict(d_mean=d_mean, d_scale=d_scale, d_quat=d_quat, d_rgbo=d_rgbo, d_color=d_rgbo[:, :3],
                d_opacity=d_rgbo[:, 3])


class RenderStep:
    def __init__(self, n: int, cams, background=(0.0, 0.0, 0.0), early_termination=True, device=None,
                 headroom: float = 1.05, buffers: int = 2, view_streams: int = 16, reducer=None,
                 batched_projection: bool = True):
        """reducer: a dist.GradReducer -- the step's gradients are summed over
        the ranks of its process group, the all-reduce overlapped with the
        (last view's, or the batched) projection backward (view-sharded data
        parallelism).  batched_projection: with several views, every view
        runs its raster backward only and one gs_frame_views_project_backward
        pass does all views' projection backward (parameters read once, sums
        written once) instead of one read-modify-write pass per view."""
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.reducer = reducer
        self.n = int(n)
        self.cams = [c if isinstance(c, ops.CameraParams) else ops.CameraParams.of(c) for c in cams]
        self.bg = tuple(float(b) for b in background)
        self.et = bool(early_termination)
        self.headroom = headroom
        self.batched = bool(batched_projection) and len(self.cams) > 1
        # batched forward projection too, when every view bins depth-first (large scenes)
        self.batched_fwd = self.batched and ops.frames_projectable(self.n, self.cams)
        self.nbuf = buffers
        z = lambda *shape: torch.zeros(shape, device=self.dev, dtype=torch.float32)
        self.sets = []
        for _ in range(buffers):
            self.sets.append(dict(
                params=[z(n, 3), z(n, 3), z(n, 4), z(n), z(n, 3)],
                d_images=[z(c.height, c.width, 3) for c in self.cams],
                grads=z(14 * n),
                meta=torch.zeros((len(self.cams), 4), device=self.dev, dtype=torch.int64),
                d_view=z(len(self.cams), 4, 4),
                frames=[None] * len(self.cams),
                graph=None))
        self.caps = None
        self.wss = None
        # further view streams (multi-view steps): with the batched projections the views are
        # independent; config 3 measured 2: 1236, 3: 1256, 4: 1274, 6: 1298, 8: 1306, 16: 1313,
        # 32: 1306 frames/s (bench.py --streams); 16 by default
        self.aux = [torch.cuda.Stream(self.dev) for _ in range(max(0, min(view_streams, len(self.cams)) - 1))]

    # -------------------------------------------------------------- set-up
    def _size(self, k: int):
        """One checked frame per view: the static intersection capacities."""
        s = self.sets[k]
        m, sc, q, o, c = s["params"]
        L = _lib.load()
        self.caps, self.wss, self.binnings = [], [], []
        for cam, d in zip(self.cams, s["d_images"]):
            fr = ops.frame_forward(m, sc, q, o, c, cam, self.bg, self.et)
            self.binnings.append(fr.binning)
            cap = int(fr.needed_capacity * self.headroom) + 4096
            self.caps.append(cap)
            self.wss.append(ops.frame_workspace(self.n, cap, cam.width, cam.height, self.dev))

    def _body(self, k: int):
        """All views of one step.  Several views alternate between the view
        streams (each view has its own workspace); a view's projection
        backward -- the read-modify-write accumulation into the step's
        gradients -- waits for the previous view's, so the views are summed
        in order, while forwards and raster backwards of neighbouring views
        overlap.  (Within a view the raster backward's fp32 atomics already
        make the low bits order-dependent.)"""
        s = self.sets[k]
        m, sc, q, o, c = s["params"]
        out = unpack(s["grads"], self.n)
        main = torch.cuda.current_stream(self.dev)
        sts = [main] + self.aux
        if self.batched_fwd:  # every view's projection in one pass over the Gaussians
            ops.frames_project(m, sc, q, o, self.cams, self.caps, self.wss)
        for a in sts[1:]:
            a.wait_stream(main)
        bwd_done = None
        for vi, (cam, d) in enumerate(zip(self.cams, s["d_images"])):
            st = sts[vi % len(sts)]
            with torch.cuda.stream(st):
                fr = ops.frame_forward(m, sc, q, o, c, cam, self.bg, self.et, capacity=self.caps[vi],
                                       check_meta=False, ws=self.wss[vi], binning=self.binnings[vi],
                                       projected=self.batched_fwd)
                last = vi == len(self.cams) - 1
                if self.batched or (last and self.reducer is not None):
                    # the projection backward runs afterwards (batched over the views, and/or
                    # bucketed under the all-reduce in replay())
                    ops.frame_backward(fr, m, sc, q, c, d, project=False)
                else:
                    g = ops.frame_backward(fr, m, sc, q, c, d, out=out, accumulate=vi > 0,
                                           wait_before_accumulate=bwd_done)
                    s["d_view"][vi].copy_(g["d_view"])
                s["meta"][vi].copy_(fr.meta()[:4])
                s["frames"][vi] = fr
                if len(sts) > 1:
                    bwd_done = torch.cuda.Event()
                    bwd_done.record(st)
        for a in sts[1:]:
            main.wait_stream(a)
        if self.batched and self.reducer is None:
            ops.frame_views_project_backward(s["frames"], m, sc, q, out, s["d_view"])

    def _capture(self):
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            for k in range(self.nbuf):
                self._body(k)  # warm-up (allocations) outside capture
        torch.cuda.current_stream(self.dev).wait_stream(side)
        for k in range(self.nbuf):
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                self._body(k)
            self.sets[k]["graph"] = graph

    def prime(self, params, d_images):
        """Load one step's inputs, size the capacities and capture."""
        for k in range(self.nbuf):
            self.load(k, params, d_images)
        self._size(0)
        self._capture()

    # ------------------------------------------------------------- stepping
    def load(self, k: int, params, d_images, stream=None):
        """Copy (non-blocking from pinned host, or device) into buffer set k.
        stream: one stream, or a list of streams the copies are split over
        in chunks (several DMA streams in flight: on some hosts one stream
        gets well under the link's host-to-device bandwidth)."""
        s = self.sets[k]
        streams = stream if isinstance(stream, (list, tuple)) else [stream or torch.cuda.current_stream(self.dev)]
        pairs = [(dst.view(-1), src.reshape(-1)) for dst, src in zip(s["params"], params)]
        pairs += [(dst.view(-1), src.reshape(-1)) for dst, src in zip(s["d_images"], d_images)]
        chunks = []
        for dst, src in pairs:
            parts = max(1, min(len(streams), dst.numel() * 4 // (1 << 20)))  # >= 1 MiB per chunk
            chunks += list(zip(dst.chunk(parts), src.chunk(parts)))
        for i, (dst, src) in enumerate(chunks):
            with torch.cuda.stream(streams[i % len(streams)]):
                dst.copy_(src, non_blocking=True)

    def replay(self, k: int):
        self.sets[k]["graph"].replay()
        if self.reducer is not None:
            # the last view's projection backward in Gaussian buckets, each
            # bucket's all-reduce overlapping the next buckets (dist.py)
            s = self.sets[k]
            nv = len(self.cams)
            if self.batched:
                works = self.reducer.views(s["frames"], s["params"], unpack(s["grads"], self.n), s["d_view"])
            else:
                works = self.reducer.last_view(s["frames"][nv - 1], s["params"], unpack(s["grads"], self.n),
                                               s["d_view"][nv - 1], accumulate=nv > 1)
            self.reducer.wait(works)

    def d_view(self, k: int) -> torch.Tensor:
        """Per-view d_view (views, 4, 4) of buffer set k's last replay (per
        camera: not reduced over ranks)."""
        return self.sets[k]["d_view"]

    def grads(self, k: int) -> torch.Tensor:
        return self.sets[k]["grads"]

    def meta(self, k: int) -> torch.Tensor:
        return self.sets[k]["meta"]

    def result(self, k: int, meta_host=None):
        """Check buffer set k's last replay: raise on a status error; on a
        capacity overflow grow the capacities, re-capture and re-run it.
        Returns the flat device gradient buffer (see unpack)."""
        m = (meta_host if meta_host is not None else self.meta(k).cpu()).tolist()
        for row in m:
            ops.raise_status(int(row[0]))
        if any(ops.needed_capacity(row) > cap for row, cap in zip(m, self.caps)):
            self._size(k)
            self._capture()
            self.replay(k)
            return self.result(k)
        return self.grads(k)

    def step(self, params, d_images) -> torch.Tensor:
        """One synchronous step (load, replay, check); returns gradients."""
        self.load(0, params, d_images)
        self.replay(0)
        return self.result(0)


# host->device copy streams of pipeline.  On a box whose single-stream pinned
# copies ran at 14-16 GB/s (28 GB/s over 8 streams in isolation,
# tools/pcie_bw.py) config 1's e2e rate per process was 1.45-1.96 k frames/s
# with 1 stream, 1.2-2.8 k with 4 and 1.4-2.6 k with 8 (bimodal, no clear
# winner), so the default stays 1.  GS_H2D_STREAMS=k overrides.
H2D_STREAMS = int(os.environ.get("GS_H2D_STREAMS", "1"))


def pipeline(engine: RenderStep, host_params, host_d_images, out_host, steps: int, allreduce=None, flush=None):
    """`steps` end-to-end steps with double buffering: the H2D copies of step
    k+1 and the D2H read of step k-1 overlap the replay of step k (copy
    engines vs SMs).  Every step copies its inputs from pinned host memory
    and reads its gradients (and frame metadata) back.  out_host: one pinned
    (14 n) tensor per buffer set.  Returns the pinned meta tensors (status,
    intersection count per view) of the last step of each buffer set, for
    RenderStep.result().  The caller synchronizes."""
    dev = engine.dev
    comp = torch.cuda.current_stream(dev)
    h2d = [torch.cuda.Stream(dev) for _ in range(H2D_STREAMS)]
    d2h = torch.cuda.Stream(dev)
    nb = engine.nbuf
    loaded = [torch.cuda.Event() for _ in range(nb)]
    done = [torch.cuda.Event() for _ in range(nb)]
    read = [torch.cuda.Event() for _ in range(nb)]
    metas = [torch.empty((len(engine.cams), 4), dtype=torch.int64).pin_memory() for _ in range(nb)]
    for e in read + done:
        e.record(comp)
    for k in range(steps):
        b = k % nb
        for st in h2d:
            st.wait_event(done[b])  # the replay that last read set b finished
        engine.load(b, host_params, host_d_images, stream=h2d)
        for st in h2d[1:]:
            h2d[0].wait_stream(st)
        loaded[b].record(h2d[0])
        if flush is not None:
            flush.zero_()  # benchmarking: evict L2 (workspace comes from HBM); overlaps this step's H2D
        comp.wait_event(loaded[b])
        comp.wait_event(read[b])  # set b's previous gradients were read back
        engine.replay(b)
        if allreduce is not None:
            allreduce(engine.grads(b))  # data-parallel views: sum over ranks
        done[b].record(comp)
        d2h.wait_event(done[b])
        with torch.cuda.stream(d2h):
            out_host[b].copy_(engine.grads(b), non_blocking=True)
            metas[b].copy_(engine.meta(b), non_blocking=True)
        read[b].record(d2h)
    for e in read:
        comp.wait_event(e)
    return metas
