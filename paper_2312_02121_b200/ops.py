"""Device pipeline and autograd for the splatting hot path.

Host code is Python/PyTorch: PyTorch owns every device buffer (caching
allocator) and the stream; each stage is one call into libsplat_b200.so
(``include/splat_b200.h``).  There is no CPU fallback: CPU tensors are
rejected and a missing library raises.

Stages (reference functions they replace, sg/ = /root/reference/pkg/src/splatgrad):
  project        sg/projection.py:115-145 (+ sg/raster_forward.py:86-92,246-252)
  bin_sort       sg/binning.py:27-65
  raster_fwd     sg/raster_forward.py:116-172,222-243
  raster_bwd     sg/raster_backward.py:47-108,166-205
  project_bwd    sg/proj_backward.py:178-223
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import torch

from . import _lib
from ._lib import check

TILE = 16


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


@dataclass
class CameraParams:
    """Host-side pinhole camera (fields of sg/core.py:59-129 Camera)."""

    view: list            # 4x4 nested list (row-major, world -> camera)
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float
    far: float

    @staticmethod
    def of(cam) -> "CameraParams":
        v = cam.view
        if isinstance(v, torch.Tensor):
            v = v.detach().to("cpu", torch.float64).tolist()
        else:
            v = [[float(x) for x in row] for row in v]
        return CameraParams(v, float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy), int(cam.width),
                            int(cam.height), float(cam.near), float(cam.far))

    def c(self) -> _lib.GsCamera:
        return _lib.make_camera(self.view, self.fx, self.fy, self.cx, self.cy, self.width, self.height,
                                self.near, self.far)

    @property
    def tiles_x(self) -> int:
        return (self.width + TILE - 1) // TILE

    @property
    def tiles_y(self) -> int:
        return (self.height + TILE - 1) // TILE


def set_option(name: str, value: int) -> None:
    """Process-wide tuning option of libsplat_b200.so (gs_set_option), e.g.
    set_option("binning", 1) forces the depth-first frame binning."""
    check(_lib.load().gs_set_option(name.encode(), int(value)), "gs_set_option")


def frame_binning(n: int, cam) -> str:
    """The tile binning gs_frame_forward uses for n Gaussians on this view
    under the current options: "depth_first", "scatter" or "direct"."""
    b = int(_lib.load().gs_frame_binning(int(n), int(cam.width), int(cam.height)))
    return {1: "depth_first", 2: "scatter", 3: "direct"}[b]


def frame_tile_emit(n: int, cam) -> bool:
    """Whether gs_frame_forward's depth-first binning uses the tile-sorted
    emission for n Gaussians on this view (gs_frame_tile_emit)."""
    return bool(_lib.load().gs_frame_tile_emit(int(n), int(cam.width), int(cam.height)))


def get_option(name: str) -> int:
    """Current value of a gs_set_option option (gs_get_option)."""
    v = int(_lib.load().gs_get_option(name.encode()))
    if v < 0:
        check(v, "gs_get_option")
    return v


def _check_param(name, t, cols):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if t.dtype != torch.float32:
        raise ValueError(f"{name} must be float32, got {t.dtype}")
    if cols is None:
        if t.dim() != 1:
            raise ValueError(f"{name} must have shape (N,), got {tuple(t.shape)}")
    elif t.dim() != 2 or t.shape[1] != cols:
        raise ValueError(f"{name} must have shape (N, {cols}), got {tuple(t.shape)}")
    return t.contiguous()


def check_params(means, scales, quats, opacities, colors=None):
    means = _check_param("means", means, 3)
    n = means.shape[0]
    scales = _check_param("scales", scales, 3)
    quats = _check_param("quats", quats, 4)
    opacities = _check_param("opacities", opacities, None)
    out = [means, scales, quats, opacities]
    if colors is not None:
        out.append(_check_param("colors", colors, 3))
    for name, t in zip(("scales", "quats", "opacities", "colors"), out[1:]):
        if t.shape[0] != n:
            raise ValueError(f"{name} has {t.shape[0]} rows, expected {n}")
    return out


# --------------------------------------------------------------------- stages

@dataclass
class Projection:
    xydr: torch.Tensor      # (N,4) mean2d.x, mean2d.y, depth, radius bits
    conic: torch.Tensor     # (N,4) A, B, C, opacity
    tiles: torch.Tensor     # (N,) int32 (uint32 counts; 0 = culled)
    cov2d: torch.Tensor | None  # (N,3) a, b, c (only when requested)

    @property
    def radius(self) -> torch.Tensor:
        return self.xydr[:, 3].contiguous().view(torch.int32)


def project(means, scales, quats, opacities, cam: CameraParams, *, want_cov=False,
            status: torch.Tensor | None = None) -> Projection:
    """Stage 1 (gs_project_fwd).  ``status`` (int64[1], init -1) collects errors."""
    L = _lib.load()
    n = means.shape[0]
    dev = means.device
    xydr = torch.empty((n, 4), device=dev, dtype=torch.float32)
    conic = torch.empty((n, 4), device=dev, dtype=torch.float32)
    tiles = torch.empty((n,), device=dev, dtype=torch.int32)
    cov = torch.empty((n, 3), device=dev, dtype=torch.float32) if want_cov else None
    if status is None:
        status = torch.full((1,), -1, device=dev, dtype=torch.int64)
    camc = cam.c()
    check(L.gs_project_fwd(_ptr(means), _ptr(scales), _ptr(quats), _ptr(opacities), n, C.byref(camc),
                           _ptr(xydr), _ptr(conic), _ptr(tiles), _ptr(cov), _ptr(status), _stream()),
          "gs_project_fwd")
    return Projection(xydr, conic, tiles, cov)


def raise_status(status_value: int) -> None:
    """Turn the device status word into the reference's ValueError."""
    if status_value == -1:
        return
    s = status_value & 0xFFFFFFFFFFFFFFFF
    idx, code = s >> 8, s & 0xFF
    raise ValueError(f"gaussian {idx}: {_lib.ERR_MESSAGES.get(code, f'error {code}')}")


def scan_tiles(tiles: torch.Tensor, total: torch.Tensor) -> torch.Tensor:
    L = _lib.load()
    n = tiles.shape[0]
    offsets = torch.empty((n,), device=tiles.device, dtype=torch.int32)
    wsb = L.gs_scan_workspace_bytes(n)
    ws = torch.empty((wsb,), device=tiles.device, dtype=torch.uint8)
    check(L.gs_scan_tiles(_ptr(tiles), _ptr(offsets), n, _ptr(ws), wsb, _ptr(total), _stream()), "gs_scan_tiles")
    return offsets


@dataclass
class Bins:
    ranges: torch.Tensor       # (tiles, 2) int32 [start, end)
    sorted_keys: torch.Tensor  # (I,) int64 (tile << 32 | depth bits)
    sorted_vals: torch.Tensor  # (I,) int32 Gaussian ids
    n_isect: int


def tile_bits(n_tiles: int) -> int:
    return max(1, math.ceil(math.log2(n_tiles))) if n_tiles > 1 else 1


def sort_pairs_(keys: torch.Tensor, vals: torch.Tensor, end_bit: int):
    """gs_sort_pairs (stable onesweep radix sort of bits [0, end_bit)) on
    int64 keys / int32 values; returns the sorted (keys, vals)."""
    L = _lib.load()
    n = keys.shape[0]
    if n == 0:
        return keys, vals
    keys_alt = torch.empty_like(keys)
    vals_alt = torch.empty_like(vals)
    wsb = L.gs_sort_workspace_bytes(n, end_bit)
    ws = torch.empty((wsb,), device=keys.device, dtype=torch.uint8)
    sel = C.c_int(0)
    check(L.gs_sort_pairs(_ptr(keys), _ptr(keys_alt), _ptr(vals), _ptr(vals_alt), n, end_bit, _ptr(ws), wsb,
                          C.byref(sel), _stream()), "gs_sort_pairs")
    return (keys_alt, vals_alt) if sel.value else (keys, vals)


def emit_and_sort(proj: Projection, offsets: torch.Tensor, n_isect: int, cam: CameraParams,
                  sort: bool = True, key_bits: str = "tile_depth") -> Bins:
    """Stage 2 after the scan: key emission, onesweep sort, tile ranges.
    key_bits="tile" sorts on the tile id only (stable: index order per bin,
    sg/binning.py:27-47 assign_tiles); "tile_depth" on (tile, depth)
    (sg/binning.py:50-65 sort_bins)."""
    L = _lib.load()
    dev = proj.xydr.device
    n = proj.xydr.shape[0]
    n_tiles = cam.tiles_x * cam.tiles_y
    keys = torch.empty((n_isect,), device=dev, dtype=torch.int64)
    vals = torch.empty((n_isect,), device=dev, dtype=torch.int32)
    st = _stream()
    check(L.gs_emit_keys(_ptr(proj.xydr), _ptr(offsets), _ptr(proj.tiles), n, cam.width, cam.height,
                         _ptr(keys), _ptr(vals), st), "gs_emit_keys")
    if sort and n_isect > 0:
        if key_bits == "tile":
            keys, vals = sort_pairs_((keys >> 32).contiguous(), vals, tile_bits(n_tiles))
            keys = (keys << 32).contiguous()
        else:
            keys, vals = sort_pairs_(keys, vals, 32 + tile_bits(n_tiles))
    ranges = torch.empty((n_tiles, 2), device=dev, dtype=torch.int32)
    if sort:
        check(L.gs_tile_ranges(_ptr(keys), n_isect, _ptr(ranges), n_tiles, st), "gs_tile_ranges")
    return Bins(ranges, keys, vals, n_isect)


def tile_counts(xydr: torch.Tensor, cam: CameraParams) -> torch.Tensor:
    """Tiles touched by each (mean2d, radius) square (gs_tile_counts)."""
    L = _lib.load()
    n = xydr.shape[0]
    tiles = torch.empty((n,), device=xydr.device, dtype=torch.int32)
    check(L.gs_tile_counts(_ptr(xydr), n, cam.width, cam.height, _ptr(tiles), _stream()), "gs_tile_counts")
    return tiles


def depth_rank(depths, dev) -> "np.ndarray":
    """Rank of each float64 depth under a STABLE ascending sort (ties keep the
    given order), computed with the device radix sort on order-preserving
    transforms of the IEEE-754 bits."""
    import numpy as np
    d = torch.as_tensor(np.ascontiguousarray(depths, np.float64), device=dev)
    bits = d.view(torch.int64)
    neg = bits < 0
    # order-preserving map to unsigned: flip all bits of negatives, set the sign bit of positives
    key = torch.where(neg, ~bits, bits ^ torch.tensor(-(1 << 63), device=dev, dtype=torch.int64))
    idx = torch.arange(d.shape[0], device=dev, dtype=torch.int32)
    _, perm = sort_pairs_(key.contiguous(), idx, 64)
    rank = torch.empty_like(perm)
    rank[perm.long()] = torch.arange(d.shape[0], device=dev, dtype=torch.int32)
    return rank.cpu().numpy().astype(np.int64)


def stable_sort_pairs(keys, vals, dev, end_bit: int):
    """Host convenience: stable device sort of int64 keys carrying int values."""
    import numpy as np
    k = torch.as_tensor(np.ascontiguousarray(keys, np.int64), device=dev)
    v = torch.as_tensor(np.ascontiguousarray(vals, np.int32), device=dev)
    _, sv = sort_pairs_(k, v, end_bit)
    return sv.cpu().numpy().astype(np.int64)


def bin_sort(proj: Projection, cam: CameraParams, status: torch.Tensor | None = None) -> Bins:
    """Scan + one 16-byte D2H read (status word and intersection count) +
    emission + sort + ranges.  Raises the reference's ValueError on bad input."""
    dev = proj.xydr.device
    meta = torch.empty((2,), device=dev, dtype=torch.int64)
    if status is not None:
        meta[0:1].copy_(status)
    else:
        meta[0] = -1
    offsets = scan_tiles(proj.tiles, meta[1:2])
    host = meta.cpu()
    raise_status(int(host[0]))
    return emit_and_sort(proj, offsets, int(host[1]), cam)


@dataclass
class FrameState:
    """What the backward pass needs (autograd ctx payload, cf. RenderResult
    of sg/raster_forward.py:62-70)."""

    cam: CameraParams
    background: tuple
    early_termination: bool
    proj: Projection
    bins: Bins
    final_T: torch.Tensor
    n_contrib: torch.Tensor
    counts_fwd: torch.Tensor | None = None
    extra: dict = field(default_factory=dict)


def raster_fwd(proj: Projection, bins: Bins, colors, cam: CameraParams, background, early_termination=True,
               counts: torch.Tensor | None = None):
    L = _lib.load()
    dev = proj.xydr.device
    H, W = cam.height, cam.width
    image = torch.empty((H, W, 3), device=dev, dtype=torch.float32)
    final_T = torch.empty((H, W), device=dev, dtype=torch.float32)
    n_contrib = torch.empty((H, W), device=dev, dtype=torch.int32)
    bg = (C.c_float * 3)(*[float(b) for b in background])
    check(L.gs_raster_fwd(_ptr(bins.ranges), _ptr(bins.sorted_vals), _ptr(proj.xydr), _ptr(proj.conic),
                          _ptr(colors), bg, W, H, 1 if early_termination else 0, _ptr(image), _ptr(final_T),
                          _ptr(n_contrib), _ptr(counts), _stream()), "gs_raster_fwd")
    return image, final_T, n_contrib


def raster_bwd(state: FrameState, colors, d_image, counts: torch.Tensor | None = None):
    """Screen-space gradients per scene Gaussian (Splat2DGrads,
    sg/raster_backward.py:24-44): returns (d_rgbo (N,4), d_geo (N,4), d_c11 (N,))."""
    L = _lib.load()
    cam = state.cam
    n = state.proj.xydr.shape[0]
    dev = state.proj.xydr.device
    d_rgbo = torch.zeros((n, 4), device=dev, dtype=torch.float32)
    d_geo = torch.zeros((n, 4), device=dev, dtype=torch.float32)
    d_c11 = torch.zeros((n,), device=dev, dtype=torch.float32)
    bg = (C.c_float * 3)(*[float(b) for b in state.background])
    check(L.gs_raster_bwd(_ptr(state.bins.ranges), _ptr(state.bins.sorted_vals), _ptr(state.proj.xydr),
                          _ptr(state.proj.conic), _ptr(colors), bg, cam.width, cam.height, _ptr(state.final_T),
                          _ptr(state.n_contrib), _ptr(d_image), _ptr(d_rgbo), _ptr(d_geo), _ptr(d_c11),
                          _ptr(counts), _stream()), "gs_raster_bwd")
    return d_rgbo, d_geo, d_c11


def project_bwd(means, scales, quats, cam: CameraParams, tiles, d_geo, d_c11):
    L = _lib.load()
    n = means.shape[0]
    dev = means.device
    d_means = torch.empty((n, 3), device=dev, dtype=torch.float32)
    d_scales = torch.empty((n, 3), device=dev, dtype=torch.float32)
    d_quats = torch.empty((n, 4), device=dev, dtype=torch.float32)
    d_view = torch.empty((4, 4), device=dev, dtype=torch.float32)
    wsb = L.gs_project_bwd_workspace_bytes(n)
    ws = torch.empty((wsb,), device=dev, dtype=torch.uint8)
    camc = cam.c()
    check(L.gs_project_bwd(_ptr(means), _ptr(scales), _ptr(quats), n, C.byref(camc), _ptr(tiles), _ptr(d_geo),
                           _ptr(d_c11), _ptr(d_means), _ptr(d_scales), _ptr(d_quats), _ptr(d_view), _ptr(ws), wsb,
                           _stream()), "gs_project_bwd")
    return d_means, d_scales, d_quats, d_view


# ------------------------------------------------------------- whole frame
#
# Production path: two C-ABI calls per view (gs_frame_forward /
# gs_frame_backward, csrc/frame.cu), no host synchronisation inside, the
# intersection buffers sized by a capacity.  `check=True` (default) reads
# the 16-byte meta word after the forward to raise the reference's
# ValueError on bad input and to re-run when the capacity was too small.

_capacity_hint: dict = {}
_binning_hint: dict = {}  # (n, W, H) -> the binning a skewed view fell back to
_BINNING_CODE = {"auto": 0, "depth_first": 1, "scatter": 2, "direct": 3}
# Direct binning sizes every tile's bin by the longest per-replica segment of
# any tile (csrc/raster.cu), so a view whose pairs crowd into a few tiles
# would need tiles x 8 x that many slots (e.g. 80k Gaussians on 4 of 4096
# tiles: ~82 M slots, ~4 GB); when it needs more than DIRECT_SKEW x the pair
# count (and over DIRECT_FLOOR slots) the frame re-runs with scatter binning,
# whose room is the pair count itself.
DIRECT_SKEW = 4
DIRECT_FLOOR = 1 << 20


class _binning_option:
    """Select the frame binning for one call (gs_set_option is process-wide)."""

    def __init__(self, binning):
        self.code = None if binning in (None, "auto") else _BINNING_CODE[binning]

    def __enter__(self):
        if self.code is not None:
            self.prev = get_option("binning")
            set_option("binning", self.code)

    def __exit__(self, *exc):
        if self.code is not None:
            set_option("binning", self.prev)


def _default_capacity(n: int, key) -> int:
    hint = _capacity_hint.get(key)
    if hint is not None:
        return hint
    return max(1 << 16, 8 * n)


def needed_capacity(meta) -> int:
    """Intersection capacity a frame needs, from its meta words: the total,
    or under direct binning tiles x the longest tile list if larger."""
    return max(int(meta[1]), int(meta[2]))


@dataclass
class Frame:
    """One rendered view kept alive for its backward (cf. RenderResult,
    sg/raster_forward.py:62-70).  Owns its workspace."""

    cam: CameraParams
    background: tuple
    early_termination: bool
    n: int
    capacity: int
    ws: torch.Tensor
    image: torch.Tensor
    final_T: torch.Tensor
    n_contrib: torch.Tensor
    counts_fwd: torch.Tensor | None = None
    meta_host: tuple | None = None
    extra: dict = field(default_factory=dict)  # adapters' payload (api.render)
    binning: str | None = None  # the binning this frame was forced to (None: the library's choice)

    def view(self) -> _lib.GsFrameView:
        v = _lib.GsFrameView()
        check(_lib.load().gs_frame_view_of(self.n, self.capacity, self.cam.width, self.cam.height,
                                           self.ws.data_ptr(), C.byref(v)), "gs_frame_view_of")
        return v

    def meta(self) -> torch.Tensor:
        """The device meta words: [0] status, [1] total intersections, [2]
        capacity needed (direct binning: tiles x the longest list), [3] the
        direct-binning tile stride (0: compact bins), [4] the forward zeroed
        the backward accumulators, [5,6] the visible depth keys' min / max,
        [7] visible Gaussians, [8] depth-sort passes (depth-first binning)."""
        v = self.view()
        off = v.meta - self.ws.data_ptr()
        return self.ws[off:off + 72].view(torch.int64)

    def _meta_host(self) -> tuple:
        if self.meta_host is None:
            self.meta_host = tuple(int(x) for x in self.meta().cpu())
        return self.meta_host

    @property
    def n_isect(self) -> int:
        return self._meta_host()[1]

    @property
    def needed_capacity(self) -> int:
        return needed_capacity(self._meta_host())

    def tensors(self) -> dict:
        """Device views of the frame's intermediates (for tests/adapters)."""
        v = self.view()
        base = self.ws.data_ptr()
        n, W, H = self.n, self.cam.width, self.cam.height
        nt = self.cam.tiles_x * self.cam.tiles_y

        def sl(ptr, count, dtype, shape):
            off = ptr - base
            esz = torch.tensor([], dtype=dtype).element_size()
            return self.ws[off:off + count * esz].view(dtype).view(shape)

        m = min(self.n_isect, self.capacity)
        ranges = sl(v.ranges2, 2 * nt, torch.int32, (nt, 2))
        stride = self._meta_host()[3]
        if stride > 0:  # direct binning: tile t's list at [t * stride, + count) -> compact (tile order)
            cnt = (ranges[:, 1] - ranges[:, 0]).long()
            src = torch.repeat_interleave(ranges[:, 0].long(), cnt)
            pos = torch.arange(int(cnt.sum()), device=cnt.device) - torch.repeat_interleave(
                torch.cumsum(cnt, 0) - cnt, cnt)
            sorted_vals = sl(v.sorted_vals, self.capacity, torch.int32, (self.capacity,))[src + pos].contiguous()
            sorted_tile_keys = torch.repeat_interleave(torch.arange(nt, device=cnt.device, dtype=torch.int32), cnt)
            end = torch.cumsum(cnt, 0)
            ranges = torch.stack([end - cnt, end], 1).to(torch.int32)
            ranges[cnt == 0] = 0  # empty tiles: (0, 0), as the other binnings write them
        else:  # compact tile-ordered lists; the tile keys follow from the ranges (the
            # tile-sorted emission writes no keys)
            sorted_vals = sl(v.sorted_vals, m, torch.int32, (m,))
            cnt = (ranges[:, 1] - ranges[:, 0]).long()
            sorted_tile_keys = torch.repeat_interleave(torch.arange(nt, device=cnt.device, dtype=torch.int32), cnt)
        mh = self._meta_host()
        n_sorted = min(mh[7], n)  # depth-first binning: the visible Gaussians by (depth, index)
        dptr = v.depth_order_alt if mh[8] & 1 else v.depth_order
        return dict(xydr=sl(v.xydr4, 4 * n, torch.float32, (n, 4)), conic=sl(v.conic4, 4 * n, torch.float32, (n, 4)),
                    tiles=sl(v.tiles, n, torch.int32, (n,)), depth_order=sl(dptr, n_sorted, torch.int32, (n_sorted,)),
                    sorted_tile_keys=sorted_tile_keys, sorted_vals=sorted_vals, ranges=ranges,
                    d_geo=sl(v.d_geo4 - 16, 8 * n, torch.float32, (n, 8))[:, 4:8],  # rows of [d_rgbo | d_geo]
                    d_c11=sl(v.d_c11, n, torch.float32, (n,)),
                    rec_count=sl(v.rec_count, 4 * nt, torch.int32, (nt, 4)))


def frame_workspace(n: int, capacity: int, width: int, height: int, device) -> torch.Tensor:
    """A frame workspace (gs_frame_workspace_bytes) marked not clean
    (gs_frame_workspace_init), for callers that keep one across frames."""
    L = _lib.load()
    ws = torch.empty((L.gs_frame_workspace_bytes(n, capacity, width, height),), device=device, dtype=torch.uint8)
    check(L.gs_frame_workspace_init(n, capacity, width, height, ws.data_ptr(), _stream()),
          "gs_frame_workspace_init")
    return ws


def frame_forward(means, scales, quats, opacities, colors, cam: CameraParams, background=(0.0, 0.0, 0.0),
                  early_termination=True, *, capacity: int | None = None, counts=False, check_meta=True,
                  ws: torch.Tensor | None = None, events=None, binning: str | None = None,
                  projected: bool = False) -> Frame:
    """gs_frame_forward: image, final_T, n_contrib of one view.  binning:
    force "depth_first" / "scatter" / "direct" for this call (default: the
    library's choice, or the scatter fallback a skewed view of this size
    needed before -- see DIRECT_SKEW).  projected: frames_project already
    projected this view into `ws` (gs_frame_forward_projected; needs the
    capacity and workspace given, check_meta=False, no counts)."""
    L = _lib.load()
    if projected:
        if ws is None or capacity is None or check_meta or counts:
            raise ValueError("frame_forward(projected=True) needs ws and capacity, check_meta=False, no counts")
        means, scales, quats, opacities, colors = check_params(means, scales, quats, opacities, colors)
        n, dev, H, W = means.shape[0], means.device, cam.height, cam.width
        image = torch.empty((H, W, 3), device=dev, dtype=torch.float32)
        final_T = torch.empty((H, W), device=dev, dtype=torch.float32)
        n_contrib = torch.empty((H, W), device=dev, dtype=torch.int32)
        camc = cam.c()
        bg = (C.c_float * 3)(*[float(b) for b in background])
        check(L.gs_frame_forward_projected(_ptr(means), _ptr(scales), _ptr(quats), _ptr(opacities), _ptr(colors), n,
                                           C.byref(camc), bg, 1 if early_termination else 0, int(capacity),
                                           _ptr(ws), ws.numel(), _ptr(image), _ptr(final_T), _ptr(n_contrib),
                                           _event_array(events), _stream()), "gs_frame_forward_projected")
        return Frame(cam, tuple(float(b) for b in background), bool(early_termination), n, int(capacity), ws, image,
                     final_T, n_contrib, None, binning="depth_first")
    means, scales, quats, opacities, colors = check_params(means, scales, quats, opacities, colors)
    n = means.shape[0]
    dev = means.device
    key = (n, cam.width, cam.height)
    cap = int(capacity) if capacity is not None else _default_capacity(n, key)
    H, W = cam.height, cam.width
    camc = cam.c()
    bg = (C.c_float * 3)(*[float(b) for b in background])
    bsel = binning or _binning_hint.get(key)
    while True:
        wsb = L.gs_frame_workspace_bytes(n, cap, W, H)
        if ws is None or ws.numel() < wsb:
            ws = frame_workspace(n, cap, W, H, dev)
        image = torch.empty((H, W, 3), device=dev, dtype=torch.float32)
        final_T = torch.empty((H, W), device=dev, dtype=torch.float32)
        n_contrib = torch.empty((H, W), device=dev, dtype=torch.int32)
        cnt = torch.zeros((4,), device=dev, dtype=torch.int64) if counts else None
        with _binning_option(bsel):
            check(L.gs_frame_forward(_ptr(means), _ptr(scales), _ptr(quats), _ptr(opacities), _ptr(colors), n,
                                     C.byref(camc), bg, 1 if early_termination else 0, cap, _ptr(ws), ws.numel(),
                                     _ptr(image), _ptr(final_T), _ptr(n_contrib), _ptr(cnt), _event_array(events),
                                     _stream()), "gs_frame_forward")
        fr = Frame(cam, tuple(float(b) for b in background), bool(early_termination), n, cap, ws, image, final_T,
                   n_contrib, cnt, binning=bsel)
        if not check_meta:
            return fr
        m = fr._meta_host()
        raise_status(m[0])
        if m[3] > 0 and binning is None and m[2] > max(DIRECT_SKEW * m[1], DIRECT_FLOOR):
            bsel = _binning_hint[key] = "scatter"  # skewed view: direct binning's room would explode
            cap = _capacity_hint[key] = max(1 << 16, int(m[1] * 1.25) + 1024)
            ws = None
            continue
        need = needed_capacity(m)
        _capacity_hint[key] = max(1 << 16, int(need * 1.25) + 1024)
        if need <= cap:
            return fr
        cap = _capacity_hint[key]
        ws = None


def frames_project(means, scales, quats, opacities, cams, capacities, workspaces) -> None:
    """gs_frames_project: the depth-first projection of every view of a step
    (each into its own workspace, sized for its capacity) in one pass over
    the Gaussians; each view then continues with
    frame_forward(..., projected=True)."""
    L = _lib.load()
    nv = len(cams)
    if nv == 0:
        return
    n = means.shape[0]
    camc = (_lib.GsCamera * nv)(*[c.c() for c in cams])
    caps = (C.c_int64 * nv)(*[int(c) for c in capacities])
    wss = (C.c_void_p * nv)(*[w.data_ptr() for w in workspaces])
    wsb = (C.c_size_t * nv)(*[w.numel() for w in workspaces])
    vp = lambda a: C.cast(a, C.c_void_p)
    check(L.gs_frames_project(_ptr(means), _ptr(scales), _ptr(quats), _ptr(opacities), n, nv, camc, vp(caps),
                              vp(wss), vp(wsb), _stream()), "gs_frames_project")


def frames_projectable(n: int, cams) -> bool:
    """Whether every view would use depth-first binning (gs_frames_project)."""
    return all(frame_binning(n, c) == "depth_first" for c in cams)


def _event_array(events):
    """torch.cuda.Event list -> void*[] of raw cudaEvent_t handles (None -> NULL)."""
    if not events:
        return None
    arr = (C.c_void_p * len(events))()
    for i, e in enumerate(events):
        arr[i] = None if e is None else int(e.cuda_event)
    return arr


def frame_backward(fr: Frame, means, scales, quats, colors, d_image, *, counts=False, events=None, out=None,
                   accumulate=False, keep_screen=False, wait_before_accumulate=None, project=True):
    """gs_frame_backward: the SceneGradients fields (sg/proj_backward.py:25-50).
    out: optional dict of contiguous output tensors d_mean (n,3), d_scale
    (n,3), d_quat (n,4), d_rgbo (n,4) to write (accumulate=False) or add
    this view's gradients into (accumulate=True).  keep_screen: leave the
    screen-space gradients (Splat2DGrads) readable through fr.tensors()
    (d_geo, d_c11); otherwise the projection backward clears them as it
    reads them, so the next frame needs no zeroing pass.
    wait_before_accumulate: a torch.cuda.Event the stream waits on between
    the raster backward and the projection backward (which adds into `out`):
    views of one step on several streams then overlap their raster backwards
    and serialise only the accumulation.  project=False: raster backward
    only -- the screen-space gradients stay in the workspace
    (frame_screen_grads) for frame_project_backward, e.g. after a reduction
    across ranks."""
    L = _lib.load()
    H, W = fr.cam.height, fr.cam.width
    if tuple(d_image.shape) != (H, W, 3):
        raise ValueError(f"d_image must have shape {(H, W, 3)}, got {tuple(d_image.shape)}")  # sg/raster_backward.py:180-183
    d_image = d_image.contiguous().to(torch.float32)
    n = fr.n
    dev = means.device
    if out is not None:
        d_means, d_scales, d_quats, d_rgbo = out["d_mean"], out["d_scale"], out["d_quat"], out["d_rgbo"]
        for t, cols in ((d_means, 3), (d_scales, 3), (d_quats, 4), (d_rgbo, 4)):
            if t.shape != (n, cols) or not t.is_contiguous() or t.dtype != torch.float32:
                raise ValueError("frame_backward: out tensors must be contiguous float32 (n, 3|3|4|4)")
    else:
        if accumulate:
            raise ValueError("frame_backward: accumulate needs out tensors")
        d_means = torch.empty((n, 3), device=dev, dtype=torch.float32)
        d_scales = torch.empty((n, 3), device=dev, dtype=torch.float32)
        d_quats = torch.empty((n, 4), device=dev, dtype=torch.float32)
        d_rgbo = torch.empty((n, 4), device=dev, dtype=torch.float32)
    d_view = torch.empty((4, 4), device=dev, dtype=torch.float32)
    cnt = torch.zeros((3,), device=dev, dtype=torch.int64) if counts else None
    camc = fr.cam.c()
    bg = (C.c_float * 3)(*fr.background)
    flags = (1 if accumulate else 0) | (2 if keep_screen else 0) | (0 if project else 8)
    if wait_before_accumulate is not None:
        flags |= 4
        events = (list(events) + [None] * 3)[:3] if events else [None, None, None]
        events.append(wait_before_accumulate)
    check(L.gs_frame_backward(_ptr(means), _ptr(scales), _ptr(quats), _ptr(colors), n, C.byref(camc), bg,
                              fr.capacity, _ptr(fr.ws), fr.ws.numel(), _ptr(fr.final_T), _ptr(fr.n_contrib),
                              _ptr(d_image), _ptr(d_means), _ptr(d_scales), _ptr(d_quats), _ptr(d_rgbo),
                              _ptr(d_view), flags, _ptr(cnt), _event_array(events), _stream()),
          "gs_frame_backward")
    return dict(d_mean=d_means, d_scale=d_scales, d_quat=d_quats, d_opacity=d_rgbo[:, 3], d_color=d_rgbo[:, :3],
                d_view=d_view, d_rgbo=d_rgbo, counts=cnt)


def frame_screen_grads(fr: Frame):
    """The screen-space gradient accumulators of a frame (after
    frame_backward(project=False)): rows (n, 8) = [d_color 3, d_opacity,
    d_mean2d 2, d_cov00, d_cov01] and d_c11 (n,) -- device views into the
    workspace, reducible in place across ranks.  Every Gaussian is marked
    touched (gs_frame_view.touched): rows changed by the caller are then all
    read by the projection backward."""
    v = fr.view()
    base = fr.ws.data_ptr()
    off = v.touched - base
    fr.ws[off:off + 4 * ((fr.n + 31) // 32)].fill_(255)
    off = v.bwd_accum - base
    rows = fr.ws[off:off + 32 * fr.n].view(torch.float32).view(fr.n, 8)
    off = v.d_c11 - base
    return rows, fr.ws[off:off + 4 * fr.n].view(torch.float32)


def frame_project_backward(fr: Frame, means, scales, quats, out: dict, d_view: torch.Tensor, begin=0, end=None, *,
                           accumulate=False, add_view=False, keep_screen=False, vis_from_grads=False):
    """gs_frame_project_backward: the projection backward of frame `fr`
    (sg/proj_backward.py:178-223) over Gaussians [begin, end) from the
    screen-space gradients in its workspace, into `out` (d_mean, d_scale,
    d_quat, d_rgbo full (n, .) tensors; rows begin..end-1 written or, with
    accumulate, added to) and d_view (4x4; overwritten or, with add_view,
    added to).  vis_from_grads: a Gaussian this frame culled but whose rows
    are non-zero (summed over tile bands) is treated as visible."""
    L = _lib.load()
    n = fr.n
    end = n if end is None else int(end)
    camc = fr.cam.c()
    flags = (1 if accumulate else 0) | (2 if keep_screen else 0) | (16 if add_view else 0) | \
        (32 if vis_from_grads else 0)
    check(L.gs_frame_project_backward(_ptr(means), _ptr(scales), _ptr(quats), n, C.byref(camc), fr.capacity,
                                      _ptr(fr.ws), fr.ws.numel(), int(begin), end, _ptr(out["d_mean"]),
                                      _ptr(out["d_scale"]), _ptr(out["d_quat"]), _ptr(out["d_rgbo"]), _ptr(d_view),
                                      flags, _stream()), "gs_frame_project_backward")


def frame_views_project_backward(frames, means, scales, quats, out: dict, d_views: torch.Tensor, begin=0, end=None,
                                 *, accumulate=False, add_view=False, keep_screen=False):
    """gs_frame_views_project_backward: the projection backward of every
    frame in `frames` (one per view, each after frame_backward(project=False)
    on its own workspace) in one pass over Gaussians [begin, end):
    sg/proj_backward.py:178-223 per view, summed over the views, into `out`
    (d_mean, d_scale, d_quat, d_rgbo full (n, .) tensors; rows written or,
    with accumulate, added to) and d_views (views, 4, 4; per view,
    overwritten or, with add_view, added to)."""
    L = _lib.load()
    nv = len(frames)
    if nv == 0:
        return
    n = frames[0].n
    end = n if end is None else int(end)
    if any(f.n != n for f in frames):
        raise ValueError("frame_views_project_backward: frames of different scenes")
    if tuple(d_views.shape) != (nv, 4, 4) or not d_views.is_contiguous():
        raise ValueError("frame_views_project_backward: d_views must be contiguous (views, 4, 4)")
    cams = (_lib.GsCamera * nv)(*[f.cam.c() for f in frames])
    caps = (C.c_int64 * nv)(*[f.capacity for f in frames])
    wss = (C.c_void_p * nv)(*[f.ws.data_ptr() for f in frames])
    wsb = (C.c_size_t * nv)(*[f.ws.numel() for f in frames])
    flags = (1 if accumulate else 0) | (2 if keep_screen else 0) | (16 if add_view else 0)
    vp = lambda a: C.cast(a, C.c_void_p)
    check(L.gs_frame_views_project_backward(_ptr(means), _ptr(scales), _ptr(quats), n, nv, cams, vp(caps), vp(wss),
                                            vp(wsb),
                                            int(begin), end, _ptr(out["d_mean"]), _ptr(out["d_scale"]),
                                            _ptr(out["d_quat"]), _ptr(out["d_rgbo"]), _ptr(d_views), flags,
                                            _stream()), "gs_frame_views_project_backward")


# ------------------------------------------------------ staged (per-stage) path
# The same frame through the individual stage entry points and the 64-bit
# (tile << 32 | depth) key sort; used by the parity harness (it exposes every
# intermediate, including cov2d) and checked equal to the frame path.

def render_forward(means, scales, quats, opacities, colors, cam: CameraParams, background=(0.0, 0.0, 0.0),
                   early_termination=True, *, want_cov=False, counts=False):
    """project -> bin/sort -> raster fwd.  Returns (image (H,W,3), FrameState)."""
    means, scales, quats, opacities, colors = check_params(means, scales, quats, opacities, colors)
    status = torch.full((1,), -1, device=means.device, dtype=torch.int64)
    proj = project(means, scales, quats, opacities, cam, want_cov=want_cov, status=status)
    bins = bin_sort(proj, cam, status)
    cnt = torch.zeros((4,), device=means.device, dtype=torch.int64) if counts else None
    image, final_T, n_contrib = raster_fwd(proj, bins, colors, cam, background, early_termination, cnt)
    state = FrameState(cam, tuple(float(b) for b in background), bool(early_termination), proj, bins, final_T,
                       n_contrib, cnt)
    return image, state


def render_backward(state: FrameState, means, scales, quats, colors, d_image, *, counts=False):
    """raster bwd -> projection bwd.  Returns dict of SceneGradients fields
    (sg/proj_backward.py:25-50) as tensors plus the screen-space grads."""
    H, W = state.cam.height, state.cam.width
    if tuple(d_image.shape) != (H, W, 3):
        raise ValueError(f"d_image must have shape {(H, W, 3)}, got {tuple(d_image.shape)}")  # sg/raster_backward.py:180-183
    d_image = d_image.contiguous().to(torch.float32)
    cnt = torch.zeros((3,), device=means.device, dtype=torch.int64) if counts else None
    d_rgbo, d_geo, d_c11 = raster_bwd(state, colors, d_image, cnt)
    d_means, d_scales, d_quats, d_view = project_bwd(means, scales, quats, state.cam, state.proj.tiles, d_geo, d_c11)
    return dict(d_mean=d_means, d_scale=d_scales, d_quat=d_quats, d_opacity=d_rgbo[:, 3], d_color=d_rgbo[:, :3],
                d_view=d_view, d_rgbo=d_rgbo, d_geo=d_geo, d_c11=d_c11, counts=cnt)


class RasterizeGaussians(torch.autograd.Function):
    """Differentiable render of one view (production frame path).

    forward(means (N,3), scales (N,3), quats (N,4) (w,x,y,z), opacities (N,),
            colors (N,3), viewmat (4,4), camera (fx, fy, cx, cy, W, H, near, far),
            background (3,), early_termination) -> image (H, W, 3), final_T, n_contrib
    backward returns d_means, d_scales, d_quats, d_opacities, d_colors,
    d_viewmat -- field by field the reference's SceneGradients
    (sg/proj_backward.py:34-39).
    """

    @staticmethod
    def forward(ctx, means, scales, quats, opacities, colors, viewmat, intrinsics, background, early_termination):
        fx, fy, cx, cy, W, H, near, far = intrinsics
        cam = CameraParams(viewmat.detach().to("cpu", torch.float64).tolist(), fx, fy, cx, cy, W, H, near, far)
        fr = frame_forward(means, scales, quats, opacities, colors, cam, background, early_termination)
        ctx.frame = fr
        ctx.view_device = viewmat.device
        ctx.save_for_backward(means, scales, quats, colors)
        ctx.mark_non_differentiable(fr.final_T, fr.n_contrib)
        return fr.image, fr.final_T, fr.n_contrib

    @staticmethod
    def backward(ctx, d_image, _d_T, _d_nc):
        means, scales, quats, colors = ctx.saved_tensors
        g = frame_backward(ctx.frame, means.contiguous(), scales.contiguous(), quats.contiguous(),
                           colors.contiguous(), d_image)
        ctx.frame = None  # release the workspace
        return (g["d_mean"], g["d_scale"], g["d_quat"], g["d_opacity"], g["d_color"],
                g["d_view"].to(ctx.view_device), None, None, None)


def rasterize(means, scales, quats, opacities, colors, viewmat, fx, fy, cx, cy, width, height, near=0.01,
              far=100.0, background=(0.0, 0.0, 0.0), early_termination=True):
    """Autograd entry point: returns (image (H,W,3), final_T (H,W), n_contrib (H,W))."""
    if not isinstance(viewmat, torch.Tensor):
        viewmat = torch.as_tensor(viewmat, dtype=torch.float32)
    return RasterizeGaussians.apply(means, scales, quats, opacities, colors, viewmat,
                                    (fx, fy, cx, cy, int(width), int(height), near, far),
                                    tuple(float(b) for b in background), bool(early_termination))
