"""The reference's Python API on the B200 path (drop-in boundary).

Same names, argument meaning and error behaviour as the public API of the
reference package (`sg/__init__.py:4-119`, sg/ = /root/reference/pkg/src/
splatgrad) for the hot path:

  render, render_brute_force        sg/raster_forward.py:255-294
  scene_backward                    sg/proj_backward.py:178-223
  accumulate_image_backward         sg/raster_backward.py:166-205
  project_gaussian                  sg/projection.py:115-145
  assign_tiles, sort_bins           sg/binning.py:27-65
  eval_alpha, composite_pixel       sg/raster_forward.py:175-219
  composite_pixel_backward,
  transmittance_replay              sg/raster_backward.py:111-163

plus the value types they exchange (Gaussian3D, Camera, ProjectedGaussian,
TileGrid, RenderResult, RenderAux, ImageBuffer, Splat2DGrads,
SceneGradients).  All arithmetic runs in the CUDA kernels of
libsplat_b200.so (fp32); this module only converts between the reference's
list-of-dataclasses / float64 numpy world and device tensors.  Results are
float64 arrays holding the fp32 values, so callers written against the
reference work unchanged.  Requires a CUDA device (no CPU fallback).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np
import torch

from . import ops, pixels

# constants (sg/binning.py:8, sg/projection.py:17, sg/raster_forward.py:21-30, sg/core.py:13)
TILE_SIZE = 16
DILATION = 0.3
ALPHA_MIN = 1.0 / 255.0
ALPHA_MAX = 0.999
T_MIN = 1e-4
SIGMA_CUT = 4.5
QUAT_NORM_EPS = 1e-12


def _as_f64(value, shape, name):
    arr = np.asarray(value, dtype=np.float64)
    if arr.shape != shape:
        raise ValueError(f"{name} must have shape {shape}, got {arr.shape}")
    return arr


@dataclass
class Gaussian3D:
    """sg/core.py:23-56."""

    mean: np.ndarray
    scale: np.ndarray
    quat: np.ndarray
    opacity: float
    color: np.ndarray

    def __post_init__(self):
        self.mean = _as_f64(self.mean, (3,), "mean")
        self.scale = _as_f64(self.scale, (3,), "scale")
        self.quat = _as_f64(self.quat, (4,), "quat")
        self.opacity = float(self.opacity)
        self.color = _as_f64(self.color, (3,), "color")

    def validate(self):
        if not np.all(np.isfinite(self.mean)):
            raise ValueError("mean must be finite")
        if not np.all(np.isfinite(self.scale)) or np.any(self.scale <= 0.0):
            raise ValueError("scale components must be positive")
        if np.sqrt(np.dot(self.quat, self.quat)) <= QUAT_NORM_EPS:
            raise ValueError("quat norm is too small")
        if not 0.0 <= self.opacity <= 1.0:
            raise ValueError("opacity must lie in [0, 1]")
        if np.any(self.color < 0.0) or np.any(self.color > 1.0):
            raise ValueError("color channels must lie in [0, 1]")


@dataclass
class Camera:
    """sg/core.py:59-129 (view = 4x4 world-to-camera)."""

    view: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float
    far: float

    def __post_init__(self):
        self.view = _as_f64(self.view, (4, 4), "view")
        self.fx, self.fy, self.cx, self.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        self.width, self.height = int(self.width), int(self.height)
        self.near, self.far = float(self.near), float(self.far)

    @property
    def rotation(self):
        return self.view[:3, :3]

    @property
    def translation(self):
        return self.view[:3, 3]

    def projection_matrix(self):
        n, f = self.near, self.far
        p = np.zeros((4, 4))
        p[0, 0] = 2.0 * self.fx / self.width
        p[1, 1] = 2.0 * self.fy / self.height
        p[2, 2] = (f + n) / (f - n)
        p[2, 3] = -2.0 * f * n / (f - n)
        p[3, 2] = 1.0
        return p

    def validate(self):
        if not np.all(np.isfinite(self.view)):
            raise ValueError("view must be finite")
        r = self.rotation
        if np.max(np.abs(r @ r.T - np.eye(3))) > 1e-9:
            raise ValueError("view rotation block must be orthonormal")
        if abs(np.linalg.det(r) - 1.0) > 1e-9:
            raise ValueError("view rotation block must have determinant +1")
        if np.max(np.abs(self.view[3] - np.array([0.0, 0.0, 0.0, 1.0]))) > 1e-12:
            raise ValueError("view bottom row must be [0, 0, 0, 1]")
        if not 0.0 < self.near < self.far:
            raise ValueError("clip planes must satisfy 0 < near < far")
        if self.width < 1 or self.height < 1:
            raise ValueError("image dimensions must be at least 1 pixel")
        if self.fx <= 0.0 or self.fy <= 0.0:
            raise ValueError("focal lengths must be positive")


@dataclass
class ProjectedGaussian:
    """sg/projection.py:20-33."""

    t_cam: np.ndarray
    mean2d: np.ndarray
    cov2d: np.ndarray
    depth: float
    radius: int
    source_index: int


@dataclass
class TileGrid:
    """sg/binning.py:11-24 (bins hold indices into `projected`)."""

    tile_size: int
    tiles_x: int
    tiles_y: int
    bins: list

    def bin_at(self, tx, ty):
        return self.bins[ty * self.tiles_x + tx]


@dataclass
class ImageBuffer:
    width: int
    height: int
    channels: np.ndarray


@dataclass
class RenderAux:
    final_T: np.ndarray
    n_contrib: np.ndarray


class PixelAux(NamedTuple):
    """sg/raster_forward.py:57-59."""

    final_T: float
    n_contrib: int


@dataclass
class RenderResult:
    """sg/raster_forward.py:62-70, plus the device state of the frame."""

    image: ImageBuffer
    aux: RenderAux
    grid: TileGrid
    projected: list
    background: np.ndarray
    _gpu: object = field(default=None, repr=False)


@dataclass
class Splat2DGrads:
    """sg/raster_backward.py:24-44."""

    d_color: np.ndarray
    d_opacity: np.ndarray
    d_mean2d: np.ndarray
    d_cov2d: np.ndarray

    @classmethod
    def zeros(cls, n):
        return cls(np.zeros((n, 3)), np.zeros(n), np.zeros((n, 2)), np.zeros((n, 2, 2)))


@dataclass
class SceneGradients:
    """sg/proj_backward.py:25-50."""

    d_mean: np.ndarray
    d_scale: np.ndarray
    d_quat: np.ndarray
    d_opacity: np.ndarray
    d_color: np.ndarray
    d_view: np.ndarray

    @classmethod
    def zeros(cls, n):
        return cls(np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 4)), np.zeros(n), np.zeros((n, 3)),
                   np.zeros((4, 4)))


# ------------------------------------------------------------------ helpers

def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2312_02121_b200.api needs a CUDA device (there is no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def _scene_tensors(scene, dev):
    n = len(scene)
    means = np.zeros((n, 3), np.float32)
    scales = np.zeros((n, 3), np.float32)
    quats = np.zeros((n, 4), np.float32)
    opac = np.zeros(n, np.float32)
    colors = np.zeros((n, 3), np.float32)
    for i, g in enumerate(scene):
        means[i], scales[i], quats[i], opac[i], colors[i] = g.mean, g.scale, g.quat, g.opacity, g.color
    t = lambda a: torch.as_tensor(a, device=dev)
    return t(means), t(scales), t(quats), t(opac), t(colors)


def _np(t):
    return t.detach().cpu().numpy()


def _projected_list(camera, scene, proj: ops.Projection):
    """ProjectedGaussian records (compacted, source order) from the device
    projection; t_cam is the camera-space point the kernel projected."""
    xydr = _np(proj.xydr)
    cov = _np(proj.cov2d).astype(np.float64)
    vis = np.nonzero(_np(proj.tiles) > 0)[0]
    radius = xydr[:, 3].copy().view(np.int32)
    out = []
    V = camera.view
    for i in vis:
        m = scene[i].mean
        t_cam = V @ np.array([m[0], m[1], m[2], 1.0])
        c = cov[i]
        out.append(ProjectedGaussian(t_cam=t_cam, mean2d=xydr[i, :2].astype(np.float64),
                                     cov2d=np.array([[c[0], c[1]], [c[1], c[2]]]), depth=float(xydr[i, 2]),
                                     radius=int(radius[i]), source_index=int(i)))
    return out, vis


def _grid_from_bins(bins: ops.Bins, cam: ops.CameraParams, vis):
    remap = -np.ones(int(vis.max()) + 1 if len(vis) else 1, np.int64)
    remap[vis] = np.arange(len(vis))
    ranges = _np(bins.ranges).astype(np.int64)
    vals = remap[_np(bins.sorted_vals).astype(np.int64)] if bins.n_isect else np.zeros(0, np.int64)
    lists = [vals[a:b].tolist() for a, b in ranges]
    return TileGrid(TILE_SIZE, cam.tiles_x, cam.tiles_y, lists)


# ------------------------------------------------------------------ API

def render(scene, camera: Camera, background, *, early_termination=True) -> RenderResult:
    """sg/raster_forward.py:255-271 on the GPU, through the production frame
    path (gs_frame_forward: the frame binning, raster_fwd_kernel with commit
    records -- what bench.py times).  The ProjectedGaussian list (which needs
    cov2d, not stored by the frame) comes from the stage projection kernel,
    the same arithmetic bit for bit."""
    dev = _device()
    bg = np.asarray(background, dtype=np.float64)
    cam = ops.CameraParams.of(camera)
    t = _scene_tensors(scene, dev)
    fr = ops.frame_forward(*t, cam, tuple(bg), early_termination)
    proj = ops.project(t[0], t[1], t[2], t[3], cam, want_cov=True)
    tv = fr.tensors()
    projected, vis = _projected_list(camera, scene, proj)
    grid = _grid_from_bins(ops.Bins(tv["ranges"], None, tv["sorted_vals"], fr.n_isect), cam, vis)
    fr.extra = dict(tensors=t, tv=tv)
    return RenderResult(image=ImageBuffer(cam.width, cam.height, _np(fr.image).astype(np.float64)),
                        aux=RenderAux(_np(fr.final_T).astype(np.float64), _np(fr.n_contrib).astype(np.int64)),
                        grid=grid, projected=projected, background=bg, _gpu=fr)


def render_brute_force(scene, camera: Camera, background, *, early_termination=True) -> RenderResult:
    """sg/raster_forward.py:274-294: every tile composites the full global
    (depth, index) order -- same raster kernel, one list for all tiles."""
    dev = _device()
    bg = np.asarray(background, dtype=np.float64)
    cam = ops.CameraParams.of(camera)
    t = _scene_tensors(scene, dev)
    means, scales, quats, opac, colors = ops.check_params(*t)
    status = torch.full((1,), -1, device=dev, dtype=torch.int64)
    proj = ops.project(means, scales, quats, opac, cam, want_cov=True, status=status)
    ops.raise_status(int(status.item()))
    projected, vis = _projected_list(camera, scene, proj)
    order = sorted(range(len(projected)), key=lambda i: (projected[i].depth, projected[i].source_index))
    gids = torch.as_tensor(np.asarray([projected[i].source_index for i in order], np.int32), device=dev)
    n_tiles = cam.tiles_x * cam.tiles_y
    ranges = torch.zeros((n_tiles, 2), device=dev, dtype=torch.int32)
    ranges[:, 1] = len(order)
    bins = ops.Bins(ranges, torch.zeros(len(order), device=dev, dtype=torch.int64), gids.contiguous(), len(order))
    image, final_T, n_contrib = ops.raster_fwd(proj, bins, colors, cam, tuple(bg), early_termination)
    st = ops.FrameState(cam, tuple(bg), bool(early_termination), proj, bins, final_T, n_contrib)
    st.extra["tensors"] = t
    grid = TileGrid(TILE_SIZE, cam.tiles_x, cam.tiles_y, [list(order) for _ in range(n_tiles)])
    return RenderResult(ImageBuffer(cam.width, cam.height, _np(image).astype(np.float64)),
                        RenderAux(_np(final_T).astype(np.float64), _np(n_contrib).astype(np.int64)), grid, projected,
                        bg, st)


def _check_dimage(result, d_image):
    d_image = np.asarray(d_image, dtype=np.float64)
    h, w = result.image.height, result.image.width
    if d_image.shape != (h, w, 3):
        raise ValueError(f"d_image must have shape {(h, w, 3)}, got {d_image.shape}")  # sg/raster_backward.py:180-183
    return d_image


def _state(scene, result):
    st = result._gpu
    if st is None:
        raise ValueError("result was not produced by paper_2312_02121_b200.api.render")
    t = st.extra.get("tensors")
    if t is None or t[0].shape[0] != len(scene):
        t = _scene_tensors(scene, _device())
    return st, t


def _stage_state(st) -> ops.FrameState:
    """A frame-path result as the stage kernels' FrameState (its own
    projection, compacted bins, final_T and n_contrib)."""
    if isinstance(st, ops.FrameState):
        return st
    tv = st.extra.get("tv") or st.tensors()
    proj = ops.Projection(tv["xydr"], tv["conic"], tv["tiles"], None)
    bins = ops.Bins(tv["ranges"], None, tv["sorted_vals"], st.n_isect)
    return ops.FrameState(st.cam, st.background, st.early_termination, proj, bins, st.final_T, st.n_contrib)


def accumulate_image_backward(scene, result: RenderResult, d_image) -> Splat2DGrads:
    """sg/raster_backward.py:166-205 on the GPU (screen-space gradients):
    the list-staging raster backward (gs_raster_bwd) over the frame's own
    projection and bins."""
    d_image = _check_dimage(result, d_image)
    st, t = _state(scene, result)
    d = torch.as_tensor(d_image.astype(np.float32), device=t[0].device)
    d_rgbo, d_geo, d_c11 = ops.raster_bwd(_stage_state(st), t[4], d)
    geo = _np(d_geo).astype(np.float64)
    c11 = _np(d_c11).astype(np.float64)
    rgbo = _np(d_rgbo).astype(np.float64)
    cov = np.stack([geo[:, 2], geo[:, 3], geo[:, 3], c11], axis=1).reshape(-1, 2, 2)
    return Splat2DGrads(d_color=rgbo[:, :3].copy(), d_opacity=rgbo[:, 3].copy(), d_mean2d=geo[:, :2].copy(),
                        d_cov2d=cov)


def scene_backward(scene, camera: Camera, result: RenderResult, d_image) -> SceneGradients:
    """sg/proj_backward.py:178-223 on the GPU: gs_frame_backward (the record-
    driven raster backward + the projection backward) for a render() result;
    the stage kernels for a render_brute_force() result."""
    d_image = _check_dimage(result, d_image)
    st, t = _state(scene, result)
    d = torch.as_tensor(d_image.astype(np.float32), device=t[0].device)
    if isinstance(st, ops.FrameState):
        g = ops.render_backward(st, t[0], t[1], t[2], t[4], d)
    else:
        g = ops.frame_backward(st, t[0], t[1], t[2], t[4], d)
    f = lambda x: _np(x).astype(np.float64)
    return SceneGradients(d_mean=f(g["d_mean"]), d_scale=f(g["d_scale"]), d_quat=f(g["d_quat"]),
                          d_opacity=f(g["d_opacity"]).copy(), d_color=f(g["d_color"]).copy(), d_view=f(g["d_view"]))


def project_gaussian(g: Gaussian3D, camera: Camera, source_index=0):
    """sg/projection.py:115-145 for one splat (a batch of one on the GPU).
    Returns ProjectedGaussian, or None when culled; raises ValueError on
    degenerate input like the reference."""
    dev = _device()
    t = _scene_tensors([g], dev)
    cam = ops.CameraParams.of(camera)
    status = torch.full((1,), -1, device=dev, dtype=torch.int64)
    proj = ops.project(*t[:4], cam, want_cov=True, status=status)
    s = int(status.item())
    if s != -1:
        raise ValueError(ops._lib.ERR_MESSAGES.get(s & 0xFF, "degenerate input"))
    projected, _ = _projected_list(camera, [g], proj)
    if not projected:
        return None
    p = projected[0]
    p.source_index = source_index
    return p


def _proj_tensors(projected, dev):
    """(x, y, depth, radius) rows for the binning kernels.  The tile rectangle
    depends on mean2d only through floor(mean2d) (r is an integer), so the
    float64 means are passed as their exact integer floors: the device bins
    equal the reference's fp64 floor((m -/+ r) / 16) exactly."""
    n = len(projected)
    xydr = np.zeros((n, 4), np.float32)
    for i, p in enumerate(projected):
        xydr[i, 0], xydr[i, 1], xydr[i, 2] = np.floor(p.mean2d[0]), np.floor(p.mean2d[1]), p.depth
    rad = np.asarray([p.radius for p in projected], np.int32)
    xydr[:, 3] = rad.view(np.float32)
    return torch.as_tensor(xydr, device=dev), torch.as_tensor(rad, device=dev)


def assign_tiles(projected, width, height) -> TileGrid:
    """sg/binning.py:27-47 on the GPU: bins (unsorted = index order) of the
    tiles each closed bbox square touches."""
    dev = _device()
    cam = ops.CameraParams(np.eye(4).tolist(), 1.0, 1.0, 0.0, 0.0, int(width), int(height), 0.1, 1.0)
    n_tiles = cam.tiles_x * cam.tiles_y
    if not projected:
        return TileGrid(TILE_SIZE, cam.tiles_x, cam.tiles_y, [[] for _ in range(n_tiles)])
    xydr, rad = _proj_tensors(projected, dev)
    tiles = ops.tile_counts(xydr, cam)
    total = torch.zeros((1,), device=dev, dtype=torch.int64)
    offsets = ops.scan_tiles(tiles, total)
    # stable sort on the tile id only keeps the emission (= index) order per bin
    bins = ops.emit_and_sort(ops.Projection(xydr, xydr, tiles, None), offsets, int(total.item()), cam,
                             key_bits="tile")
    return _grid_from_bins(bins, cam, np.arange(len(projected)))


def sort_bins(grid: TileGrid, projected) -> TileGrid:
    """sg/binning.py:50-65 on the GPU: every bin stably sorted by
    (depth, source_index).  The fp64 depths are ranked exactly on the device
    (stable sort of their IEEE bits), so ties and order match the reference."""
    dev = _device()
    if not projected:
        return TileGrid(grid.tile_size, grid.tiles_x, grid.tiles_y, [list(b) for b in grid.bins])
    n = len(projected)
    order = sorted(range(n), key=lambda i: projected[i].source_index)  # secondary key: source_index
    rank = ops.depth_rank(np.asarray([projected[i].depth for i in order], np.float64), dev)
    rank_of = np.empty(n, np.int64)
    rank_of[np.asarray(order)] = rank
    sizes = [len(b) for b in grid.bins]
    flat = np.asarray([j for b in grid.bins for j in b], np.int64)
    tile_of = np.repeat(np.arange(len(grid.bins)), sizes)
    keys = (tile_of.astype(np.int64) << 32) | rank_of[flat]
    sorted_idx = ops.stable_sort_pairs(keys, flat, dev, end_bit=32 + ops.tile_bits(len(grid.bins)))
    out, pos = [], 0
    for sz in sizes:
        out.append(sorted_idx[pos:pos + sz].tolist())
        pos += sz
    return TileGrid(grid.tile_size, grid.tiles_x, grid.tiles_y, out)


# ------------------------------------------------------------------ per-pixel API

def _splat_arrays(projected, scene, dev):
    """Device splat records of `projected` (sg/raster_forward.py:95-113
    _pack_splats): xydr (m,4), conic (m,4) (A, B, C, opacity), colors (m,3),
    and the source indices."""
    m = len(projected)
    xydr = np.zeros((m, 4), np.float32)
    cov = np.zeros((m, 3), np.float32)
    opac = np.zeros(m, np.float32)
    colors = np.zeros((m, 3), np.float32)
    src = np.zeros(m, np.int64)
    for j, p in enumerate(projected):
        c = np.asarray(p.cov2d, np.float64)
        xydr[j, :2] = np.asarray(p.mean2d, np.float64)
        cov[j] = c[0, 0], c[0, 1], c[1, 1]
        if scene is not None:
            g = scene[p.source_index]
            opac[j], colors[j] = g.opacity, g.color
        src[j] = p.source_index
    t = lambda a: torch.as_tensor(a, device=dev)
    conic = pixels.conic_from_cov(t(cov), t(opac))
    return t(xydr), conic, t(colors), src


def eval_alpha(g, opacity, pixel_center):
    """sg/raster_forward.py:175-196 on the GPU: (alpha, delta, sigma)."""
    dev = _device()
    c = np.asarray(g.cov2d, np.float64)
    xydr = torch.as_tensor(np.array([[g.mean2d[0], g.mean2d[1], 0.0, 0.0]], np.float32), device=dev)
    conic = pixels.conic_from_cov(torch.as_tensor(np.array([[c[0, 0], c[0, 1], c[1, 1]]], np.float32), device=dev),
                                  torch.as_tensor(np.array([opacity], np.float32), device=dev))
    pix = torch.as_tensor(np.asarray(pixel_center, np.float64).reshape(1, 2).astype(np.float32), device=dev)
    alpha, delta, sigma = pixels.eval_alpha(xydr, conic, torch.zeros(1, dtype=torch.int32, device=dev), pix)
    return float(alpha.item()), _np(delta)[0].astype(np.float64), float(sigma.item())


def _one_query(sorted_bin, pixel_center, dev):
    idx = np.asarray(list(sorted_bin), np.int64)
    bin_ptr = torch.as_tensor(np.array([0, len(idx)], np.int64), device=dev)
    bin_idx = torch.as_tensor(idx.astype(np.int32), device=dev)
    pix = torch.as_tensor(np.asarray(pixel_center, np.float64).reshape(1, 2).astype(np.float32), device=dev)
    return bin_ptr, bin_idx, pix


def composite_pixel(sorted_bin, projected, scene, pixel_center, background, early_termination=True):
    """sg/raster_forward.py:199-219 on the GPU: (color 3-vector,
    PixelAux(final_T, n_contrib))."""
    dev = _device()
    xydr, conic, colors, _ = _splat_arrays(projected, scene, dev)
    bin_ptr, bin_idx, pix = _one_query(sorted_bin, pixel_center, dev)
    color, T, nc = pixels.composite_pixels(xydr, conic, colors, bin_ptr, bin_idx, pix,
                                           np.asarray(background, np.float64), early_termination)
    return _np(color)[0].astype(np.float64), PixelAux(float(T.item()), int(nc.item()))


def _pixel_backward(sorted_bin, projected, scene, pixel_center, background, aux_entry, d_pixel, want_t_log):
    dev = _device()
    xydr, conic, colors, src = _splat_arrays(projected, scene, dev)
    bin_ptr, bin_idx, pix = _one_query(sorted_bin, pixel_center, dev)
    fT = torch.as_tensor(np.array([aux_entry.final_T], np.float32), device=dev)
    nc = torch.as_tensor(np.array([aux_entry.n_contrib], np.int32), device=dev)
    d = torch.as_tensor(np.asarray(d_pixel, np.float64).reshape(1, 3).astype(np.float32), device=dev)
    return src, pixels.composite_pixels_backward(xydr, conic, colors, bin_ptr, bin_idx, pix,
                                                 np.asarray(background, np.float64), fT, nc, d,
                                                 want_t_log=want_t_log)


def composite_pixel_backward(sorted_bin, projected, scene, pixel_center, background, aux_entry,
                             d_pixel) -> Splat2DGrads:
    """sg/raster_backward.py:111-135 on the GPU: one row per scene Gaussian."""
    src, (d_rgbo, d_geo, d_c11, _) = _pixel_backward(sorted_bin, projected, scene, pixel_center, background,
                                                     aux_entry, d_pixel, False)
    rgbo, geo, c11 = (_np(x).astype(np.float64) for x in (d_rgbo, d_geo, d_c11))
    grads = Splat2DGrads.zeros(len(scene))
    np.add.at(grads.d_color, src, rgbo[:, :3])
    np.add.at(grads.d_opacity, src, rgbo[:, 3])
    np.add.at(grads.d_mean2d, src, geo[:, :2])
    cov = np.stack([geo[:, 2], geo[:, 3], geo[:, 3], c11], axis=1).reshape(-1, 2, 2)
    np.add.at(grads.d_cov2d, src, cov)
    return grads


def transmittance_replay(sorted_bin, projected, scene, pixel_center, background, aux_entry):
    """sg/raster_backward.py:138-163 on the GPU: (bin position, T) pairs in
    back-to-front order, one per splat that contributed in the forward."""
    _, (_, _, _, t_log) = _pixel_backward(sorted_bin, projected, scene, pixel_center, background, aux_entry,
                                          np.zeros(3), True)
    t = _np(t_log).astype(np.float64)
    return [(pos, float(t[pos])) for pos in range(len(t) - 1, -1, -1) if np.isfinite(t[pos])]
