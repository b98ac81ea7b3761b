"""The path in float64 on the device: csrc/f64.cu.

render64 / backward64 are the fp64 counterparts of ops.render_forward /
ops.render_backward (same stages: projection, (depth, index) binning,
compositing, compositing backward, projection backward) with the reference's
fp64 arithmetic, for the finite-difference audit (gradcheck.py) and fp64
parity.  One host sync per frame (the intersection total sizes the buffers).
Inputs are float64 CUDA tensors; there is no CPU path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib, ops
from ._lib import check

TILE = 16


def _d(t, name, cols):
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise ValueError(f"{name} must be a float64 CUDA tensor (there is no CPU path)")
    if (cols is None and t.dim() != 1) or (cols is not None and (t.dim() != 2 or t.shape[1] != cols)):
        raise ValueError(f"{name} has shape {tuple(t.shape)}")
    return t.contiguous()


def camera64(cam) -> _lib.GsCamera64:
    c = cam if isinstance(cam, ops.CameraParams) else ops.CameraParams.of(cam)
    return _lib.make_camera64(c.view, c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.near, c.far)


@dataclass
class Frame64:
    cam: ops.CameraParams
    background: tuple
    early_termination: bool
    n: int
    mean2d: torch.Tensor     # (n, 2), rows of depth-culled / erroring Gaussians are 0
    cov3: torch.Tensor       # (n, 3) (a, b, c) of the dilated 2d covariance
    depth: torch.Tensor      # (n,)
    radius: torch.Tensor     # (n,) int32
    tiles: torch.Tensor      # (n,) uint32 as int32, 0 = culled
    ranges: torch.Tensor     # (n_tiles, 2) int32
    vals: torch.Tensor       # (n_isect,) int32 Gaussian ids, per tile in (depth, index) order
    n_isect: int
    image: torch.Tensor      # (H, W, 3)
    final_T: torch.Tensor
    n_contrib: torch.Tensor
    ws: torch.Tensor

    def bins(self):
        """Per-tile lists of scene indices (host)."""
        r = self.ranges.cpu().tolist()
        v = self.vals.cpu().tolist()
        return [v[a:b] for a, b in r]


def render64(means, scales, quats, opacities, colors, cam, background=(0.0, 0.0, 0.0),
             early_termination=True) -> Frame64:
    L = _lib.load()
    means, scales, quats = _d(means, "means", 3), _d(scales, "scales", 3), _d(quats, "quats", 4)
    opacities, colors = _d(opacities, "opacities", None), _d(colors, "colors", 3)
    cp = cam if isinstance(cam, ops.CameraParams) else ops.CameraParams.of(cam)
    n = means.shape[0]
    dev = means.device
    st = ops._stream()
    c64 = camera64(cp)
    f = lambda *s: torch.zeros(s, device=dev, dtype=torch.float64)
    mean2d, cov3, depth = f(n, 2), f(n, 3), f(n)
    radius = torch.zeros(n, device=dev, dtype=torch.int32)
    tiles = torch.zeros(n, device=dev, dtype=torch.int32)
    dkeys = torch.zeros(n, device=dev, dtype=torch.int64)
    status = torch.full((1,), -1, device=dev, dtype=torch.int64)
    check(L.gs_project64(means.data_ptr(), scales.data_ptr(), quats.data_ptr(), n, C.byref(c64), mean2d.data_ptr(),
                         cov3.data_ptr(), depth.data_ptr(), radius.data_ptr(), tiles.data_ptr(), dkeys.data_ptr(),
                         status.data_ptr(), st), "gs_project64")
    n_tiles = cp.tiles_x * cp.tiles_y
    total = torch.zeros(1, device=dev, dtype=torch.int64)
    ws0 = torch.empty(L.gs_bin64_workspace_bytes(n, 0, n_tiles), device=dev, dtype=torch.uint8)
    check(L.gs_bin64_count(tiles.data_ptr(), n, ws0.data_ptr(), ws0.numel(), total.data_ptr(), st), "gs_bin64_count")
    ops.raise_status(int(status.item()))
    n_isect = int(total.item())
    ws = torch.zeros(L.gs_bin64_workspace_bytes(n, n_isect, n_tiles), device=dev, dtype=torch.uint8)
    ws[:ws0.numel()].copy_(ws0)  # the scan's offsets live in the shared prefix
    ranges = torch.zeros((n_tiles, 2), device=dev, dtype=torch.int32)
    vals_ptr = C.c_void_p()
    check(L.gs_bin64_sort(mean2d.data_ptr(), radius.data_ptr(), tiles.data_ptr(), dkeys.data_ptr(), n, n_isect,
                          cp.width, cp.height, ws.data_ptr(), ws.numel(), ranges.data_ptr(), C.byref(vals_ptr), st),
          "gs_bin64_sort")
    off = (vals_ptr.value or ws.data_ptr()) - ws.data_ptr()
    vals = ws[off:off + 4 * n_isect].view(torch.int32)
    H, W = cp.height, cp.width
    image, final_T = f(H, W, 3), f(H, W)
    n_contrib = torch.zeros((H, W), device=dev, dtype=torch.int32)
    bg = (C.c_double * 3)(*[float(b) for b in background])
    check(L.gs_raster64_fwd(ranges.data_ptr(), vals.data_ptr() if n_isect else None, mean2d.data_ptr(),
                            cov3.data_ptr(), opacities.data_ptr(), colors.data_ptr(), bg, W, H,
                            1 if early_termination else 0, image.data_ptr(), final_T.data_ptr(),
                            n_contrib.data_ptr(), st), "gs_raster64_fwd")
    return Frame64(cp, tuple(float(b) for b in background), bool(early_termination), n, mean2d, cov3, depth, radius,
                   tiles, ranges, vals, n_isect, image, final_T, n_contrib, ws)


def backward64(fr: Frame64, means, scales, quats, opacities, colors, d_image) -> dict:
    """Screen-space (d9) and scene gradients in float64 (SceneGradients
    fields, sg/proj_backward.py:25-50)."""
    L = _lib.load()
    H, W = fr.cam.height, fr.cam.width
    if tuple(d_image.shape) != (H, W, 3):
        raise ValueError(f"d_image must have shape {(H, W, 3)}, got {tuple(d_image.shape)}")
    d_image = _d(d_image.reshape(-1, 3), "d_image", 3)
    means, scales, quats = _d(means, "means", 3), _d(scales, "scales", 3), _d(quats, "quats", 4)
    opacities, colors = _d(opacities, "opacities", None), _d(colors, "colors", 3)
    n = fr.n
    dev = means.device
    st = ops._stream()
    d9 = torch.zeros((n, 9), device=dev, dtype=torch.float64)
    bg = (C.c_double * 3)(*fr.background)
    check(L.gs_raster64_bwd(fr.ranges.data_ptr(), fr.vals.data_ptr() if fr.n_isect else None, fr.mean2d.data_ptr(),
                            fr.cov3.data_ptr(), opacities.data_ptr(), colors.data_ptr(), bg, W, H,
                            fr.final_T.data_ptr(), fr.n_contrib.data_ptr(), d_image.data_ptr(), d9.data_ptr(), st),
          "gs_raster64_bwd")
    f = lambda *s: torch.zeros(s, device=dev, dtype=torch.float64)
    d_means, d_scales, d_quats, d_view = f(n, 3), f(n, 3), f(n, 4), f(4, 4)
    pws = torch.empty(L.gs_project64_bwd_workspace_bytes(n), device=dev, dtype=torch.uint8)
    c64 = camera64(fr.cam)
    check(L.gs_project64_bwd(means.data_ptr(), scales.data_ptr(), quats.data_ptr(), n, C.byref(c64),
                             fr.tiles.data_ptr(), d9.data_ptr(), d_means.data_ptr(), d_scales.data_ptr(),
                             d_quats.data_ptr(), d_view.data_ptr(), pws.data_ptr(), pws.numel(), st),
          "gs_project64_bwd")
    return dict(d_mean=d_means, d_scale=d_scales, d_quat=d_quats, d_opacity=d9[:, 3], d_color=d9[:, :3],
                d_view=d_view, d_mean2d=d9[:, 4:6],
                d_cov2d=torch.stack([d9[:, 6], d9[:, 7], d9[:, 7], d9[:, 8]], 1).reshape(n, 2, 2), d9=d9)
