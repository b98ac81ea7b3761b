"""fp64 CPU oracle for the splatting hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and
only as the checker or the timed CPU baseline -- never as the product path.

It wraps ``oracle/splat_oracle.c`` (a plain-C, float64 restatement of
``/root/reference/pkg/src/splatgrad``; every C function cites the reference
file:line it follows) through ctypes.  The C library is pinned against golden
vectors produced by the real reference (``tests/golden/make_golden.py``).

Array conventions: inputs are float64 numpy arrays indexed by *scene*
Gaussian; bins are CSR (``bin_ptr[tiles+1]``, ``bin_idx[I]``) over scene
indices, in sorted (depth, index) order.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libsplat_oracle.so")
TILE = 16
ERR_MESSAGES = {
    1: "scale components must be positive",                       # sg/core.py:189-191
    2: "quaternion norm is too small to define an orientation",   # sg/core.py:160-163
    3: "degenerate projection: homogeneous component is ~0",      # sg/projection.py:54-55
    4: "2d covariance must be positive definite",                 # sg/projection.py:108-109
}

_lib = None


class _Cam(C.Structure):
    _fields_ = [("view", C.c_double * 16), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("width", C.c_int64),
                ("height", C.c_int64), ("near_plane", C.c_double), ("far_plane", C.c_double)]


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc -fopenmp)."""
    if force or not os.path.exists(LIB_PATH) or (
            os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "splat_oracle.c"))):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        i64 = C.c_int64
        L.orc_project.argtypes = [i64, P, P, P, P, P, P, P, P, P, P, P, C.c_int]
        L.orc_project.restype = C.c_int
        L.orc_bin_count.argtypes = [i64, P, P, P, i64, i64, P]
        L.orc_bin_count.restype = i64
        L.orc_bin_fill.argtypes = [i64, P, P, P, P, i64, i64, P, P, P, C.c_int]
        L.orc_bin_fill.restype = None
        L.orc_raster_fwd.argtypes = [i64, i64, P, P, P, P, P, P, P, C.c_int, P, P, P, P, P, P, P, C.c_int]
        L.orc_raster_fwd.restype = None
        L.orc_raster_bwd.argtypes = [i64, i64, P, P, P, P, P, P, P, P, P, P, i64, P, P, P, P, P, C.c_int]
        L.orc_raster_bwd.restype = None
        L.orc_project_bwd.argtypes = [i64, P, P, P, P, P, P, P, P, P, P, P, P, C.c_int]
        L.orc_project_bwd.restype = C.c_int
        L.orc_eval_alpha.argtypes = [i64, P, P, P, P, P, P]
        L.orc_eval_alpha.restype = None
        L.orc_composite_pixels.argtypes = [i64, P, P, P, P, P, P, P, P, P, P, P, P, P, P]
        L.orc_composite_pixels.restype = None
        L.orc_composite_pixels_bwd.argtypes = [i64, P, P, P, P, P, P, P, P, P, P, P, P, P]
        L.orc_composite_pixels_bwd.restype = None
        L.orc_max_threads.argtypes = []
        L.orc_max_threads.restype = C.c_int
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().orc_max_threads())


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _d(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


@dataclass
class Camera:
    """Same fields as the reference Camera (sg/core.py:59-129)."""

    view: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float
    far: float

    def c(self) -> _Cam:
        cam = _Cam()
        v = _d(self.view).reshape(16)
        for k in range(16):
            cam.view[k] = float(v[k])
        cam.fx, cam.fy, cam.cx, cam.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        cam.width, cam.height = int(self.width), int(self.height)
        cam.near_plane, cam.far_plane = float(self.near), float(self.far)
        return cam

    @staticmethod
    def of(spec) -> "Camera":
        return Camera(view=np.asarray(spec.view, np.float64), fx=spec.fx, fy=spec.fy, cx=spec.cx,
                      cy=spec.cy, width=spec.width, height=spec.height, near=spec.near, far=spec.far)


def tiles_xy(width: int, height: int):
    return (width + TILE - 1) // TILE, (height + TILE - 1) // TILE


def project(means, scales, quats, cam: Camera, nthreads: int = 0) -> dict:
    """sg/projection.py:115-145 for every Gaussian; raises ValueError like
    the reference at the first offending (non depth-culled) Gaussian."""
    means, scales, quats = _d(means, (-1, 3)), _d(scales, (-1, 3)), _d(quats, (-1, 4))
    n = means.shape[0]
    out = dict(visible=np.zeros(n, np.int8), t_cam=np.zeros((n, 4)), mean2d=np.zeros((n, 2)),
               cov2d=np.zeros((n, 3)), depth=np.zeros(n), radius=np.zeros(n, np.int64))
    err_idx = np.zeros(1, np.int64)
    camc = cam.c()
    code = lib().orc_project(n, _p(means), _p(scales), _p(quats), C.byref(camc), _p(out["visible"]),
                             _p(out["t_cam"]), _p(out["mean2d"]), _p(out["cov2d"]), _p(out["depth"]),
                             _p(out["radius"]), _p(err_idx), nthreads)
    if code:
        raise ValueError(f"gaussian {int(err_idx[0])}: {ERR_MESSAGES[code]}")
    return out


def bin_tiles(visible, mean2d, radius, depth, width, height, sort=True):
    """sg/binning.py:27-65 -> CSR (bin_ptr, bin_idx) over scene indices."""
    visible = np.ascontiguousarray(visible, dtype=np.int8)
    mean2d = _d(mean2d, (-1, 2))
    radius = np.ascontiguousarray(radius, dtype=np.int64)
    depth = _d(depth)
    n = visible.shape[0]
    tx, ty = tiles_xy(width, height)
    count = np.zeros(tx * ty, np.int64)
    total = lib().orc_bin_count(n, _p(visible), _p(mean2d), _p(radius), width, height, _p(count))
    ptr = np.zeros(tx * ty + 1, np.int64)
    idx = np.zeros(max(total, 1), np.int64)
    lib().orc_bin_fill(n, _p(visible), _p(mean2d), _p(radius), _p(depth), width, height, _p(count),
                       _p(ptr), _p(idx), 1 if sort else 0)
    return ptr, idx[:total]


def raster_fwd(width, height, bin_ptr, bin_idx, mean2d, cov2d, opac, colors, bg,
               early_termination=True, margins=False, nthreads: int = 0) -> dict:
    """sg/raster_forward.py:116-172,222-243 over all tiles."""
    bin_ptr = np.ascontiguousarray(bin_ptr, np.int64)
    bin_idx = np.ascontiguousarray(bin_idx, np.int64)
    mean2d, cov2d = _d(mean2d, (-1, 2)), _d(cov2d, (-1, 3))
    opac, colors, bg = _d(opac), _d(colors, (-1, 3)), _d(bg)
    out = dict(image=np.zeros((height, width, 3)), final_T=np.zeros((height, width)),
               n_contrib=np.zeros((height, width), np.int64), counts=np.zeros(4, np.int64))
    null = C.c_void_p(0)
    if margins:
        out["margin"] = np.zeros((height, width))
        out["margin_pos"] = np.zeros((height, width), np.int64)
        out["margin_kind"] = np.zeros((height, width), np.int8)
    lib().orc_raster_fwd(width, height, _p(bin_ptr), _p(bin_idx), _p(mean2d), _p(cov2d), _p(opac),
                         _p(colors), _p(bg), 1 if early_termination else 0, _p(out["image"]),
                         _p(out["final_T"]), _p(out["n_contrib"]),
                         _p(out["margin"]) if margins else null,
                         _p(out["margin_pos"]) if margins else null,
                         _p(out["margin_kind"]) if margins else null,
                         _p(out["counts"]), nthreads)
    return out


def raster_bwd(width, height, bin_ptr, bin_idx, mean2d, cov2d, opac, colors, bg, final_T,
               n_contrib, d_image, nthreads: int = 0) -> dict:
    """sg/raster_backward.py:47-108,166-205 -> Splat2DGrads per scene Gaussian."""
    bin_ptr = np.ascontiguousarray(bin_ptr, np.int64)
    bin_idx = np.ascontiguousarray(bin_idx, np.int64)
    mean2d, cov2d = _d(mean2d, (-1, 2)), _d(cov2d, (-1, 3))
    opac, colors, bg = _d(opac), _d(colors, (-1, 3)), _d(bg)
    final_T = _d(final_T)
    n_contrib = np.ascontiguousarray(n_contrib, np.int64)
    d_image = _d(d_image)
    n = mean2d.shape[0]
    out = dict(d_color=np.zeros((n, 3)), d_opacity=np.zeros(n), d_mean2d=np.zeros((n, 2)),
               d_cov2d=np.zeros((n, 2, 2)), counts=np.zeros(3, np.int64))
    lib().orc_raster_bwd(width, height, _p(bin_ptr), _p(bin_idx), _p(mean2d), _p(cov2d), _p(opac),
                         _p(colors), _p(bg), _p(final_T), _p(n_contrib), _p(d_image), n,
                         _p(out["d_color"]), _p(out["d_opacity"]), _p(out["d_mean2d"]),
                         _p(out["d_cov2d"]), _p(out["counts"]), nthreads)
    return out


def project_bwd(means, scales, quats, cam: Camera, visible, t_cam, d_mean2d, d_cov2d,
                nthreads: int = 0) -> dict:
    """sg/proj_backward.py:178-223 per visible Gaussian (loop body :200-222)."""
    means, scales, quats = _d(means, (-1, 3)), _d(scales, (-1, 3)), _d(quats, (-1, 4))
    visible = np.ascontiguousarray(visible, np.int8)
    t_cam = _d(t_cam, (-1, 4))
    d_mean2d, d_cov2d = _d(d_mean2d, (-1, 2)), _d(d_cov2d, (-1, 4))
    n = means.shape[0]
    out = dict(d_mean=np.zeros((n, 3)), d_scale=np.zeros((n, 3)), d_quat=np.zeros((n, 4)),
               d_view=np.zeros((4, 4)))
    camc = cam.c()
    lib().orc_project_bwd(n, _p(means), _p(scales), _p(quats), C.byref(camc), _p(visible), _p(t_cam),
                          _p(d_mean2d), _p(d_cov2d), _p(out["d_mean"]), _p(out["d_scale"]),
                          _p(out["d_quat"]), _p(out["d_view"]), nthreads)
    return out


def render(means, scales, quats, opacities, colors, cam: Camera, background,
           early_termination=True, margins=False, nthreads: int = 0) -> dict:
    """sg/raster_forward.py:255-271 render (project -> bin -> sort -> composite)."""
    pr = project(means, scales, quats, cam, nthreads)
    ptr, idx = bin_tiles(pr["visible"], pr["mean2d"], pr["radius"], pr["depth"], cam.width, cam.height)
    fw = raster_fwd(cam.width, cam.height, ptr, idx, pr["mean2d"], pr["cov2d"], opacities, colors,
                    background, early_termination, margins, nthreads)
    fw.update(pr)
    fw["bin_ptr"], fw["bin_idx"] = ptr, idx
    return fw


def scene_backward(means, scales, quats, opacities, colors, cam: Camera, background, fwd: dict,
                   d_image, nthreads: int = 0) -> dict:
    """sg/proj_backward.py:178-223 scene_backward on a render() result."""
    rb = raster_bwd(cam.width, cam.height, fwd["bin_ptr"], fwd["bin_idx"], fwd["mean2d"], fwd["cov2d"],
                    opacities, colors, background, fwd["final_T"], fwd["n_contrib"], d_image, nthreads)
    pb = project_bwd(means, scales, quats, cam, fwd["visible"], fwd["t_cam"], rb["d_mean2d"],
                     rb["d_cov2d"].reshape(-1, 4), nthreads)
    return dict(d_mean=pb["d_mean"], d_scale=pb["d_scale"], d_quat=pb["d_quat"],
                d_opacity=rb["d_opacity"], d_color=rb["d_color"], d_view=pb["d_view"],
                d_mean2d=rb["d_mean2d"], d_cov2d=rb["d_cov2d"], counts=rb["counts"])


# ------------------------------------------------------------------ per-pixel API

def eval_alpha(splat, pix, mean2d, cov2d, opac) -> np.ndarray:
    """sg/raster_forward.py:175-196 for q pairs -> (q,4) alpha, dx, dy, sigma."""
    splat = np.ascontiguousarray(splat, np.int64)
    pix, mean2d, cov2d, opac = _d(pix, (-1, 2)), _d(mean2d, (-1, 2)), _d(cov2d, (-1, 3)), _d(opac)
    out = np.zeros((len(splat), 4))
    lib().orc_eval_alpha(len(splat), _p(splat), _p(pix), _p(mean2d), _p(cov2d), _p(opac), _p(out))
    return out


def composite_pixels(bin_ptr, bin_idx, pix, et, mean2d, cov2d, opac, colors, bg) -> dict:
    """sg/raster_forward.py:199-219 for q queries (own bin + et flag each)."""
    bin_ptr = np.ascontiguousarray(bin_ptr, np.int64)
    bin_idx = np.ascontiguousarray(bin_idx, np.int64)
    q = len(bin_ptr) - 1
    et = np.ascontiguousarray(np.broadcast_to(np.asarray(et, np.int8), (q,)))
    pix, mean2d, cov2d = _d(pix, (-1, 2)), _d(mean2d, (-1, 2)), _d(cov2d, (-1, 3))
    opac, colors, bg = _d(opac), _d(colors, (-1, 3)), _d(bg)
    out = dict(color=np.zeros((q, 3)), final_T=np.zeros(q), n_contrib=np.zeros(q, np.int64), margin=np.zeros(q),
               margin_kind=np.zeros(q, np.int8))
    lib().orc_composite_pixels(q, _p(bin_ptr), _p(bin_idx), _p(pix), _p(et), _p(mean2d), _p(cov2d), _p(opac),
                               _p(colors), _p(bg), _p(out["color"]), _p(out["final_T"]), _p(out["n_contrib"]),
                               _p(out["margin"]), _p(out["margin_kind"]))
    return out


def composite_pixels_bwd(bin_ptr, bin_idx, pix, mean2d, cov2d, opac, colors, bg, final_T, n_contrib, d_pix,
                         t_log=False) -> dict:
    """sg/raster_backward.py:111-163 for q queries -> per-splat d9 rows
    (d_color 3, d_opacity, d_mean2d 2, d_cov 00, 01, 11) and the replay log."""
    bin_ptr = np.ascontiguousarray(bin_ptr, np.int64)
    bin_idx = np.ascontiguousarray(bin_idx, np.int64)
    q = len(bin_ptr) - 1
    pix, mean2d, cov2d = _d(pix, (-1, 2)), _d(mean2d, (-1, 2)), _d(cov2d, (-1, 3))
    opac, colors, bg, final_T, d_pix = _d(opac), _d(colors, (-1, 3)), _d(bg), _d(final_T), _d(d_pix, (-1, 3))
    n_contrib = np.ascontiguousarray(n_contrib, np.int64)
    d9 = np.zeros((mean2d.shape[0], 9))
    log = np.zeros(len(bin_idx)) if t_log else None
    lib().orc_composite_pixels_bwd(q, _p(bin_ptr), _p(bin_idx), _p(pix), _p(mean2d), _p(cov2d), _p(opac),
                                   _p(colors), _p(bg), _p(final_T), _p(n_contrib), _p(d_pix), _p(d9),
                                   _p(log) if t_log else C.c_void_p(0))
    return dict(d9=d9, t_log=log)
