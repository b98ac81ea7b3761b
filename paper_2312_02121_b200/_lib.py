"""ctypes binding of libsplat_b200.so (the C ABI in include/splat_b200.h).

There is no fallback: if the shared library is missing or cannot be loaded
the import of the ops fails loudly with instructions to build it.
"""

from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsplat_b200.so")
# A/B builds of one kernel variant (tools/build_variant.py) load through this
LIB_PATH = os.environ.get("GS_LIB_PATH") or LIB_PATH

# Every symbol include/splat_b200.h declares (tests check the export table).
EXPORTS = (
    "gs_last_error", "gs_version", "gs_device_sm_count", "gs_set_option", "gs_get_option",
    "gs_project_fwd",
    "gs_scan_workspace_bytes", "gs_scan_tiles", "gs_emit_keys",
    "gs_sort_workspace_bytes", "gs_sort_pairs", "gs_tile_counts", "gs_tile_ranges",
    "gs_raster_fwd", "gs_raster_bwd",
    "gs_project_bwd_workspace_bytes", "gs_project_bwd",
    "gs_frame_workspace_bytes", "gs_frame_workspace_init", "gs_frame_binning", "gs_frame_tile_emit", "gs_frame_view_of",
    "gs_frame_forward", "gs_frame_forward_projected", "gs_frames_project", "gs_frame_backward", "gs_frame_project_backward", "gs_frame_views_project_backward",
    "gs_activate", "gs_loss_l2", "gs_adam_step",
    "gs_conic_from_cov", "gs_eval_alpha", "gs_composite_pixels", "gs_composite_pixels_bwd",
    "gs_project64", "gs_bin64_workspace_bytes", "gs_bin64_count", "gs_bin64_sort", "gs_raster64_fwd",
    "gs_raster64_bwd", "gs_project64_bwd_workspace_bytes", "gs_project64_bwd", "gs_op64",
)

ERR_MESSAGES = {  # include/splat_b200.h gs_error_code -> the reference's ValueError text
    1: "scale components must be positive",                      # sg/core.py:189-191
    2: "quaternion norm is too small to define an orientation",  # sg/core.py:160-163
    3: "degenerate projection: homogeneous component is ~0",     # sg/projection.py:54-55
    4: "2d covariance must be positive definite",                # sg/projection.py:108-109
    5: "point is behind the camera",                             # sg/projection.py:75-76
}


class GsCamera(C.Structure):
    _fields_ = [("view", C.c_float * 16), ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float),
                ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("near_plane", C.c_float), ("far_plane", C.c_float)]


class GsCamera64(C.Structure):
    _fields_ = [("view", C.c_double * 16), ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double),
                ("cy", C.c_double), ("width", C.c_int32), ("height", C.c_int32),
                ("near_plane", C.c_double), ("far_plane", C.c_double)]


class GsFrameView(C.Structure):
    _fields_ = [(name, C.c_void_p) for name in (
        "xydr4", "conic4", "tiles", "depth_order", "sorted_tile_keys", "sorted_vals", "ranges2", "meta",
        "d_geo4", "d_c11", "bwd_accum")] + [("bwd_accum_bytes", C.c_size_t), ("rec_count", C.c_void_p),
                                                       ("depth_order_alt", C.c_void_p),
                                                       ("touched", C.c_void_p)]


class SplatLibError(RuntimeError):
    pass


_lib = None


def load():
    """Load and type the library (raises if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SplatLibError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2312_02121_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P, i64, i32, sz = C.c_void_p, C.c_int64, C.c_int32, C.c_size_t
    cam = C.POINTER(GsCamera)
    sig = {
        "gs_last_error": ([], C.c_char_p),
        "gs_version": ([], C.c_int),
        "gs_device_sm_count": ([], C.c_int),
        "gs_project_fwd": ([P, P, P, P, i64, cam, P, P, P, P, P, P], C.c_int),
        "gs_scan_workspace_bytes": ([i64], sz),
        "gs_scan_tiles": ([P, P, i64, P, sz, P, P], C.c_int),
        "gs_emit_keys": ([P, P, P, i64, i32, i32, P, P, P], C.c_int),
        "gs_sort_workspace_bytes": ([i64, C.c_int], sz),
        "gs_sort_pairs": ([P, P, P, P, i64, C.c_int, P, sz, C.POINTER(C.c_int), P], C.c_int),
        "gs_tile_counts": ([P, i64, i32, i32, P, P], C.c_int),
        "gs_tile_ranges": ([P, i64, P, i32, P], C.c_int),
        "gs_raster_fwd": ([P, P, P, P, P, C.POINTER(C.c_float), i32, i32, C.c_int, P, P, P, P, P], C.c_int),
        "gs_raster_bwd": ([P, P, P, P, P, C.POINTER(C.c_float), i32, i32, P, P, P, P, P, P, P, P], C.c_int),
        "gs_project_bwd_workspace_bytes": ([i64], sz),
        "gs_project_bwd": ([P, P, P, i64, cam, P, P, P, P, P, P, P, P, sz, P], C.c_int),
        "gs_frame_workspace_bytes": ([i64, i64, i32, i32], sz),
        "gs_frame_binning": ([i64, i32, i32], C.c_int),
        "gs_frame_tile_emit": ([i64, i32, i32], C.c_int),
        "gs_frame_view_of": ([i64, i64, i32, i32, P, C.POINTER(GsFrameView)], C.c_int),
        "gs_frame_workspace_init": ([i64, i64, i32, i32, P, P], C.c_int),
        "gs_frame_forward": ([P, P, P, P, P, i64, cam, C.POINTER(C.c_float), C.c_int, i64, P, sz, P, P, P, P, P,
                              P], C.c_int),
        "gs_frame_backward": ([P, P, P, P, i64, cam, C.POINTER(C.c_float), i64, P, sz, P, P, P, P, P, P, P, P,
                               C.c_int, P, P, P], C.c_int),
        "gs_frame_project_backward": ([P, P, P, i64, cam, i64, P, sz, i64, i64, P, P, P, P, P, C.c_int, P], C.c_int),
        "gs_frame_forward_projected": ([P, P, P, P, P, i64, cam, C.POINTER(C.c_float), C.c_int, i64, P, sz, P, P, P,
                                        P, P], C.c_int),
        "gs_frames_project": ([P, P, P, P, i64, i32, cam, P, P, P, P], C.c_int),
        "gs_frame_views_project_backward": ([P, P, P, i64, i32, cam, P, P, P, i64, i64, P, P, P, P, P, C.c_int, P],
                                            C.c_int),
    }
    f32 = C.c_float
    sig.update({
        "gs_activate": ([P, P, P, P, i64, P], C.c_int),
        "gs_loss_l2": ([P, P, i64, P, P, P], C.c_int),
        "gs_adam_step": ([P, P, P, P, P, P, P, P, P, P, P, P, P, i64, C.c_int, C.POINTER(f32), f32, f32, f32, P],
                         C.c_int),
        "gs_conic_from_cov": ([P, P, i64, P, P, P], C.c_int),
        "gs_eval_alpha": ([P, P, P, P, i64, P, P, P, P], C.c_int),
        "gs_composite_pixels": ([P, P, P, P, P, P, i64, C.POINTER(f32), C.c_int, P, P, P, P], C.c_int),
        "gs_composite_pixels_bwd": ([P, P, P, P, P, P, i64, C.POINTER(f32), P, P, P, P, P, P, P, P], C.c_int),
    })
    cam64 = C.POINTER(GsCamera64)
    f64p = C.POINTER(C.c_double)
    sig.update({
        "gs_project64": ([P, P, P, i64, cam64, P, P, P, P, P, P, P, P], C.c_int),
        "gs_set_option": ([C.c_char_p, C.c_int], C.c_int),
        "gs_get_option": ([C.c_char_p], C.c_int),
        "gs_bin64_workspace_bytes": ([i64, i64, C.c_int32], C.c_size_t),
        "gs_bin64_count": ([P, i64, P, C.c_size_t, P, P], C.c_int),
        "gs_bin64_sort": ([P, P, P, P, i64, i64, C.c_int32, C.c_int32, P, C.c_size_t, P,
                           C.POINTER(C.c_void_p), P], C.c_int),
        "gs_raster64_fwd": ([P, P, P, P, P, P, f64p, C.c_int32, C.c_int32, C.c_int, P, P, P, P], C.c_int),
        "gs_raster64_bwd": ([P, P, P, P, P, P, f64p, C.c_int32, C.c_int32, P, P, P, P, P], C.c_int),
        "gs_project64_bwd_workspace_bytes": ([i64], C.c_size_t),
        "gs_project64_bwd": ([P, P, P, i64, cam64, P, P, P, P, P, P, P, C.c_size_t, P], C.c_int),
        "gs_op64": ([C.c_int, i64, P, P, C.c_int32, cam64, P, P], C.c_int),
    })
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = load().gs_last_error().decode(errors="replace")
        raise SplatLibError(f"{what}: {msg}" if what else msg)


def make_camera64(view, fx, fy, cx, cy, width, height, near, far) -> GsCamera64:
    c = GsCamera64()
    flat = [float(v) for row in view for v in row] if hasattr(view[0], "__len__") else [float(v) for v in view]
    if len(flat) != 16:
        raise ValueError("view must have shape (4, 4)")
    for k in range(16):
        c.view[k] = flat[k]
    c.fx, c.fy, c.cx, c.cy = float(fx), float(fy), float(cx), float(cy)
    c.width, c.height = int(width), int(height)
    c.near_plane, c.far_plane = float(near), float(far)
    return c


def make_camera(view, fx, fy, cx, cy, width, height, near, far) -> GsCamera:
    c = GsCamera()
    flat = [float(v) for row in view for v in row] if hasattr(view[0], "__len__") else [float(v) for v in view]
    if len(flat) != 16:
        raise ValueError("view must have shape (4, 4)")
    for k in range(16):
        c.view[k] = flat[k]
    c.fx, c.fy, c.cx, c.cy = float(fx), float(fy), float(cx), float(cy)
    c.width, c.height = int(width), int(height)
    c.near_plane, c.far_plane = float(near), float(far)
    return c
