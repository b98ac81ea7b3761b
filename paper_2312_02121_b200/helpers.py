"""The reference's per-splat helper functions (the scalar building blocks
the fused kernels inline), each run on the device in float64 through
gs_op64 (csrc/ops64.cu) -- the remaining names of sg/__init__.py:64-119:

  quat_to_rotmat, compose_covariance_3d, Cov3DBundle, frobenius_inner   sg/core.py:132-204
  world_to_camera, camera_to_pixel, projection_jacobian,
  project_covariance, bounding_radius                                   sg/projection.py:36-112
  mean2d_backward, cov2d_backward, world_backward,
  covariance3d_backward                                                 sg/proj_backward.py:53-175

Same signatures, argument meaning, return types and ValueError messages as
the reference; inputs are numpy-convertible, results float64 numpy.  Each
call is a batch of one on the GPU (there is no CPU path).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

OP_QUAT_TO_ROTMAT, OP_COMPOSE_COV3D, OP_FROBENIUS, OP_WORLD_TO_CAMERA, OP_CAMERA_TO_PIXEL = 1, 2, 3, 4, 5
OP_PROJECTION_JACOBIAN, OP_PROJECT_COVARIANCE, OP_BOUNDING_RADIUS, OP_MEAN2D_BACKWARD = 6, 7, 8, 9
OP_COV2D_BACKWARD, OP_WORLD_BACKWARD, OP_COV3D_BACKWARD = 10, 11, 12


@dataclass
class Cov3DBundle:
    """sg/core.py:132-143: R, S (diag scale), M = R S and sigma = M M^T."""

    R: np.ndarray
    S: np.ndarray
    M: np.ndarray
    sigma: np.ndarray


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2312_02121_b200.helpers needs a CUDA device (there is no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def _f64(a, shape=None):
    arr = np.asarray(a, dtype=np.float64)
    if shape is not None:
        arr = arr.reshape(shape)
    return arr


def _cam64(camera):
    if camera is None:
        return None
    v = np.asarray(camera.view, np.float64)
    return _lib.make_camera64(v.tolist(), camera.fx, camera.fy, camera.cx, camera.cy, camera.width, camera.height,
                              camera.near, camera.far)


def _run(op, inputs, out_sizes, camera=None, cols=0):
    """One gs_op64 call over a batch of one; returns the outputs (float64
    numpy, flat) or raises the reference's ValueError."""
    dev = _device()
    ins = [torch.as_tensor(np.ascontiguousarray(_f64(x).reshape(-1)), device=dev) for x in inputs]
    outs = [torch.zeros(k, device=dev, dtype=torch.float64) for k in out_sizes]
    status = torch.full((1,), -1, device=dev, dtype=torch.int64)
    in_arr = (C.c_void_p * max(1, len(ins)))(*[t.data_ptr() for t in ins])
    out_arr = (C.c_void_p * len(outs))(*[t.data_ptr() for t in outs])
    cam = _cam64(camera)
    _lib.check(_lib.load().gs_op64(op, 1, in_arr, out_arr, int(cols), C.byref(cam) if cam is not None else None,
                                   status.data_ptr(), torch.cuda.current_stream(dev).cuda_stream), "gs_op64")
    s = int(status.item())
    if s != -1:
        raise ValueError(_lib.ERR_MESSAGES.get(s & 0xFF, "degenerate input"))
    return [o.cpu().numpy() for o in outs]


# ---------------------------------------------------------------- sg/core.py

def quat_to_rotmat(quat):
    """sg/core.py:146-171: rotation matrix of a (w, x, y, z) quaternion
    (normalised first)."""
    q = np.asarray(quat, dtype=np.float64)
    if q.shape != (4,):
        raise ValueError(f"quat must have shape (4,), got {q.shape}")
    return _run(OP_QUAT_TO_ROTMAT, [q], [9])[0].reshape(3, 3)


def compose_covariance_3d(quat, scale):
    """sg/core.py:174-195: Cov3DBundle(R, S, M = R S, sigma = M M^T)."""
    s = np.asarray(scale, dtype=np.float64)
    if s.shape != (3,):
        raise ValueError(f"scale must have shape (3,), got {s.shape}")
    if np.any(s <= 0.0):
        raise ValueError("scale components must be positive")
    q = np.asarray(quat, dtype=np.float64)
    if q.shape != (4,):
        raise ValueError(f"quat must have shape (4,), got {q.shape}")
    R, S, M, sig = (x.reshape(3, 3) for x in _run(OP_COMPOSE_COV3D, [q, s], [9, 9, 9, 9]))
    return Cov3DBundle(R=R, S=S, M=M, sigma=sig)


def frobenius_inner(x, y):
    """sg/core.py:198-204: sum of elementwise products, Tr(X^T Y)."""
    a = np.asarray(x, dtype=np.float64)
    b = np.asarray(y, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    if a.size == 0:
        return 0.0
    return float(_run(OP_FROBENIUS, [a, b], [1], cols=a.size)[0][0])


# ---------------------------------------------------------- sg/projection.py

def world_to_camera(mean, camera):
    """sg/projection.py:36-42: view @ [mean, 1] (4-vector)."""
    return _run(OP_WORLD_TO_CAMERA, [_f64(mean)[:3]], [4], camera)[0]


def camera_to_pixel(t_cam, camera):
    """sg/projection.py:45-61: pixel coordinates through the perspective
    matrix (= fx tx/tz + 0.5 + cx, the reference's +0.5 convention)."""
    return _run(OP_CAMERA_TO_PIXEL, [_f64(t_cam)[:4]], [2], camera)[0]


def projection_jacobian(t_cam, camera):
    """sg/projection.py:64-82: [[fx/tz, 0, -fx tx/tz^2], [0, fy/tz, -fy ty/tz^2]]."""
    return _run(OP_PROJECTION_JACOBIAN, [_f64(t_cam)[:4]], [6], camera)[0].reshape(2, 3)


def project_covariance(J, R_cw, sigma):
    """sg/projection.py:85-96: (J R_cw) sigma (J R_cw)^T + 0.3 I."""
    return _run(OP_PROJECT_COVARIANCE, [_f64(J, (2, 3)), _f64(R_cw, (3, 3)), _f64(sigma, (3, 3))], [4])[0].reshape(2, 2)


def bounding_radius(cov2d):
    """sg/projection.py:99-112: ceil(3 sqrt(lambda_max)) of the 2x2 covariance."""
    return int(_run(OP_BOUNDING_RADIUS, [_f64(cov2d, (2, 2))], [1])[0][0])


# -------------------------------------------------------- sg/proj_backward.py

def mean2d_backward(d_mean2d, t_cam, camera):
    """sg/proj_backward.py:53-77: dL/dt (4-vector) of a pixel-coordinate gradient."""
    return _run(OP_MEAN2D_BACKWARD, [_f64(d_mean2d)[:2], _f64(t_cam)[:4]], [4], camera)[0]


def cov2d_backward(d_cov2d, T_proj, sigma, J, R_cw, t_cam, camera):
    """sg/proj_backward.py:88-121: (d_sigma 3x3, d_t 4-vector)."""
    d_sigma, d_t = _run(OP_COV2D_BACKWARD, [_f64(d_cov2d, (2, 2)), _f64(T_proj, (2, 3)), _f64(sigma, (3, 3)),
                                            _f64(J, (2, 3)), _f64(R_cw, (3, 3)), _f64(t_cam)[:4]], [9, 4], camera)
    return d_sigma.reshape(3, 3), d_t


def world_backward(d_t_total, camera, mean):
    """sg/proj_backward.py:124-136: (d_mean 3-vector, d_view 4x4)."""
    d_mean, d_view = _run(OP_WORLD_BACKWARD, [_f64(d_t_total)[:4], _f64(mean)[:3]], [3, 16], camera)
    return d_mean, d_view.reshape(4, 4)


def covariance3d_backward(d_sigma, bundle: Cov3DBundle, quat, scale):
    """sg/proj_backward.py:151-175: (d_quat 4-vector (w, x, y, z), d_scale 3-vector)."""
    del scale  # carried by bundle.S, as in the reference
    d_quat, d_scale = _run(OP_COV3D_BACKWARD, [_f64(d_sigma, (3, 3)), _f64(bundle.R, (3, 3)), _f64(bundle.S, (3, 3)),
                                               _f64(bundle.M, (3, 3)), _f64(quat)[:4]], [4, 3])
    return d_quat, d_scale
