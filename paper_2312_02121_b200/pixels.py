"""Per-pixel API on the device: batched wrappers of
gs_conic_from_cov / gs_eval_alpha / gs_composite_pixels /
gs_composite_pixels_bwd (include/splat_b200.h).

A query is one pixel centre with its own depth-ordered bin (CSR
``bin_ptr`` int64 (q+1), ``bin_idx`` int32 into the splat arrays).  The
reference's one-pixel functions (api.composite_pixel, ...) are batches of
one; tests and diagnostics batch thousands.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import check
from .ops import _check_param, _stream


def _f32(t, name, cols):
    return _check_param(name, t, cols)


def conic_from_cov(cov3: torch.Tensor, opacities: torch.Tensor) -> torch.Tensor:
    """(m,3) covariance terms (a, b, c) + opacities -> (m,4) conic (A, B, C, o)
    (sg/raster_forward.py:86-92).  Raises ValueError like the reference when
    a covariance is not invertible."""
    cov3 = _f32(cov3, "cov3", 3)
    m = cov3.shape[0]
    conic = torch.empty((m, 4), device=cov3.device, dtype=torch.float32)
    status = torch.full((1,), -1, device=cov3.device, dtype=torch.int64)
    if m:
        check(_lib.load().gs_conic_from_cov(cov3.data_ptr(), _f32(opacities, "opacities", None).data_ptr(), m,
                                            conic.data_ptr(), status.data_ptr(), _stream()), "gs_conic_from_cov")
        if int(status.item()) != -1:
            raise ValueError("2d covariance is not invertible")  # sg/raster_forward.py:89-90
    return conic


def eval_alpha(xydr: torch.Tensor, conic: torch.Tensor, splat: torch.Tensor, pix: torch.Tensor):
    """sg/raster_forward.py:175-196 for q (splat, pixel centre) pairs.
    Returns alpha (q), delta (q,2), sigma (q)."""
    q = int(splat.shape[0])
    dev = xydr.device
    alpha = torch.empty(q, device=dev, dtype=torch.float32)
    delta = torch.empty((q, 2), device=dev, dtype=torch.float32)
    sigma = torch.empty(q, device=dev, dtype=torch.float32)
    if q:
        check(_lib.load().gs_eval_alpha(_f32(xydr, "xydr", 4).data_ptr(), _f32(conic, "conic", 4).data_ptr(),
                                        splat.to(torch.int32).contiguous().data_ptr(),
                                        _f32(pix, "pix", 2).data_ptr(), q, alpha.data_ptr(), delta.data_ptr(),
                                        sigma.data_ptr(), _stream()), "gs_eval_alpha")
    return alpha, delta, sigma


def _bins(bin_ptr, bin_idx, dev):
    bp = torch.as_tensor(bin_ptr, dtype=torch.int64, device=dev).contiguous()
    bi = torch.as_tensor(bin_idx, dtype=torch.int32, device=dev).contiguous()
    return bp, bi


def composite_pixels(xydr, conic, colors, bin_ptr, bin_idx, pix, background, early_termination=True):
    """sg/raster_forward.py:199-219 for q queries.  Returns color (q,3),
    final_T (q), n_contrib (q)."""
    dev = pix.device
    xydr, conic, colors = _f32(xydr, "xydr", 4), _f32(conic, "conic", 4), _f32(colors, "colors", 3)
    bp, bi = _bins(bin_ptr, bin_idx, dev)
    q = int(bp.shape[0]) - 1
    color = torch.empty((q, 3), device=dev, dtype=torch.float32)
    T = torch.empty(q, device=dev, dtype=torch.float32)
    nc = torch.empty(q, device=dev, dtype=torch.int32)
    bg = (C.c_float * 3)(*[float(b) for b in background])
    if q:
        check(_lib.load().gs_composite_pixels(xydr.data_ptr(), conic.data_ptr(), colors.data_ptr(), bp.data_ptr(),
                                              bi.data_ptr(), _f32(pix, "pix", 2).data_ptr(), q, bg,
                                              int(bool(early_termination)), color.data_ptr(), T.data_ptr(),
                                              nc.data_ptr(), _stream()), "gs_composite_pixels")
    return color, T, nc


def composite_pixels_backward(xydr, conic, colors, bin_ptr, bin_idx, pix, background, final_T, n_contrib,
                              d_pixels, *, want_t_log=False):
    """sg/raster_backward.py:111-163 for q queries.  Returns per-splat
    d_rgbo (m,4), d_geo (m,4), d_c11 (m) and, with want_t_log, the replayed
    T per bin entry (NaN where the entry did not contribute)."""
    dev = pix.device
    xydr, conic, colors = _f32(xydr, "xydr", 4), _f32(conic, "conic", 4), _f32(colors, "colors", 3)
    bp, bi = _bins(bin_ptr, bin_idx, dev)
    q = int(bp.shape[0]) - 1
    m = int(xydr.shape[0])
    d_rgbo = torch.zeros((m, 4), device=dev, dtype=torch.float32)
    d_geo = torch.zeros((m, 4), device=dev, dtype=torch.float32)
    d_c11 = torch.zeros(m, device=dev, dtype=torch.float32)
    t_log = torch.empty(int(bi.shape[0]), device=dev, dtype=torch.float32) if want_t_log else None
    bg = (C.c_float * 3)(*[float(b) for b in background])
    if q:
        check(_lib.load().gs_composite_pixels_bwd(
            xydr.data_ptr(), conic.data_ptr(), colors.data_ptr(), bp.data_ptr(), bi.data_ptr(),
            _f32(pix, "pix", 2).data_ptr(), q, bg, _f32(final_T, "final_T", None).data_ptr(),
            n_contrib.to(torch.int32).contiguous().data_ptr(), _f32(d_pixels, "d_pixels", 3).data_ptr(),
            d_rgbo.data_ptr(), d_geo.data_ptr(), d_c11.data_ptr(), None if t_log is None else t_log.data_ptr(),
            _stream()), "gs_composite_pixels_bwd")
    return d_rgbo, d_geo, d_c11, t_log
