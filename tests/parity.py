"""Parity harness: GPU path vs the fp64 oracle (test infrastructure).

Stage isolation: the oracle is fed ``fp64(fp32(x))`` of the
GPU's inputs, and for the later stages the GPU's own fp32 intermediates, so a
mismatch is attributed to the stage that produced it.  fp32-vs-fp64 branch
flips (sigma cut 4.5, alpha >= 1/255, alpha clamp 0.999, T < 1e-4) are
classified with the oracle's per-pixel decision margin -- the branch-margin
idea of sg/gradcheck.py:276-348 _pixel_safety_mask -- and LISTED; every
other pixel is held to the north-star tolerance.
"""

from __future__ import annotations

import glob
import os

import numpy as np

import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
IMG_TOL = 1e-4          # BASELINE north star: images within 1e-4 max-abs
GRAD_REL = 1e-3         # parameter gradients within 1e-3 relative
FLIP_EPS = 2e-3         # relative decision margin under which fp32 may flip
GRAD_FLOOR = 0.1        # per-element floor: 0.1 * rms of the class
KIND = {0: "none", 1: "sigma<=4.5", 2: "alpha>=1/255", 3: "alpha_raw<0.999", 4: "T<1e-4"}
GRAD_CLASSES = ("d_mean", "d_scale", "d_quat", "d_opacity", "d_color", "d_view")


def golden_names():
    # frame fixtures (make_golden.py); pixel.npz is the per-pixel API's own
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if os.path.basename(p) not in ("pixel.npz", "audit_scenes.npz"))


def load_pixel_golden():
    """tests/golden/pixel.npz (make_golden_pixel.py) with per-splat arrays in
    the oracle's layout: cov3 (a, b, c) and the scene rows gathered per
    projected splat."""
    z = dict(np.load(os.path.join(GOLDEN, "pixel.npz")))
    src = z["source_index"]
    z["cov3"] = z["cov2d"].reshape(-1, 4)[:, [0, 1, 3]]
    z["ea_cov3"] = z["ea_cov2d"].reshape(-1, 4)[:, [0, 1, 3]]
    z["p_opacity"] = z["s_opacity"][src]
    z["p_color"] = z["s_color"][src]
    return z


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    d = {k: z[k] for k in z.files}
    fx, fy, cx, cy, near, far = (float(v) for v in d["intr"])
    W, H = (int(v) for v in d["size"])
    d["camera"] = O.Camera(d["view"].astype(np.float64), fx, fy, cx, cy, W, H, near, far)
    d["et"] = bool(d["early_termination"])
    d["inputs"] = tuple(d[k].astype(np.float64) for k in ("means", "scales", "quats", "opacities", "colors"))
    return d


def ranges_to_csr(ranges, vals, n_tiles):
    ranges = np.asarray(ranges, dtype=np.int64).reshape(n_tiles, 2)
    cnt = ranges[:, 1] - ranges[:, 0]
    ptr = np.zeros(n_tiles + 1, np.int64)
    ptr[1:] = np.cumsum(cnt)
    nz = cnt > 0
    assert np.array_equal(ranges[nz, 0], ptr[:-1][nz]), "tile ranges are not contiguous in tile order"
    return ptr, np.asarray(vals, dtype=np.int64)


def _np(t):
    return t.detach().cpu().numpy()


class GpuFrame:
    """One GPU render (forward) whose backward can be run for any d_image."""

    def __init__(self, inputs, cam, background, et, device, counts=False):
        import torch
        from paper_2312_02121_b200 import ops

        self.torch, self.ops = torch, ops
        self.device = device
        f32 = lambda a, cols: torch.as_tensor(np.ascontiguousarray(np.asarray(a, np.float32).reshape(
            (-1, cols) if cols else (-1,))), device=device)
        means, scales, quats, opac, colors = inputs
        self.t = (f32(means, 3), f32(scales, 3), f32(quats, 4), f32(opac, 0), f32(colors, 3))
        self.cam = cam
        self.cp = ops.CameraParams.of(cam)
        self.background = tuple(float(b) for b in np.asarray(background, np.float64))
        m, s, q, o, c = self.t
        self.image_t, self.state = ops.render_forward(m, s, q, o, c, self.cp, self.background, et, want_cov=True,
                                                      counts=counts)
        torch.cuda.synchronize()
        st = self.state
        n_tiles = self.cp.tiles_x * self.cp.tiles_y
        xydr = _np(st.proj.xydr)
        tiles = _np(st.proj.tiles)
        ptr, idx = ranges_to_csr(_np(st.bins.ranges), _np(st.bins.sorted_vals), n_tiles)
        self.out = dict(
            visible=(tiles > 0).astype(np.int8), tiles=tiles, mean2d=xydr[:, :2].astype(np.float64),
            depth=xydr[:, 2].astype(np.float64), radius=xydr[:, 3].copy().view(np.int32).astype(np.int64),
            conic=_np(st.proj.conic), cov2d=_np(st.proj.cov2d).astype(np.float64),
            bin_ptr=ptr, bin_idx=idx, sorted_keys=_np(st.bins.sorted_keys),
            image=_np(self.image_t).astype(np.float64), final_T=_np(st.final_T).astype(np.float64),
            n_contrib=_np(st.n_contrib).astype(np.int64),
        )
        if counts:
            self.out["counts_fwd"] = _np(st.counts_fwd)

    def backward(self, d_image, counts=False):
        torch = self.torch
        m, s, q, o, c = self.t
        d = torch.as_tensor(np.ascontiguousarray(np.asarray(d_image, np.float32)), device=self.device)
        g = self.ops.render_backward(self.state, m, s, q, c, d, counts=counts)
        torch.cuda.synchronize()
        geo = _np(g["d_geo"]).astype(np.float64)
        c11 = _np(g["d_c11"]).astype(np.float64)
        out = {k: _np(g[k]).astype(np.float64) for k in GRAD_CLASSES}
        out["d_mean2d"] = geo[:, :2]
        out["d_cov2d"] = np.stack([geo[:, 2], geo[:, 3], geo[:, 3], c11], axis=1).reshape(-1, 2, 2)
        if counts:
            out["counts_bwd"] = _np(g["counts"])
        return out


def bins_from_gpu_projection(gpu_out, cam):
    """sg/binning.py:27-65 fed with the GPU's fp32 projection (bit-exact rule)."""
    return O.bin_tiles(gpu_out["visible"], gpu_out["mean2d"], gpu_out["radius"], gpu_out["depth"], cam.width,
                       cam.height)


def classify_image(img, ref, margin, margin_kind, tol=IMG_TOL, eps=FLIP_EPS):
    err = np.max(np.abs(img - ref), axis=-1)
    bad = err > tol
    flip = bad & (margin < eps)
    real = bad & ~flip
    kinds = {}
    for k in np.unique(margin_kind[flip]):
        kinds[KIND[int(k)]] = int(np.sum(margin_kind[flip] == k))
    nonflip = ~(margin < eps)
    return dict(max_err=float(err.max()) if err.size else 0.0,
                max_err_safe=float(err[nonflip].max()) if np.any(nonflip) else 0.0,
                n_bad=int(bad.sum()), n_flip=int(flip.sum()), n_real=int(real.sum()), flip_kinds=kinds,
                real_pixels=np.argwhere(real)[:10].tolist())


def grad_gate(g, ref, rel=GRAD_REL, floor=GRAD_FLOOR):
    g = np.asarray(g, np.float64).reshape(-1)
    ref = np.asarray(ref, np.float64).reshape(-1)
    nrm = np.linalg.norm(ref)
    rel_l2 = float(np.linalg.norm(g - ref) / nrm) if nrm > 0 else float(np.linalg.norm(g))
    rms = float(np.sqrt(np.mean(ref ** 2))) if ref.size else 0.0
    lim = rel * np.maximum(np.abs(ref), floor * rms)
    ratio = np.abs(g - ref) / (lim + 1e-300)
    viol = np.abs(g - ref) > lim
    if nrm == 0:
        viol = np.abs(g) > 1e-30
    return dict(rel_l2=rel_l2, n_viol=int(viol.sum()), worst_ratio=float(ratio.max()) if ratio.size else 0.0,
                ok=(rel_l2 <= rel) and not viol.any())


def stage_isolated(frame: GpuFrame, inputs, cam, d_image, nthreads=0):
    """Oracle forward on the GPU's projection+bins (with margins), a branch-
    safe d_image mask, GPU and oracle backward on that masked d_image."""
    means, scales, quats, opac, colors = inputs
    g = frame.out
    fw = O.raster_fwd(cam.width, cam.height, g["bin_ptr"], g["bin_idx"], g["mean2d"], g["cov2d"], opac, colors,
                      frame.background, frame.state.early_termination, margins=True, nthreads=nthreads)
    safe = fw["margin"] >= FLIP_EPS
    d_masked = np.asarray(d_image, np.float64) * safe[..., None]
    d_masked = d_masked.astype(np.float32).astype(np.float64)
    rb = O.raster_bwd(cam.width, cam.height, g["bin_ptr"], g["bin_idx"], g["mean2d"], g["cov2d"], opac, colors,
                      frame.background, fw["final_T"], fw["n_contrib"], d_masked, nthreads=nthreads)
    pr = O.project(means, scales, quats, cam, nthreads=nthreads)
    vis = g["visible"]
    pb = O.project_bwd(means, scales, quats, cam, vis, pr["t_cam"], rb["d_mean2d"], rb["d_cov2d"].reshape(-1, 4),
                       nthreads=nthreads)
    ref = dict(d_mean=pb["d_mean"], d_scale=pb["d_scale"], d_quat=pb["d_quat"], d_opacity=rb["d_opacity"],
               d_color=rb["d_color"], d_view=pb["d_view"], d_mean2d=rb["d_mean2d"], d_cov2d=rb["d_cov2d"],
               counts_bwd=rb["counts"])
    gg = frame.backward(d_masked)
    return fw, safe, ref, gg


def projection_diffs(gpu_out, pr):
    """Compare GPU projection to the oracle's fp64 projection; list borderline
    cases by cause (visibility / radius ceil)."""
    vis_g, vis_o = gpu_out["visible"].astype(bool), pr["visible"].astype(bool)
    both = vis_g & vis_o
    rad_diff = np.nonzero(both & (gpu_out["radius"] != pr["radius"]))[0]
    causes = []
    for i in rad_diff:
        # radius = ceil(3 sqrt(lambda)): a flip needs 3 sqrt(lambda) within rounding of an integer
        a, b, c = pr["cov2d"][i]
        lam = 0.5 * (a + c) + np.sqrt(0.25 * (a - c) ** 2 + b * b)
        x = 3.0 * np.sqrt(lam)
        causes.append(("radius-ceil", int(i), float(abs(x - round(x)))))
    for i in np.nonzero(vis_g != vis_o)[0]:
        causes.append(("visibility", int(i), float(pr["depth"][i])))
    m2 = np.abs(gpu_out["mean2d"][both] - pr["mean2d"][both]).max() if both.any() else 0.0
    cov_rel = (np.abs(gpu_out["cov2d"][both] - pr["cov2d"][both]).max(axis=1) /
               np.abs(pr["cov2d"][both]).max(axis=1)).max() if both.any() else 0.0
    return dict(n_vis_gpu=int(vis_g.sum()), n_vis_oracle=int(vis_o.sum()), n_vis_diff=int((vis_g != vis_o).sum()),
                n_radius_diff=int(len(rad_diff)), causes=causes, mean2d_max_abs=float(m2),
                cov2d_max_rel=float(cov_rel))


def classify_bins(g_ptr, g_idx, r_ptr, r_idx, gpu_depth, gpu_rect_fn=None, ref_rect_fn=None):
    """Explain every tile whose GPU list differs from the reference's.

    Causes: "depth-tie" (same members; the order differs only among splats
    whose fp32 depths are equal, which the GPU orders by index while the
    fp64 reference orders by the unrounded depth) and "rect" (membership
    differs because the fp32 and fp64 tile rectangles differ, i.e. a radius
    ceil / mean2d borderline case).  Anything else is "unexplained".
    """
    n_tiles = len(g_ptr) - 1
    causes = {"depth-tie": 0, "rect": 0, "unexplained": 0}
    details = []
    for t in range(n_tiles):
        a = g_idx[g_ptr[t]:g_ptr[t + 1]]
        b = r_idx[r_ptr[t]:r_ptr[t + 1]]
        if len(a) == len(b) and np.array_equal(a, b):
            continue
        if set(a.tolist()) == set(b.tolist()):
            key = sorted(b.tolist(), key=lambda j: (np.float32(gpu_depth[j]), j))
            if key == a.tolist():
                causes["depth-tie"] += 1
                details.append(("depth-tie", t))
                continue
            causes["unexplained"] += 1
            details.append(("order", t))
            continue
        sym = set(a.tolist()) ^ set(b.tolist())
        ok = gpu_rect_fn is not None and all(gpu_rect_fn(j, t) != ref_rect_fn(j, t) for j in sym)
        causes["rect" if ok else "unexplained"] += 1
        details.append(("rect" if ok else "membership", t, sorted(sym)[:5]))
    return causes, details


def rect_contains(mean2d, radius, width, height):
    tx_n = (width + 15) // 16
    ty_n = (height + 15) // 16

    def fn(j, t):
        tx, ty = t % tx_n, t // tx_n
        x, y, r = float(mean2d[j][0]), float(mean2d[j][1]), int(radius[j])
        x0 = max(0, int(np.floor((x - r) / 16))); x1 = min(tx_n - 1, int(np.floor((x + r) / 16)))
        y0 = max(0, int(np.floor((y - r) / 16))); y1 = min(ty_n - 1, int(np.floor((y + r) / 16)))
        return x0 <= tx <= x1 and y0 <= ty <= y1
    return fn
