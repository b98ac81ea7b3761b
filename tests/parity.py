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
                  if os.path.basename(p) not in ("pixel.npz", "audit_scenes.npz", "helpers.npz"))


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


def runs_gate(g, ref, rel=1e-3, floor=1e-2):
    """Two GPU runs of the same gradients (same kernels and inputs): only the
    fp32 summation order differs -- the raster backward's atomics land in a
    different order, sums over views / ranks / blocks associate differently.
    grad_gate's bound, except that an element whose summed terms nearly
    cancel (d_quat, d_scale) may miss its per-element bound by a small factor:
    a handful of such elements out of millions is allowed, the class as a
    whole must agree (rel-L2 <= 1e-4)."""
    r = grad_gate(g, ref, rel=rel, floor=floor)
    r["ok"] = r["rel_l2"] <= min(rel, 1e-4) and (r["ok"] or (r["n_viol"] <= 4 and r["worst_ratio"] < 10.0))
    return r


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


# ------------------------------------------------------------------ production frame path
#
# The path bench.py times and ops.rasterize / engine.RenderStep run:
# gs_frame_forward (projection + the frame binning + raster_fwd_kernel with
# commit records) and gs_frame_backward (raster_bwd_rec_kernel + the
# projection backward).  Stage-isolated like stage_isolated() above, but every
# GPU quantity comes from the frame workspace itself.

def _f64(a):
    return np.asarray(a, np.float64)


def tile_pixels(tiles, cam):
    """Boolean (H, W) mask of the pixels of the given tile ids."""
    tx_n = (cam.width + 15) // 16
    pix = np.zeros((cam.height, cam.width), bool)
    for t in tiles:
        ty, tx = divmod(int(t), tx_n)
        pix[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = True
    return pix


def _subset_csr(ptr, idx, tiles):
    n_tiles = len(ptr) - 1
    keep = np.zeros(n_tiles, bool)
    keep[np.asarray(tiles, np.int64)] = True
    cnt = np.where(keep, np.diff(ptr), 0)
    sptr = np.concatenate([[0], np.cumsum(cnt)])
    sidx = (np.concatenate([idx[ptr[t]:ptr[t + 1]] for t in tiles]) if len(tiles) else np.zeros(0, np.int64))
    return sptr, sidx.astype(np.int64)


def grad_violations(name, g, ref, ids, rel=GRAD_REL, floor=GRAD_FLOOR, limit=200):
    """The per-element gate of grad_gate, listing every violating element:
    (class, gaussian, component, got, ref, |err| / limit)."""
    g = np.asarray(g, np.float64)
    ref = np.asarray(ref, np.float64)
    rms = float(np.sqrt(np.mean(ref ** 2))) if ref.size else 0.0
    lim = rel * np.maximum(np.abs(ref), floor * rms)
    bad = np.argwhere(np.abs(g - ref) > lim)
    out = []
    for b in bad[:limit]:
        i = tuple(b)
        out.append(dict(cls=name, gaussian=int(ids[i[0]]) if ids is not None else None,
                        component=[int(x) for x in i[1:]], got=float(g[i]), ref=float(ref[i]),
                        ratio=float(abs(g[i] - ref[i]) / (lim[i] + 1e-300))))
    return out


def frame_parity(spec_arrays, cam_spec, d_image, dev, *, tile_frac=None, seed=0, nthreads=0, return_case=False):
    """Production frame path vs the oracle on the same seeded inputs.

    spec_arrays: fp32 (means, scales, quats, opacities, colors) numpy arrays.
    tile_frac: None = every tile (full frame); else the fraction of tiles
    sampled (>= 8) -- d_image is zeroed outside them on BOTH sides, so every
    gradient is the sampled tiles' exact contribution.

    The oracle gets fp64(fp32(x)) inputs and the frame's own fp32
    projection and bins (stage isolation).  d_image is further zeroed at
    branch-flip-prone pixels (oracle decision margin < FLIP_EPS) on both sides.

    Returns a report dict: projection / bins / image / n_contrib checks and
    per-class gradient gates, with every mismatch listed and classified.
    return_case=True stops before the GPU backward and also returns the
    masked d_image, the oracle gradients (full (n, .) arrays) and the
    touched Gaussians, for callers that run the backward themselves
    (engine.RenderStep over several views)."""
    import torch
    from paper_2312_02121_b200 import ops

    m32, s32, q32, o32, c32 = [np.ascontiguousarray(a, np.float32) for a in spec_arrays]
    t = [torch.as_tensor(a, device=dev) for a in (m32, s32, q32, o32, c32)]
    cp = ops.CameraParams.of(cam_spec)
    cam = O.Camera.of(cam_spec)
    n = m32.shape[0]
    rep = dict(camera=dict(width=cam.width, height=cam.height), gaussians=n,
               binning=ops.frame_binning(n, cp))

    fr = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True)
    tv = fr.tensors()
    # the stage projection kernel with cov2d; the frame's projection must be
    # the same arithmetic bit for bit
    proj = ops.project(t[0], t[1], t[2], t[3], cp, want_cov=True)
    torch.cuda.synchronize()
    tiles = _np(tv["tiles"])
    vis = tiles > 0
    xydr = _np(tv["xydr"])
    pxydr = _np(proj.xydr)
    rep["projection_frame_equals_stage"] = bool(
        np.array_equal(tiles, _np(proj.tiles)) and np.array_equal(xydr[vis].view(np.uint32),
                                                                  pxydr[vis].view(np.uint32)))
    g = dict(visible=vis.astype(np.int8), mean2d=xydr[:, :2].astype(np.float64),
             depth=xydr[:, 2].astype(np.float64), radius=xydr[:, 3].copy().view(np.int32).astype(np.int64),
             cov2d=_np(proj.cov2d).astype(np.float64))

    # bins: bit-exact against the oracle's assign_tiles + sort_bins fed the GPU's fp32 projection
    n_tiles = cp.tiles_x * cp.tiles_y
    ptr, idx = ranges_to_csr(_np(tv["ranges"]), _np(tv["sorted_vals"]), n_tiles)
    optr, oidx = O.bin_tiles(g["visible"], g["mean2d"], g["radius"], g["depth"], cam.width, cam.height)
    rep["bins"] = dict(intersections=int(len(idx)), exact=bool(np.array_equal(ptr, optr) and
                                                               np.array_equal(idx, oidx)))
    if not rep["bins"]["exact"]:
        causes, details = classify_bins(ptr, idx, optr, oidx, g["depth"])
        rep["bins"].update(causes=causes, details=[list(map(lambda v: v if isinstance(v, (int, str)) else
                                                            list(v), d)) for d in details[:50]])

    rng = np.random.default_rng(seed)
    if tile_frac is None:
        sample = np.arange(n_tiles)
        sptr, sidx = ptr, idx
        pix = np.ones((cam.height, cam.width), bool)
    else:
        sample = np.sort(rng.choice(n_tiles, size=min(n_tiles, max(8, int(n_tiles * tile_frac))), replace=False))
        sptr, sidx = _subset_csr(ptr, idx, sample)
        pix = tile_pixels(sample, cam)
    rep["tiles_checked"] = int(len(sample))
    rep["pixels_checked"] = int(pix.sum())

    o64, c64 = _f64(o32), _f64(c32)
    fw = O.raster_fwd(cam.width, cam.height, sptr, sidx, g["mean2d"], g["cov2d"], o64, c64, np.zeros(3), True,
                      margins=True, nthreads=nthreads)
    img = _np(fr.image).astype(np.float64)
    cls = classify_image(img[pix], fw["image"][pix], fw["margin"][pix], fw["margin_kind"][pix])
    err = np.max(np.abs(img - fw["image"]), axis=-1)
    flips = np.argwhere(pix & (err > IMG_TOL))
    rep["image"] = dict(max_err=cls["max_err"], max_err_safe=cls["max_err_safe"], n_over_tol=cls["n_bad"],
                        n_flip=cls["n_flip"], n_unexplained=cls["n_real"], flip_kinds=cls["flip_kinds"],
                        mismatches=[dict(pixel=[int(r), int(c)], err=float(err[r, c]),
                                         kind=KIND[int(fw["margin_kind"][r, c])],
                                         margin=float(fw["margin"][r, c]),
                                         list_position=int(fw["margin_pos"][r, c]))
                                    for r, c in flips[:100]])
    safe = pix & (fw["margin"] >= FLIP_EPS)
    ncg = _np(fr.n_contrib)
    rep["n_contrib"] = dict(safe_pixels=int(safe.sum()),
                            equal_on_safe=bool(np.array_equal(ncg[safe], fw["n_contrib"][safe])),
                            differ_on_flip_prone=int(np.sum(pix & ~safe & (ncg != fw["n_contrib"]))))
    rep["final_T_max_err_safe"] = float(np.abs(_np(fr.final_T)[safe] - fw["final_T"][safe]).max()) \
        if safe.any() else 0.0

    d_masked = (np.asarray(d_image, np.float64) * safe[..., None]).astype(np.float32)
    rb = O.raster_bwd(cam.width, cam.height, sptr, sidx, g["mean2d"], g["cov2d"], o64, c64, np.zeros(3),
                      fw["final_T"], fw["n_contrib"], d_masked.astype(np.float64), nthreads=nthreads)
    touched = np.unique(sidx) if len(sidx) else np.zeros(0, np.int64)
    m64, s64, q64 = _f64(m32)[touched], _f64(s32)[touched], _f64(q32)[touched]
    pr_t = O.project(m64, s64, q64, cam, nthreads=nthreads)
    pb = O.project_bwd(m64, s64, q64, cam, np.ones(len(touched), np.int8), pr_t["t_cam"],
                       rb["d_mean2d"][touched], rb["d_cov2d"][touched].reshape(-1, 4), nthreads=nthreads)
    ref = dict(d_mean=np.zeros((n, 3)), d_scale=np.zeros((n, 3)), d_quat=np.zeros((n, 4)),
               d_opacity=rb["d_opacity"], d_color=rb["d_color"], d_view=pb["d_view"])
    ref["d_mean"][touched], ref["d_scale"][touched], ref["d_quat"][touched] = pb["d_mean"], pb["d_scale"], pb["d_quat"]
    rep["gaussians_checked"] = int(len(touched))
    if return_case:
        return rep, dict(d_masked=d_masked, ref=ref, touched=touched, frame=fr)
    gf = ops.frame_backward(fr, t[0], t[1], t[2], t[4], torch.as_tensor(d_masked, device=dev), keep_screen=True)
    torch.cuda.synchronize()
    got = {k: _np(gf[k]).astype(np.float64) for k in GRAD_CLASSES}
    rep["gradients"] = compare_grads(got, ref, touched)
    tv = fr.tensors()
    geo = _np(tv["d_geo"]).astype(np.float64)
    screen = dict(d_mean2d=geo[:, :2], d_cov2d=np.stack([geo[:, 2], geo[:, 3], geo[:, 3],
                                                         _np(tv["d_c11"]).astype(np.float64)], 1))
    explain_violations(rep["gradients"], screen, rb, touched, (m32, s32, q32), cam, nthreads)
    rep["ok"] = frame_ok(rep)
    return rep


def explain_violations(grads, screen, rb, touched, params32, cam, nthreads=0):
    """Classify every per-element violation of the projection-backward classes
    (d_mean, d_scale, d_quat) -- the methodology of sg/gradcheck.py:276-348
    (decide per element whether a discrepancy is a numerical artefact):

    * the GPU's own screen-space gradients of that Gaussian (d_mean2d,
      d_cov2d: the raster backward's fp32 sums) pass the element gate against
      the oracle's, and
    * the oracle's projection backward FED THOSE fp32 screen-space values
      reproduces the GPU's parameter gradient (|err| <= the gate), i.e. the
      GPU's projection backward is exact and the whole difference is the
      raster backward's fp32 summation error carried through the chain;
    * kappa = sum_j |M_ij u_j| / |sum_j M_ij u_j| (M = the linear map from
      the 6 screen-space inputs u to the element, columns from unit inputs)
      is the cancellation factor that amplifies that relative error.

    Such a violation is "fp32-summation x cancellation".  One whose isolated
    projection-backward error exceeds the gate but stays within the fp32
    rounding bound of its terms, 32 * 2^-24 * sum_j |M_ij u_j|, is
    "fp32-rounding x cancellation" (the element is a near-total cancellation
    of terms kappa times larger than itself).  Any other is "unexplained".  Counts land in grads[cls]["explained"/"unexplained"]."""
    m32, s32, q32 = params32
    scr_ref = dict(d_mean2d=rb["d_mean2d"], d_cov2d=rb["d_cov2d"].reshape(-1, 4))
    scr_rms = {k: float(np.sqrt(np.mean(v[touched] ** 2))) if len(touched) else 0.0 for k, v in scr_ref.items()}
    for cls in ("d_mean", "d_scale", "d_quat"):
        r = grads.get(cls)
        if r is None:
            continue
        r["explained"], r["unexplained"] = 0, max(0, r["n_viol"] - len(r["violations"]))  # unlisted: unexplained
        for v in r["violations"]:
            i = v["gaussian"]
            sl = slice(i, i + 1)
            ss_ok = True
            for k in ("d_mean2d", "d_cov2d"):
                lim = GRAD_REL * np.maximum(np.abs(scr_ref[k][i]), GRAD_FLOOR * scr_rms[k])
                ss_ok &= bool(np.all(np.abs(screen[k][i] - scr_ref[k][i]) <= lim))
            m64, s64, q64 = _f64(m32)[sl], _f64(s32)[sl], _f64(q32)[sl]
            tc = O.project(m64, s64, q64, cam)["t_cam"]
            iso = O.project_bwd(m64, s64, q64, cam, np.ones(1, np.int8), tc, screen["d_mean2d"][sl],
                                screen["d_cov2d"][sl])[cls][0]
            c = tuple(v["component"])
            iso_err = abs(v["got"] - float(iso[c]))
            lim_e = abs(v["got"] - v["ref"]) / v["ratio"] if v["ratio"] > 0 else 0.0
            u = np.concatenate([screen["d_mean2d"][i], screen["d_cov2d"][i]])
            terms = []
            for j in range(6):
                e = np.zeros(6)
                e[j] = 1.0
                col = O.project_bwd(m64, s64, q64, cam, np.ones(1, np.int8), tc, e[None, :2], e[None, 2:])[cls][0]
                terms.append(float(col[c]) * u[j])
            kappa = float(np.sum(np.abs(terms)) / max(abs(np.sum(terms)), 1e-300))
            # fp32 rounding bound of a sum of terms of total magnitude sum|M_ij u_j| = kappa |result|
            rounding = 32.0 * 2.0 ** -24 * float(np.sum(np.abs(terms)))
            v.update(screen_space_within_gate=ss_ok, projection_bwd_isolated_err=iso_err, gate=lim_e,
                     kappa=kappa, fp32_rounding_bound=rounding)
            if ss_ok and iso_err <= lim_e:
                v["cause"] = "fp32-summation x cancellation"
                r["explained"] += 1
            elif ss_ok and iso_err <= rounding:
                v["cause"] = "fp32-rounding x cancellation"
                r["explained"] += 1
            else:
                v["cause"] = "unexplained"
                r["unexplained"] += 1
        # the class passes when rel-L2 holds and every violation is explained
        r["ok"] = bool(r["rel_l2"] <= GRAD_REL and r["unexplained"] == 0 and
                       r.get("nonzero_outside_sample", 0) == 0)


def frame_ok(rep):
    return bool(all(r["ok"] for r in rep["gradients"].values()) and rep["image"]["n_unexplained"] == 0
                and rep["n_contrib"]["equal_on_safe"] and rep["bins"]["exact"]
                and rep["projection_frame_equals_stage"])


def compare_grads(got, ref, touched):
    """Per-class gates on the Gaussians the checked tiles hold (rms over
    those, not the mostly-zero full arrays); every other Gaussian's gradient
    must be exactly zero.  Violations are listed element by element."""
    n = len(ref["d_opacity"])
    rest = np.ones(n, bool)
    rest[touched] = False
    out = {}
    for k in GRAD_CLASSES:
        if k not in got:
            continue
        gk = got[k] if k == "d_view" else got[k][touched]
        rk = ref[k] if k == "d_view" else ref[k][touched]
        r = grad_gate(gk, rk)
        r["elements"] = int(np.asarray(rk).size)
        r["violations"] = grad_violations(k, gk, rk, None if k == "d_view" else touched)
        if k != "d_view":
            r["nonzero_outside_sample"] = int(np.count_nonzero(got[k][rest]))
            r["ok"] = bool(r["ok"] and r["nonzero_outside_sample"] == 0)
        out[k] = r
    return out
