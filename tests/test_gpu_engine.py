"""GPU: engine.RenderStep / pipeline (captured fwd+bwd graphs, double-
buffered host I/O) give the per-call frame path's gradients, and recover
from an intersection-capacity overflow like the per-call path."""

import numpy as np
import pytest
import torch

from parity import load_golden

pytestmark = pytest.mark.gpu


def _per_call(ops, params, cam, d_image):
    fr = ops.frame_forward(*params, cam, (0.0, 0.0, 0.0), True)
    g = ops.frame_backward(fr, params[0], params[1], params[2], params[4], d_image)
    return torch.cat([g["d_mean"].reshape(-1), g["d_scale"].reshape(-1), g["d_quat"].reshape(-1),
                      g["d_rgbo"].reshape(-1)])


def _close(a, b):
    a, b = a.cpu().numpy().astype(np.float64), b.cpu().numpy().astype(np.float64)
    n = len(a) // 14
    for lo, hi in ((0, 3 * n), (3 * n, 6 * n), (6 * n, 10 * n), (10 * n, 14 * n)):  # per gradient class
        scale = np.abs(b[lo:hi]).max() + 1e-30
        assert np.max(np.abs(a[lo:hi] - b[lo:hi])) / scale < 1e-4  # atomic summation order only


def test_step_and_pipeline_match_per_call(cuda):
    from paper_2312_02121_b200 import engine as E, ops
    g = load_golden("config0")
    params = [torch.as_tensor(np.asarray(a, np.float32), device=cuda) for a in g["inputs"]]
    cam = ops.CameraParams.of(g["camera"])
    rng = np.random.default_rng(0)
    d_image = torch.as_tensor(rng.normal(size=(cam.height, cam.width, 3)).astype(np.float32), device=cuda)
    ref = _per_call(ops, params, cam, d_image)

    eng = E.RenderStep(len(params[0]), [cam], device=cuda)
    eng.prime(params, [d_image])
    _close(eng.step(params, [d_image]), ref)

    host = [p.cpu().pin_memory() for p in params]
    dh = [d_image.cpu().pin_memory()]
    out = [torch.empty((14 * len(params[0]),)).pin_memory() for _ in range(eng.nbuf)]
    metas = E.pipeline(eng, host, dh, out, 5)
    torch.cuda.synchronize()
    for b, mh in enumerate(metas):
        eng.result(b, mh)
        _close(out[b], ref)


def test_step_recovers_from_capacity_overflow(cuda):
    from paper_2312_02121_b200 import engine as E, ops
    g = load_golden("config0")
    params = [torch.as_tensor(np.asarray(a, np.float32), device=cuda) for a in g["inputs"]]
    cam = ops.CameraParams.of(g["camera"])
    d_image = torch.ones((cam.height, cam.width, 3), device=cuda)
    small = [p.clone() for p in params]
    small[1] = small[1] * 0.25  # smaller splats -> fewer intersections when sizing
    eng = E.RenderStep(len(params[0]), [cam], device=cuda, headroom=1.0)
    eng.prime(small, [d_image])
    cap0 = eng.caps[0]
    got = eng.step(params, [d_image])
    assert eng.caps[0] > cap0  # grew and re-captured
    _close(got, _per_call(ops, params, cam, d_image))


def test_step_raises_reference_errors(cuda):
    from paper_2312_02121_b200 import engine as E, ops
    g = load_golden("config0")
    params = [torch.as_tensor(np.asarray(a, np.float32), device=cuda) for a in g["inputs"]]
    cam = ops.CameraParams.of(g["camera"])
    d_image = torch.ones((cam.height, cam.width, 3), device=cuda)
    eng = E.RenderStep(len(params[0]), [cam], device=cuda)
    eng.prime(params, [d_image])
    bad = [p.clone() for p in params]
    bad[1].neg_()  # non-positive scales (sg/core.py:189-191)
    with pytest.raises(ValueError, match="scale"):
        eng.step(bad, [d_image])


def test_multi_view_accumulation(cuda):
    """Two views in one step: the accumulate path equals the sum of the
    per-call gradients of each view."""
    from paper_2312_02121_b200 import engine as E, ops
    g = load_golden("config0")
    params = [torch.as_tensor(np.asarray(a, np.float32), device=cuda) for a in g["inputs"]]
    cam = ops.CameraParams.of(g["camera"])
    cam2 = ops.CameraParams(cam.view, cam.fx * 1.1, cam.fy * 1.1, cam.cx, cam.cy, cam.width, cam.height, cam.near,
                            cam.far)
    rng = np.random.default_rng(1)
    d1 = torch.as_tensor(rng.normal(size=(cam.height, cam.width, 3)).astype(np.float32), device=cuda)
    d2 = torch.as_tensor(rng.normal(size=(cam.height, cam.width, 3)).astype(np.float32), device=cuda)
    ref = _per_call(ops, params, cam, d1) + _per_call(ops, params, cam2, d2)
    eng = E.RenderStep(len(params[0]), [cam, cam2], device=cuda)
    eng.prime(params, [d1, d2])
    _close(eng.step(params, [d1, d2]), ref)


def test_multi_view_step_sums_views(cuda):
    """Three views on two streams (engine._body): the step's gradients are
    the sum of the per-call frames' gradients, every view's meta is read."""
    from paper_2312_02121_b200 import engine as E, ops
    g = load_golden("config0")
    params = [torch.as_tensor(np.asarray(a, np.float32), device=cuda) for a in g["inputs"]]
    cam0 = ops.CameraParams.of(g["camera"])
    cams = []
    for k, ang in enumerate((0.0, 0.15, -0.2)):
        c, s_ = np.cos(ang), np.sin(ang)
        view = np.array(cam0.view, np.float64)
        view[:3, :3] = np.array([[c, 0.0, s_], [0.0, 1.0, 0.0], [-s_, 0.0, c]]) @ view[:3, :3]
        cams.append(ops.CameraParams(view.tolist(), cam0.fx, cam0.fy, cam0.cx, cam0.cy, cam0.width, cam0.height,
                                     cam0.near, cam0.far))
    rng = np.random.default_rng(1)
    d_imgs = [torch.as_tensor(rng.normal(size=(cam0.height, cam0.width, 3)).astype(np.float32), device=cuda)
              for _ in cams]
    ref = sum(_per_call(ops, params, c, d) for c, d in zip(cams, d_imgs))
    eng = E.RenderStep(len(params[0]), cams, device=cuda)
    eng.prime(params, d_imgs)
    _close(eng.step(params, d_imgs), ref)
    m = eng.meta(0).cpu()
    assert m.shape == (3, 4) and bool((m[:, 0] == -1).all()) and bool((m[:, 1] > 0).all())


def _views(ops, cam0, angles):
    cams = []
    for ang in angles:
        c, s_ = np.cos(ang), np.sin(ang)
        view = np.array(cam0.view, np.float64)
        view[:3, :3] = np.array([[c, 0.0, s_], [0.0, 1.0, 0.0], [-s_, 0.0, c]]) @ view[:3, :3]
        cams.append(ops.CameraParams(view.tolist(), cam0.fx, cam0.fy, cam0.cx, cam0.cy, cam0.width, cam0.height,
                                     cam0.near, cam0.far))
    return cams


def test_views_project_backward_equals_per_view(cuda):
    """gs_frame_views_project_backward (all views' projection backward in one
    pass over the Gaussians) equals the per-view projection backward summed
    over the views, per gradient class and per view's d_view; the screen-
    space rows are cleared and the workspaces stamped clean (the next frames
    give the same result again)."""
    from paper_2312_02121_b200 import engine as E, ops
    g = load_golden("config0")
    params = [torch.as_tensor(np.asarray(a, np.float32), device=cuda) for a in g["inputs"]]
    m, s, q, o, c = params
    n = len(m)
    cams = _views(ops, ops.CameraParams.of(g["camera"]), (0.0, 0.1, -0.15, 0.3))
    rng = np.random.default_rng(5)
    d_imgs = [torch.as_tensor(rng.normal(size=(cm.height, cm.width, 3)).astype(np.float32), device=cuda)
              for cm in cams]
    ref = {k: torch.zeros((n, w), device=cuda) for k, w in (("d_mean", 3), ("d_scale", 3), ("d_quat", 4),
                                                             ("d_rgbo", 4))}
    ref_views = []
    for cm, d in zip(cams, d_imgs):
        fr = ops.frame_forward(*params, cm, (0.0, 0.0, 0.0), True)
        gv = ops.frame_backward(fr, m, s, q, c, d)
        for k in ref:
            ref[k] += gv[k]
        ref_views.append(gv["d_view"])
    for rep in range(2):
        frames = []
        for cm, d in zip(cams, d_imgs):
            fr = ops.frame_forward(*params, cm, (0.0, 0.0, 0.0), True)
            ops.frame_backward(fr, m, s, q, c, d, project=False)
            frames.append(fr)
        out = {k: torch.full_like(v, 7.0) for k, v in ref.items()}
        d_views = torch.full((len(cams), 4, 4), 3.0, device=cuda)
        ops.frame_views_project_backward(frames, m, s, q, out, d_views)
        torch.cuda.synchronize()
        for k in ref:
            a, b = out[k].cpu().double().numpy(), ref[k].cpu().double().numpy()
            assert np.abs(a - b).max() <= 1e-4 * (np.abs(b).max() + 1e-30), (rep, k)
        for v, dv in enumerate(ref_views):
            a, b = d_views[v].cpu().double().numpy(), dv.cpu().double().numpy()
            assert np.abs(a - b).max() <= 1e-4 * (np.abs(b).max() + 1e-30), (rep, v)
        for fr in frames:
            tv = fr.tensors()
            assert not bool(tv["d_geo"].any()) and not bool(tv["d_c11"].any())  # rows cleared
    # accumulate / add_view add onto the outputs
    frames = []
    for cm, d in zip(cams, d_imgs):
        fr = ops.frame_forward(*params, cm, (0.0, 0.0, 0.0), True)
        ops.frame_backward(fr, m, s, q, c, d, project=False)
        frames.append(fr)
    out = {k: v.clone() for k, v in ref.items()}
    d_views = torch.stack(ref_views).clone()
    ops.frame_views_project_backward(frames, m, s, q, out, d_views, accumulate=True, add_view=True)
    for k in ref:
        a, b = out[k].cpu().double().numpy(), 2 * ref[k].cpu().double().numpy()
        assert np.abs(a - b).max() <= 1e-4 * (np.abs(b).max() + 1e-30), k


def test_views_project_backward_reads_caller_written_rows(cuda):
    """The batched projection backward reads only the rows the raster
    backward marked (gs_frame_view.touched); frame_screen_grads hands the rows
    out for in-place changes (e.g. a sum over ranks) and marks every Gaussian,
    so rows the caller changed or wrote -- here doubled, plus a row for an
    off-screen Gaussian no raster backward touched -- are all read: the result
    equals the per-view projection backward over the same rows (which treats
    a culled Gaussian with non-zero rows as visible)."""
    from paper_2312_02121_b200 import ops
    g = load_golden("config0")
    params = [torch.as_tensor(np.asarray(a, np.float32), device=cuda) for a in g["inputs"]]
    m, s, q, o, c = params
    n = len(m)
    cams = []
    for dx in (2.5, -2.5):  # the scene shifted sideways: part of it off screen
        c0 = ops.CameraParams.of(g["camera"])
        view = np.array(c0.view, np.float64)
        view[0, 3] += dx
        cams.append(ops.CameraParams(view.tolist(), c0.fx, c0.fy, c0.cx, c0.cy, c0.width, c0.height, c0.near,
                                     c0.far))
    rng = np.random.default_rng(7)
    frames, saved, injected = [], [], 0
    for cm in cams:
        d = torch.as_tensor(rng.normal(size=(cm.height, cm.width, 3)).astype(np.float32), device=cuda)
        fr = ops.frame_forward(*params, cm, (0.0, 0.0, 0.0), True)
        ops.frame_backward(fr, m, s, q, c, d, project=False)
        rows, c11 = ops.frame_screen_grads(fr)
        # a Gaussian in front of the camera but off screen: never marked, rows zero
        tv = fr.tensors()
        zero = torch.nonzero((rows == 0).all(1) & (c11 == 0) & (tv["tiles"] == 0) & (tv["xydr"][:, 2] > 1.0)).flatten()
        rows.mul_(2.0)
        if len(zero):
            rows[zero[0]] = torch.tensor([0.1, -0.2, 0.3, 0.05, 0.5, -0.4, 0.02, 0.01], device=cuda)
            c11[zero[0]] = 0.03
            injected += 1
        frames.append(fr)
        saved.append((rows.clone(), c11.clone()))
    assert injected > 0
    shape = (("d_mean", 3), ("d_scale", 3), ("d_quat", 4), ("d_rgbo", 4))
    out = {k: torch.zeros((n, w), device=cuda) for k, w in shape}
    d_views = torch.zeros((len(cams), 4, 4), device=cuda)
    ops.frame_views_project_backward(frames, m, s, q, out, d_views)
    ref = {k: torch.zeros((n, w), device=cuda) for k, w in shape}
    for vi, (fr, (rows, c11)) in enumerate(zip(frames, saved)):
        r2, c2 = ops.frame_screen_grads(fr)  # (the batched pass cleared them)
        r2.copy_(rows)
        c2.copy_(c11)
        dv = torch.zeros((4, 4), device=cuda)
        ops.frame_project_backward(fr, m, s, q, ref, dv, accumulate=vi > 0, vis_from_grads=True)
        a, b = d_views[vi].cpu().double().numpy(), dv.cpu().double().numpy()
        assert np.abs(a - b).max() <= 1e-4 * (np.abs(b).max() + 1e-30), vi
    for k in ref:
        a, b = out[k].cpu().double().numpy(), ref[k].cpu().double().numpy()
        assert np.abs(a - b).max() <= 1e-4 * (np.abs(b).max() + 1e-30), k


def test_frames_project_equals_per_view_projection(cuda):
    """gs_frames_project (every view's depth-first projection in one pass)
    then gs_frame_forward_projected per view give the per-view
    gs_frame_forward's frames bit for bit (same operations, same order),
    including the error a bad Gaussian raises in a view that sees it."""
    from paper_2312_02121_b200 import ops
    from paper_2312_02121_b200.scenes import make_config
    spec = make_config(3, n_override=450_000, n_views=3)  # > 400k: depth-first binning
    params = [torch.as_tensor(a, device=cuda) for a in (spec.means, spec.scales, spec.quats, spec.opacities,
                                                        spec.colors)]
    n = spec.n
    cams = [ops.CameraParams.of(c) for c in spec.cameras]
    assert ops.frames_projectable(n, cams)
    refs = [ops.frame_forward(*params, cm, (0.0, 0.0, 0.0), True) for cm in cams]
    caps = [r.capacity for r in refs]
    wss = [ops.frame_workspace(n, cap, cm.width, cm.height, cuda) for cap, cm in zip(caps, cams)]
    ops.frames_project(*params[:4], cams, caps, wss)
    for r, cm, cap, ws in zip(refs, cams, caps, wss):
        fr = ops.frame_forward(*params, cm, (0.0, 0.0, 0.0), True, capacity=cap, ws=ws, check_meta=False,
                               projected=True)
        assert torch.equal(fr.image, r.image) and torch.equal(fr.final_T, r.final_T)
        assert torch.equal(fr.n_contrib, r.n_contrib)
        ta, tb = fr.tensors(), r.tensors()
        for k in ("xydr", "conic", "tiles", "ranges", "sorted_vals", "depth_order"):
            assert torch.equal(ta[k], tb[k]), k
        assert torch.equal(fr.meta().cpu()[:9], r.meta().cpu()[:9])
    bad = [p.clone() for p in params]
    bad[1][123] = -1.0  # a non-positive scale (sg/core.py:189-191): the error of every view that sees it
    ops.frames_project(*bad[:4], cams, caps, wss)
    errs = 0
    for cm, cap, ws in zip(cams, caps, wss):
        fr = ops.frame_forward(*bad, cm, (0.0, 0.0, 0.0), True, capacity=cap, ws=ws, check_meta=False,
                               projected=True)
        ref = ops.frame_forward(*bad, cm, (0.0, 0.0, 0.0), True, check_meta=False)
        st = int(fr.meta().cpu()[0])
        assert st == int(ref.meta().cpu()[0])
        if st != -1:
            errs += 1
            with pytest.raises(ValueError, match="scale"):
                ops.raise_status(st)
    assert errs > 0


def test_batched_projections_over_32_views(cuda):
    """More views than one batched launch takes (MV_MAX = 32): both batched
    projections loop over groups of views -- forward bit for bit the per-view
    frames, backward the per-view sums; Gaussian ranges (the bucketed
    multi-GPU path) add up to the whole."""
    from paper_2312_02121_b200 import ops
    from paper_2312_02121_b200.scenes import make_config
    spec = make_config(3, n_override=420_000, n_views=32)  # > 400k Gaussians: depth-first views
    params = [torch.as_tensor(a, device=cuda) for a in (spec.means, spec.scales, spec.quats, spec.opacities,
                                                        spec.colors)]
    m, s, q, o, c = params
    n = spec.n
    # small views (1/4 scale) keep the 36 workspaces cheap; 4 more views turned off the ring's first
    cams = []
    for cs in spec.cameras:
        cp = ops.CameraParams.of(cs)
        cams.append(ops.CameraParams(cp.view, cp.fx / 4, cp.fy / 4, cp.cx / 4, cp.cy / 4, cp.width // 4,
                                     cp.height // 4, cp.near, cp.far))
    cams += _views(ops, cams[0], (0.05, 0.1, -0.05, -0.1))
    assert ops.frames_projectable(n, cams)
    rng = np.random.default_rng(9)
    d_imgs = [torch.as_tensor(rng.normal(size=(cm.height, cm.width, 3)).astype(np.float32), device=cuda)
              for cm in cams]
    refs = [ops.frame_forward(*params, cm, (0.0, 0.0, 0.0), True) for cm in cams]
    caps = [r.capacity for r in refs]
    wss = [ops.frame_workspace(n, cap, cm.width, cm.height, cuda) for cap, cm in zip(caps, cams)]
    ops.frames_project(m, s, q, o, cams, caps, wss)
    frames = []
    for r, cm, cap, ws, d in zip(refs, cams, caps, wss, d_imgs):
        fr = ops.frame_forward(*params, cm, (0.0, 0.0, 0.0), True, capacity=cap, ws=ws, check_meta=False,
                               projected=True)
        assert torch.equal(fr.image, r.image)
        ops.frame_backward(fr, m, s, q, c, d, project=False)
        frames.append(fr)
    ref = {k: torch.zeros((n, w), device=cuda) for k, w in (("d_mean", 3), ("d_scale", 3), ("d_quat", 4),
                                                             ("d_rgbo", 4))}
    for r, d in zip(refs, d_imgs):
        gv = ops.frame_backward(r, m, s, q, c, d)
        for k in ref:
            ref[k] += gv[k]
    # views split over two calls (the second adding): bit for bit the one-call
    # sums (d_view: the same terms, grouped by the calls' work batches)
    one = {k: torch.zeros_like(v) for k, v in ref.items()}
    two = {k: torch.full_like(v, 7.0) for k, v in ref.items()}
    dv1, dv2 = torch.zeros((len(cams), 4, 4), device=cuda), torch.zeros((len(cams), 4, 4), device=cuda)
    ops.frame_views_project_backward(frames, m, s, q, one, dv1, keep_screen=True)
    ops.frame_views_project_backward(frames[:13], m, s, q, two, dv2[:13], keep_screen=True)
    ops.frame_views_project_backward(frames[13:], m, s, q, two, dv2[13:], accumulate=True, keep_screen=True)
    for k in ref:
        assert torch.equal(one[k], two[k]), k
    assert torch.allclose(dv1, dv2, rtol=1e-5, atol=1e-6 * dv1.abs().max().item())
    out = {k: torch.zeros_like(v) for k, v in ref.items()}
    d_views = torch.zeros((len(cams), 4, 4), device=cuda)
    half = n // 2 // 256 * 256
    ops.frame_views_project_backward(frames, m, s, q, out, d_views, 0, half)
    ops.frame_views_project_backward(frames, m, s, q, out, d_views, half, n, add_view=True)
    for k in ref:
        a, b = out[k].cpu().double().numpy(), ref[k].cpu().double().numpy()
        assert np.abs(a - b).max() <= 1e-4 * (np.abs(b).max() + 1e-30), k


def test_batched_and_per_view_engine_agree(cuda):
    """RenderStep with the batched projection backward (default for several
    views) and with one projection backward per view give the same step."""
    from paper_2312_02121_b200 import engine as E, ops
    g = load_golden("config0")
    params = [torch.as_tensor(np.asarray(a, np.float32), device=cuda) for a in g["inputs"]]
    cams = _views(ops, ops.CameraParams.of(g["camera"]), (0.0, 0.2, -0.1))
    rng = np.random.default_rng(2)
    d_imgs = [torch.as_tensor(rng.normal(size=(cm.height, cm.width, 3)).astype(np.float32), device=cuda)
              for cm in cams]
    a = E.RenderStep(len(params[0]), cams, device=cuda)
    b = E.RenderStep(len(params[0]), cams, device=cuda, batched_projection=False)
    assert a.batched and not b.batched
    a.prime(params, d_imgs)
    b.prime(params, d_imgs)
    ga, gb = a.step(params, d_imgs).clone(), b.step(params, d_imgs).clone()
    _close(ga, gb)
    dva, dvb = a.d_view(0).cpu().double().numpy(), b.d_view(0).cpu().double().numpy()
    assert np.abs(dva - dvb).max() <= 1e-4 * np.abs(dvb).max()


def test_pipeline_from_write_combined_staging(cuda):
    """Inputs staged in write-combined pinned memory (engine.host_staging)
    give the same gradients as the per-call path."""
    from paper_2312_02121_b200 import engine as E, ops
    g = load_golden("config0")
    params = [torch.as_tensor(np.asarray(a, np.float32), device=cuda) for a in g["inputs"]]
    cam = ops.CameraParams.of(g["camera"])
    rng = np.random.default_rng(3)
    d_image = torch.as_tensor(rng.normal(size=(cam.height, cam.width, 3)).astype(np.float32), device=cuda)
    ref = _per_call(ops, params, cam, d_image)
    host = []
    for p in params + [d_image]:
        t = E.host_staging(tuple(p.shape))
        assert t.is_pinned()
        t.copy_(p.cpu())
        host.append(t)
    eng = E.RenderStep(len(params[0]), [cam], device=cuda)
    eng.prime(params, [d_image])
    out = [torch.empty((14 * len(params[0]),)).pin_memory() for _ in range(eng.nbuf)]
    metas = E.pipeline(eng, host[:5], host[5:], out, 4)
    torch.cuda.synchronize()
    for b, mh in enumerate(metas):
        eng.result(b, mh)
        _close(out[b], ref)
