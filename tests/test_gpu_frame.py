"""GPU: the production frame path (gs_frame_forward/backward, depth-first
binning, capacity buffers, no host sync) against the staged stage-by-stage
path (64-bit key sort) and the oracle."""

import numpy as np
import pytest
import torch

import oracle as O
from parity import GRAD_CLASSES, classify_image, golden_names, grad_gate, load_golden, runs_gate

pytestmark = pytest.mark.gpu


def _tensors(inputs, dev):
    m, s, q, o, c = inputs
    f = lambda a, sh: torch.as_tensor(np.asarray(a, np.float32).reshape(sh), device=dev).contiguous()
    return f(m, (-1, 3)), f(s, (-1, 3)), f(q, (-1, 4)), f(o, (-1,)), f(c, (-1, 3))


def _both(inputs, cam, bg, et, d_image, dev, capacity=None):
    from paper_2312_02121_b200 import ops
    t = _tensors(inputs, dev)
    cp = ops.CameraParams.of(cam)
    bg = tuple(float(b) for b in np.asarray(bg))
    img_s, st = ops.render_forward(*t, cp, bg, et)
    g_s = ops.render_backward(st, t[0], t[1], t[2], t[4], torch.as_tensor(np.asarray(d_image, np.float32), device=dev))
    fr = ops.frame_forward(*t, cp, bg, et, capacity=capacity)
    g_f = ops.frame_backward(fr, t[0], t[1], t[2], t[4], torch.as_tensor(np.asarray(d_image, np.float32), device=dev))
    torch.cuda.synchronize()
    return st, g_s, img_s, fr, g_f


@pytest.mark.parametrize("name", golden_names())
def test_frame_equals_staged_on_golden(name, cuda):
    g = load_golden(name)
    st, g_s, img_s, fr, g_f = _both(g["inputs"], g["camera"], g["background"], g["et"], g["d_image"], cuda)
    # identical decisions => bitwise identical forward outputs and per-tile lists
    assert torch.equal(fr.image, img_s)
    assert torch.equal(fr.final_T, st.final_T)
    assert torch.equal(fr.n_contrib, st.n_contrib)
    tv = fr.tensors()
    assert fr.n_isect == st.bins.n_isect
    assert torch.equal(tv["ranges"], st.bins.ranges)
    assert torch.equal(tv["sorted_vals"], st.bins.sorted_vals)
    assert torch.equal(tv["sorted_tile_keys"].long(), (st.bins.sorted_keys >> 32))
    for k in GRAD_CLASSES:
        a, b = g_f[k].cpu().numpy(), g_s[k].cpu().numpy()
        r = runs_gate(a, b)  # only the fp32 summation order differs (atomics, reduction tree)
        assert r["ok"], (name, k, r)


@pytest.fixture(params=[(1, 1, 1), (1, 1, 0), (2, 1, 1), (2, 0, 1), (3, 1, 1)],
                ids=["depth_first", "depth_first_onesweep", "scatter", "scatter_sort_kernel", "direct"])
def binning(request, cuda):
    """Run a test under every frame binning strategy (gs_set_option): the
    depth-first one with the tile-sorted emission and with emission + onesweep
    by tile, the scatter one with its per-tile sort fused into the raster
    forward and as its own kernel."""
    from paper_2312_02121_b200 import ops
    ops.set_option("binning", request.param[0])
    ops.set_option("fuse_sort", request.param[1])
    ops.set_option("tile_emit", request.param[2])
    yield request.param[0]
    ops.set_option("binning", 0)
    ops.set_option("fuse_sort", 1)
    ops.set_option("tile_emit", 1)


def _modes():
    """(binning, tile_emit) of every list-producing path."""
    return [(1, 1), (1, 0), (2, 1), (3, 1)]


@pytest.mark.parametrize("name", golden_names())
def test_binning_strategies_agree(name, binning, cuda):
    """Depth-first and scatter binning give the same lists, bit for
    bit (both are sg/binning.py:50-65's (depth, source_index) order)."""
    g = load_golden(name)
    st, g_s, img_s, fr, g_f = _both(g["inputs"], g["camera"], g["background"], g["et"], g["d_image"], cuda)
    tv = fr.tensors()
    assert torch.equal(tv["ranges"], st.bins.ranges)
    assert torch.equal(tv["sorted_vals"], st.bins.sorted_vals)
    assert torch.equal(fr.image, img_s)


def test_depth_order_is_stable_sort(cuda):
    g = load_golden("dense_ties")  # has exact depth ties
    from paper_2312_02121_b200 import ops
    t = _tensors(g["inputs"], cuda)
    ops.set_option("binning", 1)  # depth_order exists in the depth-first strategy
    try:
        fr = ops.frame_forward(*t, ops.CameraParams.of(g["camera"]), (0.0, 0.0, 0.0), True)
    finally:
        ops.set_option("binning", 0)
    tv = fr.tensors()
    order = tv["depth_order"].cpu().numpy()
    depth = tv["xydr"][:, 2].cpu().numpy()
    vis = tv["tiles"].cpu().numpy() > 0
    key = np.where(vis, depth.view(np.uint32), np.uint32(0xFFFFFFFF)).astype(np.uint64)
    ref = np.lexsort((np.arange(len(key)), key))[:int(vis.sum())]  # culled ones are dropped
    assert np.array_equal(order, ref)


@pytest.mark.parametrize("depth_lo,depth_hi,passes", [(3.0, 3.0, 1), (2.0, 7.9, 3), (0.02, 90.0, 4), (1.0, 1.0001, 2)])
def test_depth_sort_relative_keys(depth_lo, depth_hi, passes, cuda):
    """The depth sort ranks keys relative to the visible minimum and runs
    only the 8-bit passes their width needs (meta[8]); culled Gaussians are
    dropped by the first pass.  Order = stable (depth bits, index) of the
    visible ones, whatever the width; bins equal the 64-bit staged sort."""
    from paper_2312_02121_b200 import ops
    rng = np.random.default_rng(int(depth_hi * 100))
    n = 60000
    z = rng.uniform(depth_lo, depth_hi, n) if depth_hi > depth_lo else np.full(n, depth_lo)
    z[::7] = -1.0  # behind the camera: culled
    means = np.stack([rng.uniform(-0.3, 0.3, n) * z, rng.uniform(-0.3, 0.3, n) * z, z], 1)
    means[::11, 0] += 50.0 * np.abs(z[::11])  # off-screen: culled
    scales = np.exp(rng.uniform(np.log(0.002), np.log(0.01), (n, 3))) * np.abs(z)[:, None]
    quats = rng.normal(size=(n, 4))
    opac = rng.uniform(0.05, 0.95, n)
    colors = rng.uniform(0, 1, (n, 3))
    t = _tensors((means, scales, quats, opac, colors), cuda)
    cp = ops.CameraParams(np.eye(4).tolist(), 300.0, 300.0, 320.0, 240.0, 640, 480, 0.01, 100.0)
    ops.set_option("binning", 1)
    try:
        fr = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True)
    finally:
        ops.set_option("binning", 0)
    meta = fr.meta().cpu().numpy()
    tv = fr.tensors()
    vis = tv["tiles"].cpu().numpy() > 0
    assert int(meta[7]) == int(vis.sum()) and int(meta[8]) == passes, (meta[5:9], passes)
    depth = tv["xydr"][:, 2].cpu().numpy().view(np.uint32).astype(np.uint64)
    key = np.where(vis, depth, np.uint64(0xFFFFFFFF))
    ref = np.lexsort((np.arange(n), key))[:int(vis.sum())]
    assert np.array_equal(tv["depth_order"].cpu().numpy(), ref)
    img_s, st = ops.render_forward(*t, cp, (0.0, 0.0, 0.0), True)
    assert torch.equal(tv["sorted_vals"], st.bins.sorted_vals) and torch.equal(fr.image, img_s)


@pytest.mark.parametrize("config", [0, 1])
def test_frame_config_vs_oracle(config, cuda):
    from paper_2312_02121_b200 import ops
    from paper_2312_02121_b200.scenes import make_config
    spec = make_config(config)
    cam = spec.cameras[0]
    t = _tensors((spec.means, spec.scales, spec.quats, spec.opacities, spec.colors), cuda)
    fr = ops.frame_forward(*t, ops.CameraParams.of(cam), (0.0, 0.0, 0.0), True)
    torch.cuda.synchronize()
    f64 = lambda a: np.asarray(a, np.float64)
    ref = O.render(f64(spec.means), f64(spec.scales), f64(spec.quats), f64(spec.opacities), f64(spec.colors),
                   O.Camera.of(cam), np.zeros(3), True, margins=True)
    c = classify_image(fr.image.cpu().numpy().astype(np.float64), ref["image"], ref["margin"], ref["margin_kind"])
    print(f"config{config}: max err {c['max_err']:.2e}, safe max {c['max_err_safe']:.2e}, flips {c['n_flip']} "
          f"{c['flip_kinds']}")
    assert c["n_real"] == 0, c
    assert fr.n_isect == len(ref["bin_idx"]) or abs(fr.n_isect - len(ref["bin_idx"])) < 1e-4 * len(ref["bin_idx"])


def test_capacity_overflow_reruns(cuda):
    from paper_2312_02121_b200 import ops
    g = load_golden("cfg0_mini")
    t = _tensors(g["inputs"], cuda)
    cp = ops.CameraParams.of(g["camera"])
    full = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True)
    small = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True, capacity=100)  # forces a re-run
    assert small.capacity >= small.n_isect > 100
    assert torch.equal(full.image, small.image)
    # unchecked run with too small a capacity reports the true total
    raw = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True, capacity=100, check_meta=False)
    m = raw.meta().cpu()
    assert int(m[1]) == full.n_isect and int(m[0]) == -1


@pytest.mark.parametrize("tile_emit", [1, 0])
def test_depth_first_capacity_overflow_reruns(tile_emit, cuda):
    """Depth-first binning over capacity: the tile scan leaves every range
    empty and the emission writes nothing; the re-run at the reported total
    equals a frame sized right."""
    from paper_2312_02121_b200 import ops
    g = load_golden("cfg0_mini")
    t = _tensors(g["inputs"], cuda)
    cp = ops.CameraParams.of(g["camera"])
    ops.set_option("binning", 1)
    ops.set_option("tile_emit", tile_emit)
    try:
        full = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True)
        small = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True, capacity=100)
        raw = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True, capacity=100, check_meta=False)
        m = raw.meta().cpu()
        assert int(m[1]) == full.n_isect and int(m[0]) == -1
        assert small.capacity >= small.n_isect > 100
        assert torch.equal(full.image, small.image)
        assert torch.equal(full.tensors()["sorted_vals"], small.tensors()["sorted_vals"])
    finally:
        ops.set_option("binning", 0)
        ops.set_option("tile_emit", 1)


def test_frame_errors_and_empty(cuda):
    from paper_2312_02121_b200 import ops
    cp = ops.CameraParams(np.eye(4).tolist(), 16.0, 16.0, 8.0, 8.0, 16, 16, 0.1, 100.0)
    z = lambda *s: torch.zeros(s, device=cuda)
    means = torch.tensor([[0.0, 0.0, 4.0], [0.0, 0.0, 4.0]], device=cuda)
    scales = torch.tensor([[0.1, 0.1, 0.1], [0.1, -1.0, 0.1]], device=cuda)
    quats = torch.tensor([[1.0, 0, 0, 0], [1.0, 0, 0, 0]], device=cuda)
    with pytest.raises(ValueError, match="gaussian 1: scale"):
        ops.frame_forward(means, scales, quats, z(2) + 0.5, z(2, 3), cp)
    fr = ops.frame_forward(z(0, 3), z(0, 3), z(0, 4), z(0), z(0, 3), cp, (0.2, 0.4, 0.6))
    img = fr.image.cpu().numpy()
    assert np.allclose(img, np.array([0.2, 0.4, 0.6], np.float32)[None, None, :])
    assert fr.final_T.min().item() == 1.0 and fr.n_contrib.max().item() == 0
    g = ops.frame_backward(fr, z(0, 3), z(0, 3), z(0, 4), z(0, 3), torch.ones(16, 16, 3, device=cuda))
    assert g["d_view"].abs().max().item() == 0.0


@pytest.mark.parametrize("tile_emit", [1, 0])
def test_depth_first_all_culled_and_errors(tile_emit, cuda):
    """Depth-first binning (both variants) on a scene with nothing visible
    (every Gaussian behind the camera or off screen): background image, no
    intersections, zero gradients; and the reference's error for a bad
    Gaussian that the view sees."""
    from paper_2312_02121_b200 import ops
    cp = ops.CameraParams(np.eye(4).tolist(), 16.0, 16.0, 8.0, 8.0, 16, 16, 0.1, 100.0)
    n = 3000
    means = torch.zeros((n, 3), device=cuda)
    means[:, 2] = -5.0  # behind the camera
    means[::2, 0], means[::2, 2] = 1e4, 5.0  # off screen
    scales = torch.full((n, 3), 0.1, device=cuda)
    quats = torch.zeros((n, 4), device=cuda)
    quats[:, 0] = 1.0
    opac = torch.full((n,), 0.5, device=cuda)
    cols = torch.rand((n, 3), device=cuda)
    ops.set_option("binning", 1)
    ops.set_option("tile_emit", tile_emit)
    try:
        fr = ops.frame_forward(means, scales, quats, opac, cols, cp, (0.2, 0.4, 0.6))
        assert fr.n_isect == 0 and int(fr.meta().cpu()[7]) == 0
        assert np.allclose(fr.image.cpu().numpy(), np.array([0.2, 0.4, 0.6], np.float32)[None, None, :])
        g = ops.frame_backward(fr, means, scales, quats, cols, torch.ones(16, 16, 3, device=cuda))
        for k in ("d_mean", "d_scale", "d_quat", "d_rgbo", "d_view"):
            assert g[k].abs().max().item() == 0.0, k
        bad = scales.clone()
        means2 = means.clone()
        means2[7] = torch.tensor([0.0, 0.0, 4.0], device=cuda)  # visible
        bad[7, 1] = -1.0
        with pytest.raises(ValueError, match="gaussian 7: scale"):
            ops.frame_forward(means2, bad, quats, opac, cols, cp)
    finally:
        ops.set_option("binning", 0)
        ops.set_option("tile_emit", 1)


def test_autograd_matches_frame(cuda):
    from paper_2312_02121_b200 import ops
    g = load_golden("rot_ragged")
    t = [x.clone().requires_grad_(True) for x in _tensors(g["inputs"], cuda)]
    cam = g["camera"]
    view = torch.tensor(cam.view, dtype=torch.float32, requires_grad=True)
    img, T, nc = ops.rasterize(*t, view, cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, cam.near, cam.far,
                               tuple(g["background"]), True)
    d = torch.as_tensor(np.asarray(g["d_image"], np.float32), device=cuda)
    img.backward(d)
    ref = {k: g["g_" + k] for k in GRAD_CLASSES}
    got = dict(d_mean=t[0].grad, d_scale=t[1].grad, d_quat=t[2].grad, d_opacity=t[3].grad, d_color=t[4].grad,
               d_view=view.grad)
    for k in GRAD_CLASSES:
        r = grad_gate(got[k].detach().cpu().numpy(), ref[k])
        assert r["ok"], (k, r)


def test_forward_bitwise_deterministic(cuda):
    """forward outputs and tile lists are bitwise identical run to
    run (the backward may differ through atomic order, which the north star
    allows); the analogue of tests/test_acceptance.py:265-284 for the GPU."""
    from paper_2312_02121_b200 import ops
    from paper_2312_02121_b200.scenes import make_config
    spec = make_config(1)
    t = _tensors((spec.means, spec.scales, spec.quats, spec.opacities, spec.colors), cuda)
    cam = ops.CameraParams.of(spec.cameras[0])
    outs = []
    for _ in range(3):
        fr = ops.frame_forward(*t, cam, (0.1, 0.2, 0.3), True)
        tv = fr.tensors()
        outs.append((fr.image.clone(), fr.final_T.clone(), fr.n_contrib.clone(), tv["ranges"].clone(),
                     tv["sorted_vals"].clone()))
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert torch.equal(a, b)


@pytest.mark.parametrize("config", [1, 2])
def test_binning_strategies_agree_on_configs(config, cuda):
    """All binnings on BASELINE configs: config 2's lists run to thousands of
    entries, so the long-list CTA sort (len > 512) of the scatter and direct
    paths is covered besides the shared-memory sort."""
    from paper_2312_02121_b200 import ops
    from paper_2312_02121_b200.scenes import make_config
    spec = make_config(config, n_views=1)
    t = _tensors((spec.means, spec.scales, spec.quats, spec.opacities, spec.colors), cuda)
    cam = ops.CameraParams.of(spec.cameras[0])
    got = {}
    try:
        for mode in _modes():
            ops.set_option("binning", mode[0])
            ops.set_option("tile_emit", mode[1])
            fr = ops.frame_forward(*t, cam, (0.0, 0.0, 0.0), True)
            tv = fr.tensors()
            got[mode] = (tv["ranges"].clone(), tv["sorted_vals"].clone(), fr.image.clone())
            del fr, tv
    finally:
        ops.set_option("binning", 0)
        ops.set_option("tile_emit", 1)
    lens = (got[(1, 1)][0][:, 1] - got[(1, 1)][0][:, 0])
    if config == 2:
        assert int(lens.max()) > 512
    for m in _modes()[1:]:
        for a, b in zip(got[(1, 1)], got[m]):
            assert torch.equal(a, b)


def test_scatter_binning_ties_in_long_lists(cuda):
    """Scatter binning writes a tile's pairs in arbitrary order; exact depth
    ties must still come out in source-index order, in the shared-memory
    per-tile sort (<= 512 entries) and in the chunked long-list sort alike.
    2400 splats over a 64x64 image (16 tiles, lists of 0 to ~1700 entries),
    a third of them at one exact
    depth and a third at another, checked against depth-first binning (a
    stable global sort, sg/binning.py:50-65's (depth, index) order)."""
    from paper_2312_02121_b200 import ops
    rng = np.random.default_rng(7)
    n = 2400
    means = np.zeros((n, 3), np.float32)
    means[:, 0] = rng.uniform(-0.5, 0.5, n)
    means[:, 1] = rng.uniform(-0.5, 0.5, n)
    means[:, 2] = rng.uniform(-0.5, 0.5, n)
    means[0::3, 2] = 0.25   # exact ties
    means[1::3, 2] = -0.125
    scales = np.exp(rng.uniform(np.log(0.01), np.log(0.2), (n, 3))).astype(np.float32)
    quats = rng.normal(size=(n, 4)).astype(np.float32)
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    opac = rng.uniform(0.2, 0.9, n).astype(np.float32)
    cols = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    view = [[1.0, 0, 0, 0], [0, 1.0, 0, 0], [0, 0, 1.0, 4.0], [0, 0, 0, 1.0]]
    cam = ops.CameraParams(view=view, fx=60.0, fy=60.0, cx=31.5, cy=31.5, width=64, height=64, near=0.1, far=100.0)
    t = _tensors((means, scales, quats, opac, cols), cuda)
    got = {}
    try:
        for mode in _modes():
            ops.set_option("binning", mode[0])
            ops.set_option("tile_emit", mode[1])
            fr = ops.frame_forward(*t, cam, (0.0, 0.0, 0.0), True)
            tv = fr.tensors()
            got[mode] = (tv["ranges"].clone(), tv["sorted_vals"].clone(), fr.image.clone())
    finally:
        ops.set_option("binning", 0)
        ops.set_option("tile_emit", 1)
    lens = got[(1, 1)][0][:, 1] - got[(1, 1)][0][:, 0]
    assert int(lens.max()) > 512 and bool(((lens > 1) & (lens <= 512)).any())
    for m in _modes()[1:]:
        for a, b in zip(got[(1, 1)], got[m]):
            assert torch.equal(a, b)


def test_direct_binning_tile_overflow_reruns(cuda):
    """Direct binning gives every tile capacity / tiles slots in 8 replica
    segments: a capacity above the total but below what the longest segment
    needs must report the capacity it needs (meta[2]) and re-run to the
    same frame."""
    from paper_2312_02121_b200 import ops
    g = load_golden("cfg0_mini")
    t = _tensors(g["inputs"], cuda)
    cp = ops.CameraParams.of(g["camera"])
    ops.set_option("binning", 3)
    try:
        full = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True)
        tv = full.tensors()
        lens = tv["ranges"][:, 1] - tv["ranges"][:, 0]
        nt = lens.numel()
        need = full.needed_capacity  # tiles x 8 replica segments x the longest segment
        assert need % (8 * nt) == 0 and need >= nt * int(lens.max()) and need > full.n_isect
        raw = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True, capacity=need - 1, check_meta=False)
        m = raw.meta().cpu()
        assert int(m[0]) == -1 and int(m[1]) == full.n_isect and int(m[2]) == need
        small = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True, capacity=full.n_isect + 1)  # re-runs
        assert small.capacity >= need
        assert torch.equal(small.image, full.image)
        assert torch.equal(small.tensors()["sorted_vals"], tv["sorted_vals"])
    finally:
        ops.set_option("binning", 0)


def test_option_change_between_forward_and_backward(cuda):
    """The backward follows what its forward did (the raster order exists
    only for compact bins: meta[3]), not the options at backward time."""
    from paper_2312_02121_b200 import ops
    from paper_2312_02121_b200.scenes import make_config
    spec = make_config(1, n_views=1)  # 2500 tiles: more than one raster wave, so a raster order is used
    t = _tensors((spec.means, spec.scales, spec.quats, spec.opacities, spec.colors), cuda)
    cam = ops.CameraParams.of(spec.cameras[0])
    d = torch.as_tensor(np.asarray(spec.d_images[0], np.float32), device=cuda)
    ref = ops.frame_backward(ops.frame_forward(*t, cam, (0.0, 0.0, 0.0), True), t[0], t[1], t[2], t[4], d)
    try:
        for fwd_mode, bwd_mode in ((3, 2), (2, 3)):
            ops.set_option("binning", fwd_mode)
            fr = ops.frame_forward(*t, cam, (0.0, 0.0, 0.0), True)
            ops.set_option("binning", bwd_mode)
            g = ops.frame_backward(fr, t[0], t[1], t[2], t[4], d)
            for k in GRAD_CLASSES:
                r = runs_gate(g[k].cpu().numpy(), ref[k].cpu().numpy())
                assert r["ok"], (fwd_mode, bwd_mode, k, r)
    finally:
        ops.set_option("binning", 0)


def test_backward_accumulators_stay_clean(cuda):
    """The projection backward clears the screen-space accumulators as it
    reads them, so the next forward skips its zeroing pass; a workspace that
    is dirty (garbage, another layout, or a backward that kept its
    screen-space gradients) is re-zeroed by the forward (clean-word
    signature).  Every sequence must give the fresh-workspace gradients."""
    from paper_2312_02121_b200 import ops
    g = load_golden("config0")
    t = _tensors(g["inputs"], cuda)
    cp = ops.CameraParams.of(g["camera"])
    rng = np.random.default_rng(5)
    d = torch.as_tensor(rng.normal(size=(cp.height, cp.width, 3)).astype(np.float32), device=cuda)

    def grads(fr, **kw):
        out = ops.frame_backward(fr, t[0], t[1], t[2], t[4], d, **kw)
        torch.cuda.synchronize()
        return {k: out[k].clone() for k in ("d_mean", "d_scale", "d_quat", "d_rgbo")}

    def same(a, b):
        for k in a:
            # only the fp32 atomic order differs (a dirty accumulator would be off by O(1))
            r = runs_gate(a[k].cpu().numpy(), b[k].cpu().numpy(), rel=1e-4)
            assert r["ok"], (k, r)

    ref = grads(ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True))
    fr = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True)
    cap = fr.capacity
    same(grads(fr), ref)
    same(grads(fr), ref)  # a second backward of the same forward: the first left the rows zero
    same(grads(fr, keep_screen=True), ref)
    tv = fr.tensors()
    assert float(tv["d_geo"].abs().sum()) > 0  # kept readable
    fr2 = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True, capacity=cap, ws=fr.ws)  # forward re-zeroes
    same(grads(fr2), ref)
    assert float(fr2.tensors()["d_geo"].abs().sum()) == 0.0  # cleared by the projection backward
    # garbage workspace, marked not clean
    ws = ops.frame_workspace(t[0].shape[0], cap, cp.width, cp.height, cuda)
    ws.random_(0, 255)
    L = ops._lib.load()
    L.gs_frame_workspace_init(t[0].shape[0], cap, cp.width, cp.height, ws.data_ptr(), ops._stream())
    same(grads(ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True, capacity=cap, ws=ws)), ref)
    # the same workspace used for a smaller scene (another layout) and back
    m = t[0].shape[0] // 2
    half = [x[:m].contiguous() for x in t]
    frh = ops.frame_forward(*half, cp, (0.0, 0.0, 0.0), True, capacity=cap, ws=ws)
    ops.frame_backward(frh, half[0], half[1], half[2], half[4], d, keep_screen=True)
    same(grads(ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True, capacity=cap, ws=ws)), ref)


def test_skewed_view_falls_back_from_direct_binning(cuda):
    """direct binning sizes every tile's bin by the longest
    segment of any tile, so 80k Gaussians crowded into 4 of 4096 tiles would
    need ~82 M slots; the frame falls back to scatter binning (room = the pair
    count) and renders the same frame."""
    from paper_2312_02121_b200 import ops
    rng = np.random.default_rng(11)
    n = 80_000
    z = rng.uniform(3.0, 5.0, n)
    means = np.stack([rng.uniform(-0.02, 0.02, n) * z, rng.uniform(-0.02, 0.02, n) * z, z], 1)
    scales = np.full((n, 3), 0.002) * z[:, None]
    quats = rng.normal(size=(n, 4))
    t = _tensors((means, scales, quats, rng.uniform(0.05, 0.3, n), rng.uniform(0, 1, (n, 3))), cuda)
    cp = ops.CameraParams(np.eye(4).tolist(), 400.0, 400.0, 512.0, 512.0, 1024, 1024, 0.01, 100.0)  # 4096 tiles
    assert ops.frame_binning(n, cp) == "direct"
    fr = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True)
    assert fr.binning == "scatter" and fr.capacity <= 2 * fr.n_isect + (1 << 16), (fr.capacity, fr.n_isect)
    ref = ops.frame_forward(*t, cp, (0.0, 0.0, 0.0), True, binning="depth_first")
    assert torch.equal(fr.image, ref.image) and torch.equal(fr.n_contrib, ref.n_contrib)
    d = torch.ones((cp.height, cp.width, 3), device=cuda)
    ga = ops.frame_backward(fr, t[0], t[1], t[2], t[4], d)
    gb = ops.frame_backward(ref, t[0], t[1], t[2], t[4], d)
    for k in ("d_mean", "d_rgbo"):
        r = runs_gate(ga[k].cpu().numpy(), gb[k].cpu().numpy())
        assert r["ok"], (k, r)
