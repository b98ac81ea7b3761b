"""GPU: the per-pixel API (eval_alpha, composite_pixel,
composite_pixel_backward, transmittance_replay).

* against the reference's own outputs (tests/golden/pixel.npz, made by
  make_golden_pixel.py), with fp32-vs-fp64 branch flips classified by the
  oracle's decision margins (tests/parity.py FLIP_EPS);
* against the tile rasterizers: a query at a rendered pixel's centre with
  its tile's bin reproduces image / final_T / n_contrib BIT FOR BIT, and the
  per-pixel backward summed over the queried pixels equals the tile backward
  for a d_image supported on those pixels (up to fp32 summation order);
* the reference's per-pixel KATs (tests/test_forward.py:48-216,
  tests/test_backward_raster.py:50-98) through api.* with fp32 tolerances.

Tolerances (fp32 path vs fp64 reference): sigma rel 1e-5 + 1e-6 abs; alpha
and colour 1e-5 abs (north star 1e-4); transmittance replay rel 2e-4 (the
clamp value 0.999 is not representable: 1 - 0.999f differs from 1 - 0.999 by
1.3e-5 relative per clamped splat); gradients tests/parity.py grad_gate
(rel-L2 1e-3 + per-element floor).
"""

import numpy as np
import pytest
import torch

import oracle as O
from parity import FLIP_EPS, grad_gate, load_golden, load_pixel_golden

pytestmark = pytest.mark.gpu


def _t(a, dev, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a), device=dev).to(dtype)


def _np(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def gold(cuda):
    from paper_2312_02121_b200 import pixels
    z = load_pixel_golden()
    m = len(z["source_index"])
    xydr = np.zeros((m, 4), np.float32)
    xydr[:, :2] = z["mean2d"]
    conic = pixels.conic_from_cov(_t(z["cov3"], cuda), _t(z["p_opacity"], cuda))
    return z, _t(xydr, cuda), conic, _t(z["p_color"], cuda)


def test_eval_alpha_vs_reference(gold, cuda):
    from paper_2312_02121_b200 import pixels
    z = gold[0]
    n = len(z["ea_opacity"])
    xydr = np.zeros((n, 4), np.float32)
    xydr[:, :2] = z["ea_mean2d"]
    conic = pixels.conic_from_cov(_t(z["ea_cov3"], cuda), _t(z["ea_opacity"], cuda))
    alpha, delta, sigma = pixels.eval_alpha(_t(xydr, cuda), conic, _t(np.arange(n), cuda, torch.int32),
                                            _t(z["ea_pix"], cuda))
    ref = z["ea_out"]
    np.testing.assert_allclose(_np(delta), ref[:, 1:3], rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(_np(sigma), ref[:, 3], rtol=1e-5, atol=1e-6)
    araw = z["ea_opacity"] * np.exp(-ref[:, 3])
    safe = ((np.abs(ref[:, 3] - 4.5) / 4.5 >= FLIP_EPS) & (np.abs(araw - 1 / 255) * 255 >= FLIP_EPS)
            & (np.abs(araw - 0.999) / 0.999 >= FLIP_EPS))
    assert safe.mean() > 0.9
    np.testing.assert_allclose(_np(alpha)[safe], ref[safe, 0], rtol=0, atol=1e-5)
    assert np.array_equal(_np(alpha)[safe] == 0, ref[safe, 0] == 0)


def _safe_queries(z):
    o = O.composite_pixels(z["bin_ptr"], z["bin_idx"], z["q_pix"], z["q_et"], z["mean2d"], z["cov3"],
                           z["p_opacity"], z["p_color"], z["background"])
    return o["margin"] >= FLIP_EPS


def test_composite_pixel_vs_reference(gold, cuda):
    from paper_2312_02121_b200 import pixels
    z, xydr, conic, colors = gold
    safe = _safe_queries(z)
    assert safe.mean() > 0.8
    colors_out, T, nc = [], [], []
    for et in (0, 1):  # the fixture mixes early-termination flags per query
        c, t, n = pixels.composite_pixels(xydr, conic, colors, z["bin_ptr"], z["bin_idx"], _t(z["q_pix"], cuda),
                                          z["background"], bool(et))
        colors_out.append(_np(c)), T.append(_np(t)), nc.append(_np(n))
    pick = z["q_et"].astype(bool)
    col = np.where(pick[:, None], colors_out[1], colors_out[0])
    T = np.where(pick, T[1], T[0])
    nc = np.where(pick, nc[1], nc[0])
    assert np.array_equal(nc[safe], z["q_nc"][safe])
    np.testing.assert_allclose(col[safe], z["q_color"][safe], rtol=0, atol=1e-5)
    np.testing.assert_allclose(T[safe], z["q_T"][safe], rtol=1e-4, atol=1e-7)


def test_composite_backward_and_replay_vs_reference(gold, cuda):
    from paper_2312_02121_b200 import pixels
    z, xydr, conic, colors = gold
    safe = _safe_queries(z)
    src = z["source_index"]
    got = {k: [] for k in ("c", "o", "m", "v")}
    ref = {k: [] for k in ("c", "o", "m", "v")}
    for q in np.nonzero(safe)[0]:
        sl = slice(int(z["bin_ptr"][q]), int(z["bin_ptr"][q + 1]))
        ptr = np.array([0, sl.stop - sl.start])
        d_rgbo, d_geo, d_c11, t_log = pixels.composite_pixels_backward(
            xydr, conic, colors, ptr, z["bin_idx"][sl], _t(z["q_pix"][q:q + 1], cuda), z["background"],
            _t(z["q_T"][q:q + 1], cuda), _t(z["q_nc"][q:q + 1], cuda, torch.int32), _t(z["d_pix"][q:q + 1], cuda),
            want_t_log=True)
        rgbo, geo, c11 = _np(d_rgbo), _np(d_geo), _np(d_c11)
        # projected row j -> scene row src[j]
        got["c"].append(rgbo[:, :3]), ref["c"].append(z["g_color"][q][src])
        got["o"].append(rgbo[:, 3]), ref["o"].append(z["g_opacity"][q][src])
        got["m"].append(geo[:, :2]), ref["m"].append(z["g_mean2d"][q][src])
        got["v"].append(np.stack([geo[:, 2], geo[:, 3], c11], 1))
        ref["v"].append(z["g_cov2d"][q][src].reshape(-1, 4)[:, [0, 1, 3]])
        t = _np(t_log)
        pairs = [(p, t[p]) for p in range(len(t) - 1, -1, -1) if np.isfinite(t[p])]
        r = slice(int(z["r_ptr"][q]), int(z["r_ptr"][q + 1]))
        assert [p for p, _ in pairs] == z["r_pos"][r].tolist()
        if pairs:
            np.testing.assert_allclose([v for _, v in pairs], z["r_T"][r], rtol=2e-4)
    for k in got:
        r = grad_gate(np.concatenate(got[k]), np.concatenate(ref[k]))
        assert r["ok"], (k, r)


@pytest.fixture(scope="module")
def frame(cuda):
    from paper_2312_02121_b200 import ops
    g = load_golden("config0")
    t = [_t(a, cuda) for a in g["inputs"]]
    cam = ops.CameraParams.of(g["camera"])
    image, st = ops.render_forward(*t, cam, tuple(g["background"]), g["et"], want_cov=True)
    torch.cuda.synchronize()
    return g, t, cam, image, st


def _tile_queries(cam, st, per_tile, seed):
    """`per_tile` random pixels of every tile, each with its tile's bin."""
    rng = np.random.default_rng(seed)
    ranges = _np(st.bins.ranges).astype(np.int64)
    vals = _np(st.bins.sorted_vals).astype(np.int64)
    rows, cols, ptr, idx = [], [], [0], []
    for tile in range(cam.tiles_x * cam.tiles_y):
        ty, tx = divmod(tile, cam.tiles_x)
        for _ in range(per_tile):
            r = min(cam.height - 1, ty * 16 + int(rng.integers(0, 16)))
            c = min(cam.width - 1, tx * 16 + int(rng.integers(0, 16)))
            rows.append(r), cols.append(c)
            idx.append(vals[ranges[tile, 0]:ranges[tile, 1]])
            ptr.append(ptr[-1] + len(idx[-1]))
    rows, cols = np.array(rows), np.array(cols)
    pix = np.stack([cols + 0.5, rows + 0.5], 1).astype(np.float32)
    return rows, cols, pix, np.array(ptr, np.int64), np.concatenate(idx)


def test_queries_reproduce_the_frame_bitwise(frame, cuda):
    from paper_2312_02121_b200 import pixels
    g, (m, s, q, o, c), cam, image, st = frame
    rows, cols, pix, ptr, idx = _tile_queries(cam, st, 6, 0)
    # the conic rebuilt from the projected covariance equals the projection's own
    vis = st.proj.tiles > 0
    conic = pixels.conic_from_cov(st.proj.cov2d[vis].contiguous(), o[vis].contiguous())
    assert torch.equal(conic, st.proj.conic[vis])
    color, T, nc = pixels.composite_pixels(st.proj.xydr, st.proj.conic, c, ptr, idx, _t(pix, cuda),
                                           st.background, st.early_termination)
    img = _np(image)
    assert np.array_equal(_np(color), img[rows, cols])
    assert np.array_equal(_np(T), _np(st.final_T)[rows, cols])
    assert np.array_equal(_np(nc), _np(st.n_contrib)[rows, cols])

    # backward: d_image supported on the queried pixels (unique ones)
    from paper_2312_02121_b200 import ops
    _, first = np.unique(rows * cam.width + cols, return_index=True)
    slices = [idx[ptr[k]:ptr[k + 1]] for k in first]
    rows, cols, pix = rows[first], cols[first], pix[first]
    ptr = np.concatenate([[0], np.cumsum([len(x) for x in slices])]).astype(np.int64)
    idx = np.concatenate(slices)
    rng = np.random.default_rng(1)
    d_pix = rng.normal(size=(len(rows), 3)).astype(np.float32)
    d_image = np.zeros((cam.height, cam.width, 3), np.float32)
    d_image[rows, cols] = d_pix
    d_rgbo, d_geo, d_c11 = ops.raster_bwd(st, c, _t(d_image, cuda))
    p_rgbo, p_geo, p_c11, _ = pixels.composite_pixels_backward(
        st.proj.xydr, st.proj.conic, c, ptr, idx, _t(pix, cuda), st.background, st.final_T[rows, cols].contiguous(),
        st.n_contrib[rows, cols].contiguous(), _t(d_pix, cuda))
    for a, b in ((p_rgbo, d_rgbo), (p_geo, d_geo), (p_c11, d_c11)):
        r = grad_gate(_np(a), _np(b), rel=1e-4, floor=1e-2)  # summation order only
        assert r["ok"], r


# ---- reference KATs through api.* (tests/test_forward.py, test_backward_raster.py)

def _splat2d(api, mean, cov, src=0):
    return api.ProjectedGaussian(t_cam=np.array([0.0, 0.0, 1.0]), mean2d=np.asarray(mean, np.float64),
                                 cov2d=np.asarray(cov, np.float64), depth=1.0, radius=3, source_index=src)


def _g3(api, opacity, color):
    return api.Gaussian3D(mean=np.zeros(3), scale=np.ones(3), quat=np.array([1.0, 0, 0, 0]), opacity=opacity,
                          color=np.asarray(color, np.float64))


def test_api_eval_alpha_kats(cuda):
    from paper_2312_02121_b200 import api
    g = _splat2d(api, [3.5, 7.5], np.eye(2))
    a, d, s = api.eval_alpha(g, 0.7, np.array([3.5, 7.5]))
    assert s == 0.0 and np.all(d == 0.0) and a == np.float32(0.7)
    g = _splat2d(api, [0.0, 0.0], np.eye(2))
    a, d, s = api.eval_alpha(g, 1.0, np.array([1.0, 0.0]))
    assert abs(s - 0.5) < 1e-7 and abs(a - np.exp(-0.5)) < 1e-6
    assert api.eval_alpha(g, 1.0, np.array([4.0, 0.0]))[0] == 0.0      # sigma 8 > cutoff
    assert api.eval_alpha(g, 1e-5, np.array([0.0, 0.0]))[0] == 0.0     # below ALPHA_MIN
    assert api.eval_alpha(g, 1.0, np.array([0.0, 0.0]))[0] == np.float32(api.ALPHA_MAX)
    with pytest.raises(ValueError, match="not invertible"):
        api.eval_alpha(_splat2d(api, [0, 0], [[1.0, 1.0], [1.0, 1.0]]), 0.5, np.array([0.0, 0.0]))


def test_api_composite_kats(cuda):
    from paper_2312_02121_b200 import api
    px = np.array([0.5, 0.5])
    bg = np.array([0.1, 0.2, 0.3])
    color, aux = api.composite_pixel([], [], [], px, bg)
    assert np.allclose(color, bg) and aux == api.PixelAux(1.0, 0)
    p = [_splat2d(api, px, np.eye(2) * 4.0, 0), _splat2d(api, px, np.eye(2) * 4.0, 1)]
    scene = [_g3(api, 0.5, [1.0, 0.0, 0.0]), _g3(api, 0.5, [0.0, 1.0, 0.0])]
    color, aux = api.composite_pixel([0], p, scene, px, np.zeros(3))
    assert np.allclose(color, [0.5, 0, 0]) and aux.final_T == 0.5 and aux.n_contrib == 1
    color, aux = api.composite_pixel([0, 1], p, scene, px, np.zeros(3))
    assert np.allclose(color, [0.5, 0.25, 0]) and aux.final_T == 0.25 and aux.n_contrib == 2
    # a skipped (too faint) splat is not counted
    faint = [_g3(api, 1e-4, [1, 1, 1]), _g3(api, 0.5, [0.0, 1.0, 0.0])]
    color, aux = api.composite_pixel([0, 1], p, faint, px, np.zeros(3))
    assert aux.n_contrib == 2 and np.allclose(color, [0, 0.5, 0])
    # early stop: the stopping splat is not composited
    dense = [_splat2d(api, px, np.eye(2) * 4.0, i) for i in range(3)]
    opaque = [_g3(api, 1.0, [1, 0, 0]), _g3(api, 1.0, [0, 1, 0]), _g3(api, 1.0, [0, 0, 1])]
    _, aux = api.composite_pixel([0, 1, 2], dense, opaque, px, np.zeros(3))
    assert aux.n_contrib == 1 and abs(aux.final_T - 1e-3) < 1e-7
    _, aux = api.composite_pixel([0, 1, 2], dense, opaque, px, np.zeros(3), early_termination=False)
    assert aux.n_contrib == 3


def test_api_backward_and_replay_kats(cuda):
    from paper_2312_02121_b200 import api
    px = np.array([0.5, 0.5])
    p = [_splat2d(api, px, np.eye(2) * 4.0, 0)]
    scene = [_g3(api, 0.5, [1.0, 0.0, 0.0])]
    _, aux = api.composite_pixel([0], p, scene, px, np.zeros(3))
    gr = api.composite_pixel_backward([0], p, scene, px, np.zeros(3), aux, np.ones(3))
    np.testing.assert_allclose(gr.d_color[0], [0.5, 0.5, 0.5], rtol=1e-6)
    np.testing.assert_allclose(gr.d_opacity[0], 1.0, rtol=1e-6)
    np.testing.assert_allclose(gr.d_mean2d[0], [0.0, 0.0], atol=1e-7)
    _, aux1 = api.composite_pixel([0], p, scene, px, np.ones(3))
    gr = api.composite_pixel_backward([0], p, scene, px, np.ones(3), aux1, np.ones(3))
    np.testing.assert_allclose(gr.d_opacity[0], -2.0, rtol=1e-6)
    # replay order back to front, T before the front splat exactly 1
    p3 = [_splat2d(api, px, np.eye(2) * 4.0, i) for i in range(3)]
    s3 = [_g3(api, 0.5, [1, 0, 0]) for _ in range(3)]
    _, aux = api.composite_pixel([0, 1, 2], p3, s3, px, np.zeros(3))
    pairs = api.transmittance_replay([0, 1, 2], p3, s3, px, np.zeros(3), aux)
    assert [q for q, _ in pairs] == [2, 1, 0]
    assert dict(pairs)[0] == 1.0


def test_api_replay_matches_forward_walk(cuda):
    """Acceptance criterion 3 (tests/test_acceptance.py:95-130) on the GPU
    path: the replayed T equals the forward T recomputed by walking the bin
    with eval_alpha, within the fp32 tolerance (rel 2e-4)."""
    from paper_2312_02121_b200 import api
    g = load_golden("cfg0_mini")
    m, s, q, o, c = g["inputs"]
    scene = [api.Gaussian3D(mean=m[i], scale=s[i], quat=q[i], opacity=o[i], color=c[i]) for i in range(len(m))]
    cam = g["camera"]
    camera = api.Camera(view=cam.view, fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, width=cam.width,
                        height=cam.height, near=cam.near, far=cam.far)
    res = api.render(scene, camera, g["background"])
    rng = np.random.default_rng(3)
    checked = 0
    for _ in range(24):
        row, col = int(rng.integers(0, cam.height)), int(rng.integers(0, cam.width))
        sbin = res.grid.bin_at(col // 16, row // 16)
        px = np.array([col + 0.5, row + 0.5])
        aux = api.PixelAux(float(res.aux.final_T[row, col]), int(res.aux.n_contrib[row, col]))
        pairs = api.transmittance_replay(sbin, res.projected, scene, px, g["background"], aux)
        t, fwd = 1.0, {}
        for pos, idx in enumerate(sbin):
            if pos >= aux.n_contrib:
                break
            p = res.projected[idx]
            alpha, _, _ = api.eval_alpha(p, scene[p.source_index].opacity, px)
            if alpha == 0.0:
                continue
            fwd[pos] = t
            t *= 1.0 - alpha
        assert len(pairs) == len(fwd)
        for pos, tr in pairs:
            assert abs(tr - fwd[pos]) <= 2e-4 * fwd[pos]
            checked += 1
    assert checked > 0
