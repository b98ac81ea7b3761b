"""GPU parity at BASELINE sizes (configs 0-4), SURVEY.md §8c stage isolation.

Full-frame oracle comparisons at configs 0-1; at configs 2-4 the oracle runs
stage-isolated on samples: projection on a random subset of Gaussians, bins
on the GPU's own projection (bit-exact), compositing and its backward on a
random ~2% of tiles (all other tiles' bins emptied and their d_image zeroed
on both sides), projection backward on those screen-space gradients.  Plus
size-independent properties of the full frame.
"""

import numpy as np
import pytest
import torch

import oracle as O
from parity import FLIP_EPS, classify_image, grad_gate, projection_diffs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _frame(spec, view, dev):
    from paper_2312_02121_b200 import ops
    t = lambda a: torch.as_tensor(a, device=dev)
    m, s, q, o, c = t(spec.means), t(spec.scales), t(spec.quats), t(spec.opacities), t(spec.colors)
    cam = ops.CameraParams.of(spec.cameras[view])
    image, st = ops.render_forward(m, s, q, o, c, cam, (0.0, 0.0, 0.0), True, want_cov=True)
    torch.cuda.synchronize()
    return (m, s, q, o, c), cam, image, st


def _np(t):
    return t.detach().cpu().numpy()


def _gpu_proj(st):
    xydr = _np(st.proj.xydr)
    return dict(visible=(_np(st.proj.tiles) > 0).astype(np.int8), mean2d=xydr[:, :2].astype(np.float64),
                depth=xydr[:, 2].astype(np.float64), radius=xydr[:, 3].copy().view(np.int32).astype(np.int64),
                cov2d=_np(st.proj.cov2d).astype(np.float64))


def _csr(st, n_tiles):
    r = _np(st.bins.ranges).astype(np.int64)
    cnt = r[:, 1] - r[:, 0]
    ptr = np.concatenate([[0], np.cumsum(cnt)])
    return ptr, _np(st.bins.sorted_vals).astype(np.int64)


@pytest.mark.parametrize("config,view", [(2, 0), (3, 5), (4, 0)])
def test_config_stage_isolated(config, view, cuda):
    from paper_2312_02121_b200 import ops
    from paper_2312_02121_b200.scenes import make_config
    spec = make_config(config, n_views=view + 1)
    f64 = lambda a: np.asarray(a, np.float64)
    (m, s, q, o, c), cam, image, st = _frame(spec, view, cuda)
    ocam = O.Camera.of(spec.cameras[view])
    n = spec.n
    g = _gpu_proj(st)
    rng = np.random.default_rng(config)

    # --- projection on a random sample of Gaussians
    sample = np.sort(rng.choice(n, size=min(n, 200_000), replace=False))
    pr = O.project(f64(spec.means)[sample], f64(spec.scales)[sample], f64(spec.quats)[sample], ocam)
    gs = {k: v[sample] for k, v in g.items()}
    d = projection_diffs(gs, pr)
    assert d["n_vis_diff"] <= max(3, 1e-4 * len(sample)), d
    assert d["n_radius_diff"] <= max(5, 1e-4 * len(sample)), d
    assert all(c[0] in ("radius-ceil", "visibility") for c in d["causes"])
    assert d["cov2d_max_rel"] < 1e-3, d

    # --- bins: bit-exact against the oracle fed the GPU's fp32 projection
    n_tiles = cam.tiles_x * cam.tiles_y
    ptr, idx = _csr(st, n_tiles)
    optr, oidx = O.bin_tiles(g["visible"], g["mean2d"], g["radius"], g["depth"], cam.width, cam.height)
    assert np.array_equal(ptr, optr) and np.array_equal(idx, oidx)

    # --- compositing on ~2% of tiles (others emptied), then its backward
    tiles = np.sort(rng.choice(n_tiles, size=max(8, n_tiles // 50), replace=False))
    keep = np.zeros(n_tiles, bool)
    keep[tiles] = True
    cnt = np.where(keep, np.diff(ptr), 0)
    sptr = np.concatenate([[0], np.cumsum(cnt)])
    sidx = np.concatenate([idx[ptr[t]:ptr[t + 1]] for t in tiles]) if len(tiles) else np.zeros(0, np.int64)
    fw = O.raster_fwd(cam.width, cam.height, sptr, sidx, g["mean2d"], g["cov2d"], f64(spec.opacities),
                      f64(spec.colors), np.zeros(3), True, margins=True)
    pix = np.zeros((cam.height, cam.width), bool)
    for t in tiles:
        ty, tx = divmod(int(t), cam.tiles_x)
        pix[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = True
    img = _np(image).astype(np.float64)
    cls = classify_image(img[pix], fw["image"][pix], fw["margin"][pix], fw["margin_kind"][pix])
    print(f"config{config}: tiles {len(tiles)}, max err {cls['max_err']:.2e}, safe {cls['max_err_safe']:.2e}, "
          f"flips {cls['n_flip']} {cls['flip_kinds']}")
    assert cls["n_real"] == 0, cls
    safe = pix & (fw["margin"] >= FLIP_EPS)
    assert np.array_equal(_np(st.n_contrib)[safe], fw["n_contrib"][safe])

    d_image = np.asarray(spec.d_images[view], np.float64) * safe[..., None]
    d_image = d_image.astype(np.float32)
    gg = ops.render_backward(st, m, s, q, c, torch.as_tensor(d_image, device=cuda))
    rb = O.raster_bwd(cam.width, cam.height, sptr, sidx, g["mean2d"], g["cov2d"], f64(spec.opacities),
                      f64(spec.colors), np.zeros(3), fw["final_T"], fw["n_contrib"], d_image.astype(np.float64))
    geo = _np(gg["d_geo"]).astype(np.float64)
    # gate on the Gaussians the sampled tiles hold (rms over those, not the
    # mostly-zero full arrays); everything else must be exactly zero
    touched = np.unique(sidx)
    rest = np.ones(n, bool)
    rest[touched] = False
    for name, got, ref in (("d_color", _np(gg["d_color"]), rb["d_color"]),
                           ("d_opacity", _np(gg["d_opacity"]), rb["d_opacity"]),
                           ("d_mean2d", geo[:, :2], rb["d_mean2d"])):
        r = grad_gate(got[touched], ref[touched])
        assert r["ok"], (config, name, r)
        assert not np.any(got[rest]), name
    pb = O.project_bwd(f64(spec.means)[touched], f64(spec.scales)[touched], f64(spec.quats)[touched], ocam,
                       np.ones(len(touched), np.int8),
                       O.project(f64(spec.means)[touched], f64(spec.scales)[touched], f64(spec.quats)[touched],
                                 ocam)["t_cam"],
                       rb["d_mean2d"][touched], rb["d_cov2d"][touched].reshape(-1, 4))
    for name in ("d_mean", "d_scale", "d_quat"):
        r = grad_gate(_np(gg[name])[touched], pb[name])
        assert r["ok"], (config, name, r)


@pytest.mark.parametrize("config", [2, 4])
def test_full_frame_properties(config, cuda):
    from paper_2312_02121_b200 import ops
    from paper_2312_02121_b200.scenes import make_config
    spec = make_config(config)
    (m, s, q, o, c), cam, image, st = _frame(spec, 0, cuda)
    n_tiles = cam.tiles_x * cam.tiles_y
    keys = st.bins.sorted_keys
    tiles = (keys >> 32)
    assert bool((tiles[1:] >= tiles[:-1]).all())
    same = tiles[1:] == tiles[:-1]
    dep = (keys & 0xFFFFFFFF)
    assert bool(((dep[1:] >= dep[:-1]) | ~same).all())  # depth ascending within a tile
    r = st.bins.ranges.long()
    cnt = r[:, 1] - r[:, 0]
    assert int(cnt.sum()) == st.bins.n_isect == int(st.proj.tiles.long().sum())
    nc = st.n_contrib.long()
    T = st.final_T
    assert float(T.max()) <= 1.0 and float(T.min()) > 0.0
    assert bool((nc >= 0).all())
    # n_contrib never exceeds the pixel's bin length
    H, W = cam.height, cam.width
    tile_of = (torch.arange(H, device=cuda)[:, None] // 16) * cam.tiles_x + torch.arange(W, device=cuda)[None] // 16
    assert bool((nc <= cnt[tile_of]).all())
    assert float(image.min()) >= 0.0 and float(image.max()) <= 1.0 + 1e-5
    # the frame path renders the same frame bit for bit
    fr = ops.frame_forward(m, s, q, o, c, cam, (0.0, 0.0, 0.0), True)
    assert torch.equal(fr.image, image) and torch.equal(fr.n_contrib, st.n_contrib)
