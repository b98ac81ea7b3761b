"""GPU: the fit step around the hot path (sg/optimize.py) -- loss history vs
an fp64 restatement of the same loop on the oracle, and the reference's
acceptance criterion 5 (100-splat 64x64 fit cuts the loss by >= 95%,
tests/test_acceptance.py:219-263)."""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _hidden_scene(api):
    # the scene criterion 5 fits (same distributions as the reference test, own code)
    rng = np.random.default_rng(42)
    camera = api.Camera(view=np.eye(4), fx=64.0, fy=64.0, cx=31.5, cy=31.5, width=64, height=64, near=0.1, far=100.0)
    scene = []
    for _ in range(100):
        px, py = rng.uniform(4.0, 60.0), rng.uniform(4.0, 60.0)
        depth = rng.uniform(2.0, 6.0)
        mean = np.array([(px - camera.cx) * depth / camera.fx, (py - camera.cy) * depth / camera.fy, depth])
        scale = rng.uniform(1.5, 4.0, size=3) * depth / camera.fx
        scene.append(api.Gaussian3D(mean=mean, scale=scale, quat=rng.normal(size=4),
                                    opacity=float(rng.uniform(0.4, 0.9)), color=rng.uniform(0.0, 1.0, size=3)))
    return scene, camera


def _arrays(scene):
    return (np.array([g.mean for g in scene]), np.array([g.scale for g in scene]), np.array([g.quat for g in scene]),
            np.array([g.opacity for g in scene]), np.array([g.color for g in scene]))


def _oracle_fit(target, camera, config, init, iterations):
    """fp64 restatement of sg/optimize.py:96-190 on the oracle (test only)."""
    ocam = O.Camera(camera.view, camera.fx, camera.fy, camera.cx, camera.cy, camera.width, camera.height, camera.near,
                    camera.far)
    means, scales, quats, opac, colors = [np.asarray(a, np.float64) for a in _arrays(init)]
    log_s = np.log(scales)
    op = np.clip(opac, 1e-4, 1 - 1e-4)
    logits = np.log(op) - np.log1p(-op)
    state = {k: [np.zeros_like(p), np.zeros_like(p)] for k, p in
             (("m", means), ("s", log_s), ("q", quats), ("o", logits), ("c", colors))}
    bg = np.asarray(config.background, np.float64)

    def adam(p, g, k, lr, step):
        m, v = state[k]
        m[...] = config.beta1 * m + (1 - config.beta1) * g
        v[...] = config.beta2 * v + (1 - config.beta2) * g * g
        mh, vh = m / (1 - config.beta1 ** step), v / (1 - config.beta2 ** step)
        return p - lr * mh / (np.sqrt(vh) + config.eps)

    hist = []
    for it in range(iterations):
        s = np.exp(log_s)
        o = 1 / (1 + np.exp(-logits))
        fw = O.render(means, s, quats, o, colors, ocam, bg, True)
        resid = fw["image"] - target
        hist.append(float(np.sum(resid * resid)))
        g = O.scene_backward(means, s, quats, o, colors, ocam, bg, fw, 2 * resid)
        step = it + 1
        means = adam(means, g["d_mean"], "m", config.lr_mean, step)
        log_s = adam(log_s, g["d_scale"] * s, "s", config.lr_scale, step)
        quats = adam(quats, g["d_quat"], "q", config.lr_quat, step)
        logits = adam(logits, g["d_opacity"] * o * (1 - o), "o", config.lr_opacity, step)
        colors = np.clip(adam(colors, g["d_color"], "c", config.lr_color, step), 0, 1)
    return hist


def test_fit_loss_history_matches_oracle(cuda):
    from paper_2312_02121_b200 import api, fitting as F
    truth, camera = _hidden_scene(api)
    bg = (0.1, 0.1, 0.1)
    target = api.render(truth, camera, np.asarray(bg)).image.channels
    config = F.FitConfig(n_gaussians=100, iterations=20, background=bg, seed=0)
    init = F.init_random(config, camera, target)
    _, hist = F.fit(target, camera, config, init=init)
    ref = _oracle_fit(target, camera, config, init, 20)
    np.testing.assert_allclose(hist[0], ref[0], rtol=1e-4)
    # Adam normalises steps, so fp32/fp64 trajectories separate slowly; the
    # loss curve must track the fp64 one closely over the first iterations
    np.testing.assert_allclose(hist, ref, rtol=2e-2)


def test_fit_criterion5_loss_cut(cuda):
    from paper_2312_02121_b200 import api, fitting as F
    truth, camera = _hidden_scene(api)
    bg = (0.1, 0.1, 0.1)
    target = api.render(truth, camera, np.asarray(bg)).image.channels
    config = F.FitConfig(n_gaussians=100, iterations=1000, background=bg, seed=0)
    scene, history = F.fit(target, camera, config)
    history = np.asarray(history)
    reduction = 1.0 - history[-1] / history[0]
    smoothed = np.convolve(history, np.ones(50) / 50.0, mode="valid")
    drift = float(np.max(np.diff(smoothed)))
    print(f"fit: loss {history[0]:.2f} -> {history[-1]:.2f} ({100 * reduction:.1f}% cut), smoothed drift {drift:.1e}")
    assert reduction >= 0.95
    # The reference holds the 50-iteration moving average to drift <= 1e-9
    # (fp64, deterministic).  On the fp32 path the gradient sums use atomics,
    # so the plateau of the curve carries fp32 noise: non-increasing up to
    # 1e-5 of the initial loss.
    assert drift <= 1e-5 * history[0]
    assert len(scene) == 100 and all(0.0 <= g.opacity <= 1.0 for g in scene)


def test_fit_rejects_bad_target(cuda):
    from paper_2312_02121_b200 import api, fitting as F
    _, camera = _hidden_scene(api)
    with pytest.raises(ValueError, match="target shape"):
        F.fit(np.zeros((10, 10, 3)), camera, F.FitConfig(iterations=1))
    with pytest.raises(ValueError, match="unsupported loss"):
        F.fit(np.zeros((64, 64, 3)), camera, F.FitConfig(iterations=1, loss="l1"))
