"""Generate golden fixtures by running the REAL reference (splatgrad) here.

Run in the build container only (``/root/reference`` is absent on the GPU
box):  ``python tests/golden/make_golden.py``.  The fixtures it writes
(``tests/golden/*.npz``) are committed; tests never import the reference.

Each fixture stores fp32-exact inputs (generated in fp64, rounded to fp32 so
the GPU path and the fp64 oracle see identical values), the reference's
``render`` outputs (``sg/raster_forward.py:255-271``), its sorted tile bins
(``sg/binning.py:27-65``) re-expressed as CSR over *scene* indices, its
``accumulate_image_backward`` screen-space gradients
(``sg/raster_backward.py:166-205``) and its ``scene_backward`` gradients
(``sg/proj_backward.py:178-223``).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


def _f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def _view_from_quat(q, t):
    import splatgrad as sg
    v = np.eye(4)
    v[:3, :3] = sg.quat_to_rotmat(q)
    v[:3, 3] = t
    return v


def _frustum_scene(rng, n, cam, depth_range=(2.0, 8.0), scale_px=(1.0, 3.0),
                   opacity=(0.2, 0.95)):
    """Splats back-projected onto visible pixels (same idea as the
    reference's tests/helpers.py frustum_scene, written independently)."""
    R = cam["view"][:3, :3]
    t = cam["view"][:3, 3]
    px = rng.uniform(1.0, cam["width"] - 1.0, size=n)
    py = rng.uniform(1.0, cam["height"] - 1.0, size=n)
    z = rng.uniform(*depth_range, size=n)
    tc = np.stack([(px - 0.5 - cam["cx"]) * z / cam["fx"],
                   (py - 0.5 - cam["cy"]) * z / cam["fy"], z], axis=1)
    means = (tc - t) @ R  # R^T (tc - t)
    scales = rng.uniform(*scale_px, size=(n, 3)) * (z / cam["fx"])[:, None]
    quats = rng.normal(size=(n, 4))
    opac = rng.uniform(*opacity, size=n)
    colors = rng.uniform(0.0, 1.0, size=(n, 3))
    return means, scales, quats, opac, colors


def _camera(width, height, fx=None, view=None, near=0.1, far=100.0, cx=None, cy=None):
    fx = float(max(width, height)) if fx is None else fx
    return dict(
        view=np.eye(4) if view is None else view, fx=fx, fy=fx,
        cx=(width - 1) / 2.0 if cx is None else cx,
        cy=(height - 1) / 2.0 if cy is None else cy,
        width=width, height=height, near=near, far=far,
    )


def build_cases():
    cases = {}
    # 1. rotated camera, non-zero background, ragged edge tiles (37x29)
    rng = np.random.default_rng(1001)
    cam = _camera(37, 29)
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    ang = 0.25
    q = np.concatenate([[np.cos(ang / 2)], np.sin(ang / 2) * axis])
    cam["view"] = _view_from_quat(q, rng.uniform(-0.2, 0.2, size=3))
    cases["rot_ragged"] = (cam, _frustum_scene(rng, 60, cam), rng.uniform(0, 1, 3), True)
    # 2. dense, high opacity -> heavy early termination; forced depth ties
    rng = np.random.default_rng(1002)
    cam = _camera(48, 32)
    m, s, qq, o, c = _frustum_scene(rng, 140, cam, opacity=(0.6, 0.99), scale_px=(2.0, 5.0))
    # exact depth ties: copy z of earlier splats (identity view => depth = z)
    m[30:40, 2] = m[0:10, 2]
    cases["dense_ties"] = (cam, (m, s, qq, o, c), np.zeros(3), True)
    # 3. same dense scene without early termination
    cases["dense_noet"] = (cam, (m, s, qq, o, c), np.array([0.1, 0.2, 0.3]), False)
    # 4. culling: behind camera, beyond far, off-screen, plus visible ones
    rng = np.random.default_rng(1003)
    cam = _camera(32, 32, near=0.5, far=20.0)
    m, s, qq, o, c = _frustum_scene(rng, 30, cam)
    m[0] = [0.0, 0.0, -3.0]        # behind
    m[1] = [0.0, 0.0, 0.3]         # inside near
    m[2] = [0.0, 0.0, 25.0]        # beyond far
    m[3] = [40.0, 0.0, 3.0]        # far off to the side
    m[4] = [-40.0, 5.0, 3.0]
    cases["culling"] = (cam, (m, s, qq, o, c), np.array([0.5, 0.5, 0.5]), True)
    # 5. config-0 distributions, scaled down (1500 splats, 80x64, off-centre pp)
    rng = np.random.default_rng(1004)
    n = 1500
    means = rng.uniform(-1.0, 1.0, size=(n, 3))
    scales = np.exp(rng.uniform(np.log(0.005), np.log(0.05), size=(n, 3)))
    quats = rng.normal(size=(n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    opac = 1.0 / (1.0 + np.exp(-rng.normal(size=n)))
    colors = rng.uniform(0, 1, size=(n, 3))
    view = np.eye(4)
    view[2, 3] = 4.0
    cam = _camera(80, 64, fx=80.0, view=view, near=0.01, far=100.0, cx=40.0, cy=32.0)
    cases["cfg0_mini"] = (cam, (means, scales, quats, opac, colors), np.zeros(3), True)
    # 6. empty frame: everything culled
    rng = np.random.default_rng(1005)
    cam = _camera(20, 18)
    m, s, qq, o, c = _frustum_scene(rng, 5, cam)
    m[:, 2] = -1.0
    cases["all_culled"] = (cam, (m, s, qq, o, c), np.array([0.25, 0.5, 0.75]), True)
    return cases


def run_case(sg, cam_d, params, bg, et, rng):
    means, scales, quats, opac, colors = [_f32(p) for p in params]
    view = _f32(cam_d["view"])
    cam = sg.Camera(view=view, fx=cam_d["fx"], fy=cam_d["fy"], cx=cam_d["cx"],
                    cy=cam_d["cy"], width=cam_d["width"], height=cam_d["height"],
                    near=cam_d["near"], far=cam_d["far"])
    scene = [sg.Gaussian3D(mean=means[i], scale=scales[i], quat=quats[i],
                           opacity=float(opac[i]), color=colors[i])
             for i in range(len(means))]
    bg = _f32(bg)
    res = sg.render(scene, cam, bg, early_termination=et)
    d_image = _f32(rng.normal(size=(cam.height, cam.width, 3)))
    splat = sg.accumulate_image_backward(scene, res, d_image)
    grads = sg.scene_backward(scene, cam, res, d_image)
    proj = res.projected
    src = np.array([p.source_index for p in proj], dtype=np.int64)
    # bins as CSR over SCENE indices (source_index), in sorted order
    ptr = [0]
    idx = []
    for b in res.grid.bins:
        idx.extend(int(proj[j].source_index) for j in b)
        ptr.append(len(idx))
    out = dict(
        means=means, scales=scales, quats=quats, opacities=opac, colors=colors,
        view=view, intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.near, cam.far]),
        size=np.array([cam.width, cam.height], dtype=np.int64),
        background=bg, early_termination=np.array(et),
        image=res.image.channels, final_T=res.aux.final_T, n_contrib=res.aux.n_contrib,
        proj_source=src,
        proj_t_cam=np.array([p.t_cam for p in proj]).reshape(-1, 4),
        proj_mean2d=np.array([p.mean2d for p in proj]).reshape(-1, 2),
        proj_cov2d=np.array([p.cov2d for p in proj]).reshape(-1, 2, 2),
        proj_depth=np.array([p.depth for p in proj], dtype=np.float64),
        proj_radius=np.array([p.radius for p in proj], dtype=np.int64),
        bin_ptr=np.array(ptr, dtype=np.int64), bin_idx=np.array(idx, dtype=np.int64),
        d_image=d_image,
        s_d_color=splat.d_color, s_d_opacity=splat.d_opacity,
        s_d_mean2d=splat.d_mean2d, s_d_cov2d=splat.d_cov2d,
        g_d_mean=grads.d_mean, g_d_scale=grads.d_scale, g_d_quat=grads.d_quat,
        g_d_opacity=grads.d_opacity, g_d_color=grads.d_color, g_d_view=grads.d_view,
    )
    return out


def config0_case():
    """BASELINE config 0 exactly as paper_2312_02121_b200.scenes builds it."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2312_02121_b200.scenes import make_config
    spec = make_config(0)
    c = spec.cameras[0]
    cam = dict(view=c.view, fx=c.fx, fy=c.fy, cx=c.cx, cy=c.cy, width=c.width,
               height=c.height, near=c.near, far=c.far)
    params = (spec.means, spec.scales, spec.quats, spec.opacities, spec.colors)
    return cam, params, spec.background, True, spec.d_images[0]


class _FixedRng:
    def __init__(self, arr):
        self.arr = arr

    def normal(self, size):
        assert tuple(size) == self.arr.shape
        return self.arr


def main():
    sys.path.insert(0, REF_SRC)
    import splatgrad as sg  # noqa: E402  (reference, read-only)

    rng = np.random.default_rng(7)
    cases = build_cases()
    cases["config0"] = config0_case()
    for name, case in cases.items():
        cam, params, bg, et = case[:4]
        r = _FixedRng(np.asarray(case[4], np.float64)) if len(case) > 4 else rng
        out = run_case(sg, cam, params, bg, et, r)
        # inputs are fp32-exact by construction: store them losslessly as fp32
        for k in ("means", "scales", "quats", "opacities", "colors", "view", "background", "d_image"):
            assert np.array_equal(out[k].astype(np.float32).astype(np.float64), out[k]), k
            out[k] = out[k].astype(np.float32)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(f"{name}: N={len(out['means'])} visible={len(out['proj_source'])} "
              f"I={len(out['bin_idx'])} -> {os.path.relpath(path)}")


if __name__ == "__main__":
    main()
