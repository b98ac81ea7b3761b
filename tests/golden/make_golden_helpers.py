"""Golden vectors for the per-splat helpers (paper_2312_02121_b200.helpers),
made by running the REAL reference (splatgrad) here:

    python tests/golden/make_golden_helpers.py      # writes tests/golden/helpers.npz

Run in the build container only (``/root/reference`` is absent on the GPU
box); tests never import the reference.  For K random cases (a random
Gaussian in front of a random camera, the way sg/projection.py:115-145
chains the helpers) it stores every helper's inputs and the reference's
outputs: quat_to_rotmat, compose_covariance_3d (sg/core.py:146-204),
world_to_camera, camera_to_pixel, projection_jacobian, project_covariance,
bounding_radius (sg/projection.py:36-112), mean2d_backward, cov2d_backward,
world_backward, covariance3d_backward (sg/proj_backward.py:53-175) and
frobenius_inner.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


def main(k=64, seed=7):
    sys.path.insert(0, REF_SRC)
    import splatgrad as sg
    rng = np.random.default_rng(seed)
    rows = {key: [] for key in (
        "quat", "scale", "mean", "view", "intr", "R", "S", "M", "sigma", "t_cam", "mean2d", "J", "Rcw", "cov2d",
        "radius", "d_mean2d", "dt_mean2d", "d_cov2d", "T_proj", "d_sigma", "dt_cov2d", "d_t_total", "d_mean",
        "d_view", "d_quat", "d_scale", "frob_x", "frob_y", "frob")}
    while len(rows["quat"]) < k:
        q = rng.normal(size=4) * rng.uniform(0.2, 3.0)
        s = np.exp(rng.uniform(np.log(0.01), np.log(0.5), 3))
        cq = rng.normal(size=4)
        view = np.eye(4)
        view[:3, :3] = sg.quat_to_rotmat(cq)
        view[:3, 3] = rng.uniform(-1, 1, 3) + np.array([0, 0, 5.0])
        W, H = int(rng.integers(32, 200)), int(rng.integers(32, 200))
        fx, fy = rng.uniform(50, 300), rng.uniform(50, 300)
        cx, cy = rng.uniform(0, W), rng.uniform(0, H)
        cam = sg.Camera(view=view, fx=fx, fy=fy, cx=cx, cy=cy, width=W, height=H, near=0.01, far=100.0)
        mean = view[:3, :3].T @ (np.array([rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(2, 8)]) - view[:3, 3])
        t = sg.world_to_camera(mean, cam)
        if t[2] <= 0.1:
            continue
        b = sg.compose_covariance_3d(q, s)
        J = sg.projection_jacobian(t, cam)
        Rcw = cam.rotation
        cov2d = sg.project_covariance(J, Rcw, b.sigma)
        g2 = rng.normal(size=2)
        G = rng.normal(size=(2, 2))
        T_proj = J @ Rcw
        d_sigma, dt_c = sg.cov2d_backward(G, T_proj, b.sigma, J, Rcw, t, cam)
        d_t_total = rng.normal(size=4)
        d_mean, d_view = sg.world_backward(d_t_total, cam, mean)
        dS = rng.normal(size=(3, 3))
        d_quat, d_scale = sg.covariance3d_backward(dS, b, q, s)
        fx_, fy_ = rng.normal(size=(3, 4)), rng.normal(size=(3, 4))
        for key, v in (("quat", q), ("scale", s), ("mean", mean), ("view", view),
                       ("intr", np.array([fx, fy, cx, cy, W, H, 0.01, 100.0])), ("R", b.R), ("S", b.S), ("M", b.M),
                       ("sigma", b.sigma), ("t_cam", t), ("mean2d", sg.camera_to_pixel(t, cam)), ("J", J),
                       ("Rcw", Rcw), ("cov2d", cov2d), ("radius", sg.bounding_radius(cov2d)), ("d_mean2d", g2),
                       ("dt_mean2d", sg.mean2d_backward(g2, t, cam)), ("d_cov2d", G), ("T_proj", T_proj),
                       ("d_sigma", d_sigma), ("dt_cov2d", dt_c), ("d_t_total", d_t_total), ("d_mean", d_mean),
                       ("d_view", d_view), ("d_quat", d_quat), ("d_scale", d_scale), ("frob_x", fx_),
                       ("frob_y", fy_), ("frob", sg.frobenius_inner(fx_, fy_))):
            rows[key].append(np.asarray(v))
        rows.setdefault("dS", []).append(dS)
    np.savez(os.path.join(HERE, "helpers.npz"), **{key: np.stack(v) for key, v in rows.items()})
    print("wrote helpers.npz with", k, "cases")


if __name__ == "__main__":
    main()
