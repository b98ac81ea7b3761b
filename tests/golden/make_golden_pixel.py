"""Golden fixtures for the per-pixel API, made by running the REAL reference.

Run in the build container only: ``python tests/golden/make_golden_pixel.py``
writes ``tests/golden/pixel.npz`` (committed; tests never import the
reference).  Inputs are fp32-exact so the GPU and the fp64 restatement see
the reference's exact values.  Splats are given directly in screen space
(ProjectedGaussian with random mean2d / SPD cov2d), which is what the
per-pixel functions consume:

  eval_alpha                  sg/raster_forward.py:175-196   (ea_* arrays)
  composite_pixel             sg/raster_forward.py:199-219   (q_color, q_T, q_nc)
  composite_pixel_backward    sg/raster_backward.py:111-135  (g_* per query, per splat)
  transmittance_replay        sg/raster_backward.py:138-163  (r_pos / r_T CSR)
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


def _f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def main():
    sys.path.insert(0, REF_SRC)
    import splatgrad as sg
    from splatgrad.projection import ProjectedGaussian

    rng = np.random.default_rng(2312)
    out = {}

    # ---- eval_alpha: random splats and pixel centres, some far, some tiny
    n_ea = 400
    means = _f32(rng.uniform(-6, 6, size=(n_ea, 2)))
    mats = rng.normal(size=(n_ea, 2, 2)) * rng.uniform(0.3, 2.0, size=(n_ea, 1, 1))
    covs = _f32(mats @ np.transpose(mats, (0, 2, 1)) + 0.3 * np.eye(2))
    opac = _f32(np.where(rng.uniform(size=n_ea) < 0.1, rng.uniform(1e-4, 5e-3, n_ea), rng.uniform(0.05, 1.0, n_ea)))
    pix = _f32(means + rng.normal(size=(n_ea, 2)) * rng.uniform(0.0, 4.0, size=(n_ea, 1)))
    ea = np.zeros((n_ea, 4))
    for i in range(n_ea):
        g = ProjectedGaussian(t_cam=np.array([0.0, 0.0, 1.0]), mean2d=means[i], cov2d=covs[i], depth=1.0, radius=1,
                              source_index=0)
        a, d, s = sg.eval_alpha(g, float(opac[i]), pix[i])
        ea[i] = a, d[0], d[1], s
    out.update(ea_mean2d=means, ea_cov2d=covs, ea_opacity=opac, ea_pix=pix, ea_out=ea)

    # ---- compositing queries over one shared set of screen-space splats
    m = 48
    mean2d = rng.uniform(0, 24, size=(m, 2))
    mean2d[:16] = 12.0 + rng.normal(size=(16, 2))  # a dense cluster: early termination around (12, 12)
    mean2d = _f32(mean2d)
    mats = rng.normal(size=(m, 2, 2)) * rng.uniform(0.8, 3.0, size=(m, 1, 1))
    mats[:16] = np.eye(2) * rng.uniform(3.0, 5.0, size=(16, 1, 1))
    cov2d = _f32(mats @ np.transpose(mats, (0, 2, 1)) + 0.3 * np.eye(2))
    # scene rows are a permutation of the projected rows (source_index)
    src = rng.permutation(m)
    s_opac = _f32(rng.uniform(0.2, 0.99, size=m))
    s_opac[src[:16]] = 0.97
    s_opac[src[16:20]] = 1.0  # alpha clamp at 0.999
    s_color = _f32(rng.uniform(0, 1, size=(m, 3)))
    projected = [ProjectedGaussian(t_cam=np.array([0.0, 0.0, 1.0]), mean2d=mean2d[j], cov2d=cov2d[j],
                                   depth=float(j), radius=1, source_index=int(src[j])) for j in range(m)]
    scene = [sg.Gaussian3D(mean=np.zeros(3), scale=np.ones(3), quat=np.array([1.0, 0, 0, 0]),
                           opacity=float(s_opac[i]), color=s_color[i]) for i in range(m)]
    bg = _f32([0.15, 0.25, 0.35])
    n_q = 96
    q_pix = np.concatenate([np.floor(rng.uniform(0, 24, size=(n_q // 2, 2))) + 0.5,
                            rng.uniform(0, 24, size=(n_q - n_q // 2, 2))])
    q_pix[::4] = 12.0 + rng.uniform(-2, 2, size=(len(q_pix[::4]), 2))
    q_pix = _f32(q_pix)
    q_et = (np.arange(n_q) % 3 != 2).astype(np.int8)
    bins, ptr = [], [0]
    for q in range(n_q):
        k = int(rng.integers(0, m + 1)) if q % 8 else m  # ragged, some empty, some full
        b = rng.permutation(m)[:k]
        bins.extend(b.tolist())
        ptr.append(len(bins))
    q_color = np.zeros((n_q, 3))
    q_T = np.zeros(n_q)
    q_nc = np.zeros(n_q, np.int64)
    d_pix = _f32(rng.normal(size=(n_q, 3)))
    g_color = np.zeros((n_q, m, 3))
    g_opac = np.zeros((n_q, m))
    g_mean = np.zeros((n_q, m, 2))
    g_cov = np.zeros((n_q, m, 2, 2))
    r_pos, r_T, r_ptr = [], [], [0]
    for q in range(n_q):
        b = bins[ptr[q]:ptr[q + 1]]
        col, aux = sg.composite_pixel(b, projected, scene, q_pix[q], bg, early_termination=bool(q_et[q]))
        q_color[q], q_T[q], q_nc[q] = col, aux.final_T, aux.n_contrib
        gr = sg.composite_pixel_backward(b, projected, scene, q_pix[q], bg, aux, d_pix[q])
        g_color[q], g_opac[q], g_mean[q], g_cov[q] = gr.d_color, gr.d_opacity, gr.d_mean2d, gr.d_cov2d
        for pos, t in sg.transmittance_replay(b, projected, scene, q_pix[q], bg, aux):
            r_pos.append(pos)
            r_T.append(t)
        r_ptr.append(len(r_pos))
    out.update(mean2d=mean2d, cov2d=cov2d, source_index=src, s_opacity=s_opac, s_color=s_color, background=bg,
               q_pix=q_pix, q_et=q_et, bin_ptr=np.asarray(ptr, np.int64), bin_idx=np.asarray(bins, np.int64),
               q_color=q_color, q_T=q_T, q_nc=q_nc, d_pix=d_pix, g_color=g_color, g_opacity=g_opac,
               g_mean2d=g_mean, g_cov2d=g_cov, r_ptr=np.asarray(r_ptr, np.int64), r_pos=np.asarray(r_pos, np.int64),
               r_T=np.asarray(r_T, np.float64))
    path = os.path.join(HERE, "pixel.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
