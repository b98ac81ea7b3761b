"""Quadrant culling statistics (ignoring early termination): for every
(tile-list entry, 8x8 quadrant) pair, does the current staging test (clamped
ellipse-extent box), an exact ellipse-vs-rectangle test, or the pixel-centre
sigma cut keep it?"""
import sys

import numpy as np
import torch

from paper_2312_02121_b200 import ops
from paper_2312_02121_b200.scenes import make_config

for cfg in [int(a) for a in sys.argv[1:]]:
    spec = make_config(cfg, n_views=1)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.as_tensor(a, device=dev)
    cam = ops.CameraParams.of(spec.cameras[0])
    fr = ops.frame_forward(t(spec.means), t(spec.scales), t(spec.quats), t(spec.opacities), t(spec.colors), cam,
                           (0.0, 0.0, 0.0), True)
    T = fr.tensors()
    r = T["ranges"].cpu().numpy().astype(np.int64)
    vals = T["sorted_vals"].cpu().numpy().astype(np.int64)
    xy = T["xydr"].cpu().numpy()
    q = T["conic"].cpu().numpy().astype(np.float64)
    rad = xy[:, 3].view(np.int32).astype(np.float64)
    ln = r[:, 1] - r[:, 0]
    tile = np.repeat(np.arange(len(ln)), ln)
    ids = np.concatenate([vals[a:b] for a, b in r]) if ln.sum() else np.zeros(0, np.int64)
    tx, ty = tile % cam.tiles_x, tile // cam.tiles_x
    mx, my = xy[ids, 0].astype(np.float64), xy[ids, 1].astype(np.float64)
    A, B, Cc = q[ids, 0], q[ids, 1], q[ids, 2]
    det = A * Cc - B * B
    rr = rad[ids] + 1
    rx = np.minimum(rr, 3.003 * np.sqrt(Cc / det) + 1)
    ry = np.minimum(rr, 3.003 * np.sqrt(A / det) + 1)
    tot = dict(box=0, exact=0, pix=0, g05=0, g1=0)
    offs = np.arange(8) + 0.5
    for w in range(4):
        x0 = tx * 16 + (w & 1) * 8 + 0.5
        y0 = ty * 16 + (w >> 1) * 8 + 0.5
        box = (mx + rx >= x0) & (mx - rx <= x0 + 7) & (my + ry >= y0) & (my - ry <= y0 + 7)
        tot["box"] += box.sum()
        # exact: min over the rectangle [x0, x0+7] x [y0, y0+7] of d^T Q d <= 9
        lo_x, hi_x, lo_y, hi_y = x0 - mx, x0 + 7 - mx, y0 - my, y0 + 7 - my
        inside = (lo_x <= 0) & (hi_x >= 0) & (lo_y <= 0) & (hi_y >= 0)
        best = np.where(inside, 0.0, np.inf)
        for dx in (lo_x, hi_x):
            dy = np.clip(-B * dx / Cc, lo_y, hi_y)
            best = np.minimum(best, A * dx * dx + 2 * B * dx * dy + Cc * dy * dy)
        for dy in (lo_y, hi_y):
            dx = np.clip(-B * dy / A, lo_x, hi_x)
            best = np.minimum(best, A * dx * dx + 2 * B * dx * dy + Cc * dy * dy)
        tot["exact"] += (best <= 9.0).sum()
        for key, g in (("g05", 0.5), ("g1", 1.0)):
            lx, hx, ly, hy = lo_x - g, hi_x + g, lo_y - g, hi_y + g
            ins = (lx <= 0) & (hx >= 0) & (ly <= 0) & (hy >= 0)
            bb = np.where(ins, 0.0, np.inf)
            for dx in (lx, hx):
                dy = np.clip(-B * dx / Cc, ly, hy)
                bb = np.minimum(bb, A * dx * dx + 2 * B * dx * dy + Cc * dy * dy)
            for dy in (ly, hy):
                dx = np.clip(-B * dy / A, lx, hx)
                bb = np.minimum(bb, A * dx * dx + 2 * B * dx * dy + Cc * dy * dy)
            tot[key] += (bb <= 9.0 * 1.002).sum()
        pm = np.zeros(len(ids), bool)
        for oy in offs - 0.5:
            dy = y0 + oy - my
            for ox in offs - 0.5:
                dx = x0 + ox - mx
                pm |= 0.5 * (A * dx * dx + 2 * B * dx * dy + Cc * dy * dy) <= 4.5
        tot["pix"] += pm.sum()
    E = len(ids)
    print(f"config{cfg}: entries={E} quadrant-entries={4*E} box={tot['box']} ({tot['box']/(4*E):.3f}) "
          f"exact={tot['exact']} ({tot['exact']/(4*E):.3f}) g05={tot['g05']/(4*E):.3f} g1={tot['g1']/(4*E):.3f} pix={tot['pix']} ({tot['pix']/(4*E):.3f})", flush=True)
