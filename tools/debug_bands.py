"""Emulate the 2-band split of a config-4 frame in one process and locate the
Gaussians whose gradient differs most from the full frame's."""
import numpy as np
import torch

from paper_2312_02121_b200 import dist as D
from paper_2312_02121_b200 import engine as E
from paper_2312_02121_b200 import ops
from paper_2312_02121_b200.scenes import make_config

spec = make_config(4, n_override=400_000)
dev = torch.device("cuda", 0)
P = [torch.as_tensor(a, device=dev) for a in (spec.means, spec.scales, spec.quats, spec.opacities, spec.colors)]
full = ops.CameraParams.of(spec.cameras[0])
proj = ops.project(*P[:4], full)
work = D.tile_row_work_from_projection(proj.xydr, full.height, full.width)
bands = D.band_rows(work, 2, full.height)
print("bands", bands)
frames, rows_sum, c11_sum = [], None, None
for r0, r1 in bands:
    cam = D.band_camera(full, r0, r1)
    fr = ops.frame_forward(*P, cam, (0.0, 0.0, 0.0), True)
    ops.frame_backward(fr, P[0], P[1], P[2], P[4], torch.as_tensor(np.ascontiguousarray(spec.d_images[0][r0:r1]), device=dev), project=False)
    rows, c11 = ops.frame_screen_grads(fr)
    rows_sum = rows.clone() if rows_sum is None else rows_sum + rows
    c11_sum = c11.clone() if c11_sum is None else c11_sum + c11
    frames.append(fr)
fr = frames[0]
rows, c11 = ops.frame_screen_grads(fr)
rows.copy_(rows_sum); c11.copy_(c11_sum)
flat = torch.zeros(14 * spec.n, device=dev); dv = torch.zeros(4, 4, device=dev)
ops.frame_project_backward(fr, P[0], P[1], P[2], E.unpack(flat, spec.n), dv, vis_from_grads=True)
ff = ops.frame_forward(*P, full, (0.0, 0.0, 0.0), True)
g = ops.frame_backward(ff, P[0], P[1], P[2], P[4], torch.as_tensor(spec.d_images[0], device=dev), keep_screen=True)
tv = ff.tensors()
u = E.unpack(flat, spec.n)
a, b = u["d_mean"].cpu().numpy(), g["d_mean"].cpu().numpy()
err = np.abs(a - b).max(1)
idx = np.argsort(err)[::-1][:10]
geo_full = tv["d_geo"].cpu().numpy(); geo_band = rows_sum[:, 4:].cpu().numpy()
tiles0 = frames[0].tensors()["tiles"].cpu().numpy(); tiles1 = frames[1].tensors()["tiles"].cpu().numpy()
tf = tv["tiles"].cpu().numpy()
xy = tv["xydr"].cpu().numpy()
for i in idx:
    print(i, "err", err[i], "ref", b[i], "got", a[i], "tiles full/b0/b1", tf[i], tiles0[i], tiles1[i], "y", xy[i, 1],
          "r", xy[i, 3:4].view(np.int32)[0], "geo full", geo_full[i], "band", geo_band[i])
print("rows max diff", np.abs(geo_full - geo_band).max(), "n rows differing >1e-3 rel:",
      int((np.abs(geo_full - geo_band).max(1) > 1e-3 * (np.abs(geo_full).max(1) + 1e-6)).sum()))
