"""One frame-path forward+backward (gs_frame_forward / gs_frame_backward: commit records, the grouped
record backward) under each binning, for compute-sanitizer:
  compute-sanitizer --tool memcheck|racecheck python tools/sanitize_frame_path.py [n]"""
import sys

import torch

from paper_2312_02121_b200 import ops
from paper_2312_02121_b200.scenes import make_config

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
spec = make_config(1, n_override=n)
dev = torch.device("cuda", 0)
t = lambda a: torch.as_tensor(a, device=dev)
m, s, q, o, c = t(spec.means), t(spec.scales), t(spec.quats), t(spec.opacities), t(spec.colors)
cam = ops.CameraParams.of(spec.cameras[0])
d_img = t(spec.d_images[0])
for mode in (1, 2, 3):  # depth-first, scatter, direct
    ops.set_option("binning", mode)
    fr = ops.frame_forward(m, s, q, o, c, cam, (0.0, 0.0, 0.0), True)
    g = ops.frame_backward(fr, m, s, q, c, d_img)
    torch.cuda.synchronize()
    print("binning", mode, "ok", float(g["d_mean"].abs().sum()), flush=True)
ops.set_option("binning", 0)
