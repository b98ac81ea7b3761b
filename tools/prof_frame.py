"""One frame (frame_forward + frame_backward) of a BASELINE config, for ncu.

  ncu --set full -k regex:... python tools/prof_frame.py 4
"""
import sys

import torch

from paper_2312_02121_b200 import ops
from paper_2312_02121_b200.scenes import make_config

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = make_config(cfg, n_views=1)
dev = torch.device("cuda", 0)
t = lambda a: torch.as_tensor(a, device=dev)
m, s, q, o, c = t(spec.means), t(spec.scales), t(spec.quats), t(spec.opacities), t(spec.colors)
cam = ops.CameraParams.of(spec.cameras[0])
d_image = torch.ones((cam.height, cam.width, 3), device=dev)
fr = ops.frame_forward(m, s, q, o, c, cam, (0.0, 0.0, 0.0), True)
cap = int(fr.needed_capacity * 1.05) + 4096
for _ in range(reps):
    fr = ops.frame_forward(m, s, q, o, c, cam, (0.0, 0.0, 0.0), True, capacity=cap)
    g = ops.frame_backward(fr, m, s, q, c, d_image)
torch.cuda.synchronize()
print("frame ok", fr.n_isect)
