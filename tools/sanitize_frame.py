"""Run one staged forward+backward of a BASELINE config (for compute-sanitizer)."""
import sys

import numpy as np
import torch

from paper_2312_02121_b200 import ops
from paper_2312_02121_b200.scenes import make_config

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
spec = make_config(cfg, n_views=1)
dev = torch.device("cuda", 0)
t = lambda a: torch.as_tensor(a, device=dev)
m, s, q, o, c = t(spec.means), t(spec.scales), t(spec.quats), t(spec.opacities), t(spec.colors)
cam = ops.CameraParams.of(spec.cameras[0])
image, st = ops.render_forward(m, s, q, o, c, cam, (0.0, 0.0, 0.0), True)
torch.cuda.synchronize()
print("fwd ok", st.bins.n_isect, flush=True)
g = ops.render_backward(st, m, s, q, c, torch.ones_like(image))
torch.cuda.synchronize()
print("bwd ok", flush=True)
