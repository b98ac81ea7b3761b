"""Tile-list length statistics of a config (for binning design decisions)."""
import sys

import numpy as np
import torch

from paper_2312_02121_b200 import ops
from paper_2312_02121_b200.scenes import make_config

for cfg in [int(a) for a in sys.argv[1:]]:
    spec = make_config(cfg, n_views=1)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.as_tensor(a, device=dev)
    m, s, q, o, c = t(spec.means), t(spec.scales), t(spec.quats), t(spec.opacities), t(spec.colors)
    cam = ops.CameraParams.of(spec.cameras[0])
    fr = ops.frame_forward(m, s, q, o, c, cam, (0.0, 0.0, 0.0), True)
    r = fr.tensors()["ranges"].cpu().numpy().astype(np.int64)
    ln = r[:, 1] - r[:, 0]
    print(f"config{cfg}: n={spec.n} tiles={len(ln)} isect={ln.sum()} mean={ln.mean():.0f} "
          f"p50={np.percentile(ln, 50):.0f} p99={np.percentile(ln, 99):.0f} max={ln.max()} "
          f">2048: {(ln > 2048).sum()} >4096: {(ln > 4096).sum()} >8192: {(ln > 8192).sum()}")
