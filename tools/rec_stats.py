"""Distribution of the forward's commit records per (tile, quadrant warp) --
the record backward's work per warp -- for one view of a config.

  python tools/rec_stats.py 3
"""
import sys

import numpy as np
import torch

from paper_2312_02121_b200 import ops
from paper_2312_02121_b200.scenes import make_config

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
spec = make_config(cfg, n_views=1)
dev = torch.device("cuda", 0)
t = [torch.as_tensor(a, device=dev) for a in (spec.means, spec.scales, spec.quats, spec.opacities, spec.colors)]
cam = ops.CameraParams.of(spec.cameras[0])
fr = ops.frame_forward(*t, cam, (0.0, 0.0, 0.0), True)
tv = fr.tensors()
rc = tv["rec_count"].cpu().numpy().astype(np.int64)
lens = (tv["ranges"][:, 1] - tv["ranges"][:, 0]).cpu().numpy()
w = rc.reshape(-1)
print(f"config{cfg}: tiles {len(rc)} records {w.sum()} per warp mean {w.mean():.1f} p50 {np.median(w):.0f} "
      f"p99 {np.percentile(w, 99):.0f} max {w.max()}  list len mean {lens.mean():.0f} max {lens.max()}")
top = np.sort(w)[::-1]
print("top warps:", top[:10].tolist(), " share of records in top 1% warps:",
      round(float(top[:max(1, len(top) // 100)].sum() / w.sum()), 3))
