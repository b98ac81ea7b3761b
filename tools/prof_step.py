"""One multi-view step of a BASELINE config through engine.RenderStep (the
batched projections, every view's binning and rasterizers), for ncu.

  ncu --profile-from-start off --set full -k regex:... python tools/prof_step.py 3 [views] [reps]
"""
import sys

import torch

from paper_2312_02121_b200 import engine as E
from paper_2312_02121_b200 import ops
from paper_2312_02121_b200.scenes import make_config

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
views = int(sys.argv[2]) if len(sys.argv) > 2 else 32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
spec = make_config(cfg, n_views=views)
dev = torch.device("cuda", 0)
params = [torch.as_tensor(a, device=dev) for a in (spec.means, spec.scales, spec.quats, spec.opacities, spec.colors)]
cams = [ops.CameraParams.of(c) for c in spec.cameras]
d_imgs = [torch.as_tensor(d, device=dev) for d in spec.d_images]
eng = E.RenderStep(spec.n, cams, device=dev)
eng.prime(params, d_imgs)
eng.step(params, d_imgs)  # warm
torch.cuda.synchronize()
torch.cuda.profiler.start()  # ncu --profile-from-start off: only the timed steps
for _ in range(reps):
    eng.step(params, d_imgs)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("step ok", len(cams), "views")
