"""Where the e2e (engine.pipeline) step time goes: host enqueue time per
step vs the device time per step, on config 1 (one view)."""
import time

import numpy as np
import torch

from paper_2312_02121_b200 import engine as E
from paper_2312_02121_b200.scenes import make_config

spec = make_config(1, n_views=1)
dev = torch.device("cuda", 0)


def staged(a, wc):
    a = np.ascontiguousarray(a, dtype=np.float32)
    t = E.host_staging(a.shape) if wc else torch.empty(a.shape).pin_memory()
    t.copy_(torch.from_numpy(a))
    return t


for wc in (True, False):
    host = [staged(a, wc) for a in (spec.means, spec.scales, spec.quats, spec.opacities, spec.colors)]
    dimgs = [staged(spec.d_images[0], wc)]
    eng = E.RenderStep(spec.n, [spec.cameras[0]], device=dev)
    eng.prime(host, dimgs)
    out = [torch.empty((14 * spec.n,)).pin_memory() for _ in range(eng.nbuf)]
    for flush in (None, torch.empty(192 << 18, device=dev)):
        E.pipeline(eng, host, dimgs, out, 5, None, flush)
        torch.cuda.synchronize()
        steps = 40
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        E.pipeline(eng, host, dimgs, out, steps, None, flush)
        e1.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"wc={wc} flush={flush is not None}: enqueue {1e3 * (t1 - t0) / steps:.3f} ms/step, "
              f"device {e0.elapsed_time(e1) / steps:.3f} ms/step, wall {1e3 * (t2 - t0) / steps:.3f} ms/step")
    g0 = time.perf_counter()
    for _ in range(40):
        eng.replay(0)
    torch.cuda.synchronize()
    print(f"replay only: {1e3 * (time.perf_counter() - g0) / 40:.3f} ms/step")
