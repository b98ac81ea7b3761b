import torch
from paper_2312_02121_b200 import ops
from paper_2312_02121_b200.scenes import make_config
for cfg in (2, 3, 4):
    spec = make_config(cfg, n_views=4 if cfg == 3 else 1)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.as_tensor(a, device=dev)
    m, s, q, o, c = t(spec.means), t(spec.scales), t(spec.quats), t(spec.opacities), t(spec.colors)
    for cv in spec.cameras[:4]:
        cam = ops.CameraParams.of(cv)
        fr = ops.frame_forward(m, s, q, o, c, cam, (0.0, 0.0, 0.0), True)
        tl = fr.tensors()["tiles"]
        print(cfg, spec.n, "visible", int((tl != 0).sum()), "isect", fr.n_isect, flush=True)
