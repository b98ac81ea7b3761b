import torch, sys
sys.path.insert(0, '.')
from paper_2312_02121_b200 import ops, _lib
from paper_2312_02121_b200.scenes import make_config
spec = make_config(0)
dev = torch.device('cuda')
t = lambda a: torch.as_tensor(a, device=dev)
m, s, q, o, c = [t(spec.means), t(spec.scales), t(spec.quats), t(spec.opacities), t(spec.colors)]
cam = ops.CameraParams.of(spec.cameras[0])
fr = ops.frame_forward(m, s, q, o, c, cam)
cap = fr.n_isect + 1000
L = _lib.load()
ws = ops.frame_workspace(spec.n, cap, cam.width, cam.height, dev)
for use_ev in (False, True):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    for e in evs: e.record()
    torch.cuda.synchronize()
    def step():
        return ops.frame_forward(m, s, q, o, c, cam, capacity=cap, check_meta=False, ws=ws, events=evs if use_ev else None)
    side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2): step()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g):
            step()
        g.replay(); torch.cuda.synchronize()
        print('use_ev', use_ev, 'ok', [evs[i].elapsed_time(evs[i+1]) for i in range(5)] if use_ev else '')
    except Exception as ex:
        print('use_ev', use_ev, 'FAILED', ex)
