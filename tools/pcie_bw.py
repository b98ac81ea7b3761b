"""Pinned host<->device copy bandwidth at the e2e step sizes (13.3 MB H2D, 5.6 MB D2H)."""
import torch, time
n = 13_280_000 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
o = torch.empty(5_600_000 // 4, dtype=torch.float32).pin_memory()
dd = torch.empty(5_600_000 // 4, dtype=torch.float32, device="cuda")
for _ in range(5):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("H2D GB/s", 50 * 13.28e6 / (e0.elapsed_time(e1) / 1e3) / 1e9)
e0.record()
for _ in range(50):
    o.copy_(dd, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("D2H GB/s", 50 * 5.6e6 / (e0.elapsed_time(e1) / 1e3) / 1e9)
import os; print("cpus", os.cpu_count(), os.sched_getaffinity(0).__len__())
# the same H2D bytes split over k copy streams
for k in (2, 4, 8):
    sts = [torch.cuda.Stream() for _ in range(k)]
    chunks_h = h.chunk(k)
    chunks_d = d.chunk(k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        for st, a, b in zip(sts, chunks_d, chunks_h):
            with torch.cuda.stream(st):
                a.copy_(b, non_blocking=True)
    torch.cuda.synchronize()
    print(f"H2D GB/s over {k} streams", 50 * 13.28e6 / (time.perf_counter() - t0) / 1e9)

# write-combined pinned staging (cudaHostAllocWriteCombined): host writes once, the DMA engine reads
import ctypes
import numpy as np

rt = ctypes.CDLL("libcudart.so") if False else None
try:
    from cuda.bindings import runtime as cr  # cuda-python
except Exception:  # noqa: BLE001
    from cuda import cudart as cr
err, ptr = cr.cudaHostAlloc(13_280_000, cr.cudaHostAllocWriteCombined)
buf = (ctypes.c_float * n).from_address(int(ptr))
hw = torch.from_numpy(np.ctypeslib.as_array(buf))
print("WC tensor pinned:", hw.is_pinned())
for _ in range(5):
    d.copy_(hw, non_blocking=True)
torch.cuda.synchronize()
e0.record()
for _ in range(50):
    d.copy_(hw, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("H2D write-combined GB/s", 50 * 13.28e6 / (e0.elapsed_time(e1) / 1e3) / 1e9)
