"""B200-native (sm_100a) differentiable Gaussian-splatting hot path.

Drop-in for the reference `splatgrad` render path (project -> tile-bin/sort
-> rasterize forward -> rasterize backward -> projection backward).  Kernels
live in libsplat_b200.so (csrc/, C ABI in include/splat_b200.h); this package
is the host side: `ops` (device pipeline + torch.autograd.Function) and
`api` (the reference's Python API names on top of it).
"""

__version__ = "0.1.0"
