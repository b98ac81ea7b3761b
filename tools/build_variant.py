"""Build an A/B variant of the library: the given sources recompiled with
extra nvcc flags, linked with the regular objects into
_ab/<name>/libsplat_b200.so (load it with GS_LIB_PATH=...).

  python tools/build_variant.py <name> <src.cu>[,<src.cu>] -DFOO=1 ...
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_02121_b200 import build as B  # noqa: E402

name, srcs, flags = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
B.build()
out = os.path.join(B.ROOT, "_ab", name)
os.makedirs(out, exist_ok=True)
objs = []
for o in sorted(os.listdir(B.OBJ)):
    src = o[:-2] + ".cu"
    if src in srcs:
        obj = os.path.join(out, o)
        cmd = [B._nvcc()] + B.NVCC_FLAGS + flags + ["-c", os.path.join(B.CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stdout + r.stderr)
        objs.append(obj)
    else:
        objs.append(os.path.join(B.OBJ, o))
lib = os.path.join(out, "libsplat_b200.so")
subprocess.run([B._nvcc()] + B.ARCH + ["-shared", "-o", lib] + objs, check=True)
print(lib)
