"""Audit-scene fixtures made by running the REAL reference's generator
(sg/gradcheck.py make_audit_scene) here: tests/golden/audit_scenes.npz pins
paper_2312_02121_b200.gradcheck's seeded generator to the same draws.
Run in the build container only: python tests/golden/make_golden_audit.py"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    from splatgrad.gradcheck import make_audit_scene
    out = {}
    for seed in (0, 1, 4):
        scene, camera, target, bg, mask = make_audit_scene(seed, 16 if seed % 2 == 0 else 32)
        out[f"s{seed}_means"] = np.array([g.mean for g in scene])
        out[f"s{seed}_view"] = camera.view
        out[f"s{seed}_bg"] = np.asarray(bg)
        out[f"s{seed}_mask"] = np.asarray(mask)
    np.savez_compressed(os.path.join(HERE, "audit_scenes.npz"), **out)
    print("wrote audit_scenes.npz", {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
