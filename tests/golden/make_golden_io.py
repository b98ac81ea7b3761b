"""File-format fixtures made by the REAL reference (sg/cli.py): a scene
document (serialize_scene) and a PPM (write_image) of a fixed buffer, plus
the error messages of a few malformed documents.  Run in the build
container only: python tests/golden/make_golden_io.py"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    import splatgrad as sg
    from splatgrad.cli import parse_scene, serialize_scene, write_image
    rng = np.random.default_rng(7)
    view = np.eye(4)
    view[:3, :3] = sg.quat_to_rotmat(np.array([0.9, 0.1, -0.2, 0.3]))
    view[:3, 3] = [0.1, -0.2, 0.3]
    cam = sg.Camera(view=view, fx=40.0, fy=41.5, cx=15.5, cy=11.25, width=32, height=24, near=0.1, far=50.0)
    scene = [sg.Gaussian3D(mean=rng.normal(size=3), scale=rng.uniform(0.1, 1, 3), quat=rng.normal(size=4),
                           opacity=float(rng.uniform()), color=rng.uniform(size=3)) for _ in range(4)]
    bg = np.array([0.1, 0.25, 1.0])
    with open(os.path.join(HERE, "io_scene.json"), "w") as fh:
        fh.write(serialize_scene(scene, cam, bg))
    buf = sg.ImageBuffer(width=5, height=3, channels=np.linspace(-0.2, 1.2, 45).reshape(3, 5, 3))
    write_image(buf, os.path.join(HERE, "io_image.ppm"))
    bad = {}
    doc = json.loads(serialize_scene(scene, cam, bg))
    cases = {
        "extra_top": dict(doc, extra=1),
        "bad_version": dict(doc, version=2),
        "bad_opacity": dict(doc, gaussians=[dict(doc["gaussians"][0], opacity=1.5)]),
        "bad_scale_len": dict(doc, gaussians=[dict(doc["gaussians"][0], scale=[1.0, 2.0])]),
        "bool_entry": dict(doc, gaussians=[dict(doc["gaussians"][0], color=[True, 0.0, 0.0])]),
        "float_width": dict(doc, camera=dict(doc["camera"], width=32.0)),
        "bad_background": dict(doc, background=[0.0, 2.0, 0.0]),
        "missing_fx": dict(doc, camera={k: v for k, v in doc["camera"].items() if k != "fx"}),
        "gaussian_extra": dict(doc, gaussians=[doc["gaussians"][0], dict(doc["gaussians"][1], w=1)]),
        "non_rigid_view": dict(doc, camera=dict(doc["camera"], view=[2.0] + doc["camera"]["view"][1:])),
    }
    for name, d in cases.items():
        try:
            parse_scene(json.dumps(d))
            bad[name] = {"doc": d, "error": None}
        except ValueError as exc:
            bad[name] = {"doc": d, "error": str(exc)}
    with open(os.path.join(HERE, "io_errors.json"), "w") as fh:
        json.dump(bad, fh, indent=1)
    print("wrote io_scene.json io_image.ppm io_errors.json")


if __name__ == "__main__":
    main()
