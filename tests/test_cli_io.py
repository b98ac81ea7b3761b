"""CPU: scene JSON and PPM formats (paper_2312_02121_b200.cli) against files
and error messages made by the reference (tests/golden/make_golden_io.py),
plus the format round trips of tests/test_io.py (sg/cli.py:61-197)."""

import json
import os

import numpy as np
import pytest

from paper_2312_02121_b200 import api, cli

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _text(name):
    with open(os.path.join(GOLDEN, name), "r", encoding="utf-8") as fh:
        return fh.read()


def test_serialize_is_byte_identical_to_reference():
    ref = _text("io_scene.json")
    scene, cam, bg = cli.parse_scene(ref)
    assert cli.serialize_scene(scene, cam, bg) == ref
    assert cli.parse_scene(ref.encode("utf-8"))[1].width == 32


def test_round_trip_exact():
    scene, cam, bg = cli.parse_scene(_text("io_scene.json"))
    s2, c2, b2 = cli.parse_scene(cli.serialize_scene(scene, cam, bg))
    assert np.array_equal(c2.view, cam.view) and np.array_equal(b2, bg)
    for a, b in zip(scene, s2):
        assert np.array_equal(a.mean, b.mean) and np.array_equal(a.quat, b.quat) and a.opacity == b.opacity


def test_errors_match_reference_messages():
    cases = json.loads(_text("io_errors.json"))
    for name, c in cases.items():
        if c["error"] is None:
            cli.parse_scene(json.dumps(c["doc"]))
            continue
        with pytest.raises(ValueError) as ei:
            cli.parse_scene(json.dumps(c["doc"]))
        assert str(ei.value) == c["error"], name


def test_invalid_json():
    with pytest.raises(ValueError, match="not valid JSON"):
        cli.parse_scene("{nope")


def test_ppm_bytes_match_reference(tmp_path):
    buf = api.ImageBuffer(5, 3, np.linspace(-0.2, 1.2, 45).reshape(3, 5, 3))
    p = tmp_path / "a.ppm"
    cli.write_image(buf, str(p))
    with open(os.path.join(GOLDEN, "io_image.ppm"), "rb") as fh:
        assert p.read_bytes() == fh.read()
    img = cli.read_image(str(p))
    assert img.shape == (3, 5, 3) and img.min() == 0.0 and img.max() == 1.0


def test_ppm_quantization_and_header(tmp_path):
    p = tmp_path / "b.ppm"
    vals = np.array([0.0, 0.5 / 255, 1.0, 0.499 / 255, 254.5 / 255, 1.0]).reshape(1, 2, 3)
    cli.write_image(api.ImageBuffer(2, 1, vals), str(p))
    assert list(p.read_bytes()[-6:]) == [0, 1, 255, 0, 255, 255]
    q = tmp_path / "c.ppm"
    q.write_bytes(b"P6\n# comment\n2 1\n# another\n255\n" + bytes(range(6)))
    assert np.allclose(cli.read_image(str(q)).ravel() * 255, range(6))
    for data, msg in ((b"P5\n1 1\n255\n\x00", "not a binary PPM"), (b"P6\n1 1\n65535\n" + bytes(6), "maxval"),
                      (b"P6\n2 2\n255\n" + bytes(5), "payload size"), (b"P6\n1", "truncated")):
        q.write_bytes(data)
        with pytest.raises(ValueError, match=msg):
            cli.read_image(str(q))


def test_usage_error_exits_2():
    with pytest.raises(SystemExit) as ei:
        cli.main(["render"])
    assert ei.value.code == 2


def test_missing_file_exits_2(tmp_path, capsys):
    assert cli.main(["render", str(tmp_path / "none.json"), "-o", str(tmp_path / "x.ppm")]) == 2
    assert "error:" in capsys.readouterr().err
