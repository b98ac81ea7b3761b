"""GPU: the command line (cli.main; sg/cli.py:214-315) end to end:
render / --aux / --brute-force, gradcheck (single seed, report, failing
tolerance -> exit 1), fit (tests/test_cli.py cases)."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture()
def scene_file():
    return os.path.join(GOLDEN, "io_scene.json")


def test_render_writes_the_api_image(tmp_path, scene_file, cuda):
    from paper_2312_02121_b200 import api, cli
    out, aux = tmp_path / "r.ppm", tmp_path / "t.ppm"
    assert cli.main(["render", scene_file, "-o", str(out), "--aux", str(aux)]) == 0
    with open(scene_file) as fh:
        scene, cam, bg = cli.parse_scene(fh.read())
    res = api.render(scene, cam, bg)
    expect = np.floor(np.clip(res.image.channels, 0, 1) * 255 + 0.5) / 255
    assert np.array_equal(cli.read_image(str(out)), expect)
    t = cli.read_image(str(aux))
    assert np.array_equal(t[..., 0], np.floor(np.clip(res.aux.final_T, 0, 1) * 255 + 0.5) / 255)
    bf = tmp_path / "b.ppm"
    assert cli.main(["render", scene_file, "-o", str(bf), "--brute-force"]) == 0
    assert np.max(np.abs(cli.read_image(str(bf)) - cli.read_image(str(out)))) <= 1.0 / 255


def test_invalid_scene_exits_2(tmp_path, capsys, cuda):
    from paper_2312_02121_b200 import cli
    p = tmp_path / "bad.json"
    p.write_text('{"version": 2}')
    assert cli.main(["render", str(p), "-o", str(tmp_path / "x.ppm")]) == 2
    assert "error:" in capsys.readouterr().err


def test_gradcheck_command(tmp_path, capsys, cuda):
    from paper_2312_02121_b200 import cli
    rep = tmp_path / "rep.json"
    assert cli.main(["gradcheck", "--seed", "3", "--report", str(rep)]) == 0
    d = json.loads(rep.read_text())
    assert list(d) == ["3"] and d["3"]["passed"] and set(d["3"]["classes"]) == {
        "mean", "scale", "quat", "opacity", "color", "view"}
    assert cli.main(["gradcheck", "--seed", "3", "--tol-rel", "1e-14", "--tol-abs", "1e-20"]) == 1
    assert "FAIL" in capsys.readouterr().out


def test_fit_command(tmp_path, cuda):
    from paper_2312_02121_b200 import api, cli
    target = tmp_path / "t.ppm"
    ys, xs = np.mgrid[0:24, 0:32]
    img = np.stack([xs / 31.0, ys / 23.0, 0.5 + 0 * xs], -1)
    cli.write_image(api.ImageBuffer(32, 24, img), str(target))
    out, losses = tmp_path / "fit.json", tmp_path / "loss.txt"
    assert cli.main(["fit", str(target), "-n", "30", "--iters", "60", "-o", str(out), "--loss-out",
                     str(losses)]) == 0
    hist = [float(x) for x in losses.read_text().split()]
    assert len(hist) == 60 and hist[-1] < hist[0]
    scene, cam, bg = cli.parse_scene(out.read_text())
    assert len(scene) == 30 and cam.width == 32 and cam.height == 24
    res = api.render(scene, cam, bg)
    assert res.image.channels.shape == (24, 32, 3)
    assert cli.main(["fit", str(tmp_path / "none.ppm"), "-o", str(out)]) == 2
