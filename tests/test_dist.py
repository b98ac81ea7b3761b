"""CPU: multi-process sharding logic (paper_2312_02121_b200.dist) with gloo,
world_size 2, checked against the fp64 oracle:

* view sharding: each rank renders its views, the gradient all-reduce equals
  the serial sum over all views (BASELINE config 3's decomposition);
* tile-band sharding: each rank renders a band camera, band images tile the
  full frame and the all-reduced band gradients equal the full frame's
  (BASELINE config 4's decomposition).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle as O
from paper_2312_02121_b200 import dist as D
from paper_2312_02121_b200.scenes import CameraSpec, look_at
from parity import load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_views_partition():
    for world in (1, 2, 3, 4, 8):
        got = sorted(v for r in range(world) for v in D.shard_views(32, world, r))
        assert got == list(range(32))


def test_band_rows_cover_and_balance():
    rng = np.random.default_rng(0)
    for height in (16, 100, 2160):
        n_rows = (height + 15) // 16
        work = rng.integers(0, 1000, size=n_rows).astype(float)
        for world in (1, 2, 4, 8):
            bands = D.band_rows(work, world, height)
            assert len(bands) == world
            assert bands[0][0] == 0 and bands[-1][1] == height
            for (a0, a1), (b0, b1) in zip(bands[:-1], bands[1:]):
                assert a1 == b0 and a0 <= a1
            for a0, _ in bands:
                assert a0 % 16 == 0 or a0 == height
            if world <= n_rows and work.sum() > 0:
                per = [work[a0 // 16:(a1 + 15) // 16].sum() for a0, a1 in bands]
                assert max(per) <= work.sum() / world + work.max() + 1e-9


def _scene():
    g = load_golden("cfg0_mini")
    return g["inputs"], g["camera"]


def _views(cam, n):
    out = []
    for k in range(n):
        th = 2 * np.pi * k / n
        c = (4.0 * np.sin(th), 0.3 * np.cos(th), -4.0 * np.cos(th))
        out.append(O.Camera(look_at(c), cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, cam.near, cam.far))
    return out


def _grads(inputs, cam, d_image):
    fw = O.render(*inputs, cam, np.zeros(3), True, nthreads=1)
    sb = O.scene_backward(*inputs, cam, np.zeros(3), fw, d_image, nthreads=1)
    n = len(inputs[0])
    flat = np.zeros((n, D.GRAD_COLS))
    flat[:, 0:3], flat[:, 3:6], flat[:, 6:10] = sb["d_mean"], sb["d_scale"], sb["d_quat"]
    flat[:, 10:13], flat[:, 13] = sb["d_color"], sb["d_opacity"]
    return fw, flat, sb["d_view"]


def _worker(rank, world, port, mode, out_path):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    inputs, cam = _scene()
    rng = np.random.default_rng(5)
    if mode == "views":
        views = _views(cam, 4)
        dimgs = [rng.normal(size=(cam.height, cam.width, 3)) for _ in views]
        flat = torch.zeros((len(inputs[0]), D.GRAD_COLS), dtype=torch.float64)
        for v in D.shard_views(len(views), world, rank):
            _, f, _ = _grads(inputs, views[v], dimgs[v])
            flat += torch.from_numpy(f)
        D.allreduce_grads(flat)
        extra = torch.zeros(1, dtype=torch.float64)
    else:
        d_image = rng.normal(size=(cam.height, cam.width, 3))
        work = np.ones((cam.height + 15) // 16)
        r0, r1 = D.band_rows(work, world, cam.height)[rank]
        bcam = D.band_camera(cam, r0, r1)
        fw, f, dv = _grads(inputs, bcam, d_image[r0:r1])
        flat = torch.from_numpy(f)
        D.allreduce_grads(flat)
        dvt = torch.from_numpy(dv.copy())
        D.allreduce_grads(dvt)
        img = torch.zeros((cam.height, cam.width, 3), dtype=torch.float64)
        img[r0:r1] = torch.from_numpy(fw["image"])
        D.allreduce_grads(img)
        extra = torch.cat([dvt.reshape(-1), img.reshape(-1)])
    if rank == 0:
        torch.save({"flat": flat, "extra": extra}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def _run(mode, tmp_path):
    out = str(tmp_path / f"{mode}.pt")
    mp.spawn(_worker, args=(2, _free_port(), mode, out), nprocs=2, join=True)
    return torch.load(out)


def test_view_sharded_allreduce_gloo(tmp_path):
    res = _run("views", tmp_path)
    inputs, cam = _scene()
    rng = np.random.default_rng(5)
    views = _views(cam, 4)
    dimgs = [rng.normal(size=(cam.height, cam.width, 3)) for _ in views]
    ref = sum(_grads(inputs, v, d)[1] for v, d in zip(views, dimgs))
    np.testing.assert_allclose(res["flat"].numpy(), ref, rtol=1e-10, atol=1e-12)


def test_band_sharded_allreduce_gloo(tmp_path):
    res = _run("bands", tmp_path)
    inputs, cam = _scene()
    rng = np.random.default_rng(5)
    d_image = rng.normal(size=(cam.height, cam.width, 3))
    fw, ref, dv = _grads(inputs, cam, d_image)
    extra = res["extra"].numpy()
    np.testing.assert_allclose(extra[:16].reshape(4, 4), dv, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(extra[16:].reshape(cam.height, cam.width, 3), fw["image"], atol=1e-12)
    scale = np.abs(ref).max(axis=0, keepdims=True) + 1e-30
    assert np.max(np.abs(res["flat"].numpy() - ref) / scale) < 1e-9
