"""Multi-GPU sharding of the splatting step (one process per GPU).

Two decompositions, both exact because every quantity the backward sums is
linear in the per-pixel contributions (sg/proj_backward.py:206-222 is linear
in d_mean2d/d_cov2d; sg/raster_backward.py:166-205 sums over pixels):

* by camera view (BASELINE config 3): rank r renders views r, r+N, ...;
  Gaussian parameters are replicated and the per-Gaussian gradients
  (14 fp32: mean 3, scale 3, quat 4, color 3, opacity 1) are summed with one
  NCCL all-reduce.  d_view stays per camera.
* by horizontal tile bands of one large frame (BASELINE config 4): rank r
  renders the pixel rows [r0, r1) of the frame as a band camera -- same view
  and focal lengths, height r1 - r0, principal point cy - r0 (r0 a multiple of
  16, so tiles align).  Gaussians not reaching the band are culled by the
  ordinary off-screen rule; the per-tile lists are the full frame's lists for
  those tiles.  The band gradients (and d_view) sum to the full frame's.

The host-side logic (view assignment, balanced band split, the flat gradient
layout) is plain Python so it is tested on CPU with gloo (tests/test_dist.py).
"""

from __future__ import annotations

import math

import numpy as np

TILE = 16
GRAD_COLS = 14  # d_mean 3 | d_scale 3 | d_quat 4 | d_color 3 | d_opacity 1


def shard_views(n_views: int, world: int, rank: int) -> list:
    """Round-robin view assignment (every view exactly once across ranks)."""
    return list(range(rank, n_views, world))


def band_rows(tile_row_work, world: int, height: int) -> list:
    """Split the frame's tile rows into `world` contiguous bands of about equal
    work (e.g. intersections per tile row).  Every rank computes the same
    split from the same counts, so no exchange is needed.  Returns pixel-row
    ranges [(r0, r1), ...]; r0 is a multiple of 16; bands may be empty."""
    w = np.asarray(tile_row_work, dtype=np.float64)
    n_rows = len(w)
    assert n_rows == math.ceil(height / TILE)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        # first tile row whose prefix reaches the target, never before the previous cut
        t = int(np.searchsorted(cum, target, side="left"))
        t = min(max(t, cuts[-1]), n_rows)
        cuts.append(t)
    cuts.append(n_rows)
    return [(min(a * TILE, height), min(b * TILE, height)) for a, b in zip(cuts[:-1], cuts[1:])]


def band_camera(cam, r0: int, r1: int):
    """The band [r0, r1) of `cam` as a camera of its own (cy shifted)."""
    from dataclasses import replace
    return replace(cam, height=int(r1 - r0), cy=float(cam.cy) - float(r0))


def tile_row_work_from_projection(xydr, height: int, width: int):
    """Intersections per tile row from a projection (xydr rows, radius bits
    in .w, 0 = culled), computed on the device with torch."""
    import torch
    x, y = xydr[:, 0], xydr[:, 1]
    r = xydr[:, 3].contiguous().view(torch.int32)
    vis = r > 0
    tiles_x = (width + TILE - 1) // TILE
    tiles_y = (height + TILE - 1) // TILE
    rf = r.to(torch.float32)
    ty0 = torch.clamp(torch.floor((torch.floor(y) - rf) / TILE), 0, tiles_y - 1).long()
    ty1 = torch.clamp(torch.floor((torch.floor(y) + rf) / TILE), 0, tiles_y - 1).long()
    tx0 = torch.clamp(torch.floor((torch.floor(x) - rf) / TILE), 0, tiles_x - 1)
    tx1 = torch.clamp(torch.floor((torch.floor(x) + rf) / TILE), 0, tiles_x - 1)
    wx = (tx1 - tx0 + 1).clamp(min=0)
    diff = torch.zeros(tiles_y + 1, device=xydr.device, dtype=torch.float64)
    diff.index_add_(0, ty0[vis], wx[vis].double())
    diff.index_add_(0, ty1[vis] + 1, -wx[vis].double())
    return torch.cumsum(diff[:-1], 0).cpu().numpy()


def pack_grads(out, d_mean, d_scale, d_quat, d_color, d_opacity, accumulate=False):
    """Write (or add) one view's gradients into the flat (N, 14) buffer."""
    cols = ((0, 3, d_mean), (3, 6, d_scale), (6, 10, d_quat), (10, 13, d_color))
    for a, b, g in cols:
        if accumulate:
            out[:, a:b].add_(g)
        else:
            out[:, a:b].copy_(g)
    if accumulate:
        out[:, 13].add_(d_opacity)
    else:
        out[:, 13].copy_(d_opacity)
    return out


def allreduce_grads(flat, group=None):
    """Sum the flat per-Gaussian gradients over all ranks (NCCL on GPUs,
    gloo on CPU)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


# ------------------------------------------------------------------ device-side reductions
#
# View sharding (config 3): every rank accumulates its views' gradients into
# one flat buffer; the sum over ranks is an all-reduce of the 14 fp32 per
# Gaussian.  Only the LAST view's projection backward stands between the
# local sum and that reduction, so it runs in Gaussian buckets and each
# bucket's all-reduce starts as soon as the bucket is written (NCCL's stream
# waits for the launching stream at call time), overlapping the following
# buckets' projection backward.  Tile bands (config 4): the ranks hold
# disjoint pixel bands of one frame, so the screen-space gradients (9 fp32
# per Gaussian: d_color 3, d_opacity, d_mean2d 2, d_cov 3) are summed first
# and every rank then runs the projection backward on the summed rows
# (sg/proj_backward.py:206-222 is linear in them), ending with identical
# gradients and d_view on every rank.

def bucket_bounds(n: int, buckets: int, align: int = 256) -> list:
    """[a, b) Gaussian ranges of about equal size (multiples of `align`)."""
    buckets = max(1, int(buckets))
    per = (n + buckets - 1) // buckets
    step = max(align, (per + align - 1) // align * align)
    out, a = [], 0
    while a < n:
        b = min(n, a + step)
        out.append((a, b))
        a = b
    return out or [(0, 0)]


class GradReducer:
    """Sum the flat gradient buffer (engine.unpack layout) over ranks,
    overlapped with the last view's projection backward (`buckets` ranges)."""

    def __init__(self, n: int, buckets: int = 4, group=None):
        self.n = int(n)
        self.bounds = bucket_bounds(self.n, buckets)
        self.group = group

    def last_view(self, fr, params, out: dict, d_view, accumulate: bool) -> list:
        """Projection backward of the last view (after
        ops.frame_backward(project=False)) bucket by bucket, each bucket's
        4 gradient slices all-reduced asynchronously.  Returns the works."""
        import torch.distributed as dist
        from . import ops
        m, s, q = params[0], params[1], params[2]
        works = []
        for a, b in self.bounds:
            ops.frame_project_backward(fr, m, s, q, out, d_view, a, b, accumulate=accumulate, add_view=a > 0)
            for key in ("d_mean", "d_scale", "d_quat", "d_rgbo"):
                works.append(dist.all_reduce(out[key][a:b], op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        return works

    def views(self, frames, params, out: dict, d_views, accumulate: bool = False) -> list:
        """The batched projection backward of all of this rank's views (each
        after ops.frame_backward(project=False)) bucket by bucket, each
        bucket's 4 gradient slices all-reduced asynchronously.  Returns the
        works."""
        import torch.distributed as dist
        from . import ops
        m, s, q = params[0], params[1], params[2]
        works = []
        for a, b in self.bounds:
            ops.frame_views_project_backward(frames, m, s, q, out, d_views, a, b, accumulate=accumulate,
                                             add_view=a > 0)
            for key in ("d_mean", "d_scale", "d_quat", "d_rgbo"):
                works.append(dist.all_reduce(out[key][a:b], op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        return works

    @staticmethod
    def wait(works) -> None:
        for w in works:
            w.wait()


def band_backward(fr, params, d_image, out: dict, d_view, group=None) -> None:
    """Tile-band backward of one frame split over ranks: raster backward of
    this rank's band, sum of the 9 screen-space fp32 per Gaussian over
    ranks, then the projection backward of the summed rows (identical
    gradients and d_view on every rank)."""
    import torch.distributed as dist
    from . import ops
    m, s, q, _, c = params
    ops.frame_backward(fr, m, s, q, c, d_image, project=False)
    rows, c11 = ops.frame_screen_grads(fr)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(rows, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(c11, op=dist.ReduceOp.SUM, group=group)
    ops.frame_project_backward(fr, m, s, q, out, d_view, vis_from_grads=True)
