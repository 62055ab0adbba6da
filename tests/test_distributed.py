"""View sharding + the one all-reduce per step, on CPU with gloo (world size 2).

The multi-GPU step (paper_2107_12672_b200/distributed.py) deals views
round-robin to ranks and sums [d_volume | d_tf | d_dt | loss] with one
all-reduce.  Here each rank computes its views' gradients with the CPU oracle
(the kernels need a GPU) and the real FlatGrads packing + torch.distributed
collective combine them; the result must equal the single-process sum over all
views, i.e. the reference's view-ordered sum (tasks.py:266-268, 428-430).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2107_12672_b200.distributed import FlatGrads, shard_views


def test_shard_views_partition():
    for n_views, world in ((64, 1), (64, 2), (64, 8), (7, 3), (3, 8)):
        shards = [shard_views(n_views, r, world) for r in range(world)]
        flat = sorted(v for s in shards for v in s)
        assert flat == list(range(n_views))
        sizes = [len(s) for s in shards]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_views(4, 2, 2)


def test_flatgrads_views():
    f = FlatGrads.zeros(10, 8, "cpu")
    f.d_volume[:] = 1.0
    f.d_tf[:] = 2.0
    f.d_stepsize[:] = 3.0
    f.loss[:] = 4.0
    assert f.buf.shape == (10,) and f.buf.dtype == torch.float32
    assert f.tail.shape == (10,) and f.tail.dtype == torch.float64
    assert f.buf.sum() == 10 and f.tail[:8].sum() == 16
    assert f.tail[8] == 3 and f.tail[9] == 4
    f.zero_()
    assert f.buf.abs().sum() == 0 and f.tail.abs().sum() == 0


def _scene():
    from oracle import dvr_oracle as O
    rng = np.random.default_rng(3)
    vol = rng.uniform(0.1, 0.9, (6, 6, 6)).astype(np.float32).astype(np.float64)
    tex = rng.uniform(0.2, 1.5, (8, 4)).astype(np.float32).astype(np.float64)
    poses = [(20.0 + 47.0 * k, -30.0 + 17.0 * k) for k in range(5)]
    views = [O.View(lon, lat, 2.3, width=6, height=5) for lon, lat in poses]
    refs = [rng.uniform(0, 1, (5, 6, 4)) for _ in views]
    return O.Grid(vol), tex, views, refs, 0.09


def _rank_grads(rank, world):
    """This rank's share: forward, L1 seed over the GLOBAL count, adjoint; oracle math."""
    from oracle import dvr_oracle as O
    grid, tex, views, refs, dt = _scene()
    count = sum(r.size for r in refs)
    flat = FlatGrads.zeros(grid.flat.size, tex.size, "cpu")
    loss = 0.0
    for v in shard_views(len(views), rank, world):
        img = O.render_view(grid, tex, views[v], dt)
        loss += float(np.abs(img - refs[v]).sum()) / count
        seed = np.sign(img - refs[v]) / count
        g = O.adjoint_view(grid, tex, views[v], dt, seed, ["volume", "tf", "stepsize"], image=img)
        flat.d_volume.add_(torch.from_numpy(g["d_volume"].ravel().astype(np.float32)))
        flat.d_tf.add_(torch.from_numpy(g["d_tf"].ravel()))
        flat.d_stepsize.add_(float(g["d_stepsize"]))
    flat.loss.add_(loss)
    return flat


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        flat = _rank_grads(rank, world)
        flat.allreduce()
        if rank == 0:
            torch.save((flat.buf.clone(), flat.tail.clone()), out_path)   # (views of one buffer)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_allreduce_equals_single_process_sum(tmp_path):
    world = 2
    out = str(tmp_path / "buf.pt")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    got, got_tail = torch.load(out)
    full = _rank_grads(0, 1)             # one process, every view
    assert torch.allclose(got, full.buf, rtol=1e-5, atol=1e-7)
    # the fp64 tail is summed in fp64 (no fp32 round trip)
    assert torch.allclose(got_tail, full.tail, rtol=1e-12, atol=1e-15)
    # and the shards really split the work: each rank alone is not the total
    part = _rank_grads(0, world)
    assert not torch.allclose(part.buf, full.buf)
