"""View-sharded tomography step with 2 ranks (distributed.ShardedStep).

Both ranks run on cuda:0 over the gloo backend: each rank's kernels are
independent (its own views, workspace and stream) and the one collective of
the step -- the all-reduce of [d_volume | d_tf | d_dt | loss] -- runs on the
host, so nothing on the device waits on the other rank.  The reduced
gradient and loss must equal the single-process step over all views, and
after one TomographyIteration both replicas hold the same volume.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs():
    import torch
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.scenes import absorption_ramp_texels, fibonacci_poses, phantom
    dev = torch.device("cuda", 0)
    truth = torch.from_numpy(phantom("sphere", 20, seed=0).astype(np.float32)).to(dev)
    tx = torch.from_numpy(absorption_ramp_texels(16, 3.0).astype(np.float32)).to(dev)
    ll = torch.tensor(fibonacci_poses(7), dtype=torch.float64, device=dev)
    rig = R.Rig(24, 24)
    cams = R.camera_array(ll, 2.0, (0.0, 0.0, 0.0), 30.0)
    refs, _ = R.forward(truth, tx, cams, 0.01, rig)
    est = (0.8 * truth + 0.05).contiguous()
    return est, tx, ll, refs, rig


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from paper_2107_12672_b200.distributed import ShardedStep, TomographyIteration, shard_views
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        est, tx, ll, refs, rig = _inputs()
        mine = shard_views(ll.shape[0], rank, world)
        step = ShardedStep(est, tx, ll[mine].contiguous(), refs[mine].contiguous(), 0.01, rig,
                           targets=("volume", "tf"), total_elements=refs.numel())
        f = step.run()
        torch.save(f.buf.cpu(), os.path.join(out_dir, f"grad{rank}.pt"))
        it = TomographyIteration(step, lr=0.05, lam=0.1)
        it.run()
        torch.save(est.cpu(), os.path.join(out_dir, f"vol{rank}.pt"))
    finally:
        dist.destroy_process_group()


def test_two_rank_step_equals_single_process(tmp_path):
    import torch
    import torch.multiprocessing as mp
    from conftest import rel_l2
    from paper_2107_12672_b200.distributed import ShardedStep
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    est, tx, ll, refs, rig = _inputs()
    single = ShardedStep(est, tx, ll, refs, 0.01, rig, targets=("volume", "tf")).run()
    g0 = torch.load(tmp_path / "grad0.pt")
    g1 = torch.load(tmp_path / "grad1.pt")
    assert torch.equal(g0, g1)                        # every rank holds the reduced sum
    assert rel_l2(g0.double().numpy(), single.buf.double().cpu().numpy()) <= 1e-5
    v0 = torch.load(tmp_path / "vol0.pt")
    v1 = torch.load(tmp_path / "vol1.pt")
    assert torch.equal(v0, v1)                        # replicas stay identical


def test_torchrun_single_rank_runs_nccl(tmp_path):
    """bench.py under torch.distributed.run with one rank on the GPU: the NCCL process
    group forms (its INIT log names the communicator: nranks 1) and the bench's
    collectives -- the sample-count all-reduce and the max-over-ranks step time -- run
    through NCCL; one JSON line comes out.  (The pool gives one GPU: N > 1 runs the same
    code with the view sharding the gloo tests cover.)"""
    import json
    import subprocess
    import sys
    from conftest import ROOT
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "bench.py"), "--gpus", "1", "--config", "C1", "--steps", "2",
           "--warmup", "3", "--no-extras", "--no-cpu-baseline"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env=dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT"))
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 0
    log = p.stdout + p.stderr
    assert "NCCL INFO" in log, log[-2000:]
    assert "nranks 1" in log.lower() or "nRanks 1" in log, log[-2000:]
