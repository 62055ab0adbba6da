"""bench.py's multi-rank launch path on CPU (gloo): ``python bench.py --gpus N`` outside
torchrun re-launches itself under torch.distributed.run with N ranks, the ranks
shard the views round-robin (tasks.py:106-110) and one all-reduce sums their
contributions; rank 0 alone prints the JSON line."""

from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stdout + p.stderr
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return [json.loads(ln) for ln in lines]


def test_gpus_2_spawns_two_ranks_and_reduces():
    out = _run("--gpus", "2", "--dry-run", "--steps", "1", "--warmup", "0")
    assert len(out) == 1, out                     # rank 0 only
    d = out[0]
    assert d["n_gpus"] == 2 and d["backend"] == "gloo"
    assert d["views_rank0"] == list(range(0, 64, 2))
    assert d["loss_sum"] == d["expected"]         # every view counted exactly once


def test_gpus_1_runs_in_process():
    out = _run("--gpus", "1", "--dry-run", "--config", "C2")
    assert len(out) == 1 and out[0]["n_gpus"] == 1
    assert out[0]["loss_sum"] == out[0]["expected"] == 36.0


def test_spawn_is_skipped_under_torchrun(monkeypatch):
    sys.path.insert(0, ROOT)
    import bench
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.maybe_spawn(bench.parse(["--gpus", "2"])) is None
    monkeypatch.delenv("WORLD_SIZE")
    assert bench.maybe_spawn(bench.parse(["--gpus", "1"])) is None
    assert bench.maybe_spawn(bench.parse(["--gpus", "4", "--impl", "reference"])) is None
