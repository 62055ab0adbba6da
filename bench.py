#!/usr/bin/env python
"""Benchmark: forward + adjoint DiffDVR step, samples/s and rays/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

Workload (default C4, BASELINE.json configs[3]): absorption tomography, 256^3
sphere phantom, 64 views at 512x512, dt = 0.2 voxel, absorption-ramp TF
(R=64, tau 3), gradients w.r.t. the density.  One step = one optimisation
iteration of the reference's tomography loop (tasks.py:397-481): cell-record
pack, forward march of the rank's views, fused L1 loss/seed, adjoint
(inversion trick), the all-reduce of [d_volume | fp64 tail] (N > 1),
smoothness prior, Adam + [0,1] projection -- all libddvr kernels.

Fixed state: every timed step (and every e2e step) starts from the SAME
estimate -- iteration 1 of the optimisation, 0.85 * truth + 0.1 * U(0,1),
which has no exact zeros (dense: the empty-space skips find nothing) -- with
the Adam moments reset, so the number does not depend on --steps/--warmup.
Extra keys time the tape-free walk and a converged (sparse) estimate the same
way and count the samples the skips actually marched (device counters).

Views are dealt round-robin to ranks; the total work is fixed (strong
scaling).  ``python bench.py --gpus N`` outside torchrun re-launches itself
under torch.distributed.run with N ranks (NCCL, one GPU per rank).

Own arm: device-timed with CUDA events, L2 flushed (512 MiB write) before
every timed step, max over ranks.  ``e2e`` repeats the step through the
public API with host (pinned) buffers: H2D of the volume and the rank's
reference images and D2H of the updated volume and the loss inside the timed
region (same fixed state as ``value``).

``--impl reference``: the reference algorithm on the host CPU (the fp64 NumPy
oracle restatement, oracle/dvr_oracle.py -- voldiff itself is pure Python and
cannot travel), one row band per core, on a bounded sample of the same
workload, extrapolated; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# algorithmic bytes (SURVEY.md 8d / BASELINE.md 3): fp32 density, 8 corners, no reuse
FWD_B_PER_SAMPLE, FWD_B_PER_RAY = 32, 16
ADJ_B_PER_SAMPLE = {"volume": 64, "tf": 32, "camera": 32, "stepsize": 32}
ADJ_B_PER_RAY = 32
NCU_FILE = os.path.join(ROOT, "profiles", "ncu_r02.json")


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="C4")
    p.add_argument("--impl", default="own", choices=["own", "reference"])
    p.add_argument("--cpu-seconds", type=float, default=15.0,
                   help="target CPU time of the cpu_baseline sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extras", action="store_true",
                   help="skip the tape-free / sparse-state / e2e legs (profiling runs)")
    p.add_argument("--sparse-iters", type=int, default=24,
                   help="optimisation iterations before the sparse-state measurement")
    p.add_argument("--views", type=int, default=0,
                   help="profiling aid: use only the first N views (not a bench result)")
    p.add_argument("--layout", default="cells", choices=["cells", "voxels"])
    p.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                   help="replay each timed iteration from a captured CUDA graph (1 GPU); "
                        "auto: on for launch-bound steps (density target, < 1e7 samples)")
    p.add_argument("--unfused", action="store_true",
                   help="separate forward / L1 / adjoint launches instead of the fused step")
    p.add_argument("--fused", action="store_true",
                   help="the fused step also for camera / stepsize targets with the TF target")
    p.add_argument("--no-empty-skip", action="store_true",
                   help="band tape without the empty-brick skip of the march")
    p.add_argument("--no-band-tape", action="store_true",
                   help="fused absorption step without the 1-bit-per-sample band tape "
                        "(DDVR_FLAG_BAND_TAPE; the walk then re-gathers the cell records)")
    p.add_argument("--deterministic", action="store_true",
                   help="bitwise-reproducible gradients (DDVR_FLAG_DETERMINISTIC: int64 "
                        "fixed-point cell moments, fixed-order camera / stepsize sums)")
    p.add_argument("--split-walk", action="store_true",
                   help="band tape: march and walk as two kernels (DDVR_FLAG_SPLIT_WALK)")
    p.add_argument("--ray-split", default="auto", choices=["auto", "1", "2", "4", "8"],
                   help="fused TF-target steps: threads per ray (DDVR_FLAG_RAY_SPLIT_*; auto "
                        "splits steps too small to fill the GPU, e.g. C1)")
    p.add_argument("--sort-views", action="store_true",
                   help="experiment: order the views by direction (latitude bands, then "
                        "longitude) so that neighbouring views are similar")
    p.add_argument("--dry-run", action="store_true",
                   help="launcher / collective check without kernels (gloo on CPU if no GPU)")
    return p.parse_args(argv)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy-based burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


RED_SECTORS_PEAK = 2 * 93.9e9   # profiles/r02_bulk_red_probe.txt, 64 MB, mode 0


def ncu_entry(config, kernel):
    """The committed ncu --set full numbers of one kernel launch at the bench's fixed
    state (tools/ncu_summary.py --json-out), or None."""
    try:
        with open(NCU_FILE) as f:
            return json.load(f).get(f"{config}/{kernel}")
    except Exception:
        return None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled every 10 ms through NVML
    in a background thread while the timed region runs (one sample at the start
    and one at the end at least, so even a 1 ms region has samples)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index, period=0.01):
        self.index, self.period = index, period
        self.samples = []
        self._stop = threading.Event()
        self._nvml = None

    def _sample(self):
        import pynvml as nv
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        try:
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        self.samples.append((sm, rs))

    def _loop(self):
        while not self._stop.wait(self.period):
            try:
                self._sample()
            except Exception:
                return

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nvml = nv
            idx = self.index
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                try:
                    idx = int(vis.split(",")[self.index])
                except ValueError:
                    pass
            self._h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._sample()
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
        except Exception:
            self._nvml = None
        return self

    def __exit__(self, *exc):
        if self._nvml is not None:
            try:
                self._sample()
            except Exception:
                pass
            self._stop.set()
            self._t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "source": "nvml unavailable"}
        reasons = sorted({n for _, rs in self.samples for n, bit in self.REASONS.items()
                          if rs & bit})
        return {"sm_mhz": float(np.median([s for s, _ in self.samples])),
                "sm_max_mhz": float(self.max_mhz), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml, 10 ms period"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args):
    """``--gpus N`` outside torchrun: re-launch this script under torch.distributed.run
    with N ranks on this node (the driver's own launch line), return its exit code."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def init_group(world, dev):
    """NCCL (GPU) or gloo (dry run on CPU) process group; NCCL logs its communicator
    setup (NCCL_DEBUG=INFO, INIT) so the rank count is visible in the output."""
    import torch.distributed as dist
    if dev.type == "cuda":
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    return dist


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle on the host cores
# ---------------------------------------------------------------------------


_CPU = {}


def _cpu_band(job):
    """One row band of one view: oracle forward march, then the adjoint from the image."""
    from oracle import dvr_oracle as O
    cfg, grid, tex = _CPU["cfg"], _CPU["grid"], _CPU["tex"]
    view_idx, r0, r1 = job
    lon, lat = cfg.view_poses()[view_idx]
    view = O.View(lon, lat, cfg.radius, fov_y_deg=cfg.fov, width=cfg.image, height=cfg.image)
    b = O.make_band(grid, view, cfg.dt, r0, r1)
    img, _ = O.march(grid, tex, b, cfg.dt)
    seed = np.random.default_rng(r0).normal(size=img.shape)   # dense: no zero-skipping
    O.adjoint_view(grid, tex, view, cfg.dt, seed, list(cfg.targets), image=img, rows=(r0, r1))
    return int(b.n.sum()), int(b.n.size)


def cpu_sample(cfg, target_seconds, cores=None):
    """Time fwd + adjoint of the CPU oracle on a bounded sample of the workload.

    The reference parallelises over row tiles (renderer.py:243-247) and views
    (tasks.py:106-110) with threads; its NumPy path is GIL-bound at these band
    sizes, so the port runs one row band per core in forked processes (a
    stronger baseline than threads).  The sample is ``cores`` central row
    bands of view 0, each sized for ~target_seconds of work at ~0.75 M
    samples/s per core.  Returns (samples/s, rays/s, cores, description).
    """
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    from oracle import dvr_oracle as O

    cores = cores or max(1, len(os.sched_getaffinity(0)))
    _CPU["cfg"] = cfg
    _CPU["grid"] = O.Grid(cfg.volume().astype(np.float64))
    _CPU["tex"] = cfg.texels()
    lon, lat = cfg.view_poses()[0]
    view = O.View(lon, lat, cfg.radius, fov_y_deg=cfg.fov, width=cfg.image, height=cfg.image)
    mid = cfg.image // 2
    per_row = int(O.make_band(_CPU["grid"], view, cfg.dt, mid, mid + 1).n.sum())
    rows = int(np.clip(target_seconds * 0.75e6 // max(per_row, 1), 1, max(1, cfg.image // cores)))
    r0 = max(0, mid - rows * cores // 2)
    jobs = [(0, a, min(a + rows, cfg.image)) for a in range(r0, min(r0 + rows * cores, cfg.image),
                                                            rows)]
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=len(jobs), mp_context=mp.get_context("fork")) as ex:
        res = list(ex.map(_cpu_band, jobs))
    el = time.perf_counter() - t0
    samples = sum(r[0] for r in res)
    rays = sum(r[1] for r in res)
    desc = (f"{cfg.name} view 0 rows [{jobs[0][1]},{jobs[-1][2]}) = {rays} rays, {samples} "
            f"samples, fwd+adjoint ({'+'.join(cfg.targets)}) in fp64 NumPy (oracle port), "
            f"{len(jobs)} row bands of {rows} rows on {len(jobs)} forked processes, {el:.1f} s")
    return samples / el, rays / el, len(jobs), desc


def cpu_baseline_json(cfg, sps, cores, desc):
    total = cfg_samples(cfg)
    return {"value": sps, "unit": "samples/s", "cores": cores, "kind": "port",
            "cpu_model": cpu_model(), "sample": desc, "extrapolated": True,
            "extrapolation": (f"samples/s of the central row bands of view 0; the full "
                              f"{cfg.name} step ({total} samples) would take "
                              f"{total / sps:.0f} s at this rate" if total else None)}


def cfg_samples(cfg):
    """Sum of the reference's step counts over every ray of the config."""
    try:
        with np.load(os.path.join(ROOT, "tests", "golden", "counts.npz")) as z:
            return int(z[cfg.name + "_samples"])
    except Exception:
        return None


def run_reference(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    vals = []
    for i in range(args.warmup + args.steps):
        sps, rps, cores, desc = cpu_sample(cfg, args.cpu_seconds / 2)
        if i >= args.warmup:
            vals.append((sps, rps, cores, desc))
    sps = float(np.mean([v[0] for v in vals]))
    rps = float(np.mean([v[1] for v in vals]))
    line = {
        "impl": "reference",
        "metric": "fwd+adjoint samples/s", "value": sps, "unit": "samples/s",
        "rays_per_s": rps, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_json(cfg, args.gpus),
        "cpu_baseline": cpu_baseline_json(cfg, sps, vals[-1][2], vals[-1][3]),
        "e2e": {"value": sps, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_json(cfg, n):
    return {"workload": f"{cfg.name}: {cfg.title}", "volume": [cfg.vol_dim] * 3,
            "image": [cfg.image, cfg.image], "views": cfg.views, "dt_voxels": cfg.dt_vox,
            "tf": list(map(str, cfg.tf)), "targets": list(cfg.targets),
            "parallelism": f"views round-robin over {n} GPU(s), all-reduce of the gradients",
            "l2": "flushed before every timed step (512 MiB write)"}


# ---------------------------------------------------------------------------
# own arm
# ---------------------------------------------------------------------------


def run_dry(args, cfg):
    """Launcher / collective check without kernels: every rank fills its share of the
    flat gradient buffers, one all-reduce, rank 0 prints a JSON line with the sums."""
    import torch

    from paper_2107_12672_b200.distributed import FlatGrads, shard_views
    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    dev = torch.device("cuda", local) if torch.cuda.is_available() else torch.device("cpu")
    # (under torchrun even one rank forms the process group: the collectives then run)
    dist = init_group(world, dev) if world > 1 or "WORLD_SIZE" in os.environ else None
    mine = shard_views(cfg.views, rank, world)
    f = FlatGrads.zeros(1024, 16, dev)
    t0 = time.perf_counter()
    for v in mine:   # a stand-in per-view contribution (view index + 1)
        f.d_volume.add_(float(v + 1))
        f.d_tf.add_(float(v + 1))
        f.loss.add_(float(v + 1))
    f.allreduce()
    el = time.perf_counter() - t0
    if rank == 0:
        print(json.dumps({"metric": "dry run", "dry_run": True, "n_gpus": world,
                          "backend": dist.get_backend() if dist else None,
                          "views_rank0": mine, "loss_sum": float(f.loss),
                          "expected": cfg.views * (cfg.views + 1) / 2,
                          "seconds": el}), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


class _Timer:
    """CUDA events on the launching stream around one step: start, post_forward,
    pre_adjoint, post_adjoint (ShardedStep hooks) and end."""

    KEYS = ("start", "post_forward", "pre_adjoint", "post_adjoint", "end")

    def __init__(self, torch):
        self.torch = torch
        self.e = {k: torch.cuda.Event(enable_timing=True) for k in self.KEYS}

    def rec(self, k):
        self.e[k].record(self.torch.cuda.current_stream())

    def ms(self, a, b):
        return self.e[a].elapsed_time(self.e[b])


def run_own(args, cfg):
    import torch

    from paper_2107_12672_b200 import _native as N
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.distributed import ShardedStep, TomographyIteration, shard_views

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # (under torchrun even one rank forms the process group: NCCL init and the
    # max-over-ranks / all-reduce collectives run)
    dist = init_group(world, dev) if world > 1 or "WORLD_SIZE" in os.environ else None
    N.lib()

    # --- synthetic inputs of the named shape ---
    truth = torch.from_numpy(cfg.volume()).to(dev)
    tex = torch.from_numpy(cfg.texels().astype(np.float32)).to(dev)
    poses = cfg.view_poses()
    if args.sort_views:   # latitude bands of 22.5 degrees, serpentine in longitude
        def _key(p):
            band = int((p[1] + 90.0) // 22.5)
            return (band, p[0] if band % 2 == 0 else -p[0])
        poses = sorted(poses, key=_key)
    if args.views:
        poses = poses[: args.views]
    mine = shard_views(len(poses), rank, world)
    ll = torch.tensor([poses[i] for i in mine], dtype=torch.float64, device=dev).reshape(-1, 2)
    rig = R.Rig(cfg.image, cfg.image)
    cams = R.camera_array(ll, cfg.radius, (0.0, 0.0, 0.0), cfg.fov)
    refs, _ = R.forward(truth, tex, cams, cfg.dt, rig, with_depth=False,
                        cells=R.pack_cells(truth) if args.layout == "cells" else None)
    g = torch.Generator(device=dev).manual_seed(7)
    # the fixed state every timed step starts from: iteration 1, no exact zeros
    est0 = (0.85 * truth + 0.1 * torch.rand(truth.shape, generator=g, device=dev)).contiguous()
    est = est0.clone()
    total_elems = 4 * cfg.image * cfg.image * len(poses)
    volume_target = "volume" in cfg.targets

    def make_step(band_tape):
        return ShardedStep(est, tex, ll, refs, cfg.dt, rig, targets=cfg.targets,
                           total_elements=total_elems, radius=cfg.radius, fov_y_deg=cfg.fov,
                           layout=args.layout,
                           fused=False if args.unfused else (True if args.fused else "auto"),
                           band_tape=band_tape, empty_skip=not args.no_empty_skip,
                           split_walk=args.split_walk, deterministic=args.deterministic,
                           ray_split=args.ray_split if args.ray_split == "auto"
                           else int(args.ray_split))

    step = make_step(False if args.no_band_tape else "auto")
    small = cfg_samples(cfg) is not None and cfg_samples(cfg) < 10 ** 7
    graphed = (args.graph == "on" or (args.graph == "auto" and small)) and world == 1 \
        and volume_target and not args.views
    # density targets run the whole optimisation iteration (prior + Adam + projection)
    runner = (TomographyIteration(step, lr=0.02, lam=0.5, graph=graphed) if volume_target
              else step)

    def restore(state):
        """Back to a fixed state: the estimate (and Adam's moments / step counter)."""
        if runner is step:
            est.copy_(state)
        else:
            runner.reset(state)

    _, n_steps, _ = R.ray_setup(cams, cfg.dt, rig, dims=tuple(truth.shape))
    local_samples = int(n_steps.to(torch.int64).sum().item())
    local_rays = n_steps.numel()
    t = torch.tensor([local_samples, local_rays], dtype=torch.int64, device=dev)
    if dist:
        dist.all_reduce(t)
    total_samples, total_rays = int(t[0]), int(t[1])
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        v = torch.tensor([x], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    def timed_steps(r, state, n, clk=None):
        """n steps of runner ``r``, each from ``state``; per-step _Timer list."""
        out = []
        for _ in range(n):
            restore(state)
            flush.zero_()
            barrier()
            torch.cuda.synchronize()
            tm = _Timer(torch)
            tm.rec("start")
            if graphed and r is runner:        # one replay: no per-kernel events inside
                r.run()
                for k in ("post_forward", "pre_adjoint", "post_adjoint"):
                    tm.rec(k)
            else:
                r.run(hook=tm.rec)
            tm.rec("end")
            torch.cuda.synchronize()
            out.append(tm)
        return out

    def count_samples(s, state):
        """Samples / skipped samples of one (untimed) step at ``state``: device counters."""
        if not getattr(s, "fused", False):
            return None
        stats = torch.zeros(4, dtype=torch.int64, device=dev)
        s.stats = stats
        restore(state)
        s.run()
        torch.cuda.synchronize()
        s.stats = None
        c = [int(x) for x in stats.cpu()]
        return {"samples": c[0], "march_skipped": c[1], "walk_skipped": c[2],
                "samples_marched": c[0] - c[1], "samples_walked": c[0] - c[2], "rays": c[3]}

    for _ in range(args.warmup):
        restore(est0)
        runner.run()
    torch.cuda.synchronize()

    launches0 = N.launch_count()
    with ClockSampler(local) as clk:
        tms = timed_steps(runner, est0, args.steps)
    launches = N.launch_count() - launches0
    step_ms = [tm.ms("start", "end") for tm in tms]
    fwd_ms = [tm.ms("start", "post_forward") for tm in tms]
    adj_ms = [tm.ms("pre_adjoint", "post_adjoint") for tm in tms]
    if graphed:   # replays launch the captured kernels; the breakdown comes from eager steps
        launches = runner.graph_launches * args.steps
        eager = TomographyIteration(step, lr=0.02, lam=0.5)
        eager.adam = runner.adam
        tm2 = timed_steps(eager, est0, max(2, args.steps))
        fwd_ms = [tm.ms("start", "post_forward") for tm in tm2]
        adj_ms = [tm.ms("pre_adjoint", "post_adjoint") for tm in tm2]
    ms_per_step = max_over_ranks(sum(step_ms)) / args.steps
    counts = count_samples(step, est0)

    # gather roofline: the same rays and held record gathers, one FADD
    # per sample (ddvr_gather_probe), at the same dense state, timed like the kernels
    probe_ms = None
    if step.cells is not None:
        restore(est0)
        R.pack_cells(step.density, step.cells)
        pm = []
        for _ in range(3):
            flush.zero_()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            R.gather_probe(step.density, step.cams, cfg.dt, rig, step.cells, hold=True)
            b.record()
            torch.cuda.synchronize()
            pm.append(a.elapsed_time(b))
        probe_ms = float(np.median(pm))

    extras = {}
    fused = getattr(step, "fused", False)
    band = getattr(step, "band_tape", False)
    if not args.no_extras and volume_target and fused and not graphed:
        # the inversion-only (tape-free) walk: O(pixels) memory, the paper's contract
        if band:
            nt = make_step(False)
            it = TomographyIteration(nt, lr=0.02, lam=0.5)
            for _ in range(max(1, args.warmup)):
                it.reset(est0)
                it.run()
            r_ms = max_over_ranks(sum(tm.ms("start", "end")
                                      for tm in _timed_with(it, est0, args.steps, flush, barrier,
                                                            torch))) / args.steps
            extras["tape_free"] = {
                "value": total_samples / (r_ms / 1e3), "ms_per_step": r_ms,
                "walk": "inversion-only walk: re-gathers the cell records back to front, "
                        "no per-sample tape (O(pixels) state)",
                "workspace_bytes": int(nt.workspace.numel() * 4)}
            del nt, it
            torch.cuda.empty_cache()
        # a converged estimate: the optimisation grows exact zeros outside the object,
        # which the empty-space skips step over (the data-dependent speed-up)
        restore(est0)
        for _ in range(args.sparse_iters):
            runner.run()
        torch.cuda.synchronize()
        est_sparse = est.clone()
        sp = timed_steps(runner, est_sparse, args.steps)
        sp_ms = max_over_ranks(sum(tm.ms("start", "end") for tm in sp)) / args.steps
        extras["sparse_state"] = {
            "value": total_samples / (sp_ms / 1e3), "ms_per_step": sp_ms,
            "state": f"estimate after {args.sparse_iters} iterations from the dense state "
                     f"(restored before every timed step; Adam moments reset)",
            "zero_voxels_frac": float((est_sparse == 0).float().mean()),
            "counts": count_samples(step, est_sparse)}

    # --- e2e through the public API with host buffers, same fixed state ---
    e2e = None
    if not args.no_extras:
        host_vol = torch.empty(est.shape, dtype=torch.float32, pin_memory=True)
        host_vol.copy_(est0.cpu())
        host_refs = torch.empty(refs.shape, dtype=torch.float32, pin_memory=True)
        host_refs.copy_(refs.cpu())
        # the step's result: the updated density after an optimiser step (volume
        # targets), else the gradients it computes (fp64 tail, per-view camera)
        if runner is not step:
            result = est.reshape(-1)
        else:
            result = torch.cat([step.flat.tail, step.d_camera.reshape(-1)]) \
                if step.mask & 1 else step.flat.tail
        host_res = torch.empty(result.numel(), dtype=result.dtype, pin_memory=True)
        host_loss = torch.empty(1, dtype=torch.float64, pin_memory=True)
        e2e_ms = []
        for i in range(args.warmup + args.steps):
            restore(est0)
            flush.zero_()
            barrier()
            torch.cuda.synchronize()
            st = torch.cuda.current_stream()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            est.copy_(host_vol, non_blocking=True)
            if graphed:   # the graph reads step.refs: copy first, then replay
                refs.copy_(host_refs, non_blocking=True)
                runner.run()
            else:
                runner.run(refs_host=host_refs)  # refs H2D overlaps pack + forward
            if runner is step:
                result = torch.cat([step.flat.tail, step.d_camera.reshape(-1)]) \
                    if step.mask & 1 else step.flat.tail
            host_res.copy_(result, non_blocking=True)
            host_loss.copy_(step.flat.loss, non_blocking=True)
            b.record(st)
            torch.cuda.synchronize()
            if i >= args.warmup:
                e2e_ms.append(a.elapsed_time(b))
        e2e_ms_step = max_over_ranks(sum(e2e_ms)) / args.steps
        e2e = {"value": total_samples / (e2e_ms_step / 1e3), "unit": "samples/s",
               "ms_per_step": e2e_ms_step,
               "h2d_bytes_per_step": host_vol.numel() * 4 + host_refs.numel() * 4,
               "d2h_bytes_per_step": host_res.numel() * host_res.element_size() + 8,
               "state": "the same fixed state as value (restored before every step)"}

    if rank == 0:
        line = report(args, cfg, step, runner, world, mine, total_samples, total_rays,
                      local_samples, local_rays, ms_per_step, fwd_ms, adj_ms, probe_ms, counts,
                      extras, e2e, launches, clk, graphed)
        if world == 1 and not args.no_cpu_baseline:
            sps, _, cores, desc = cpu_sample(cfg, args.cpu_seconds)
            line["cpu_baseline"] = cpu_baseline_json(cfg, sps, cores, desc)
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def _timed_with(r, state, n, flush, barrier, torch):
    out = []
    for _ in range(n):
        r.reset(state)
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        tm = _Timer(torch)
        tm.rec("start")
        r.run(hook=tm.rec)
        tm.rec("end")
        torch.cuda.synchronize()
        out.append(tm)
    return out


def report(args, cfg, step, runner, world, mine, total_samples, total_rays, local_samples,
           local_rays, ms_per_step, fwd_ms, adj_ms, probe_ms, counts, extras, e2e, launches,
           clk, graphed):
    peak, peak_src = peaks()
    fused = getattr(step, "fused", False)
    band = getattr(step, "band_tape", False)
    adj_b = max(ADJ_B_PER_SAMPLE[t] for t in cfg.targets)
    adj_bytes = adj_b * local_samples + ADJ_B_PER_RAY * local_rays
    fwd_bytes = FWD_B_PER_SAMPLE * local_samples + FWD_B_PER_RAY * local_rays
    adj_s = float(np.mean(adj_ms)) / 1e3
    fwd_s = float(np.mean(fwd_ms)) / 1e3
    if fused:   # one kernel marches forward, forms the L1 seed and walks back
        adj_bytes += fwd_bytes
        adj_b += FWD_B_PER_SAMPLE
    ray_b = ADJ_B_PER_RAY + (FWD_B_PER_RAY if fused else 0)
    kkey = ("fused_tape" if band else "fused") if fused else "adjoint"
    kname = ("dvr_adjoint_kernel<FUSED> (forward + L1 seed + adjoint per ray)" if fused
             else "dvr_adjoint_kernel")
    nc = ncu_entry(cfg.name, kkey)
    model_gbs = adj_bytes / adj_s / 1e9
    roof = {"bound": "hbm", "kernel": kname, "peak": peak, "unit": "GB/s",
            "peak_source": peak_src, "launch_ms": adj_s * 1e3,
            "model_bytes_per_launch": adj_bytes,
            "model": f"{adj_b} B/sample + {ray_b} B/ray (SURVEY 8d: 8 corner gathers "
                     f"(+8 scatters) per sample, no cache reuse)",
            "model_achieved": model_gbs, "model_frac": model_gbs / peak}
    if nc:
        traffic = float(nc["dram_bytes"]) * (local_samples / nc["samples"]
                                             if nc.get("samples") else 1.0)
        roof.update({
            "achieved": traffic / adj_s / 1e9, "frac": traffic / adj_s / 1e9 / peak,
            "traffic": traffic,
            "traffic_source": f"ncu --set full, one launch at the bench's fixed dense state "
                              f"({nc.get('file')}); achieved = that launch's DRAM bytes / the "
                              f"live launch time",
            "ncu": {k: nc[k] for k in ("issue_active_pct", "warp_inst_per_sample",
                                       "l1tex_pct", "l2_pct", "dram_pct",
                                       "red_requests_per_s", "gather_requests_per_sample",
                                       "occupancy_pct", "registers", "duration_ms")
                    if k in nc}})
        if nc.get("red_sectors") and nc["red_sectors"] / nc["duration_ms"] > 1e6:   # > 1 G/s
            # the kernel's density / TF gradient reds against the measured red ceiling:
            # 2 x red.v4 per 32-byte record into an L2-resident array, random records,
            # 94 G records/s = 188 G sectors/s (tools/probes/bulk_red_probe.cu mode 0,
            # profiles/r02_bulk_red_probe.txt)
            sectors = float(nc["red_sectors"]) * (local_samples / nc["samples"]
                                                  if nc.get("samples") else 1.0)
            roof["atomics"] = {
                "bound": "L2 reds", "sectors_per_launch": sectors,
                "achieved": sectors / adj_s, "peak": RED_SECTORS_PEAK, "unit": "sectors/s",
                "frac": sectors / adj_s / RED_SECTORS_PEAK,
                "peak_source": "measured: bulk_red_probe mode 0 (2 x red.v4 per 32-byte "
                               "record, random records, 64 MB L2-resident array)",
                "pct_of_l2_red_peak_ncu": nc.get("red_sectors_pct_of_l2_peak")}
    else:
        roof.update({"achieved": model_gbs, "frac": model_gbs / peak, "traffic": None,
                     "traffic_source": "no ncu capture of this kernel at this state: "
                                       "achieved = the byte model (not evidence)"})
    if fused:
        kernels = {"pack_cells": {"ms": fwd_s * 1e3},
                   "fused_forward_adjoint": {"ms": adj_s * 1e3},
                   "share_of_step": {"pack_cells": fwd_s * 1e3 / ms_per_step,
                                     "fused_forward_adjoint": adj_s * 1e3 / ms_per_step}}
    else:
        kernels = {"forward": {"ms": fwd_s * 1e3}, "adjoint": {"ms": adj_s * 1e3},
                   "share_of_step": {"forward": fwd_s * 1e3 / ms_per_step,
                                     "adjoint": adj_s * 1e3 / ms_per_step}}
    line = {
        "metric": "fwd+adjoint samples/s",
        "value": total_samples / (ms_per_step / 1e3),
        "unit": "samples/s",
        "rays_per_s": total_rays / (ms_per_step / 1e3),
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_json(cfg, world),
        "samples_per_step": total_samples, "rays_per_step": total_rays,
        "roofline": roof,
        "kernels": kernels,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if counts:
        line["counts"] = dict(counts, note="one untimed step at the same state, device "
                                           "counters (rank 0's views)")
    if probe_ms:
        probe_rate = local_samples / (probe_ms / 1e3)
        gr = {"probe": "ddvr_gather_probe: the same rays, fixed-point stepping and held "
                       "256-bit record gathers, one FADD per sample, every sample marched",
              "samples_per_s": probe_rate * world, "probe_ms": probe_ms}
        if fused:
            # the fused kernel gathers along every ray twice (forward + walk), or
            # once with the band tape (the walk reads 1 bit per sample instead)
            passes = 1 if band else 2
            gr["record_gather_passes"] = passes
            gr["fused_frac"] = local_samples / adj_s / probe_rate
            gr["fused_frac_per_gather_pass"] = passes * local_samples / adj_s / probe_rate
        else:
            gr["forward_frac"] = local_samples / fwd_s / probe_rate
            gr["adjoint_frac"] = local_samples / adj_s / probe_rate
        line["gather_roofline"] = gr
    line.update(extras)
    if runner is not step:
        line["config"]["state"] = (
            "fixed: every timed step is iteration 1 of the optimisation from 0.85*truth + "
            "0.1*U(0,1) (no exact zeros), estimate and Adam state restored before each step")
    line["config"]["step"] = (("fused forward+L1+adjoint" if fused else "forward, L1, adjoint") +
                              (", band tape (1 bit/sample, DDVR_FLAG_BAND_TAPE)" if band
                               else "") +
                              (", empty-brick skip in the march" if band and step.empty_skip
                               else "") +
                              (", deterministic (int64 cell moments)" if step.deterministic
                               else "") +
                              (", march and walk as two kernels" if band and step.split_walk
                               else "") + (", CUDA-graph replay" if graphed else ""))
    if len(mine) > 1:   # CTA order of the adjoint / fused kernels (cta_view_tile)
        line["config"]["cta_order"] = (f"view groups of {os.environ.get('DDVR_VGROUP', '4')} "
                                       f"views per tile")
    if fused:   # threads per ray of the fused kernel (DDVR_FLAG_RAY_SPLIT_*, ddvr_ray_split)
        from paper_2107_12672_b200 import _native as N
        sflags = (0 if step.ray_split == "auto" else N.FLAG_RAY_SPLIT[step.ray_split]) | \
            (N.FLAG_DETERMINISTIC if step.deterministic else 0)
        k = int(N.lib().ddvr_ray_split(step.mask, local_rays, sflags))
        line["config"]["lanes_per_ray"] = k
        if k > 1:
            line["config"]["step"] += f", {k} lanes per ray (segment-split rays)"
    if band:
        from paper_2107_12672_b200 import _native as N
        from paper_2107_12672_b200 import raymarch as R
        import ctypes
        vol, _, prm = R._descs(step.density, step.texels, step.rig, step.dt, False, step.cells)
        line["memory"] = {
            "band_tape_bytes": int(N.lib().ddvr_band_tape_bytes(ctypes.byref(vol), len(mine),
                                                                 ctypes.byref(prm))),
            "cells_bytes": int(step.cells.numel() * 4),
            "workspace_bytes": int(step.workspace.numel() * 4)}
    return line


def main():
    args = parse()
    rc = maybe_spawn(args)
    if rc is not None:
        sys.exit(rc)
    from paper_2107_12672_b200.scenes import CONFIGS
    cfg = CONFIGS[args.config]
    if args.dry_run:
        run_dry(args, cfg)
    elif args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_own(args, cfg)


if __name__ == "__main__":
    main()
