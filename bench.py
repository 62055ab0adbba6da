#!/usr/bin/env python
"""Benchmark: forward + adjoint DiffDVR step, samples/s and rays/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

Workload (default C4, BASELINE.json configs[3]): absorption tomography, 256^3
sphere phantom, 64 views at 512x512, dt = 0.2 voxel, absorption-ramp TF
(R=64, tau 3), gradients w.r.t. the density.  One step = one optimisation
iteration of the reference's tomography loop (tasks.py:397-481): cell-record
pack, forward march of the rank's views, fused L1 loss/seed, adjoint
(inversion trick), ONE all-reduce of [d_volume | d_tf | d_dt | loss] (N > 1),
smoothness prior, Adam + [0,1] projection -- all libddvr kernels.  Views are dealt round-robin to
ranks; the total work is fixed (strong scaling).  Synthetic data: the
reference images are rendered from the phantom, the optimised volume is a
perturbed copy.

Own arm: device-timed with CUDA events, L2 flushed (512 MiB write) before
every timed step, max over ranks.  ``e2e`` repeats the step through the public
API with host (pinned) buffers: H2D of the volume and the rank's reference
images and D2H of the updated volume and the loss inside the timed region.

``--impl reference``: the reference algorithm on the host CPU (the fp64 NumPy
oracle restatement, oracle/dvr_oracle.py -- voldiff itself is pure Python and
cannot travel), row-band thread pool like renderer.py:243-247, on a bounded
sample of the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# algorithmic bytes (SURVEY.md 8d / BASELINE.md 3): fp32 density, 8 corners, no reuse
FWD_B_PER_SAMPLE, FWD_B_PER_RAY = 32, 16
ADJ_B_PER_SAMPLE = {"volume": 64, "tf": 32, "camera": 32, "stepsize": 32}
ADJ_B_PER_RAY = 32


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="C4")
    p.add_argument("--impl", default="own", choices=["own", "reference"])
    p.add_argument("--cpu-seconds", type=float, default=15.0,
                   help="target CPU time of the cpu_baseline sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--views", type=int, default=0,
                   help="profiling aid: use only the first N views (not a bench result)")
    p.add_argument("--layout", default="cells", choices=["cells", "voxels"])
    p.add_argument("--graph", action="store_true",
                   help="replay each timed iteration from a captured CUDA graph (1 GPU)")
    p.add_argument("--unfused", action="store_true",
                   help="separate forward / L1 / adjoint launches instead of the fused step")
    p.add_argument("--no-empty-skip", action="store_true",
                   help="band tape without the empty-brick skip of the march")
    p.add_argument("--no-band-tape", action="store_true",
                   help="fused absorption step without the 1-bit-per-sample band tape "
                        "(DDVR_FLAG_BAND_TAPE; the walk then re-gathers the cell records)")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config, kernel):
    """dram read+write bytes per launch from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(config, {}).get(kernel)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


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
        "cpu_baseline": {"value": sps, "unit": "samples/s", "cores": vals[-1][2], "kind": "port",
                         "sample": vals[-1][3]},
        "e2e": {"value": sps, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_json(cfg, n):
    return {"workload": f"{cfg.name}: {cfg.title}", "volume": [cfg.vol_dim] * 3,
            "image": [cfg.image, cfg.image], "views": cfg.views, "dt_voxels": cfg.dt_vox,
            "tf": list(map(str, cfg.tf)), "targets": list(cfg.targets),
            "parallelism": f"views round-robin over {n} GPU(s), 1 all-reduce/step",
            "l2": "flushed before every timed step (512 MiB write)"}


# ---------------------------------------------------------------------------
# own arm
# ---------------------------------------------------------------------------


def run_own(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2107_12672_b200 import _native as N
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.distributed import ShardedStep, TomographyIteration, shard_views

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    N.lib()

    # --- synthetic inputs of the named shape ---
    truth = torch.from_numpy(cfg.volume()).to(dev)
    tex = torch.from_numpy(cfg.texels().astype(np.float32)).to(dev)
    poses = cfg.view_poses()
    if args.views:
        poses = poses[: args.views]
    mine = shard_views(len(poses), rank, world)
    ll = torch.tensor([poses[i] for i in mine], dtype=torch.float64, device=dev).reshape(-1, 2)
    rig = R.Rig(cfg.image, cfg.image)
    cams = R.camera_array(ll, cfg.radius, (0.0, 0.0, 0.0), cfg.fov)
    refs, _ = R.forward(truth, tex, cams, cfg.dt, rig, with_depth=False,
                        cells=R.pack_cells(truth) if args.layout == "cells" else None)
    g = torch.Generator(device=dev).manual_seed(7)
    est = (0.85 * truth + 0.1 * torch.rand(truth.shape, generator=g, device=dev)).contiguous()
    total_elems = 4 * cfg.image * cfg.image * len(poses)
    step = ShardedStep(est, tex, ll, refs, cfg.dt, rig, targets=cfg.targets,
                       total_elements=total_elems, radius=cfg.radius, fov_y_deg=cfg.fov,
                       layout=args.layout, fused=False if args.unfused else "auto",
                       band_tape=False if args.no_band_tape else "auto",
                       empty_skip=not args.no_empty_skip)
    # density targets run the whole optimisation iteration (prior + Adam + projection)
    graphed = args.graph and world == 1 and "volume" in cfg.targets
    runner = (TomographyIteration(step, lr=0.02, lam=0.5, graph=graphed)
              if "volume" in cfg.targets else step)
    _, n_steps, _ = R.ray_setup(cams, cfg.dt, rig, dims=tuple(truth.shape))
    local_samples = int(n_steps.to(torch.int64).sum().item())
    local_rays = n_steps.numel()
    t = torch.tensor([local_samples, local_rays], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(t)
    total_samples, total_rays = int(t[0]), int(t[1])
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    # per-kernel events on the launching stream: step start, forward end,
    # adjoint start, adjoint end, step end
    def timed_step(r=None):
        r = r or runner
        st = torch.cuda.current_stream()
        e = {k: torch.cuda.Event(enable_timing=True)
             for k in ("start", "post_forward", "pre_adjoint", "post_adjoint", "end")}
        e["start"].record(st)
        if graphed and r is runner:        # one replay: no per-kernel events inside
            runner.run()
            for k in ("post_forward", "pre_adjoint", "post_adjoint"):
                e[k].record(st)
        else:
            r.run(hook=lambda k: e[k].record(st))
        e["end"].record(st)
        return e

    for _ in range(args.warmup):
        runner.run()
    torch.cuda.synchronize()

    launches0 = N.launch_count()
    step_ms, fwd_ms, adj_ms = [], [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            torch.cuda.synchronize()
            e = timed_step()
            torch.cuda.synchronize()
            step_ms.append(e["start"].elapsed_time(e["end"]))
            fwd_ms.append(e["start"].elapsed_time(e["post_forward"]))
            adj_ms.append(e["pre_adjoint"].elapsed_time(e["post_adjoint"]))
    launches = N.launch_count() - launches0
    if graphed:   # replays launch the captured kernels; the breakdown comes from eager steps
        launches = runner.graph_launches * args.steps
        eager = TomographyIteration(step, lr=0.02, lam=0.5)
        fwd_ms, adj_ms = [], []
        for _ in range(max(2, args.steps)):
            flush.zero_()
            torch.cuda.synchronize()
            e = timed_step(eager)
            torch.cuda.synchronize()
            fwd_ms.append(e["start"].elapsed_time(e["post_forward"]))
            adj_ms.append(e["pre_adjoint"].elapsed_time(e["post_adjoint"]))
    # gather roofline: the same rays and held record gathers, one FADD
    # per sample (ddvr_gather_probe), timed like the kernels
    probe_ms = None
    if step.cells is not None:
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
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = float(tot.item()) / args.steps

    # --- e2e through the public API with host buffers ---
    host_vol = torch.empty(est.shape, dtype=torch.float32, pin_memory=True)
    host_vol.copy_(est.cpu())
    host_refs = torch.empty(refs.shape, dtype=torch.float32, pin_memory=True)
    host_refs.copy_(refs.cpu())
    # the step's result: the updated density after an optimiser step (volume
    # targets), else the gradients it computes (tf / stepsize flat tail, camera)
    if runner is not step:
        result = est.reshape(-1)
    else:
        tail = step.flat.buf[step.flat.d_volume.numel():]
        result = torch.cat([tail, step.d_camera.reshape(-1).float()]) \
            if step.mask & 1 else tail
    host_grad = torch.empty(result.numel(), dtype=torch.float32, pin_memory=True)
    host_loss = torch.empty(1, dtype=torch.float32, pin_memory=True)
    e2e_ms = []
    for i in range(args.warmup + args.steps):
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
        f = step.flat
        if runner is step:
            tail = f.buf[f.d_volume.numel():]
            result = torch.cat([tail, step.d_camera.reshape(-1).float()]) \
                if step.mask & 1 else tail
        host_grad.copy_(result, non_blocking=True)
        host_loss.copy_(f.loss, non_blocking=True)
        b.record(st)
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
    te = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms_step = float(te.item()) / args.steps
    h2d = host_vol.numel() * 4 + host_refs.numel() * 4
    d2h = host_grad.numel() * 4 + 4

    if rank == 0:
        peak, peak_src = peaks()
        adj_b = ADJ_B_PER_SAMPLE[cfg.targets[0]] if len(cfg.targets) == 1 else max(
            ADJ_B_PER_SAMPLE[t] for t in cfg.targets)
        adj_bytes = adj_b * local_samples + ADJ_B_PER_RAY * local_rays
        fwd_bytes = FWD_B_PER_SAMPLE * local_samples + FWD_B_PER_RAY * local_rays
        adj_s = float(np.mean(adj_ms)) / 1e3
        fwd_s = float(np.mean(fwd_ms)) / 1e3
        fused = getattr(step, "fused", False)
        if fused:   # one kernel marches forward, forms the L1 seed and walks back
            adj_bytes += fwd_bytes
            adj_b += FWD_B_PER_SAMPLE
        adj_gbs = adj_bytes / adj_s / 1e9
        fwd_gbs = fwd_bytes / fwd_s / 1e9
        traffic = ncu_traffic(cfg.name, ("fused_tape" if getattr(step, "band_tape", False)
                                         else "fused") if fused else "adjoint")
        kname = ("dvr_adjoint_kernel<FUSED> (forward + L1 seed + adjoint per ray)" if fused
                 else "dvr_adjoint_kernel")
        ray_b = ADJ_B_PER_RAY + (FWD_B_PER_RAY if fused else 0)
        note = ("algorithmic bytes charge 8 corner gathers (+8 scatters) per sample with no "
                "cache reuse (SURVEY 8d)")
        if traffic:
            note += (f"; ncu measures {traffic / adj_bytes:.2f}x those bytes of DRAM traffic per "
                     "launch (L1/L2 reuse), so frac > 1 is reuse, not missing work; the "
                     "limiters are instruction issue and L1 wavefronts (record gathers, "
                     "cell-run vector reds): profiles/r01_ncu_c4_full_fused_skip.txt")
        if fused:
            kernels = {
                "pack_cells": {"ms": fwd_s * 1e3},
                "fused_forward_adjoint": {"ms": adj_s * 1e3, "achieved_gbs": adj_gbs,
                                          "frac": adj_gbs / peak, "traffic": traffic},
                "share_of_step": {"pack_cells": fwd_s * 1e3 / ms_per_step,
                                  "fused_forward_adjoint": adj_s * 1e3 / ms_per_step}}
        else:
            kernels = {
                "forward": {"ms": fwd_s * 1e3, "achieved_gbs": fwd_gbs, "frac": fwd_gbs / peak,
                            "bytes_model": f"{FWD_B_PER_SAMPLE} B/sample + {FWD_B_PER_RAY} B/ray",
                            "traffic": ncu_traffic(cfg.name, "forward")},
                "adjoint": {"ms": adj_s * 1e3, "achieved_gbs": adj_gbs, "frac": adj_gbs / peak},
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
            "roofline": {"bound": "hbm", "kernel": kname,
                         "achieved": adj_gbs, "peak": peak, "unit": "GB/s",
                         "frac": adj_gbs / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": adj_bytes,
                         "bytes_model": f"{adj_b} B/sample + {ray_b} B/ray",
                         "launch_ms": adj_s * 1e3, "peak_source": peak_src, "note": note},
            "kernels": kernels,
            "e2e": {"value": total_samples / (e2e_ms_step / 1e3), "unit": "samples/s",
                    "ms_per_step": e2e_ms_step, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if probe_ms:
            probe_rate = local_samples / (probe_ms / 1e3)
            gr = {"probe": "ddvr_gather_probe: the same rays, fixed-point stepping and held "
                           "256-bit record gathers, one FADD per sample (6 CTAs/SM)",
                  "samples_per_s": probe_rate * world, "probe_ms": probe_ms}
            if fused:
                # the fused kernel gathers along every ray twice (forward + walk), or
                # once with the band tape (the walk reads 1 bit per sample instead)
                passes = 1 if getattr(step, "band_tape", False) else 2
                gr["record_gather_passes"] = passes
                gr["fused_frac"] = passes * local_samples / adj_s / probe_rate
            else:
                gr["forward_frac"] = local_samples / fwd_s / probe_rate
                gr["adjoint_frac"] = local_samples / adj_s / probe_rate
            line["gather_roofline"] = gr
        if runner is not step:
            line["config"]["iterations"] = (
                "one optimisation run: value times iterations W+1..W+K, e2e the next W+K; "
                "the estimate changes every iteration (Adam + [0,1] projection), and as its "
                "empty space grows the march and the walk skip more of it")
        line["config"]["step"] = (("fused forward+L1+adjoint" if getattr(step, "fused", False)
                                   else "forward, L1, adjoint") +
                                  (", band tape (1 bit/sample, DDVR_FLAG_BAND_TAPE)"
                                   if getattr(step, "band_tape", False) else "") +
                                  (", empty-brick skip in the march"
                                   if getattr(step, "band_tape", False) and step.empty_skip
                                   else "") +
                                  (", CUDA-graph replay" if graphed else ""))
        if world == 1 and not args.no_cpu_baseline:
            sps, rps, cores, desc = cpu_sample(cfg, args.cpu_seconds)
            line["cpu_baseline"] = {"value": sps, "unit": "samples/s", "cores": cores,
                                    "kind": "port", "sample": desc}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    from paper_2107_12672_b200.scenes import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_own(args, cfg)


if __name__ == "__main__":
    main()
