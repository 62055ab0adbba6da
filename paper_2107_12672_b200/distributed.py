"""View-sharded optimisation step over N GPUs (one process per GPU, NCCL).

The reference sums per-view gradients in view order on one host
(``_volume_loss_and_grad``, tasks.py:397-432; TF variant tasks.py:258-270).
Here views are dealt round-robin to ranks (rank r takes views r, r+N, ...),
every rank renders and differentiates its own views with the replicated
volume and TF, and the sums are combined by an all-reduce over two flat
buffers:

    buf  fp32  [ d_volume (X*Y*Z) ]                      (the large one)
    tail fp64  [ d_tf (R*4) | d_stepsize (1) | loss (1) ] (a few hundred bytes)

The tail stays fp64 as the kernels produce it: the reference sums per-view
gradients in fp64, and the stepsize gradient is cancellation-heavy.  The L1
seeds only need the global element count, known statically
(objectives.py:51-53), so the forward/adjoint need no communication at all.
Camera gradients are per view and stay local.

The packing and the collective are plain torch.distributed, so the same code
runs with ``gloo`` on CPU tensors in the tests and ``nccl`` on the GPUs.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native as N
from . import raymarch as R


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """Round-robin view indices of ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return list(range(rank, n_views, world))


@dataclass
class FlatGrads:
    """The all-reduced quantities of a step: ``buf`` fp32 d_volume, ``tail`` fp64
    [d_tf | d_stepsize | loss] (the kernels accumulate d_tf, d_dt and the loss
    in fp64 directly into the tail's views).  ``zeros`` places both, plus one fp64
    ``aux`` slot that is not reduced (the iteration's prior value), in one byte
    buffer ``raw``, so zeroing a step is a single fill (one graph node)."""

    n_vox: int
    n_tf: int
    buf: torch.Tensor
    tail: torch.Tensor
    raw: torch.Tensor | None = None
    aux: torch.Tensor | None = None

    @classmethod
    def zeros(cls, n_vox: int, n_tf: int, device) -> "FlatGrads":
        n_tail = n_tf + 2
        off = (8 * (n_tail + 1) + 255) // 256 * 256          # buf 256-byte aligned
        raw = torch.zeros(off + 4 * n_vox, dtype=torch.uint8, device=device)
        tail = raw[: 8 * n_tail].view(torch.float64)
        aux = raw[8 * n_tail: 8 * (n_tail + 1)].view(torch.float64)
        buf = raw[off: off + 4 * n_vox].view(torch.float32)
        return cls(n_vox, n_tf, buf, tail, raw, aux)

    @property
    def d_volume(self) -> torch.Tensor:
        return self.buf

    @property
    def d_tf(self) -> torch.Tensor:
        return self.tail[: self.n_tf]

    @property
    def d_stepsize(self) -> torch.Tensor:
        return self.tail[self.n_tf: self.n_tf + 1]

    @property
    def loss(self) -> torch.Tensor:
        return self.tail[self.n_tf + 1:]

    def zero_(self) -> None:
        if self.raw is not None:
            self.raw.zero_()
        else:
            self.buf.zero_()
            self.tail.zero_()

    def allreduce(self, group=None) -> None:
        """Sum both buffers over all ranks in place (the fp32 volume gradient and the
        small fp64 tail; no-op at world size 1)."""
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.buf, op=dist.ReduceOp.SUM, group=group)
            dist.all_reduce(self.tail, op=dist.ReduceOp.SUM, group=group)


class ShardedStep:
    """One forward + L1 + adjoint + all-reduce step over this rank's views.

    density (X,Y,Z) fp32, texels (R,4) fp32 on this rank's GPU (replicated);
    refs: (V_local, H, W, 4) fp32 reference images of the local views;
    lonlat: (V_local, 2) poses; ``total_elements`` = 4*H*W*V_global.

    With cell records (the default layout) the forward, the L1 seed and the
    adjoint run as one fused kernel per ray (ddvr_forward_adjoint_l1);
    ``fused=False`` keeps the three separate launches (ddvr_forward,
    ddvr_l1_loss, ddvr_adjoint).  ``fused="auto"`` (default) fuses unless the
    camera or stepsize target comes with the TF target: those walks carry fp64
    sums and texel runs (~128 registers, 2 CTAs/SM), which would hold the fused
    forward phase there while the separate forward runs 5 CTAs/SM.  Camera /
    stepsize alone fuse (64-register walks: C3 82.3 vs 78.6 G samples/s
    separate).  ``keep_images``: also write the rendered
    images / optical depth of the fused step into ``img`` / ``depth``.
    ``deterministic``: camera / stepsize gradients reduced from per-CTA partials in a
    fixed order (DDVR_FLAG_DETERMINISTIC), bitwise reproducible step to step.
    ``stats`` (fused step, measurement only): (4,) int64 device counters the kernel adds
    [samples, march-skipped samples, walk-skipped samples, rays] to on every run.
    ``band_tape`` (fused volume-only steps): the march stores one bit per sample
    for the affine absorption walk, which then re-gathers no cell records
    (DDVR_FLAG_BAND_TAPE; 4.7 GB at C4).  "auto" uses it when it fits
    min(8 GiB, a quarter of the free device memory).  ``empty_skip`` (band tape):
    the march skips 32-sample blocks in all-zero 8^3-cell bricks (bitwise the same
    step; False marches every block, DDVR_FLAG_NO_EMPTY_SKIP).  ``split_walk`` (band
    tape): march and walk as two kernels instead of one (DDVR_FLAG_SPLIT_WALK).
    ``ray_split`` (fused TF-target steps): threads per ray (1, 2, 4, 8 or "auto",
    DDVR_FLAG_RAY_SPLIT_*).
    """

    def __init__(self, density, texels, lonlat, refs, dt, rig: R.Rig, *, targets=("volume",),
                 total_elements=None, radius=2.0, center=(0.0, 0.0, 0.0), fov_y_deg=30.0,
                 group=None, layout="cells", fused="auto", keep_images=False, chunks=4,
                 deterministic=False, band_tape="auto", empty_skip=True, stats=None,
                 split_walk=False, ray_split="auto"):
        self.density, self.texels, self.refs, self.dt, self.rig = density, texels, refs, dt, rig
        if ray_split != "auto" and ray_split not in N.FLAG_RAY_SPLIT:
            from .errors import InvalidParameterError
            raise InvalidParameterError(f"ray_split must be 'auto', 1, 2, 4 or 8, not {ray_split!r}")
        R.validate_cameras(lonlat, radius, fov_y_deg)   # field.py:147-156
        self.cams = R.camera_array(lonlat, radius, center, fov_y_deg)
        self.mask = 0
        for t in targets:
            self.mask |= N.TARGET_BITS[t]
        self.count = float(total_elements if total_elements is not None else refs.numel())
        self.group = group
        dev = density.device
        V = self.cams.shape[0]
        self.flat = FlatGrads.zeros(density.numel(), texels.numel(), dev)
        self.img = torch.empty(V, rig.band_rows, rig.width, 4, dtype=torch.float32, device=dev)
        self.seed = torch.empty_like(self.img)
        self.depth = torch.empty(V, rig.band_rows, rig.width, dtype=torch.float32, device=dev)
        # the fp64 outputs are views of the all-reduced tail (no cast, no copy)
        self.d_tf64 = self.flat.d_tf.view(texels.shape)
        self.d_dt64 = self.flat.d_stepsize
        # camera gradients are per view (d/d(lon, lat) per degree, field.py:11), so
        # they stay with the rank that owns the view: (V_local, 2), not all-reduced
        self.d_camera = torch.zeros(V, 2, dtype=torch.float64, device=dev)
        self.loss64 = self.flat.loss
        # cell records (rebuilt from the density every step) + adjoint workspace
        self.cells = (torch.empty(R.cells_numel(density.shape), dtype=torch.float32, device=dev)
                      if layout == "cells" else None)
        self.deterministic = bool(deterministic)
        self.empty_skip = bool(empty_skip)
        # measurement counters of the fused step (forward_adjoint_l1 ``stats``)
        self.stats = stats
        self.split_walk = bool(split_walk)
        self.ray_split = ray_split
        if fused == "auto":
            pos = self.mask & (N.TARGET_CAMERA | N.TARGET_STEPSIZE)
            fused = not (pos and self.mask & N.TARGET_TF)
        self.fused = bool(fused) and self.cells is not None
        vol, _, prm = R._descs(density, texels, rig, dt, False, self.cells)
        self.band_tape = bool(band_tape) and self.fused and self.mask == N.TARGET_VOLUME
        if self.band_tape and band_tape == "auto":   # <= min(8 GiB, a quarter of free HBM)
            need = int(N.lib().ddvr_band_tape_bytes(ctypes.byref(vol), V, ctypes.byref(prm)))
            free = torch.cuda.mem_get_info(dev)[0] if dev.type == "cuda" else 0
            self.band_tape = need <= min(8 << 30, free // 4)
        extra = R.extra_workspace_bytes(vol, prm, V, self.mask, self.deterministic,
                                        self.band_tape)
        self.workspace = R.workspace_for(density, self.mask, self.cells, texels, extra)
        self._copy_stream = None
        self.keep_images = keep_images
        # view chunks of the fused step when the refs come from the host: chunk k
        # waits only for its own refs, so the copy of the rest overlaps compute.
        # The first chunk is small (1/16 of the views) so the first kernel starts
        # after a short copy; the rest split evenly.
        n = max(1, min(chunks, V))
        if n > 1 and V >= 2 * n:
            first = max(1, V // 16)
            edges = [0] + [first + round(k * (V - first) / (n - 1)) for k in range(n)]
        else:
            edges = [round(k * V / n) for k in range(n + 1)]
        self._chunks = [slice(a, b) for a, b in zip(edges[:-1], edges[1:]) if b > a]

    def _stage_refs(self, refs_host, chunks):
        """Start the host->device copy of this step's reference images on a side
        stream, one piece per view chunk; return the events the loss waits on.
        The refs are first needed by the L1 seed, after the forward march of
        the chunk, so the copy overlaps the pack and the compute."""
        if refs_host is None:
            return None
        if tuple(refs_host.shape) != tuple(self.refs.shape):
            raise ValueError(f"refs_host shape {tuple(refs_host.shape)} != {tuple(self.refs.shape)}")
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(self.refs.device)
        main = torch.cuda.current_stream(self.refs.device)
        self._copy_stream.wait_stream(main)          # the previous step's loss read self.refs
        events = []
        with torch.cuda.stream(self._copy_stream):
            for sl in chunks:
                self.refs[sl].copy_(refs_host[sl], non_blocking=True)
                done = torch.cuda.Event()
                done.record(self._copy_stream)
                events.append(done)
        return events

    def run(self, hook=None, refs_host=None) -> FlatGrads:
        """One step; ``hook(name)`` (optional) is called at "post_forward",
        "pre_adjoint" and "post_adjoint" in stream order (for CUDA events).
        ``refs_host``: pinned host copy of this step's reference images, copied
        to the device on a side stream, overlapped with the forward."""
        import ctypes
        hook = hook or (lambda name: None)
        chunks = self._chunks if (self.fused and refs_host is not None) else [slice(None)]
        refs_ready = self._stage_refs(refs_host, chunks)
        f = self.flat
        f.zero_()
        if self.mask & N.TARGET_CAMERA:
            self.d_camera.zero_()
        V = self.cams.shape[0]
        if V and self.fused:
            R.pack_cells(self.density, self.cells)
            hook("post_forward")
            hook("pre_adjoint")
            main = torch.cuda.current_stream(self.refs.device)
            want = lambda bit, t: t if self.mask & bit else None  # noqa: E731
            for k, sl in enumerate(chunks):
                if refs_ready is not None:
                    main.wait_event(refs_ready[k])
                # one workspace for the whole step: zeroed by the first chunk,
                # folded into the gradients by the last
                last = k == len(chunks) - 1
                R.forward_adjoint_l1(
                    self.density, self.texels, self.cams[sl], self.dt, self.rig, self.refs[sl],
                    self.count, self.mask, cells=self.cells, loss=self.loss64,
                    d_volume=want(N.TARGET_VOLUME, f.d_volume), d_tf=want(N.TARGET_TF, self.d_tf64),
                    d_camera=want(N.TARGET_CAMERA, self.d_camera[sl]),
                    d_dt=want(N.TARGET_STEPSIZE, self.d_dt64), workspace=self.workspace,
                    image_out=self.img[sl] if self.keep_images else None,
                    depth_out=self.depth[sl] if self.keep_images else None,
                    ws_continue=k > 0 and self.workspace is not None,
                    ws_defer=not last and self.workspace is not None,
                    deterministic=self.deterministic, band_tape=self.band_tape,
                    empty_skip=self.empty_skip, stats=self.stats, split_walk=self.split_walk,
                    ray_split=self.ray_split)
            hook("post_adjoint")
        elif V:
            if self.cells is not None:
                R.pack_cells(self.density, self.cells)
            vol, tf, prm = R._descs(self.density, self.texels, self.rig, self.dt, False,
                                    self.cells)
            if self.deterministic:
                prm.flags |= N.FLAG_DETERMINISTIC
            lib = N.lib()
            st = R._stream_ptr()
            N.check(lib.ddvr_forward(ctypes.byref(vol), ctypes.byref(tf), self.cams.data_ptr(), V,
                                     ctypes.byref(prm), self.img.data_ptr(), self.depth.data_ptr(),
                                     st))
            hook("post_forward")
            if refs_ready is not None:
                torch.cuda.current_stream(self.refs.device).wait_event(refs_ready[0])
            N.check(lib.ddvr_l1_loss(self.img.data_ptr(), self.refs.data_ptr(), self.img.numel(),
                                     self.count, self.seed.data_ptr(), self.loss64.data_ptr(), st))
            want = lambda bit, t: t.data_ptr() if self.mask & bit else None  # noqa: E731
            hook("pre_adjoint")
            N.check(lib.ddvr_adjoint(ctypes.byref(vol), ctypes.byref(tf), self.cams.data_ptr(), V,
                                     ctypes.byref(prm), self.img.data_ptr(),
                                     self.depth.data_ptr(), self.seed.data_ptr(), self.mask,
                                     want(N.TARGET_VOLUME, f.d_volume),
                                     want(N.TARGET_TF, self.d_tf64),
                                     want(N.TARGET_CAMERA, self.d_camera),
                                     want(N.TARGET_STEPSIZE, self.d_dt64),
                                     self.workspace.data_ptr()
                                     if self.workspace is not None else None,
                                     self.workspace.numel() * 4 if self.workspace is not None
                                     else 0, st))
            hook("post_adjoint")
        f.allreduce(self.group)
        return f


class TomographyIteration:
    """One full absorption-tomography iteration on device (tasks.py:397-481).

    ShardedStep (forward + L1 seed + adjoint + all-reduce) followed by the
    volume smoothness prior (objectives.py:72-92, weight ``lam``), one Adam
    update and the [0,1] projection (optim.py:45-89).  Every rank applies the
    same update to its replica after the all-reduce, so replicas stay equal.

    ``check_finite`` (default on, optim.py:28-30): a non-finite gradient skips the
    update on the device (sticky flag) and raises NumericalAbortError on the host
    without a per-iteration synchronisation -- the flag is copied to pinned host
    memory after each iteration and checked at the start of the next ``run`` once
    that copy has landed, or by ``check()``, which waits for it.
    """

    def __init__(self, step: ShardedStep, *, lr: float = 0.02, lam: float = 0.5,
                 check_finite: bool = True, graph: bool = False):
        from .optim import AdamState
        self.step = step
        self.lam = lam
        self.check_finite = check_finite
        self._flag_host = None
        self._flag_evt = None
        # graph: after two eager warm-up iterations one iteration is captured in a
        # CUDA graph and replayed (launch-bound small problems); single process
        # only, Adam's step counter lives on the device
        self.graph = graph
        self.adam = AdamState(lr=lr, device_step=graph)
        self._g = None
        self._out = None
        self._eager = 0
        self.graph_launches = 0      # libddvr kernels in the captured graph
        if graph and dist.is_available() and dist.is_initialized() and \
                dist.get_world_size(step.group) > 1:
            raise ValueError("graph capture of the step is single-process only")

    def run(self, hook=None, refs_host=None):
        """One iteration -> (loss (1,) f64, prior (1,) f64) on device.  With ``graph``
        the hook and refs_host are not available (the graph replays fixed work)."""
        self._raise_if_flagged(block=False)
        out = self._run(hook, refs_host)
        self._post_flag()
        return out

    def check(self) -> None:
        """Wait for the last iteration's non-finite flag; raise NumericalAbortError
        if any iteration so far saw a non-finite gradient."""
        self._raise_if_flagged(block=True)

    def reset(self, density=None) -> None:
        """Restore a fixed state (measurement): optionally copy ``density`` into the
        optimised volume, and zero the Adam moments and step counter."""
        if density is not None:
            self.step.density.copy_(density)
        self.adam.reset()

    def _post_flag(self):
        if not self.check_finite or self.adam.flag is None:
            return
        dev = self.step.density.device
        if self._flag_host is None:
            self._flag_host = torch.zeros(1, dtype=torch.int32,
                                          pin_memory=dev.type == "cuda")
            self._flag_evt = torch.cuda.Event() if dev.type == "cuda" else None
        self._flag_host.copy_(self.adam.flag, non_blocking=True)
        if self._flag_evt is not None:
            self._flag_evt.record()

    def _raise_if_flagged(self, block):
        from .errors import NumericalAbortError
        if self._flag_host is None:
            return
        if self._flag_evt is not None:
            if block:
                self._flag_evt.synchronize()
            elif not self._flag_evt.query():
                return
        if int(self._flag_host[0]):
            raise NumericalAbortError("non-finite gradients passed to the optimizer")

    def _run(self, hook, refs_host):
        if not self.graph:
            return self._iterate(hook, refs_host)
        if hook is not None or refs_host is not None:
            raise ValueError("a graphed iteration takes no hook or refs_host")
        if self._g is None and self._eager < 2:
            self._eager += 1
            return self._iterate(None, None)
        if self._g is None:
            side = torch.cuda.Stream(self.step.density.device)
            side.wait_stream(torch.cuda.current_stream(self.step.density.device))
            self._g = torch.cuda.CUDAGraph()
            n0 = N.launch_count()
            with torch.cuda.graph(self._g, stream=side):
                self._out = self._iterate(None, None)
            self.graph_launches = N.launch_count() - n0
            torch.cuda.current_stream(self.step.density.device).wait_stream(side)
        self._g.replay()
        return self._out

    def _iterate(self, hook, refs_host):
        from .optim import prior_volume
        f = self.step.run(hook=hook, refs_host=refs_host)
        density = self.step.density
        grad = f.d_volume.view(density.shape)
        # grad += lam * d prior; the value into the step's zeroed aux slot
        prior = prior_volume(density, self.lam, grad, out=f.aux)
        self.adam.update(density, grad, project="volume",
                         check_finite="defer" if self.check_finite else False)
        return f.loss, prior
