"""Tensor-level raymarcher over CUDA tensors: ops and the autograd Function.

This is the B200 product path: torch owns device memory and streams, every
compute step is a libddvr kernel reached through the C ABI (``_native``).

    images = render_views(density, texels, lonlat, dt, rig)     # differentiable

``DiffDVR.backward`` launches ONE adjoint kernel whose target mask is
``ctx.needs_input_grad`` and saves only the output images and the per-pixel
optical depth: O(pixels) memory, the paper's inversion trick
(renderer.py:540-543, 576-580).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _native as N
from .errors import InvalidInputError, InvalidParameterError, UnsupportedConfigurationError

EPS_POLE_DEG = 1e-3    # field.py:24


# transfer-function representation by parameter-row width:
#   (R, 4) texel table [r, g, b, tau]           (field.py:540-549)
#   (K, 5) piecewise-linear knots [pos, r, g, b, tau]   (no reference implementation)
#   (G, 6) Gaussians [mu, sigma, r, g, b, tau]          (tasks.py:751-766 optical model)
TF_KINDS = {4: N.TF_TEXTURE, 5: N.TF_PIECEWISE, 6: N.TF_GAUSSIAN}


@dataclass(frozen=True)
class Rig:
    """Static geometry shared by every view of a batch.

    The image size is common to all views (images are (V, H, W, 4));
    ``rows`` restricts every view to a row band [r0, r1) (renderer.py:491).
    """

    width: int
    height: int
    box_min: tuple = (-0.5, -0.5, -0.5)
    box_max: tuple = (0.5, 0.5, 0.5)
    rows: tuple | None = None

    @property
    def band(self) -> tuple:
        return self.rows if self.rows is not None else (0, self.height)

    @property
    def band_rows(self) -> int:
        r0, r1 = self.band
        return r1 - r0


def _stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def _require(t: torch.Tensor, name: str, dtype, *, ndim=None, align16=False):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InvalidInputError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise InvalidInputError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise InvalidInputError(f"{name} must be contiguous")
    if ndim is not None and t.dim() != ndim:
        raise InvalidInputError(f"{name} must have {ndim} dims, got shape {tuple(t.shape)}")
    if align16 and t.data_ptr() % 16:
        raise InvalidInputError(f"{name} must be 16-byte aligned")


def camera_array(lonlat: torch.Tensor, radius=2.0, center=(0.0, 0.0, 0.0),
                 fov_y_deg=30.0) -> torch.Tensor:
    """(V, 8) float64 device array of ddvr_camera records from (V, 2) lon/lat degrees."""
    ll = lonlat.detach().to(torch.float64)
    V = ll.shape[0]
    dev = ll.device
    rad = torch.as_tensor(radius, dtype=torch.float64, device=dev).reshape(-1, 1).expand(V, 1)
    ctr = torch.as_tensor(center, dtype=torch.float64, device=dev).reshape(-1, 3).expand(V, 3)
    fov = torch.as_tensor(fov_y_deg, dtype=torch.float64, device=dev).reshape(-1, 1).expand(V, 1)
    pad = torch.zeros(V, 1, dtype=torch.float64, device=dev)
    return torch.cat([ll, rad, ctr, fov, pad], dim=1).contiguous()


def validate_cameras(lonlat, radius, fov_y_deg):
    """Host-side checks of field.py:147-156 (one device->host copy)."""
    ll = torch.as_tensor(lonlat).detach().to("cpu", torch.float64)
    if ll.numel() and bool((ll[:, 1].abs() >= 90.0 - EPS_POLE_DEG).any()):
        raise InvalidParameterError("latitude violates the pole exclusion")
    if bool((torch.as_tensor(radius, dtype=torch.float64) <= 0).any()):
        raise InvalidParameterError("camera radius must be positive")
    f = torch.as_tensor(fov_y_deg, dtype=torch.float64)
    if bool(((f <= 0) | (f >= 180)).any()):
        raise InvalidParameterError("vertical field of view must be in (0, 180)")


def _descs(density, texels, rig: Rig, dt: float, early_stop: bool, cells=None):
    _require(density, "density", torch.float32, ndim=3)
    _require(texels, "texels", torch.float32, ndim=2)
    kind = TF_KINDS.get(int(texels.shape[1]))
    if kind is None or texels.shape[0] < 1:
        raise InvalidParameterError("transfer function must have shape (R, 4) texels, "
                                    "(K, 5) piecewise knots or (G, 6) Gaussians")
    if kind == N.TF_TEXTURE and texels.data_ptr() % 16:
        raise InvalidInputError("texels must be 16-byte aligned")
    if cells is not None:
        _require(cells, "cells", torch.float32)
        if cells.data_ptr() % 32 or cells.numel() != cells_numel(density.shape):
            raise InvalidInputError("cell records do not match the density (use pack_cells)")
    vol = N.DdvrVolume(density.data_ptr(), (ctypes.c_int32 * 3)(*density.shape),
                       (ctypes.c_double * 3)(*rig.box_min), (ctypes.c_double * 3)(*rig.box_max),
                       cells.data_ptr() if cells is not None else None)
    tf = N.DdvrTf(kind, texels.shape[0], texels.data_ptr())
    r0, r1 = rig.band
    prm = N.DdvrParams(float(dt), rig.width, rig.height, r0, r1, 1 if early_stop else 0, 0,
                       None, 0)
    return vol, tf, prm


def cells_numel(dims) -> int:
    """Floats in the padded cell-record copy of a (X,Y,Z) volume: 8 per cell, (X+1)(Y+1)(Z+1) cells."""
    n = 8
    for d in dims:
        n *= int(d) + 1
    return n


def pack_cells(density: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Cell-record copy of ``density``: the 8 corners of every cell in 32 bytes.

    One 256-bit load per sample instead of 8 scalar gathers (ddvr_pack_cells).
    Costs 8x the volume's memory; rebuild after every density update.
    """
    _require(density, "density", torch.float32, ndim=3)
    n = cells_numel(density.shape)
    if out is None or out.numel() != n:
        out = torch.empty(n, dtype=torch.float32, device=density.device)
    vol = N.DdvrVolume(density.data_ptr(), (ctypes.c_int32 * 3)(*density.shape),
                       (ctypes.c_double * 3)(-0.5, -0.5, -0.5), (ctypes.c_double * 3)(0.5, 0.5, 0.5),
                       None)
    N.check(N.lib().ddvr_pack_cells(ctypes.byref(vol), out.data_ptr(), _stream_ptr()))
    return out


def _set_tape(prm, tape, tape_stride):
    """Stored memory mode (renderer.py:507-513): one transmittance per sample."""
    if tape is not None:
        _require(tape, "tape", torch.float32)
        prm.tape = tape.data_ptr()
        prm.tape_stride = int(tape_stride)


def forward(density, texels, cams, dt: float, rig: Rig, *, early_stop=False, with_depth=True,
            cells=None, tape=None, tape_stride=0):
    """Images (V, rows, W, 4) fp32 and ray optical depth S (V, rows, W), T = exp(-S) (or None)."""
    _require(cams, "cameras", torch.float64, ndim=2)
    vol, tf, prm = _descs(density, texels, rig, dt, early_stop, cells)
    _set_tape(prm, tape, tape_stride)
    V = cams.shape[0]
    img = torch.empty(V, rig.band_rows, rig.width, 4, dtype=torch.float32, device=density.device)
    depth = (torch.empty(V, rig.band_rows, rig.width, dtype=torch.float32, device=density.device)
             if with_depth else None)
    N.check(N.lib().ddvr_forward(ctypes.byref(vol), ctypes.byref(tf), cams.data_ptr(), V,
                                 ctypes.byref(prm), img.data_ptr(),
                                 depth.data_ptr() if depth is not None else None, _stream_ptr()))
    return img, depth


def forward_grad(density, texels, cams, dt: float, rig: Rig, wrt: str = "camera", *,
                 cells=None):
    """(image (V,rows,W,4), jacobian (V,rows,W,4,p)) by forward mode (renderer.py:410-464).

    wrt "camera": p = 2, d/d(lon, lat) per degree; "stepsize": p = 1.
    """
    _require(cams, "cameras", torch.float64, ndim=2)
    if wrt not in ("camera", "stepsize"):
        raise UnsupportedConfigurationError(
            f"forward mode supports camera and stepsize, not {wrt!r}")
    vol, tf, prm = _descs(density, texels, rig, dt, False, cells)
    V = cams.shape[0]
    p = 2 if wrt == "camera" else 1
    dev = density.device
    img = torch.empty(V, rig.band_rows, rig.width, 4, dtype=torch.float32, device=dev)
    jac = torch.empty(V, rig.band_rows, rig.width, 4, p, dtype=torch.float32, device=dev)
    N.check(N.lib().ddvr_forward_grad(ctypes.byref(vol), ctypes.byref(tf), cams.data_ptr(), V,
                                      ctypes.byref(prm), N.TARGET_BITS[wrt], img.data_ptr(),
                                      jac.data_ptr(), _stream_ptr()))
    return img, jac


def _color_descs(color, rig: Rig, dt: float, early_stop: bool, tape=None, tape_stride=0):
    _require(color, "colour volume", torch.float32, ndim=4, align16=True)
    if color.shape[3] != 4:
        raise InvalidParameterError("color volume must have shape (X, Y, Z, 4)")
    vol = N.DdvrVolume(color.data_ptr(), (ctypes.c_int32 * 3)(*color.shape[:3]),
                       (ctypes.c_double * 3)(*rig.box_min), (ctypes.c_double * 3)(*rig.box_max),
                       None)
    r0, r1 = rig.band
    prm = N.DdvrParams(float(dt), rig.width, rig.height, r0, r1, 1 if early_stop else 0, 0,
                       None, 0)
    _set_tape(prm, tape, tape_stride)
    return vol, prm


def forward_color(color, cams, dt: float, rig: Rig, *, early_stop=False, tape=None,
                  tape_stride=0):
    """Images and optical depth of a pre-shaded (X,Y,Z,4) colour volume (renderer.py:404-407)."""
    _require(cams, "cameras", torch.float64, ndim=2)
    vol, prm = _color_descs(color, rig, dt, early_stop, tape, tape_stride)
    V = cams.shape[0]
    img = torch.empty(V, rig.band_rows, rig.width, 4, dtype=torch.float32, device=color.device)
    depth = torch.empty(V, rig.band_rows, rig.width, dtype=torch.float32, device=color.device)
    N.check(N.lib().ddvr_forward_color(ctypes.byref(vol), cams.data_ptr(), V, ctypes.byref(prm),
                                       img.data_ptr(), depth.data_ptr(), _stream_ptr()))
    return img, depth


def adjoint_color(color, cams, dt: float, rig: Rig, image, depth, seed, d_color, *, tape=None,
                  tape_stride=0):
    """d_color += d sum(seed * image) / d colour values (renderer.py:703-709)."""
    _require(cams, "cameras", torch.float64, ndim=2)
    vol, prm = _color_descs(color, rig, dt, False, tape, tape_stride)
    V = cams.shape[0]
    shape = (V, rig.band_rows, rig.width, 4)
    _require(seed, "seed", torch.float32)
    if tuple(seed.shape) != shape:
        raise InvalidInputError(f"seed shape {tuple(seed.shape)} does not match image {shape}")
    _require(d_color, "d_color", torch.float32, align16=True)
    N.check(N.lib().ddvr_adjoint_color(
        ctypes.byref(vol), cams.data_ptr(), V, ctypes.byref(prm),
        image.data_ptr() if image is not None else None,
        depth.data_ptr() if depth is not None else None, seed.data_ptr(), d_color.data_ptr(),
        _stream_ptr()))


def workspace_for(density, mask: int, cells=None, texels=None, extra: int = 0):
    """Device workspace ddvr_adjoint needs for this layout, TF and mask (or None):
    cell-gradient records (volume target, cell layout) + TF-gradient slots
    (tf target; needs ``texels`` for the TF shape), + ``extra`` bytes after the
    256-aligned end (the deterministic mode's partials, ddvr_deterministic_bytes)."""
    if mask & N.TARGET_TF and texels is None:
        raise InvalidParameterError("the tf target's workspace depends on the TF: pass texels")
    if texels is None:
        texels = torch.zeros(1, 4, dtype=torch.float32, device=density.device)
    vol, tf, _ = _descs(density, texels, Rig(1, 1), 1.0, False, cells)
    need = int(N.lib().ddvr_adjoint_workspace_bytes(ctypes.byref(vol), ctypes.byref(tf), mask))
    if extra:
        need = ((need + 255) & ~255) + int(extra)
    if need == 0:
        return None
    return torch.empty((need + 3) // 4, dtype=torch.float32, device=density.device)


def extra_workspace_bytes(vol, prm, n_views: int, mask: int, deterministic=False,
                          band_tape=False) -> int:
    """Bytes after the 256-aligned adjoint workspace for the optional modes: the
    deterministic partials, then (256-aligned) the band tape (include/ddvr.h)."""
    lib = N.lib()
    det = int(lib.ddvr_deterministic_bytes(ctypes.byref(vol), n_views, ctypes.byref(prm), mask)) \
        if deterministic else 0
    band = int(lib.ddvr_band_tape_bytes(ctypes.byref(vol), n_views, ctypes.byref(prm))) \
        if band_tape and mask == N.TARGET_VOLUME else 0
    if not band:
        return det
    return ((det + 255) & ~255) + band


def forward_adjoint_l1(density, texels, cams, dt: float, rig: Rig, refs, count: float, mask: int,
                       *, cells, loss, d_volume=None, d_tf=None, d_camera=None, d_dt=None,
                       workspace=None, image_out=None, depth_out=None, ws_continue=False,
                       ws_defer=False, deterministic=False, band_tape=False,
                       empty_skip=True, stats=None, split_walk=False, ray_split="auto"):
    """One fused step over these views: forward march, L1 seed sign(image - ref)/count
    and adjoint walk per ray in one kernel (ddvr_forward_adjoint_l1).  loss (fp64,
    device) += sum |image - ref| / count; gradients accumulate (+=) as in adjoint().
    One step split over several calls (view chunks) shares ``workspace``: every
    call but the first passes ws_continue, every call but the last ws_defer.
    ``deterministic``: bitwise reproducible d_camera / d_dt (DDVR_FLAG_DETERMINISTIC);
    ``band_tape``: the march stores 1 bit per sample for the affine absorption walk,
    which then gathers no records (DDVR_FLAG_BAND_TAPE, volume target); with it the
    march skips 32-sample blocks in all-zero bricks unless ``empty_skip`` is False
    (DDVR_FLAG_NO_EMPTY_SKIP; bitwise the same outputs either way).  A
    caller-provided workspace needs those extra bytes too (extra_workspace_bytes).
    ``split_walk`` (band tape): march and walk as two kernels (DDVR_FLAG_SPLIT_WALK)
    instead of one (the same outputs).
    ``ray_split`` (TF target without camera / stepsize): threads per ray, 1, 2, 4 or 8
    consecutive lanes marching and walking one sample segment each; "auto" picks it
    from the ray count (DDVR_FLAG_RAY_SPLIT_*).
    ``stats`` (measurement, optional): (4,) int64 device tensor the kernel adds
    [samples, samples the march skipped, samples the walk skipped, rays] to."""
    _require(cams, "cameras", torch.float64, ndim=2)
    if cells is None:
        raise InvalidParameterError("the fused step needs cell records (pack_cells)")
    vol, tf, prm = _descs(density, texels, rig, dt, False, cells)
    V = cams.shape[0]
    shape = (V, rig.band_rows, rig.width, 4)
    _require(refs, "reference images", torch.float32)
    if tuple(refs.shape) != shape:
        raise InvalidInputError(f"refs shape {tuple(refs.shape)} does not match image {shape}")
    _require(loss, "loss", torch.float64)
    for buf, name, dt_ in ((d_volume, "d_volume", torch.float32), (d_tf, "d_tf", torch.float64),
                           (d_camera, "d_camera", torch.float64), (d_dt, "d_dt", torch.float64),
                           (image_out, "image_out", torch.float32),
                           (depth_out, "depth_out", torch.float32)):
        if buf is not None:
            _require(buf, name, dt_)
    extra = extra_workspace_bytes(vol, prm, V, mask, deterministic, band_tape)
    if workspace is None:
        if ws_continue or ws_defer:
            raise InvalidParameterError("a step split over calls needs a shared workspace")
        workspace = workspace_for(density, mask, cells, texels, extra)
    prm.flags = (N.FLAG_WS_CONTINUE if ws_continue else 0) | (N.FLAG_WS_DEFER if ws_defer else 0) \
        | (N.FLAG_DETERMINISTIC if deterministic else 0) | (N.FLAG_BAND_TAPE if band_tape else 0) \
        | (0 if empty_skip else N.FLAG_NO_EMPTY_SKIP) | (N.FLAG_SPLIT_WALK if split_walk else 0)
    if ray_split != "auto":
        if ray_split not in N.FLAG_RAY_SPLIT:
            raise InvalidParameterError(f"ray_split must be 'auto', 1, 2, 4 or 8, not {ray_split!r}")
        prm.flags |= N.FLAG_RAY_SPLIT[ray_split]
    if stats is not None:
        _require(stats, "stats", torch.int64)
        if stats.numel() < 4:
            raise InvalidInputError("stats needs 4 int64 counters")
        prm.stats = stats.data_ptr()
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    ws_bytes = workspace.numel() * 4 if workspace is not None else 0
    N.check(N.lib().ddvr_forward_adjoint_l1(
        ctypes.byref(vol), ctypes.byref(tf), cams.data_ptr(), V, ctypes.byref(prm),
        refs.data_ptr(), float(count), mask, ptr(image_out), ptr(depth_out), loss.data_ptr(),
        ptr(d_volume), ptr(d_tf), ptr(d_camera), ptr(d_dt), ptr(workspace), ws_bytes,
        _stream_ptr()))


def adjoint(density, texels, cams, dt: float, rig: Rig, image, depth, seed, mask: int, *,
            d_volume=None, d_tf=None, d_camera=None, d_dt=None, cells=None, workspace=None,
            tape=None, tape_stride=0, deterministic=False):
    """Accumulate gradients of sum(seed * image) into the given buffers (+=).
    ``deterministic``: d_camera / d_dt from per-CTA partials reduced in a fixed
    order (bitwise reproducible; DDVR_FLAG_DETERMINISTIC)."""
    _require(cams, "cameras", torch.float64, ndim=2)
    vol, tf, prm = _descs(density, texels, rig, dt, False, cells)
    _set_tape(prm, tape, tape_stride)
    V = cams.shape[0]
    shape = (V, rig.band_rows, rig.width, 4)
    _require(seed, "seed", torch.float32)
    if tuple(seed.shape) != shape:
        raise InvalidInputError(f"seed shape {tuple(seed.shape)} does not match image {shape}")
    if image is not None:
        _require(image, "image", torch.float32)
        if tuple(image.shape) != shape:
            raise InvalidInputError("provided image does not match the camera size")
    if depth is not None:
        _require(depth, "optical depth", torch.float32)
    for buf, name, dt_ in ((d_volume, "d_volume", torch.float32), (d_tf, "d_tf", torch.float64),
                           (d_camera, "d_camera", torch.float64), (d_dt, "d_dt", torch.float64)):
        if buf is not None:
            _require(buf, name, dt_)
    extra = int(N.lib().ddvr_deterministic_bytes(ctypes.byref(vol), V, ctypes.byref(prm), mask)) \
        if deterministic else 0
    if deterministic:
        prm.flags |= N.FLAG_DETERMINISTIC
    if workspace is None:
        workspace = workspace_for(density, mask, cells, texels, extra)
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    ws_bytes = workspace.numel() * 4 if workspace is not None else 0
    N.check(N.lib().ddvr_adjoint(ctypes.byref(vol), ctypes.byref(tf), cams.data_ptr(), V,
                                 ctypes.byref(prm), ptr(image), ptr(depth), seed.data_ptr(),
                                 mask, ptr(d_volume), ptr(d_tf), ptr(d_camera), ptr(d_dt),
                                 ptr(workspace), ws_bytes, _stream_ptr()))


def l1_loss_seed(images: torch.Tensor, refs: torch.Tensor, count: float | None = None):
    """(loss (1,) float64, seed like images) of mean |x - y| (objectives.py:38-54)."""
    _require(images, "images", torch.float32)
    _require(refs, "refs", torch.float32)
    if images.shape != refs.shape:
        raise InvalidInputError(f"image shape {tuple(images.shape)} != reference shape "
                                f"{tuple(refs.shape)}")
    count = float(images.numel()) if count is None else float(count)
    seed = torch.empty_like(images)
    loss = torch.zeros(1, dtype=torch.float64, device=images.device)
    N.check(N.lib().ddvr_l1_loss(images.data_ptr(), refs.data_ptr(), images.numel(), count,
                                 seed.data_ptr(), loss.data_ptr(), _stream_ptr()))
    return loss, seed


def gather_probe(density, cams, dt: float, rig: Rig, cells, hold: bool = True):
    """Per-ray checksums of the gather-roofline microbenchmark (ddvr_gather_probe):
    the march's record gathers with one FADD per sample instead of the shading."""
    _require(cams, "cameras", torch.float64, ndim=2)
    tex = torch.zeros(1, 4, dtype=torch.float32, device=density.device)
    vol, _, prm = _descs(density, tex, rig, dt, False, cells)
    out = torch.empty(cams.shape[0], rig.band_rows, rig.width, dtype=torch.float32,
                      device=density.device)
    N.check(N.lib().ddvr_gather_probe(ctypes.byref(vol), cams.data_ptr(), cams.shape[0],
                                      ctypes.byref(prm), int(hold), out.data_ptr(),
                                      _stream_ptr()))
    return out


def opacity_entropy(images: torch.Tensor, with_seed: bool = True):
    """Per image of an (..., H, W, 4) float32 batch: (H (V,) f64, seed like images or None,
    degenerate (V,) bool) of the normalised alpha entropy (objectives.py:95-126)."""
    _require(images, "images", torch.float32)
    if images.dim() < 3 or images.shape[-1] != 4:
        raise InvalidInputError("images must have shape (..., H, W, 4)")
    v = images.reshape(-1, images.shape[-3] * images.shape[-2], 4)
    out = torch.empty(v.shape[0], 4, dtype=torch.float64, device=images.device)
    seed = torch.empty_like(images) if with_seed else None
    N.check(N.lib().ddvr_opacity_entropy(v.data_ptr(), v.shape[1], v.shape[0], out.data_ptr(),
                                         seed.data_ptr() if seed is not None else None,
                                         _stream_ptr()))
    degenerate = (out[:, 1] <= 0) | (v.shape[1] < 2)
    return out[:, 0], seed, degenerate


def ray_setup(cams, dt: float, rig: Rig, dims=(2, 2, 2)):
    """(tn_tf (V,rows,W,2) f64, n_steps (V,rows,W) i32, flags i32) for parity tests."""
    _require(cams, "cameras", torch.float64, ndim=2)
    vol = N.DdvrVolume(None, (ctypes.c_int32 * 3)(*dims), (ctypes.c_double * 3)(*rig.box_min),
                       (ctypes.c_double * 3)(*rig.box_max), None)
    r0, r1 = rig.band
    prm = N.DdvrParams(float(dt), rig.width, rig.height, r0, r1, 0, 0, None, 0)
    V = cams.shape[0]
    dev = cams.device
    tn_tf = torch.empty(V, rig.band_rows, rig.width, 2, dtype=torch.float64, device=dev)
    n = torch.empty(V, rig.band_rows, rig.width, dtype=torch.int32, device=dev)
    fl = torch.empty_like(n)
    N.check(N.lib().ddvr_ray_setup(ctypes.byref(vol), cams.data_ptr(), V, ctypes.byref(prm),
                                   tn_tf.data_ptr(), n.data_ptr(), fl.data_ptr(), _stream_ptr()))
    return tn_tf, n, fl


class DiffDVR(torch.autograd.Function):
    """images = DiffDVR.apply(density, texels, lonlat, dt, rig, radius, center, fov, layout).

    density (X,Y,Z) fp32, texels (R,4) fp32, lonlat (V,2) degrees, dt a 0-d
    tensor (stepsize).  Gradients: density, texels, lonlat (per degree), dt.
    layout "cells" packs the density into 32-byte cell records (one 256-bit
    load per sample, 8x the volume's memory); "voxels" gathers 8 corners.
    """

    @staticmethod
    def forward(ctx, density, texels, lonlat, dt, rig: Rig, radius, center, fov, layout="cells"):
        cams = camera_array(lonlat.to(density.device), radius, center, fov)
        dtv = float(dt.detach()) if isinstance(dt, torch.Tensor) else float(dt)
        density = density.contiguous()
        cells = pack_cells(density) if layout == "cells" else None
        img, depth = forward(density, texels.contiguous(), cams, dtv, rig, cells=cells)
        ctx.save_for_backward(density, texels, img, depth)
        ctx.cams, ctx.dt, ctx.rig, ctx.cells = cams, dtv, rig, cells
        ctx.lonlat_meta = (lonlat.dtype, lonlat.device)
        ctx.dt_meta = (dt.dtype, dt.device) if isinstance(dt, torch.Tensor) else None
        ctx.mark_non_differentiable(depth)
        return img

    @staticmethod
    def backward(ctx, grad_img):
        density, texels, img, depth = ctx.saved_tensors
        need = ctx.needs_input_grad
        mask = ((N.TARGET_VOLUME if need[0] else 0) | (N.TARGET_TF if need[1] else 0)
                | (N.TARGET_CAMERA if need[2] else 0) | (N.TARGET_STEPSIZE if need[3] else 0))
        if mask == 0:
            return (None,) * 9
        dev = density.device
        d_vol = torch.zeros_like(density) if need[0] else None
        d_tf = torch.zeros(texels.shape, dtype=torch.float64, device=dev) if need[1] else None
        d_cam = (torch.zeros(ctx.cams.shape[0], 2, dtype=torch.float64, device=dev)
                 if need[2] else None)
        d_dt = torch.zeros(1, dtype=torch.float64, device=dev) if need[3] else None
        adjoint(density.contiguous(), texels.contiguous(), ctx.cams, ctx.dt, ctx.rig, img, depth,
                grad_img.contiguous().to(torch.float32), mask, d_volume=d_vol, d_tf=d_tf,
                d_camera=d_cam, d_dt=d_dt, cells=ctx.cells)
        g_tf = d_tf.to(texels.dtype) if d_tf is not None else None
        g_cam = (d_cam.to(dtype=ctx.lonlat_meta[0], device=ctx.lonlat_meta[1])
                 if d_cam is not None else None)
        g_dt = None
        if d_dt is not None and ctx.dt_meta is not None:
            g_dt = d_dt.reshape(()).to(dtype=ctx.dt_meta[0], device=ctx.dt_meta[1])
        return d_vol, g_tf, g_cam, g_dt, None, None, None, None, None


def render_views(density, texels, lonlat, dt, rig: Rig, *, radius=2.0, center=(0.0, 0.0, 0.0),
                 fov_y_deg=30.0, layout="cells"):
    """Differentiable images (V, rows, W, 4) of ``lonlat`` views (autograd-aware)."""
    if not isinstance(dt, torch.Tensor):
        dt = torch.tensor(float(dt), dtype=torch.float64)
    if float(dt.detach()) <= 0.0:
        raise InvalidParameterError("stepsize must be positive")
    if layout not in ("cells", "voxels"):
        raise InvalidParameterError(f"unknown volume layout {layout!r}")
    # field.py:147-156: a latitude at the pole degenerates the camera frame (NaN images
    # and gradients), so it is rejected here like the reference's SphericalCamera does
    validate_cameras(lonlat, radius, fov_y_deg)
    return DiffDVR.apply(density, texels, lonlat, dt, rig, radius, center, fov_y_deg, layout)
