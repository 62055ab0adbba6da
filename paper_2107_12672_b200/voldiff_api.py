"""Drop-in replacement for the reference's render / loss API (voldiff).

Same names, signatures, argument meaning and exceptions as
``voldiff.renderer.render`` (renderer.py:393-401), ``render_adjoint``
(renderer.py:688-700) and ``voldiff.objectives.l1_loss`` (objectives.py:38-54),
plus the domain dataclasses they take (field.py:35-156, renderer.py:56-118).
Inputs may be the reference's own objects (duck-typed ``.values``,
``.texels``, camera fields) or the classes below.  Results come back as
float64 NumPy, like the reference.

Every numerical result is computed by libddvr on the current CUDA device; the
``threads`` keyword is accepted and ignored (the GPU replaces the tile pool,
renderer.py:243-247).  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _native as N
from . import raymarch as R
from .errors import (
    InvalidInputError,
    InvalidParameterError,
    UnsupportedConfigurationError,
)

EPS_POLE_DEG = 1e-3      # field.py:24
EPS_ALPHA = 1e-6         # field.py:25
TILE_ROWS = 64           # renderer.py:44 (only used for the stored-mode memory counter)
_TARGETS = ("none", "camera", "stepsize", "tf", "volume")     # renderer.py:47
_MEMORY_MODES = ("inversion", "stored")                        # renderer.py:48


# ---------------------------------------------------------------------------
# domain types (field.py:35-156; renderer.py:56-118)
# ---------------------------------------------------------------------------


@dataclass
class DensityVolume:
    """3D scalar grid (X,Y,Z) on a world box (field.py:35-77)."""

    values: np.ndarray
    box_min: np.ndarray = dc_field(default_factory=lambda: np.array([-0.5, -0.5, -0.5]))
    box_max: np.ndarray = dc_field(default_factory=lambda: np.array([0.5, 0.5, 0.5]))

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=np.float64)
        self.box_min = np.asarray(self.box_min, dtype=np.float64).reshape(3)
        self.box_max = np.asarray(self.box_max, dtype=np.float64).reshape(3)
        if self.values.ndim != 3 or min(self.values.shape) < 1:
            raise InvalidParameterError("volume values must be a non-empty 3D array")
        if not np.all(np.isfinite(self.values)):
            raise InvalidParameterError("volume contains non-finite densities")
        if not np.all(self.box_max > self.box_min):
            raise InvalidParameterError("world box must have positive extent on each axis")

    @property
    def dims(self):
        return self.values.shape

    @property
    def extent(self):
        return self.box_max - self.box_min

    @property
    def voxel_size(self):
        return self.extent / np.asarray(self.values.shape, dtype=np.float64)


@dataclass
class ColorVolume:
    """Per-voxel rgb emission plus absorption, shape (X, Y, Z, 4) (field.py:80-105)."""

    values: np.ndarray
    box_min: np.ndarray = dc_field(default_factory=lambda: np.array([-0.5, -0.5, -0.5]))
    box_max: np.ndarray = dc_field(default_factory=lambda: np.array([0.5, 0.5, 0.5]))

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=np.float64)
        self.box_min = np.asarray(self.box_min, dtype=np.float64).reshape(3)
        self.box_max = np.asarray(self.box_max, dtype=np.float64).reshape(3)
        if self.values.ndim != 4 or self.values.shape[3] != 4:
            raise InvalidParameterError("color volume must have shape (X, Y, Z, 4)")
        if not np.all(np.isfinite(self.values)):
            raise InvalidParameterError("color volume contains non-finite entries")
        if not np.all(self.box_max > self.box_min):
            raise InvalidParameterError("world box must have positive extent on each axis")

    @property
    def dims(self):
        return self.values.shape[:3]

    @property
    def voxel_size(self):
        return (self.box_max - self.box_min) / np.asarray(self.values.shape[:3], dtype=np.float64)


@dataclass
class TransferFunction:
    """R texels of (r, g, b, tau) with linear interpolation (field.py:108-127)."""

    texels: np.ndarray

    def __post_init__(self):
        self.texels = np.asarray(self.texels, dtype=np.float64)
        if self.texels.ndim != 2 or self.texels.shape[1] != 4 or self.texels.shape[0] < 1:
            raise InvalidParameterError("transfer function must have shape (R, 4), R >= 1")
        if not np.all(np.isfinite(self.texels)):
            raise InvalidParameterError("transfer function contains non-finite entries")

    @property
    def resolution(self):
        return self.texels.shape[0]


@dataclass
class SphericalCamera:
    """Camera on a sphere around ``center`` looking at it, up = +Y (field.py:130-156)."""

    lon_deg: float
    lat_deg: float
    radius: float
    center: np.ndarray = dc_field(default_factory=lambda: np.zeros(3))
    fov_y_deg: float = 30.0
    width: int = 64
    height: int = 64

    def __post_init__(self):
        self.lon_deg = float(self.lon_deg) % 360.0
        self.lat_deg = float(self.lat_deg)
        self.radius = float(self.radius)
        self.center = np.asarray(self.center, dtype=np.float64).reshape(3)
        if abs(self.lat_deg) >= 90.0 - EPS_POLE_DEG:
            raise InvalidParameterError(f"latitude {self.lat_deg} deg violates the pole exclusion")
        if self.radius <= 0.0:
            raise InvalidParameterError("camera radius must be positive")
        if not 0.0 < self.fov_y_deg < 180.0:
            raise InvalidParameterError("vertical field of view must be in (0, 180)")
        if self.width < 1 or self.height < 1:
            raise InvalidParameterError("image size must be at least 1x1")


@dataclass
class ImageRGBA:
    """Premultiplied rgb + accumulated opacity, shape (H, W, 4) (renderer.py:56-81)."""

    data: np.ndarray

    def __post_init__(self):
        self.data = np.asarray(self.data, dtype=np.float64)
        if self.data.ndim != 3 or self.data.shape[2] != 4:
            raise InvalidInputError("image data must have shape (H, W, 4)")

    @classmethod
    def zeros(cls, width, height):
        return cls(np.zeros((height, width, 4)))

    @property
    def width(self):
        return self.data.shape[1]

    @property
    def height(self):
        return self.data.shape[0]

    @property
    def alpha(self):
        return self.data[..., 3]


@dataclass
class RenderConfig:
    """Stepsize, differentiation target and adjoint memory mode (renderer.py:84-106)."""

    dt: float
    target: str = "none"
    memory_mode: str = "inversion"
    precision: str = "double"

    def __post_init__(self):
        _validate_config(self)

    @property
    def dtype(self):
        return np.float64 if self.precision == "double" else np.float32


@dataclass
class GradientSet:
    """Gradients for the selected target; the others stay None (renderer.py:109-118)."""

    d_stepsize: float | None = None
    d_camera: np.ndarray | None = None
    d_tf: np.ndarray | None = None
    d_volume: np.ndarray | None = None
    d_color: np.ndarray | None = None
    state_floats: int = 0


def _validate_config(cfg):
    dt = float(cfg.dt)
    if not dt > 0.0:
        raise InvalidParameterError("stepsize must be positive")
    if cfg.target not in _TARGETS:
        raise InvalidParameterError(f"unknown differentiation target {cfg.target!r}")
    if getattr(cfg, "memory_mode", "inversion") not in _MEMORY_MODES:
        raise InvalidParameterError(f"unknown memory mode {cfg.memory_mode!r}")
    if getattr(cfg, "precision", "double") not in ("double", "single"):
        raise InvalidParameterError("precision must be 'double' or 'single'")
    cfg.dt = dt


# ---------------------------------------------------------------------------
# compositing algebra on single states (renderer.py:126-174); host helpers
# ---------------------------------------------------------------------------


def blend(state, sample):
    """One front-to-back compositing step (renderer.py:126-138)."""
    state = np.asarray(state, np.float64)
    sample = np.asarray(sample, np.float64)
    vis = 1.0 - state[..., 3:4]
    out = np.empty(np.broadcast_shapes(state.shape, sample.shape))
    out[..., :3] = state[..., :3] + vis * sample[..., :3]
    out[..., 3:4] = state[..., 3:4] + vis * sample[..., 3:4]
    return out


def blend_invert(nxt, sample):
    """Exact inverse of :func:`blend` given the blended sample (renderer.py:141-152)."""
    nxt = np.asarray(nxt, np.float64)
    sample = np.asarray(sample, np.float64)
    a_s = sample[..., 3]
    if np.any(a_s > 1.0 - EPS_ALPHA + 1e-15):
        raise InvalidInputError("sample opacity exceeds the invertibility clamp")
    a_prev = (a_s - nxt[..., 3]) / (a_s - 1.0)
    out = np.empty(np.broadcast_shapes(nxt.shape, sample.shape))
    out[..., :3] = nxt[..., :3] - (1.0 - a_prev)[..., None] * sample[..., :3]
    out[..., 3] = a_prev
    return out


def blend_adjoint(state, sample, next_hat):
    """(state_hat, sample_hat) = transpose of the blend Jacobian (renderer.py:155-174)."""
    state = np.asarray(state, np.float64)
    sample = np.asarray(sample, np.float64)
    next_hat = np.asarray(next_hat, np.float64)
    vis = 1.0 - state[..., 3]
    shape = np.broadcast_shapes(state.shape, sample.shape, next_hat.shape)
    state_hat = np.empty(shape)
    sample_hat = np.empty(shape)
    state_hat[..., :3] = next_hat[..., :3]
    state_hat[..., 3] = (1.0 - sample[..., 3]) * next_hat[..., 3] - np.sum(
        sample[..., :3] * next_hat[..., :3], axis=-1)
    sample_hat[..., :3] = vis[..., None] * next_hat[..., :3]
    sample_hat[..., 3] = vis * next_hat[..., 3]
    return state_hat, sample_hat


# ---------------------------------------------------------------------------
# upload helpers
# ---------------------------------------------------------------------------


def _device():
    if not torch.cuda.is_available():
        raise N.NativeLibraryError("no CUDA device: the B200 raymarcher has no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


# Device copies of recently used density arrays: the reference's pipelines call render /
# render_adjoint once per view with the same DensityVolume (tasks.py:397-432), so the
# volume is uploaded and its cell records packed once per optimisation step, not once
# per view and call.  An entry is found by the identity of the ``values`` array (held
# weakly: a new DensityVolume -- what adam_step / project_params produce, tasks.py:
# 473-480 -- is a new entry) and validated against its data pointer, shape and a
# checksum of every 61st element (in-place writes to a cached array between calls are
# outside the reference's contract: inputs are read-only).
_VOLUME_CACHE: list = []
_VOLUME_CACHE_SIZE = 2


def _fingerprint(values: np.ndarray):
    flat = values.reshape(-1)
    return (values.__array_interface__["data"][0], values.shape, values.dtype.str,
            float(np.add.reduce(flat[::61], dtype=np.float64)),
            float(flat[-1]) if flat.size else 0.0)


def _device_volume(values: np.ndarray, dev):
    """(density fp32, cell records) on ``dev`` for ``values``, cached (see above)."""
    import weakref
    fp = _fingerprint(values)
    for k, (ref, key, d, dens, cells) in enumerate(_VOLUME_CACHE):
        if ref() is values and key == fp and d == dev:
            _VOLUME_CACHE.insert(0, _VOLUME_CACHE.pop(k))
            return dens, cells
    dens = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32)).to(dev)
    cells = R.pack_cells(dens)
    try:
        ref = weakref.ref(values)
    except TypeError:          # (not weak-referenceable: never cached)
        return dens, cells
    _VOLUME_CACHE.insert(0, (ref, fp, dev, dens, cells))
    del _VOLUME_CACHE[_VOLUME_CACHE_SIZE:]
    return dens, cells


def _upload(volume, tf, cam, dev):
    values = np.asarray(volume.values)
    if values.ndim != 3:
        raise InvalidParameterError("volume values must be a non-empty 3D array")
    dens, cells = _device_volume(values, dev)
    tex = torch.from_numpy(np.ascontiguousarray(np.asarray(tf.texels), dtype=np.float32)).to(dev)
    if tex.dim() != 2 or tex.shape[1] != 4:
        raise InvalidParameterError("transfer function must have shape (R, 4), R >= 1")
    ll = torch.tensor([[float(cam.lon_deg), float(cam.lat_deg)]], dtype=torch.float64)
    cams = R.camera_array(ll.to(dev), float(cam.radius),
                          tuple(np.asarray(cam.center, np.float64).reshape(3)),
                          float(cam.fov_y_deg))
    rig = R.Rig(int(cam.width), int(cam.height),
                tuple(np.asarray(volume.box_min, np.float64).reshape(3)),
                tuple(np.asarray(volume.box_max, np.float64).reshape(3)))
    return dens, tex, cams, rig, cells


def _image_from(img, depth):
    """fp64 ImageRGBA; the ray optical depth S (T = exp(-S)) rides along.

    alpha = A is accurate as A -> 0; S keeps T accurate as T -> 0.
    ``render_adjoint(image=...)`` starts the inversion from the attached S
    when the image came from :func:`render`, else from S = -ln(1 - alpha).
    """
    out = ImageRGBA(img[0].to(torch.float64).cpu().numpy())
    out._ddvr_depth = depth[0].cpu().numpy()
    return out


# ---------------------------------------------------------------------------
# public entry points
# ---------------------------------------------------------------------------


def render(volume, tf, cam, cfg, *, threads: int = 1) -> ImageRGBA:
    """Direct volume rendering (renderer.py:393-401); early termination only for target none."""
    _validate_config(cfg)
    dev = _device()
    dens, tex, cams, rig, cells = _upload(volume, tf, cam, dev)
    img, depth = R.forward(dens, tex, cams, cfg.dt, rig, early_stop=(cfg.target == "none"),
                           cells=cells)
    return _image_from(img, depth)


def fibonacci_views(count: int, radius: float, center=(0.0, 0.0, 0.0), fov_y_deg: float = 30.0,
                    width: int = 64, height: int = 64):
    """Golden-angle spiral of cameras on the sphere (tasks.py:118-128)."""
    from .scenes import fibonacci_poses
    return [SphericalCamera(lon, lat, radius, center, fov_y_deg, width, height)
            for lon, lat in fibonacci_poses(count)]


def render_forward_grad(volume, tf, cam, cfg, *, threads: int = 1):
    """Image and its per-pixel Jacobian by forward mode (renderer.py:410-464).

    Targets ``camera`` (p=2, per degree) and ``stepsize`` (p=1); returns
    ``(ImageRGBA, jacobian (H, W, 4, p) float64)``.
    """
    _validate_config(cfg)
    if cfg.target not in ("camera", "stepsize"):
        raise UnsupportedConfigurationError(
            f"forward mode supports camera and stepsize, not {cfg.target!r}")
    dev = _device()
    dens, tex, cams, rig, cells = _upload(volume, tf, cam, dev)
    img, jac = R.forward_grad(dens, tex, cams, cfg.dt, rig, cfg.target,
                              cells=cells)
    return (ImageRGBA(img[0].to(torch.float64).cpu().numpy()),
            jac[0].to(torch.float64).cpu().numpy())


def _upload_color(cv, cam, dev):
    values = np.asarray(cv.values)
    if values.ndim != 4 or values.shape[3] != 4:
        raise InvalidParameterError("color volume must have shape (X, Y, Z, 4)")
    col = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32)).to(dev)
    ll = torch.tensor([[float(cam.lon_deg), float(cam.lat_deg)]], dtype=torch.float64)
    cams = R.camera_array(ll.to(dev), float(cam.radius),
                          tuple(np.asarray(cam.center, np.float64).reshape(3)),
                          float(cam.fov_y_deg))
    rig = R.Rig(int(cam.width), int(cam.height),
                tuple(np.asarray(cv.box_min, np.float64).reshape(3)),
                tuple(np.asarray(cv.box_max, np.float64).reshape(3)))
    return col, cams, rig


def render_colorvol(cv, cam, cfg, *, threads: int = 1) -> ImageRGBA:
    """Render a pre-shaded colour volume (renderer.py:404-407)."""
    _validate_config(cfg)
    dev = _device()
    col, cams, rig = _upload_color(cv, cam, dev)
    img, depth = R.forward_color(col, cams, cfg.dt, rig, early_stop=(cfg.target == "none"))
    return _image_from(img, depth)


def render_colorvol_adjoint(cv, cam, cfg, seed, *, threads: int = 1, image=None) -> GradientSet:
    """Adjoint for the pre-shaded colour volume; target must be ``volume`` (renderer.py:703-709)."""
    _validate_config(cfg)
    if cfg.target != "volume":
        raise UnsupportedConfigurationError("color volumes differentiate per-voxel rgba only")
    seed_arr = seed.data if hasattr(seed, "data") and not isinstance(seed, np.ndarray) else seed
    seed_arr = np.asarray(seed_arr, dtype=np.float64)
    H, W = int(cam.height), int(cam.width)
    if seed_arr.shape != (H, W, 4):
        raise InvalidInputError(f"seed shape {seed_arr.shape} does not match image {(H, W, 4)}")
    dev = _device()
    col, cams, rig = _upload_color(cv, cam, dev)
    stored = getattr(cfg, "memory_mode", "inversion") == "stored"
    tape, stride, n_steps = None, 0, None
    if stored:
        n_steps = _stored_tape_len(cams, cfg.dt, rig)
        stride = max(int(n_steps.max().item()), 1)
        tape = torch.empty(H * W * stride, dtype=torch.float32, device=dev)
    if image is None or stored:
        img_t, depth_t = R.forward_color(col, cams, cfg.dt, rig, tape=tape, tape_stride=stride)
    else:
        img_arr = image.data if hasattr(image, "data") and not isinstance(image, np.ndarray) \
            else image
        img_arr = np.asarray(img_arr, np.float64)
        if img_arr.shape != (H, W, 4):
            raise InvalidInputError("provided image does not match the camera size")
        img_t = torch.from_numpy(img_arr.astype(np.float32)).to(dev).reshape(1, H, W, 4)
        s_np = getattr(image, "_ddvr_depth", None)
        if s_np is None or np.shape(s_np) != (H, W):
            with np.errstate(divide="ignore"):
                s_np = -np.log1p(-np.clip(img_arr[..., 3], 0.0, 1.0))
        depth_t = torch.from_numpy(np.asarray(s_np, np.float32)).to(dev).reshape(1, H, W)
    seed_t = torch.from_numpy(seed_arr.astype(np.float32)).to(dev).reshape(1, H, W, 4)
    d_col = torch.zeros_like(col)
    R.adjoint_color(col, cams, cfg.dt, rig, img_t, depth_t, seed_t, d_col, tape=tape,
                    tape_stride=stride)
    if stored:
        n_cpu = n_steps[0].cpu().numpy()
        state = 8 * H * W + sum(int(n_cpu[r:r + TILE_ROWS].max()) * n_cpu[r:r + TILE_ROWS].size
                                for r in range(0, H, TILE_ROWS))
    else:
        state = 8 * H * W
    return GradientSet(d_color=d_col.to(torch.float64).cpu().numpy(), state_floats=int(state))


def _stored_tape_len(cams, dt, rig):
    _, n, _ = R.ray_setup(cams, dt, rig)
    return n


def render_adjoint(volume, tf, cam, cfg, seed, *, threads: int = 1, image=None) -> GradientSet:
    """Gradient of sum(seed * image) for ``cfg.target`` (renderer.py:688-700, 655-685)."""
    _validate_config(cfg)
    if cfg.target == "none":
        raise UnsupportedConfigurationError("adjoint requires a differentiation target")
    seed_arr = seed.data if hasattr(seed, "data") and not isinstance(seed, np.ndarray) else seed
    seed_arr = np.asarray(seed_arr, dtype=np.float64)
    H, W = int(cam.height), int(cam.width)
    if seed_arr.shape != (H, W, 4):
        raise InvalidInputError(f"seed shape {seed_arr.shape} does not match image {(H, W, 4)}")
    img_arr = None
    if image is not None:
        img_arr = image.data if hasattr(image, "data") and not isinstance(image, np.ndarray) \
            else image
        img_arr = np.asarray(img_arr, dtype=np.float64)
        if img_arr.shape != (H, W, 4):
            raise InvalidInputError("provided image does not match the camera size")
    dev = _device()
    dens, tex, cams, rig, cells = _upload(volume, tf, cam, dev)
    stored = getattr(cfg, "memory_mode", "inversion") == "stored"
    tape = None
    n_steps = None
    stride = 0
    if stored:
        n_steps = _stored_tape_len(cams, cfg.dt, rig)
        stride = max(int(n_steps.max().item()), 1)
        tape = torch.empty(H * W * stride, dtype=torch.float32, device=dev)
        img_t, depth_t = R.forward(dens, tex, cams, cfg.dt, rig, cells=cells, tape=tape,
                                   tape_stride=stride)
    elif img_arr is None:
        img_t, depth_t = R.forward(dens, tex, cams, cfg.dt, rig, cells=cells)
    else:
        img_t = torch.from_numpy(img_arr.astype(np.float32)).to(dev).reshape(1, H, W, 4)
        s_np = getattr(image, "_ddvr_depth", None)
        if s_np is None or np.shape(s_np) != (H, W):
            with np.errstate(divide="ignore"):
                s_np = -np.log1p(-np.clip(img_arr[..., 3], 0.0, 1.0))
        depth_t = torch.from_numpy(np.asarray(s_np, np.float32)).to(dev).reshape(1, H, W)
    seed_t = torch.from_numpy(seed_arr.astype(np.float32)).to(dev).reshape(1, H, W, 4)
    bit = N.TARGET_BITS[cfg.target]
    d_vol = torch.zeros_like(dens) if bit == N.TARGET_VOLUME else None
    d_tf = torch.zeros(tex.shape, dtype=torch.float64, device=dev) if bit == N.TARGET_TF else None
    d_cam = torch.zeros(1, 2, dtype=torch.float64, device=dev) if bit == N.TARGET_CAMERA else None
    d_dt = torch.zeros(1, dtype=torch.float64, device=dev) if bit == N.TARGET_STEPSIZE else None
    R.adjoint(dens, tex, cams, cfg.dt, rig, img_t, depth_t, seed_t, bit, d_volume=d_vol,
              d_tf=d_tf, d_camera=d_cam, d_dt=d_dt, cells=cells, tape=tape, tape_stride=stride)
    # per-ray state: inversion keeps (C, A) and the constant seed, 8 floats per ray,
    # independent of the step count (renderer.py:513); stored mode keeps a tape
    # of one transmittance per sample, n_max per 64-row tile.
    if stored:
        n_cpu = n_steps[0].cpu().numpy()
        state = 8 * H * W + sum(int(n_cpu[r:r + TILE_ROWS].max()) * n_cpu[r:r + TILE_ROWS].size
                                for r in range(0, H, TILE_ROWS))
    else:
        state = 8 * H * W
    out = GradientSet(state_floats=int(state))
    if d_vol is not None:
        out.d_volume = d_vol.to(torch.float64).cpu().numpy()
    if d_tf is not None:
        out.d_tf = d_tf.cpu().numpy()
    if d_cam is not None:
        out.d_camera = d_cam[0].cpu().numpy()
    if d_dt is not None:
        out.d_stepsize = float(d_dt.item())
    return out


def opacity_entropy(image):
    """(H, seed (H,W,4) float64 with only alpha populated, degenerate) of the
    normalised Shannon entropy of the alpha channel (objectives.py:95-126)."""
    data = image.data if isinstance(image, ImageRGBA) or hasattr(image, "alpha") \
        else np.asarray(image, np.float64)
    data = np.asarray(data, np.float64)
    if data.ndim != 3 or data.shape[2] != 4:
        raise InvalidInputError("image data must have shape (H, W, 4)")
    t = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float32)).to(_device())
    h, seed, degenerate = R.opacity_entropy(t[None])
    return float(h[0]), seed[0].to(torch.float64).cpu().numpy(), bool(degenerate[0])


def l1_loss(images, refs):
    """(mean |x - y|, [sign(x - y)/count]) over all images (objectives.py:38-54)."""
    if len(images) != len(refs):
        raise InvalidInputError("image and reference counts differ")
    arr = lambda im: im.data if isinstance(im, ImageRGBA) or hasattr(im, "alpha") \
        else np.asarray(im, np.float64)  # noqa: E731
    xs = [np.asarray(arr(im), np.float64) for im in images]
    ys = [np.asarray(arr(r), np.float64) for r in refs]
    for x, y in zip(xs, ys):
        if x.shape != y.shape:
            raise InvalidInputError(f"image shape {x.shape} != reference shape {y.shape}")
    count = sum(x.size for x in xs)
    if count == 0:
        return 0.0, [np.zeros_like(x) for x in xs]
    dev = _device()
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    seeds = []
    for x, y in zip(xs, ys):
        xt = torch.from_numpy(x.astype(np.float32).ravel()).to(dev)
        yt = torch.from_numpy(y.astype(np.float32).ravel()).to(dev)
        st = torch.empty_like(xt)
        N.check(N.lib().ddvr_l1_loss(xt.data_ptr(), yt.data_ptr(), xt.numel(), float(count),
                                     st.data_ptr(), loss.data_ptr(), R._stream_ptr()))
        seeds.append(st.to(torch.float64).cpu().numpy().reshape(x.shape))
    return float(loss.item()), seeds



# ---------------------------------------------------------------------------
# point-wise field functions (field.py:186-600; SURVEY 8a rows a1, a4-a6, a9,
# a10): fp64 device kernels with the reference's operation order
# ---------------------------------------------------------------------------


def _dev64(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


def _box(a):
    return (ctypes.c_double * 3)(*np.asarray(a, np.float64).reshape(3))


def _field_call(volume, points, spatial: bool):
    values = np.asarray(volume.values, np.float64)
    if values.ndim != 3:
        raise InvalidParameterError("volume values must be a non-empty 3D array")
    pts = np.asarray(points, dtype=np.float64)
    if pts.shape[-1:] != (3,):
        raise InvalidInputError("points must have a trailing axis of 3")
    shape = pts.shape[:-1]
    n = int(np.prod(shape, dtype=np.int64))
    dev = _device()
    vt, pt = _dev64(values, dev), _dev64(pts.reshape(n, 3), dev)
    val = torch.empty(n, dtype=torch.float64, device=dev)
    sp = torch.empty(n, 3, dtype=torch.float64, device=dev) if spatial else None
    w = torch.empty(n, 8, dtype=torch.float64, device=dev) if spatial else None
    c = torch.empty(n, 8, dtype=torch.int64, device=dev) if spatial else None
    N.check(N.lib().ddvr_field_sample(
        vt.data_ptr(), (ctypes.c_int32 * 3)(*values.shape), _box(volume.box_min),
        _box(volume.box_max), pt.data_ptr(), n, val.data_ptr(),
        sp.data_ptr() if spatial else None, w.data_ptr() if spatial else None,
        c.data_ptr() if spatial else None, R._stream_ptr()))
    if not spatial:
        return val.cpu().numpy().reshape(shape)
    return (sp.cpu().numpy().reshape(shape + (3,)), w.cpu().numpy().reshape(shape + (8,)),
            c.cpu().numpy().reshape(shape + (8,)))


def trilinear_sample(volume, points) -> np.ndarray:
    """Density at world points, 0 outside the box, clamped to [0, 1] (field.py:352-358)."""
    return _field_call(volume, points, spatial=False)


def trilinear_gradients(volume, points):
    """(spatial (...,3), weights (...,8), corner_indices (...,8)) (field.py:503-517)."""
    return _field_call(volume, points, spatial=True)


def _tf_call(tf, d, grads: bool):
    tex = np.asarray(tf.texels, np.float64)
    if tex.ndim != 2 or tex.shape[1] != 4:
        raise InvalidParameterError("transfer function must have shape (R, 4), R >= 1")
    d = np.asarray(d, dtype=np.float64)
    shape = d.shape
    n = int(d.size)
    dev = _device()
    tt, dt_ = _dev64(tex, dev), _dev64(d.reshape(n), dev)
    out = torch.empty(n, 4, dtype=torch.float64, device=dev) if not grads else None
    sl = torch.empty(n, 4, dtype=torch.float64, device=dev) if grads else None
    w = torch.empty(n, 2, dtype=torch.float64, device=dev) if grads else None
    ix = torch.empty(n, 2, dtype=torch.int64, device=dev) if grads else None
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    N.check(N.lib().ddvr_tf_lookup(tt.data_ptr(), tex.shape[0], dt_.data_ptr(), n, ptr(out),
                                   ptr(sl), ptr(w), ptr(ix), R._stream_ptr()))
    if not grads:
        return out.cpu().numpy().reshape(shape + (4,))
    return (sl.cpu().numpy().reshape(shape + (4,)), w.cpu().numpy().reshape(shape + (2,)),
            ix.cpu().numpy().reshape(shape + (2,)))


def tf_sample(tf, d) -> np.ndarray:
    """(rgb emission, tau) (..., 4) for densities d, clamp-to-edge (field.py:552-555)."""
    return _tf_call(tf, d, grads=False)


def tf_gradients(tf, d):
    """(slope (...,4), weights (...,2), texel_indices (...,2)) (field.py:558-579)."""
    return _tf_call(tf, d, grads=True)


def opacity_from_density(tau, dt):
    """(alpha, dalpha/dtau) of one segment, alpha <= 1 - EPS_ALPHA (field.py:587-600)."""
    tau = np.asarray(tau, dtype=np.float64)
    shape, n = tau.shape, int(tau.size)
    dev = _device()
    tt = _dev64(tau.reshape(n), dev)
    a = torch.empty(n, dtype=torch.float64, device=dev)
    da_ = torch.empty(n, dtype=torch.float64, device=dev)
    N.check(N.lib().ddvr_opacity(tt.data_ptr(), n, float(dt), a.data_ptr(), da_.data_ptr(),
                                 R._stream_ptr()))
    return a.cpu().numpy().reshape(shape), da_.cpu().numpy().reshape(shape)


def _camera_call(cam, u, v, jac: bool):
    u = np.asarray(u, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    W, H = int(cam.width), int(cam.height)
    if np.any(u < 0) or np.any(u >= W) or np.any(v < 0) or np.any(v >= H):   # field.py:231-236
        raise InvalidParameterError("pixel coordinates outside image bounds")
    u, v = np.broadcast_arrays(u, v)
    shape, n = u.shape, int(u.size)
    c = (ctypes.c_double * N.CAMERA_DOUBLES)(
        float(cam.lon_deg), float(cam.lat_deg), float(cam.radius),
        *np.asarray(cam.center, np.float64).reshape(3), float(cam.fov_y_deg), 0.0)
    dev = _device()
    ut, vt = _dev64(u.reshape(n), dev), _dev64(v.reshape(n), dev)
    o = torch.empty(n, 3, dtype=torch.float64, device=dev)
    d = torch.empty(n, 3, dtype=torch.float64, device=dev)
    jo = torch.empty(n, 3, 2, dtype=torch.float64, device=dev) if jac else None
    jd = torch.empty(n, 3, 2, dtype=torch.float64, device=dev) if jac else None
    N.check(N.lib().ddvr_camera_rays(c, W, H, ut.data_ptr(), vt.data_ptr(), n, o.data_ptr(),
                                     d.data_ptr(), jo.data_ptr() if jac else None,
                                     jd.data_ptr() if jac else None, R._stream_ptr()))
    if jac:
        return jo.cpu().numpy().reshape(shape + (3, 2)), jd.cpu().numpy().reshape(shape + (3, 2))
    return o.cpu().numpy().reshape(shape + (3,)), d.cpu().numpy().reshape(shape + (3,))


def camera_from_sphere(cam, u, v):
    """(origin, unit direction) through the centre of pixel (u, v) (field.py:239-250)."""
    return _camera_call(cam, u, v, jac=False)


def camera_gradients(cam, u, v):
    """(j_origin, j_direction) (..., 3, 2) w.r.t. (lon, lat) per degree (field.py:253-271)."""
    return _camera_call(cam, u, v, jac=True)


# ---------------------------------------------------------------------------
# the steps either side of the path: objectives.py:57-92,
# optim.py:16-129 under the reference's names, on the libddvr kernels of optim.py
# (fp32 parameters, fp64 reductions)
# ---------------------------------------------------------------------------

TAU_MAX_DEFAULT = 100.0   # optim.py:12


def smoothness_prior_tf(tf):
    """(mean squared adjacent-texel difference, gradient (R,4)) (objectives.py:57-69)."""
    from . import optim as P
    tex = np.asarray(tf.texels if hasattr(tf, "texels") else tf, np.float64)
    if tex.shape[0] < 2:
        return 0.0, np.zeros_like(tex)
    dev = _device()
    g = torch.zeros(tex.shape, dtype=torch.float64, device=dev)
    val = P.prior_tf(torch.from_numpy(tex.astype(np.float32)).to(dev), 1.0, g)
    return float(val.item()), g.cpu().numpy()


def smoothness_prior_volume(volume):
    """(mean squared forward difference, gradient (X,Y,Z)) (objectives.py:72-92)."""
    from . import optim as P
    v = np.asarray(volume.values if hasattr(volume, "values") else volume, np.float64)
    if v.ndim != 3:
        raise InvalidParameterError("volume values must be a non-empty 3D array")
    dev = _device()
    vt = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).to(dev)
    g = torch.zeros_like(vt)
    val = P.prior_volume(vt, 1.0, g)
    return float(val.item()), g.to(torch.float64).cpu().numpy()


@dataclass
class OptimState:
    """Adam moment accumulators for one parameter vector (optim.py:15-25)."""

    lr: float
    m: np.ndarray | None = None
    v: np.ndarray | None = None
    step: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


def _params_pair(params, grads):
    p = np.asarray(params, dtype=np.float64)
    g = np.asarray(grads, dtype=np.float64)
    if p.shape != g.shape:
        raise InvalidParameterError("parameter/gradient shape mismatch")
    dev = _device()
    return (p, torch.from_numpy(np.ascontiguousarray(p, np.float32)).to(dev),
            torch.from_numpy(np.ascontiguousarray(g, np.float32)).to(dev))


def gd_step(params, grads, lr: float):
    """params - lr * grads (optim.py:33-42); NumericalAbortError on non-finite grads."""
    from .errors import NumericalAbortError
    p, pt, gt = _params_pair(params, grads)
    if lr <= 0.0:
        raise InvalidParameterError("learning rate must be positive")
    flag = torch.zeros(1, dtype=torch.int32, device=pt.device)
    N.check(N.lib().ddvr_gd_step(pt.data_ptr(), gt.data_ptr(), pt.numel(), float(lr),
                                 flag.data_ptr(), R._stream_ptr()))
    if int(flag.item()):
        raise NumericalAbortError("non-finite gradients passed to the optimizer")
    return pt.to(torch.float64).cpu().numpy().reshape(p.shape)


def adam_step(state, params, grads):
    """One Adam update with bias correction; returns ``(new state, params)`` (optim.py:45-67)."""
    from . import optim as P
    p, pt, gt = _params_pair(params, grads)
    st = P.AdamState(lr=float(state.lr), beta1=float(state.beta1), beta2=float(state.beta2),
                     eps=float(state.eps), step=int(state.step))
    dev = pt.device
    st.m = (torch.zeros_like(pt) if state.m is None else
            torch.from_numpy(np.ascontiguousarray(state.m, np.float32)).to(dev).reshape(pt.shape))
    st.v = (torch.zeros_like(pt) if state.v is None else
            torch.from_numpy(np.ascontiguousarray(state.v, np.float32)).to(dev).reshape(pt.shape))
    st.flag = torch.zeros(1, dtype=torch.int32, device=dev)
    st.update(pt, gt, project=None)
    new = OptimState(lr=state.lr, m=st.m.to(torch.float64).cpu().numpy().reshape(p.shape),
                     v=st.v.to(torch.float64).cpu().numpy().reshape(p.shape), step=st.step,
                     beta1=state.beta1, beta2=state.beta2, eps=state.eps)
    return new, pt.to(torch.float64).cpu().numpy().reshape(p.shape)


def project_params(params, target: str, tau_max: float = TAU_MAX_DEFAULT):
    """Clamp parameters into their physical range; idempotent (optim.py:70-89)."""
    p = np.asarray(params, dtype=np.float64)
    inf = float("inf")
    if target == "volume":
        cfg = (1, 0.0, 1.0, 0.0, 1.0)
    elif target in ("tf", "color"):
        cfg = (4, 0.0, float(tau_max), 0.0, inf)
    else:
        raise InvalidParameterError(f"unknown projection target {target!r}")
    dev = _device()
    pt = torch.from_numpy(np.ascontiguousarray(p, np.float32)).to(dev)
    a = N.DdvrAdam(0.0, 0.0, 0.0, 0.0, 0, *cfg)
    N.check(N.lib().ddvr_project(pt.data_ptr(), pt.numel(), ctypes.byref(a), R._stream_ptr()))
    return pt.to(torch.float64).cpu().numpy().reshape(p.shape)


def upsample_volume(volume):
    """Double the grid resolution per axis, world box unchanged (optim.py:114-129)."""
    from . import optim as P
    if isinstance(volume, ColorVolume) or (hasattr(volume, "values")
                                           and np.ndim(volume.values) == 4):
        vals = np.asarray(volume.values, np.float64)
        dev = _device()
        chans = [P.upsample_volume(torch.from_numpy(np.ascontiguousarray(vals[..., c], np.float32))
                                   .to(dev)) for c in range(vals.shape[3])]
        up = torch.stack(chans, dim=3).to(torch.float64).cpu().numpy()
        return ColorVolume(up, np.array(volume.box_min, np.float64),
                           np.array(volume.box_max, np.float64))
    if not hasattr(volume, "values"):
        raise InvalidParameterError("upsample_volume expects a density or color volume")
    vals = np.asarray(volume.values, np.float64)
    up = P.upsample_volume(torch.from_numpy(np.ascontiguousarray(vals, np.float32)).to(_device()))
    return DensityVolume(up.to(torch.float64).cpu().numpy(), np.array(volume.box_min, np.float64),
                         np.array(volume.box_max, np.float64))


# ---------------------------------------------------------------------------
# synthetic inputs of the benchmarks under the reference's names
# ---------------------------------------------------------------------------


def make_phantom(kind: str, dims, seed: int = 0, box_min=(-0.5, -0.5, -0.5),
                 box_max=(0.5, 0.5, 0.5)) -> DensityVolume:
    """Stock phantom as a DensityVolume (phantoms.py:26-72); host NumPy, input data only."""
    from .scenes import phantom
    return DensityVolume(phantom(kind, dims, seed, box_min, box_max), np.asarray(box_min),
                         np.asarray(box_max))


def make_absorption_ramp_tf(resolution: int = 64, tau_scale: float = 3.0) -> TransferFunction:
    """Emission-free TF with absorption linear in density (tasks.py:348-356)."""
    from .scenes import absorption_ramp_texels
    return TransferFunction(absorption_ramp_texels(resolution, tau_scale))


def preset_tf(name: str, resolution: int = 16, tau_scale: float = 4.0) -> TransferFunction:
    """Stock transfer functions grayscale / warm / gaussian (tasks.py:359-388)."""
    from .scenes import preset_texels
    return TransferFunction(preset_texels(name, resolution, tau_scale))
