"""Volume / transfer-function / image files (drop-in for voldiff.fileio, fileio.py:1-127).

Same names, file formats and exceptions as the reference:

* volumes: ``<stem>.raw`` little-endian float32 in **x-fastest** order plus a
  ``<stem>.json`` sidecar {schema_version, dims, box_min, box_max[, value_range]}
  (fileio.py:27-71);
* transfer functions: JSON {schema_version, texels} (fileio.py:74-91);
* images: binary PPM composited over white, or a raw float32 rgba dump
  (fileio.py:94-127).

The host functions parse and write the formats byte-for-byte like the
reference (they return the reference's float64 dataclasses).  The device
loaders are the path a tomography run uses to put a real volume into HBM:
``load_volume_device`` reads the raw body straight into pinned memory, copies
it to the GPU and lets ``ddvr_volume_from_raw`` swap x-fastest -> z-fastest
with the ``value_range`` normalisation fused; ``save_volume_device`` and
``images_to_ppm`` run the reverse swap and the PPM quantiser on the device so
only the file bytes cross PCIe.
"""

from __future__ import annotations

import ctypes
import json
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from .errors import CorruptFileError, InvalidParameterError, MissingMetadataError
from .voldiff_api import DensityVolume, ImageRGBA, TransferFunction

SCHEMA_VERSION = 1      # fileio.py:19


def _stem(path) -> Path:
    p = Path(path)
    return p.with_suffix("") if p.suffix in (".raw", ".json") else p


def _write_sidecar(stem: Path, dims, box_min, box_max) -> None:
    sidecar = {
        "schema_version": SCHEMA_VERSION,
        "dims": [int(d) for d in dims],
        "box_min": [float(c) for c in box_min],
        "box_max": [float(c) for c in box_max],
    }
    stem.with_suffix(".json").write_text(json.dumps(sidecar, indent=2) + "\n")


def _read_meta(path):
    """Sidecar checks in the reference's order (fileio.py:45-63)."""
    stem = _stem(path)
    raw_path, meta_path = stem.with_suffix(".raw"), stem.with_suffix(".json")
    if not meta_path.exists():
        raise MissingMetadataError(f"sidecar not found: {meta_path}")
    if not raw_path.exists():
        raise CorruptFileError(f"raw data not found: {raw_path}")
    meta = json.loads(meta_path.read_text())
    for key in ("dims", "box_min", "box_max"):
        if key not in meta:
            raise MissingMetadataError(f"sidecar missing field {key!r}")
    dims = tuple(int(d) for d in meta["dims"])
    if len(dims) != 3 or min(dims) < 1:
        raise MissingMetadataError(f"invalid dims {dims} in sidecar")
    size = raw_path.stat().st_size
    expected = dims[0] * dims[1] * dims[2] * 4
    if size != expected:
        raise CorruptFileError(
            f"{raw_path}: expected {expected} bytes for dims {dims}, found {size}")
    vr = meta.get("value_range")
    if vr is not None:
        lo, hi = (float(v) for v in vr)
        if hi <= lo:
            raise MissingMetadataError("value_range must be increasing")
        vr = (lo, hi)
    return raw_path, dims, vr, np.asarray(meta["box_min"], np.float64), \
        np.asarray(meta["box_max"], np.float64)


# ---------------------------------------------------------------------------
# host formats (byte-identical to the reference)
# ---------------------------------------------------------------------------


def save_volume(volume, path) -> Path:
    """Write ``<stem>.raw`` plus its JSON sidecar; returns the raw path (fileio.py:27-40)."""
    stem = _stem(path)
    raw_path = stem.with_suffix(".raw")
    data = np.asarray(volume.values, dtype="<f4")
    raw_path.write_bytes(data.ravel(order="F").tobytes())
    _write_sidecar(stem, data.shape, volume.box_min, volume.box_max)
    return raw_path


def load_volume(path) -> DensityVolume:
    """Read a raw volume through its sidecar; normalises if a range is given (fileio.py:43-71)."""
    raw_path, dims, vr, bmin, bmax = _read_meta(path)
    values = np.frombuffer(raw_path.read_bytes(), dtype="<f4").reshape(dims, order="F")
    values = values.astype(np.float64)
    if vr is not None:
        values = (values - vr[0]) / (vr[1] - vr[0])
    return DensityVolume(values, bmin, bmax)


def save_tf(tf, path) -> Path:
    """Texels as JSON (fileio.py:74-80)."""
    p = Path(path)
    p.write_text(json.dumps({
        "schema_version": SCHEMA_VERSION,
        "texels": [[float(c) for c in row] for row in np.asarray(tf.texels)],
    }, indent=2) + "\n")
    return p


def load_tf(path) -> TransferFunction:
    """fileio.py:83-91."""
    p = Path(path)
    if not p.exists():
        raise MissingMetadataError(f"transfer function file not found: {p}")
    meta = json.loads(p.read_text())
    if "texels" not in meta:
        raise MissingMetadataError("transfer function file missing 'texels'")
    return TransferFunction(np.asarray(meta["texels"], dtype=np.float64))


def _image_format(p: Path, fmt):
    if fmt is None:
        fmt = {"ppm": "ppm", "rgba": "raw-rgba"}.get(p.suffix.lstrip("."), None)
        if fmt is None:
            raise InvalidParameterError(f"cannot infer image format from {p.suffix!r}")
    if fmt not in ("ppm", "raw-rgba"):
        raise InvalidParameterError(f"unknown image format {fmt!r}")
    return fmt


def save_image(img, path, fmt: str | None = None) -> Path:
    """Binary PPM over white or raw float32 rgba (fileio.py:94-115).

    ``img`` is an ImageRGBA (host) or an (H, W, 4) float32 CUDA tensor, which
    is quantised on the device by ``ddvr_image_to_ppm``.
    """
    p = Path(path)
    fmt = _image_format(p, fmt)
    if isinstance(img, torch.Tensor):
        if img.dim() != 3 or img.shape[2] != 4:
            raise InvalidParameterError("image tensor must have shape (H, W, 4)")
        H, W = int(img.shape[0]), int(img.shape[1])
        if fmt == "ppm":
            body = images_to_ppm(img[None])[0]
        else:
            body = img.detach().to(torch.float32).cpu().numpy().astype("<f4").tobytes()
    else:
        data = np.asarray(img.data, dtype=np.float64)
        H, W = data.shape[0], data.shape[1]
        if fmt == "ppm":
            rgb = data[..., :3] + (1.0 - data[..., 3:4])     # premultiplied over white
            body = np.round(255.0 * np.clip(rgb, 0.0, 1.0)).astype(np.uint8).tobytes()
        else:
            body = np.asarray(data, dtype="<f4").tobytes()
    if fmt == "ppm":
        p.write_bytes(f"P6\n{W} {H}\n255\n".encode("ascii") + body)
    else:
        p.write_bytes(body)
    return p


def load_image_rgba(path, width: int, height: int) -> ImageRGBA:
    """Read back a raw-rgba dump written by save_image (fileio.py:118-127)."""
    blob = Path(path).read_bytes()
    expected = width * height * 4 * 4
    if len(blob) != expected:
        raise CorruptFileError(
            f"{path}: expected {expected} bytes for {width}x{height} rgba, found {len(blob)}")
    return ImageRGBA(np.frombuffer(blob, dtype="<f4").reshape(height, width, 4)
                     .astype(np.float64))


# ---------------------------------------------------------------------------
# device paths (HBM-resident volumes and image batches)
# ---------------------------------------------------------------------------


def _ptr(t) -> int:
    return t.data_ptr() if t is not None else 0


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def load_volume_device(path, device=None):
    """Load a raw volume into HBM as the (X,Y,Z) z-fastest float32 tensor.

    Same checks and exceptions as load_volume.  The raw body is read into
    pinned memory, copied once, and swapped/normalised by
    ``ddvr_volume_from_raw``.  Returns (values, box_min, box_max).
    """
    raw_path, dims, vr, bmin, bmax = _read_meta(path)
    device = torch.device(device if device is not None else "cuda")
    if device.type != "cuda":
        raise InvalidParameterError("load_volume_device needs a CUDA device")
    n = dims[0] * dims[1] * dims[2]
    host = torch.empty(n, dtype=torch.float32, pin_memory=True)
    with open(raw_path, "rb") as f:
        got = f.readinto(memoryview(host.numpy()).cast("B"))
    if got != 4 * n:
        raise CorruptFileError(f"{raw_path}: short read ({got} of {4 * n} bytes)")
    raw = host.to(device, non_blocking=True)
    out = torch.empty(dims, dtype=torch.float32, device=device)
    rng = (ctypes.c_double * 2)(*vr) if vr is not None else None
    with torch.cuda.device(device):
        N.check(N.lib().ddvr_volume_from_raw(_ptr(raw), (ctypes.c_int32 * 3)(*dims), rng,
                                             _ptr(out), _stream(device)))
    return out, bmin, bmax


def save_volume_device(values: torch.Tensor, box_min, box_max, path) -> Path:
    """Write a device (X,Y,Z) volume as ``<stem>.raw`` + sidecar (fileio.py:27-40)."""
    if values.dim() != 3 or not values.is_cuda:
        raise InvalidParameterError("values must be an (X, Y, Z) CUDA tensor")
    v = values.detach().to(torch.float32).contiguous()
    raw = torch.empty(v.numel(), dtype=torch.float32, device=v.device)
    dims = tuple(int(d) for d in v.shape)
    with torch.cuda.device(v.device):
        N.check(N.lib().ddvr_volume_to_raw(_ptr(v), (ctypes.c_int32 * 3)(*dims), _ptr(raw),
                                           _stream(v.device)))
    host = torch.empty(v.numel(), dtype=torch.float32, pin_memory=True)
    host.copy_(raw)
    stem = _stem(path)
    raw_path = stem.with_suffix(".raw")
    raw_path.write_bytes(host.numpy().astype("<f4", copy=False).tobytes())
    _write_sidecar(stem, dims, box_min, box_max)
    return raw_path


def images_to_ppm(images: torch.Tensor) -> list[bytes]:
    """PPM bodies (rgb over white, uint8) for a (V, H, W, 4) float32 CUDA batch."""
    if images.dim() != 4 or images.shape[3] != 4 or not images.is_cuda:
        raise InvalidParameterError("images must be a (V, H, W, 4) CUDA tensor")
    img = images.detach().to(torch.float32).contiguous()
    V, H, W = (int(s) for s in img.shape[:3])
    out = torch.empty(V * H * W * 3, dtype=torch.uint8, device=img.device)
    with torch.cuda.device(img.device):
        N.check(N.lib().ddvr_image_to_ppm(_ptr(img), V * H * W, _ptr(out),
                                          _stream(img.device)))
    host = out.cpu().numpy().reshape(V, H * W * 3)
    return [host[v].tobytes() for v in range(V)]


def save_images_ppm(images: torch.Tensor, paths) -> list[Path]:
    """Write one PPM per view of a device image batch."""
    paths = [Path(p) for p in paths]
    if len(paths) != int(images.shape[0]):
        raise InvalidParameterError("need one path per view")
    H, W = int(images.shape[1]), int(images.shape[2])
    header = f"P6\n{W} {H}\n255\n".encode("ascii")
    for p, body in zip(paths, images_to_ppm(images)):
        p.write_bytes(header + body)
    return paths


__all__ = ["SCHEMA_VERSION", "save_volume", "load_volume", "save_tf", "load_tf", "save_image",
           "load_image_rgba", "load_volume_device", "save_volume_device", "images_to_ppm",
           "save_images_ppm"]
