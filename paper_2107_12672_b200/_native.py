"""ctypes binding of libddvr.so (include/ddvr.h) -- the only door to the kernels.

There is no CPU fallback: if the shared library is missing or fails to load,
every call raises ``NativeLibraryError``.  The library is built in-tree by
``paper_2107_12672_b200/_build.py`` (``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os

from .errors import (
    InvalidInputError,
    InvalidParameterError,
    UnsupportedConfigurationError,
    VoldiffError,
)

LIB_PATH = os.environ.get("DDVR_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                      "libddvr.so")
ABI_VERSION = 4

TARGET_CAMERA = 1
TARGET_STEPSIZE = 2
TARGET_TF = 4
TARGET_VOLUME = 8
TARGET_BITS = {"camera": TARGET_CAMERA, "stepsize": TARGET_STEPSIZE, "tf": TARGET_TF,
               "volume": TARGET_VOLUME}

FLAG_WS_CONTINUE = 1   # ddvr_params.flags (include/ddvr.h)
FLAG_WS_DEFER = 2
FLAG_DETERMINISTIC = 4
FLAG_BAND_TAPE = 8
FLAG_NO_EMPTY_SKIP = 16
FLAG_SPLIT_WALK = 32
FLAG_RAY_SPLIT = {1: 64, 2: 128, 4: 256, 8: 512}   # DDVR_FLAG_RAY_SPLIT_OFF / _2 / _4 / _8
TF_TEXTURE = 0
TF_PIECEWISE = 1
TF_GAUSSIAN = 2

EXPORTED = ("ddvr_forward", "ddvr_adjoint", "ddvr_forward_adjoint_l1",
            "ddvr_adjoint_workspace_bytes", "ddvr_deterministic_bytes", "ddvr_band_tape_bytes", "ddvr_ray_split", "ddvr_cells_bytes", "ddvr_pack_cells", "ddvr_forward_grad", "ddvr_forward_color",
            "ddvr_adjoint_color", "ddvr_l1_loss", "ddvr_opacity_entropy", "ddvr_gather_probe",
            "ddvr_ray_setup",
            "ddvr_prior_volume",
            "ddvr_prior_tf", "ddvr_adam_step", "ddvr_adam_step_device",
            "ddvr_upsample_volume", "ddvr_project", "ddvr_gd_step", "ddvr_field_sample",
            "ddvr_tf_lookup", "ddvr_opacity", "ddvr_camera_rays", "ddvr_volume_from_raw",
            "ddvr_volume_to_raw", "ddvr_image_to_ppm", "ddvr_last_error",
            "ddvr_abi_version", "ddvr_launch_count")


class NativeLibraryError(VoldiffError, RuntimeError):
    """libddvr.so is missing, stale or failed to load (no fallback exists)."""


class CudaError(VoldiffError, RuntimeError):
    """A CUDA launch failed inside libddvr."""


class DdvrVolume(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dims", ctypes.c_int32 * 3),
                ("box_min", ctypes.c_double * 3), ("box_max", ctypes.c_double * 3),
                ("cells", ctypes.c_void_p)]


class DdvrTf(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("count", ctypes.c_int32), ("params", ctypes.c_void_p)]


class DdvrParams(ctypes.Structure):
    _fields_ = [("dt", ctypes.c_double), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("row0", ctypes.c_int32), ("row1", ctypes.c_int32),
                ("early_stop", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("tape", ctypes.c_void_p), ("tape_stride", ctypes.c_int64),
                ("stats", ctypes.c_void_p)]


class DdvrAdam(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("step", ctypes.c_int32), ("stride", ctypes.c_int32),
                ("lo", ctypes.c_float), ("hi", ctypes.c_float), ("lo_other", ctypes.c_float),
                ("hi_other", ctypes.c_float)]


CAMERA_DOUBLES = 8   # sizeof(ddvr_camera) / 8: lon, lat, radius, cx, cy, cz, fov, reserved

_lib = None


def _bind(lib):
    P = ctypes.POINTER
    vp = ctypes.c_void_p
    lib.ddvr_forward.argtypes = [P(DdvrVolume), P(DdvrTf), vp, ctypes.c_int32, P(DdvrParams),
                                 vp, vp, vp]
    lib.ddvr_forward.restype = ctypes.c_int
    lib.ddvr_adjoint.argtypes = [P(DdvrVolume), P(DdvrTf), vp, ctypes.c_int32, P(DdvrParams),
                                 vp, vp, vp, ctypes.c_uint32, vp, vp, vp, vp, vp,
                                 ctypes.c_int64, vp]
    lib.ddvr_adjoint.restype = ctypes.c_int
    lib.ddvr_forward_adjoint_l1.argtypes = [P(DdvrVolume), P(DdvrTf), vp, ctypes.c_int32,
                                            P(DdvrParams), vp, ctypes.c_double, ctypes.c_uint32,
                                            vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int64, vp]
    lib.ddvr_forward_adjoint_l1.restype = ctypes.c_int
    lib.ddvr_forward_grad.argtypes = [P(DdvrVolume), P(DdvrTf), vp, ctypes.c_int32,
                                      P(DdvrParams), ctypes.c_uint32, vp, vp, vp]
    lib.ddvr_forward_grad.restype = ctypes.c_int
    lib.ddvr_forward_color.argtypes = [P(DdvrVolume), vp, ctypes.c_int32, P(DdvrParams), vp, vp,
                                       vp]
    lib.ddvr_forward_color.restype = ctypes.c_int
    lib.ddvr_adjoint_color.argtypes = [P(DdvrVolume), vp, ctypes.c_int32, P(DdvrParams), vp, vp,
                                       vp, vp, vp]
    lib.ddvr_adjoint_color.restype = ctypes.c_int
    lib.ddvr_adjoint_workspace_bytes.argtypes = [P(DdvrVolume), P(DdvrTf), ctypes.c_uint32]
    lib.ddvr_adjoint_workspace_bytes.restype = ctypes.c_int64
    lib.ddvr_deterministic_bytes.argtypes = [P(DdvrVolume), ctypes.c_int32, P(DdvrParams),
                                             ctypes.c_uint32]
    lib.ddvr_deterministic_bytes.restype = ctypes.c_int64
    lib.ddvr_band_tape_bytes.argtypes = [P(DdvrVolume), ctypes.c_int32, P(DdvrParams)]
    lib.ddvr_band_tape_bytes.restype = ctypes.c_int64
    lib.ddvr_ray_split.argtypes = [ctypes.c_uint32, ctypes.c_int64, ctypes.c_int32]
    lib.ddvr_ray_split.restype = ctypes.c_int32
    lib.ddvr_cells_bytes.argtypes = [P(ctypes.c_int32)]
    lib.ddvr_cells_bytes.restype = ctypes.c_int64
    lib.ddvr_pack_cells.argtypes = [P(DdvrVolume), vp, vp]
    lib.ddvr_pack_cells.restype = ctypes.c_int
    lib.ddvr_l1_loss.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_double, vp, vp, vp]
    lib.ddvr_l1_loss.restype = ctypes.c_int
    lib.ddvr_opacity_entropy.argtypes = [vp, ctypes.c_int64, ctypes.c_int32, vp, vp, vp]
    lib.ddvr_opacity_entropy.restype = ctypes.c_int
    lib.ddvr_gather_probe.argtypes = [P(DdvrVolume), vp, ctypes.c_int32, P(DdvrParams),
                                      ctypes.c_int32, vp, vp]
    lib.ddvr_gather_probe.restype = ctypes.c_int
    lib.ddvr_ray_setup.argtypes = [P(DdvrVolume), vp, ctypes.c_int32, P(DdvrParams), vp, vp, vp,
                                   vp]
    lib.ddvr_ray_setup.restype = ctypes.c_int
    i3 = P(ctypes.c_int32)
    lib.ddvr_prior_volume.argtypes = [vp, i3, ctypes.c_double, vp, vp, vp]
    lib.ddvr_prior_volume.restype = ctypes.c_int
    lib.ddvr_prior_tf.argtypes = [vp, ctypes.c_int32, ctypes.c_double, vp, vp, vp]
    lib.ddvr_prior_tf.restype = ctypes.c_int
    lib.ddvr_adam_step.argtypes = [vp, vp, vp, vp, ctypes.c_int64, P(DdvrAdam), vp, vp]
    lib.ddvr_adam_step.restype = ctypes.c_int
    lib.ddvr_adam_step_device.argtypes = [vp, vp, vp, vp, ctypes.c_int64, P(DdvrAdam), vp, vp,
                                          vp]
    lib.ddvr_adam_step_device.restype = ctypes.c_int
    lib.ddvr_upsample_volume.argtypes = [vp, i3, vp, vp]
    lib.ddvr_upsample_volume.restype = ctypes.c_int
    lib.ddvr_project.argtypes = [vp, ctypes.c_int64, P(DdvrAdam), vp]
    lib.ddvr_project.restype = ctypes.c_int
    lib.ddvr_gd_step.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_double, vp, vp]
    lib.ddvr_gd_step.restype = ctypes.c_int
    d3 = P(ctypes.c_double)
    lib.ddvr_field_sample.argtypes = [vp, i3, d3, d3, vp, ctypes.c_int64, vp, vp, vp, vp, vp]
    lib.ddvr_field_sample.restype = ctypes.c_int
    lib.ddvr_tf_lookup.argtypes = [vp, ctypes.c_int32, vp, ctypes.c_int64, vp, vp, vp, vp, vp]
    lib.ddvr_tf_lookup.restype = ctypes.c_int
    lib.ddvr_opacity.argtypes = [vp, ctypes.c_int64, ctypes.c_double, vp, vp, vp]
    lib.ddvr_opacity.restype = ctypes.c_int
    lib.ddvr_camera_rays.argtypes = [d3, ctypes.c_int32, ctypes.c_int32, vp, vp, ctypes.c_int64,
                                     vp, vp, vp, vp, vp]
    lib.ddvr_camera_rays.restype = ctypes.c_int
    lib.ddvr_volume_from_raw.argtypes = [vp, i3, P(ctypes.c_double), vp, vp]
    lib.ddvr_volume_from_raw.restype = ctypes.c_int
    lib.ddvr_volume_to_raw.argtypes = [vp, i3, vp, vp]
    lib.ddvr_volume_to_raw.restype = ctypes.c_int
    lib.ddvr_image_to_ppm.argtypes = [vp, ctypes.c_int64, vp, vp]
    lib.ddvr_image_to_ppm.restype = ctypes.c_int
    lib.ddvr_last_error.argtypes = []
    lib.ddvr_last_error.restype = ctypes.c_char_p
    lib.ddvr_abi_version.argtypes = []
    lib.ddvr_abi_version.restype = ctypes.c_int32
    lib.ddvr_launch_count.argtypes = []
    lib.ddvr_launch_count.restype = ctypes.c_int64


def lib():
    """The loaded library; raises NativeLibraryError if it cannot be loaded."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        try:
            handle = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name in EXPORTED:
            if not hasattr(handle, name):
                raise NativeLibraryError(f"{LIB_PATH} does not export {name}")
        _bind(handle)
        if handle.ddvr_abi_version() != ABI_VERSION:
            raise NativeLibraryError(
                f"{LIB_PATH} ABI {handle.ddvr_abi_version()} != expected {ABI_VERSION}")
        _lib = handle
    return _lib


def check(rc: int) -> None:
    """Map a ddvr_status to the reference exception classes (errors.py:4-33)."""
    if rc == 0:
        return
    msg = lib().ddvr_last_error().decode(errors="replace")
    if rc == 1:
        raise InvalidParameterError(msg)
    if rc == 2:
        raise InvalidInputError(msg)
    if rc == 3:
        raise UnsupportedConfigurationError(msg)
    raise CudaError(msg or f"ddvr status {rc}")


def launch_count() -> int:
    return int(lib().ddvr_launch_count())
