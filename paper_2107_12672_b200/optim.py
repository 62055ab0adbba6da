"""The steps either side of the path, on device.

Every tomography / TF-reconstruction iteration of the reference
(tasks.py:397-481, 258-340) follows the adjoint with a smoothness prior, one
Adam update and a projection; multiresolution runs upsample the volume
between levels.  These run as libddvr kernels here:

    smoothness_prior_volume  objectives.py:72-92   -> prior_volume
    smoothness_prior_tf      objectives.py:57-69   -> prior_tf
    adam_step                optim.py:45-67        -> AdamState.step (fused with)
    project_params           optim.py:70-89           the projection
    NumericalAbortError      optim.py:28-30           (non-finite gradients)
    upsample_volume          optim.py:92-129       -> upsample_volume
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from . import _native as N
from .errors import InvalidParameterError, NumericalAbortError
from .raymarch import _require, _stream_ptr

TAU_MAX_DEFAULT = 100.0   # optim.py:12


def _dims(values):
    return (ctypes.c_int32 * 3)(*values.shape)


def prior_volume(values: torch.Tensor, weight: float = 1.0, grad: torch.Tensor | None = None,
                 out: torch.Tensor | None = None):
    """weight * smoothness_prior_volume: returns the value (1,) f64; grad += weight * dP/dv.
    ``out``: a (1,) f64 device tensor the value is ADDED to (the caller zeroes it),
    instead of a fresh zeroed one."""
    _require(values, "volume", torch.float32, ndim=3)
    if out is None:
        out = torch.zeros(1, dtype=torch.float64, device=values.device)
    else:
        _require(out, "prior value", torch.float64)
        if out.numel() != 1:
            raise InvalidParameterError("the prior value output holds one float64")
    if grad is not None:
        _require(grad, "gradient", torch.float32)
    N.check(N.lib().ddvr_prior_volume(values.data_ptr(), _dims(values), float(weight),
                                      grad.data_ptr() if grad is not None else None,
                                      out.data_ptr(), _stream_ptr()))
    return out


def prior_tf(texels: torch.Tensor, weight: float = 1.0, grad: torch.Tensor | None = None):
    """weight * smoothness_prior_tf: value (1,) f64; grad (R,4) f64 += weight * dP/dtexels."""
    _require(texels, "texels", torch.float32, ndim=2)
    out = torch.zeros(1, dtype=torch.float64, device=texels.device)
    if grad is not None:
        _require(grad, "gradient", torch.float64)
    N.check(N.lib().ddvr_prior_tf(texels.data_ptr(), texels.shape[0], float(weight),
                                  grad.data_ptr() if grad is not None else None, out.data_ptr(),
                                  _stream_ptr()))
    return out


@dataclass
class AdamState:
    """Adam moments of one parameter tensor (OptimState, optim.py:15-25), on device."""

    lr: float
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    step: int = 0
    m: torch.Tensor | None = None
    v: torch.Tensor | None = None
    flag: torch.Tensor | None = field(default=None, repr=False)
    # device_step: the step counter lives on the device (ddvr_adam_step_device), so
    # the update can be captured in a CUDA graph and replayed; no host sync
    device_step: bool = False
    state: torch.Tensor | None = field(default=None, repr=False)

    def reset(self) -> None:
        """Back to the state before the first update (moments zeroed, t = 0), keeping
        the buffers (and any CUDA graph that captured them) in place."""
        self.step = 0
        for t in (self.m, self.v, self.flag, self.state):
            if t is not None:
                t.zero_()

    def update(self, params: torch.Tensor, grads: torch.Tensor, project: str | None = None,
               tau_max: float = TAU_MAX_DEFAULT, check_finite=True) -> None:
        """One in-place Adam step + projection (``volume``: [0,1]; ``tf``: rgb >= 0,
        tau in [0, tau_max]; None: unconstrained).  Raises NumericalAbortError
        (and leaves the parameters untouched) on a non-finite gradient; with
        ``device_step`` the update is still skipped on the device but nothing is
        raised (no host synchronisation).  ``check_finite="defer"``: no host
        synchronisation either; the device flag ``self.flag`` is sticky (never
        re-zeroed), so once set every later update is skipped too, and the
        caller raises when it reads the flag (TomographyIteration)."""
        _require(params, "params", torch.float32)
        _require(grads, "grads", torch.float32)
        if params.shape != grads.shape:
            raise InvalidParameterError("parameter/gradient shape mismatch")
        if self.m is None:
            self.m = torch.zeros_like(params)
            self.v = torch.zeros_like(params)
            self.flag = torch.zeros(1, dtype=torch.int32, device=params.device)
        inf = float("inf")
        if project == "volume":
            cfg = (1, 0.0, 1.0, 0.0, 1.0)
        elif project == "tf":
            cfg = (4, 0.0, float(tau_max), 0.0, inf)
        elif project is None:
            cfg = (1, -inf, inf, -inf, inf)
        else:
            raise InvalidParameterError(f"unknown projection target {project!r}")
        a = N.DdvrAdam(self.lr, self.beta1, self.beta2, self.eps, self.step + 1, *cfg)
        defer = check_finite == "defer"
        if check_finite and not defer:
            self.flag.zero_()
        if self.device_step:
            if self.state is None:
                self.state = torch.zeros(4, dtype=torch.int32, device=params.device)
                self.state[0] = self.step
            N.check(N.lib().ddvr_adam_step_device(
                params.data_ptr(), grads.data_ptr(), self.m.data_ptr(), self.v.data_ptr(),
                params.numel(), ctypes.byref(a), self.state.data_ptr(),
                self.flag.data_ptr() if check_finite else None, _stream_ptr()))
            return
        N.check(N.lib().ddvr_adam_step(params.data_ptr(), grads.data_ptr(), self.m.data_ptr(),
                                       self.v.data_ptr(), params.numel(), ctypes.byref(a),
                                       self.flag.data_ptr() if check_finite else None,
                                       _stream_ptr()))
        if check_finite and not defer and int(self.flag.item()):
            raise NumericalAbortError("non-finite gradients passed to the optimizer")
        self.step += 1


def upsample_volume(values: torch.Tensor) -> torch.Tensor:
    """(2X, 2Y, 2Z) linear upsampling with edge extrapolation (optim.py:92-129)."""
    _require(values, "volume", torch.float32, ndim=3)
    out = torch.empty(tuple(2 * d for d in values.shape), dtype=torch.float32,
                      device=values.device)
    N.check(N.lib().ddvr_upsample_volume(values.data_ptr(), _dims(values), out.data_ptr(),
                                         _stream_ptr()))
    return out
