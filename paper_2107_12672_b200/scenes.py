"""Synthetic inputs of the benchmark configurations.

Host-side NumPy generators for the density volumes, transfer-function texel
tables and camera poses the reference uses for its pipelines.  They restate:

* phantoms   ``voldiff/phantoms.py:13-72`` (sphere, shells, blobs, asymmetric),
* TF presets ``voldiff/tasks.py:348-388`` (grayscale, warm, gaussian,
  absorption; and the absorption ramp of ``make_absorption_ramp_tf``),
* views      ``voldiff/tasks.py:118-128`` (golden-angle Fibonacci spiral).

These only build inputs; nothing here is on the GPU hot path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_LAT_LIMIT = 90.0 - 1e-3 - 0.1                      # tasks.py:50
_GOLDEN_ANGLE_DEG = 137.50776405003785               # tasks.py:49


def _node_grid(dims, box_min, box_max):
    axes = [box_min[a] + (np.arange(dims[a]) + 0.5) * (box_max[a] - box_min[a]) / dims[a]
            for a in range(3)]
    return np.meshgrid(*axes, indexing="ij")


def _smoothstep(t):
    t = np.clip(t, 0.0, 1.0)
    return t * t * (3.0 - 2.0 * t)


def phantom(kind: str, dims, seed: int = 0, box_min=(-0.5, -0.5, -0.5),
            box_max=(0.5, 0.5, 0.5)) -> np.ndarray:
    """Density grid (X,Y,Z) float64 in [0,1] (phantoms.py:26-72)."""
    if isinstance(dims, int):
        dims = (dims, dims, dims)
    box_min = np.asarray(box_min, np.float64)
    box_max = np.asarray(box_max, np.float64)
    x, y, z = _node_grid(dims, box_min, box_max)
    c = 0.5 * (box_min + box_max)
    half = float(np.min(0.5 * (box_max - box_min)))
    r = np.sqrt((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2)
    if kind == "sphere":
        r0, r1 = 0.45 * half, 0.85 * half
        d = 1.0 - _smoothstep((r - r0) / (r1 - r0))
    elif kind == "shells":
        d = (0.85 * np.exp(-(((r - 0.32 * half) / (0.11 * half)) ** 2))
             + 0.45 * np.exp(-(((r - 0.70 * half) / (0.11 * half)) ** 2)))
    elif kind in ("blobs", "asymmetric"):
        rng = np.random.default_rng(seed)
        d = np.zeros(dims)
        for _ in range(6):
            p = c + rng.uniform(-0.55, 0.55, 3) * half
            s = rng.uniform(0.16, 0.38) * half
            amp = rng.uniform(0.4, 1.0)
            d += amp * np.exp(-(((x - p[0]) ** 2 + (y - p[1]) ** 2 + (z - p[2]) ** 2)
                                / (2 * s * s)))
        if kind == "asymmetric":
            p = c + np.array([0.62, 0.18, -0.10]) * half
            s = 0.14 * half
            d += 1.2 * np.exp(-(((x - p[0]) ** 2 + (y - p[1]) ** 2 + (z - p[2]) ** 2)
                                / (2 * s * s)))
    else:
        raise ValueError(f"unknown phantom kind {kind!r}")
    return np.clip(d, 0.0, 1.0)


def preset_texels(name: str, resolution: int = 16, tau_scale: float = 4.0) -> np.ndarray:
    """(R,4) texel table of a stock TF (tasks.py:359-388)."""
    d = (np.arange(resolution) + 0.5) / resolution
    t = np.zeros((resolution, 4))
    if name == "grayscale":
        t[:, 0] = t[:, 1] = t[:, 2] = d
        t[:, 3] = tau_scale * d
    elif name == "warm":
        t[:, 0] = d
        t[:, 1] = 0.3 + 0.2 * d
        t[:, 2] = 1.0 - d
        t[:, 3] = tau_scale * d
    elif name == "gaussian":
        bump = np.exp(-(((d - 0.5) / 0.09) ** 2))
        t[:, 0] = 0.9 * bump
        t[:, 1] = 0.6 * bump
        t[:, 2] = 0.2 * bump
        t[:, 3] = tau_scale * bump
    elif name == "absorption":
        t[:, 3] = tau_scale * d
    else:
        raise ValueError(f"unknown transfer-function preset {name!r}")
    return t


def absorption_ramp_texels(resolution: int = 64, tau_scale: float = 3.0) -> np.ndarray:
    """Emission-free ramp with an exactly-zero first texel (tasks.py:348-356)."""
    t = np.zeros((resolution, 4))
    t[:, 3] = tau_scale * np.arange(resolution) / max(resolution - 1, 1)
    return t


def fibonacci_poses(count: int):
    """(lon, lat) degrees of ``count`` golden-angle views (tasks.py:118-128)."""
    poses = []
    for k in range(count):
        zk = 1.0 - 2.0 * (k + 0.5) / count
        lat = math.degrees(math.asin(max(-1.0, min(1.0, zk))))
        lat = max(-_LAT_LIMIT, min(_LAT_LIMIT, lat))
        poses.append(((k * _GOLDEN_ANGLE_DEG) % 360.0, lat))
    return poses


@dataclass
class BenchConfig:
    """One row of SURVEY.md section 8's configuration table."""

    name: str
    title: str
    vol_dim: int
    phantom: str
    image: int
    views: int
    dt_vox: float                  # stepsize in voxels of the volume
    tf: tuple                      # ("preset", name, R, tau) | ("ramp", R, tau)
    targets: tuple
    radius: float = 2.0
    fov: float = 30.0
    poses: list = field(default_factory=list)

    @property
    def dt(self) -> float:
        return self.dt_vox / self.vol_dim

    def texels(self) -> np.ndarray:
        if self.tf[0] == "ramp":
            return absorption_ramp_texels(self.tf[1], self.tf[2])
        return preset_texels(self.tf[1], self.tf[2], self.tf[3])

    def volume(self) -> np.ndarray:
        """fp32-representable density (float32 array)."""
        return phantom(self.phantom, self.vol_dim, seed=0).astype(np.float32)

    def view_poses(self):
        if self.views == 1:
            return [(30.0, 20.0)]          # SphericalCamera(30, 20, 2.0), cli.py:101-104
        return fibonacci_poses(self.views)


CONFIGS = {
    "C1": BenchConfig("C1", "synthetic 64^3, 128x128, 1 view, PL(texel) TF, density+TF grads",
                      64, "blobs", 128, 1, 1.0, ("preset", "warm", 64, 8.0), ("volume", "tf")),
    "C2": BenchConfig("C2", "TF reconstruction: 128^3, 256x256, 8 views, texture TF, TF grads",
                      128, "shells", 256, 8, 1.0, ("preset", "warm", 64, 4.0), ("tf",)),
    "C3": BenchConfig("C3", "viewpoint: 256^3, 512x512, 1 view, camera+stepsize grads",
                      256, "asymmetric", 512, 1, 0.5, ("preset", "grayscale", 64, 4.0),
                      ("camera", "stepsize")),
    "C4": BenchConfig("C4", "absorption tomography: 256^3, 64 views at 512x512, density grads",
                      256, "sphere", 512, 64, 0.2, ("ramp", 64, 3.0), ("volume",)),
    "C5": BenchConfig("C5", "EA tomography: 512^3, 128 views at 1024x1024, Gaussian TF, "
                            "density grads", 512, "shells", 1024, 128, 0.2,
                      ("preset", "gaussian", 64, 6.0), ("volume",)),
}
