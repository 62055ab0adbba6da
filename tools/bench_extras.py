"""Measurements for the SURVEY 8f rows around the hot path (one B200).

    python tools/bench_extras.py > profiles/r01_extras.json

Each entry: the operation, its work unit, the median CUDA-event time over 5 runs
(after 2 warm-ups, L2 flushed before each run) and the rate:
- forward-mode camera Jacobian (render_forward_grad) at C3 (1 view 512^2, 256^3);
- pre-shaded colour volume forward + adjoint (render_colorvol(_adjoint)) on a
  256^3 RGBA volume, 16 views at 512^2, dt 0.2 voxel;
- the raw x-fastest -> z-fastest device import (load_volume_device's kernel) and
  the reverse, 512^3 f32, in GB/s against the HBM peak;
- opacity_entropy and the PPM quantiser over 64 images of 512^2, GB/s.
"""
import json
import os
import sys
import ctypes

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2107_12672_b200 import _native as N                     # noqa: E402
from paper_2107_12672_b200 import fileio as F                       # noqa: E402
from paper_2107_12672_b200 import raymarch as R                     # noqa: E402
from paper_2107_12672_b200.scenes import CONFIGS, fibonacci_poses, phantom  # noqa: E402

dev = torch.device("cuda")
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6548.2) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6548.2


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ms = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.median(ms))


def samples_of(cams, dt, rig, dims):
    _, n, _ = R.ray_setup(cams, dt, rig, dims=dims)
    return int(n.to(torch.int64).sum())


out = {}

# forward-mode camera Jacobian at C3
c3 = CONFIGS["C3"]
vol = torch.from_numpy(c3.volume()).to(dev)
tex = torch.from_numpy(c3.texels().astype(np.float32)).to(dev)
cams = R.camera_array(torch.tensor(c3.view_poses(), dtype=torch.float64, device=dev), c3.radius,
                      (0.0, 0.0, 0.0), c3.fov)
rig = R.Rig(c3.image, c3.image)
cells = R.pack_cells(vol)
ns = samples_of(cams, c3.dt, rig, tuple(vol.shape))
ms = timed(lambda: R.forward_grad(vol, tex, cams, c3.dt, rig, "camera", cells=cells))
out["forward_grad_camera_C3"] = {"unit": "samples/s", "samples": ns, "ms": ms,
                                 "rate": ns / (ms / 1e3)}

# colour volume forward + adjoint, 256^3 RGBA, 16 views
n = 256
dens = phantom("sphere", n, seed=0).astype(np.float32)
rng = np.random.default_rng(0)
rgba = np.concatenate([rng.uniform(0, 1, (n, n, n, 3)).astype(np.float32) * dens[..., None],
                       3.0 * dens[..., None]], axis=3)
col = torch.from_numpy(np.ascontiguousarray(rgba)).to(dev)
poses = fibonacci_poses(16)
ccams = R.camera_array(torch.tensor(poses, dtype=torch.float64, device=dev), 2.0,
                       (0.0, 0.0, 0.0), 30.0)
crig = R.Rig(512, 512)
dt = 0.2 / n
ns = samples_of(ccams, dt, crig, (n, n, n))
img, depth = R.forward_color(col, ccams, dt, crig)
seed = torch.randn_like(img)
dcol = torch.zeros_like(col)
ms_f = timed(lambda: R.forward_color(col, ccams, dt, crig))
ms_a = timed(lambda: R.adjoint_color(col, ccams, dt, crig, img, depth, seed, dcol))
out["colour_volume_256_16views"] = {
    "unit": "samples/s", "samples": ns, "forward_ms": ms_f, "adjoint_ms": ms_a,
    "forward_rate": ns / (ms_f / 1e3), "adjoint_rate": ns / (ms_a / 1e3),
    "bytes_model": "128 B/sample (8 float4 corners) forward; + 128 B scattered adjoint"}

# raw volume import / export, 512^3 f32
dims = (512, 512, 512)
raw = torch.rand(int(np.prod(dims)), device=dev)
dst = torch.empty(dims, device=dev)
d3 = (ctypes.c_int32 * 3)(*dims)
st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
rng2 = (ctypes.c_double * 2)(0.0, 2.0)
ms_i = timed(lambda: N.check(N.lib().ddvr_volume_from_raw(raw.data_ptr(), d3, rng2,
                                                          dst.data_ptr(), st())))
ms_o = timed(lambda: N.check(N.lib().ddvr_volume_to_raw(dst.data_ptr(), d3, raw.data_ptr(),
                                                        st())))
nbytes = 2 * 4 * raw.numel()
out["volume_import_512"] = {"unit": "GB/s", "bytes": nbytes, "ms": ms_i,
                            "rate": nbytes / (ms_i / 1e3) / 1e9,
                            "frac_of_hbm": nbytes / (ms_i / 1e3) / 1e9 / peak}
out["volume_export_512"] = {"unit": "GB/s", "bytes": nbytes, "ms": ms_o,
                            "rate": nbytes / (ms_o / 1e3) / 1e9,
                            "frac_of_hbm": nbytes / (ms_o / 1e3) / 1e9 / peak}

# opacity entropy and PPM quantisation over 64 x 512^2 images
imgs = torch.rand(64, 512, 512, 4, device=dev)
ms_e = timed(lambda: R.opacity_entropy(imgs))
eb = 2 * imgs.numel() * 4            # read images twice (sums, seed) + write the seed
out["opacity_entropy_64x512"] = {"unit": "GB/s", "bytes": eb + imgs.numel() * 4, "ms": ms_e,
                                 "rate": (eb + imgs.numel() * 4) / (ms_e / 1e3) / 1e9}
ppm = torch.empty(64 * 512 * 512 * 3, dtype=torch.uint8, device=dev)
ms_p = timed(lambda: N.check(N.lib().ddvr_image_to_ppm(imgs.data_ptr(), 64 * 512 * 512,
                                                       ppm.data_ptr(), st())))
pb = imgs.numel() * 4 + ppm.numel()
out["ppm_64x512"] = {"unit": "GB/s", "bytes": pb, "ms": ms_p, "rate": pb / (ms_p / 1e3) / 1e9,
                     "frac_of_hbm": pb / (ms_p / 1e3) / 1e9 / peak}
print(json.dumps(out, indent=1))
