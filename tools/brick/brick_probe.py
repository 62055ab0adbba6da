"""Experiment: gather-only probe over z-linear vs 2x2x2-bricked cell records (C4 rays).

    python tools/brick/brick_probe.py       # GPU; builds tools/brick/libbrick.so first
"""
import ctypes
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from paper_2107_12672_b200 import _native as N           # noqa: E402
from paper_2107_12672_b200 import raymarch as R          # noqa: E402
from paper_2107_12672_b200.scenes import CONFIGS         # noqa: E402

so = os.path.join(HERE, "libbrick.so")
subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
                "-I", os.path.join(ROOT, "paper_2107_12672_b200", "csrc"), "-o", so,
                os.path.join(HERE, "brick_probe.cu")], check=True)
lib = ctypes.CDLL(so)
dev = torch.device("cuda")
cfg = CONFIGS["C4"]
vol = torch.from_numpy(cfg.volume()).to(dev)
ll = torch.tensor(cfg.view_poses(), dtype=torch.float64, device=dev)
cams = R.camera_array(ll, cfg.radius, (0.0, 0.0, 0.0), cfg.fov)
rig = R.Rig(512, 512)
cells = R.pack_cells(vol)
X, Y, Z = vol.shape
nb = ((X + 2) // 2) * ((Y + 2) // 2) * ((Z + 2) // 2) * 8 * 8
bricks = torch.zeros(nb, dtype=torch.float32, device=dev)
out = torch.empty(64, 512, 512, dtype=torch.float32, device=dev)
tx = torch.zeros(1, 4, device=dev)
v, _, prm = R._descs(vol, tx, rig, cfg.dt, False, cells)
st = torch.cuda.current_stream().cuda_stream
lib.brick_run(ctypes.byref(v), ctypes.c_void_p(cams.data_ptr()), 64, ctypes.byref(prm), 1,
              ctypes.c_void_p(cells.data_ptr()), ctypes.c_void_p(bricks.data_ptr()),
              ctypes.c_void_p(out.data_ptr()), 1, ctypes.c_void_p(st))
ref = None
for mode in (0, 1, 0, 1):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    lib.brick_run(ctypes.byref(v), ctypes.c_void_p(cams.data_ptr()), 64, ctypes.byref(prm), mode,
                  ctypes.c_void_p(cells.data_ptr()), ctypes.c_void_p(bricks.data_ptr()),
                  ctypes.c_void_p(out.data_ptr()), 0, ctypes.c_void_p(st))
    b.record()
    torch.cuda.synchronize()
    s = float(out.double().sum())
    ref = ref if ref is not None else s
    print(f"{'bricked' if mode else 'linear '} {a.elapsed_time(b):7.2f} ms  checksum {s:.6e} "
          f"({'same' if abs(s - ref) <= 1e-6 * abs(ref) else 'DIFFERENT'})")

ctr = torch.zeros(148, dtype=torch.int32, device=dev)
for cps in (6, 12, 6, 12):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    lib.sm_run(ctypes.byref(v), ctypes.c_void_p(cams.data_ptr()), 64, ctypes.byref(prm),
               ctypes.c_void_p(cells.data_ptr()), ctypes.c_void_p(ctr.data_ptr()),
               ctypes.c_void_p(out.data_ptr()), cps, ctypes.c_void_p(st))
    b.record()
    torch.cuda.synchronize()
    s = float(out.double().sum())
    print(f"sm-local persistent ({cps} CTAs/SM launched) {a.elapsed_time(b):7.2f} ms  checksum {s:.6e} "
          f"({'same' if abs(s - ref) <= 1e-6 * abs(ref) else 'DIFFERENT'})")

stats = torch.zeros(1, dtype=torch.int32, device=dev)
for K in (8, 16, 32, 8, 16, 32):
    stats.zero_()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    lib.staged_run(ctypes.byref(v), ctypes.c_void_p(cams.data_ptr()), 64, ctypes.byref(prm),
                   ctypes.c_void_p(cells.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                   ctypes.c_void_p(stats.data_ptr()), K, ctypes.c_void_p(st))
    b.record()
    torch.cuda.synchronize()
    s = float(out.double().sum())
    print(f"smem-staged K={K:2d} {a.elapsed_time(b):7.2f} ms  fallback windows {int(stats[0])}  "
          f"checksum {s:.6e} ({'same' if abs(s - ref) <= 1e-6 * abs(ref) else 'DIFFERENT'})")
