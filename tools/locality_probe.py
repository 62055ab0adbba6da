"""Does the march pay for L2 misses?  Time forward + volume adjoint per sample
for C4-like scenes whose cell records fit L2 (128^3: 69 MB) or not (256^3:
543 MB, 192^3: 229 MB), same image and dt in voxels.  Prints G samples/s.

    python tools/locality_probe.py        # GPU
"""
import dataclasses
import sys

import torch

sys.path.insert(0, ".")
from paper_2107_12672_b200 import raymarch as R                     # noqa: E402
from paper_2107_12672_b200.scenes import CONFIGS, phantom            # noqa: E402

dev = torch.device("cuda")
base = CONFIGS["C4"]
for n in (128, 192, 256, 320):
    cfg = dataclasses.replace(base, vol_dim=n)
    vol = torch.from_numpy(phantom("sphere", n, seed=0).astype("float32")).to(dev)
    tex = torch.from_numpy(cfg.texels().astype("float32")).to(dev)
    poses = cfg.view_poses()[:16]
    ll = torch.tensor(poses, dtype=torch.float64, device=dev)
    cams = R.camera_array(ll, cfg.radius, (0.0, 0.0, 0.0), cfg.fov)
    dt = cfg.dt
    rig = R.Rig(512, 512)
    cells = R.pack_cells(vol)
    _, n_steps, _ = R.ray_setup(cams, dt, rig, dims=(n, n, n))
    samples = int(n_steps.to(torch.int64).sum())
    img, depth = R.forward(vol, tex, cams, dt, rig, cells=cells)
    seed = torch.randn_like(img)
    ws = R.workspace_for(vol, 8, cells)
    d = torch.zeros_like(vol)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for it in range(3):
        ev[0].record()
        img, depth = R.forward(vol, tex, cams, dt, rig, cells=cells)
        ev[1].record()
        R.adjoint(vol, tex, cams, dt, rig, img, depth, seed, 8, d_volume=d, cells=cells,
                  workspace=ws)
        ev[2].record()
        torch.cuda.synchronize()
    f, a = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    print(f"{n}^3 cells {cells.numel() * 4 / 2**20:7.0f} MiB  samples {samples / 1e9:.2f} G  "
          f"fwd {samples / f / 1e6:6.1f} G/s  adj {samples / a / 1e6:6.1f} G/s")
