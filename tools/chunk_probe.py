"""Would running each ray's adjoint right after its forward help?  Proxy:
forward+adjoint over 64 C4 views batched (one launch each) vs in chunks of
k views (fwd(chunk) -> adj(chunk)), so a chunk's cells are still in L2.

    python tools/chunk_probe.py        # GPU
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2107_12672_b200 import raymarch as R                     # noqa: E402
from paper_2107_12672_b200.scenes import CONFIGS                     # noqa: E402

dev = torch.device("cuda")
cfg = CONFIGS["C4"]
vol = torch.from_numpy(cfg.volume()).to(dev)
tex = torch.from_numpy(cfg.texels().astype("float32")).to(dev)
ll = torch.tensor(cfg.view_poses(), dtype=torch.float64, device=dev)
cams = R.camera_array(ll, cfg.radius, (0.0, 0.0, 0.0), cfg.fov)
rig = R.Rig(512, 512)
cells = R.pack_cells(vol)
ws = R.workspace_for(vol, 8, cells)
d = torch.zeros_like(vol)
img, depth = R.forward(vol, tex, cams, cfg.dt, rig, cells=cells)
seed = torch.randn_like(img)
for k in (64, 16, 8, 4, 2):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for it in range(3):
        ev[0].record()
        for c in range(0, 64, k):
            sl = slice(c, c + k)
            im, de = R.forward(vol, tex, cams[sl], cfg.dt, rig, cells=cells)
            R.adjoint(vol, tex, cams[sl], cfg.dt, rig, im, de, seed[sl].contiguous(), 8,
                      d_volume=d, cells=cells, workspace=ws)
        ev[1].record()
        torch.cuda.synchronize()
    print(f"chunk {k:3d} views: fwd+adj {ev[0].elapsed_time(ev[1]):7.2f} ms")
