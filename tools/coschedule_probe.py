"""Does running forward and adjoint warps side by side help?  C4 views split in
two halves A, B: sequential fwd(A) fwd(B) adj(A) adj(B) vs fwd(A); {adj(A) on
stream 2 || fwd(B)}; adj(B).  A large gain argues for a fused per-ray
forward -> seed -> adjoint kernel (different bottlenecks share the SMs).

    python tools/coschedule_probe.py        # GPU
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
A, B = slice(0, 32), slice(32, 64)
wsA, wsB = R.workspace_for(vol, 8, cells), R.workspace_for(vol, 8, cells)
dA, dB = torch.zeros_like(vol), torch.zeros_like(vol)
img, depth = R.forward(vol, tex, cams, cfg.dt, rig, cells=cells)
seed = torch.randn_like(img)
s2 = torch.cuda.Stream()


def adj(sl, d, ws):
    R.adjoint(vol, tex, cams[sl], cfg.dt, rig, img[sl], depth[sl], seed[sl].contiguous(), 8,
              d_volume=d, cells=cells, workspace=ws)


def fwd(sl):
    return R.forward(vol, tex, cams[sl], cfg.dt, rig, cells=cells)


for mode in ("sequential", "overlap", "sequential", "overlap"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if mode == "sequential":
        fwd(A); fwd(B); adj(A, dA, wsA); adj(B, dB, wsB)
    else:
        fwd(A)
        ev = torch.cuda.Event(); ev.record()
        s2.wait_event(ev)
        with torch.cuda.stream(s2):
            adj(A, dA, wsA)
        fwd(B)
        torch.cuda.current_stream().wait_stream(s2)
        adj(B, dB, wsB)
    e1.record()
    torch.cuda.synchronize()
    print(f"{mode:10s} {e0.elapsed_time(e1):7.2f} ms")
