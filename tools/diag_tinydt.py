"""Diagnostic: tiny-dt camera gradient, inversion vs stored tape vs fp64 oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import dvr_oracle as O
from paper_2107_12672_b200 import raymarch as R
rng = np.random.default_rng(5)
vol = rng.uniform(0.05, 0.95, (8, 8, 8)).astype(np.float32)
tex = rng.uniform(0.05, 1.0, (8, 4)).astype(np.float32)
W, H, radius = 9, 7, 2.2
for dt in (0.04, 2e-3, 5e-4, 2.5e-4):
    view = O.View(33.0, 21.0, radius, fov_y_deg=35.0, width=W, height=H)
    seed = rng.normal(size=(H, W, 4))
    g = O.Grid(vol.astype(np.float64))
    img_o = O.render_view(g, tex.astype(np.float64), view, dt)
    ref = O.adjoint_view(g, tex.astype(np.float64), view, dt, seed, ["camera", "stepsize"], image=img_o)
    dev = torch.device("cuda")
    dens = torch.from_numpy(vol).to(dev); tx = torch.from_numpy(tex).to(dev)
    cams = R.camera_array(torch.tensor([[33.0, 21.0]], dtype=torch.float64, device=dev), radius, (0.0, 0.0, 0.0), 35.0)
    rig = R.Rig(W, H)
    _, n, _ = R.ray_setup(cams, dt, rig)
    stride = int(n.max().item())
    tape = torch.empty(W * H * stride, device=dev)
    img, trans = R.forward(dens, tx, cams, dt, rig, tape=tape, tape_stride=stride)
    s = torch.from_numpy(seed.astype(np.float32)).to(dev)[None].contiguous()
    for mode in ("inversion", "stored"):
        dc = torch.zeros(1, 2, dtype=torch.float64, device=dev); dd = torch.zeros(1, dtype=torch.float64, device=dev)
        kw = dict(tape=tape, tape_stride=stride) if mode == "stored" else {}
        R.adjoint(dens, tx, cams, dt, rig, img, trans, s, 3, d_camera=dc, d_dt=dd, **kw)
        c = dc.cpu().numpy()[0]
        print(f"dt={dt:g} n_max={stride} {mode:9s} cam={c} ref={ref['d_camera']} rel={np.linalg.norm(c-ref['d_camera'])/np.linalg.norm(ref['d_camera']):.2e} "
              f"dt_rel={abs(dd.item()-ref['d_stepsize'])/abs(ref['d_stepsize']):.2e}")
