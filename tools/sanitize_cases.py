"""Small GPU cases for compute-sanitizer (race / memory checking).

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py

Runs every libddvr kernel family once on small inputs: the C1 step (fused forward +
L1 + adjoint, volume + TF targets, then prior + Adam + projection), the C2-shaped TF-target
step, the C3-shaped camera / stepsize adjoint (separate forward and adjoint), a C4-shaped
absorption step with the band tape, the empty-brick skip and the split march / walk kernels
on a volume with exact empty space, a Gaussian-TF (C5-shaped) emitting step, the stored
(tape) mode, both volume layouts through autograd, forward-mode Jacobians, colour volumes
and the entropy objective.  Prints
"SANITIZE_CASES_OK" at the end.  ``--config-band``: also the C4 step at full size (8 rows).

With the bounds-checked library (DDVR_LIB=.../libddvr_checked.so, built with
-DDDVR_CHECKED) every record gather, cell-gradient flush and brick lookup is checked
against the padded record grid (tests/test_gpu_checked.py).
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2107_12672_b200 import raymarch as R  # noqa: E402
from paper_2107_12672_b200.distributed import ShardedStep, TomographyIteration  # noqa: E402
from paper_2107_12672_b200.scenes import (absorption_ramp_texels, fibonacci_poses,  # noqa: E402
                                          phantom, preset_texels)


def dev_t(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def step_case(n, img, views, tex, targets, dt_vox=0.5, kind="blobs", sparse=False, **kw):
    truth = phantom(kind, n, seed=0).astype(np.float32)
    est = np.clip(0.8 * truth + 0.05, 0, 1).astype(np.float32)
    if sparse:
        est = np.where(truth > 0, est, 0.0).astype(np.float32)
    ll = torch.tensor(fibonacci_poses(views) if views > 1 else [(30.0, 20.0)],
                      dtype=torch.float64, device="cuda")
    rig = R.Rig(img, img)
    dt = dt_vox / n
    tx = dev_t(tex)
    cams = R.camera_array(ll, 2.0, (0.0, 0.0, 0.0), 30.0)
    refs, _ = R.forward(dev_t(truth), tx, cams, dt, rig)
    e = dev_t(est)
    step = ShardedStep(e, tx, ll, refs, dt, rig, targets=targets, **kw)
    if "volume" in targets:
        it = TomographyIteration(step, lr=0.02, lam=0.5)
        for _ in range(2):
            it.run()
        it.check()
    else:
        step.run()
    torch.cuda.synchronize()
    return step


def main():
    torch.cuda.init()
    # C1-shaped: volume + TF targets, fused step, Adam
    step_case(24, 24, 1, preset_texels("warm", 16, 8.0), ("volume", "tf"), dt_vox=1.0)
    # C2-shaped: TF target only, several views
    step_case(24, 20, 3, preset_texels("warm", 16, 4.0), ("tf",), dt_vox=1.0, kind="shells")
    # C3-shaped: camera + stepsize (separate forward and adjoint)
    step_case(24, 20, 1, preset_texels("grayscale", 16, 4.0), ("camera", "stepsize"))
    step_case(24, 20, 1, preset_texels("grayscale", 16, 4.0), ("camera", "stepsize"),
              deterministic=True)
    # C4-shaped: absorption ramp, band tape, empty-brick skip (exact zeros), split kernels
    ramp = absorption_ramp_texels(32, 3.0)
    for split in (False, True):
        s = step_case(40, 24, 3, ramp, ("volume",), dt_vox=0.2, kind="sphere", sparse=True,
                      split_walk=split)
        assert s.band_tape
    step_case(40, 24, 3, ramp, ("volume",), dt_vox=0.2, kind="sphere", band_tape=False)
    # C5-shaped: Gaussian texel TF (emitting), volume target
    step_case(24, 20, 2, preset_texels("gaussian", 16, 6.0), ("volume",), dt_vox=0.2,
              kind="shells")
    # stored (tape) mode, forward-mode Jacobian, voxel layout, through the autograd path
    vol = dev_t(phantom("blobs", 16, seed=1)).requires_grad_(True)
    tx = dev_t(preset_texels("warm", 8, 6.0)).requires_grad_(True)
    ll = torch.tensor([[30.0, 20.0], [75.0, -10.0]], dtype=torch.float64, device="cuda",
                      requires_grad=True)
    dtt = torch.tensor(1.0 / 16, dtype=torch.float64, requires_grad=True)
    for layout in ("cells", "voxels"):
        img = R.render_views(vol, tx, ll, dtt, R.Rig(12, 10), layout=layout)
        img.square().sum().backward()
    cams = R.camera_array(ll.detach(), 2.0, (0.0, 0.0, 0.0), 30.0)
    rig = R.Rig(12, 10)
    _, n, _ = R.ray_setup(cams, 1.0 / 16, rig)
    stride = int(n.max())
    tape = torch.zeros(2 * 12 * 10 * stride, dtype=torch.float32, device="cuda")
    img, depth = R.forward(vol.detach(), tx.detach(), cams, 1.0 / 16, rig, tape=tape,
                           tape_stride=stride)
    seed = torch.randn_like(img)
    dv = torch.zeros_like(vol)
    R.adjoint(vol.detach(), tx.detach(), cams, 1.0 / 16, rig, img, depth, seed, 8, d_volume=dv,
              cells=R.pack_cells(vol.detach()), tape=tape, tape_stride=stride)
    for wrt in ("camera", "stepsize"):
        R.forward_grad(vol.detach(), tx.detach(), cams, 1.0 / 16, rig, wrt)
    # colour volume (X,Y,Z,4) forward + adjoint, entropy objective
    color = torch.rand(12, 12, 12, 4, device="cuda")
    cimg, cdepth = R.forward_color(color, cams, 1.0 / 12, rig)
    dcol = torch.zeros_like(color)
    R.adjoint_color(color, cams, 1.0 / 12, rig, cimg, cdepth, torch.randn_like(cimg), dcol)
    R.opacity_entropy(cimg)
    if "--config-band" in sys.argv:   # the full-size C4 geometry (256^3, 512^2) on 8 rows
        from paper_2107_12672_b200.scenes import CONFIGS
        c = CONFIGS["C4"]
        truth = c.volume()
        est = np.where(truth > 0, np.clip(0.7 * truth + 0.05, 0, 1), 0.0).astype(np.float32)
        ll = torch.tensor(c.view_poses()[:3], dtype=torch.float64, device="cuda")
        rig = R.Rig(c.image, c.image, rows=(252, 260))
        tx = dev_t(c.texels())
        cams = R.camera_array(ll, c.radius, (0.0, 0.0, 0.0), c.fov)
        refs, _ = R.forward(dev_t(truth), tx, cams, c.dt, rig)
        for split in (False, True):
            ShardedStep(dev_t(est), tx, ll, refs, c.dt, rig, split_walk=split).run()
    torch.cuda.synchronize()
    print("SANITIZE_CASES_OK")


if __name__ == "__main__":
    main()
