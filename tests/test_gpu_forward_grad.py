"""Forward-mode Jacobians (render_forward_grad, renderer.py:410-464) vs the reference.

tests/golden/forward_grad.npz holds voldiff's own per-pixel Jacobians for the
camera (p=2) and stepsize (p=1) targets on random gradcheck scenes, plus the
stepsize closed-form scene (test_renderer.py:166-175).  Also checks the
forward/adjoint consistency the reference asserts (test_renderer.py:231-238):
sum(seed * J) equals the adjoint gradient for the same seed.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu
SCENES = (500, 501, 502, 2001)


def _scene(g, s, dev):
    import torch
    from paper_2107_12672_b200 import raymarch as R
    lon, lat, radius, cx, cy, cz, fov, W, H = g[f"s{s}_cam"]
    dens = torch.from_numpy(g[f"s{s}_volume"]).to(dev)
    tex = torch.from_numpy(g[f"s{s}_texels"]).to(dev)
    cams = R.camera_array(torch.tensor([[lon, lat]], dtype=torch.float64, device=dev), radius,
                          (cx, cy, cz), fov)
    return dens, tex, cams, R.Rig(int(W), int(H)), float(g[f"s{s}_dt"])


@pytest.mark.parametrize("s", SCENES)
@pytest.mark.parametrize("wrt", ["camera", "stepsize"])
@pytest.mark.parametrize("layout", ["cells", "voxels"])
def test_forward_grad_matches_reference(cuda, s, wrt, layout):
    import torch
    from paper_2107_12672_b200 import raymarch as R
    g = golden("forward_grad")
    dens, tex, cams, rig, dt = _scene(g, s, cuda)
    cells = R.pack_cells(dens) if layout == "cells" else None
    img, jac = R.forward_grad(dens, tex, cams, dt, rig, wrt, cells=cells)
    assert rel_l2(img[0].double().cpu().numpy(), g[f"s{s}_{wrt}_image"]) <= 1e-5
    assert rel_l2(jac[0].double().cpu().numpy(), g[f"s{s}_{wrt}_jac"]) <= 1e-4
    # forward mode == adjoint (test_renderer.py:231-238): sum(seed * J) vs the adjoint
    seed = torch.randn(img.shape, device=cuda, generator=torch.Generator(device=cuda).manual_seed(s))
    img2, depth = R.forward(dens, tex, cams, dt, rig, cells=cells)
    if wrt == "camera":
        d = torch.zeros(1, 2, dtype=torch.float64, device=cuda)
        R.adjoint(dens, tex, cams, dt, rig, img2, depth, seed, 1, d_camera=d, cells=cells)
    else:
        d = torch.zeros(1, dtype=torch.float64, device=cuda)
        R.adjoint(dens, tex, cams, dt, rig, img2, depth, seed, 2, d_dt=d, cells=cells)
    fwd = (seed.double()[..., None] * jac.double()).sum(dim=(0, 1, 2, 3))
    assert rel_l2(fwd.cpu().numpy(), d.reshape(-1).cpu().numpy()) <= 1e-4


def test_stepsize_closed_form(cuda):
    """d alpha / d dt = tau0 n exp(-tau0 n dt) at the centre pixel (test_renderer.py:166-175)."""
    import torch
    from paper_2107_12672_b200 import raymarch as R
    dens = torch.ones(8, 8, 8, device=cuda)
    tex = torch.tensor(np.tile([0.4, 0.4, 0.4, 1.3], (2, 1)), dtype=torch.float32, device=cuda)
    cams = R.camera_array(torch.tensor([[0.0, 0.0]], dtype=torch.float64, device=cuda), 2.0,
                          (0.0, 0.0, 0.0), 8.0)
    _, jac = R.forward_grad(dens, tex, cams, 0.05, R.Rig(9, 9), "stepsize",
                            cells=R.pack_cells(dens))
    tau0, n, dt = float(np.float32(1.3)), 20, 0.05
    expected = tau0 * n * np.exp(-tau0 * n * dt)
    got = float(jac[0, 4, 4, 3, 0])
    assert abs(got - expected) / expected < 1e-5
    g = golden("forward_grad")
    assert rel_l2(jac[0].double().cpu().numpy(), g["kat_stepsize_jac"]) <= 1e-5


def test_dropin_render_forward_grad(cuda):
    import paper_2107_12672_b200 as vd
    g = golden("forward_grad")
    s = 501
    lon, lat, radius, cx, cy, cz, fov, W, H = g[f"s{s}_cam"]
    vol = vd.DensityVolume(g[f"s{s}_volume"].astype(np.float64))
    tf = vd.TransferFunction(g[f"s{s}_texels"].astype(np.float64))
    cam = vd.SphericalCamera(lon, lat, radius, (cx, cy, cz), fov, int(W), int(H))
    img, jac = vd.render_forward_grad(vol, tf, cam, vd.RenderConfig(dt=float(g[f"s{s}_dt"]),
                                                                    target="camera"))
    assert jac.shape == (int(H), int(W), 4, 2) and jac.dtype == np.float64
    assert rel_l2(jac, g[f"s{s}_camera_jac"]) <= 1e-4
    with pytest.raises(vd.UnsupportedConfigurationError):
        vd.render_forward_grad(vol, tf, cam, vd.RenderConfig(dt=0.1, target="tf"))
