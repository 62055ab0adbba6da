"""Pre-shaded colour volumes on the GPU vs the reference (tests/golden/color.npz).

render_colorvol / render_colorvol_adjoint (renderer.py:404-407, 703-709):
per-channel trilinear without the [0,1] clamp, negative tau, an off-centre
anisotropic box and a camera inside the box; inversion and stored modes.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu
KEYS = ["a", "b", "c"]


@pytest.mark.parametrize("key", KEYS)
def test_color_tensor_path(cuda, key):
    import torch
    from paper_2107_12672_b200 import raymarch as R
    g = golden("color")
    lon, lat, radius, cx, cy, cz, fov, W, H = g[f"{key}_cam"]
    col = torch.from_numpy(np.ascontiguousarray(g[f"{key}_values"])).to(cuda)
    cams = R.camera_array(torch.tensor([[lon, lat]], dtype=torch.float64, device=cuda), radius,
                          (cx, cy, cz), fov)
    box = g[f"{key}_box"]
    rig = R.Rig(int(W), int(H), tuple(box[0]), tuple(box[1]))
    dt = float(g[f"{key}_dt"])
    img, depth = R.forward_color(col, cams, dt, rig)
    assert rel_l2(img[0].double().cpu().numpy(), g[f"{key}_image"]) <= 1e-5
    img2, _ = R.forward_color(col, cams, dt, rig, early_stop=True)
    assert rel_l2(img2[0].double().cpu().numpy(), g[f"{key}_image_none"]) <= 1e-4
    seed = torch.from_numpy(g[f"{key}_seed"].astype(np.float32)).to(cuda)[None].contiguous()
    d = torch.zeros_like(col)
    R.adjoint_color(col, cams, dt, rig, img, depth, seed, d)
    assert rel_l2(d.double().cpu().numpy(), g[f"{key}_inversion_d_color"]) <= 1e-4


@pytest.mark.parametrize("key", KEYS)
@pytest.mark.parametrize("mode", ["inversion", "stored"])
def test_color_dropin(cuda, key, mode):
    import paper_2107_12672_b200 as vd
    g = golden("color")
    lon, lat, radius, cx, cy, cz, fov, W, H = g[f"{key}_cam"]
    box = g[f"{key}_box"]
    cv = vd.ColorVolume(g[f"{key}_values"].astype(np.float64), box[0], box[1])
    cam = vd.SphericalCamera(lon, lat, radius, (cx, cy, cz), fov, int(W), int(H))
    dt = float(g[f"{key}_dt"])
    img = vd.render_colorvol(cv, cam, vd.RenderConfig(dt=dt, target="volume"))
    assert rel_l2(img.data, g[f"{key}_image"]) <= 1e-5
    cfg = vd.RenderConfig(dt=dt, target="volume", memory_mode=mode)
    gs = vd.render_colorvol_adjoint(cv, cam, cfg, g[f"{key}_seed"], image=img)
    assert gs.d_color.shape == cv.values.shape
    assert rel_l2(gs.d_color, g[f"{key}_{mode}_d_color"]) <= 1e-4
    with pytest.raises(vd.UnsupportedConfigurationError):
        vd.render_colorvol_adjoint(cv, cam, vd.RenderConfig(dt=dt, target="tf"), g[f"{key}_seed"])
