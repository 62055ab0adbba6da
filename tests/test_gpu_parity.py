"""CUDA path vs the reference (golden fixtures) and the CPU oracle -- parity proper.

Tolerances (stated by BASELINE.json's north star as "relative L2 per image and
per gradient tensor"):
  * n_steps: bit-exact (integer work);
  * image: rel-L2 <= 1e-5 (fp32 march with fp64 ray setup);
  * every gradient tensor (d_volume, d_tf, d_camera, d_stepsize): rel-L2 <= 1e-4,
    which also covers fp32 atomic-order non-determinism.
All calls go through the C ABI (libddvr.so) via the package's host layer.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, golden_names, rel_l2

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-5
GRAD_TOL = 1e-4
TARGETS = ("tf", "volume", "camera", "stepsize")
BIT = {"camera": 1, "stepsize": 2, "tf": 4, "volume": 8}


def _torch():
    import torch
    return torch


def _setup(g, dev, volume=None, rows=None, layout="cells"):
    torch = _torch()
    from paper_2107_12672_b200 import raymarch as R
    cam = g["cam"]
    lon, lat, radius, cx, cy, cz, fov, W, H = cam
    vol = g["volume"] if volume is None else volume
    dens = torch.from_numpy(np.ascontiguousarray(vol, np.float32)).to(dev)
    tex = torch.from_numpy(np.ascontiguousarray(g["texels"], np.float32)).to(dev)
    ll = torch.tensor([[lon, lat]], dtype=torch.float64, device=dev)
    cams = R.camera_array(ll, radius, (cx, cy, cz), fov)
    box = g.get("box", np.array([[-0.5] * 3, [0.5] * 3]))
    rig = R.Rig(int(W), int(H), tuple(box[0]), tuple(box[1]),
                rows=tuple(int(r) for r in rows) if rows is not None else None)
    cells = R.pack_cells(dens) if layout == "cells" else None
    return dens, tex, cams, rig, float(g["dt"]), cells


def _grads(dens, tex, cams, rig, dt, img, trans, seed, targets, cells=None, tape=None,
           stride=0):
    torch = _torch()
    from paper_2107_12672_b200 import raymarch as R
    dev = dens.device
    mask = 0
    for t in targets:
        mask |= BIT[t]
    out = {
        "volume": torch.zeros_like(dens) if "volume" in targets else None,
        "tf": torch.zeros(tex.shape, dtype=torch.float64, device=dev) if "tf" in targets else None,
        "camera": (torch.zeros(cams.shape[0], 2, dtype=torch.float64, device=dev)
                   if "camera" in targets else None),
        "stepsize": torch.zeros(1, dtype=torch.float64, device=dev) if "stepsize" in targets else None,
    }
    R.adjoint(dens, tex, cams, dt, rig, img, trans, seed, mask, d_volume=out["volume"],
              d_tf=out["tf"], d_camera=out["camera"], d_dt=out["stepsize"], cells=cells,
              tape=tape, tape_stride=stride)
    torch.cuda.synchronize()
    return {k: v.double().cpu().numpy() for k, v in out.items() if v is not None}


SCENES = golden_names("kat_") + golden_names("rand_")


@pytest.mark.parametrize("name", SCENES)
def test_ray_setup_bit_exact(cuda, name):
    from paper_2107_12672_b200 import raymarch as R
    g = golden(name)
    dens, tex, cams, rig, dt, _ = _setup(g, cuda, layout="voxels")
    _, n, _ = R.ray_setup(cams, dt, rig, dims=g["volume"].shape)
    np.testing.assert_array_equal(n[0].cpu().numpy().ravel(), g["n_steps"].ravel())


@pytest.mark.parametrize("name", SCENES)
@pytest.mark.parametrize("layout", ["cells", "voxels"])
def test_image_matches_reference(cuda, name, layout):
    from paper_2107_12672_b200 import raymarch as R
    g = golden(name)
    dens, tex, cams, rig, dt, cells = _setup(g, cuda, layout=layout)
    img, trans = R.forward(dens, tex, cams, dt, rig, cells=cells)
    got = img[0].double().cpu().numpy()
    ref = g["image"]
    if np.linalg.norm(ref) == 0:
        assert np.abs(got).max() == 0.0
    else:
        assert rel_l2(got, ref) <= IMG_TOL
    T = np.exp(-trans[0].double().cpu().numpy())      # forward's optical depth S, T = exp(-S)
    np.testing.assert_allclose(1.0 - T, got[..., 3], atol=2e-6)
    if "image_none" in g:   # early ray termination (renderer.py:331-335)
        img2, _ = R.forward(dens, tex, cams, dt, rig, early_stop=True, cells=cells)
        ref2 = g["image_none"]
        got2 = img2[0].double().cpu().numpy()
        if np.linalg.norm(ref2) == 0:
            assert np.abs(got2).max() == 0.0
        else:
            assert rel_l2(got2, ref2) <= 1e-4


@pytest.mark.parametrize("name", SCENES)
@pytest.mark.parametrize("mode", ["inversion", "stored"])
@pytest.mark.parametrize("layout", ["cells", "voxels"])
def test_gradients_match_reference(cuda, name, mode, layout):
    torch = _torch()
    from paper_2107_12672_b200 import raymarch as R
    g = golden(name)
    keys = [k for k in g if k.startswith(mode + "_") and not k.endswith("state_floats")]
    if not keys:
        pytest.skip(f"no {mode} fixtures for {name}")
    dens, tex, cams, rig, dt, cells = _setup(g, cuda, layout=layout)
    seed = torch.from_numpy(np.asarray(g["seed"], np.float32)).to(cuda)[None].contiguous()
    tape, stride = None, 0
    if mode == "stored":
        H, W = rig.height, rig.width
        _, n, _ = R.ray_setup(cams, dt, rig)
        stride = max(int(n.max().item()), 1)
        tape = torch.full((H * W * stride,), float("nan"), dtype=torch.float32, device=cuda)
    img, trans = R.forward(dens, tex, cams, dt, rig, cells=cells, tape=tape, tape_stride=stride)
    targets = [k.split("_", 1)[1] for k in keys]
    for t in targets:   # one target per call, as the reference
        got = _grads(dens, tex, cams, rig, dt, img, trans, seed, [t], cells=cells, tape=tape,
                     stride=stride)[t]
        ref = np.asarray(g[f"{mode}_{t}"], np.float64).reshape(got.shape)
        if np.linalg.norm(ref) < 1e-300:
            assert np.abs(got).max() <= 1e-7, (t, np.abs(got).max())
        else:
            assert rel_l2(got, ref) <= GRAD_TOL, (t, rel_l2(got, ref))
    if mode == "inversion" and len(targets) > 1:
        # all targets in ONE adjoint launch reproduce each single-target result
        both = _grads(dens, tex, cams, rig, dt, img, trans, seed, targets, cells=cells)
        for t in targets:
            ref = np.asarray(g[f"{mode}_{t}"], np.float64).reshape(both[t].shape)
            if np.linalg.norm(ref) > 1e-300:
                assert rel_l2(both[t], ref) <= GRAD_TOL


CONFIG_CASES = ["C1", "C2", "C3", "C4", "C5"]
# C5's Gaussian texel TF is sharply peaked: fp32-level density rounding alone
# moves the reference's own band gradient by 1.03e-4 rel-L2 (oracle experiment,
# tools/fp32_floor_c5.py); the bar is 2.5x that floor.
BAND_TOL = {("C5", "volume"): 2.5e-4}


@pytest.mark.parametrize("name", CONFIG_CASES)
@pytest.mark.parametrize("layout", ["cells", "voxels"])
def test_config_band_matches_reference(cuda, name, layout):
    """Full C1 view and row bands of view 0 at C2..C5 against the reference."""
    torch = _torch()
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.scenes import CONFIGS
    g = golden(name)
    c = CONFIGS[name]
    vol = c.volume()
    probe = vol.astype(np.float64).reshape(-1)[:: max(1, vol.size // 4096)]
    np.testing.assert_array_equal(probe, g["volume_probe"])
    rows = g["rows"]
    g = dict(g, volume=vol)
    dens, tex, cams, rig, dt, cells = _setup(g, cuda, rows=rows, layout=layout)
    tn_tf, n, _ = R.ray_setup(cams, dt, rig, dims=vol.shape)
    np.testing.assert_array_equal(n[0].cpu().numpy().ravel(), g["n_steps"].ravel())
    np.testing.assert_allclose(tn_tf[0].cpu().numpy().reshape(-1, 2).T, g["tn_tf"], rtol=0,
                               atol=1e-12)
    img, trans = R.forward(dens, tex, cams, dt, rig, cells=cells)
    assert rel_l2(img[0].double().cpu().numpy(), g["image"]) <= IMG_TOL
    seed = torch.from_numpy(g["seed_band"].astype(np.float32)).to(cuda)[None].contiguous()
    targets = [k.split("_", 1)[1] for k in g if k.startswith("inversion_")]
    targets = sorted({t.replace("_idx", "").replace("_val", "") for t in targets})
    got = _grads(dens, tex, cams, rig, dt, img, trans, seed, targets, cells=cells)
    for t in targets:
        if t == "volume" and "inversion_volume_idx" in g:
            ref = np.zeros(vol.size)
            ref[g["inversion_volume_idx"]] = g["inversion_volume_val"]
        else:
            ref = g[f"inversion_{t}"]
        err = rel_l2(got[t], ref)
        assert err <= BAND_TOL.get((name, t), GRAD_TOL), (name, t, err)


def test_sample_totals_match_reference(cuda):
    """Sum of n_steps over every ray of every config == the reference's count."""
    torch = _torch()
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.scenes import CONFIGS
    counts = golden("counts")
    for name, c in CONFIGS.items():
        ll = torch.tensor(c.view_poses(), dtype=torch.float64, device=cuda)
        cams = R.camera_array(ll, c.radius, (0.0, 0.0, 0.0), c.fov)
        total = 0
        for v0 in range(0, c.views, 16):
            _, n, _ = R.ray_setup(cams[v0:v0 + 16].contiguous(), c.dt, R.Rig(c.image, c.image))
            total += int(n.to(torch.int64).sum().item())
        assert total == int(counts[name + "_samples"]), name
