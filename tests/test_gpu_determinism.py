"""DDVR_FLAG_DETERMINISTIC (SURVEY 8b "Threading / determinism"): the camera and
stepsize gradients are summed per CTA and reduced in a fixed order, so repeated
runs agree BIT FOR BIT; the default mode (fp64 atomics across CTAs) agrees with
it to fp64 rounding.  Also: the deterministic sums still match the oracle, and
a step split over view chunks gives the same per-view camera gradients.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _scene(cuda, views=6, W=40, H=36):
    import torch
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.scenes import fibonacci_poses, phantom, preset_texels
    vol = torch.from_numpy(phantom("asymmetric", 32, seed=0).astype(np.float32)).to(cuda)
    tex = torch.from_numpy(preset_texels("grayscale", 16, 4.0).astype(np.float32)).to(cuda)
    ll = torch.tensor(fibonacci_poses(views), dtype=torch.float64, device=cuda)
    cams = R.camera_array(ll, 2.0, (0.0, 0.0, 0.0), 30.0)
    rig = R.Rig(W, H)
    dt = 0.5 / 32
    img, depth = R.forward(vol, tex, cams, dt, rig)
    seed = torch.from_numpy(np.random.default_rng(7).normal(size=tuple(img.shape))
                            .astype(np.float32)).to(cuda)
    return vol, tex, cams, rig, dt, img, depth, seed


def _grads(cuda, sc, deterministic, cells=None):
    import torch
    from paper_2107_12672_b200 import raymarch as R
    vol, tex, cams, rig, dt, img, depth, seed = sc
    d_cam = torch.zeros(cams.shape[0], 2, dtype=torch.float64, device=cuda)
    d_dt = torch.zeros(1, dtype=torch.float64, device=cuda)
    R.adjoint(vol, tex, cams, dt, rig, img, depth, seed, 3, d_camera=d_cam, d_dt=d_dt,
              cells=cells, deterministic=deterministic)
    return d_cam.cpu().numpy(), float(d_dt.item())


@pytest.mark.parametrize("layout", ["voxels", "cells"])
def test_camera_and_stepsize_are_bitwise_reproducible(cuda, layout):
    from paper_2107_12672_b200 import raymarch as R
    sc = _scene(cuda)
    cells = R.pack_cells(sc[0]) if layout == "cells" else None
    runs = [_grads(cuda, sc, True, cells) for _ in range(4)]
    for cam, dt in runs[1:]:
        assert np.array_equal(cam, runs[0][0]) and dt == runs[0][1]
    cam_a, dt_a = _grads(cuda, sc, False, cells)          # atomics: fp64 rounding apart
    assert np.allclose(cam_a, runs[0][0], rtol=1e-12, atol=1e-14 * np.abs(cam_a).max())
    assert abs(dt_a - runs[0][1]) <= 1e-12 * abs(dt_a)


def test_deterministic_sums_match_the_oracle(cuda):
    from oracle import dvr_oracle as O
    from paper_2107_12672_b200.scenes import fibonacci_poses, phantom, preset_texels
    sc = _scene(cuda, views=2, W=24, H=20)
    cam, dt_g = _grads(cuda, sc, True)
    grid = O.Grid(phantom("asymmetric", 32, seed=0).astype(np.float32))
    tex = preset_texels("grayscale", 16, 4.0).astype(np.float32).astype(np.float64)
    seed = sc[7].double().cpu().numpy()
    want_cam, want_dt = [], 0.0
    for k, (lon, lat) in enumerate(fibonacci_poses(2)):
        v = O.View(lon, lat, 2.0, (0, 0, 0), 30.0, 24, 20)
        g = O.adjoint_view(grid, tex, v, 0.5 / 32, seed[k], ["camera", "stepsize"])
        want_cam.append(np.asarray(g["d_camera"], np.float64).reshape(2))
        want_dt += float(g["d_stepsize"])
    assert rel_l2(cam, np.stack(want_cam)) <= 1e-4
    assert abs(dt_g - want_dt) <= 1e-4 * abs(want_dt)


def test_fused_chunks_keep_per_view_camera_sums(cuda):
    """Each call reduces its own partials: per-view camera gradients of a step split
    into view chunks equal the single call's bit for bit."""
    import torch
    from paper_2107_12672_b200 import raymarch as R
    vol, tex, cams, rig, dt, img, depth, seed = _scene(cuda)
    cells = R.pack_cells(vol)
    refs = (img + 0.05 * seed).contiguous()
    count = float(refs.numel())

    def run(splits):
        d_cam = torch.zeros(cams.shape[0], 2, dtype=torch.float64, device=cuda)
        d_dt = torch.zeros(1, dtype=torch.float64, device=cuda)
        loss = torch.zeros(1, dtype=torch.float64, device=cuda)
        ws = None
        bounds = np.linspace(0, cams.shape[0], splits + 1).astype(int)
        for k, (a, b) in enumerate(zip(bounds[:-1], bounds[1:])):
            if ws is None:
                import ctypes
                from paper_2107_12672_b200 import _native as N
                _, _, prm = R._descs(vol, tex, rig, dt, False, cells)
                vold, _, prm = R._descs(vol, tex, rig, dt, False, cells)
                extra = int(N.lib().ddvr_deterministic_bytes(ctypes.byref(vold),
                                                              int(cams.shape[0]),
                                                              ctypes.byref(prm), 3))
                ws = R.workspace_for(vol, 3, cells, tex, extra)
            R.forward_adjoint_l1(vol, tex, cams[a:b], dt, rig, refs[a:b], count, 3, cells=cells,
                                 loss=loss, d_camera=d_cam[a:b], d_dt=d_dt, workspace=ws,
                                 ws_continue=k > 0, ws_defer=k < splits - 1, deterministic=True)
        return d_cam.cpu().numpy(), float(d_dt.item()), float(loss.item())

    one, three = run(1), run(3)
    assert np.array_equal(one[0], three[0])
    assert abs(one[1] - three[1]) <= 1e-13 * abs(one[1])
    again = run(3)
    assert np.array_equal(again[0], three[0]) and again[1] == three[1]


@pytest.mark.parametrize("fused", [True, False])
def test_sharded_step_deterministic(cuda, fused):
    """ShardedStep(deterministic=True) (C3-style camera + stepsize targets): two steps
    give identical per-view camera gradients and stepsize gradient."""
    from test_gpu_step import _step
    step, _ = _step(cuda, "cells", targets=("camera", "stepsize"), fused=fused,
                    deterministic=True)
    a = step.run()
    cam_a, dt_a = step.d_camera.clone(), a.d_stepsize.clone()
    b = step.run()
    assert bool((step.d_camera == cam_a).all()) and bool((b.d_stepsize == dt_a).all())


def _det_scene(cuda, texels, n=28, views=4, W=30, H=26):
    import torch
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.scenes import fibonacci_poses, phantom
    truth = torch.from_numpy(phantom("sphere", n, seed=0).astype(np.float32)).to(cuda)
    tex = torch.from_numpy(texels.astype(np.float32)).to(cuda)
    ll = torch.tensor(fibonacci_poses(views), dtype=torch.float64, device=cuda)
    rig = R.Rig(W, H)
    dt = 0.2 / n
    cams = R.camera_array(ll, 2.0, (0.0, 0.0, 0.0), 30.0)
    refs, _ = R.forward(truth, tex, cams, dt, rig)
    est = (0.8 * truth + 0.1).contiguous()
    return est, tex, ll, refs, dt, rig


@pytest.mark.parametrize("tf", ["ramp", "warm"])
@pytest.mark.parametrize("chunks", [1, 3])
def test_density_gradient_is_bitwise_reproducible(cuda, tf, chunks):
    """DDVR_FLAG_DETERMINISTIC with the volume target: int64 fixed-point cell moments,
    so the fused step's d_volume is the same bits on every run (band tape / absorption
    walk for the ramp, the emitting inversion walk for the warm TF), also when the step
    is split into view chunks, and equals the fp32-atomic result to rounding."""
    import torch
    from paper_2107_12672_b200.distributed import ShardedStep
    from paper_2107_12672_b200.scenes import absorption_ramp_texels, preset_texels
    texels = absorption_ramp_texels(32, 3.0) if tf == "ramp" else preset_texels("warm", 16, 6.0)
    est, tex, ll, refs, dt, rig = _det_scene(cuda, texels)
    host = refs.cpu().pin_memory() if chunks > 1 else None
    runs = []
    for _ in range(3):
        step = ShardedStep(est, tex, ll, refs, dt, rig, deterministic=True, chunks=chunks)
        runs.append(step.run(refs_host=host).d_volume.clone())
    assert float(runs[0].abs().max()) > 0
    for r in runs[1:]:
        assert torch.equal(r, runs[0])
    plain = ShardedStep(est, tex, ll, refs, dt, rig).run().d_volume
    assert rel_l2(runs[0].double().cpu().numpy(), plain.double().cpu().numpy()) <= 1e-6


def test_adjoint_density_gradient_is_bitwise_reproducible(cuda):
    """ddvr_adjoint (one call, arbitrary seed): the scale comes from max|seed|."""
    import torch
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.scenes import preset_texels
    est, tex, ll, refs, dt, rig = _det_scene(cuda, preset_texels("warm", 16, 6.0))
    cams = R.camera_array(ll, 2.0, (0.0, 0.0, 0.0), 30.0)
    cells = R.pack_cells(est)
    img, depth = R.forward(est, tex, cams, dt, rig, cells=cells)
    seed = torch.randn(img.shape, generator=torch.Generator(device=cuda).manual_seed(3),
                       device=cuda)
    outs = []
    for det in (True, True, False):
        dv = torch.zeros_like(est)
        R.adjoint(est, tex, cams, dt, rig, img, depth, seed, 8, d_volume=dv, cells=cells,
                  deterministic=det)
        outs.append(dv)
    assert torch.equal(outs[0], outs[1])
    assert rel_l2(outs[0].double().cpu().numpy(), outs[2].double().cpu().numpy()) <= 1e-6
