"""The on-device tomography step (distributed.ShardedStep / TomographyIteration).

One step = pack cells, forward over this rank's views, fused L1 loss + seed over
the global element count (objectives.py:38-54), adjoint, all-reduce (a no-op
at world size 1).  Checked against the oracle's per-view forward / L1 /
adjoint sum (the same restatement tests/test_distributed.py reduces over gloo
ranks), for both volume layouts, with device-resident and host-staged
reference images.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2
from test_distributed import _rank_grads, _scene

pytestmark = pytest.mark.gpu


def _step(cuda, layout, targets=("volume", "tf", "stepsize"), **kw):
    import torch
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.distributed import ShardedStep
    grid, tex, views, refs, dt = _scene()
    vol = torch.from_numpy(grid.values.astype(np.float32)).to(cuda)
    tx = torch.from_numpy(tex.astype(np.float32)).to(cuda)
    ll = torch.tensor([[v.lon_deg, v.lat_deg] for v in views], dtype=torch.float64, device=cuda)
    rf = torch.from_numpy(np.stack(refs).astype(np.float32)).to(cuda)
    step = ShardedStep(vol, tx, ll, rf, dt, R.Rig(6, 5), targets=targets, radius=2.3,
                       layout=layout, **kw)
    return step, rf


@pytest.mark.parametrize("layout,fused", [("cells", True), ("cells", False), ("voxels", False)])
def test_step_matches_oracle(cuda, layout, fused):
    """fused: ddvr_forward_adjoint_l1 (one kernel per ray); else forward + l1 + adjoint."""
    step, _ = _step(cuda, layout, fused=fused)
    assert step.fused == fused
    f = step.run()
    ref = _rank_grads(0, 1)
    assert abs(float(f.loss) - float(ref.loss)) <= 1e-5 * abs(float(ref.loss))
    for name in ("d_volume", "d_tf", "d_stepsize"):
        got = getattr(f, name).double().cpu().numpy()
        want = getattr(ref, name).double().numpy()
        assert rel_l2(got, want) <= 1e-4, (name, rel_l2(got, want))


def test_host_staged_refs_are_identical(cuda):
    """refs_host: the copy runs on a side stream and the loss kernel waits for it."""
    step, rf = _step(cuda, "cells", fused=True)
    a = step.run().buf.clone()
    host = rf.cpu().pin_memory()
    rf.zero_()                        # the step must use the staged copy, not stale data
    b = step.run(refs_host=host).buf.clone()
    # (equal up to the order of the fp32 atomic reductions)
    assert rel_l2(b.double().cpu().numpy(), a.double().cpu().numpy()) <= 1e-6
    with pytest.raises(ValueError):
        step.run(refs_host=host[:1])


def test_tomography_iterations_reduce_the_loss(cuda):
    """A few full iterations (step + prior + Adam + projection) recover the
    density that rendered the references (tasks.py:397-481)."""
    import torch
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.distributed import ShardedStep, TomographyIteration
    from paper_2107_12672_b200.scenes import absorption_ramp_texels, fibonacci_poses, phantom
    truth = torch.from_numpy(phantom("sphere", 24, seed=0).astype(np.float32)).to(cuda)
    tx = torch.from_numpy(absorption_ramp_texels(32, 3.0).astype(np.float32)).to(cuda)
    ll = torch.tensor(fibonacci_poses(12), dtype=torch.float64, device=cuda)
    rig = R.Rig(32, 32)
    cams = R.camera_array(ll, 2.0, (0.0, 0.0, 0.0), 30.0)
    refs, _ = R.forward(truth, tx, cams, 0.2 / 24, rig)
    est = torch.full_like(truth, 0.3)
    it = TomographyIteration(ShardedStep(est, tx, ll, refs, 0.2 / 24, rig), lr=0.05, lam=0.0)
    losses = [float(it.run()[0]) for _ in range(25)]
    assert losses[-1] < 0.5 * losses[0]
    assert float(est.min()) >= 0.0 and float(est.max()) <= 1.0   # projection (optim.py:78-89)


@pytest.mark.parametrize("fused", ["auto", True, False])
def test_step_camera_gradients_stay_per_view(cuda, fused):
    """C3-style targets: d/d(lon, lat) per view (field.py:11), kept by the owning rank
    ("auto" runs the separate kernels for these targets)."""
    from oracle import dvr_oracle as O
    step, _ = _step(cuda, "cells", targets=("camera", "stepsize"), fused=fused)
    assert step.fused == (fused is not False)   # camera / stepsize alone: "auto" fuses
    f = step.run()
    grid, tex, views, refs, dt = _scene()
    count = sum(r.size for r in refs)
    want = []
    for v, ref in zip(views, refs):
        img = O.render_view(grid, tex, v, dt)
        g = O.adjoint_view(grid, tex, v, dt, np.sign(img - ref) / count, ["camera"], image=img)
        want.append(np.asarray(g["d_camera"], np.float64).reshape(2))
    got = step.d_camera.cpu().numpy()
    assert got.shape == (len(views), 2)
    assert rel_l2(got, np.stack(want)) <= 1e-4
    assert float(f.d_stepsize) != 0.0


def test_fused_step_images_and_chunks(cuda):
    """keep_images: the fused step's images equal forward(); host-staged refs in
    chunks give the single-launch result."""
    from paper_2107_12672_b200 import raymarch as R
    step, rf = _step(cuda, "cells", keep_images=True, chunks=3, fused=True)
    f1 = step.run().buf.clone()
    img, depth = R.forward(step.density, step.texels, step.cams, step.dt, step.rig,
                           cells=step.cells)
    assert rel_l2(step.img.double().cpu().numpy(), img.double().cpu().numpy()) <= 1e-6
    assert rel_l2(step.depth.double().cpu().numpy(), depth.double().cpu().numpy()) <= 1e-6
    host = rf.cpu().pin_memory()
    f2 = step.run(refs_host=host).buf.clone()      # 3 chunks, each waits for its refs
    assert rel_l2(f2.double().cpu().numpy(), f1.double().cpu().numpy()) <= 1e-6


def test_graphed_iterations_follow_the_eager_trajectory(cuda):
    """TomographyIteration(graph=True): two eager warm-ups, then one captured CUDA
    graph replayed per iteration (device-side Adam counter)."""
    import torch
    from paper_2107_12672_b200.distributed import TomographyIteration
    vols = []
    for graph in (False, True):
        step, _ = _step(cuda, "cells", targets=("volume",))
        it = TomographyIteration(step, lr=0.05, lam=0.1, graph=graph)
        losses = [float(it.run()[0]) for _ in range(6)]
        vols.append(step.density.clone())
        assert losses[-1] < losses[0]
    assert rel_l2(vols[1].double().cpu().numpy(), vols[0].double().cpu().numpy()) <= 1e-5
    with pytest.raises(ValueError):
        it.run(refs_host=torch.zeros(1))


@pytest.mark.parametrize("kind", ["piecewise", "gaussian"])
def test_fused_step_analytic_tfs(cuda, kind):
    """The fused kernel's forward dispatch and walk for the (K,5) piecewise-linear
    and (G,6) Gaussian TFs equal the separate launches (volume + tf targets)."""
    import torch
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.distributed import ShardedStep
    grid, _, views, refs, dt = _scene()
    rng = np.random.default_rng(8)
    if kind == "piecewise":
        pos = np.sort(np.concatenate([[0.0, 1.0], rng.uniform(0.05, 0.95, 5)]))
        tf = np.column_stack([pos, rng.uniform(0.1, 1.0, (7, 3)), rng.uniform(0.2, 2.5, 7)])
    else:
        tf = np.column_stack([rng.uniform(0.2, 0.8, 4), rng.uniform(0.05, 0.3, 4),
                              rng.uniform(0.1, 1.0, (4, 3)), rng.uniform(0.5, 3.0, 4)])
    vol = torch.from_numpy(grid.values.astype(np.float32)).to(cuda)
    tx = torch.from_numpy(tf.astype(np.float32)).to(cuda)
    ll = torch.tensor([[v.lon_deg, v.lat_deg] for v in views], dtype=torch.float64, device=cuda)
    rf = torch.from_numpy(np.stack(refs).astype(np.float32)).to(cuda)
    bufs = []
    for fused in (True, False):
        step = ShardedStep(vol, tx, ll, rf, dt, R.Rig(6, 5), targets=("volume", "tf"),
                           radius=2.3, fused=fused)
        assert step.fused == fused
        bufs.append(step.run().buf.double().cpu().numpy())
    assert rel_l2(bufs[0], bufs[1]) <= 1e-5


def test_fused_step_row_band(cuda):
    """A row band (renderer.py:491 tiles) through the fused kernel equals the
    separate launches on the same band."""
    import torch
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.distributed import ShardedStep
    grid, tex, views, refs, dt = _scene()
    vol = torch.from_numpy(grid.values.astype(np.float32)).to(cuda)
    tx = torch.from_numpy(tex.astype(np.float32)).to(cuda)
    ll = torch.tensor([[v.lon_deg, v.lat_deg] for v in views], dtype=torch.float64, device=cuda)
    rf = torch.from_numpy(np.stack(refs).astype(np.float32)[:, 1:4]).to(cuda).contiguous()
    bufs = []
    for fused in (True, False):
        step = ShardedStep(vol, tx, ll, rf, dt, R.Rig(6, 5, rows=(1, 4)),
                           targets=("volume", "tf", "stepsize"), radius=2.3, fused=fused)
        bufs.append(step.run().buf.double().cpu().numpy())
    assert rel_l2(bufs[0], bufs[1]) <= 1e-5


def _ramp_scene(cuda, n=24, views=6, W=32, H=30, texels=None):
    import torch
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.scenes import absorption_ramp_texels, fibonacci_poses, phantom
    truth = torch.from_numpy(phantom("sphere", n, seed=0).astype(np.float32)).to(cuda)
    tex = torch.from_numpy((absorption_ramp_texels(64, 3.0) if texels is None else texels)
                           .astype(np.float32)).to(cuda)
    ll = torch.tensor(fibonacci_poses(views), dtype=torch.float64, device=cuda)
    rig = R.Rig(W, H)
    dt = 0.2 / n
    cams = R.camera_array(ll, 2.0, (0.0, 0.0, 0.0), 30.0)
    refs, _ = R.forward(truth, tex, cams, dt, rig)
    est = (0.8 * truth + 0.1).contiguous()
    return est, tex, ll, refs, dt, rig


@pytest.mark.parametrize("chunks", [1, 3])
def test_band_tape_step_equals_gathering_walk(cuda, chunks):
    """DDVR_FLAG_BAND_TAPE: the absorption walk from the march's band bits gives the
    gathering walk's gradient (same runs and moments; atomics order aside) and the
    oracle's, also when the step is split into view chunks."""
    import torch
    from oracle import dvr_oracle as O
    from paper_2107_12672_b200.distributed import ShardedStep
    est, tex, ll, refs, dt, rig = _ramp_scene(cuda)
    out = {}
    for tape in (False, True):
        step = ShardedStep(est, tex, ll, refs, dt, rig, band_tape=tape, chunks=chunks)
        assert step.fused and step.band_tape == tape
        f = step.run(refs_host=refs.cpu().pin_memory() if chunks > 1 else None)
        out[tape] = (f.d_volume.double().cpu().numpy(), float(f.loss))
    assert rel_l2(out[True][0], out[False][0]) <= 1e-6
    # (the band-tape march sums each 32-sample word's optical depth in fp32 before the
    # fp64 ray total: images, hence the L1 loss, agree to fp32 rounding)
    assert abs(out[True][1] - out[False][1]) <= 1e-6 * abs(out[False][1])
    grid = O.Grid(est.cpu().numpy().astype(np.float64))
    t64 = tex.cpu().numpy().astype(np.float64)
    count = refs.numel()
    want = np.zeros(tuple(est.shape))
    for k, (lon, lat) in enumerate(ll.cpu().numpy()):
        v = O.View(lon, lat, 2.0, (0, 0, 0), 30.0, rig.width, rig.height)
        img = O.render_view(grid, t64, v, dt)
        seed = np.sign(img - refs[k].cpu().numpy().astype(np.float64)) / count
        want += O.adjoint_view(grid, t64, v, dt, seed, ["volume"], image=img)["d_volume"]
    assert rel_l2(out[True][0], want) <= 1e-4


def test_band_tape_is_ignored_off_the_affine_walk(cuda):
    """A non-affine emission-free TF takes the table walk: the tape flag changes
    nothing (the kernel only uses it on the affine band walk)."""
    from paper_2107_12672_b200.distributed import ShardedStep
    rng = np.random.default_rng(2)
    tex = np.zeros((16, 4))
    tex[:, 3] = np.sort(rng.uniform(0.0, 4.0, 16))
    est, tx, ll, refs, dt, rig = _ramp_scene(cuda, texels=tex)
    g = [ShardedStep(est, tx, ll, refs, dt, rig, band_tape=t).run().d_volume.double().cpu()
         .numpy() for t in (False, True)]
    assert rel_l2(g[1], g[0]) <= 1e-6


def test_band_tape_auto_and_workspace(cuda):
    """"auto" turns the tape on when it fits; a too-small workspace is refused."""
    import ctypes
    import torch
    from paper_2107_12672_b200 import _native as N
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.distributed import ShardedStep
    est, tex, ll, refs, dt, rig = _ramp_scene(cuda)
    assert ShardedStep(est, tex, ll, refs, dt, rig).band_tape
    assert not ShardedStep(est, tex, ll, refs, dt, rig, targets=("volume", "tf")).band_tape
    cells = R.pack_cells(est)
    cams = R.camera_array(ll, 2.0, (0.0, 0.0, 0.0), 30.0)
    ws = R.workspace_for(est, 8, cells, tex)           # no room for the tape
    loss = torch.zeros(1, dtype=torch.float64, device=cuda)
    from paper_2107_12672_b200.errors import InvalidInputError
    with pytest.raises(InvalidInputError, match="band tape"):
        R.forward_adjoint_l1(est, tex, cams, dt, rig, refs, float(refs.numel()), 8, cells=cells,
                             loss=loss, d_volume=torch.zeros_like(est), workspace=ws,
                             band_tape=True)
    vol, _, prm = R._descs(est, tex, rig, dt, False, cells)
    words = int(N.lib().ddvr_band_tape_bytes(ctypes.byref(vol), 6, ctypes.byref(prm)))
    assert words > 0 and words % 256 == 0


@pytest.mark.parametrize("n,dt_vox", [(24, 0.2), (40, 0.05)])
def test_band_tape_skips_empty_blocks_exactly(cuda, n, dt_vox):
    """An estimate with exactly empty space (the sphere phantom: density 0 outside
    the ball, so whole 32-sample tape words are 0 and the walk skips them, and
    empty cell runs skip their flush) gives the gathering walk's gradient and the
    oracle's."""
    import torch
    from oracle import dvr_oracle as O
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.distributed import ShardedStep
    from paper_2107_12672_b200.scenes import absorption_ramp_texels, fibonacci_poses, phantom
    truth = phantom("sphere", n, seed=0).astype(np.float32)
    est_np = np.where(truth > 0, np.clip(0.7 * truth + 0.05, 0, 1), 0.0).astype(np.float32)
    est = torch.from_numpy(est_np).to(cuda)
    tex = torch.from_numpy(absorption_ramp_texels(64, 3.0).astype(np.float32)).to(cuda)
    ll = torch.tensor(fibonacci_poses(5), dtype=torch.float64, device=cuda)
    rig = R.Rig(28, 26)
    dt = dt_vox / n
    cams = R.camera_array(ll, 2.0, (0.0, 0.0, 0.0), 30.0)
    refs, _ = R.forward(torch.from_numpy(truth).to(cuda), tex, cams, dt, rig)
    got = {}
    for tape in (False, True):
        step = ShardedStep(est, tex, ll, refs, dt, rig, band_tape=tape)
        assert step.band_tape == tape
        got[tape] = step.run().d_volume.double().cpu().numpy()
    assert np.abs(got[True]).max() > 0
    assert rel_l2(got[True], got[False]) <= 1e-6
    grid = O.Grid(est_np.astype(np.float64))
    t64 = tex.cpu().numpy().astype(np.float64)
    want = np.zeros((n, n, n))
    for k, (lon, lat) in enumerate(ll.cpu().numpy()):
        v = O.View(lon, lat, 2.0, (0, 0, 0), 30.0, rig.width, rig.height)
        img = O.render_view(grid, t64, v, dt)
        seed = np.sign(img - refs[k].cpu().numpy().astype(np.float64)) / refs.numel()
        want += O.adjoint_view(grid, t64, v, dt, seed, ["volume"], image=img)["d_volume"]
    assert rel_l2(got[True], want) <= 1e-4


def _brick_map_np(vol: np.ndarray) -> np.ndarray:
    """The brick occupancy map the fused band-tape step builds (ddvr_abi.cu
    brick_occupancy_kernel), restated: padded cell s (storage index, cell s-1) is
    occupied when one of its edge-clamped corners is nonzero; brick b = cells
    [8b, 8b+8) per axis."""
    nz = np.pad(vol != 0, 1, mode="edge")          # padded[p] = voxel clamp(p-1)
    cell = np.zeros(tuple(d + 1 for d in vol.shape), bool)
    for dx in (0, 1):
        for dy in (0, 1):
            for dz in (0, 1):
                cell |= nz[dx:dx + cell.shape[0], dy:dy + cell.shape[1], dz:dz + cell.shape[2]]
    nb = tuple((d + 8) >> 3 for d in vol.shape)
    occ = np.zeros(nb, bool)
    for b in np.ndindex(*nb):
        occ[b] = cell[8 * b[0]:8 * b[0] + 8, 8 * b[1]:8 * b[1] + 8, 8 * b[2]:8 * b[2] + 8].any()
    return occ


@pytest.mark.parametrize("dt_vox", [0.2, 0.11, 0.5])
def test_band_tape_empty_brick_skip_is_exact(cuda, dt_vox):
    """The march's empty-space skip (32-sample blocks whose samples all lie in
    unoccupied bricks) changes nothing: image and optical depth bitwise, the band tape
    bitwise, the loss and the density gradient to atomic-order rounding -- against the
    same call with DDVR_FLAG_NO_EMPTY_SKIP.  The occupancy map itself equals the numpy
    restatement, and the gradient matches the oracle.  dt 0.5 voxel: a block can span
    more than 8 cells on an axis, so those rays march every block."""
    import ctypes
    import torch
    from oracle import dvr_oracle as O
    from paper_2107_12672_b200 import _native as N
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.scenes import absorption_ramp_texels, fibonacci_poses
    n = 72
    g = np.stack(np.meshgrid(*[np.arange(n)] * 3, indexing="ij"), -1).astype(np.float64)
    r = np.linalg.norm(g - np.array([44.0, 34.0, 30.0]), axis=-1)
    est_np = np.where(r < 14, np.clip(1.0 - r / 16, 0, 1), 0.0).astype(np.float32)
    truth = np.where(r < 12, 0.8, 0.0).astype(np.float32)
    est = torch.from_numpy(est_np).to(cuda)
    tex = torch.from_numpy(absorption_ramp_texels(64, 3.0).astype(np.float32)).to(cuda)
    ll = torch.tensor(fibonacci_poses(6), dtype=torch.float64, device=cuda)
    rig = R.Rig(40, 36)
    dt = dt_vox / n
    cams = R.camera_array(ll, 2.0, (0.0, 0.0, 0.0), 30.0)
    refs, _ = R.forward(torch.from_numpy(truth).to(cuda), tex, cams, dt, rig)
    cells = R.pack_cells(est)
    vol, _, prm = R._descs(est, tex, rig, dt, False, cells)
    band = int(N.lib().ddvr_band_tape_bytes(ctypes.byref(vol), 6, ctypes.byref(prm)))
    base = int(N.lib().ddvr_adjoint_workspace_bytes(
        ctypes.byref(vol), ctypes.byref(N.DdvrTf(N.TF_TEXTURE, 64, tex.data_ptr())),
        N.TARGET_VOLUME))
    base = (base + 255) & ~255
    nb = ((n + 8) >> 3) ** 3
    map_bytes = (2 * nb + 255) & ~255
    ctas = 6 * ((rig.width + 15) // 16) * ((rig.height + 15) // 16)
    rayk_bytes = (ctas * 256 * 4 + 255) & ~255
    tape_bytes = band - map_bytes - rayk_bytes
    out = {}
    for skip in (True, False, "no map", "split"):
        # "no map": a workspace that ends after the tape (the map and the walk weights
        # are optional: no skip); "split": march and walk as two kernels
        # (DDVR_FLAG_SPLIT_WALK)
        size = base + (tape_bytes if skip == "no map" else band)
        ws = torch.zeros(size // 4, dtype=torch.float32, device=cuda)
        img = torch.empty(6, rig.band_rows, rig.width, 4, dtype=torch.float32, device=cuda)
        depth = torch.empty(6, rig.band_rows, rig.width, dtype=torch.float32, device=cuda)
        loss = torch.zeros(1, dtype=torch.float64, device=cuda)
        dv = torch.zeros_like(est)
        R.forward_adjoint_l1(est, tex, cams, dt, rig, refs, float(refs.numel()), N.TARGET_VOLUME,
                             cells=cells, loss=loss, d_volume=dv, workspace=ws, image_out=img,
                             depth_out=depth, band_tape=True,
                             empty_skip=skip is True or skip == "split",
                             split_walk=skip == "split")
        raw = ws.view(torch.uint8).cpu().numpy()
        out[skip] = dict(img=img.cpu().numpy(), depth=depth.cpu().numpy(), loss=loss.item(),
                         dv=dv.double().cpu().numpy(), tape=raw[base:base + tape_bytes],
                         occ=raw[base + tape_bytes:base + tape_bytes + nb])
    a, b = out[True], out[False]
    for c in (out["no map"], out["split"]):   # one kernel or two: the same step
        np.testing.assert_array_equal(a["img"], c["img"])
        np.testing.assert_array_equal(a["depth"], c["depth"])
        np.testing.assert_array_equal(a["tape"], c["tape"])
        assert a["loss"] == pytest.approx(c["loss"], rel=1e-12)
        assert rel_l2(a["dv"], c["dv"]) <= 1e-6
    want_map = _brick_map_np(est_np).ravel()
    assert want_map.any() and not want_map.all()
    np.testing.assert_array_equal(a["occ"].astype(bool), want_map)
    assert not b["occ"].any()        # NO_EMPTY_SKIP builds no map
    np.testing.assert_array_equal(a["img"], b["img"])
    np.testing.assert_array_equal(a["depth"], b["depth"])
    np.testing.assert_array_equal(a["tape"], b["tape"])
    assert a["loss"] == pytest.approx(b["loss"], rel=1e-12)
    assert np.abs(a["dv"]).max() > 0
    assert rel_l2(a["dv"], b["dv"]) <= 1e-6
    grid = O.Grid(est_np.astype(np.float64))
    t64 = tex.cpu().numpy().astype(np.float64)
    want = np.zeros((n, n, n))
    for k, (lon, lat) in enumerate(ll.cpu().numpy()):
        v = O.View(lon, lat, 2.0, (0, 0, 0), 30.0, rig.width, rig.height)
        im = O.render_view(grid, t64, v, dt)
        seed = np.sign(im - refs[k].cpu().numpy().astype(np.float64)) / refs.numel()
        want += O.adjoint_view(grid, t64, v, dt, seed, ["volume"], image=im)["d_volume"]
    assert rel_l2(a["dv"], want) <= 1e-4


@pytest.mark.parametrize("kind", ["texture", "piecewise", "gaussian"])
@pytest.mark.parametrize("targets", [("tf",), ("volume", "tf")])
def test_fused_step_ray_split_matches_one_thread_per_ray(cuda, kind, targets):
    """Segment-split rays (DDVR_FLAG_RAY_SPLIT_2/4/8) against one thread per ray, for
    every TF kind and both split masks: the composed image, the L1 loss and every
    gradient agree up to fp32 reassociation (segments shorter than SPLIT included: the
    scene's rays have 3-40 samples)."""
    import torch
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.distributed import ShardedStep
    rng = np.random.default_rng(21)
    n = 20
    vol = torch.from_numpy(rng.uniform(0.0, 1.0, (n, n, n)).astype(np.float32)).to(cuda)
    if kind == "texture":
        tf = rng.uniform(0.1, 1.0, (16, 4)) * np.array([1, 1, 1, 6.0])
    elif kind == "piecewise":
        pos = np.sort(np.concatenate([[0.0, 1.0], rng.uniform(0.05, 0.95, 5)]))
        tf = np.column_stack([pos, rng.uniform(0.1, 1.0, (7, 3)), rng.uniform(0.2, 6.0, 7)])
    else:
        tf = np.column_stack([rng.uniform(0.2, 0.8, 4), rng.uniform(0.05, 0.3, 4),
                              rng.uniform(0.1, 1.0, (4, 3)), rng.uniform(0.5, 6.0, 4)])
    tx = torch.from_numpy(tf.astype(np.float32)).to(cuda)
    ll = torch.tensor([[25.0, 10.0], [200.0, -40.0], [95.0, 65.0]], dtype=torch.float64,
                      device=cuda)
    W, H = 21, 19
    # references at -1 or 2: every seed sign is fixed away from image == ref (an image
    # change of 1e-7 cannot flip a pixel's seed)
    refs = torch.from_numpy(rng.choice([-1.0, 2.0], (3, H, W, 4)).astype(np.float32)).to(cuda)
    out = {}
    for split in (1, 2, 4, 8):
        step = ShardedStep(vol, tx, ll, refs, 0.6 / n, R.Rig(W, H), targets=targets,
                           radius=2.0, keep_images=True, ray_split=split)
        assert step.fused
        f = step.run()
        torch.cuda.synchronize()
        out[split] = (step.img.double().cpu().numpy(), float(f.loss),
                      f.d_tf.double().cpu().numpy(), f.d_volume.double().cpu().numpy())
    img1, loss1, dtf1, dvol1 = out[1]
    assert np.abs(dtf1).max() > 0
    for split in (2, 4, 8):
        img, loss, dtf, dvol = out[split]
        assert rel_l2(img, img1) <= 1e-6, (split, rel_l2(img, img1))
        assert abs(loss - loss1) <= 1e-6 * abs(loss1)
        assert rel_l2(dtf, dtf1) <= 1e-5, (split, rel_l2(dtf, dtf1))
        if "volume" in targets:
            assert rel_l2(dvol, dvol1) <= 1e-5, (split, rel_l2(dvol, dvol1))


@pytest.mark.parametrize("split", [2, 4])
def test_fused_camera_step_ray_split_matches_one_thread_per_ray(cuda, split):
    """Camera / stepsize targets with forced segment-split rays (DDVR_FLAG_RAY_SPLIT_2/4):
    every segment walks with its samples' whole-ray indices (t = i dt) and its partial
    sums go through the same per-ray Jacobian chain (linear in them), so the per-view
    camera gradients, the stepsize gradient, the image and the loss agree with one thread
    per ray up to the summation order."""
    import torch
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.distributed import ShardedStep
    rng = np.random.default_rng(31)
    n = 20
    vol = torch.from_numpy(rng.uniform(0.0, 1.0, (n, n, n)).astype(np.float32)).to(cuda)
    tf = rng.uniform(0.1, 1.0, (16, 4)) * np.array([1, 1, 1, 6.0])
    tx = torch.from_numpy(tf.astype(np.float32)).to(cuda)
    ll = torch.tensor([[25.0, 10.0], [200.0, -40.0], [95.0, 65.0]], dtype=torch.float64,
                      device=cuda)
    W, H = 21, 19
    refs = torch.from_numpy(rng.choice([-1.0, 2.0], (3, H, W, 4)).astype(np.float32)).to(cuda)
    out = {}
    for k in (1, split):
        step = ShardedStep(vol, tx, ll, refs, 0.6 / n, R.Rig(W, H), targets=("camera", "stepsize"),
                           radius=2.0, keep_images=True, fused=True, ray_split=k)
        f = step.run()
        torch.cuda.synchronize()
        out[k] = (step.img.double().cpu().numpy(), float(f.loss),
                  step.d_camera.double().cpu().numpy(), float(f.d_stepsize))
    img1, loss1, cam1, dt1 = out[1]
    img, loss, cam, dtk = out[split]
    assert np.abs(cam1).max() > 0 and dt1 != 0.0
    assert rel_l2(img, img1) <= 1e-6
    assert abs(loss - loss1) <= 1e-6 * abs(loss1)
    assert rel_l2(cam, cam1) <= 1e-5, rel_l2(cam, cam1)
    assert abs(dtk - dt1) <= 1e-5 * abs(dt1)
