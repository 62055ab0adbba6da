"""The benchmarked step at the configs' full sizes against the reference.

tests/golden/{C4,C5}_step_*.npz come from voldiff itself (oracle/gen_golden.py
step_cases): the tomography loop body of tasks.py:397-432 -- render of the
estimate, l1_loss against reference images rendered from the truth, render_adjoint
with that seed -- on row bands of the config's views at the full volume (256^3 /
512^3) and image (512^2 / 1024^2).  The GPU runs the same bands through
``ShardedStep`` (ddvr_forward_adjoint_l1), i.e. the kernels bench.py times, with
the band tape and the empty-space skips on and off:

* ``dense``: 0.85 truth + 0.1 U(0,1), the bench's iteration-1 state (no exact zeros);
* ``sparse`` (C4): the truth's support only, exact zeros outside the sphere, so the
  march's empty-brick skip and the walk's zero-word skip run over real empty space.

tests/golden/{C1,C2}_step_dense.npz (gen_golden.py tf_step_cases) hold the fused
TF-target steps the same way: C1 (64^3, one full 128^2 view, volume + TF targets) and
C2 (128^3, 16 rows of two 256^2 views, TF target), with d_tf in fp64.

Bars: image rel-L2 <= 1e-5, loss <= 1e-5 relative, d_volume and d_tf rel-L2 <= 1e-4.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, rel_l2

IMG_TOL = 1e-5
GRAD_TOL = 1e-4   # every case, C5 included (measured 1.0e-5 there: profiles/r02_parity.json;
# fp32-level density noise alone moves the reference's own C5 band gradient by 1e-5 .. 4e-5,
# profiles/r02_fp32_floor_c5.txt)


def _f32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def step_estimate(name: str, kind: str) -> np.ndarray:
    """The estimate of a step fixture: the generator and seed of gen_golden.step_cases
    (one default_rng(99) stream drawn for C4 then C5; tf_step_cases: default_rng(77),
    C1 then C2)."""
    from paper_2107_12672_b200.scenes import CONFIGS
    order = ("C1", "C2") if name in ("C1", "C2") else ("C4", "C5")
    rng = np.random.default_rng(77 if name in ("C1", "C2") else 99)
    for nm in order:
        truth = CONFIGS[nm].volume().astype(np.float64)
        u = rng.uniform(size=truth.shape)
        if nm == name:
            if kind == "dense":
                return _f32(0.85 * truth + 0.1 * u)
            return _f32(np.where(truth > 0, np.clip(0.7 * truth + 0.05, 0, 1), 0.0))
    raise KeyError(name)


@pytest.mark.parametrize("case", ["C4_step_dense", "C4_step_sparse", "C1_step_dense",
                                  "C2_step_dense"])
def test_step_estimates_are_reproduced(case):
    """(CPU) the tests rebuild exactly the estimate the fixture was computed from."""
    g = golden(case)
    name, _, kind = case.split("_")
    est = step_estimate(name, kind)
    np.testing.assert_array_equal(est.reshape(-1)[:: max(1, est.size // 4096)], g["est_probe"])


# (case, band tape, empty skip, split walk)
MODES = [("C4_step_dense", True, True, False), ("C4_step_dense", False, True, False),
         ("C4_step_dense", True, True, True),
         ("C4_step_sparse", True, True, False), ("C4_step_sparse", True, False, False),
         ("C4_step_sparse", False, True, False), ("C4_step_sparse", True, True, True),
         ("C5_step_dense", False, True, False)]


@pytest.mark.gpu
@pytest.mark.parametrize("case,tape,skip,split", MODES)
def test_fused_step_matches_reference_at_config_scale(cuda, case, tape, skip, split):
    import torch
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.distributed import ShardedStep
    from paper_2107_12672_b200.scenes import CONFIGS
    g = golden(case)
    name, _, kind = case.split("_")
    c = CONFIGS[name]
    est_np = step_estimate(name, kind)
    np.testing.assert_array_equal(est_np.reshape(-1)[:: max(1, est_np.size // 4096)],
                                  g["est_probe"])
    est = torch.from_numpy(est_np.astype(np.float32)).to(cuda)
    tex = torch.from_numpy(g["texels"]).to(cuda)
    poses = c.view_poses()
    ll = torch.tensor([poses[int(k)] for k in g["views"]], dtype=torch.float64, device=cuda)
    r0, r1 = (int(r) for r in g["rows"])
    rig = R.Rig(c.image, c.image, rows=(r0, r1))
    refs = torch.from_numpy(g["refs"]).to(cuda).contiguous()
    stats = torch.zeros(4, dtype=torch.int64, device=cuda)
    step = ShardedStep(est, tex, ll, refs, float(g["dt"]), rig, targets=("volume",),
                       total_elements=float(g["count"]), radius=c.radius, fov_y_deg=c.fov,
                       keep_images=True, band_tape=tape, empty_skip=skip, split_walk=split,
                       stats=stats)
    assert step.fused and step.band_tape == (tape and name == "C4")
    f = step.run()
    img = step.img.double().cpu().numpy()
    assert rel_l2(img, g["image"]) <= IMG_TOL
    assert abs(float(f.loss) - float(g["loss"])) <= IMG_TOL * float(g["loss"])
    want = np.zeros(est_np.size)
    want[g["volume_idx"]] = g["volume_val"]
    got = f.d_volume.double().cpu().numpy()
    err = rel_l2(got, want)
    assert err <= GRAD_TOL, err
    s = [int(x) for x in stats.cpu()]
    _, n, _ = R.ray_setup(step.cams, float(g["dt"]), rig, dims=tuple(est.shape))
    assert s[0] == int(n.to(torch.int64).sum()) and s[3] == n.numel()
    if kind == "sparse" and step.band_tape:
        assert s[2] > 0                        # the walk skipped empty tape words
        assert (s[1] > 0) == skip              # the march skipped empty bricks


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["C1_step_dense", "C2_step_dense"])
@pytest.mark.parametrize("graph,split", [(False, "auto"), (True, "auto"), (False, 1), (False, 2),
                                         (False, 4), (False, 8)])
def test_tf_step_matches_reference_at_config_scale(cuda, case, graph, split):
    """The fused TF-target step (C1: volume + TF, C2: TF) the bench times, eagerly and
    replayed from a CUDA graph (bench.py's default for C1), with the default and every
    forced segment split of the rays (DDVR_FLAG_RAY_SPLIT_*: 1, 2, 4, 8 threads per ray;
    the C1 and C2 bands have few enough rays that "auto" splits them)."""
    import torch
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.distributed import ShardedStep
    from paper_2107_12672_b200.scenes import CONFIGS
    g = golden(case)
    name = case.split("_")[0]
    c = CONFIGS[name]
    est_np = step_estimate(name, "dense")
    np.testing.assert_array_equal(est_np.reshape(-1)[:: max(1, est_np.size // 4096)],
                                  g["est_probe"])
    est = torch.from_numpy(est_np.astype(np.float32)).to(cuda)
    tex = torch.from_numpy(g["texels"]).to(cuda)
    poses = c.view_poses()
    ll = torch.tensor([poses[int(k)] for k in g["views"]], dtype=torch.float64, device=cuda)
    r0, r1 = (int(r) for r in g["rows"])
    rig = R.Rig(c.image, c.image, rows=(r0, r1))
    refs = torch.from_numpy(g["refs"]).to(cuda).contiguous()
    targets = tuple(c.targets)
    step = ShardedStep(est, tex, ll, refs, float(g["dt"]), rig, targets=targets,
                       total_elements=float(g["count"]), radius=c.radius, fov_y_deg=c.fov,
                       keep_images=True, ray_split=split)
    assert step.fused
    if graph:
        step.run()                              # warm up outside the capture
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            f = step.run()
        for _ in range(2):                      # every replay zeroes and refills the grads
            gr.replay()
        torch.cuda.synchronize()
    else:
        f = step.run()
    img = step.img.double().cpu().numpy()
    assert rel_l2(img, g["image"]) <= IMG_TOL
    assert abs(float(f.loss) - float(g["loss"])) <= IMG_TOL * float(g["loss"])
    err = rel_l2(f.d_tf.double().cpu().numpy().reshape(-1), g["d_tf"].reshape(-1))
    assert err <= GRAD_TOL, err
    if "volume" in targets:
        want = np.zeros(est_np.size)
        want[g["volume_idx"]] = g["volume_val"]
        err = rel_l2(f.d_volume.double().cpu().numpy().reshape(-1), want)
        assert err <= GRAD_TOL, err
