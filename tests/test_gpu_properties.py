"""Autograd path, edge cases and full-size (C4) properties of the CUDA path.

At C4/C5 sizes the fp64 oracle cannot run the whole workload, so full-size
checks use properties that hold independently of size: linearity of the
adjoint in its seed, agreement of the two volume layouts, the sum of
per-view gradients equal to the multi-view launch, exact sample counts, and
finite outputs.  Small cases are compared with the oracle directly.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

BITS = {"camera": 1, "stepsize": 2, "tf": 4, "volume": 8}


def _t():
    import torch
    return torch


def _oracle(vol, tex, views, dt, seeds, targets):
    from oracle import dvr_oracle as O
    g = O.Grid(vol.astype(np.float64))
    imgs, outs = [], []
    for v, s in zip(views, seeds):
        img = O.render_view(g, tex.astype(np.float64), v, dt)
        imgs.append(img)
        outs.append(O.adjoint_view(g, tex.astype(np.float64), v, dt, s, targets, image=img))
    return imgs, outs


def test_autograd_multiview_matches_oracle(cuda):
    torch = _t()
    from oracle import dvr_oracle as O
    from paper_2107_12672_b200 import Rig, render_views
    rng = np.random.default_rng(11)
    vol = rng.uniform(0.1, 0.9, (10, 12, 9)).astype(np.float32)
    tex = rng.uniform(0.1, 1.5, (16, 4)).astype(np.float32)
    poses = [(15.0, 25.0), (140.0, -40.0), (260.0, 5.0)]
    H, W, dt = 11, 13, 0.05
    dens = torch.from_numpy(vol).to(cuda).requires_grad_(True)
    tx = torch.from_numpy(tex).to(cuda).requires_grad_(True)
    ll = torch.tensor(poses, dtype=torch.float64, device=cuda, requires_grad=True)
    dtt = torch.tensor(dt, dtype=torch.float64, requires_grad=True)
    seeds = rng.normal(size=(3, H, W, 4)).astype(np.float32)
    img = render_views(dens, tx, ll, dtt, Rig(W, H), radius=2.4, fov_y_deg=35.0)
    (img * torch.from_numpy(seeds).to(cuda)).sum().backward()
    views = [O.View(lon, lat, 2.4, fov_y_deg=35.0, width=W, height=H) for lon, lat in poses]
    imgs, outs = _oracle(vol, tex, views, dt, seeds.astype(np.float64),
                         ["volume", "tf", "camera", "stepsize"])
    assert rel_l2(img.detach().cpu().numpy(), np.stack(imgs)) <= 1e-5
    assert rel_l2(dens.grad.cpu().numpy(), sum(o["d_volume"] for o in outs)) <= 1e-4
    assert rel_l2(tx.grad.cpu().numpy(), sum(o["d_tf"] for o in outs)) <= 1e-4
    assert rel_l2(ll.grad.cpu().numpy(), np.stack([o["d_camera"] for o in outs])) <= 1e-4
    assert rel_l2(dtt.grad.numpy(), sum(o["d_stepsize"] for o in outs)) <= 1e-4


def test_autograd_only_requested_targets(cuda):
    torch = _t()
    from paper_2107_12672_b200 import Rig, render_views
    dens = torch.rand(6, 6, 6, device=cuda, requires_grad=True)
    tx = torch.rand(8, 4, device=cuda)
    ll = torch.tensor([[10.0, 20.0]], dtype=torch.float64, device=cuda)
    img = render_views(dens, tx, ll, 0.05, Rig(5, 5))
    img.sum().backward()
    assert dens.grad is not None and tx.grad is None and ll.grad is None


# R2048: 2048 independent random texels (slope ~ +-2000, a kink at every texel
# boundary) put the gradients on the fp32 floor: the fp64 oracle itself moves
# by up to 1.37e-4 (camera) under fp32-level density noise
# (tools/fp32_floor_r2048.py), so that case is held to 2.5x its floor; the
# smooth 2048-texel table (R2048s) keeps the standard bar.
GRAD_BAR = {"R2048": 3.5e-4}


@pytest.mark.parametrize("case", ["inside_box", "tiny_dt", "big_dt", "R2048", "R2048s",
                                  "row_band", "one_pixel", "flat_volume", "single_voxel",
                                  "axis_aligned", "R1"])
def test_edge_cases_match_oracle(cuda, case):
    torch = _t()
    from oracle import dvr_oracle as O
    from paper_2107_12672_b200 import raymarch as R
    rng = np.random.default_rng(5)
    vol = rng.uniform(0.05, 0.95, (8, 8, 8)).astype(np.float32)
    tex = rng.uniform(0.05, 1.0, (8, 4)).astype(np.float32)
    radius, W, H, dt, rows = 2.2, 9, 7, 0.04, None
    lon, lat = 33.0, 21.0
    if case == "flat_volume":     # a size-1 axis: every cell clamps to one voxel layer
        vol = rng.uniform(0.05, 0.95, (1, 6, 5)).astype(np.float32)
    elif case == "single_voxel":  # 1x1x1: a constant field inside the box
        vol = np.full((1, 1, 1), 0.6, np.float32)
    elif case == "axis_aligned":  # w parallel to two slab pairs (renderer.py:194-197)
        lon, lat = 0.0, 0.0
        W = H = 1
    elif case == "R1":            # one texel: both lookup indices 0, zero slope
        tex = rng.uniform(0.05, 1.0, (1, 4)).astype(np.float32)
    if case == "inside_box":      # clamped rays: the eye is inside the volume (renderer.py:201)
        radius = 0.3
    elif case == "tiny_dt":       # ~2.6k samples per ray: inversion drift, fixed-point positions
        dt = 5e-4
    elif case == "big_dt":        # 1-3 samples per ray
        dt = 0.7
    elif case == "R2048":
        tex = rng.uniform(0.05, 1.0, (2048, 4)).astype(np.float32)
    elif case == "R2048s":
        x = (np.arange(2048) + 0.5) / 2048
        tex = np.stack([0.5 + 0.4 * np.sin(6 * x + k) for k in range(3)] +
                       [2.0 + 1.5 * np.sin(9 * x)], axis=1).astype(np.float32)
    elif case == "row_band":
        rows = (3, 6)
    elif case == "one_pixel":
        W = H = 1
    view = O.View(lon, lat, radius, fov_y_deg=35.0, width=W, height=H)
    r0, r1 = rows if rows else (0, H)
    seed = rng.normal(size=(r1 - r0, W, 4)).astype(np.float32)
    (img_o,), (out,) = _oracle(vol, tex, [view], dt, [seed.astype(np.float64)],
                               ["volume", "tf", "camera", "stepsize"]) if rows is None else \
        _band_oracle(vol, tex, view, dt, seed, rows)
    dens = torch.from_numpy(vol).to(cuda)
    tx = torch.from_numpy(tex).to(cuda)
    cams = R.camera_array(torch.tensor([[lon, lat]], dtype=torch.float64, device=cuda), radius,
                          (0.0, 0.0, 0.0), 35.0)
    rig = R.Rig(W, H, rows=rows)
    for cells in (R.pack_cells(dens), None):
        img, trans = R.forward(dens, tx, cams, dt, rig, cells=cells)
        assert rel_l2(img[0].cpu().numpy(), img_o) <= 1e-5, case
        d = {k: torch.zeros(s, dtype=dt_, device=cuda) for k, s, dt_ in
             (("volume", dens.shape, torch.float32), ("tf", tx.shape, torch.float64),
              ("camera", (1, 2), torch.float64), ("stepsize", (1,), torch.float64))}
        R.adjoint(dens, tx, cams, dt, rig, img, trans,
                  torch.from_numpy(seed).to(cuda)[None].contiguous(), 15, d_volume=d["volume"],
                  d_tf=d["tf"], d_camera=d["camera"], d_dt=d["stepsize"], cells=cells)
        for k in d:
            ref = np.asarray(out["d_" + k], np.float64)
            got = d[k].double().cpu().numpy().reshape(ref.shape)
            if np.linalg.norm(ref) == 0:
                assert np.abs(got).max() == 0.0
            else:
                assert rel_l2(got, ref) <= GRAD_BAR.get(case, 1e-4), (case, k, rel_l2(got, ref))


def _band_oracle(vol, tex, view, dt, seed, rows):
    from oracle import dvr_oracle as O
    g = O.Grid(vol.astype(np.float64))
    img = O.render_view(g, tex.astype(np.float64), view, dt, rows=rows)
    out = O.adjoint_view(g, tex.astype(np.float64), view, dt, seed.astype(np.float64),
                         ["volume", "tf", "camera", "stepsize"], image=img, rows=rows)
    return (img,), (out,)


def test_full_c4_properties(cuda):
    """All 64 views of C4 at full size: counts, finiteness, linearity, layouts, view sums."""
    torch = _t()
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.scenes import CONFIGS
    c = CONFIGS["C4"]
    dens = torch.from_numpy(c.volume()).to(cuda)
    tex = torch.from_numpy(c.texels().astype(np.float32)).to(cuda)
    ll = torch.tensor(c.view_poses(), dtype=torch.float64, device=cuda)
    cams = R.camera_array(ll, c.radius, (0.0, 0.0, 0.0), c.fov)
    rig = R.Rig(c.image, c.image)
    cells = R.pack_cells(dens)
    img, trans = R.forward(dens, tex, cams, c.dt, rig, cells=cells)
    assert torch.isfinite(img).all() and bool((img[..., 3] >= 0).all())
    assert bool((img[..., 3] < 1).all())
    g = torch.Generator(device=cuda).manual_seed(0)
    s1 = torch.randn(img.shape, generator=g, device=cuda)
    s2 = torch.randn(img.shape, generator=g, device=cuda)

    def adj(seed, cells_=cells, views=None):
        out = torch.zeros_like(dens)
        if views is None:
            R.adjoint(dens, tex, cams, c.dt, rig, img, trans, seed, 8, d_volume=out, cells=cells_)
        else:
            for v in views:
                R.adjoint(dens, tex, cams[v:v + 1].contiguous(), c.dt, rig, img[v:v + 1],
                          trans[v:v + 1], seed[v:v + 1].contiguous(), 8, d_volume=out,
                          cells=cells_)
        return out

    a1, a2, a12 = adj(s1), adj(s2), adj((s1 + s2).contiguous())
    assert torch.isfinite(a12).all()
    lin = float((a12 - a1 - a2).norm() / a12.norm())
    assert lin <= 1e-5, lin                              # linear in the seed
    vox = adj(s1, None)
    assert float((vox - a1).norm() / a1.norm()) <= 1e-5  # both layouts agree
    per_view = adj(s1, views=range(64))
    assert float((per_view - a1).norm() / a1.norm()) <= 1e-5   # view sum == one launch
    again = adj(s1)
    assert float((again - a1).norm() / a1.norm()) <= 1e-6      # atomic-order spread


def test_inversion_matches_stored_on_saturating_rays(cuda):
    """Dense rays (final T ~ 1e-6): the fp32 transmittance inversion vs the tape."""
    torch = _t()
    from paper_2107_12672_b200 import raymarch as R
    rng = np.random.default_rng(2)
    vol = rng.uniform(0.3, 0.9, (32, 32, 32)).astype(np.float32)
    tex = np.tile([0.6, 0.4, 0.3, 12.0], (16, 1)).astype(np.float32)
    tex[:, 3] *= np.linspace(0.5, 1.0, 16)
    dens = torch.from_numpy(vol).to(cuda)
    tx = torch.from_numpy(tex).to(cuda)
    cams = R.camera_array(torch.tensor([[40.0, 30.0]], dtype=torch.float64, device=cuda), 2.0,
                          (0.0, 0.0, 0.0), 30.0)
    rig = R.Rig(48, 48)
    dt = 1.0 / 128
    _, n, _ = R.ray_setup(cams, dt, rig)
    stride = int(n.max().item())
    tape = torch.empty(48 * 48 * stride, device=cuda)
    img, trans = R.forward(dens, tx, cams, dt, rig, tape=tape, tape_stride=stride)
    assert float(torch.exp(-trans).min()) < 1e-5        # really saturating (trans = depth)
    seed = torch.randn(img.shape, device=cuda)
    out = {}
    for mode in ("inversion", "stored"):
        d = torch.zeros_like(dens)
        dtf = torch.zeros(tx.shape, dtype=torch.float64, device=cuda)
        kw = dict(tape=tape, tape_stride=stride) if mode == "stored" else {}
        R.adjoint(dens, tx, cams, dt, rig, img, trans, seed, 12, d_volume=d, d_tf=dtf, **kw)
        out[mode] = (d, dtf)
    for a, b in zip(out["inversion"], out["stored"]):
        assert float((a - b).norm() / b.norm()) <= 1e-4


@pytest.mark.parametrize("kind", ["piecewise", "gaussian", "piecewise_uniform"])
def test_analytic_tf_modes_match_oracle(cuda, kind):
    """Piecewise-linear (K,5) and Gaussian (G,6) TFs: forward + every gradient vs the oracle."""
    torch = _t()
    from oracle import dvr_oracle as O
    from paper_2107_12672_b200 import raymarch as R
    rng = np.random.default_rng(21)
    vol = rng.uniform(0.05, 0.95, (9, 8, 10)).astype(np.float32)
    if kind == "gaussian":
        G = 3
        params = np.column_stack([rng.uniform(0.2, 0.8, G), rng.uniform(0.08, 0.3, G),
                                  rng.uniform(0.1, 1.0, (G, 3)), rng.uniform(0.5, 4.0, G)])
        tf_o = O.GaussianTF(params.astype(np.float32).astype(np.float64))
    else:
        K = 7
        pos = (np.arange(K) + 0.5) / K if kind == "piecewise_uniform" else \
            np.sort(rng.uniform(0.05, 0.95, K))
        params = np.column_stack([pos, rng.uniform(0.05, 1, (K, 3)), rng.uniform(0.3, 2.0, K)])
        tf_o = O.PiecewiseTF(params.astype(np.float32).astype(np.float64))
    params = params.astype(np.float32)
    view = O.View(50.0, -20.0, 2.2, fov_y_deg=35.0, width=10, height=9)
    dt = 0.05
    seed = rng.normal(size=(9, 10, 4))
    g = O.Grid(vol.astype(np.float64))
    img_o = O.render_view(g, tf_o, view, dt)
    ref = O.adjoint_view(g, tf_o, view, dt, seed, ["tf", "volume", "camera", "stepsize"],
                         image=img_o)
    dens = torch.from_numpy(vol).to(cuda)
    tx = torch.from_numpy(params).to(cuda).contiguous()
    cams = R.camera_array(torch.tensor([[50.0, -20.0]], dtype=torch.float64, device=cuda), 2.2,
                          (0.0, 0.0, 0.0), 35.0)
    rig = R.Rig(10, 9)
    for cells in (R.pack_cells(dens), None):
        img, depth = R.forward(dens, tx, cams, dt, rig, cells=cells)
        assert rel_l2(img[0].cpu().numpy(), img_o) <= 1e-5, kind
        d = {"volume": torch.zeros_like(dens),
             "tf": torch.zeros(tx.shape, dtype=torch.float64, device=cuda),
             "camera": torch.zeros(1, 2, dtype=torch.float64, device=cuda),
             "stepsize": torch.zeros(1, dtype=torch.float64, device=cuda)}
        R.adjoint(dens, tx, cams, dt, rig, img, depth,
                  torch.from_numpy(seed.astype(np.float32)).to(cuda)[None].contiguous(), 15,
                  d_volume=d["volume"], d_tf=d["tf"], d_camera=d["camera"], d_dt=d["stepsize"],
                  cells=cells)
        for k, v in d.items():
            r_ = np.asarray(ref["d_" + k], np.float64)
            assert rel_l2(v.double().cpu().numpy().reshape(r_.shape), r_) <= 1e-4, (kind, k)
    if kind == "piecewise_uniform":   # equals the texel table on the GPU too
        tex = torch.from_numpy(params[:, 1:].copy()).to(cuda)
        img_t, _ = R.forward(dens, tex, cams, dt, rig)
        assert rel_l2(img.cpu().numpy(), img_t.cpu().numpy()) <= 1e-6


def test_cell_records_are_the_trilinear_polynomial(cuda):
    """ddvr_pack_cells: padded, edge-clamped records of the polynomial
    coefficients {c0, cx, cy, cxy, cz, cxz, cyz, cxyz} (the monomial of corner
    bit b = bx | by << 1 | bz << 2 at index b) in u = f - 1/2; the polynomial
    equals the reference's lerp form (field.py:318-349)."""
    torch = _t()
    from paper_2107_12672_b200 import raymarch as R
    rng = np.random.default_rng(5)
    vol = rng.uniform(0, 1, (5, 4, 3)).astype(np.float32)
    cells = R.pack_cells(torch.from_numpy(vol).to(cuda)).cpu().numpy().astype(np.float64)
    X, Y, Z = vol.shape
    rec = cells.reshape(X + 1, Y + 1, Z + 1, 8)
    v64 = vol.astype(np.float64)
    s = np.array([[(1 if b & 1 << a else -1) for a in range(3)] for b in range(8)], np.float64)
    for i in range(-1, X):
        for j in range(-1, Y):
            for k in range(-1, Z):
                corner = np.array([v64[min(max(i + (b & 1), 0), X - 1),
                                       min(max(j + (b >> 1 & 1), 0), Y - 1),
                                       min(max(k + (b >> 2 & 1), 0), Z - 1)] for b in range(8)])
                want = np.array([corner.sum() / 8,
                                 (s[:, 0] * corner).sum() / 4, (s[:, 1] * corner).sum() / 4,
                                 (s[:, 0] * s[:, 1] * corner).sum() / 2,
                                 (s[:, 2] * corner).sum() / 4,
                                 (s[:, 0] * s[:, 2] * corner).sum() / 2,
                                 (s[:, 1] * s[:, 2] * corner).sum() / 2,
                                 (s[:, 0] * s[:, 1] * s[:, 2] * corner).sum()])
                got = rec[i + 1, j + 1, k + 1]
                np.testing.assert_allclose(got, want, atol=4e-7)
                for _ in range(3):   # polynomial == x-then-y-then-z lerps
                    f = rng.uniform(0, 1, 3)
                    ux, uy, uz = f - 0.5
                    poly = (got[0] + got[1] * ux + got[2] * uy + got[3] * ux * uy + got[4] * uz
                            + got[5] * ux * uz + got[6] * uy * uz + got[7] * ux * uy * uz)
                    a = [corner[b] + f[0] * (corner[b + 1] - corner[b]) for b in (0, 2, 4, 6)]
                    p0 = a[0] + f[1] * (a[1] - a[0])
                    p1 = a[2] + f[1] * (a[3] - a[2])
                    assert abs(poly - (p0 + f[2] * (p1 - p0))) < 1e-6
                # a replicated (clamped) axis has exactly zero odd coefficients
                if i in (-1, X - 1):
                    assert got[1] == got[3] == got[5] == got[7] == 0.0


@pytest.mark.parametrize("tau_scale,dt,shape", [(3.0, 0.02, "ramp"), (60.0, 0.02, "ramp"),
                                                (4000.0, 0.05, "ramp"), (3.0, 0.02, "bent"),
                                                (60.0, 0.02, "bent")])
@pytest.mark.parametrize("with_step", [True, False])
def test_absorption_only_walk_matches_oracle(cuda, tau_scale, dt, shape, with_step):
    """Emission-free TF, volume + camera + stepsize targets: the adjoint's
    closed-form absorption walk (tau_hat = dt seed_a T_n per ray) against the
    oracle's inversion walk.  The three scales select the degree-3, degree-7
    and general opacity modes; the last has clamped segments (a > 1 - EPS).
    "ramp" is affine in the texel index (the march evaluates it without the
    table), "bent" (tau ~ k^2) is not (the table path); without the stepsize
    target a ramp in a polynomial mode takes the table-free walk."""
    torch = _t()
    from oracle import dvr_oracle as O
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.scenes import absorption_ramp_texels
    rng = np.random.default_rng(11)
    vol = rng.uniform(0.0, 1.0, (9, 8, 7)).astype(np.float32)
    tex = absorption_ramp_texels(32, tau_scale).astype(np.float32)
    if shape == "bent":
        tex[:, 3] = (tau_scale * (np.arange(32) / 31.0) ** 2).astype(np.float32)
    view = O.View(47.0, -18.0, 2.0, fov_y_deg=40.0, width=11, height=9)
    seed = rng.normal(size=(9, 11, 4)).astype(np.float32)
    targets = ["volume", "camera", "stepsize"] if with_step else ["volume", "camera"]
    (img_o,), (out,) = _oracle(vol, tex, [view], dt, [seed.astype(np.float64)], targets)
    if tau_scale > 1000:   # the case must exercise the EPS clamp
        assert img_o[..., 3].max() > 1 - 2e-6
    dens = torch.from_numpy(vol).to(cuda)
    tx = torch.from_numpy(tex).to(cuda)
    cams = R.camera_array(torch.tensor([[47.0, -18.0]], dtype=torch.float64, device=cuda), 2.0,
                          (0.0, 0.0, 0.0), 40.0)
    rig = R.Rig(11, 9)
    for cells in (R.pack_cells(dens), None):
        img, depth = R.forward(dens, tx, cams, dt, rig, cells=cells)
        assert rel_l2(img[0].cpu().numpy(), img_o) <= 1e-5
        d = {"volume": torch.zeros_like(dens),
             "camera": torch.zeros(1, 2, dtype=torch.float64, device=cuda),
             "stepsize": torch.zeros(1, dtype=torch.float64, device=cuda)}
        R.adjoint(dens, tx, cams, dt, rig, img, depth,
                  torch.from_numpy(seed).to(cuda)[None].contiguous(), 11 if with_step else 9,
                  d_volume=d["volume"], d_camera=d["camera"],
                  d_dt=d["stepsize"] if with_step else None, cells=cells)
        for k in targets:
            ref = np.asarray(out["d_" + k], np.float64)
            got = d[k].double().cpu().numpy().reshape(ref.shape)
            assert rel_l2(got, ref) <= 1e-4, (tau_scale, k, rel_l2(got, ref))


def test_gather_probe_checksums(cuda):
    """ddvr_gather_probe (the gather-roofline microbenchmark): the held and the
    per-sample gathers read the same records, so the per-ray checksums agree."""
    torch = _t()
    from paper_2107_12672_b200 import raymarch as R
    rng = np.random.default_rng(3)
    dens = torch.from_numpy(rng.uniform(0, 1, (20, 18, 16)).astype(np.float32)).to(cuda)
    cams = R.camera_array(torch.tensor([[20.0, 10.0], [200.0, -40.0]], dtype=torch.float64,
                                       device=cuda), 2.0, (0.0, 0.0, 0.0), 30.0)
    cells = R.pack_cells(dens)
    a = R.gather_probe(dens, cams, 0.01, R.Rig(24, 20), cells, hold=True)
    b = R.gather_probe(dens, cams, 0.01, R.Rig(24, 20), cells, hold=False)
    assert torch.equal(a, b) and float(a.abs().sum()) > 0
