"""The CPU oracle (oracle/dvr_oracle.py) pinned against the reference's own outputs.

tests/golden/*.npz were produced by oracle/gen_golden.py running the reference
(voldiff, /root/reference) on fp32-representable inputs.  The oracle is a
restatement in fp64, so agreement is to round-off (<= 1e-9 relative, max norm).
Also re-checks the reference's own known-answer tests against the fixtures.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, golden_names, rel_max
from oracle import dvr_oracle as O

TOL = 1e-9
SCENES = golden_names("kat_") + golden_names("rand_")


def _scene(g):
    lon, lat, radius, cx, cy, cz, fov, W, H = g["cam"]
    grid = O.Grid(g["volume"].astype(np.float64), g["box"][0], g["box"][1])
    view = O.View(lon, lat, radius, (cx, cy, cz), fov, int(W), int(H))
    return grid, view, g["texels"].astype(np.float64), float(g["dt"])


@pytest.mark.parametrize("name", SCENES)
def test_oracle_render(name):
    g = golden(name)
    grid, view, tex, dt = _scene(g)
    img = O.render_view(grid, tex, view, dt)
    assert rel_max(img, g["image"]) <= TOL
    if "image_none" in g:
        assert rel_max(O.render_view(grid, tex, view, dt, early_stop=True), g["image_none"]) <= TOL
    band = O.make_band(grid, view, dt)
    np.testing.assert_array_equal(band.n, g["n_steps"].ravel())


@pytest.mark.parametrize("name", SCENES)
@pytest.mark.parametrize("mode", ["inversion", "stored"])
def test_oracle_adjoint(name, mode):
    g = golden(name)
    keys = [k for k in g if k.startswith(mode + "_") and not k.endswith("state_floats")]
    if not keys:
        pytest.skip("no fixtures for this mode")
    grid, view, tex, dt = _scene(g)
    targets = [k.split("_", 1)[1] for k in keys]
    out = O.adjoint_view(grid, tex, view, dt, g["seed"], targets, stored=(mode == "stored"))
    for t in targets:
        got = np.asarray(out["d_" + t], np.float64).ravel()
        ref = np.asarray(g[f"{mode}_{t}"], np.float64).ravel()
        if np.abs(ref).max() == 0.0:
            assert np.abs(got).max() == 0.0
        else:
            assert rel_max(got, ref) <= TOL, (t, rel_max(got, ref))


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_oracle_config_band(name):
    from paper_2107_12672_b200.scenes import CONFIGS
    g = golden(name)
    c = CONFIGS[name]
    vol = c.volume().astype(np.float64)
    np.testing.assert_array_equal(vol.reshape(-1)[:: max(1, vol.size // 4096)], g["volume_probe"])
    lon, lat, radius, cx, cy, cz, fov, W, H = g["cam"]
    grid = O.Grid(vol)
    view = O.View(lon, lat, radius, (cx, cy, cz), fov, int(W), int(H))
    r0, r1 = (int(r) for r in g["rows"])
    band = O.make_band(grid, view, c.dt, r0, r1)
    np.testing.assert_array_equal(band.n, g["n_steps"])
    img = O.render_view(grid, g["texels"].astype(np.float64), view, c.dt, rows=(r0, r1))
    assert rel_max(img, g["image"]) <= TOL
    targets = sorted({k.split("_")[1] for k in g if k.startswith("inversion_")})
    out = O.adjoint_view(grid, g["texels"].astype(np.float64), view, c.dt, g["seed_band"], targets,
                         image=g["image"], rows=(r0, r1))
    for t in targets:
        if t == "volume" and "inversion_volume_idx" in g:
            ref = np.zeros(vol.size)
            ref[g["inversion_volume_idx"]] = g["inversion_volume_val"]
        else:
            ref = g[f"inversion_{t}"]
        assert rel_max(out["d_" + t], ref) <= TOL, t


def test_sample_totals():
    """C1..C3 exact sample totals from the oracle's step counts."""
    from paper_2107_12672_b200.scenes import CONFIGS
    counts = golden("counts")
    for name in ("C1", "C2", "C3"):
        c = CONFIGS[name]
        grid = O.Grid(np.zeros((2, 2, 2)))
        total = 0
        for lon, lat in c.view_poses():
            view = O.View(lon, lat, c.radius, fov_y_deg=c.fov, width=c.image, height=c.image)
            total += int(O.make_band(grid, view, c.dt).n.sum())
        assert total == int(counts[name + "_samples"])
    assert int(counts["C4_samples"]) == 18_081_633_464
    assert int(counts["C5_samples"]) == 289_327_888_092


# --- the reference's own known answers, re-checked on the fixtures -------------


def test_kat_transparency():
    """1 - alpha = exp(-tau0 * chord) at the centre pixel (test_renderer.py:105-112)."""
    for tau0 in (0.1, 1.0, 10.0):
        g = golden(f"kat_transparency_{tau0:g}")
        tau_f32 = float(np.float32(tau0))
        assert abs((1.0 - g["image"][4, 4, 3]) - np.exp(-tau_f32)) < 1e-5


def test_kat_emission_closed_form():
    """c0 (1 - e^{-tau0}) exactly at any stepsize (test_renderer.py:114-122)."""
    g = golden("kat_emission")
    c0, tau0 = float(np.float32(0.7)), 2.0
    assert abs(g["image"][4, 4, 0] - c0 * (1.0 - np.exp(-tau0))) < 1e-10


def test_kat_empty_and_untouched():
    g = golden("kat_empty")
    assert np.abs(g["image"]).max() == 0.0
    u = golden("kat_untouched")["inversion_volume"]
    assert u[0, 0, 0] == 0.0 and u[-1, -1, -1] == 0.0 and np.any(u != 0.0)


def test_inversion_equals_stored_in_fixtures():
    """renderer.py inversion == stored (test_renderer.py:200-214) on the fixtures."""
    for name in golden_names("rand_"):
        g = golden(name)
        for t in ("tf", "volume", "camera", "stepsize"):
            assert rel_max(g[f"inversion_{t}"], g[f"stored_{t}"]) < 1e-5


@pytest.mark.parametrize("key", ["a", "b", "c"])
def test_oracle_color_volume(key):
    """render_colorvol / render_colorvol_adjoint (renderer.py:404-407, 703-709)."""
    g = golden("color")
    lon, lat, radius, cx, cy, cz, fov, W, H = g[f"{key}_cam"]
    cg = O.ColorGrid(g[f"{key}_values"].astype(np.float64), g[f"{key}_box"][0],
                     g[f"{key}_box"][1])
    view = O.View(lon, lat, radius, (cx, cy, cz), fov, int(W), int(H))
    dt = float(g[f"{key}_dt"])
    assert rel_max(O.render_color_view(cg, view, dt), g[f"{key}_image"]) <= TOL
    assert rel_max(O.render_color_view(cg, view, dt, early_stop=True),
                   g[f"{key}_image_none"]) <= TOL
    for mode in ("inversion", "stored"):
        got = O.adjoint_color_view(cg, view, dt, g[f"{key}_seed"], stored=(mode == "stored"))
        assert rel_max(got, g[f"{key}_{mode}_d_color"]) <= TOL


# --- point-wise field functions (tests/golden/fields.npz, field.py:186-600) ---


@pytest.mark.parametrize("name", ["a", "b"])
def test_oracle_trilinear(name):
    g = golden("fields")
    grid = O.Grid(g[f"vol_{name}"], g[f"box_{name}"][0], g[f"box_{name}"][1])
    pts = g[f"pts_{name}"]
    d, sp, w, idx = grid.density_and_grads(pts.T)
    np.testing.assert_array_equal(idx, g[f"corners_{name}"])
    assert rel_max(d, g[f"value_{name}"]) <= 1e-14
    assert rel_max(grid.density(pts.T), g[f"value_{name}"]) <= 1e-14
    assert rel_max(w, g[f"weights_{name}"]) <= 1e-14
    assert rel_max(sp, g[f"spatial_{name}"]) <= 1e-14


@pytest.mark.parametrize("R", [1, 2, 8])
def test_oracle_tf(R):
    g = golden("fields")
    out, slope, (i0, i1), (w0, w1) = O.tf_eval(g[f"tf{R}"], g[f"d{R}"])
    np.testing.assert_array_equal(out, g[f"tfs{R}"])
    np.testing.assert_array_equal(slope, g[f"slope{R}"])
    np.testing.assert_array_equal(np.stack([i0, i1], -1), g[f"ti{R}"])
    np.testing.assert_array_equal(np.stack([w0, w1], -1), g[f"tw{R}"])


def test_oracle_opacity():
    g = golden("fields")
    for k in (0, 1):
        dt = float(g[f"odt{k}"])
        tau, e, a, clamped = O.segment_opacity(g["tau"], dt)
        live = g["tau"] >= 0.0          # the oracle folds the renderer's max(tau, 0)
        np.testing.assert_array_equal(a[live], g[f"alpha{k}"][live])
        np.testing.assert_array_equal(np.where(clamped, 0.0, dt * e)[live], g[f"dalpha{k}"][live])


@pytest.mark.parametrize("k", [0, 1, 2])
def test_oracle_camera(k):
    g = golden("fields")
    c = g[f"cam{k}"]
    view = O.View(c[0], c[1], c[2], tuple(c[3:6]), c[6], int(c[7]), int(c[8]))
    o, d = O.pixel_rays(view, g[f"u{k}"], g[f"v{k}"])
    np.testing.assert_array_equal(o.T, g[f"origin{k}"])
    np.testing.assert_array_equal(d.T, g[f"dir{k}"])
    jo, jd = O.camera_jacobians(view, g[f"u{k}"], g[f"v{k}"])
    assert rel_max(np.broadcast_to(jo, g[f"jo{k}"].shape), g[f"jo{k}"]) <= 1e-12
    assert rel_max(np.moveaxis(jd, 0, 1), g[f"jd{k}"]) <= 1e-12
