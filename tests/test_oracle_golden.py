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
