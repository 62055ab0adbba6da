"""Piecewise-linear and Gaussian TF modes of the CPU oracle (no reference exists).

SURVEY.md 8c: the reference only has the texel table.  These two modes are
restated from its conventions and pinned here by (a) exact equivalence of the
piecewise-linear TF on uniform knots (r+0.5)/R with the reference-pinned texel
path, (b) central finite differences of the oracle's own fp64 render for every
TF parameter, and (c) the reference's 1-D Gaussian demo optical model
(tasks.py:751-766).  Parity of these modes is therefore "unpinned" against
the reference itself; DESIGN.md says so.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_max
from oracle import dvr_oracle as O


def _scene(seed=3):
    rng = np.random.default_rng(seed)
    grid = O.Grid(rng.uniform(0.1, 0.9, (7, 7, 7)))
    view = O.View(35.0, 25.0, 2.3, width=7, height=6)
    return rng, grid, view, 0.06


def test_piecewise_uniform_knots_equal_texels():
    rng, grid, view, dt = _scene()
    R = 9
    tex = np.column_stack([rng.uniform(0.05, 1, (R, 3)), rng.uniform(0.3, 2.0, R)])
    pl = O.PiecewiseTF(np.column_stack([(np.arange(R) + 0.5) / R, tex]))
    img_t = O.render_view(grid, tex, view, dt)
    img_p = O.render_view(grid, pl, view, dt)
    assert rel_max(img_p, img_t) < 1e-12
    seed = rng.normal(size=img_t.shape)
    gt = O.adjoint_view(grid, tex, view, dt, seed, ["tf", "volume", "camera"], image=img_t)
    gp = O.adjoint_view(grid, pl, view, dt, seed, ["tf", "volume", "camera"], image=img_p)
    assert rel_max(gp["d_volume"], gt["d_volume"]) < 1e-10
    assert rel_max(gp["d_camera"], gt["d_camera"]) < 1e-10
    assert rel_max(gp["d_tf"][:, 1:], gt["d_tf"]) < 1e-10


def _fd_check(tf_cls, params, rng, grid, view, dt, h=1e-6, tol=2e-4):
    seed = rng.normal(size=(view.height, view.width, 4))

    def loss(p):
        return float(np.sum(seed * O.render_view(grid, tf_cls(p), view, dt)))

    img = O.render_view(grid, tf_cls(params), view, dt)
    g = O.adjoint_view(grid, tf_cls(params), view, dt, seed, ["tf", "volume"], image=img)
    fd = np.zeros_like(params)
    for idx in np.ndindex(params.shape):
        e = np.zeros_like(params)
        e[idx] = h
        fd[idx] = (loss(params + e) - loss(params - e)) / (2 * h)
    assert rel_max(g["d_tf"], fd, floor=1e-9) < tol, np.abs(g["d_tf"] - fd).max()
    # density gradient through the analytic TF slope
    k = (3, 2, 4)
    e = np.zeros_like(grid.values)
    e[k] = h
    plus = O.Grid(grid.values + e)
    minus = O.Grid(grid.values - e)
    fdv = (float(np.sum(seed * O.render_view(plus, tf_cls(params), view, dt)))
           - float(np.sum(seed * O.render_view(minus, tf_cls(params), view, dt)))) / (2 * h)
    assert abs(g["d_volume"][k] - fdv) <= tol * max(abs(fdv), 1e-6)


def test_piecewise_gradients_match_finite_differences():
    rng, grid, view, dt = _scene(5)
    K = 6
    pos = np.sort(rng.uniform(0.05, 0.95, K))
    vals = np.column_stack([rng.uniform(0.05, 1, (K, 3)), rng.uniform(0.3, 2.0, K)])
    _fd_check(O.PiecewiseTF, np.column_stack([pos, vals]), rng, grid, view, dt)


def test_gaussian_gradients_match_finite_differences():
    rng, grid, view, dt = _scene(7)
    G = 3
    params = np.column_stack([rng.uniform(0.2, 0.8, G), rng.uniform(0.08, 0.3, G),
                              rng.uniform(0.1, 1.0, (G, 3)), rng.uniform(0.5, 4.0, G)])
    _fd_check(O.GaussianTF, params, rng, grid, view, dt)


def test_gaussian_matches_reference_demo_model():
    """tasks.py:751-766: g = exp(-d^2/2s^2), tau = tau_s g, emission g, opacity-weighted."""
    s2, tau_s = 0.5, 3.0
    tf = O.GaussianTF(np.array([[0.0, np.sqrt(s2), 1.0, 1.0, 1.0, tau_s]]))
    d = np.linspace(0.0, 1.0, 11)
    out = tf.eval(d)[0]
    g = np.exp(-d * d / (2 * s2))
    np.testing.assert_allclose(out, np.column_stack([g, g, g, tau_s * g]), rtol=1e-14)


@pytest.mark.parametrize("K", [1, 2])
def test_piecewise_degenerate_knot_counts(K):
    rng, grid, view, dt = _scene(9)
    params = np.column_stack([np.linspace(0.3, 0.7, K), rng.uniform(0.1, 1.0, (K, 4))])
    img = O.render_view(grid, O.PiecewiseTF(params), view, dt)
    assert np.all(np.isfinite(img))
    if K == 1:   # constant TF: every sample sees the single knot's value
        tex = params[:, 1:]
        assert rel_max(img, O.render_view(grid, tex, view, dt)) < 1e-12
