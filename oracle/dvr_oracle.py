"""CPU oracle for the DiffDVR hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The shipped path
(``paper_2107_12672_b200``) never imports anything under ``oracle/``.

What it is: an fp64 NumPy restatement of the reference package ``voldiff``
(arXiv 2107.12672, "DiffDVR"; pure Python, /root/reference/pkg/src/voldiff)
for the functions on the hot path -- camera rays, slab clipping, step counts,
trilinear sampling and its gradients, the texel transfer function, the
front-to-back march, and the adjoint walk with the inversion trick, for the
targets ``tf``, ``volume``, ``camera`` and ``stepsize``.  Each function cites
the reference lines whose semantics it follows.

Parity is PINNED: ``tests/test_oracle_golden.py`` checks this module against
``tests/golden/*.npz``, which ``oracle/gen_golden.py`` produced by running the
reference itself (imported from /root/reference in the build container).

The structure differs from the reference on purpose: rays of a row band are
processed as one vector (no 64-row tile pool), several targets are produced in
one backward walk, and per-view results are returned as plain arrays.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

EPS_ALPHA = 1e-6            # field.py:25
EPS_POLE_DEG = 1e-3         # field.py:24
ALPHA_STOP = 1.0 - 1e-4     # renderer.py:45
STEP_EPS = 1e-9             # renderer.py:212
_DEG = math.pi / 180.0      # field.py:27

TARGETS = ("camera", "stepsize", "tf", "volume")


# ---------------------------------------------------------------------------
# camera (field.py:130-156, 186-271)
# ---------------------------------------------------------------------------


@dataclass
class View:
    """One spherical pinhole camera (mirrors SphericalCamera, field.py:130-156)."""

    lon_deg: float
    lat_deg: float
    radius: float
    center: tuple = (0.0, 0.0, 0.0)
    fov_y_deg: float = 30.0
    width: int = 64
    height: int = 64

    def __post_init__(self):
        self.lon_deg = float(self.lon_deg) % 360.0            # field.py:143
        self.lat_deg = float(self.lat_deg)
        self.radius = float(self.radius)
        self.center = tuple(float(c) for c in np.asarray(self.center).reshape(3))
        if abs(self.lat_deg) >= 90.0 - EPS_POLE_DEG:          # field.py:147
            raise ValueError("pole exclusion")
        if self.radius <= 0.0 or not 0.0 < self.fov_y_deg < 180.0:
            raise ValueError("bad camera")


def _frame(view: View):
    """Eye, forward, right and up vectors (field.py:194-216), fp64.

    The arithmetic sequence follows the reference so directions agree to the
    last bit in practice (the step counts downstream are integer-exact).
    """
    lon = view.lon_deg * _DEG
    lat = view.lat_deg * _DEG
    cl, sl = math.cos(lat), math.sin(lat)
    cp, sp = math.cos(lon), math.sin(lon)
    cx, cy, cz = view.center
    eye = np.array([cx + view.radius * (cl * cp), cy + view.radius * sl,
                    cz + view.radius * (cl * sp)])
    fx, fy, fz = -(cl * cp), -sl, -(cl * sp)
    fn = math.sqrt(fx * fx + fy * fy + fz * fz)
    fx, fy, fz = fx / fn, fy / fn, fz / fn
    rx, rz = -fz, fx
    rn = math.sqrt(rx * rx + rz * rz)
    rx, rz = rx / rn, rz / rn
    up = np.array([-(rz * fy), rz * fx - rx * fz, rx * fy])
    return eye, np.array([fx, fy, fz]), np.array([rx, 0.0, rz]), up


def _screen(view: View, u, v):
    """Pixel-centre screen offsets (field.py:218-222)."""
    th = math.tan(0.5 * view.fov_y_deg * _DEG)
    su = ((np.asarray(u, np.float64) + 0.5) * (2.0 / view.width) - 1.0) * th * (
        view.width / view.height)
    sv = (1.0 - (np.asarray(v, np.float64) + 0.5) * (2.0 / view.height)) * th
    return su, sv


def pixel_rays(view: View, u, v):
    """Origins (3,n) and unit directions (3,n) through pixel centres (field.py:224-228)."""
    eye, f, r, up = _frame(view)
    su, sv = _screen(view, u, v)
    dx = f[0] + r[0] * su + up[0] * sv
    dy = f[1] + up[1] * sv
    dz = f[2] + r[2] * su + up[2] * sv
    dn = np.sqrt(dx * dx + dy * dy + dz * dz)
    n = np.shape(su)[0]
    o = np.repeat(eye[:, None], n, axis=1)
    return o, np.stack([dx / dn, dy / dn, dz / dn])


def camera_jacobians(view: View, u, v):
    """d(origin)/d(lon,lat) (3,2) and d(direction)/d(lon,lat) (3,n,2), per degree.

    Analytic derivative of the parameterisation that the reference evaluates
    over dual numbers (field.py:253-271).  With r = (sin lon, 0, -cos lon) and
    up = (-cos lon sin lat, cos lat, -sin lon sin lat) after normalisation.
    """
    lon = view.lon_deg * _DEG
    lat = view.lat_deg * _DEG
    cl, sl = math.cos(lat), math.sin(lat)
    cp, sp = math.cos(lon), math.sin(lon)
    rho = view.radius
    j_o = np.array([[-rho * cl * sp, -rho * sl * cp],
                    [0.0, rho * cl],
                    [rho * cl * cp, -rho * sl * sp]]) * _DEG
    df = np.array([[cl * sp, sl * cp], [0.0, -cl], [-cl * cp, sl * sp]]) * _DEG
    dr = np.array([[cp, 0.0], [0.0, 0.0], [sp, 0.0]]) * _DEG
    du = np.array([[sp * sl, -cp * cl], [0.0, -sl], [-cp * sl, -sp * cl]]) * _DEG
    _, f, r, up = _frame(view)
    su, sv = _screen(view, u, v)
    raw = f[:, None] + r[:, None] * su[None, :] + up[:, None] * sv[None, :]
    nrm = np.sqrt(np.sum(raw * raw, axis=0))
    d = raw / nrm
    j_d = np.empty((3, raw.shape[1], 2))
    for j in range(2):
        draw = df[:, j, None] + dr[:, j, None] * su[None, :] + du[:, j, None] * sv[None, :]
        proj = np.sum(d * draw, axis=0)
        j_d[:, :, j] = (draw - d * proj[None, :]) / nrm[None, :]
    return j_o, j_d


# ---------------------------------------------------------------------------
# ray / box clipping and step counts (renderer.py:182-214)
# ---------------------------------------------------------------------------


def clip_to_box(o, w, box_min, box_max):
    """(tn, tf, axis, clamped, miss) of rays against the box (renderer.py:182-206)."""
    bmin = np.asarray(box_min, np.float64)[:, None]
    bmax = np.asarray(box_max, np.float64)[:, None]
    with np.errstate(divide="ignore", invalid="ignore"):
        ta = (bmin - o) / w
        tb = (bmax - o) / w
    near = np.minimum(ta, tb)
    far = np.maximum(ta, tb)
    flat = w == 0.0
    inside = (o >= bmin) & (o <= bmax)
    near = np.where(flat, np.where(inside, -np.inf, np.inf), near)
    far = np.where(flat, np.where(inside, np.inf, -np.inf), far)
    axis = np.argmax(near, axis=0)
    tn = np.max(near, axis=0)
    tf_ = np.min(far, axis=0)
    clamped = tn <= 0.0
    tn = np.maximum(tn, 0.0)
    miss = ~(tf_ > tn) | ~np.isfinite(tn) | ~np.isfinite(tf_)
    return np.where(miss, 0.0, tn), np.where(miss, 0.0, tf_), axis, clamped, miss


def count_steps(tn, tf_, dt, miss):
    """n = ceil((tf - tn)/dt - 1e-9), >= 0, 0 on a miss (renderer.py:209-214)."""
    n = np.ceil((tf_ - tn) / dt - STEP_EPS).astype(np.int64)
    return np.where(miss, 0, np.maximum(n, 0))


# ---------------------------------------------------------------------------
# trilinear density (field.py:279-349, 379-500)
# ---------------------------------------------------------------------------


class Grid:
    """Voxel-centred grid over a world box; values (X,Y,Z), z fastest."""

    def __init__(self, values, box_min=(-0.5, -0.5, -0.5), box_max=(0.5, 0.5, 0.5)):
        self.values = np.asarray(values, np.float64)
        self.flat = self.values.reshape(-1)
        self.dims = self.values.shape
        self.bmin = np.asarray(box_min, np.float64).reshape(3)
        self.bmax = np.asarray(box_max, np.float64).reshape(3)
        self.scale = np.asarray(self.dims, np.float64) / (self.bmax - self.bmin)
        self.tol = 1e-9 * (self.bmax - self.bmin)           # field.py:293

    def _cell(self, pts):
        """Unclamped g, cell index, cell fraction, inside mask (field.py:279-308)."""
        g, idx, frac = [], [], []
        inside = np.ones(pts[0].shape, bool)
        for a in range(3):
            ga = (pts[a] - self.bmin[a]) * self.scale[a] - 0.5
            gc = np.clip(ga, 0.0, float(self.dims[a] - 1))
            ia = np.clip(np.floor(gc).astype(np.int64), 0, max(self.dims[a] - 2, 0))
            g.append(ga)
            idx.append(ia)
            frac.append(gc - ia)
            inside &= (pts[a] >= self.bmin[a] - self.tol[a]) & (pts[a] <= self.bmax[a] + self.tol[a])
        return g, idx, frac, inside

    def _corners(self, idx):
        """Flat indices of the 8 corners, x bit 0, y bit 1, z bit 2 (field.py:311-324)."""
        X, Y, Z = self.dims
        lo = idx
        hi = [np.minimum(idx[0] + 1, X - 1), np.minimum(idx[1] + 1, Y - 1),
              np.minimum(idx[2] + 1, Z - 1)]
        out = []
        for c in range(8):
            ix = hi[0] if c & 1 else lo[0]
            iy = hi[1] if c & 2 else lo[1]
            iz = hi[2] if c & 4 else lo[2]
            out.append((ix * Y + iy) * Z + iz)
        return np.stack(out, axis=-1)

    @staticmethod
    def _weights(frac):
        fx, fy, fz = frac
        wx = (1.0 - fx, fx)
        wy = (1.0 - fy, fy)
        wz = (1.0 - fz, fz)
        return np.stack([wx[c & 1] * wy[(c >> 1) & 1] * wz[(c >> 2) & 1] for c in range(8)],
                        axis=-1)

    def density(self, pts):
        """Clamped [0,1] density, 0 outside the box (field.py:336-349)."""
        _, idx, frac, inside = self._cell(pts)
        v = self.flat[self._corners(idx)]
        raw = np.sum(self._weights(frac) * v, axis=-1)
        return np.clip(np.where(inside, raw, 0.0), 0.0, 1.0)

    def density_and_grads(self, pts):
        """(d, spatial (n,3), w8 (n,8), idx8 (n,8)) as field.py:379-500 (clamp01 grid).

        ``spatial`` is the world-space gradient, zeroed per axis where the edge
        clamp froze the coordinate (field.py:459-484); spatial and w8 are zeroed
        where the sample is outside the box or the [0,1] clamp is active
        (field.py:486-499).
        """
        g, idx, frac, inside = self._cell(pts)
        idx8 = self._corners(idx)
        v = self.flat[idx8]
        w8 = self._weights(frac)
        raw = np.sum(w8 * v, axis=-1)
        fx, fy, fz = frac
        ex, ey, ez = 1.0 - fx, 1.0 - fy, 1.0 - fz
        # derivative along each axis: bilinear blend of the 4 edge differences
        ddx = (ey * ez * (v[:, 1] - v[:, 0]) + fy * ez * (v[:, 3] - v[:, 2])
               + ey * fz * (v[:, 5] - v[:, 4]) + fy * fz * (v[:, 7] - v[:, 6]))
        ddy = (ex * ez * (v[:, 2] - v[:, 0]) + fx * ez * (v[:, 3] - v[:, 1])
               + ex * fz * (v[:, 6] - v[:, 4]) + fx * fz * (v[:, 7] - v[:, 5]))
        ddz = (ex * ey * (v[:, 4] - v[:, 0]) + fx * ey * (v[:, 5] - v[:, 1])
               + ex * fy * (v[:, 6] - v[:, 2]) + fx * fy * (v[:, 7] - v[:, 3]))
        spatial = np.stack([
            ddx * np.where((g[0] >= 0.0) & (g[0] <= self.dims[0] - 1.0), self.scale[0], 0.0),
            ddy * np.where((g[1] >= 0.0) & (g[1] <= self.dims[1] - 1.0), self.scale[1], 0.0),
            ddz * np.where((g[2] >= 0.0) & (g[2] <= self.dims[2] - 1.0), self.scale[2], 0.0),
        ], axis=-1)
        live = (inside & (raw >= 0.0) & (raw <= 1.0)).astype(np.float64)
        d = np.clip(np.where(inside, raw, 0.0), 0.0, 1.0)
        return d, spatial * live[:, None], w8 * live[:, None], idx8


# ---------------------------------------------------------------------------
# texel transfer function (field.py:525-579, renderer.py:472-488)
# ---------------------------------------------------------------------------


def tf_eval(texels, d):
    """(out4 (n,4), slope (n,4), (i0,i1), (1-w, w)) of the texel lookup.

    Texel r is centred at (r+0.5)/R, linear in between, clamp-to-edge beyond
    (field.py:8-10, 540-549); the slope is zero in the clamp bands
    (field.py:575-576).
    """
    texels = np.asarray(texels, np.float64)
    R = texels.shape[0]
    dc = np.clip(d, 0.0, 1.0)
    t = dc * float(R) - 0.5
    f = np.clip(t, 0.0, float(R - 1))
    i0 = np.clip(np.floor(f).astype(np.int64), 0, max(R - 2, 0))
    i1 = np.minimum(i0 + 1, R - 1)
    w = f - i0
    out = (1.0 - w)[:, None] * texels[i0] + w[:, None] * texels[i1]
    live = (t >= 0.0) & (t <= R - 1.0) & (d >= 0.0) & (d <= 1.0)
    slope = (texels[i1] - texels[i0]) * float(R) * live[:, None]
    return out, slope, (i0, i1), (1.0 - w, w)


class PiecewiseTF:
    """Piecewise-linear TF on non-uniform knots: params (K,5) = [pos, r, g, b, tau].

    NO REFERENCE IMPLEMENTATION: restated from the texel TF's
    conventions (field.py:540-549, 575-576) -- linear between knots,
    clamp-to-edge outside [pos_0, pos_K-1], zero slope in the clamp bands.
    With knots at (r+0.5)/R it equals the R-texel table.  Gradients cover the
    knot values and positions.  Parity for this mode is unpinned (no reference);
    tests check it by the texel equivalence and by finite differences.
    """

    kind = "piecewise"

    def __init__(self, params):
        self.params = np.asarray(params, np.float64)
        self.pos = self.params[:, 0]
        self.val = self.params[:, 1:]

    def eval(self, d):
        K = self.pos.shape[0]
        d = np.clip(d, 0.0, 1.0)
        k = np.clip(np.searchsorted(self.pos, d, side="right") - 1, 0, max(K - 2, 0))
        k1 = np.minimum(k + 1, K - 1)
        span = self.pos[k1] - self.pos[k]
        inner = (d > self.pos[0]) & (d < self.pos[-1]) & (span > 0)
        w = np.where(inner, (d - self.pos[k]) / np.where(span > 0, span, 1.0), 0.0)
        w = np.where(d >= self.pos[-1], 1.0 if K > 1 else 0.0, w)
        out = (1.0 - w)[:, None] * self.val[k] + w[:, None] * self.val[k1]
        slope = np.where(inner[:, None],
                         (self.val[k1] - self.val[k]) / np.where(span > 0, span, 1.0)[:, None],
                         0.0)
        return out, slope, k, k1, w

    def grads(self, d, o4):
        """dL/dparams (K,5) of sum(o4 * eval(d)) (o4 (n,4) the output adjoint)."""
        out, slope, k, k1, w = self.eval(d)
        g = np.zeros_like(self.params)
        np.add.at(g[:, 1:], k, (1.0 - w)[:, None] * o4)
        np.add.at(g[:, 1:], k1, w[:, None] * o4)
        dh = np.sum(slope * o4, axis=1)              # d out / d d . o4 (0 in clamp bands)
        np.add.at(g[:, 0], k, dh * (w - 1.0))
        np.add.at(g[:, 0], k1, -dh * w)
        return g


class GaussianTF:
    """Analytic sum-of-Gaussians TF: params (G,6) = [mu, sigma, r, g, b, tau].

    out(d) = sum_j exp(-(d - mu_j)^2 / (2 sigma_j^2)) * (r_j, g_j, b_j, tau_j) on the
    clamped density.  NO REFERENCE IMPLEMENTATION: the optical model follows the
    reference's 1-D Gaussian demo (tasks.py:751-766: g = exp(-d^2/2sigma^2),
    tau = tau_s g, opacity-weighted emission g).  Parity unpinned; checked by
    finite differences and by that demo's closed form.
    """

    kind = "gaussian"

    def __init__(self, params):
        self.params = np.asarray(params, np.float64)

    def _g(self, d):
        mu, sg = self.params[:, 0], self.params[:, 1]
        z = (np.clip(d, 0.0, 1.0)[:, None] - mu[None, :])
        return z, np.exp(-(z * z) / (2.0 * sg[None, :] ** 2))

    def eval(self, d):
        rgba = self.params[:, 2:]
        z, g = self._g(d)
        out = g @ rgba
        dg = -g * z / self.params[None, :, 1] ** 2
        return out, dg @ rgba, None, None, None

    def grads(self, d, o4):
        rgba = self.params[:, 2:]
        sg = self.params[:, 1]
        z, g = self._g(d)
        proj = o4 @ rgba.T                                   # (n, G): o4 . rgba_j
        gr = np.zeros_like(self.params)
        gr[:, 2:] = g.T @ o4
        gr[:, 0] = np.sum(g * z / sg ** 2 * proj, axis=0)
        gr[:, 1] = np.sum(g * z * z / sg ** 3 * proj, axis=0)
        return gr


def _as_tf(tf):
    return tf if isinstance(tf, (PiecewiseTF, GaussianTF)) else None


def segment_opacity(tau_raw, dt):
    """(tau, e, a, a_clamped) of Beer-Lambert with the 1-EPS clamp (field.py:587-600)."""
    tau = np.maximum(tau_raw, 0.0)
    e = np.exp(-dt * tau)
    a_raw = 1.0 - e
    a_clamped = a_raw > 1.0 - EPS_ALPHA
    return tau, e, np.where(a_clamped, 1.0 - EPS_ALPHA, a_raw), a_clamped


# ---------------------------------------------------------------------------
# scene, rays of a row band
# ---------------------------------------------------------------------------


@dataclass
class Band:
    """Ray data of rows [r0, r1) of one view (renderer.py:238-240, 360-368)."""

    u: np.ndarray
    v: np.ndarray
    o: np.ndarray
    w: np.ndarray
    tn: np.ndarray
    tf: np.ndarray
    axis: np.ndarray
    clamped: np.ndarray
    miss: np.ndarray
    n: np.ndarray
    xo: np.ndarray


def make_band(grid: Grid, view: View, dt: float, r0: int = 0, r1: int | None = None) -> Band:
    r1 = view.height if r1 is None else r1
    vv, uu = np.meshgrid(np.arange(r0, r1), np.arange(view.width), indexing="ij")
    u = uu.ravel().astype(np.float64)
    v = vv.ravel().astype(np.float64)
    o, w = pixel_rays(view, u, v)
    tn, tf_, axis, clamped, miss = clip_to_box(o, w, grid.bmin, grid.bmax)
    n = count_steps(tn, tf_, dt, miss)
    return Band(u, v, o, w, tn, tf_, axis, clamped, miss, n, o + tn[None, :] * w)


# ---------------------------------------------------------------------------
# forward march (renderer.py:306-357, 376-401)
# ---------------------------------------------------------------------------


def march(grid: Grid, texels, band: Band, dt: float, *, early_stop=False, record=False):
    """Front-to-back compositing of premultiplied rgb + alpha, (n,4).

    With ``record`` returns the state before every step (the reference's
    "stored" memory mode, renderer.py:348-349).
    """
    nr = band.n.shape[0]
    acc = np.zeros((nr, 4))
    tape = [] if record else None
    steps = int(band.n.max()) if nr else 0
    for i in range(steps):
        act = i < band.n
        if early_stop:                                      # renderer.py:331-335
            act &= acc[:, 3] <= ALPHA_STOP
            if not act.any():
                break
        ti = dt * float(i)
        pts = [band.xo[k] + ti * band.w[k] for k in range(3)]
        d = grid.density(pts)
        s4 = texels.eval(d)[0] if _as_tf(texels) else tf_eval(texels, d)[0]
        _, _, a, _ = segment_opacity(s4[:, 3], dt)
        if record:
            tape.append(acc.copy())
        vis = np.where(act, 1.0 - acc[:, 3], 0.0)
        acc[:, :3] = acc[:, :3] + vis[:, None] * (a[:, None] * s4[:, :3])
        acc[:, 3] = acc[:, 3] + vis * a
    return acc, tape


def render_view(grid: Grid, texels, view: View, dt: float, *, early_stop=False,
                rows=None) -> np.ndarray:
    """Image (H', W, 4) of one view; rows = (r0, r1) restricts to a band."""
    r0, r1 = rows if rows is not None else (0, view.height)
    band = make_band(grid, view, dt, r0, r1)
    rgba, _ = march(grid, texels, band, dt, early_stop=early_stop)
    return rgba.reshape(r1 - r0, view.width, 4)


# ---------------------------------------------------------------------------
# adjoint walk with the inversion trick (renderer.py:491-685)
# ---------------------------------------------------------------------------


def adjoint_view(grid: Grid, texels, view: View, dt: float, seed, targets, *,
                 image=None, rows=None, stored=False):
    """Gradients of sum(seed * image) for each target in ``targets``.

    Back-to-front over every ray of the band; in inversion mode the state
    before a step is recovered from the state after it
    (A_prev = (a - A)/(a - 1), C_prev = C - (1 - A_prev) a c, renderer.py:579-580).
    Returns a dict with keys among d_tf (R,4), d_volume (X,Y,Z),
    d_camera (2,), d_stepsize (float).
    """
    targets = set(targets)
    analytic = _as_tf(texels)
    if not analytic:
        texels = np.asarray(texels, np.float64)
    r0, r1 = rows if rows is not None else (0, view.height)
    band = make_band(grid, view, dt, r0, r1)
    seed = np.asarray(seed, np.float64).reshape(-1, 4)
    if stored or image is None:
        final, tape = march(grid, texels, band, dt, record=stored)
    else:
        final, tape = np.asarray(image, np.float64).reshape(-1, 4), None
    nr = band.n.shape[0]
    steps = int(band.n.max()) if nr else 0
    want_pos = bool(targets & {"camera", "stepsize"})
    want_d = bool(targets & {"camera", "stepsize", "volume"})

    g_tf = np.zeros_like(analytic.params if analytic else texels)
    g_vol = np.zeros(grid.flat.shape[0])
    g_dt = 0.0
    xo_bar = np.zeros((3, nr))
    w_bar = np.zeros((3, nr))

    rgb_bar = seed[:, :3].copy()            # constant along the walk (renderer.py:540)
    alpha_bar = seed[:, 3].copy()
    col = final[:, :3].copy()
    alp = final[:, 3].copy()

    for i in range(steps - 1, -1, -1):
        act = i < band.n
        ti = dt * float(i)
        pts = [band.xo[k] + ti * band.w[k] for k in range(3)]
        d, spatial, w8, idx8 = grid.density_and_grads(pts)
        if analytic:
            out4, slope = analytic.eval(d)[:2]
        else:
            out4, slope, (i0, i1), (tw0, tw1) = tf_eval(texels, d)
        tau, e, a, a_clamped = segment_opacity(out4[:, 3], dt)
        crgb = out4[:, :3]
        cs = a[:, None] * crgb
        if stored:
            prev = tape[i]
            col_prev, alp_prev = prev[:, :3], prev[:, 3]
        else:
            alp_prev = np.where(act, (a - alp) / (a - 1.0), alp)
            col_prev = np.where(act[:, None], col - (1.0 - alp_prev)[:, None] * cs, col)
        vis = 1.0 - alp_prev
        # blend adjoint (renderer.py:583-589)
        cs_bar = vis[:, None] * rgb_bar
        seg_a_bar = vis * alpha_bar + np.sum(crgb * cs_bar, axis=-1)
        alpha_bar_next = (1.0 - a) * alpha_bar - np.sum(cs * rgb_bar, axis=-1)
        crgb_bar = a[:, None] * cs_bar
        # Beer-Lambert (renderer.py:592-596)
        a_raw_bar = np.where(a_clamped, 0.0, seg_a_bar)
        if "stepsize" in targets:
            g_dt += float(np.sum(np.where(act, tau * e * a_raw_bar, 0.0)))
        tau_bar = np.where(out4[:, 3] < 0.0, 0.0, dt * e * a_raw_bar)
        o4 = np.concatenate([crgb_bar, tau_bar[:, None]], axis=1) * act[:, None]
        if "tf" in targets and analytic:
            g_tf += analytic.grads(d, o4)
        elif "tf" in targets:                                # renderer.py:602-604
            np.add.at(g_tf, i0, tw0[:, None] * o4)
            np.add.at(g_tf, i1, tw1[:, None] * o4)
        if want_d:
            d_bar = np.sum(slope * o4, axis=-1)              # renderer.py:606
            if "volume" in targets:                          # renderer.py:607-608
                np.add.at(g_vol, idx8, w8 * d_bar[:, None])
            if want_pos:                                     # renderer.py:609-623
                x_bar = spatial * d_bar[:, None]
                if "stepsize" in targets:
                    g_dt += float(i) * float(np.sum(np.sum(band.w * x_bar.T, axis=0)))
                w_bar += ti * x_bar.T
                xo_bar += x_bar.T
        alpha_bar = np.where(act, alpha_bar_next, alpha_bar)
        col, alp = col_prev, alp_prev

    out = {}
    if "camera" in targets:                                  # renderer.py:629-643
        s = np.sum(band.w * xo_bar, axis=0)
        o_bar = xo_bar.copy()
        w_tot = w_bar + band.tn[None, :] * xo_bar
        need = ~band.clamped & ~band.miss
        for k in range(3):
            sel = need & (band.axis == k)
            wk = np.where(sel, band.w[k], 1.0)
            o_bar[k] += np.where(sel, -s / wk, 0.0)
            w_tot[k] += np.where(sel, -s * band.tn / wk, 0.0)
        j_o, j_d = camera_jacobians(view, band.u, band.v)
        out["d_camera"] = np.einsum("kn,kj->j", o_bar, j_o) + np.einsum("kn,knj->j", w_tot, j_d)
    if "stepsize" in targets:
        out["d_stepsize"] = g_dt
    if "tf" in targets:
        out["d_tf"] = g_tf
    if "volume" in targets:
        out["d_volume"] = g_vol.reshape(grid.dims)
    out["inversion_residual"] = np.concatenate([col, alp[:, None]], axis=1)
    return out


# ---------------------------------------------------------------------------
# loss seed (objectives.py:38-54)
# ---------------------------------------------------------------------------


def l1_seed(images, refs):
    """(mean |x - y|, [sign(x - y)/count]) over all images (objectives.py:38-54)."""
    count = sum(np.asarray(x).size for x in images)
    total = sum(float(np.sum(np.abs(np.asarray(x, np.float64) - np.asarray(y, np.float64))))
                for x, y in zip(images, refs)) / count
    seeds = [np.sign(np.asarray(x, np.float64) - np.asarray(y, np.float64)) / count
             for x, y in zip(images, refs)]
    return total, seeds


# ---------------------------------------------------------------------------
# pre-shaded colour volumes (renderer.py:404-407, 703-709; field.py:361-376)
# ---------------------------------------------------------------------------


class ColorGrid(Grid):
    """(X,Y,Z,4) rgb-emission + absorption grid; trilinear per channel, no clamp."""

    def __init__(self, values, box_min=(-0.5, -0.5, -0.5), box_max=(0.5, 0.5, 0.5)):
        values = np.asarray(values, np.float64)
        super().__init__(values[..., 0], box_min, box_max)
        self.rgba = values.reshape(-1, 4)
        self.cdims = values.shape

    def sample4(self, pts):
        """(n,4) channel values, 0 outside the box (field.py:361-376)."""
        _, idx, frac, inside = self._cell(pts)
        idx8 = self._corners(idx)
        w8 = self._weights(frac)
        out = np.einsum("nc,nck->nk", w8, self.rgba[idx8])
        return np.where(inside[:, None], out, 0.0), w8 * inside[:, None], idx8


def march_color(cg: ColorGrid, band: Band, dt: float, *, early_stop=False, record=False):
    """Front-to-back march of a colour volume (renderer.py:306-357, colour branch)."""
    nr = band.n.shape[0]
    acc = np.zeros((nr, 4))
    tape = [] if record else None
    steps = int(band.n.max()) if nr else 0
    for i in range(steps):
        act = i < band.n
        if early_stop:
            act &= acc[:, 3] <= ALPHA_STOP
            if not act.any():
                break
        ti = dt * float(i)
        s4, _, _ = cg.sample4([band.xo[k] + ti * band.w[k] for k in range(3)])
        _, _, a, _ = segment_opacity(s4[:, 3], dt)
        if record:
            tape.append(acc.copy())
        vis = np.where(act, 1.0 - acc[:, 3], 0.0)
        acc[:, :3] = acc[:, :3] + vis[:, None] * (a[:, None] * s4[:, :3])
        acc[:, 3] = acc[:, 3] + vis * a
    return acc, tape


def render_color_view(cg: ColorGrid, view: View, dt: float, *, early_stop=False):
    band = make_band(cg, view, dt)
    rgba, _ = march_color(cg, band, dt, early_stop=early_stop)
    return rgba.reshape(view.height, view.width, 4)


def adjoint_color_view(cg: ColorGrid, view: View, dt: float, seed, *, image=None, stored=False):
    """d sum(seed * image) / d colour values (X,Y,Z,4) (renderer.py:491-652, colour branch).

    Same inversion walk as adjoint_view; the per-corner sensitivity is
    w8 (inside-masked) times the full out4 adjoint (renderer.py:611-613).
    """
    band = make_band(cg, view, dt)
    seed = np.asarray(seed, np.float64).reshape(-1, 4)
    if stored or image is None:
        final, tape = march_color(cg, band, dt, record=stored)
    else:
        final, tape = np.asarray(image, np.float64).reshape(-1, 4), None
    steps = int(band.n.max()) if band.n.size else 0
    g = np.zeros_like(cg.rgba)
    rgb_bar, alpha_bar = seed[:, :3].copy(), seed[:, 3].copy()
    col, alp = final[:, :3].copy(), final[:, 3].copy()
    for i in range(steps - 1, -1, -1):
        act = i < band.n
        ti = dt * float(i)
        out4, w8, idx8 = cg.sample4([band.xo[k] + ti * band.w[k] for k in range(3)])
        tau, e, a, a_clamped = segment_opacity(out4[:, 3], dt)
        crgb = out4[:, :3]
        cs = a[:, None] * crgb
        if stored:
            col_prev, alp_prev = tape[i][:, :3], tape[i][:, 3]
        else:
            alp_prev = np.where(act, (a - alp) / (a - 1.0), alp)
            col_prev = np.where(act[:, None], col - (1.0 - alp_prev)[:, None] * cs, col)
        vis = 1.0 - alp_prev
        cs_bar = vis[:, None] * rgb_bar
        seg_a_bar = vis * alpha_bar + np.sum(crgb * cs_bar, axis=-1)
        alpha_bar_next = (1.0 - a) * alpha_bar - np.sum(cs * rgb_bar, axis=-1)
        a_raw_bar = np.where(a_clamped, 0.0, seg_a_bar)
        tau_bar = np.where(out4[:, 3] < 0.0, 0.0, dt * e * a_raw_bar)
        o4 = np.concatenate([a[:, None] * cs_bar, tau_bar[:, None]], axis=1) * act[:, None]
        np.add.at(g, idx8, w8[:, :, None] * o4[:, None, :])
        alpha_bar = np.where(act, alpha_bar_next, alpha_bar)
        col, alp = col_prev, alp_prev
    return g.reshape(cg.cdims)
