"""How often do lanes of one warp flush the same cell in the same adjoint step?

C4 geometry (256^3, 512^2, dt 0.2 voxel), several views and warp tiles (8x4
pixels as in pixel_of).  For each backward step, among lanes whose cell run
ends (cell changes), count distinct cells.  Prints flushes per warp-step and
the distinct/flushing ratio (the best a warp-aggregated flush could reach).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import dvr_oracle as O                       # noqa: E402
from paper_2107_12672_b200.scenes import CONFIGS          # noqa: E402

c = CONFIGS["C4"]
grid = O.Grid(np.zeros((256, 256, 256)))
rng = np.random.default_rng(0)
tot_flush = tot_distinct = tot_steps = 0
for lon, lat in c.view_poses()[:6]:
    view = O.View(lon, lat, c.radius, fov_y_deg=c.fov, width=512, height=512)
    for _ in range(12):
        x0, y0 = rng.integers(16, 60) * 8, rng.integers(32, 96) * 4
        band = O.make_band(grid, view, c.dt, y0, y0 + 4)
        sel = (band.u >= x0) & (band.u < x0 + 8)
        n = band.n[sel]
        if n.max() == 0:
            continue
        xo, w = band.xo[:, sel], band.w[:, sel]
        scale = (256 / (grid.bmax - grid.bmin))[:, None]
        steps = int(n.max())
        cells = np.full((steps, sel.sum()), -1, np.int64)
        for i in range(steps):
            g = (xo + i * c.dt * w - grid.bmin[:, None]) * scale - 0.5
            cid = np.floor(g).astype(np.int64)
            key = (cid[0] * 300 + cid[1]) * 300 + cid[2]
            cells[i] = np.where(i < n, key, -1)
        for i in range(steps - 1, 0, -1):      # backward walk: run ends when cell changes
            live = (cells[i] >= 0)
            flush = live & (cells[i - 1] != cells[i])
            k = int(flush.sum())
            tot_steps += 1
            if k:
                tot_flush += k
                tot_distinct += len(np.unique(cells[i][flush]))
print(f"flushing lanes per warp-step {tot_flush / tot_steps:.2f}, distinct cells "
      f"{tot_distinct / tot_steps:.2f}, ratio {tot_distinct / max(tot_flush, 1):.3f}")
