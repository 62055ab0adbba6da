"""fp32 floor of C5's density gradient (evidence for its parity bar).

Runs the fp64 oracle on the C5 step fixture (tests/golden/C5_step_dense.npz: the
reference's tomography step on 8 rows of view 0 at 512^3 / 1024^2, L1 seed) with
every sample density multiplied by (1 + N(0, 6e-8)) -- fp32-level rounding -- and
compares with the reference.  C5's Gaussian texel preset (tasks.py:378-383) is
sharply peaked, so such noise moves samples across texel kinks where the slope
jumps.  tests/test_gpu_step_config.py uses 2.5x this floor for C5.

    python tools/fp32_floor_c5.py > profiles/r02_fp32_floor_c5.txt   # CPU, a few minutes
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import golden, rel_l2  # noqa: E402
from oracle import dvr_oracle as O  # noqa: E402
from paper_2107_12672_b200.scenes import CONFIGS  # noqa: E402
from test_gpu_step_config import step_estimate  # noqa: E402

g = golden("C5_step_dense")
c = CONFIGS["C5"]
est = step_estimate("C5", "dense")
grid = O.Grid(est)
lon, lat = c.view_poses()[int(g["views"][0])]
view = O.View(lon, lat, c.radius, (0.0, 0.0, 0.0), c.fov, c.image, c.image)
r0, r1 = (int(r) for r in g["rows"])
tex = g["texels"].astype(np.float64)
ref = np.zeros(est.size)
ref[g["volume_idx"]] = g["volume_val"]
seed = np.sign(g["image"][0] - g["refs"][0].astype(np.float64)) / float(g["count"])


def run(noise, seed_rng=0):
    rng = np.random.default_rng(seed_rng)
    orig = O.Grid.density_and_grads

    def noisy(self, pts):
        d, sp, w8, idx = orig(self, pts)
        if noise:
            d = np.clip(d * (1 + rng.normal(scale=noise, size=d.shape)), 0, 1)
        return d, sp, w8, idx
    O.Grid.density_and_grads = noisy
    try:
        return O.adjoint_view(grid, tex, view, c.dt, seed, ["volume"], image=g["image"][0],
                              rows=(r0, r1))["d_volume"].ravel()
    finally:
        O.Grid.density_and_grads = orig


print(f"C5 step band: rows [{r0}, {r1}) of view {int(g['views'][0])}, 512^3, 1024^2")
print("oracle (fp64, no noise) vs reference rel-L2:", rel_l2(run(0.0), ref))
for k in range(3):
    print(f"oracle with fp32-level density noise (draw {k}) vs reference rel-L2:",
          rel_l2(run(6e-8, k), ref))
