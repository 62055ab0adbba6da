"""fp32 floor of the R2048 edge case (tests/test_gpu_properties.py, evidence for its bar).

The case uses 2048 independent uniform-random texels: the TF slope is ~+-2000
and jumps at every texel boundary, so fp32-level density rounding moves
samples across kinks.  This runs the fp64 oracle on the test's exact scene
with every sample density multiplied by (1 + N(0, 6e-8)) and reports the
rel-L2 of each gradient against the clean oracle, over several noise seeds.

    python tools/fp32_floor_r2048.py     # CPU, seconds
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import rel_l2                      # noqa: E402
from oracle import dvr_oracle as O               # noqa: E402

rng = np.random.default_rng(5)
vol = rng.uniform(0.05, 0.95, (8, 8, 8)).astype(np.float32)
rng.uniform(0.05, 1.0, (8, 4))                    # the default texels the case replaces
tex = rng.uniform(0.05, 1.0, (2048, 4)).astype(np.float32).astype(np.float64)
view = O.View(33.0, 21.0, 2.2, fov_y_deg=35.0, width=9, height=7)
seed = rng.normal(size=(7, 9, 4)).astype(np.float32).astype(np.float64)
grid = O.Grid(vol.astype(np.float64))
targets = ["volume", "tf", "camera", "stepsize"]
img = O.render_view(grid, tex, view, 0.04)
clean = O.adjoint_view(grid, tex, view, 0.04, seed, targets, image=img)
orig = O.Grid.density_and_grads
worst = {t: 0.0 for t in targets}
for s in range(8):
    noise = np.random.default_rng(100 + s)

    def noisy(self, pts, _n=noise):
        d, sp, w8, idx = orig(self, pts)
        return np.clip(d * (1 + _n.normal(scale=6e-8, size=d.shape)), 0, 1), sp, w8, idx

    O.Grid.density_and_grads = noisy
    out = O.adjoint_view(grid, tex, view, 0.04, seed, targets, image=img)
    O.Grid.density_and_grads = orig
    for t in targets:
        worst[t] = max(worst[t], rel_l2(np.ravel(out["d_" + t]), np.ravel(clean["d_" + t])))
print("max rel-L2 over 8 fp32-level noise draws:", {t: f"{v:.2e}" for t, v in worst.items()})
