"""fp32 floor of the C5 band's density gradient (evidence for its parity bar).

Runs the fp64 oracle with every sample density multiplied by (1 + N(0, 6e-8)),
i.e. fp32-level rounding, and compares with the reference (tests/golden/C5.npz).
C5's Gaussian texel preset (tasks.py:378-383) is sharply peaked, so such noise
moves samples across texel kinks where the slope jumps: measured rel-L2 1.03e-4.
The GPU path measures 9.95e-5 (profiles/r01_parity.json), i.e. it sits on this
floor; tests/test_gpu_parity.py therefore uses 2.5x the floor for this case.

    python tools/fp32_floor_c5.py      # CPU, ~1 min (builds the 512^3 phantom)
"""
import sys, numpy as np
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'tests'))
from conftest import golden, rel_l2
from oracle import dvr_oracle as O
from paper_2107_12672_b200.scenes import CONFIGS
g = golden("C5"); c = CONFIGS["C5"]
vol = c.volume().astype(np.float64)
lon, lat, radius, cx, cy, cz, fov, W, H = g["cam"]
grid = O.Grid(vol); view = O.View(lon, lat, radius, (cx,cy,cz), fov, int(W), int(H))
r0, r1 = (int(r) for r in g["rows"])
tex = g["texels"].astype(np.float64)
ref = np.zeros(vol.size); ref[g["inversion_volume_idx"]] = g["inversion_volume_val"]
rng = np.random.default_rng(0)
orig = O.Grid.density_and_grads
def noisy(self, pts):
    d, sp, w8, idx = orig(self, pts)
    d = np.clip(d * (1 + rng.normal(scale=6e-8, size=d.shape)), 0, 1)
    return d, sp, w8, idx
O.Grid.density_and_grads = noisy
out = O.adjoint_view(grid, tex, view, c.dt, g["seed_band"], ["volume"], image=g["image"], rows=(r0, r1))
print("rel-L2 with fp32-level density noise:", rel_l2(out["d_volume"].ravel(), ref))
