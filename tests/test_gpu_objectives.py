"""opacity_entropy on the GPU (ddvr_opacity_entropy) vs the reference's own outputs.

tests/golden/entropy.npz: voldiff.objectives.opacity_entropy (objectives.py:95-126)
on the acceptance contract's images (test_acceptance.py:135-163) and the edge
cases the reference handles explicitly: zero alphas (+1e6 seed), a negative
alpha, all-zero alpha and a single pixel (degenerate).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu
CASES = ["uniform", "onehot", "random", "zeros", "scaled", "empty", "single", "negative"]


@pytest.mark.parametrize("case", CASES)
def test_entropy_matches_reference(cuda, case):
    import paper_2107_12672_b200 as vd
    g = golden("entropy")
    h, seed, degenerate = vd.opacity_entropy(g[f"{case}_image"])
    assert degenerate == bool(g[f"{case}_degenerate"])
    assert abs(h - float(g[f"{case}_h"])) <= 1e-9
    np.testing.assert_allclose(seed, g[f"{case}_seed"], rtol=1e-6, atol=1e-9)
    assert np.all(seed[..., :3] == 0.0)


def test_entropy_batch_equals_single_images(cuda):
    """The tensor API reduces every image of a batch independently."""
    import torch
    from paper_2107_12672_b200 import raymarch as R
    g = golden("entropy")
    imgs = np.stack([g["random_image"], g["zeros_image"], g["scaled_image"]]).astype(np.float32)
    h, seed, deg = R.opacity_entropy(torch.from_numpy(imgs).to(cuda))
    for k, case in enumerate(("random", "zeros", "scaled")):
        assert abs(float(h[k]) - float(g[f"{case}_h"])) <= 1e-9
        np.testing.assert_allclose(seed[k].double().cpu().numpy(), g[f"{case}_seed"], rtol=1e-6)
    assert not bool(deg.any())


def test_entropy_contract(cuda):
    """test_acceptance.py:135-163: uniform -> 1, one-hot -> 0, scale invariance,
    seed vs central differences."""
    import paper_2107_12672_b200 as vd
    rng = np.random.default_rng(5)
    data = np.zeros((8, 8, 4))
    data[..., 3] = rng.uniform(0.01, 1.0, (8, 8)).astype(np.float32)
    h1, seed, _ = vd.opacity_entropy(data)
    scaled = data.copy()
    scaled[..., 3] = (scaled[..., 3] * 123.4).astype(np.float32)
    assert abs(vd.opacity_entropy(scaled)[0] - h1) < 1e-6
    fd_h, worst = 1e-3, 0.0          # fp32 inputs: a larger step than the reference's 1e-7
    for _ in range(12):
        i, j = rng.integers(0, 8, 2)
        dp, dm = data.copy(), data.copy()
        dp[i, j, 3] += fd_h
        dm[i, j, 3] -= fd_h
        fd = (vd.opacity_entropy(dp)[0] - vd.opacity_entropy(dm)[0]) / (2 * fd_h)
        worst = max(worst, abs(seed[i, j, 3] - fd) / max(abs(fd), 1e-9))
    assert worst < 1e-3
