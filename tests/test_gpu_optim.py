"""On-device prior / Adam / projection / upsample against the reference's outputs.

tests/golden/optim.npz holds voldiff's own smoothness_prior_volume,
smoothness_prior_tf, adam_step (3 steps), project_params and upsample_volume
on fp32-representable inputs (oracle/gen_golden.py optim_cases).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, rel_max

pytestmark = pytest.mark.gpu


def _t(a, dev, dtype=None):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev)


def test_priors_match_reference(cuda):
    import torch
    from paper_2107_12672_b200 import optim as P
    g = golden("optim")
    vol = _t(g["volume"], cuda)
    grad = torch.zeros_like(vol)
    val = P.prior_volume(vol, 0.5, grad)
    assert abs(float(val) - 0.5 * g["prior_value"]) <= 1e-6 * abs(g["prior_value"])
    assert rel_max(grad.cpu().numpy(), 0.5 * g["prior_grad"]) <= 1e-6
    tex = _t(g["texels"], cuda)
    tg = torch.zeros(tex.shape, dtype=torch.float64, device=cuda)
    tv = P.prior_tf(tex, 2.0, tg)
    assert abs(float(tv) - 2.0 * g["prior_tf_value"]) <= 1e-9 * abs(g["prior_tf_value"])
    assert rel_max(tg.cpu().numpy(), 2.0 * g["prior_tf_grad"]) <= 1e-9


def test_adam_trajectory_and_projection(cuda):
    import torch
    from paper_2107_12672_b200 import optim as P
    g = golden("optim")
    p = _t(g["volume"], cuda)
    st = P.AdamState(lr=float(g["adam_lr"]))
    for k in range(3):
        st.update(p, _t(g["adam_grads"][k], cuda), project=None)
        assert rel_max(p.cpu().numpy(), g["adam_traj"][k]) <= 1e-5
    q = _t(g["volume"], cuda)
    P.AdamState(lr=1e-30).update(q, torch.zeros_like(q), project="volume")
    np.testing.assert_allclose(q.cpu().numpy(), g["proj_vol"], atol=1e-7)
    t = _t(g["proj_tf_in"], cuda)
    P.AdamState(lr=1e-30).update(t, torch.zeros_like(t), project="tf")
    np.testing.assert_allclose(t.cpu().numpy(), g["proj_tf"], rtol=1e-6, atol=1e-6)


def test_adam_device_step_counter(cuda):
    """ddvr_adam_step_device (graph-safe): the same trajectory as the reference's
    adam_step; a skipped (non-finite) update does not advance the counter."""
    import torch
    from paper_2107_12672_b200 import optim as P
    g = golden("optim")
    p = _t(g["volume"], cuda)
    st = P.AdamState(lr=float(g["adam_lr"]), device_step=True)
    for k in range(3):
        st.update(p, _t(g["adam_grads"][k], cuda), project=None, check_finite=False)
        assert rel_max(p.cpu().numpy(), g["adam_traj"][k]) <= 1e-5
    assert int(st.state[0]) == 3
    before = p.clone()
    bad = _t(g["adam_grads"][0], cuda)
    bad.view(-1)[0] = float("nan")
    st.update(p, bad, project=None, check_finite=True)       # skipped on the device
    assert torch.equal(p, before) and int(st.state[0]) == 3


def test_adam_rejects_non_finite_gradients(cuda):
    import torch
    from paper_2107_12672_b200 import optim as P
    from paper_2107_12672_b200.errors import NumericalAbortError
    p = torch.rand(5, 6, device=cuda)
    before = p.clone()
    gr = torch.zeros_like(p)
    gr[2, 3] = float("nan")
    with pytest.raises(NumericalAbortError):
        P.AdamState(lr=0.1).update(p, gr)
    assert torch.equal(p, before)


def test_upsample_matches_reference(cuda):
    from paper_2107_12672_b200 import optim as P
    g = golden("optim")
    up = P.upsample_volume(_t(g["up_src"], cuda))
    assert up.shape == g["up"].shape
    assert rel_max(up.cpu().numpy(), g["up"]) <= 1e-6
