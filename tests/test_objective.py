"""objective_and_grad (inversion.cpp:25-73): the fused
device objective against the reference's own objective_and_grad (oracle/_ref)
and the oracle composition, bit for bit with the exact loss sum."""
import numpy as np
import pytest

from conftest import assert_bitwise


def _problem(reflib, n=40, m=36, K=2, nan_block=False):
    F = reflib.random_feasible_fields(max(n, m), 5, 0.2)[:, :n, :m].copy()
    if nan_block:  # a walled-off pocket: observed nodes there stay unreached
        F[0, 2:5, 2:5] = np.nan
    src = np.zeros((K, n, m), np.uint8)
    src[0, n // 2, m // 3] = 1
    if K > 1:
        src[1, n // 4, (2 * m) // 3] = 1
    obs = np.stack([reflib.observation_mask(src[k], seed=2024 + k) for k in range(K)])
    if nan_block:
        obs[:, 3, 3] = 1
    vals = np.random.default_rng(3).uniform(0.0, 0.8, size=(K, n, m))
    return F, src, obs, vals


@pytest.mark.parametrize("nan_block", [False, True])
def test_oracle_composition_matches_reference(oracle, reflib, nan_block):
    F, src, obs, vals = _problem(reflib, nan_block=nan_block)
    h = 1.0 / 40
    want = reflib.objective_and_grad(*F, src, obs, vals, h)
    got = oracle.objective_and_grad(*F, src, obs, vals, h)
    assert got[0] == want[0] and got[1] == want[1]
    if nan_block:
        assert want[1] > 0
    assert_bitwise(got[2], want[2])


@pytest.mark.gpu
@pytest.mark.parametrize("nan_block", [False, True])
def test_device_objective_bitwise_vs_reference(reflib, nan_block):
    import paper_2603_00035_b200 as rfk

    F, src, obs, vals = _problem(reflib, nan_block=nan_block)
    h = 1.0 / 40
    dl, un, grads = reflib.objective_and_grad(*F, src, obs, vals, h)
    o = rfk.objective_and_grad(*F, src, obs, vals, h, exact=True)
    assert o.data_loss == dl and o.unreached_observed == un
    assert_bitwise(o.grad, grads)


@pytest.mark.gpu
def test_device_objective_device_memory_and_pinned_out(reflib):
    import torch

    import paper_2603_00035_b200 as rfk

    F, src, obs, vals = _problem(reflib, K=1)
    h = 1.0 / 40
    dl, un, grads = reflib.objective_and_grad(*F, src, obs, vals, h)
    dev = [torch.tensor(x, device="cuda") for x in (*F, src, obs, vals)]
    o = rfk.objective_and_grad(*dev, h, exact=True)
    assert o.data_loss == dl
    assert_bitwise(o.grad.cpu().numpy(), grads)
    out = torch.empty((5,) + F.shape[1:], dtype=torch.float64).pin_memory().numpy()
    o2 = rfk.objective_and_grad(*F, src[0], obs[0], vals[0], h, exact=True, out=out)
    assert o2.grad is out
    assert_bitwise(out, grads)


@pytest.mark.gpu
def test_device_objective_not_converged_raises(reflib):
    import paper_2603_00035_b200 as rfk

    F, src, obs, vals = _problem(reflib, K=1)
    with pytest.raises(rfk.NotConverged):
        rfk.objective_and_grad(*F, src, obs, vals, 1.0 / 40, solve_max_iters=1)
    with pytest.raises(rfk.DimensionMismatch):
        rfk.objective_and_grad(*F, src[:, :-1], obs, vals, 1.0 / 40)
