"""GPU gradient check driver (gradcheck.py): per probe point, the finite
difference and the adjoint value equal the reference's own (solves and loss
sums are bit-identical), and the adjoint agrees with the FD."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_gradient_check_points_match_reference(reflib):
    from paper_2603_00035_b200 import gradcheck

    n = 36
    F = reflib.random_feasible_fields(n, 8, 0.2)
    src = np.zeros((1, n, n), np.uint8)
    src[0, n // 2, n // 2] = 1
    obs = reflib.observation_mask(src[0])[None]
    vals = np.zeros((1, n, n))
    h = 1.0 / n
    res = gradcheck.gradient_check(*F, src, obs, vals, h, n_points=4, eps=1e-5, seed=3)
    assert len(res.points) == 4
    _, _, adj = reflib.objective_and_grad(*F, src, obs, vals, h)
    for p in res.points:
        assert p.adjoint == adj[p.channel].ravel()[p.node]
        plus, minus = F.copy(), F.copy()
        plus[p.channel].ravel()[p.node] += 1e-5
        minus[p.channel].ravel()[p.node] -= 1e-5
        lp = reflib.loss_grad_mse(reflib.solve(*plus, src[0], h).t, obs[0], vals[0])[1]
        lm = reflib.loss_grad_mse(reflib.solve(*minus, src[0], h).t, obs[0], vals[0])[1]
        assert p.fd == (lp - lm) / 2e-5
        assert p.rel_error < 1e-4
    assert res.max_rel_error < 1e-4
