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


def test_loss_difference_equals_loss_value_difference_small(reflib):
    """The node-wise central difference (used at 4096^2) is the reference's
    loss_value difference up to the latter's cancellation."""
    import torch

    from paper_2603_00035_b200 import gradcheck
    n = 40
    F = reflib.random_feasible_fields(n, 5, 0.2)
    src = np.zeros((1, n, n), np.uint8)
    src[0, 20, 20] = 1
    obs = reflib.observation_mask(src[0])[None]
    vals = np.zeros((1, n, n))
    dev = [torch.as_tensor(x).cuda() for x in F]
    pp = [p.clone() for p in dev]
    pm = [p.clone() for p in dev]
    pp[2].view(-1)[5 * n + 9] += 1e-5
    pm[2].view(-1)[5 * n + 9] -= 1e-5
    s = torch.as_tensor(src).cuda()
    o = torch.as_tensor(obs).cuda()
    v = torch.as_tensor(vals).cuda()
    a = gradcheck.loss_difference(pp, pm, s, o, v, 1.0 / n)
    b = gradcheck.loss_value(pp, s, o, v, 1.0 / n) - gradcheck.loss_value(pm, s, o, v, 1.0 / n)
    assert abs(a - b) <= 1e-9 * abs(b) + 1e-15


def test_c3_gradient_check_4096():
    """BASELINE configs[2]: 4096^2 Randers forward + adjoint vs central
    finite differences at stencil-stable points (oracle.cpp:322-363), exact
    solves.  At this size the difference has a noise floor from the exact
    Gauss-Seidel fixed point's history dependence (it grows as 1/eps,
    profiles/r02_gradcheck_c3.json), so the check uses eps = 1e-4 and the
    median over the points."""
    from paper_2603_00035_b200 import gradcheck
    from paper_2603_00035_b200 import workload as wl
    n = 4096
    F = wl.host_fields(n, 1, 0.2)
    src = wl.host_point_source(n, n)
    obs = wl.host_observation_mask(src)
    res = gradcheck.gradient_check(*F, src[None], obs[None], np.zeros((1, n, n)), 1.0 / n, n_points=7, eps=1e-4,
                                   seed=7, fd="difference", tol=1e-300, max_iters=100, identify_tol=1e-6)
    assert len(res.points) == 7
    rel = sorted(p.rel_error for p in res.points)
    assert rel[len(rel) // 2] < 1e-3 and rel[-1] < 1e-2, [(p.node, p.channel, p.fd, p.adjoint, p.rel_error)
                                                           for p in res.points]
