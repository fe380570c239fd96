"""Edge cases of run_sweeping / solve / solve_from_values
(src/sweeper.cpp:101-174) against the reference library itself (oracle/_ref),
bit for bit: iteration caps of 0 and below, sweep orders with repeated and
out-of-range directions (the reference maps every d outside 0..2 to its
default branch, sweeper.cpp:101-121), skinny and tiny grids (fewer lines than
a 16-line band, fewer positions than a 32-position staging chunk), and the
device-pointer solve_from_values path."""
import numpy as np
import pytest

from conftest import assert_bitwise

pytestmark = pytest.mark.gpu


def _fields(rows, cols, seed=3, drift=0.2):
    from paper_2603_00035_b200 import workload as wl
    return wl.host_fields(rows, seed, drift, cols=cols)


def _src(rows, cols, pts):
    s = np.zeros((rows, cols), np.uint8)
    for r, c in pts:
        s[r, c] = 1
    return s


def _compare(reflib, F, src, h, **kw):
    import paper_2603_00035_b200 as rfk
    tol, mi, order = kw.get("tol", 1e-6), kw.get("max_iters", 50), kw.get("sweep_order", (0, 1, 2, 3))
    ref = reflib.solve(*F, src, h, tol=tol, max_iters=mi, order=list(order))
    t, rep = rfk.solve(*F, src, h, tol=tol, max_iters=mi, sweep_order=tuple(order))
    assert rep.iterations == ref.iterations
    assert rep.converged == ref.converged
    assert_bitwise(t, ref.t, f"T {kw}")
    assert_bitwise(rep.max_delta_history, ref.history[:ref.iterations], f"history {kw}")
    return t, rep


@pytest.mark.parametrize("max_iters", [0, -1, 1, 2])
def test_iteration_caps(reflib, max_iters):
    F = _fields(40, 52)
    src = _src(40, 52, [(20, 26)])
    t, rep = _compare(reflib, F, src, 1.0 / 52, max_iters=max_iters)
    if max_iters <= 0:
        assert rep.iterations == 0 and not rep.converged
        assert np.all(t[src == 0] == 1e10) and np.all(t[src == 1] == 0.0)


@pytest.mark.parametrize("order", [(0, 0, 0, 0), (3, 3, 1, 1), (0, 7, -1, 2), (2, 2, 0, 0), (1, 3, 1, 3)])
def test_sweep_orders(reflib, order):
    F = _fields(57, 70, seed=5)
    src = _src(57, 70, [(10, 60), (50, 5)])
    for tol in (1e-6, 1e-300):
        _compare(reflib, F, src, 1.0 / 70, tol=tol, max_iters=60, sweep_order=order)


@pytest.mark.parametrize("shape", [(3, 3), (3, 4096), (4096, 3), (17, 1000), (1000, 17), (5, 33), (33, 5),
                                   (16, 16), (18, 31)])
def test_skinny_and_tiny_grids(reflib, shape):
    R, C = shape
    F = _fields(R, C, seed=7)
    src = _src(R, C, [(R // 2, C // 2)])
    _compare(reflib, F, src, 1.0 / max(R, C), max_iters=200)
    if R * C <= 100000:
        _compare(reflib, F, src, 1.0 / max(R, C), tol=1e-300, max_iters=200)


def test_skinny_backward(reflib):
    """identify -> adjoint -> gradients on a grid with fewer lines than a band."""
    import paper_2603_00035_b200 as rfk
    R, C = 9, 700
    F = _fields(R, C, seed=9)
    src = _src(R, C, [(4, 350)])
    h = 1.0 / C
    t, rep = _compare(reflib, F, src, h)
    obs = (np.arange(R * C).reshape(R, C) % 3 == 0).astype(np.uint8) * (1 - src)
    g, _, _ = reflib.loss_grad_mse(t, obs, np.zeros_like(t))
    lam_r, pg_r, cl_r = reflib.backward(t, *F, src, h, g)
    lam, pg, cl = rfk.backward(t, *F, src, h, g)
    assert cl == cl_r
    assert_bitwise(lam, lam_r, "lambda")
    assert_bitwise(pg, pg_r, "gradients")


def test_solve_from_values_device_pointers(reflib):
    import torch

    import paper_2603_00035_b200 as rfk
    R, C = 48, 61
    F = _fields(R, C, seed=11)
    fixed = np.zeros((R, C), np.uint8)
    fixed[:, 0] = 1
    fixed[R // 3, C // 2] = 1
    vals = np.where(fixed == 1, np.linspace(0.0, 0.3, R)[:, None] * np.ones((1, C)), 0.0)
    h = 1.0 / C
    ref = reflib.solve(*F, fixed, h, mode=2, fixed_values=vals)
    dev = [torch.as_tensor(x).cuda() for x in F]
    t, rep = rfk.solve_from_values(*dev, torch.as_tensor(fixed).cuda(), torch.as_tensor(vals).cuda(), h)
    assert rep.iterations == ref.iterations
    assert_bitwise(t.cpu().numpy(), ref.t, "solve_from_values (device pointers)")


@pytest.mark.parametrize("scale", [1e-200, 1e-32, 1e32, 1e200])
def test_extreme_metric_magnitudes(reflib, scale):
    """Metrics scaled far outside the fast path's exponent window (hoisted
    |q| >= 2^100 or a outside 2^+-100 go to the out-of-line IEEE division and
    the exact lambda test, rfk_sweep.cu slow_update): T, K and the history
    still equal the reference's bit for bit, including products that
    overflow to +-inf in the lambda test (the reference's inf + -inf = NaN
    rejects the candidate, stencil.cpp:36-41)."""
    R, C = 40, 37
    F = list(_fields(R, C, seed=5, drift=0.0))
    F = [F[0] * scale, F[1] * scale, F[2] * scale, F[3], F[4]]
    _compare(reflib, F, _src(R, C, [(20, 18)]), 1.0 / C)
    # a band of extreme nodes inside an ordinary metric
    G = list(_fields(R, C, seed=6, drift=0.1))
    for k in range(3):
        G[k] = G[k].copy()
        G[k][10:14, :] *= scale
    _compare(reflib, G, _src(R, C, [(3, 4), (30, 30)]), 1.0 / C)
