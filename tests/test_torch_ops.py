"""Autograd bindings (paper_2603_00035_b200.torch_ops): gradients equal the
C ABI's adjoint / projection VJP exactly, and agree with central finite
differences of the forward along random smooth directions."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _fields(reflib, n=32):
    import torch
    F = reflib.random_feasible_fields(n, 11, 0.2)
    return [torch.tensor(x, device="cuda", requires_grad=True) for x in F]


def test_eikonal_solve_grad_matches_backward(reflib):
    import torch

    import paper_2603_00035_b200 as rfk
    from paper_2603_00035_b200 import torch_ops

    n = 32
    F = _fields(reflib, n)
    src = torch.zeros((n, n), dtype=torch.uint8, device="cuda")
    src[n // 2, n // 3] = 1
    obs = torch.tensor(reflib.observation_mask(src.cpu().numpy()), device="cuda").bool()
    t = torch_ops.eikonal_solve(*F, src, 1.0 / n)
    loss = 0.5 * ((t - 0.3)[obs] ** 2).sum()
    loss.backward()
    g = torch.where(obs, t.detach() - 0.3, torch.zeros_like(t))
    _, want, _ = rfk.backward(t.detach(), *(x.detach() for x in F), src, 1.0 / n, g, want_lambda=False)
    for k in range(5):
        np.testing.assert_array_equal(F[k].grad.cpu().numpy(), want[k].cpu().numpy())


def test_eikonal_solve_directional_fd(reflib):
    import torch

    from paper_2603_00035_b200 import torch_ops

    n = 32
    F = _fields(reflib, n)
    src = torch.zeros((n, n), dtype=torch.uint8, device="cuda")
    src[n // 2, n // 2] = 1
    obs = torch.tensor(reflib.observation_mask(src.cpu().numpy()), device="cuda").bool()

    def loss_of(params):
        t = torch_ops.eikonal_solve(*params, src, 1.0 / n, tol=1e-300, max_iters=200)
        return 0.5 * ((t - 0.2)[obs] ** 2).sum()

    loss_of(F).backward()
    # smooth direction (low-frequency) so the stencil choice does not flip
    yy, xx = torch.meshgrid(torch.linspace(0, 1, n, device="cuda", dtype=torch.float64),
                            torch.linspace(0, 1, n, device="cuda", dtype=torch.float64), indexing="ij")
    vs = [torch.sin(3 * xx + k) * torch.cos(2 * yy - k) for k in range(5)]
    an = sum((F[k].grad * vs[k]).sum() for k in range(5)).item()
    eps = 1e-6
    with torch.no_grad():
        lp = loss_of([F[k] + eps * vs[k] for k in range(5)]).item()
        lm = loss_of([F[k] - eps * vs[k] for k in range(5)]).item()
    fd = (lp - lm) / (2 * eps)
    assert abs(fd - an) <= 1e-4 * max(abs(fd), abs(an)), (fd, an)


def test_batched_shared_params_accumulate(reflib):
    import torch

    import paper_2603_00035_b200 as rfk
    from paper_2603_00035_b200 import torch_ops

    n = 24
    F = _fields(reflib, n)
    src = torch.zeros((2, n, n), dtype=torch.uint8, device="cuda")
    src[0, 5, 5] = 1
    src[1, 17, 12] = 1
    t = torch_ops.eikonal_solve(*F, src, 1.0 / n)
    (t.sum(dim=(1, 2)) * torch.tensor([1.0, 2.0], device="cuda", dtype=torch.float64)).sum().backward()
    g = torch.ones_like(t)
    g[1] = 2.0
    g = torch.where(t < 1e9, g, torch.zeros_like(g))
    _, want, _ = rfk.backward(t.detach(), *(x.detach() for x in F), src, 1.0 / n, g, accumulate=True,
                              want_lambda=False)
    for k in range(5):
        np.testing.assert_array_equal(F[k].grad.cpu().numpy(), want[k].cpu().numpy())


def test_projection_layer_matches_vjp_and_gradcheck():
    import torch

    from oracle import pyoracle as po
    from paper_2603_00035_b200 import torch_ops

    rng = np.random.default_rng(4)
    n = 64
    th = rng.uniform(0, np.pi, n)
    l1, l2 = rng.uniform(-0.5, 6.0, n), rng.uniform(0.05, 3.0, n)
    c, s = np.cos(th), np.sin(th)
    g = [l1 * c * c + l2 * s * s, (l1 - l2) * c * s, l1 * s * s + l2 * c * c]
    r, ph = rng.uniform(0, 2.5, n), rng.uniform(0, 2 * np.pi, n)
    x = [torch.tensor(v, device="cuda", requires_grad=True) for v in (*g, r * np.cos(ph), r * np.sin(ph))]
    cfg = (0.05, 4.0, 0.6, 1.5)
    out = torch_ops.project(*x, *cfg)
    w = [torch.tensor(rng.normal(size=n), device="cuda") for _ in range(5)]
    sum((o * wk).sum() for o, wk in zip(out, w)).backward()
    want = po.project_joint_vjp_np(*(v.detach().cpu().numpy() for v in x), *(wk.cpu().numpy() for wk in w), *cfg)
    for k in range(5):
        np.testing.assert_allclose(x[k].grad.cpu().numpy(), want[k], rtol=1e-10, atol=1e-12)
