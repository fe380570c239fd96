"""The feasibility projection fused into the load stage (north_star (3),
SURVEY §7.4): rfk_solve_projected projects each node inside the sweep's
hoist and rfk_backward_projected applies the projection's VJP inside the
gradient pass.  Both must be bitwise equal to the unfused chain
project_spd / project_drift -> solve -> backward -> project_vjp
(ParamView::project, inversion.cpp:255-279; feasibility.cpp:31-72), for every
projection mode, per-grid and shared parameters, and through the C5 torch
path."""
import numpy as np
import pytest

from conftest import assert_bitwise

pytestmark = pytest.mark.gpu


def _raw(B, R, C, seed, amp=1.0):
    """Parameters that need projecting: eigenvalues outside [0.5, 2.5] at
    many nodes (amp = 1), drift beyond tau = 0.4 in the G^-1 norm.  With a
    small amp the metric stays SPD (project_drift alone needs that)."""
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:R, 0:C] / max(R, C)
    out = []
    for b in range(B):
        ph = rng.uniform(0, 6, 5)
        g11 = 1.0 + 1.4 * amp * np.sin(5 * x + ph[0]) * np.cos(3 * y)
        g22 = 1.0 + 1.3 * amp * np.cos(4 * y + ph[1])
        g12 = 0.9 * amp * np.sin(6 * (x + y) + ph[2])
        b1 = 0.7 * np.sin(3 * y + 2 * x + ph[3])
        b2 = 0.7 * np.cos(4 * x - y + ph[4])
        out.append(np.stack([g11, g12, g22, b1, b2]))
    return np.stack(out, axis=1)  # (5, B, R, C)


def _unfused(rfk, raw, proj):
    import torch
    g11, g12, g22, b1, b2 = (x.clone() for x in raw)
    if proj.mode & 1:
        g11, g12, g22 = rfk.project_spd(g11, g12, g22, proj.eps_min, proj.lambda_max)
    if proj.mode & 2:
        b1, b2 = rfk.project_drift(b1, b2, g11, g12, g22, proj.tau, proj.euclid_cap)
    return [g11, g12, g22, b1, b2]


@pytest.mark.parametrize("mode", [1, 2, 3])
@pytest.mark.parametrize("shared", [False, True])
def test_fused_projection_equals_unfused_chain(mode, shared):
    import torch

    import paper_2603_00035_b200 as rfk
    B, R, C = 3, 61, 70
    raw_np = _raw(1 if shared else B, R, C, seed=mode, amp=1.0 if mode & 1 else 0.2)
    raw = [torch.as_tensor(raw_np[k][0] if shared else raw_np[k]).cuda() for k in range(5)]
    src = torch.zeros((B, R, C), dtype=torch.uint8, device="cuda")
    for b in range(B):
        src[b, (13 + 17 * b) % R, (7 + 23 * b) % C] = 1
    proj = rfk.Projection(mode, 0.5, 2.5, 0.4, 10.0)
    h = 1.0 / C
    # forward
    t_f, rep_f, planes = rfk.solve_projected(*raw, src, h, proj)
    fields = _unfused(rfk, raw, proj)
    t_u, rep_u = rfk.solve(*fields, src, h)
    assert np.array_equal(np.asarray(rep_f.iterations), np.asarray(rep_u.iterations))
    assert_bitwise(t_f.cpu().numpy(), t_u.cpu().numpy(), "T")
    for k in range(5):
        assert_bitwise(planes[k].cpu().numpy(), fields[k].cpu().numpy(), f"projected plane {k}")
    # some nodes were actually projected
    assert any(not torch.equal(planes[k], raw[k]) for k in range(5))
    # backward
    obs = (torch.rand((B, R, C), generator=torch.Generator("cuda").manual_seed(5), device="cuda") < 0.3)
    lg, _, _ = rfk.loss_grad_mse(t_u, obs.to(torch.uint8) * (1 - src), torch.zeros_like(t_u))
    lam_f, g_f, cl_f = rfk.backward_projected(t_f, *raw, planes, src, h, lg, proj, accumulate=shared)
    lam_u, g_u, cl_u = rfk.backward(t_u, *fields, src, h, lg, accumulate=shared)
    # the unfused VJP: elementwise over the (flattened) raw planes
    d = [g_u[k].clone() for k in range(5)]
    shp = d[0].shape
    flat = [x.reshape(-1).contiguous() for x in raw]
    dd = [x.reshape(-1).contiguous() for x in d]
    if mode == 3:
        d = [x.reshape(shp) for x in rfk.project_vjp(*flat, *dd, proj.eps_min, proj.lambda_max, proj.tau,
                                                       proj.euclid_cap)]
    elif mode == 1:
        a, b_, c = rfk.project_spd_vjp(flat[0], flat[1], flat[2], dd[0], dd[1], dd[2], proj.eps_min,
                                       proj.lambda_max)
        d = [a.reshape(shp), b_.reshape(shp), c.reshape(shp), d[3], d[4]]
    else:  # drift against the metric as given; its metric cotangent accumulates onto the solver's
        x1, y1, c11, c12, c22 = rfk.project_drift_vjp(flat[3], flat[4], flat[0], flat[1], flat[2], dd[3], dd[4],
                                                      proj.tau, proj.euclid_cap, metric_grad=True,
                                                      d_metric=dd[:3])
        d = [c11.reshape(shp), c12.reshape(shp), c22.reshape(shp), x1.reshape(shp), y1.reshape(shp)]
    assert np.array_equal(np.asarray(cl_f), np.asarray(cl_u))
    assert_bitwise(lam_f.cpu().numpy(), lam_u.cpu().numpy(), "lambda")
    for k in range(5):
        assert_bitwise(g_f[k].cpu().numpy(), d[k].cpu().numpy(), f"raw gradient {k}")


def test_c5_loss_fused_equals_unfused():
    import torch

    from paper_2603_00035_b200 import training
    n, B = 40, 3
    g = torch.Generator(device="cpu").manual_seed(4)
    cov = torch.randn((B, 3, n, n), generator=g).cuda()
    src = torch.zeros((B, n, n), dtype=torch.uint8, device="cuda")
    for b in range(B):
        src[b, 5 + 9 * b, 30 - 7 * b] = 1
    obs = (torch.rand((B, n, n), generator=g) < 0.3).to(torch.uint8).cuda()
    tgt = torch.rand((B, n, n), generator=g, dtype=torch.float64).cuda()
    # cuDNN's convolution backward may use atomics: deterministic algorithms
    # so the encoder gradients of the two runs can be compared bit for bit
    det = torch.backends.cudnn.deterministic
    torch.backends.cudnn.deterministic = True
    try:
        losses, grads = [], []
        for fused in (True, False):
            torch.manual_seed(9)
            model = training.RandersEncoder().cuda()
            loss = training.c5_loss(model, cov, src, obs, tgt, 1.0 / n, fused_projection=fused)
            loss.backward()
            losses.append(loss.item())
            grads.append([p.grad.clone() for p in model.parameters()])
    finally:
        torch.backends.cudnn.deterministic = det
    assert losses[0] == losses[1]
    for a, b in zip(*grads):
        assert torch.equal(a, b)
