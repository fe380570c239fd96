"""Adjoint-vs-finite-difference gradient check on the GPU (SURVEY.md §8f
rank 3; the reference's gradient_check, fd_gradient and stencil_stable,
src/oracle.cpp:299-363).

Every probe point costs four device solves (the central difference of the
loss, and the stencil records at both nudges); the adjoint gradient comes
from one fused objective_and_grad.  Candidate points are drawn with numpy's
generator (the reference draws with libstdc++'s mt19937_64, so the sampled
points differ; for a given point the values are the reference's bit for bit).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import api

CHANNELS = ("g11", "g12", "g22", "b1", "b2")


@dataclass
class GradCheckPoint:
    node: int
    channel: int
    fd: float
    adjoint: float
    rel_error: float


@dataclass
class GradCheckResult:
    points: list = field(default_factory=list)
    max_rel_error: float = 0.0
    skipped_unstable: int = 0
    skipped_zero: int = 0


def _torch_planes(params, device):
    import torch
    return [torch.as_tensor(np.asarray(p, np.float64), device=device).contiguous() for p in params]


def loss_value(params, sources, observed, values, h, tol=1e-6, max_iters=50, ctx=None):
    """loss_value (oracle.cpp:213-224): sum over observation sets of the exact
    sequential MSE of the converged solve."""
    total = 0.0
    for k in range(sources.shape[0]):
        t, rep = api.solve(*params, sources[k], h, tol=tol, max_iters=max_iters, ctx=ctx)
        if not rep.converged:
            raise api.NotConverged("loss_value: forward solve did not converge")
        _, loss, _ = api.loss_grad_mse(t, observed[k], values[k], exact=True, ctx=ctx)
        total += loss
    return total


def loss_difference(plus, minus, sources, observed, values, h, tol=1e-6, max_iters=50, ctx=None):
    """L(plus) - L(minus) summed node by node, sum_i 1/2 (T+_i - T-_i)(T+_i + T-_i - 2 v_i)
    over observed reached nodes: the same difference as loss_value(plus) -
    loss_value(minus), without the cancellation of two ~1e5-sized sums that
    differ in their 10th digit at 4096^2 (which leaves a central difference
    with eps = 1e-5 only ~3 significant digits)."""
    import torch
    total = 0.0
    for k in range(sources.shape[0]):
        tp, rp = api.solve(*plus, sources[k], h, tol=tol, max_iters=max_iters, ctx=ctx)
        tm, rm = api.solve(*minus, sources[k], h, tol=tol, max_iters=max_iters, ctx=ctx)
        if not (rp.converged and rm.converged):
            raise api.NotConverged("loss_difference: forward solve did not converge")
        obs = torch.as_tensor(observed[k], device=tp.device).bool()
        val = torch.as_tensor(values[k], device=tp.device)
        m = obs & (tp < 1e9) & (tm < 1e9)
        total += float((0.5 * (tp - tm) * (tp + tm - 2.0 * val))[m].sum())
    return total


def _records(params, sources, h, tol, max_iters, ctx, itol=None):
    out = []
    for k in range(sources.shape[0]):
        t, rep = api.solve(*params, sources[k], h, tol=tol, max_iters=max_iters, ctx=ctx)
        if not rep.converged:
            raise api.NotConverged("stencil identification: solve did not converge")
        r = api.identify_stencils(t, *params, sources[k], h, tol if itol is None else itol, ctx=ctx)
        out.append(tuple(np.asarray(x.cpu() if hasattr(x, "cpu") else x) for x in
                         (r.type, r.stencil, r.donor1, r.donor2)))
    return out


def gradient_check(g11, g12, g22, b1, b2, sources, observed, values, h, channels=(0, 1, 2, 3, 4),
                   n_points=20, eps=1e-5, seed=7, tol=1e-6, max_iters=50, device="cuda", ctx=None,
                   fd="loss", identify_tol=None):
    """gradient_check (oracle.cpp:322-363) with the solves on the GPU.

    sources/observed/values: (K, R, C).  Channels index (g11, g12, g22, b1, b2).
    fd="loss": the reference's central difference of loss_value (bit-identical
    to it); fd="difference": the same central difference summed node by node
    (loss_difference), for grids where the two losses cancel to a few digits.
    identify_tol: the InconsistentFixedPoint slack of identify_stencils
    (default: tol, as LossSpec uses one tol for both); an exact solve
    (tol=1e-300) needs the reference's default 1e-6 here, since an exact
    fixed point keeps "stuck" nodes slightly below their best candidate."""
    itol = tol if identify_tol is None else identify_tol
    if n_points < 1:
        raise api.InvalidArgument("gradient_check: n_points must be >= 1")
    if not channels:
        raise api.InvalidArgument("gradient_check: no channels")
    import torch
    sources = np.asarray(sources, np.uint8).reshape((-1,) + np.shape(g11))
    observed = np.asarray(observed, np.uint8).reshape(sources.shape)
    values = np.asarray(values, np.float64).reshape(sources.shape)
    R, C = np.shape(g11)
    base = [np.array(p, np.float64) for p in (g11, g12, g22, b1, b2)]
    dev_params = _torch_planes(base, device)
    src_d = torch.as_tensor(sources, device=device)
    obs_d = torch.as_tensor(observed, device=device)
    val_d = torch.as_tensor(values, device=device)
    if identify_tol is None:
        adj = api.objective_and_grad(*dev_params, src_d, obs_d, val_d, h, solve_tol=tol, solve_max_iters=max_iters,
                                     exact=True, ctx=ctx).grad.cpu().numpy()
    else:  # adjoint_gradient (oracle.cpp:226-247) with its own identify slack
        acc = None
        for k in range(src_d.shape[0]):
            t, rep = api.solve(*dev_params, src_d[k], h, tol=tol, max_iters=max_iters, ctx=ctx)
            if not rep.converged:
                raise api.NotConverged("adjoint_gradient: forward solve did not converge")
            g, _, _ = api.loss_grad_mse(t, obs_d[k], val_d[k], exact=True, ctx=ctx)
            _, pg, _ = api.backward(t, *dev_params, src_d[k], h, g, tol=itol, ctx=ctx)
            acc = pg if acc is None else acc + pg
        adj = acc.cpu().numpy()
    rng = np.random.default_rng(seed)
    out = GradCheckResult()
    is_src = sources.any(axis=0).ravel()
    for _ in range(40 * n_points):
        if len(out.points) >= n_points:
            break
        r, c = int(rng.integers(2, R - 2)), int(rng.integers(2, C - 2))
        ch = int(channels[int(rng.integers(0, len(channels)))])
        node = r * C + c
        if is_src[node]:
            continue
        # nudge (oracle.cpp:249-257) on device copies: the same IEEE add
        pp = [p.clone() for p in dev_params]
        pm = [p.clone() for p in dev_params]
        pp[ch].view(-1)[node] += eps
        pm[ch].view(-1)[node] -= eps
        rp = _records(pp, src_d, h, tol, max_iters, ctx, itol)
        rm = _records(pm, src_d, h, tol, max_iters, ctx, itol)
        if any(any(not np.array_equal(a, b) for a, b in zip(x, y)) for x, y in zip(rp, rm)):
            out.skipped_unstable += 1
            continue
        if fd == "difference":
            dl = loss_difference(pp, pm, src_d, obs_d, val_d, h, tol, max_iters, ctx)
        else:
            dl = (loss_value(pp, src_d, obs_d, val_d, h, tol, max_iters, ctx) -
                  loss_value(pm, src_d, obs_d, val_d, h, tol, max_iters, ctx))
        fdv = dl / (2.0 * eps)
        an = float(adj[ch].ravel()[node])
        denom = max(abs(fdv), abs(an))
        if denom < 1e-12:
            out.skipped_zero += 1
            continue
        rel = abs(fdv - an) / denom
        out.points.append(GradCheckPoint(node, ch, fdv, an, rel))
        out.max_rel_error = max(out.max_rel_error, rel)
    return out
