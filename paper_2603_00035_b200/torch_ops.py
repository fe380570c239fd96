"""PyTorch autograd bindings of the hot path.

The paper trains an encoder through the solver with "hybrid autodiff":
implicit differentiation for the eikonal solve and the adjoint for its
parameters, plus "differentiable projection layers"
(PAPER.md:297).  These Functions make the CUDA library usable as ordinary
autograd nodes on CUDA tensors:

* :class:`EikonalSolve` - forward ``rfk_solve``; backward the fused
  identify -> adjoint -> parameter-gradient path (``rfk_backward``), the
  implicit derivative of the converged fixed point.
* :class:`Projection` - ``ParamView::project`` for the Joint
  parameterisation (``project_spd`` then ``project_drift``,
  inversion.cpp:276-279); backward ``rfk_project_vjp``.
* :class:`ProjectedEikonalSolve` - the two fused: T = solve(project(raw));
  the projection runs inside the sweep's load stage (``rfk_solve_projected``)
  and its VJP inside the backward's gradient pass
  (``rfk_backward_projected``).  Bitwise the same values and gradients as
  ``eikonal_solve(*project(raw))``, with one pass fewer each way.

No CPU fallback: inputs must be CUDA float64 tensors.
"""
from __future__ import annotations

import torch

from . import api


def _check(*xs):
    for x in xs:
        if not (isinstance(x, torch.Tensor) and x.is_cuda):
            raise api.InvalidArgument("torch_ops: inputs must be CUDA tensors (no CPU fallback)")


# Optional collector of forward-solve results (iteration counts + arrival
# fields), used by bench.py's C5 line to count the work it timed.
_solve_stats = None


def collect_solve_stats(target):
    """Append (iterations, T, sources) of every forward solve to `target`
    (a list), or stop collecting with None."""
    global _solve_stats
    _solve_stats = target


class EikonalSolve(torch.autograd.Function):
    """T = solve(G, b, sources); dL/dG, dL/db by the adjoint method.

    Shapes follow :func:`api.solve`: parameters (R, C) shared by a batch of
    source masks (B, R, C), or per-grid (B, R, C).  With shared parameters the
    per-source gradients are summed in source order (inversion.cpp:13-21)."""

    @staticmethod
    def forward(ctx, g11, g12, g22, b1, b2, src, h, tol=1e-6, max_iters=50, ctx_rfk=None):
        _check(g11, g12, g22, b1, b2, src)
        params = [x.detach().to(torch.float64).contiguous() for x in (g11, g12, g22, b1, b2)]
        srcc = src.detach().to(torch.uint8).contiguous()
        t, rep = api.solve(*params, srcc, h, tol=tol, max_iters=max_iters, ctx=ctx_rfk)
        conv = rep.converged if isinstance(rep.converged, bool) else bool(rep.converged.all())
        if not conv:
            raise api.NotConverged("EikonalSolve: forward solve did not converge")
        if _solve_stats is not None:
            _solve_stats.append((rep.iterations, t, srcc))
        ctx.save_for_backward(t, *params, srcc)
        ctx.h, ctx.tol, ctx.rfk = h, tol, ctx_rfk
        ctx.shared = params[0].dim() == 2
        return t

    @staticmethod
    def backward(ctx, dT):
        t, g11, g12, g22, b1, b2, src = ctx.saved_tensors
        dT = dT.contiguous().to(torch.float64)
        batched = t.dim() == 3
        _, grads, _ = api.backward(t, g11, g12, g22, b1, b2, src, ctx.h, dT, tol=ctx.tol,
                                   accumulate=ctx.shared and batched, want_lambda=False, ctx=ctx.rfk)
        # grads is (5, R, C) for shared parameters, (5, B, R, C) per grid
        out = [grads[k] for k in range(5)]
        return (*out, None, None, None, None, None)


def eikonal_solve(g11, g12, g22, b1, b2, src, h, tol=1e-6, max_iters=50, ctx=None):
    """Differentiable :func:`api.solve` (returns T only)."""
    return EikonalSolve.apply(g11, g12, g22, b1, b2, src, h, tol, max_iters, ctx)


class Projection(torch.autograd.Function):
    """ParamView::project for the Joint parameterisation, differentiable."""

    @staticmethod
    def forward(ctx, g11, g12, g22, b1, b2, eps_min=1e-3, lambda_max=1e3, tau=0.95, euclid_cap=10.0,
                ctx_rfk=None):
        _check(g11, g12, g22, b1, b2)
        x = [v.detach().to(torch.float64).contiguous() for v in (g11, g12, g22, b1, b2)]
        p11, p12, p22 = api.project_spd(x[0], x[1], x[2], eps_min, lambda_max, ctx=ctx_rfk)
        q1, q2 = api.project_drift(x[3], x[4], p11, p12, p22, tau, euclid_cap, ctx=ctx_rfk)
        ctx.save_for_backward(*x)
        ctx.cfg = (eps_min, lambda_max, tau, euclid_cap)
        ctx.rfk = ctx_rfk
        return p11, p12, p22, q1, q2

    @staticmethod
    def backward(ctx, *d):
        x = ctx.saved_tensors
        d = [torch.zeros_like(x[k]) if g is None else g.contiguous().to(torch.float64) for k, g in enumerate(d)]
        out = api.project_vjp(*x, *d, *ctx.cfg, ctx=ctx.rfk)
        return (*out, None, None, None, None, None)


def project(g11, g12, g22, b1, b2, eps_min=1e-3, lambda_max=1e3, tau=0.95, euclid_cap=10.0, ctx=None):
    """Differentiable feasibility projection (project_spd, then project_drift)."""
    return Projection.apply(g11, g12, g22, b1, b2, eps_min, lambda_max, tau, euclid_cap, ctx)


class ProjectedEikonalSolve(torch.autograd.Function):
    """T = solve(ParamView::project(raw)) with the projection fused into the
    solver's load stage and its VJP into the backward's gradient pass."""

    @staticmethod
    def forward(ctx, g11, g12, g22, b1, b2, src, h, tol=1e-6, max_iters=50, eps_min=1e-3, lambda_max=1e3,
                tau=0.95, euclid_cap=10.0, ctx_rfk=None):
        _check(g11, g12, g22, b1, b2, src)
        raw = [x.detach().to(torch.float64).contiguous() for x in (g11, g12, g22, b1, b2)]
        srcc = src.detach().to(torch.uint8).contiguous()
        pc = api.Projection(3, eps_min, lambda_max, tau, euclid_cap)
        t, rep, proj = api.solve_projected(*raw, srcc, h, pc, tol=tol, max_iters=max_iters, ctx=ctx_rfk)
        conv = rep.converged if isinstance(rep.converged, bool) else bool(rep.converged.all())
        if not conv:
            raise api.NotConverged("ProjectedEikonalSolve: forward solve did not converge")
        if _solve_stats is not None:
            _solve_stats.append((rep.iterations, t, srcc))
        ctx.save_for_backward(t, *raw, proj, srcc)
        ctx.h, ctx.tol, ctx.rfk, ctx.pc = h, tol, ctx_rfk, pc
        ctx.shared = raw[0].dim() == 2
        return t

    @staticmethod
    def backward(ctx, dT):
        t, g11, g12, g22, b1, b2, proj, src = ctx.saved_tensors
        dT = dT.contiguous().to(torch.float64)
        batched = t.dim() == 3
        _, grads, _ = api.backward_projected(t, g11, g12, g22, b1, b2, proj, src, ctx.h, dT, ctx.pc, tol=ctx.tol,
                                             accumulate=ctx.shared and batched, want_lambda=False, ctx=ctx.rfk)
        out = [grads[k] for k in range(5)]
        return (*out,) + (None,) * 9


def projected_eikonal_solve(g11, g12, g22, b1, b2, src, h, tol=1e-6, max_iters=50, eps_min=1e-3, lambda_max=1e3,
                            tau=0.95, euclid_cap=10.0, ctx=None):
    """Differentiable solve of projected raw parameters, projection fused."""
    return ProjectedEikonalSolve.apply(g11, g12, g22, b1, b2, src, h, tol, max_iters, eps_min, lambda_max, tau,
                                       euclid_cap, ctx)
