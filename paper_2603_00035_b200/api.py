"""Host-side mirror of the reference API for the Randers hot path.

Names, argument meaning and error behaviour follow the reference's
``proj/include/randers`` API (solve, solve_jacobi, solve_from_values,
best_candidate, node_update, two_point_update, identify_stencils,
jacobian_entries, solve_adjoint, param_gradients, loss_grad_mse,
project_spd, project_drift, drift_norm_sq) so tests read like the
reference's own.  Every call goes through the C ABI (include/rfk.h) into
librfk.so; there is no CPU path.

Arrays may be numpy arrays (host memory: the library stages them through the
device) or CUDA torch tensors (device memory: nothing crosses PCIe).  A
leading batch dimension solves independent grids in one call.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib as L


# ---- errors: randers::Error hierarchy (include/randers/errors.hpp:8-50) ------
class Error(RuntimeError):
    pass


class DimensionMismatch(Error):
    pass


class ZeroDimension(Error):
    pass


class InvalidArgument(Error):
    pass


class InconsistentFixedPoint(Error):
    pass


class NotConverged(Error):
    pass


class NonSpdInput(Error):
    pass


class DivergedLoss(Error):
    pass


class CudaError(Error):
    pass


class NoDevice(Error):
    pass


_ERRORS = {
    L.RFK_ERR_DIMENSION_MISMATCH: DimensionMismatch,
    L.RFK_ERR_ZERO_DIMENSION: ZeroDimension,
    L.RFK_ERR_INVALID_ARGUMENT: InvalidArgument,
    L.RFK_ERR_INCONSISTENT_FIXED_POINT: InconsistentFixedPoint,
    L.RFK_ERR_CUDA: CudaError,
    L.RFK_ERR_NO_DEVICE: NoDevice,
    L.RFK_ERR_ALLOC: CudaError,
    L.RFK_ERR_NOT_CONVERGED: NotConverged,
    L.RFK_ERR_NON_SPD_INPUT: NonSpdInput,
    L.RFK_ERR_DIVERGED_LOSS: DivergedLoss,
}


class Context:
    """Owns an rfk_context (device workspace cache + stream)."""

    def __init__(self, device: int = 0):
        self.lib = L.load()
        h = C.c_void_p()
        st = self.lib.rfk_create(C.byref(h), device)
        if st != L.RFK_OK:
            raise _ERRORS.get(st, Error)(self.lib.rfk_status_string(st).decode())
        self.handle = h
        self.device = device

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.rfk_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def set_stream(self, stream_ptr: int):
        self.check(self.lib.rfk_set_stream(self.handle, C.c_void_p(stream_ptr)))
        self._stream = stream_ptr

    def bind(self, dev):
        """Device-pointer calls: the tensors must live on this context's
        device, and the library runs on torch's current stream of that device
        (ordered after the producers of the tensors; rfk_set_stream orders the
        new stream after the context's previous one)."""
        import torch

        if dev.index is not None and dev.index != self.device:
            raise InvalidArgument(f"tensors on cuda:{dev.index}, context on cuda:{self.device}")
        s = torch.cuda.current_stream(dev).cuda_stream
        if s != getattr(self, "_stream", None):
            self.set_stream(s)

    @property
    def launches(self) -> int:
        return int(self.lib.rfk_launch_count(self.handle))

    @property
    def workspace_bytes(self) -> int:
        """Device bytes held by the context's workspace cache."""
        return int(self.lib.rfk_workspace_bytes(self.handle))

    def release_workspace(self):
        """Free the context's cached device workspace."""
        self.check(self.lib.rfk_release_workspace(self.handle))

    def check(self, st: int):
        if st != L.RFK_OK:
            msg = self.lib.rfk_last_error(self.handle).decode()
            raise _ERRORS.get(st, Error)(msg)


_contexts = {}


def context(device: Optional[int] = None) -> Context:
    """The shared context of `device` (default: the current CUDA device, so
    a rank of a multi-GPU job that called torch.cuda.set_device(local_rank)
    computes on its own GPU)."""
    if device is None:
        device = 0
        try:
            import torch

            if torch.cuda.is_available() and torch.cuda.is_initialized():
                device = torch.cuda.current_device()
        except Exception:
            pass
    if device not in _contexts:
        _contexts[device] = Context(device)
    return _contexts[device]


# ---- array plumbing --------------------------------------------------------------
def _is_dev(x) -> bool:
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if _is_dev(x):
        return x.data_ptr()
    return x.ctypes.data


class _Arrays:
    """Converts inputs to contiguous arrays of one memory kind and allocates
    outputs of the same kind."""

    def __init__(self, *xs, ctx: "Context" = None):
        devs = [_is_dev(x) for x in xs if x is not None]
        self.device = bool(devs) and all(devs)
        if any(devs) and not self.device:
            raise InvalidArgument("mix of host and device arrays")
        self.mem = L.RFK_MEM_DEVICE if self.device else L.RFK_MEM_HOST
        if self.device:
            import torch

            self.torch = torch
            self.dev = next(x for x in xs if x is not None).device
            if any(x.device != self.dev for x in xs if x is not None):
                raise InvalidArgument("arrays on different devices")
            if ctx is not None:
                ctx.bind(self.dev)

    def conv(self, x, dtype):
        if x is None:
            return None
        if self.device:
            tdt = {np.float64: self.torch.float64, np.float32: self.torch.float32, np.uint8: self.torch.uint8,
                   np.int8: self.torch.int8, np.int32: self.torch.int32}[dtype]
            return x.to(dtype=tdt).contiguous()
        return np.ascontiguousarray(x, dtype=dtype)

    def empty(self, shape, dtype):
        if self.device:
            tdt = {np.float64: self.torch.float64, np.float32: self.torch.float32, np.uint8: self.torch.uint8,
                   np.int8: self.torch.int8, np.int32: self.torch.int32,
                   np.int64: self.torch.int64}[dtype]
            return self.torch.empty(shape, dtype=tdt, device=self.dev)
        return np.empty(shape, dtype=dtype)

    def zeros(self, shape, dtype):
        z = self.empty(shape, dtype)
        z[...] = 0
        return z


@dataclass
class SolveReport:
    """SolveReport (sweeper.hpp:43-47); arrays when batched."""
    iterations: object
    converged: object
    max_delta_history: object


@dataclass
class Records:
    """Per-node StencilRecord planes (adjoint.hpp:13-30)."""
    type: object
    stencil: object
    donor1: object
    donor2: object
    c: object  # (5, ...) two-point (q11,q12,q22,u1,u2) / one-point (r_edge, e_edge)
    two_point_count: object
    one_point_count: object


def _fields(A: _Arrays, g11, g12, g22, b1, b2, src, h, fixed_values=None):
    g = [A.conv(x, np.float64) for x in (g11, g12, g22, b1, b2)]
    s = A.conv(src, np.uint8)
    fv = A.conv(fixed_values, np.float64)
    shp_p, shp_s = tuple(g[0].shape), tuple(s.shape)
    for x in g[1:]:
        if tuple(x.shape) != shp_p:
            raise DimensionMismatch("solve: field dimensions disagree with grid spec")
    if len(shp_p) not in (2, 3) or len(shp_s) not in (2, 3) or shp_p[-2:] != shp_s[-2:]:
        raise DimensionMismatch("solve: field dimensions disagree with grid spec")
    rows, cols = shp_p[-2:]
    bp = shp_p[0] if len(shp_p) == 3 else 1
    bs = shp_s[0] if len(shp_s) == 3 else 1
    batch = max(bp, bs)
    if (bp not in (1, batch)) or (bs not in (1, batch)):
        raise DimensionMismatch("batch sizes disagree")
    f = L.rfk_fields()
    f.batch, f.rows, f.cols, f.h = batch, rows, cols, float(h)
    f.g11, f.g12, f.g22, f.b1, f.b2 = (_ptr(x) for x in g)
    f.param_stride = rows * cols if (len(shp_p) == 3 and bp > 1) else 0
    f.src = _ptr(s)
    f.src_stride = rows * cols if (len(shp_s) == 3 and bs > 1) else 0
    f.fixed_values = _ptr(fv)
    keep = (g, s, fv)
    batched = len(shp_p) == 3 or len(shp_s) == 3
    return f, keep, batch, rows, cols, batched


def _opts(tol, max_iters, sweep_order):
    o = L.rfk_solve_options()
    o.tol, o.max_iters = float(tol), int(max_iters)
    for i, v in enumerate(sweep_order):
        o.sweep_order[i] = int(v)
    return o


def _solve(entry, g11, g12, g22, b1, b2, src, h, tol, max_iters, sweep_order, fixed_values, ctx):
    ctx = ctx or context()
    A = _Arrays(g11, g12, g22, b1, b2, src, fixed_values, ctx=ctx)
    f, keep, B, R, Cc, batched = _fields(A, g11, g12, g22, b1, b2, src, h, fixed_values)
    t = A.empty((B, R, Cc), np.float64)
    its = A.empty((B,), np.int32)
    conv = A.empty((B,), np.int32)
    hist = A.empty((B, max(int(max_iters), 1)), np.float64)
    o = _opts(tol, max_iters, sweep_order)
    ctx.check(getattr(ctx.lib, entry)(ctx.handle, A.mem, C.byref(f), C.byref(o), _ptr(t), _ptr(its),
                                      _ptr(conv), _ptr(hist)))
    if A.device:
        its_h, conv_h = its.cpu().numpy(), conv.cpu().numpy()
        hist_h = hist.cpu().numpy()
    else:
        its_h, conv_h, hist_h = its, conv, hist
    hists = [hist_h[b, : its_h[b]].copy() for b in range(B)]
    if not batched:
        return t[0], SolveReport(int(its_h[0]), bool(conv_h[0]), hists[0])
    return t, SolveReport(its_h.copy(), conv_h.astype(bool), hists)


def solve(g11, g12, g22, b1, b2, src, h, tol=1e-6, max_iters=50, sweep_order=(0, 1, 2, 3),
          ctx: Context = None):
    """randers::solve (sweeper.hpp:60-62)."""
    return _solve("rfk_solve", g11, g12, g22, b1, b2, src, h, tol, max_iters, sweep_order, None, ctx)


def _fields_f32(A, g11, g12, g22, b1, b2, src, h):
    """rfk_fields_f32 over float32 copies of the parameter planes."""
    if A.device:
        g = [x.to(dtype=A.torch.float32).contiguous() for x in (g11, g12, g22, b1, b2)]
    else:
        g = [np.ascontiguousarray(x, dtype=np.float32) for x in (g11, g12, g22, b1, b2)]
    s = A.conv(src, np.uint8)
    shp_p, shp_s = tuple(g[0].shape), tuple(s.shape)
    for x in g[1:]:
        if tuple(x.shape) != shp_p:
            raise DimensionMismatch("solve: field dimensions disagree with grid spec")
    if len(shp_p) not in (2, 3) or len(shp_s) not in (2, 3) or shp_p[-2:] != shp_s[-2:]:
        raise DimensionMismatch("solve: field dimensions disagree with grid spec")
    R, Cc = shp_p[-2:]
    bp = shp_p[0] if len(shp_p) == 3 else 1
    bs = shp_s[0] if len(shp_s) == 3 else 1
    B = max(bp, bs)
    batched = len(shp_p) == 3 or len(shp_s) == 3
    f = L.rfk_fields_f32()
    f.batch, f.rows, f.cols, f.h = B, R, Cc, float(h)
    f.g11, f.g12, f.g22, f.b1, f.b2 = (_ptr(x) for x in g)
    f.param_stride = R * Cc if (len(shp_p) == 3 and bp > 1) else 0
    f.src = _ptr(s)
    f.src_stride = R * Cc if (len(shp_s) == 3 and bs > 1) else 0
    return f, (g, s), B, R, Cc, batched


def solve_f32(g11, g12, g22, b1, b2, src, h, tol=1e-6, max_iters=50, sweep_order=(0, 1, 2, 3),
              ctx: Context = None):
    """The fp32 mode of solve: the same exact wavefront with
    fp32 storage and arithmetic.  Inputs are converted to float32; returns a
    float32 field.  Agrees with the fp64 solve to ~1e-6 relative."""
    ctx = ctx or context()
    A = _Arrays(g11, g12, g22, b1, b2, src, ctx=ctx)
    f, keep, B, R, Cc, batched = _fields_f32(A, g11, g12, g22, b1, b2, src, h)
    if A.device:
        t = A.torch.empty((B, R, Cc), dtype=A.torch.float32, device=A.dev)
    else:
        t = np.empty((B, R, Cc), np.float32)
    its = A.empty((B,), np.int32)
    conv = A.empty((B,), np.int32)
    hist = A.empty((B, max(int(max_iters), 1)), np.float64)
    o = _opts(tol, max_iters, sweep_order)
    ctx.check(ctx.lib.rfk_solve_f32(ctx.handle, A.mem, C.byref(f), C.byref(o), _ptr(t), _ptr(its), _ptr(conv),
                                    _ptr(hist)))
    if A.device:
        its_h, conv_h, hist_h = its.cpu().numpy(), conv.cpu().numpy(), hist.cpu().numpy()
    else:
        its_h, conv_h, hist_h = its, conv, hist
    hists = [hist_h[b, : its_h[b]].copy() for b in range(B)]
    if not batched:
        return t[0], SolveReport(int(its_h[0]), bool(conv_h[0]), hists[0])
    return t, SolveReport(its_h.copy(), conv_h.astype(bool), hists)


def solve_from_values(g11, g12, g22, b1, b2, fixed, fixed_values, h, tol=1e-6, max_iters=50,
                      sweep_order=(0, 1, 2, 3), ctx: Context = None):
    """randers::solve_from_values (sweeper.hpp:72-76)."""
    return _solve("rfk_solve", g11, g12, g22, b1, b2, fixed, h, tol, max_iters, sweep_order,
                  fixed_values, ctx)


def solve_jacobi(g11, g12, g22, b1, b2, src, h, tol=1e-6, max_iters=50, ctx: Context = None):
    """randers::solve_jacobi (sweeper.hpp:66-68)."""
    return _solve("rfk_solve_jacobi", g11, g12, g22, b1, b2, src, h, tol, max_iters, (0, 1, 2, 3),
                  None, ctx)


def jacobi_iteration_budget(rows, cols):
    """sweeper.hpp:80-82."""
    return 5 * max(rows, cols) + 50


def best_candidates(nodes, t, g11, g12, g22, b1, b2, h, node_update=False, ctx: Context = None):
    """best_candidate / node_update (sweeper.cpp:8-72) at linear node indices."""
    ctx = ctx or context()
    A = _Arrays(t, g11, g12, g22, b1, b2, ctx=ctx)
    t_ = A.conv(t, np.float64)
    R, Cc = t_.shape
    f, keep, B, _, _, _ = _fields(A, g11, g12, g22, b1, b2, A.conv(np.zeros((R, Cc), np.uint8), np.uint8)
                                  if not A.device else A.torch.zeros((R, Cc), dtype=A.torch.uint8,
                                                                     device=A.dev), h)
    nd = A.conv(nodes if not A.device else A.torch.as_tensor(np.asarray(nodes), device=A.dev),
                np.int32)
    n = int(nd.shape[0])
    out = dict(t0=A.empty((n,), np.float64), type=A.empty((n,), np.int8),
               stencil=A.empty((n,), np.int8), donor1=A.empty((n,), np.int8),
               donor2=A.empty((n,), np.int8), lam1=A.empty((n,), np.float64),
               lam2=A.empty((n,), np.float64), found=A.empty((n,), np.int8))
    ctx.check(ctx.lib.rfk_best_candidate(ctx.handle, A.mem, C.byref(f), _ptr(t_), n, _ptr(nd),
                                         int(bool(node_update)),
                                         *(_ptr(out[k]) for k in ("t0", "type", "stencil", "donor1",
                                                                  "donor2", "lam1", "lam2", "found"))))
    return out


def best_candidate(r, c, t, g11, g12, g22, b1, b2, h, ctx: Context = None):
    cols = np.shape(t)[1]
    o = best_candidates(np.array([r * cols + c], np.int32), t, g11, g12, g22, b1, b2, h, False, ctx)
    return {k: (np.asarray(v.cpu() if _is_dev(v) else v)[0]) for k, v in o.items()}


def node_update(r, c, t, g11, g12, g22, b1, b2, h, ctx: Context = None):
    cols = np.shape(t)[1]
    o = best_candidates(np.array([r * cols + c], np.int32), t, g11, g12, g22, b1, b2, h, True, ctx)
    return {k: (np.asarray(v.cpu() if _is_dev(v) else v)[0]) for k, v in o.items()}


def two_point_update(t1, t2, m1, m2, g, b, ctx: Context = None):
    """two_point_update (stencil.cpp:7-43), elementwise over arrays."""
    ctx = ctx or context()
    arrs = [np.ascontiguousarray(np.atleast_1d(x), np.float64) for x in
            (t1, t2, m1[0], m1[1], m2[0], m2[1], g[0], g[1], g[2], b[0], b[1])]
    n = max(a.size for a in arrs)
    arrs = [np.ascontiguousarray(np.broadcast_to(a, (n,))) for a in arrs]
    t0, l1, l2 = (np.empty(n) for _ in range(3))
    v = np.empty(n, np.int8)
    ctx.check(ctx.lib.rfk_two_point_update(ctx.handle, L.RFK_MEM_HOST, n, *(a.ctypes.data for a in arrs),
                                           t0.ctypes.data, l1.ctypes.data, l2.ctypes.data, v.ctypes.data))
    return t0, l1, l2, v.astype(bool)


def _records_struct(rec_arrays):
    r = L.rfk_records()
    r.type, r.stencil, r.donor1, r.donor2 = (_ptr(x) for x in rec_arrays[:4])
    for k in range(5):
        r.c[k] = _ptr(rec_arrays[4][k])
    return r


def identify_stencils(t, g11, g12, g22, b1, b2, src, h, tol=1e-6, ctx: Context = None) -> Records:
    """identify_stencils (adjoint.hpp:31-33) as per-node planes."""
    ctx = ctx or context()
    A = _Arrays(t, g11, g12, g22, b1, b2, src, ctx=ctx)
    f, keep, B, R, Cc, batched = _fields(A, g11, g12, g22, b1, b2, src, h)
    t_ = A.conv(t, np.float64)
    shp = (B, R, Cc)
    planes = [A.empty(shp, np.int8) for _ in range(4)] + [A.empty((5,) + shp, np.float64)]
    rs = _records_struct(planes)
    n2, n1, bad = (np.zeros(B, np.int32), np.zeros(B, np.int32), np.zeros(B, np.int64))
    if A.device:
        n2d, n1d, badd = (A.empty((B,), np.int32), A.empty((B,), np.int32), A.empty((B,), np.int64))
        st = ctx.lib.rfk_identify(ctx.handle, A.mem, C.byref(f), _ptr(t_), float(tol), C.byref(rs),
                                  _ptr(n2d), _ptr(n1d), _ptr(badd))
        ctx.check(st)
        n2, n1 = n2d.cpu().numpy(), n1d.cpu().numpy()
    else:
        ctx.check(ctx.lib.rfk_identify(ctx.handle, A.mem, C.byref(f), _ptr(t_), float(tol), C.byref(rs),
                                       n2.ctypes.data, n1.ctypes.data, bad.ctypes.data))
    c = planes[4]
    if not batched:
        return Records(planes[0][0], planes[1][0], planes[2][0], planes[3][0], c[:, 0], int(n2[0]),
                       int(n1[0]))
    return Records(*planes[:4], c, n2, n1)


def jacobian_entries(type_, c, ctx: Context = None):
    ctx = ctx or context()
    ty = np.ascontiguousarray(np.atleast_1d(type_), np.int8)
    cc = [np.ascontiguousarray(np.broadcast_to(np.atleast_1d(x), ty.shape), np.float64) for x in c]
    n = ty.size
    d, j0, j1 = (np.empty(n) for _ in range(3))
    cl = np.empty(n, np.int8)
    ctx.check(ctx.lib.rfk_jacobian_entries(ctx.handle, L.RFK_MEM_HOST, n, ty.ctypes.data,
                                           *(x.ctypes.data for x in cc), d.ctypes.data, j0.ctypes.data,
                                           j1.ctypes.data, cl.ctypes.data))
    return d, j0, j1, cl.astype(bool)


def _rec_planes(A: _Arrays, rec: Records):
    c = rec.c
    if A.device:
        c = A.torch.stack([A.conv(c[k], np.float64) for k in range(5)])
    else:
        c = np.stack([np.ascontiguousarray(c[k], np.float64) for k in range(5)])
    return [A.conv(rec.type, np.int8), A.conv(rec.stencil, np.int8), A.conv(rec.donor1, np.int8),
            A.conv(rec.donor2, np.int8), c]


def solve_adjoint(rec: Records, t, loss_grad, ctx: Context = None):
    """solve_adjoint (adjoint.hpp:54-55): returns (lambda, clamped_diagonals)."""
    ctx = ctx or context()
    A = _Arrays(t, loss_grad, rec.type, ctx=ctx)
    t_ = A.conv(t, np.float64)
    R, Cc = t_.shape[-2:]
    B = 1 if t_.ndim == 2 else t_.shape[0]
    planes = _rec_planes(A, rec)
    rs = _records_struct(planes)
    g = A.conv(loss_grad, np.float64)
    lam = A.empty(tuple(t_.shape), np.float64)
    cl = A.empty((B,), np.int32)
    ctx.check(ctx.lib.rfk_solve_adjoint(ctx.handle, A.mem, B, R, Cc, _ptr(t_), C.byref(rs), _ptr(g),
                                        _ptr(lam), _ptr(cl)))
    clh = cl.cpu().numpy() if A.device else cl
    return lam, (int(clh[0]) if t_.ndim == 2 else clh)


def param_gradients(rec: Records, lam, h, ctx: Context = None):
    """param_gradients (adjoint.hpp:71): (5, ...) = g11, g12, g22, b1, b2."""
    ctx = ctx or context()
    A = _Arrays(lam, rec.type, ctx=ctx)
    lam_ = A.conv(lam, np.float64)
    R, Cc = lam_.shape[-2:]
    B = 1 if lam_.ndim == 2 else lam_.shape[0]
    planes = _rec_planes(A, rec)
    rs = _records_struct(planes)
    out = A.empty((5,) + tuple(lam_.shape), np.float64)
    ctx.check(ctx.lib.rfk_param_gradients(ctx.handle, A.mem, B, R, Cc, float(h), C.byref(rs), _ptr(lam_),
                                          *(_ptr(out[k]) for k in range(5))))
    return out


def loss_grad_mse(t, observed, values, exact=True, ctx: Context = None):
    """loss_grad_mse (adjoint.hpp:81): (grad, loss, unreached_observed)."""
    ctx = ctx or context()
    A = _Arrays(t, observed, values, ctx=ctx)
    t_ = A.conv(t, np.float64)
    obs = A.conv(observed, np.uint8)
    val = A.conv(values, np.float64)
    B = 1 if t_.ndim == 2 else t_.shape[0]
    n = int(t_.shape[-1] * t_.shape[-2])
    grad = A.empty(tuple(t_.shape), np.float64)
    loss = A.empty((B,), np.float64)
    unr = A.empty((B,), np.int32)
    ctx.check(ctx.lib.rfk_loss_grad_mse(ctx.handle, A.mem, B, n, _ptr(t_), _ptr(obs), _ptr(val), _ptr(grad),
                                        _ptr(loss), _ptr(unr), int(bool(exact))))
    if t_.ndim == 2:
        lh = loss.cpu().numpy() if A.device else loss
        uh = unr.cpu().numpy() if A.device else unr
        return grad, float(lh[0]), int(uh[0])
    return grad, loss, unr


def backward(t, g11, g12, g22, b1, b2, src, h, loss_grad, tol=1e-6, accumulate=False,
             want_lambda=True, ctx: Context = None):
    """Fused identify -> adjoint -> param gradients (the body of
    adjoint_gradient, oracle.cpp:226-247).  Returns (lambda, grads(5,...), clamped)."""
    ctx = ctx or context()
    A = _Arrays(t, g11, g12, g22, b1, b2, src, loss_grad, ctx=ctx)
    f, keep, B, R, Cc, batched = _fields(A, g11, g12, g22, b1, b2, src, h)
    t_ = A.conv(t, np.float64)
    lg = A.conv(loss_grad, np.float64)
    acc = bool(accumulate) and f.param_stride == 0
    gshape = (5, R, Cc) if acc or not batched else (5, B, R, Cc)
    grads = A.empty(gshape, np.float64)
    lam = A.empty(tuple(t_.shape), np.float64) if want_lambda else None
    cl = A.empty((B,), np.int32)
    bad = np.zeros(B, np.int64)
    ctx.check(ctx.lib.rfk_backward(ctx.handle, A.mem, C.byref(f), _ptr(t_), float(tol), _ptr(lg), _ptr(lam),
                                   *(_ptr(grads[k]) for k in range(5)), int(acc), _ptr(cl),
                                   bad.ctypes.data if not A.device else None))
    clh = cl.cpu().numpy() if A.device else cl
    return lam, grads, (int(clh[0]) if not batched else clh)


def backward_f32(t, g11, g12, g22, b1, b2, src, h, loss_grad, tol=1e-6, accumulate=False, ctx: Context = None):
    """The backward of the fp32 mode (rfk_backward_f32): float32 arrival field,
    parameters and loss gradient in, float32 gradients out; the identify ->
    adjoint -> gradient arithmetic runs in fp64 on the widened values.
    Returns (grads(5,...), clamped) with :func:`backward`'s shapes."""
    ctx = ctx or context()
    A = _Arrays(t, g11, g12, g22, b1, b2, src, loss_grad, ctx=ctx)
    f, keep, B, R, Cc, batched = _fields_f32(A, g11, g12, g22, b1, b2, src, h)
    t_ = A.conv(t, np.float32)
    lg = A.conv(loss_grad, np.float32)
    acc = bool(accumulate) and f.param_stride == 0
    gshape = (5, R, Cc) if acc or not batched else (5, B, R, Cc)
    grads = A.empty(gshape, np.float32)
    cl = A.empty((B,), np.int32)
    bad = np.zeros(B, np.int64)
    ctx.check(ctx.lib.rfk_backward_f32(ctx.handle, A.mem, C.byref(f), _ptr(t_), float(tol), _ptr(lg),
                                       *(_ptr(grads[k]) for k in range(5)), int(acc), _ptr(cl),
                                       bad.ctypes.data if not A.device else None))
    clh = cl.cpu().numpy() if A.device else cl
    return grads, (int(clh[0]) if not batched else clh)


@dataclass
class Projection:
    """ProjectionConfig (feasibility.hpp:9-21) plus which projections run:
    mode 1 project_spd, 2 project_drift, 3 both (ParamView::project, Joint)."""
    mode: int = 3
    eps_min: float = 1e-3
    lambda_max: float = 1e3
    tau: float = 0.95
    euclid_cap: float = 10.0

    def to_c(self):
        return L.rfk_projection(int(self.mode), float(self.eps_min), float(self.lambda_max), float(self.tau),
                                float(self.euclid_cap))


def solve_projected(g11, g12, g22, b1, b2, src, h, proj: Projection, tol=1e-6, max_iters=50,
                    sweep_order=(0, 1, 2, 3), ctx: Context = None):
    """solve on raw parameters with the feasibility projection fused into the
    load stage (rfk_solve_projected).  Returns (t, report, projected planes
    (5, ...)) -- bitwise what project_spd / project_drift followed by solve
    give."""
    ctx = ctx or context()
    A = _Arrays(g11, g12, g22, b1, b2, src, ctx=ctx)
    f, keep, B, R, Cc, batched = _fields(A, g11, g12, g22, b1, b2, src, h)
    t = A.empty((B, R, Cc), np.float64)
    its = A.empty((B,), np.int32)
    conv = A.empty((B,), np.int32)
    hist = A.empty((B, max(int(max_iters), 1)), np.float64)
    pshape = tuple(keep[0][0].shape)
    planes = [A.empty(pshape, np.float64) for _ in range(5)]
    pp = (C.c_void_p * 5)(*[_ptr(x) for x in planes])
    o = _opts(tol, max_iters, sweep_order)
    pc = proj.to_c()
    ctx.check(ctx.lib.rfk_solve_projected(ctx.handle, A.mem, C.byref(f), C.byref(pc), C.byref(o), _ptr(t), _ptr(its),
                                          _ptr(conv), _ptr(hist), pp))
    if A.device:
        its_h, conv_h, hist_h = its.cpu().numpy(), conv.cpu().numpy(), hist.cpu().numpy()
    else:
        its_h, conv_h, hist_h = its, conv, hist
    hists = [hist_h[b, : its_h[b]].copy() for b in range(B)]
    stack = A.torch.stack if A.device else np.stack
    if not batched:
        return t[0], SolveReport(int(its_h[0]), bool(conv_h[0]), hists[0]), stack(planes)
    return t, SolveReport(its_h.copy(), conv_h.astype(bool), hists), stack(planes)


def backward_projected(t, g11, g12, g22, b1, b2, projected, src, h, loss_grad, proj: Projection, tol=1e-6,
                       accumulate=False, want_lambda=True, ctx: Context = None):
    """backward with gradients with respect to the raw parameters: the
    projection's VJP runs inside the gradient pass (rfk_backward_projected).
    `projected` = the planes solve_projected returned."""
    ctx = ctx or context()
    A = _Arrays(t, g11, g12, g22, b1, b2, src, loss_grad, ctx=ctx)
    f, keep, B, R, Cc, batched = _fields(A, g11, g12, g22, b1, b2, src, h)
    pl = [A.conv(projected[k], np.float64) for k in range(5)]
    pp = (C.c_void_p * 5)(*[_ptr(x) for x in pl])
    t_ = A.conv(t, np.float64)
    lg = A.conv(loss_grad, np.float64)
    acc = bool(accumulate) and f.param_stride == 0
    gshape = (5, R, Cc) if acc or not batched else (5, B, R, Cc)
    grads = A.empty(gshape, np.float64)
    lam = A.empty(tuple(t_.shape), np.float64) if want_lambda else None
    cl = A.empty((B,), np.int32)
    bad = np.zeros(B, np.int64)
    pc = proj.to_c()
    ctx.check(ctx.lib.rfk_backward_projected(ctx.handle, A.mem, C.byref(f), C.byref(pc), pp, _ptr(t_), float(tol),
                                             _ptr(lg), _ptr(lam), *(_ptr(grads[k]) for k in range(5)), int(acc),
                                             _ptr(cl), bad.ctypes.data if not A.device else None))
    clh = cl.cpu().numpy() if A.device else cl
    return lam, grads, (int(clh[0]) if not batched else clh)


def project_spd(g11, g12, g22, eps_min=1e-3, lambda_max=1e3, ctx: Context = None):
    """project_spd (feasibility.hpp:27-31); returns projected copies."""
    ctx = ctx or context()
    A = _Arrays(g11, g12, g22, ctx=ctx)
    a, b, c = (A.conv(x, np.float64) for x in (g11, g12, g22))
    a, b, c = (x.clone() if A.device else x.copy() for x in (a, b, c))
    n = int(np.prod(tuple(a.shape)))
    ctx.check(ctx.lib.rfk_project_spd(ctx.handle, A.mem, n, _ptr(a), _ptr(b), _ptr(c), float(eps_min),
                                      float(lambda_max)))
    return a, b, c


def project_drift(b1, b2, g11, g12, g22, tau=0.95, euclid_cap=10.0, ctx: Context = None):
    """project_drift (feasibility.hpp:35-40); returns projected copies."""
    ctx = ctx or context()
    A = _Arrays(b1, b2, g11, g12, g22, ctx=ctx)
    x, y = (A.conv(v, np.float64) for v in (b1, b2))
    x, y = (v.clone() if A.device else v.copy() for v in (x, y))
    g = [A.conv(v, np.float64) for v in (g11, g12, g22)]
    n = int(np.prod(tuple(x.shape)))
    ctx.check(ctx.lib.rfk_project_drift(ctx.handle, A.mem, n, _ptr(x), _ptr(y), *(_ptr(v) for v in g),
                                        float(tau), float(euclid_cap)))
    return x, y


def drift_norm_sq(b1, b2, g11, g12, g22, ctx: Context = None):
    ctx = ctx or context()
    A = _Arrays(b1, b2, g11, g12, g22, ctx=ctx)
    v = [A.conv(x, np.float64) for x in (b1, b2, g11, g12, g22)]
    out = A.empty(tuple(v[0].shape), np.float64)
    n = int(np.prod(tuple(v[0].shape)))
    ctx.check(ctx.lib.rfk_drift_norm_sq(ctx.handle, A.mem, n, *(_ptr(x) for x in v), _ptr(out)))
    return out


# ---- projection VJP (not in the reference) ------------

def _cot(A, x):
    x = A.conv(x, np.float64)
    return x.clone() if A.device else x.copy()


def project_spd_vjp(g11, g12, g22, d_g11, d_g12, d_g22, eps_min=1e-3, lambda_max=1e3, ctx: Context = None):
    """Cotangents of project_spd's inputs from those of its outputs.

    (g11, g12, g22) are the PRE-projection channels; returns (d_g11, d_g12,
    d_g22) w.r.t. them (new arrays).  Daleckii-Krein on the eigenvalue clamp
    of feasibility.cpp:31-44; identity where the node passes through."""
    ctx = ctx or context()
    A = _Arrays(g11, g12, g22, d_g11, d_g12, d_g22, ctx=ctx)
    g = [A.conv(v, np.float64) for v in (g11, g12, g22)]
    d = [_cot(A, v) for v in (d_g11, d_g12, d_g22)]
    n = int(np.prod(tuple(g[0].shape)))
    ctx.check(ctx.lib.rfk_project_spd_vjp(ctx.handle, A.mem, n, *(_ptr(v) for v in g), float(eps_min),
                                          float(lambda_max), *(_ptr(v) for v in d)))
    return tuple(d)


def project_drift_vjp(b1, b2, g11, g12, g22, d_b1, d_b2, tau=0.95, euclid_cap=10.0, metric_grad=True,
                      d_metric=None, ctx: Context = None):
    """Cotangents through project_drift (feasibility.cpp:51-72) against a
    fixed metric.  Returns (d_b1, d_b2) and, if metric_grad, the metric's
    cotangent (d_g11, d_g12, d_g22) through the drift norm, accumulated onto
    d_metric (three planes) when given, else onto zeros."""
    ctx = ctx or context()
    A = _Arrays(b1, b2, g11, g12, g22, d_b1, d_b2, ctx=ctx)
    v = [A.conv(x, np.float64) for x in (b1, b2, g11, g12, g22)]
    db = [_cot(A, x) for x in (d_b1, d_b2)]
    if metric_grad and d_metric is not None:
        dg = [_cot(A, x) for x in d_metric]
    else:
        dg = [A.zeros(tuple(v[0].shape), np.float64) for _ in range(3)] if metric_grad else [None] * 3
    n = int(np.prod(tuple(v[0].shape)))
    ctx.check(ctx.lib.rfk_project_drift_vjp(ctx.handle, A.mem, n, *(_ptr(x) for x in v), float(tau),
                                            float(euclid_cap), *(_ptr(x) for x in db),
                                            *(_ptr(x) if x is not None else None for x in dg)))
    return (db[0], db[1], *dg) if metric_grad else (db[0], db[1])


def project_vjp(g11, g12, g22, b1, b2, d_g11, d_g12, d_g22, d_b1, d_b2, eps_min=1e-3, lambda_max=1e3,
                tau=0.95, euclid_cap=10.0, ctx: Context = None):
    """Cotangents through ParamView::project for the Joint parameterization
    (inversion.cpp:276-279: project_spd, then project_drift against the
    projected metric).  Inputs are the pre-projection channels; returns the
    five cotangent planes w.r.t. them."""
    ctx = ctx or context()
    A = _Arrays(g11, g12, g22, b1, b2, d_g11, d_g12, d_g22, d_b1, d_b2, ctx=ctx)
    v = [A.conv(x, np.float64) for x in (g11, g12, g22, b1, b2)]
    d = [_cot(A, x) for x in (d_g11, d_g12, d_g22, d_b1, d_b2)]
    n = int(np.prod(tuple(v[0].shape)))
    ctx.check(ctx.lib.rfk_project_vjp(ctx.handle, A.mem, n, *(_ptr(x) for x in v), float(eps_min),
                                      float(lambda_max), float(tau), float(euclid_cap), *(_ptr(x) for x in d)))
    return tuple(d)


# ---- fused objective (objective_and_grad, inversion.cpp:25-73) ------------------

@dataclass
class Objective:
    """Objective (inversion.hpp:47-53) without the caller-side regularizer."""
    data_loss: float
    unreached_observed: int
    grad: object  # (5, rows, cols): d/d(g11, g12, g22, b1, b2)


def objective_and_grad(g11, g12, g22, b1, b2, sources, observed, values, h, solve_tol=1e-6,
                       solve_max_iters=50, unreached_penalty_cap=1e4, exact=True, out=None,
                       ctx: Context = None):
    """Data term of randers::objective_and_grad over K observation sets in one call.

    sources/observed/values: (K, rows, cols) or (rows, cols).  The loss and the
    gradient accumulation follow the reference's order; with exact=True the loss
    sum is bit-identical to it.  `out` may supply the (5, rows, cols) gradient
    buffer (e.g. pinned host memory).  Raises NotConverged like the reference."""
    ctx = ctx or context()
    A = _Arrays(g11, g12, g22, b1, b2, sources, observed, values, out, ctx=ctx)
    g = [A.conv(x, np.float64) for x in (g11, g12, g22, b1, b2)]
    src = A.conv(sources, np.uint8)
    obs = A.conv(observed, np.uint8)
    val = A.conv(values, np.float64)
    rows, cols = tuple(g[0].shape)[-2:]
    for x in g:
        if tuple(x.shape) != (rows, cols):
            raise DimensionMismatch("objective_and_grad: field dimensions disagree with grid spec")
    K = 1 if src.ndim == 2 else int(src.shape[0])
    for x in (src, obs, val):
        if tuple(x.shape)[-2:] != (rows, cols) or (1 if x.ndim == 2 else int(x.shape[0])) != K:
            raise DimensionMismatch("objective_and_grad: observation planes disagree with grid spec")
    f = L.rfk_fields()
    f.batch, f.rows, f.cols, f.h = 1, rows, cols, float(h)
    f.g11, f.g12, f.g22, f.b1, f.b2 = (_ptr(x) for x in g)
    ob = L.rfk_observations()
    ob.count, ob.sources, ob.observed, ob.values = K, _ptr(src), _ptr(obs), _ptr(val)
    o = L.rfk_objective_options()
    o.solve_tol, o.solve_max_iters = float(solve_tol), int(solve_max_iters)
    o.unreached_penalty_cap, o.exact_sum = float(unreached_penalty_cap), int(bool(exact))
    grads = out if out is not None else A.empty((5, rows, cols), np.float64)
    dl = C.c_double(0.0)
    un = C.c_int32(0)
    ctx.check(ctx.lib.rfk_objective_and_grad(ctx.handle, A.mem, C.byref(f), C.byref(ob), C.byref(o),
                                             C.addressof(dl), C.addressof(un),
                                             *(_ptr(grads[k]) for k in range(5))))
    return Objective(dl.value, un.value, grads)
