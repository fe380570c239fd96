"""Host-side mirror of the reference's recovery API (proj/include/randers/
inversion.hpp and the regularizers of feasibility.hpp) on top of the C ABI.

``recover`` runs the whole projected first-order loop in librfk.so: the
parameter channels, Adam moments and gradients stay on the device, and only
one objective value per iteration reaches the host.  With
``InverseConfig.exact_sum`` the sums the reference takes sequentially (loss,
TV value, clip norm, relative error) are replayed in node order, which makes
every history and field bit-identical to the reference's ``recover``.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L
from .api import Context, DimensionMismatch, InvalidArgument, _Arrays, _ptr, context


class Parameterization(enum.IntEnum):  # inversion.hpp:12
    Isotropic = 0
    Diagonal = 1
    Full = 2
    DriftOnly = 3
    Joint = 4


class OptimizerKind(enum.IntEnum):  # inversion.hpp:13
    Adam = 0
    Gd = 1


class TvVariant(enum.IntEnum):  # feasibility.hpp:46
    Frobenius = 0
    LogEuclidean = 1
    Drift = 2


@dataclass
class InverseConfig:
    """InverseConfig (inversion.hpp:15-45) with ProjectionConfig's fields flattened."""
    param: Parameterization = Parameterization.Isotropic
    optimizer: OptimizerKind = OptimizerKind.Adam
    step_g: float = 1e-2
    step_b: float = 5e-3
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    grad_clip_norm: float = 1.0
    lambda_g: float = 0.0
    lambda_b: float = 0.0
    tv_variant: TvVariant = TvVariant.Frobenius
    iters: int = 300
    eps_min: float = 1e-3
    lambda_max: float = 1e3
    tau: float = 0.95
    euclid_cap: float = 10.0
    solve_tol: float = 1e-6
    solve_max_iters: int = 50
    plateau_window: int = 25
    plateau_factor: float = 0.5
    unreached_penalty_cap: float = 1e4
    exact_sum: bool = False

    def to_c(self) -> L.rfk_inverse_config:
        c = L.rfk_inverse_config()
        for name, _ in L.rfk_inverse_config._fields_:
            v = getattr(self, name)
            setattr(c, name, int(v) if name in ("param", "optimizer", "tv_variant", "iters", "solve_max_iters",
                                                "plateau_window", "exact_sum") else float(v))
        return c

    def to_reference(self) -> np.ndarray:
        """The flat array oracle/ref_capi.cpp's config_of() reads (tests only)."""
        return np.array([self.param, self.optimizer, self.step_g, self.step_b, self.beta1, self.beta2,
                         self.adam_eps, self.grad_clip_norm, self.lambda_g, self.lambda_b, self.tv_variant,
                         self.iters, self.eps_min, self.lambda_max, self.tau, self.euclid_cap, self.solve_tol,
                         self.solve_max_iters, self.plateau_window, self.plateau_factor,
                         self.unreached_penalty_cap], dtype=np.float64)


def _plane_ptrs(xs):
    arr = (C.c_void_p * max(1, len(xs)))(*[_ptr(x) for x in xs])
    return arr


def _planes(A: _Arrays, xs, shape=None):
    out = [A.conv(x, np.float64) for x in xs]
    shp = tuple(out[0].shape) if shape is None else shape
    for x in out:
        if tuple(x.shape) != shp:
            raise DimensionMismatch("channel shapes")
    return out


def tv_value_grad(channels: Sequence, variant: TvVariant = TvVariant.Frobenius, eps_tv: float = 1e-8,
                  exact: bool = True, ctx: Context = None):
    """tv_value_grad (feasibility.cpp:137-182) -> (value, [grad planes])."""
    ctx = ctx or context()
    if len(channels) < 1 or len(channels) > 3:
        raise InvalidArgument("tv_value_grad: need 1..3 channels")
    A = _Arrays(*channels, ctx=ctx)
    ch = _planes(A, channels)
    if len(ch[0].shape) != 2:
        raise DimensionMismatch("tv_value_grad: channel shapes")
    rows, cols = tuple(ch[0].shape)
    grads = [A.empty((rows, cols), np.float64) for _ in ch]
    v = C.c_double(0.0)
    ctx.check(ctx.lib.rfk_tv_value_grad(ctx.handle, A.mem, rows, cols, len(ch), int(variant), float(eps_tv),
                                        _plane_ptrs(ch), _plane_ptrs(grads), C.addressof(v), int(bool(exact))))
    return v.value, grads


def tikhonov_value_grad(channels: Sequence, weight: float, exact: bool = True, ctx: Context = None):
    """tikhonov_value_grad (feasibility.cpp:184-196) -> (value, [grad planes])."""
    ctx = ctx or context()
    if not channels:
        return 0.0, []
    A = _Arrays(*channels, ctx=ctx)
    ch = _planes(A, channels)
    grads = [A.empty(tuple(ch[0].shape), np.float64) for _ in ch]
    v = C.c_double(0.0)
    n = int(np.prod(tuple(ch[0].shape)))
    ctx.check(ctx.lib.rfk_tikhonov_value_grad(ctx.handle, A.mem, n, len(ch), float(weight), _plane_ptrs(ch),
                                              _plane_ptrs(grads), C.addressof(v), int(bool(exact))))
    return v.value, grads


def clip_global_norm(grads: Sequence, max_norm: float, exact: bool = True, ctx: Context = None) -> float:
    """clip_global_norm (inversion.cpp:75-88): scales `grads` in place (they
    must be contiguous float64 arrays/tensors) and returns the pre-clip norm."""
    ctx = ctx or context()
    A = _Arrays(*grads, ctx=ctx)
    for g in grads:
        ok = g.is_contiguous() if A.device else (g.flags["C_CONTIGUOUS"] and g.dtype == np.float64)
        if not ok:
            raise InvalidArgument("clip_global_norm: planes must be contiguous float64")
    n = int(np.prod(tuple(grads[0].shape)))
    norm = C.c_double(0.0)
    ctx.check(ctx.lib.rfk_clip_global_norm(ctx.handle, A.mem, n, len(grads), _plane_ptrs(list(grads)),
                                           float(max_norm), C.addressof(norm), int(bool(exact))))
    return norm.value


class AdamState:
    """AdamState (inversion.hpp:62-65): moments allocated on the first step."""

    def __init__(self):
        self.m = []
        self.v = []
        self.t = 0


def _check_inplace(A, xs, what):
    for x in xs:
        ok = x.is_contiguous() and x.dtype == A.torch.float64 if A.device else (
            x.flags["C_CONTIGUOUS"] and x.dtype == np.float64)
        if not ok:
            raise InvalidArgument(f"{what}: parameters must be contiguous float64")


def adam_step(state: AdamState, params: Sequence, grads: Sequence, steps: Sequence[float],
              cfg: InverseConfig = None, exact: bool = True, ctx: Context = None):
    """adam_step (inversion.cpp:90-116): updates `params` in place; the grads
    are clipped as a copy, as the reference takes them by value."""
    ctx = ctx or context()
    cfg = cfg or InverseConfig()
    A = _Arrays(*params, *grads, ctx=ctx)
    _check_inplace(A, params, "adam_step")
    g = _planes(A, grads, tuple(params[0].shape))
    if not state.m:
        state.m = [A.zeros(tuple(p.shape), np.float64) for p in params]
        state.v = [A.zeros(tuple(p.shape), np.float64) for p in params]
    n = int(np.prod(tuple(params[0].shape)))
    t = C.c_int64(state.t)
    st = (C.c_double * len(params))(*[float(s) for s in steps])
    ctx.check(ctx.lib.rfk_adam_step(ctx.handle, A.mem, n, len(params), _plane_ptrs(list(params)),
                                    _plane_ptrs(state.m), _plane_ptrs(state.v), C.addressof(t), _plane_ptrs(g), st,
                                    float(cfg.beta1), float(cfg.beta2), float(cfg.adam_eps),
                                    float(cfg.grad_clip_norm), int(bool(exact))))
    state.t = t.value


def gd_step(params: Sequence, grads: Sequence, steps: Sequence[float], cfg: InverseConfig = None,
            exact: bool = True, ctx: Context = None):
    """gd_step (inversion.cpp:118-127): updates `params` in place."""
    ctx = ctx or context()
    cfg = cfg or InverseConfig()
    A = _Arrays(*params, *grads, ctx=ctx)
    _check_inplace(A, params, "gd_step")
    g = _planes(A, grads, tuple(params[0].shape))
    n = int(np.prod(tuple(params[0].shape)))
    st = (C.c_double * len(params))(*[float(s) for s in steps])
    ctx.check(ctx.lib.rfk_gd_step(ctx.handle, A.mem, n, len(params), _plane_ptrs(list(params)), _plane_ptrs(g), st,
                                  float(cfg.grad_clip_norm), int(bool(exact))))


def relative_error(est: Sequence, truth: Sequence, exact: bool = True, ctx: Context = None) -> float:
    """relative_error (inversion.cpp:129-138)."""
    ctx = ctx or context()
    A = _Arrays(*est, *truth, ctx=ctx)
    e = _planes(A, est)
    t = _planes(A, truth, tuple(e[0].shape))
    out = C.c_double(0.0)
    n = int(np.prod(tuple(e[0].shape)))
    ctx.check(ctx.lib.rfk_relative_error(ctx.handle, A.mem, n, len(e), _plane_ptrs(e), _plane_ptrs(t),
                                         C.addressof(out), int(bool(exact))))
    return out.value


def _obs(A: _Arrays, sources, observed, values, rows, cols):
    src = A.conv(sources, np.uint8)
    obs = A.conv(observed, np.uint8)
    val = A.conv(values, np.float64)
    K = 1 if src.ndim == 2 else int(src.shape[0])
    for x in (src, obs, val):
        if tuple(x.shape)[-2:] != (rows, cols) or (1 if x.ndim == 2 else int(x.shape[0])) != K:
            raise DimensionMismatch("observation planes disagree with grid spec")
    ob = L.rfk_observations()
    ob.count, ob.sources, ob.observed, ob.values = K, _ptr(src), _ptr(obs), _ptr(val)
    return ob, (src, obs, val)


@dataclass
class FullObjective:
    """Objective (inversion.hpp:49-55)."""
    loss: float
    data_loss: float
    reg_loss: float
    unreached_observed: int
    grad: object  # (5, rows, cols): g11, g12, g22, b1, b2


def objective(g11, g12, g22, b1, b2, sources, observed, values, h, cfg: InverseConfig = None,
              ctx: Context = None) -> FullObjective:
    """randers::objective_and_grad with the TV regularizers (inversion.cpp:25-73)."""
    ctx = ctx or context()
    cfg = cfg or InverseConfig()
    A = _Arrays(g11, g12, g22, b1, b2, sources, observed, values, ctx=ctx)
    g = _planes(A, (g11, g12, g22, b1, b2))
    rows, cols = tuple(g[0].shape)[-2:]
    ob, keep = _obs(A, sources, observed, values, rows, cols)
    f = L.rfk_fields()
    f.batch, f.rows, f.cols, f.h = 1, rows, cols, float(h)
    f.g11, f.g12, f.g22, f.b1, f.b2 = (_ptr(x) for x in g)
    c = cfg.to_c()
    out = L.rfk_objective_value()
    grads = A.empty((5, rows, cols), np.float64)
    ctx.check(ctx.lib.rfk_objective(ctx.handle, A.mem, C.byref(f), C.byref(ob), C.byref(c), C.byref(out),
                                    *(_ptr(grads[k]) for k in range(5))))
    return FullObjective(out.loss, out.data_loss, out.reg_loss, out.unreached_observed, grads)


@dataclass
class RecoveryResult:
    """RecoveryResult (inversion.hpp:83-93)."""
    metric: tuple
    drift: tuple
    iso_g: Optional[object]
    loss_history: np.ndarray
    error_history: np.ndarray
    iterations: int
    final_error: float
    unreached_observed_total: int


def recover(sources, observed, values, h, cfg: InverseConfig = None, init_metric=None, init_drift=None,
            truth_metric=None, truth_drift=None, ctx: Context = None) -> RecoveryResult:
    """randers::recover (inversion.cpp:327-385) on the device.

    sources/observed/values: (K, rows, cols) observation sets.  init_*/truth_*:
    (g11, g12, g22) / (b1, b2) plane tuples or None."""
    ctx = ctx or context()
    cfg = cfg or InverseConfig()
    extra = [x for t in (init_metric, init_drift, truth_metric, truth_drift) if t is not None for x in t]
    A = _Arrays(sources, observed, values, *extra, ctx=ctx)
    src = A.conv(sources, np.uint8)
    rows, cols = tuple(src.shape)[-2:]
    ob, keep = _obs(A, sources, observed, values, rows, cols)

    def planes(t, k):
        if t is None:
            return None, None
        if len(t) != k:
            raise InvalidArgument("recover: wrong number of planes")
        p = _planes(A, t, (rows, cols))
        return p, _plane_ptrs(p)

    im, imp = planes(init_metric, 3)
    idr, idp = planes(init_drift, 2)
    tm, tmp = planes(truth_metric, 3)
    td, tdp = planes(truth_drift, 2)
    outs = [A.empty((rows, cols), np.float64) for _ in range(6)]
    iters = max(1, int(cfg.iters))
    loss_h = np.zeros(iters, np.float64)
    err_h = np.zeros(iters, np.float64)
    r = L.rfk_recovery()
    r.g11, r.g12, r.g22, r.b1, r.b2, r.iso_g = (_ptr(x) for x in outs)
    r.loss_history = loss_h.ctypes.data
    r.error_history = err_h.ctypes.data
    c = cfg.to_c()
    ctx.check(ctx.lib.rfk_recover(ctx.handle, A.mem, rows, cols, float(h), C.byref(ob), C.byref(c), imp, idp, tmp,
                                  tdp, C.byref(r)))
    has_truth = truth_metric is not None or truth_drift is not None
    it = int(r.iterations)
    return RecoveryResult(tuple(outs[:3]), tuple(outs[3:5]),
                          outs[5] if cfg.param == Parameterization.Isotropic else None, loss_h[:it],
                          err_h[:it] if has_truth else np.zeros(0), it, float(r.final_error),
                          int(r.unreached_observed_total))


def generate_observations(g11, g12, g22, b1, b2, sources, h, density, noise_level=0.0, seed=0,
                          ctx: Context = None):
    """randers::generate_observations (inversion.cpp:387-437): the solves run on
    the device, the sampling is the reference's host code.  Returns
    (observed uint8, values float64), each (K, rows, cols)."""
    ctx = ctx or context()
    A = _Arrays(g11, g12, g22, b1, b2, sources, ctx=ctx)
    g = _planes(A, (g11, g12, g22, b1, b2))
    rows, cols = tuple(g[0].shape)[-2:]
    src = A.conv(sources, np.uint8)
    K = 1 if src.ndim == 2 else int(src.shape[0])
    if tuple(src.shape)[-2:] != (rows, cols):
        raise DimensionMismatch("generate_observations: source masks disagree with grid spec")
    f = L.rfk_fields()
    f.batch, f.rows, f.cols, f.h = 1, rows, cols, float(h)
    f.g11, f.g12, f.g22, f.b1, f.b2 = (_ptr(x) for x in g)
    f.src = _ptr(src)
    obs = A.empty((K, rows, cols), np.uint8)
    val = A.empty((K, rows, cols), np.float64)
    ctx.check(ctx.lib.rfk_generate_observations(ctx.handle, A.mem, C.byref(f), K, _ptr(src), float(density),
                                                float(noise_level), int(seed), _ptr(obs), _ptr(val)))
    return obs, val


@dataclass
class MultiSourceRow:
    """MultiSourceRow (inversion.hpp:114-119)."""
    k: int
    total_observations: int
    error: float


def multi_source_recover(ks: Sequence[int], density: float, cfg: InverseConfig = None, grid_size: int = 64,
                         seed: int = 42, ctx: Context = None):
    """randers::multi_source_recover (inversion.cpp:439-503): the two-region
    isotropic benchmark, every solve and recover step on the device."""
    ctx = ctx or context()
    cfg = cfg or InverseConfig()
    ka = (C.c_int32 * len(ks))(*[int(k) for k in ks])
    rows = (L.rfk_multi_source_row * len(ks))()
    c = cfg.to_c()
    ctx.check(ctx.lib.rfk_multi_source_recover(ctx.handle, ka, len(ks), float(density), C.byref(c), int(grid_size),
                                               int(seed), rows))
    return [MultiSourceRow(r.k, r.total_observations, r.error) for r in rows]
