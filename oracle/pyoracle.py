"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU checkers.

* ``Oracle``   -> oracle/liboracle.so         (C restatement, oracle.c)
* ``RefLib``   -> oracle/_ref/libranders_ref.so (the reference library itself,
                  compiled from /root/reference/proj/src by oracle/Makefile)

Both expose the same plane-based calls so tests can compare them 1:1 with
the product's C-ABI (include/rfk.h).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / reference leg may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libranders_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i8 = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_ip = C.POINTER(C.c_int)


class CheckerError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: status {status}")
        self.status = status


@dataclass
class SolveResult:
    t: np.ndarray
    iterations: int
    converged: bool
    history: np.ndarray


@dataclass
class Records:
    type: np.ndarray
    stencil: np.ndarray
    donor1: np.ndarray
    donor2: np.ndarray
    c: np.ndarray  # (5, rows, cols)
    two_point_count: int
    one_point_count: int


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class _Checker:
    """Common wrappers over the identical plane-based signatures."""

    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle all ref)")
        self.lib = C.CDLL(path)

    # -- solve ----------------------------------------------------------------
    def solve(self, g11, g12, g22, b1, b2, src, h, tol=1e-6, max_iters=50, order=None,
              mode=0, fixed_values=None) -> SolveResult:
        rows, cols = np.shape(g11)
        t = np.empty((rows, cols), np.float64)
        hist = np.zeros(max(max_iters, 1), np.float64)
        it, conv = C.c_int(0), C.c_int(0)
        order_arr = None if order is None else (C.c_int * 4)(*order)
        fv = None if fixed_values is None else _c(fixed_values, np.float64)
        st = self._solve(rows, cols, h, *(_c(x, np.float64) for x in (g11, g12, g22, b1, b2)),
                         _c(src, np.uint8), None if fv is None else fv.ctypes.data, mode, tol, max_iters, order_arr, t,
                         C.byref(it), C.byref(conv), hist)
        if st:
            raise CheckerError(st, "solve")
        return SolveResult(t, it.value, bool(conv.value), hist[: it.value].copy())

    def identify(self, t, g11, g12, g22, b1, b2, src, h, tol=1e-6) -> Records:
        rows, cols = np.shape(t)
        codes = [np.empty((rows, cols), np.int8) for _ in range(4)]
        cc = np.empty((5, rows, cols), np.float64)
        n2, n1, extra = C.c_int(0), C.c_int(0), self._identify_extra(rows, cols)
        st = self._identify(rows, cols, h, _c(t, np.float64),
                            *(_c(x, np.float64) for x in (g11, g12, g22, b1, b2)),
                            _c(src, np.uint8), tol, *codes, cc[0], cc[1], cc[2], cc[3], cc[4],
                            C.byref(n2), C.byref(n1), extra)
        if st:
            raise CheckerError(st, "identify")
        return Records(*codes, cc, n2.value, n1.value)


class Oracle(_Checker):
    def __init__(self, path: str = ORACLE_SO):
        super().__init__(path)
        L = self.lib
        L.orc_solve.argtypes = [C.c_int, C.c_int, C.c_double] + [_dp] * 5 + [
            _u8, C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_void_p, _dp, _ip, _ip, _dp]
        L.orc_solve.restype = C.c_int
        L.orc_identify.argtypes = [C.c_int, C.c_int, C.c_double, _dp] + [_dp] * 5 + [
            _u8, C.c_double] + [_i8] * 4 + [_dp] * 5 + [_ip, _ip, _ip]
        L.orc_identify.restype = C.c_int
        L.orc_adjoint.argtypes = [C.c_int, C.c_int, _dp, _i8, _i8, _i8] + [_dp] * 5 + [
            _dp, _dp, _ip]
        L.orc_param_gradients.argtypes = [C.c_int, C.c_int, C.c_double, _i8, _i8, _i8] + [
            _dp] * 6 + [_dp] * 5
        L.orc_loss_grad_mse.argtypes = [C.c_int, _dp, _u8, _dp, _dp, C.POINTER(C.c_double), _ip]
        L.orc_project_spd.argtypes = [C.c_int, _dp, _dp, _dp, C.c_double, C.c_double]
        L.orc_project_drift.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_double, C.c_double]
        L.orc_drift_norm_sq.argtypes = [C.c_double] * 5
        L.orc_drift_norm_sq.restype = C.c_double
        L.orc_pipeline.argtypes = [C.c_int, C.c_int, C.c_double] + [_dp] * 5 + [
            _u8, _u8, _dp, C.c_double, C.c_int, _dp, _ip, _ip]
        self._bad = C.c_int(-1)

    def _solve(self, *a):
        return self.lib.orc_solve(*a)

    def _identify(self, *a):
        return self.lib.orc_identify(*a)

    def _identify_extra(self, rows, cols):
        self._bad = C.c_int(-1)
        return C.byref(self._bad)

    @property
    def bad_node(self) -> int:
        return self._bad.value

    def best_candidate(self, r, c, t, g11, g12, g22, b1, b2, h):
        L = self.lib
        if not hasattr(self, "_bc_ready"):
            class Cand(C.Structure):
                _fields_ = [("t0", C.c_double), ("type", C.c_int), ("stencil", C.c_int),
                            ("donor1", C.c_int), ("donor2", C.c_int), ("lam1", C.c_double),
                            ("lam2", C.c_double), ("found", C.c_int)]
            L.orc_best_candidate.argtypes = [C.c_int] * 4 + [C.c_double] + [_dp] * 6
            L.orc_best_candidate.restype = Cand
            self._bc_ready = True
        rows, cols = np.shape(t)
        x = L.orc_best_candidate(r, c, rows, cols, h, _c(t, np.float64),
                                 *(_c(v, np.float64) for v in (g11, g12, g22, b1, b2)))
        return dict(t0=x.t0, type=x.type, stencil=x.stencil, donor1=x.donor1, donor2=x.donor2,
                    lam1=x.lam1, lam2=x.lam2, found=bool(x.found))

    def adjoint(self, t, rec: Records, loss_grad):
        rows, cols = np.shape(t)
        lam = np.empty((rows, cols), np.float64)
        cl = C.c_int(0)
        self.lib.orc_adjoint(rows, cols, _c(t, np.float64), rec.type, rec.donor1, rec.donor2,
                             rec.c[0], rec.c[1], rec.c[2], rec.c[3], rec.c[4],
                             _c(loss_grad, np.float64), lam, C.byref(cl))
        return lam, cl.value

    def param_gradients(self, rec: Records, lam, h):
        rows, cols = np.shape(lam)
        out = np.empty((5, rows, cols), np.float64)
        self.lib.orc_param_gradients(rows, cols, h, rec.type, rec.donor1, rec.donor2, rec.c[0],
                                     rec.c[1], rec.c[2], rec.c[3], rec.c[4], _c(lam, np.float64),
                                     out[0], out[1], out[2], out[3], out[4])
        return out

    def loss_grad_mse(self, t, observed, values):
        n = np.size(t)
        grad = np.empty(np.shape(t), np.float64)
        loss, unr = C.c_double(0), C.c_int(0)
        self.lib.orc_loss_grad_mse(n, _c(t, np.float64), _c(observed, np.uint8),
                                   _c(values, np.float64), grad, C.byref(loss), C.byref(unr))
        return grad, loss.value, unr.value

    def project_spd(self, g11, g12, g22, eps_min=1e-3, lambda_max=1e3):
        a, b, c = (np.array(x, np.float64, copy=True).ravel() for x in (g11, g12, g22))
        st = self.lib.orc_project_spd(a.size, a, b, c, eps_min, lambda_max)
        if st:
            raise CheckerError(st, "project_spd")
        shp = np.shape(g11)
        return a.reshape(shp), b.reshape(shp), c.reshape(shp)

    def project_drift(self, b1, b2, g11, g12, g22, tau=0.95, euclid_cap=10.0):
        x, y = (np.array(v, np.float64, copy=True).ravel() for v in (b1, b2))
        st = self.lib.orc_project_drift(x.size, x, y, *(_c(v, np.float64).ravel() for v in (g11, g12, g22)),
                                        tau, euclid_cap)
        if st:
            raise CheckerError(st, "project_drift")
        shp = np.shape(b1)
        return x.reshape(shp), y.reshape(shp)

    def objective_and_grad(self, g11, g12, g22, b1, b2, sources, observed, values, h, solve_tol=1e-6,
                           solve_max_iters=50, penalty_cap=1e4):
        """objective_and_grad's data term (inversion.cpp:25-51) composed from
        the restated pieces, in the reference's order: per observation set
        solve, MSE loss, flat penalty on unreached observed nodes (node order),
        identify -> adjoint -> param_gradients, accumulated in set order."""
        src = np.asarray(sources)
        src, obs, val = (np.reshape(x, (-1,) + np.shape(g11)) for x in (src, observed, values))
        data_loss, unreached = 0.0, 0
        acc = np.zeros((5,) + np.shape(g11))
        for k in range(src.shape[0]):
            r = self.solve(g11, g12, g22, b1, b2, src[k], h, solve_tol, solve_max_iters)
            if not r.converged:
                raise CheckerError(8, "objective_and_grad: forward solve did not converge")
            grad, loss, unr = self.loss_grad_mse(r.t, obs[k], val[k])
            data_loss += loss
            unreached += unr
            if unr > 0:
                for i in np.flatnonzero((obs[k].ravel() != 0) & ~(r.t.ravel() < 1e9)):
                    d = penalty_cap - val[k].ravel()[i]
                    data_loss += 0.5 * d * d
            rec = self.identify(r.t, g11, g12, g22, b1, b2, src[k], h, solve_tol)
            lam, _ = self.adjoint(r.t, rec, grad)
            acc += self.param_gradients(rec, lam, h)   # elementwise, set order (inversion.cpp:13-21)
        return data_loss, unreached, acc

    def pipeline(self, g11, g12, g22, b1, b2, src, observed, values, h, tol=1e-6, max_iters=50):
        rows, cols = np.shape(g11)
        times = np.zeros(5)
        it, nrec = C.c_int(0), C.c_int(0)
        st = self.lib.orc_pipeline(rows, cols, h, *(_c(x, np.float64) for x in (g11, g12, g22, b1, b2)),
                                   _c(src, np.uint8), _c(observed, np.uint8), _c(values, np.float64),
                                   tol, max_iters, times, C.byref(it), C.byref(nrec))
        if st:
            raise CheckerError(st, "pipeline")
        return times, it.value, nrec.value


class RefLib(_Checker):
    """The reference library itself (compiled from its own sources)."""

    def __init__(self, path: str = REF_SO):
        super().__init__(path)
        L = self.lib
        L.ref_solve.argtypes = [C.c_int, C.c_int, C.c_double] + [_dp] * 5 + [
            _u8, C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_void_p, _dp, _ip, _ip, _dp]
        L.ref_identify.argtypes = [C.c_int, C.c_int, C.c_double, _dp] + [_dp] * 5 + [
            _u8, C.c_double] + [_i8] * 4 + [_dp] * 5 + [_ip, _ip, _i32]
        L.ref_backward.argtypes = [C.c_int, C.c_int, C.c_double, _dp] + [_dp] * 5 + [
            _u8, C.c_double, _dp, _dp] + [_dp] * 5 + [_ip]
        L.ref_best_candidate.argtypes = [C.c_int, C.c_int, C.c_double, _dp] + [_dp] * 5 + [
            C.c_int, _i32, C.c_int, _dp, _i8, _i8, _i8, _i8, _dp, _dp, _i8]
        L.ref_two_point_update.argtypes = [C.c_int] + [_dp] * 12 + [_dp, _dp, _dp, _i8]
        L.ref_jacobian_entries.argtypes = [C.c_int, _i8] + [_dp] * 5 + [_dp, _dp, _dp, _i8]
        L.ref_loss_grad_mse.argtypes = [C.c_int, C.c_int, _dp, _u8, _dp, _dp,
                                        C.POINTER(C.c_double), _ip]
        L.ref_project_spd.argtypes = [C.c_int, _dp, _dp, _dp, C.c_double, C.c_double]
        L.ref_project_drift.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_double, C.c_double]
        L.ref_drift_norm_sq.argtypes = [C.c_double] * 5
        L.ref_drift_norm_sq.restype = C.c_double
        L.ref_correlated_noise.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, _dp]
        L.ref_random_feasible_fields.argtypes = [C.c_int, C.c_uint64, C.c_double] + [_dp] * 5
        L.ref_observation_mask.argtypes = [C.c_int, C.c_int, _u8, C.c_uint64, C.c_double, _u8]
        L.ref_solve_batch.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double] + [_dp] * 5 + [
            C.c_void_p, C.c_double, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_solve_batch.restype = C.c_int
        L.ref_pipeline.argtypes = [C.c_int, C.c_int, C.c_double] + [_dp] * 5 + [
            _u8, _u8, _dp, C.c_double, C.c_int, C.c_int, C.c_int,
            C.POINTER(C.c_double), _dp, _ip, _ip, _ip]
        L.ref_objective_and_grad.argtypes = [C.c_int, C.c_int, C.c_double] + [_dp] * 5 + [
            C.c_int, _u8, _u8, _dp, C.c_double, C.c_int, C.c_double, C.POINTER(C.c_double), _ip] + [_dp] * 5
        self._ri = None

    def objective_and_grad(self, g11, g12, g22, b1, b2, sources, observed, values, h, solve_tol=1e-6,
                           solve_max_iters=50, penalty_cap=1e4):
        """randers::objective_and_grad (inversion.cpp:25-73), regularizers off."""
        src = _c(sources, np.uint8)
        K = 1 if src.ndim == 2 else src.shape[0]
        rows, cols = np.shape(g11)
        grads = np.zeros((5, rows, cols))
        dl, un = C.c_double(0.0), C.c_int(0)
        st = self.lib.ref_objective_and_grad(rows, cols, h, *(_c(x, np.float64) for x in (g11, g12, g22, b1, b2)),
                                             K, src.reshape(-1), _c(observed, np.uint8).reshape(-1),
                                             _c(values, np.float64).reshape(-1), solve_tol, solve_max_iters,
                                             penalty_cap, C.byref(dl), C.byref(un), *grads)
        if st:
            raise CheckerError(st, "objective_and_grad")
        return dl.value, un.value, grads

    # ---- recovery loop pieces (feasibility.cpp:106-196, inversion.cpp) ----
    @staticmethod
    def _pp(planes):
        """(void*)[k] over C-contiguous float64 numpy planes (kept alive by the caller)."""
        return (C.c_void_p * max(1, len(planes)))(*[p.ctypes.data for p in planes])

    def _sig(self, name, args):
        fn = getattr(self.lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
        return fn

    def tv_value_grad(self, channels, variant=0, eps_tv=1e-8):
        ch = [_c(x, np.float64) for x in channels]
        rows, cols = ch[0].shape
        grads = [np.zeros((rows, cols)) for _ in ch]
        v = C.c_double(0.0)
        fn = self._sig("ref_tv_value_grad", [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p,
                                             C.c_void_p, C.POINTER(C.c_double)])
        st = fn(rows, cols, len(ch), int(variant), eps_tv, self._pp(ch), self._pp(grads), C.byref(v))
        if st:
            raise CheckerError(st, "tv_value_grad")
        return v.value, grads

    def tikhonov_value_grad(self, channels, weight):
        ch = [_c(x, np.float64) for x in channels]
        rows, cols = ch[0].shape
        grads = [np.zeros((rows, cols)) for _ in ch]
        v = C.c_double(0.0)
        fn = self._sig("ref_tikhonov_value_grad", [C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_void_p,
                                                   C.POINTER(C.c_double)])
        st = fn(rows, cols, len(ch), weight, self._pp(ch), self._pp(grads), C.byref(v))
        if st:
            raise CheckerError(st, "tikhonov_value_grad")
        return v.value, grads

    def clip_global_norm(self, grads, max_norm):
        """Returns (norm, clipped copies)."""
        g = [np.array(x, dtype=np.float64, order="C", copy=True) for x in grads]
        rows, cols = g[0].shape
        nv = C.c_double(0.0)
        fn = self._sig("ref_clip_global_norm", [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_double,
                                                C.POINTER(C.c_double)])
        st = fn(rows, cols, len(g), self._pp(g), max_norm, C.byref(nv))
        if st:
            raise CheckerError(st, "clip_global_norm")
        return nv.value, g

    def adam_step(self, params, m, v, t, grads, steps, beta1=0.9, beta2=0.999, adam_eps=1e-8, clip=1.0):
        """One adam_step from state (m, v, t); returns (params, m, v, t) as new arrays."""
        P = [np.array(x, dtype=np.float64, order="C", copy=True) for x in params]
        rows, cols = P[0].shape
        M = [np.array(x, dtype=np.float64, order="C", copy=True) for x in m] if t > 0 else [np.zeros((rows, cols)) for _ in P]
        V = [np.array(x, dtype=np.float64, order="C", copy=True) for x in v] if t > 0 else [np.zeros((rows, cols)) for _ in P]
        G = [_c(x, np.float64) for x in grads]
        tt = C.c_long(t)
        stp = (C.c_double * len(P))(*steps)
        fn = self._sig("ref_adam_step", [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.POINTER(C.c_long), C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                         C.c_double, C.c_double])
        st = fn(rows, cols, len(P), self._pp(P), self._pp(M), self._pp(V), C.byref(tt), self._pp(G), stp,
                beta1, beta2, adam_eps, clip)
        if st:
            raise CheckerError(st, "adam_step")
        return P, M, V, tt.value

    def gd_step(self, params, grads, steps, clip=1.0):
        P = [np.array(x, dtype=np.float64, order="C", copy=True) for x in params]
        rows, cols = P[0].shape
        G = [_c(x, np.float64) for x in grads]
        stp = (C.c_double * len(P))(*steps)
        fn = self._sig("ref_gd_step", [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_double])
        st = fn(rows, cols, len(P), self._pp(P), self._pp(G), stp, clip)
        if st:
            raise CheckerError(st, "gd_step")
        return P

    def relative_error(self, est, truth):
        E = [_c(x, np.float64) for x in est]
        T = [_c(x, np.float64) for x in truth]
        rows, cols = E[0].shape
        out = C.c_double(0.0)
        fn = self._sig("ref_relative_error", [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                              C.POINTER(C.c_double)])
        st = fn(rows, cols, len(E), self._pp(E), self._pp(T), C.byref(out))
        if st:
            raise CheckerError(st, "relative_error")
        return out.value

    def objective(self, fields, sources, observed, values, h, cfgv):
        """Full objective_and_grad; cfgv = InverseConfig.to_reference().
        Returns (loss, data_loss, reg_loss, unreached, grads[5])."""
        F = [_c(x, np.float64) for x in fields]
        rows, cols = F[0].shape
        src = _c(sources, np.uint8)
        K = 1 if src.ndim == 2 else src.shape[0]
        obs, val = _c(observed, np.uint8), _c(values, np.float64)
        grads = [np.zeros((rows, cols)) for _ in range(5)]
        cv = _c(cfgv, np.float64)
        l, dl, rl, un = C.c_double(), C.c_double(), C.c_double(), C.c_int()
        fn = self._sig("ref_objective", [C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_double),
                                         C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int),
                                         C.c_void_p])
        st = fn(rows, cols, h, self._pp(F), K, src.ctypes.data, obs.ctypes.data, val.ctypes.data, cv.ctypes.data,
                C.byref(l), C.byref(dl), C.byref(rl), C.byref(un), self._pp(grads))
        if st:
            raise CheckerError(st, "objective")
        return l.value, dl.value, rl.value, un.value, grads

    def recover(self, sources, observed, values, h, cfgv, init=None, truth_metric=None, truth_drift=None):
        """randers::recover; init = 5 planes or None.  Returns a dict."""
        src = _c(sources, np.uint8)
        K = 1 if src.ndim == 2 else src.shape[0]
        rows, cols = src.shape[-2:]
        obs, val = _c(observed, np.uint8), _c(values, np.float64)
        cv = _c(cfgv, np.float64)
        iters = int(cv[11])
        I = [_c(x, np.float64) for x in init] if init is not None else None
        mask = (1 if truth_metric is not None else 0) | (2 if truth_drift is not None else 0)
        T = None
        if mask:
            zero = np.zeros((rows, cols))
            tm = [_c(x, np.float64) for x in truth_metric] if truth_metric is not None else [zero] * 3
            td = [_c(x, np.float64) for x in truth_drift] if truth_drift is not None else [zero] * 2
            T = tm + td
        outs = [np.zeros((rows, cols)) for _ in range(5)]
        iso = np.zeros((rows, cols))
        lh, eh = np.zeros(iters), np.zeros(iters)
        it, fe, ut = C.c_int(), C.c_double(), C.c_int()
        fn = self._sig("ref_recover", [C.c_int, C.c_int, C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double),
                                       C.POINTER(C.c_int)])
        st = fn(rows, cols, h, K, src.ctypes.data, obs.ctypes.data, val.ctypes.data, cv.ctypes.data,
                self._pp(I) if I is not None else None, self._pp(T) if T is not None else None, mask,
                self._pp(outs), iso.ctypes.data, lh.ctypes.data, eh.ctypes.data, C.byref(it), C.byref(fe),
                C.byref(ut))
        if st:
            raise CheckerError(st, "recover")
        n = it.value
        return {"fields": outs, "iso_g": iso, "loss_history": lh[:n], "error_history": eh[:n] if mask else eh[:0],
                "iterations": n, "final_error": fe.value, "unreached_observed_total": ut.value}

    def generate_observations(self, fields, sources, h, density, noise_level=0.0, seed=0):
        F = [_c(x, np.float64) for x in fields]
        rows, cols = F[0].shape
        src = _c(sources, np.uint8)
        K = 1 if src.ndim == 2 else src.shape[0]
        obs = np.zeros((K, rows, cols), np.uint8)
        val = np.zeros((K, rows, cols))
        fn = self._sig("ref_generate_observations", [C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int, C.c_void_p,
                                                     C.c_double, C.c_double, C.c_ulonglong, C.c_void_p, C.c_void_p])
        st = fn(rows, cols, h, self._pp(F), K, src.ctypes.data, density, noise_level, seed, obs.ctypes.data,
                val.ctypes.data)
        if st:
            raise CheckerError(st, "generate_observations")
        return obs, val

    def multi_source_recover(self, ks, density, cfgv, grid_size=64, seed=42):
        ka = (C.c_int * len(ks))(*ks)
        ok, ot, oe = (C.c_int * len(ks))(), (C.c_int * len(ks))(), (C.c_double * len(ks))()
        cv = _c(cfgv, np.float64)
        fn = self._sig("ref_multi_source_recover", [C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_int,
                                                    C.c_ulonglong, C.c_void_p, C.c_void_p, C.c_void_p])
        st = fn(ka, len(ks), density, cv.ctypes.data, grid_size, seed, ok, ot, oe)
        if st:
            raise CheckerError(st, "multi_source_recover")
        return [(ok[i], ot[i], oe[i]) for i in range(len(ks))]

    def _solve(self, *a):
        return self.lib.ref_solve(*a)

    def _identify(self, *a):
        return self.lib.ref_identify(*a)

    def _identify_extra(self, rows, cols):
        self._ri = np.empty((rows, cols), np.int32)
        return self._ri

    @property
    def record_index(self):
        return self._ri

    def backward(self, t, g11, g12, g22, b1, b2, src, h, loss_grad, tol=1e-6):
        rows, cols = np.shape(t)
        lam = np.empty((rows, cols), np.float64)
        out = np.empty((5, rows, cols), np.float64)
        cl = C.c_int(0)
        st = self.lib.ref_backward(rows, cols, h, _c(t, np.float64),
                                   *(_c(x, np.float64) for x in (g11, g12, g22, b1, b2)),
                                   _c(src, np.uint8), tol, _c(loss_grad, np.float64), lam,
                                   out[0], out[1], out[2], out[3], out[4], C.byref(cl))
        if st:
            raise CheckerError(st, "backward")
        return lam, out, cl.value

    def best_candidates(self, t, g11, g12, g22, b1, b2, h, nodes, node_update=False):
        rows, cols = np.shape(t)
        nodes = _c(nodes, np.int32)
        n = nodes.size
        t0, l1, l2 = (np.empty(n) for _ in range(3))
        ty, st_, d1, d2, fd = (np.empty(n, np.int8) for _ in range(5))
        s = self.lib.ref_best_candidate(rows, cols, h, _c(t, np.float64),
                                        *(_c(x, np.float64) for x in (g11, g12, g22, b1, b2)),
                                        n, nodes, int(node_update), t0, ty, st_, d1, d2, l1, l2, fd)
        if s:
            raise CheckerError(s, "best_candidate")
        return dict(t0=t0, type=ty, stencil=st_, donor1=d1, donor2=d2, lam1=l1, lam2=l2,
                    found=fd.astype(bool))

    def two_point_update(self, t1, t2, m1x, m1y, m2x, m2y, g11, g12, g22, b1, b2):
        args = [_c(np.atleast_1d(x), np.float64) for x in (t1, t2, m1x, m1y, m2x, m2y, g11, g12, g22, b1, b2)]
        n = args[0].size
        t0, l1, l2 = (np.empty(n) for _ in range(3))
        v = np.empty(n, np.int8)
        self.lib.ref_two_point_update(n, *args, t0, l1, l2, v)
        return t0, l1, l2, v.astype(bool)

    def jacobian_entries(self, type_, c):
        type_ = _c(np.atleast_1d(type_), np.int8)
        n = type_.size
        c = [_c(np.atleast_1d(x), np.float64) for x in c]
        d, j0, j1 = (np.empty(n) for _ in range(3))
        cl = np.empty(n, np.int8)
        self.lib.ref_jacobian_entries(n, type_, *c, d, j0, j1, cl)
        return d, j0, j1, cl.astype(bool)

    def loss_grad_mse(self, t, observed, values):
        rows, cols = np.shape(t)
        grad = np.empty((rows, cols))
        loss, unr = C.c_double(0), C.c_int(0)
        self.lib.ref_loss_grad_mse(rows, cols, _c(t, np.float64), _c(observed, np.uint8),
                                   _c(values, np.float64), grad, C.byref(loss), C.byref(unr))
        return grad, loss.value, unr.value

    def project_spd(self, g11, g12, g22, eps_min=1e-3, lambda_max=1e3):
        a, b, c = (np.array(x, np.float64, copy=True).ravel() for x in (g11, g12, g22))
        st = self.lib.ref_project_spd(a.size, a, b, c, eps_min, lambda_max)
        if st:
            raise CheckerError(st, "project_spd")
        shp = np.shape(g11)
        return a.reshape(shp), b.reshape(shp), c.reshape(shp)

    def project_drift(self, b1, b2, g11, g12, g22, tau=0.95, euclid_cap=10.0):
        x, y = (np.array(v, np.float64, copy=True).ravel() for v in (b1, b2))
        st = self.lib.ref_project_drift(x.size, x, y, *(_c(v, np.float64).ravel() for v in (g11, g12, g22)),
                                        tau, euclid_cap)
        if st:
            raise CheckerError(st, "project_drift")
        shp = np.shape(b1)
        return x.reshape(shp), y.reshape(shp)

    def correlated_noise(self, rows, cols, radius, seed, normalize=True):
        out = np.empty((rows, cols))
        self.lib.ref_correlated_noise(rows, cols, radius, seed, int(normalize), out)
        return out

    def random_feasible_fields(self, n, seed, drift_scale=0.2):
        # drift_scale == 0 (Riemannian, b = 0): the helper would build tau = 0,
        # which ProjectionConfig rejects; G does not depend on drift_scale.
        out = np.empty((5, n, n))
        st = self.lib.ref_random_feasible_fields(n, seed, drift_scale or 0.2, *out)
        if st:
            raise CheckerError(st, "random_feasible_fields")
        if not drift_scale:
            out[3:] = 0.0
        return out

    def observation_mask(self, src, seed=2024, frac=0.3):
        rows, cols = np.shape(src)
        out = np.empty((rows, cols), np.uint8)
        self.lib.ref_observation_mask(rows, cols, _c(src, np.uint8), seed, frac, out)
        return out

    def solve_batch(self, g11, g12, g22, b1, b2, src, h, tol=1e-6, max_iters=50):
        """Forward solves of independent problems ([nprob, rows, cols] planes),
        one thread each, concurrently (ref_solve_batch).  Returns (wall
        seconds, iterations per problem)."""
        nprob, rows, cols = np.shape(g11)
        wall = C.c_double(0)
        its = np.zeros(nprob, np.int32)
        st = self.lib.ref_solve_batch(nprob, rows, cols, h, *(_c(x, np.float64) for x in (g11, g12, g22, b1, b2)),
                                      _c(src, np.uint8).ctypes.data, tol, max_iters, C.byref(wall), its.ctypes.data)
        if st:
            raise CheckerError(st, "solve_batch")
        return wall.value, its

    def pipeline(self, g11, g12, g22, b1, b2, src, observed, values, h, tol=1e-6, max_iters=50,
                 nprob=1, nthreads=1):
        rows, cols = np.shape(g11)
        wall = C.c_double(0)
        times = np.zeros(5)
        it, nrec, conv = C.c_int(0), C.c_int(0), C.c_int(0)
        st = self.lib.ref_pipeline(rows, cols, h, *(_c(x, np.float64) for x in (g11, g12, g22, b1, b2)),
                                   _c(src, np.uint8), _c(observed, np.uint8), _c(values, np.float64),
                                   tol, max_iters, nprob, nthreads, C.byref(wall), times,
                                   C.byref(it), C.byref(nrec), C.byref(conv))
        if st:
            raise CheckerError(st, "pipeline")
        return wall.value, times, it.value, nrec.value, bool(conv.value)


def point_source(rows, cols, r=None, c=None):
    m = np.zeros((rows, cols), np.uint8)
    m[rows // 2 if r is None else r, cols // 2 if c is None else c] = 1
    return m


# ---- projection VJP reference ----------------------------
# The reference has no backward through project_spd / project_drift
# (feasibility.cpp:31-72); this analytic numpy restatement is the checker for
# the device VJP.  It is pinned by central finite differences of the oracle's
# own forward projections (tests/test_projection_vjp.py), the protocol
# SURVEY.md §8c prescribes for this row ("parity unpinned" otherwise).

def _eig_frame(a, b, c):
    half_tr = 0.5 * (a + c)
    amc = a - c
    disc = np.sqrt(0.25 * amc * amc + b * b)
    theta = 0.5 * np.arctan2(2.0 * b, amc)     # eigenvector (cos, sin) of hi, feasibility.cpp:18-20
    return half_tr + disc, half_tr - disc, np.cos(theta), np.sin(theta)


def project_spd_forward_np(a, b, c, eps_min=1e-3, lambda_max=1e3):
    """project_spd (feasibility.cpp:31-44) in numpy (host trig)."""
    hi, lo, cs, sn = _eig_frame(a, b, c)
    keep = (lo >= eps_min) & (hi <= lambda_max)
    H, L = np.clip(hi, eps_min, lambda_max), np.clip(lo, eps_min, lambda_max)
    o11 = np.where(keep, a, H * cs * cs + L * sn * sn)
    o12 = np.where(keep, b, (H - L) * cs * sn)
    o22 = np.where(keep, c, H * sn * sn + L * cs * cs)
    return o11, o12, o22


def project_spd_vjp_np(a, b, c, d11, d12, d22, eps_min=1e-3, lambda_max=1e3):
    """Daleckii-Krein VJP of the eigenvalue clamp; identity at pass-through nodes."""
    hi, lo, cs, sn = _eig_frame(a, b, c)
    keep = (lo >= eps_min) & (hi <= lambda_max)
    Fh = ((hi > eps_min) & (hi < lambda_max)).astype(float)
    Fl = ((lo > eps_min) & (lo < lambda_max)).astype(float)
    fh, fl = np.clip(hi, eps_min, lambda_max), np.clip(lo, eps_min, lambda_max)
    with np.errstate(divide="ignore", invalid="ignore"):
        F12 = np.where(hi > lo, (fh - fl) / np.where(hi > lo, hi - lo, 1.0), Fh)
    g11, g12, g22 = d11, 0.5 * d12, d22
    pvv = cs * cs * g11 + 2 * cs * sn * g12 + sn * sn * g22
    pww = sn * sn * g11 - 2 * cs * sn * g12 + cs * cs * g22
    pvw = -cs * sn * g11 + (cs * cs - sn * sn) * g12 + cs * sn * g22
    qvv, qww, qvw = Fh * pvv, Fl * pww, F12 * pvw
    r11 = cs * cs * qvv - 2 * cs * sn * qvw + sn * sn * qww
    r22 = sn * sn * qvv + 2 * cs * sn * qvw + cs * cs * qww
    r12 = cs * sn * qvv + (cs * cs - sn * sn) * qvw - cs * sn * qww
    return (np.where(keep, d11, r11), np.where(keep, d12, 2 * r12), np.where(keep, d22, r22))


def project_drift_vjp_np(x, y, g11, g12, g22, dx, dy, tau=0.95, euclid_cap=10.0):
    """VJP of project_drift (feasibility.cpp:51-72) w.r.t. b and the metric."""
    en = np.sqrt(x * x + y * y)
    c1 = en > euclid_cap
    f1 = np.where(c1, euclid_cap / np.where(c1, en, 1.0), 1.0)
    x1, y1 = x * f1, y * f1
    det = g11 * g22 - g12 * g12
    mx, my = (g22 * x1 - g12 * y1) / det, (g11 * y1 - g12 * x1) / det
    gn = np.sqrt(x1 * mx + y1 * my)
    c2 = gn > tau
    k = np.where(c2, tau * (dx * x1 + dy * y1) / np.where(c2, gn, 1.0) ** 3, 0.0)
    dg11, dg22, dg12 = 0.5 * k * mx * mx, 0.5 * k * my * my, k * mx * my
    s = np.where(c2, tau / np.where(c2, gn, 1.0), 1.0)
    dx1, dy1 = s * dx - k * mx, s * dy - k * my
    dot = np.where(c1, (x * dx1 + y * dy1) / np.where(c1, en * en, 1.0), 0.0)
    return f1 * (dx1 - x * dot), f1 * (dy1 - y * dot), dg11, dg12, dg22


def project_joint_vjp_np(g11, g12, g22, b1, b2, d11, d12, d22, db1, db2, eps_min=1e-3, lambda_max=1e3,
                         tau=0.95, euclid_cap=10.0):
    """ParamView::project, Joint (inversion.cpp:276-279): spd, then drift on the projected metric."""
    p11, p12, p22 = project_spd_forward_np(g11, g12, g22, eps_min, lambda_max)
    ox, oy, e11, e12, e22 = project_drift_vjp_np(b1, b2, p11, p12, p22, db1, db2, tau, euclid_cap)
    r11, r12, r22 = project_spd_vjp_np(g11, g12, g22, d11 + e11, d12 + e12, d22 + e22, eps_min, lambda_max)
    return r11, r12, r22, ox, oy
