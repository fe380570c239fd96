"""Generate the golden fixtures in tests/golden/ from the REFERENCE library.

Runs the unmodified reference (compiled from /root/reference/proj/src into
oracle/_ref/libranders_ref.so by `make -C oracle ref`) through its public API
(solve, solve_jacobi, solve_from_values, identify_stencils, solve_adjoint,
param_gradients, loss_grad_mse) and stores inputs and outputs as .npz.
Inputs come from the reference's own generators (correlated_noise +
project_spd/project_drift, i.e. tests/helpers.hpp random_feasible_fields),
because std::normal_distribution is libstdc++-specific.

    python tests/golden/gen_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import RefLib  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def case_fields(R: RefLib, name: str):
    if name == "iso32":
        n = 32
        g = np.zeros((5, n, n)); g[0] = g[2] = 1.0
        src = np.zeros((n, n), np.uint8); src[16, 16] = 1
        return g, src, 1.0 / n, None
    if name == "randers48x40":
        F = R.random_feasible_fields(48, 7, 0.2)[:, :, :40].copy()
        src = np.zeros((48, 40), np.uint8); src[5, 7] = 1; src[30, 33] = 1
        return F, src, 1.0 / 48, None
    if name == "riem40":
        F = R.random_feasible_fields(40, 5, 0.0)
        src = np.zeros((40, 40), np.uint8); src[20, 20] = 1
        return F, src, 1.0 / 40, None
    if name == "randers64":
        F = R.random_feasible_fields(64, 21, 0.3)
        src = np.zeros((64, 64), np.uint8); src[32, 32] = 1
        return F, src, 1.0, None
    if name == "drift81":
        n = 81
        g = np.zeros((5, n, n)); g[0] = g[2] = 1.0; g[3] = 0.3
        src = np.zeros((n, n), np.uint8); src[40, 40] = 1
        return g, src, 1.0, None
    if name == "fixed36x50":
        F = R.random_feasible_fields(50, 9, 0.15)[:, :36, :].copy()
        src = np.zeros((36, 50), np.uint8)
        src[0, :] = 1  # a fixed front along the top row with given values
        fv = np.zeros((36, 50)); fv[0, :] = np.linspace(0.0, 0.3, 50)
        return F, src, 1.0 / 50, fv
    raise KeyError(name)


CASES = ["iso32", "randers48x40", "riem40", "randers64", "drift81", "fixed36x50"]


def main():
    R = RefLib()
    for name in CASES:
        F, src, h, fv = case_fields(R, name)
        rows, cols = src.shape
        mode = 2 if fv is not None else 0
        out = dict(fields=F, src=src, h=np.float64(h))
        if fv is not None:
            out["fixed_values"] = fv
        for tag, tol, mi, order in [("default", 1e-6, 50, None), ("exact", 1e-300, 200, None),
                                    ("order3102", 1e-6, 50, (3, 1, 0, 2))]:
            s = R.solve(*F, src, h, tol=tol, max_iters=mi, order=order, mode=mode, fixed_values=fv)
            out[f"t_{tag}"] = s.t
            out[f"iters_{tag}"] = np.int32(s.iterations)
            out[f"conv_{tag}"] = np.int32(s.converged)
            out[f"hist_{tag}"] = s.history
            out[f"tol_{tag}"] = np.float64(tol)
            out[f"maxit_{tag}"] = np.int32(mi)
            out[f"order_{tag}"] = np.array(order or (0, 1, 2, 3), np.int32)
        if fv is None and rows * cols <= 48 * 48:
            budget = 5 * max(rows, cols) + 50
            s = R.solve(*F, src, h, tol=1e-6, max_iters=budget, mode=1)
            out["t_jacobi"] = s.t
            out["iters_jacobi"] = np.int32(s.iterations)
            out["hist_jacobi"] = s.history
        t = out["t_default"]
        rec = R.identify(t, *F, src, h, 1e-6)
        out.update(rec_type=rec.type, rec_stencil=rec.stencil, rec_donor1=rec.donor1,
                   rec_donor2=rec.donor2, rec_c=rec.c,
                   rec_counts=np.array([rec.two_point_count, rec.one_point_count], np.int32))
        observed = R.observation_mask(src, 2024, 0.3)
        values = np.zeros((rows, cols))
        grad, loss, unr = R.loss_grad_mse(t, observed, values)
        lam, pg, cl = R.backward(t, *F, src, h, grad, 1e-6)
        out.update(observed=observed, loss_grad=grad, loss=np.float64(loss), unreached=np.int32(unr),
                   lam=lam, param_grads=pg, clamped=np.int32(cl))
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(name, rows, cols, "K", int(out["iters_default"]), int(out["iters_exact"]),
              "rec", rec.two_point_count, rec.one_point_count, os.path.getsize(path))


if __name__ == "__main__":
    main()
