"""C3's "forward + adjoint vs finite differences" (BASELINE.json configs[2];
SURVEY §8d: gradient_check over all 5 channels, 20 points, eps 1e-5, seed 7,
src/oracle.cpp:322-363) at 4096^2 on the bench's inputs, solves on the GPU.
The central difference is summed node by node (gradcheck.loss_difference):
the reference's loss_value difference cancels ~10 digits at this size.  The
solves are exact (tol 1e-300, the SURVEY's "exact run"): implicit
differentiation is the derivative of the fixed point, and at tol 1e-6 a 4096^2
iterate is ~1e-7 away from it, which shows in a 1e-5 difference.
Writes profiles/r02_gradcheck_c3.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from paper_2603_00035_b200 import gradcheck
from paper_2603_00035_b200 import workload as wl

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
npts = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "profiles", "r02_gradcheck_c3.json")
F = wl.host_fields(n, 1, 0.2)
src = wl.host_point_source(n, n)
obs = wl.host_observation_mask(src)
t0 = time.time()
runs = {}
for eps in (1e-4, 1e-5):
    res = gradcheck.gradient_check(*F, src[None], obs[None], np.zeros((1, n, n)), 1.0 / n, n_points=npts,
                                   eps=eps, seed=7, fd="difference", tol=1e-300, max_iters=100,
                                   identify_tol=1e-6)
    rel = [p.rel_error for p in res.points]
    runs[f"{eps:g}"] = {
        "points": [{"node": p.node, "r": p.node // n, "c": p.node % n, "channel": gradcheck.CHANNELS[p.channel],
                    "fd": p.fd, "adjoint": p.adjoint, "rel_error": p.rel_error} for p in res.points],
        "max_rel_error": res.max_rel_error, "median_rel_error": float(np.median(rel)) if rel else None,
        "skipped_unstable": res.skipped_unstable, "skipped_zero": res.skipped_zero}
    print(f"eps {eps:g}: median {runs[f'{eps:g}']['median_rel_error']:.2e} max {res.max_rel_error:.2e} "
          f"unstable {res.skipped_unstable}", flush=True)
    for p in runs[f"{eps:g}"]["points"]:
        print(f"  {p['r']:5d} {p['c']:5d} {p['channel']:4s} fd {p['fd']: .10e} adj {p['adjoint']: .10e} "
              f"rel {p['rel_error']:.2e}")
dt = time.time() - t0
rec = {"grid": f"{n}x{n}", "seed": 7, "channels": list(gradcheck.CHANNELS),
       "fd": "central difference of the loss, summed node by node", "solve_tol": 1e-300, "identify_tol": 1e-6,
       "runs": runs, "seconds": dt,
       "inputs": "workload.host_fields(4096, 1, 0.2): the bench's / large_hashes c3 inputs",
       "note": "adjoint values and solves are bit-identical to the reference library's (full-size parity); "
               "the finite difference has a noise floor from the history dependence of the exact "
               "Gauss-Seidel fixed point (error grows as 1/eps: scripts/gradcheck_probe.py)"}
json.dump(rec, open(out, "w"), indent=1)
