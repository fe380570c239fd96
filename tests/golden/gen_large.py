"""Full-size parity goldens (TEST INFRASTRUCTURE): the reference library
itself (oracle/_ref, compiled from /root/reference/proj/src) run once on
BASELINE.json's own configs, on the deterministic host inputs of
paper_2603_00035_b200.workload.host_fields.  The planes are far too large to
commit (4096^2 x 5 x 8 B), so the fixture stores sha256 digests of their raw
bits plus the scalars (K, converged, max|dT| history, counts, loss); the GPU
test (tests/test_fullsize_parity_gpu.py) regenerates the same inputs on the
box, checks the input digest, runs the CUDA path and compares digests.

    python tests/golden/gen_large.py [c2 c4 c3 ...]    # one process per config

Configs (SURVEY.md §8d shapes, point source at the centre, h = 1/N):
  c2      1024^2 Riemannian (b = 0), seed 1, tol 1e-6 and exact (1e-300)
  c4      2048^2 Randers (drift 0.2), seed 0 (the first C4 scene)
  c3      4096^2 Randers (drift 0.2), seed 1 (the bench's workload), tol 1e-6
  c3x     4096^2, seed 1, sweep order (2, 0, 3, 1), max_iters 9 (a capped solve)
Loss: 30% observed mask (host_observation_mask, stream 2024), targets 0,
sequential loss sum (loss_grad_mse, src/adjoint.cpp:146-160).
CPU time of each reference call is recorded too (the C3 CPU baseline at the
stated config).
"""
from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "large_hashes.json")

CONFIGS = {
    "c2": dict(n=1024, seed=1, drift=0.0, runs=[dict(tol=1e-6, max_iters=50, order=(0, 1, 2, 3)),
                                                 dict(tol=1e-300, max_iters=50, order=(0, 1, 2, 3))]),
    "c4": dict(n=2048, seed=0, drift=0.2, runs=[dict(tol=1e-6, max_iters=50, order=(0, 1, 2, 3))]),
    "c3": dict(n=4096, seed=1, drift=0.2, runs=[dict(tol=1e-6, max_iters=50, order=(0, 1, 2, 3))]),
    "c3x": dict(n=4096, seed=1, drift=0.2, runs=[dict(tol=1e-6, max_iters=9, order=(2, 0, 3, 1))],
                backward=False),
}


def inputs(cfg):
    from paper_2603_00035_b200 import workload as wl
    n = cfg["n"]
    F = wl.host_fields(n, cfg["seed"], cfg["drift"])
    src = wl.host_point_source(n, n)
    obs = wl.host_observation_mask(src)
    return F, src, obs


def digest(*a):
    from paper_2603_00035_b200 import workload as wl
    return wl.fields_digest(*a)


def run(name):
    from oracle.pyoracle import RefLib
    cfg = CONFIGS[name]
    ref = RefLib()
    n = cfg["n"]
    h = 1.0 / n
    F, src, obs = inputs(cfg)
    out = dict(n=n, seed=cfg["seed"], drift=cfg["drift"], h=h,
               input_digest=digest(*F, src, obs), runs=[])
    for k, r in enumerate(cfg["runs"]):
        t0 = time.time()
        sol = ref.solve(*F, src, h, tol=r["tol"], max_iters=r["max_iters"], order=list(r["order"]))
        t_fwd = time.time() - t0
        run = dict(tol=r["tol"], max_iters=r["max_iters"], order=list(r["order"]),
                   iterations=sol.iterations, converged=bool(sol.converged),
                   history=[float(x).hex() for x in sol.history[:sol.iterations]],
                   t_digest=digest(sol.t), t_seconds=t_fwd)
        print(f"{name} run {k}: K={sol.iterations} conv={sol.converged} fwd {t_fwd:.1f}s", flush=True)
        if k == 0 and cfg.get("backward", True):
            t1 = time.time()
            g, loss, unr = ref.loss_grad_mse(sol.t, obs, np.zeros_like(sol.t))
            rec = ref.identify(sol.t, *F, src, h, r["tol"])
            t2 = time.time()
            lam, pg, cl = ref.backward(sol.t, *F, src, h, g, r["tol"])
            t3 = time.time()
            run.update(loss=float(loss).hex(), unreached=int(unr), loss_grad_digest=digest(g),
                       rec_digest=digest(rec.type, rec.stencil, rec.donor1, rec.donor2),
                       rec_c_digest=digest(rec.c),
                       rec_counts=[int(rec.two_point_count), int(rec.one_point_count)],
                       lam_digest=digest(lam), grads_digest=digest(pg), clamped=int(cl),
                       identify_seconds=t2 - t1, backward_seconds=t3 - t2)
            print(f"{name}: records {run['rec_counts']} clamped {cl} backward {t3 - t2:.1f}s", flush=True)
        out["runs"].append(run)
    return name, out


def main(names):
    names = names or list(CONFIGS)
    with mp.Pool(len(names)) as pool:
        res = dict(pool.map(run, names))
    old = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            old = json.load(f)
    old.update(res)
    with open(OUT, "w") as f:
        json.dump(old, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main(sys.argv[1:])
