"""Repeated batched solves + backward (concurrent slots) vs one-at-a-time, bitwise."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_00035_b200 as rfk
from paper_2603_00035_b200 import workload as wl
rng = np.random.default_rng(0)
bad = 0
for rep in range(int(os.environ.get("REPS", "30"))):
    n = int(rng.choice([64, 96, 160, 256]))
    B = int(rng.integers(2, 7))
    F = [x for x in wl.randers_fields(n, int(rng.integers(0, 100)), 0.2)]
    per_grid = bool(rng.integers(0, 2))
    if per_grid:
        F = [torch.stack([x * (1.0 + 0.03 * b) if i < 3 else x for b in range(B)]) for i, x in enumerate(F)]
    src = torch.zeros((B, n, n), dtype=torch.uint8, device="cuda")
    for b in range(B):
        src[b, int(rng.integers(0, n)), int(rng.integers(0, n))] = 1
    T, r = rfk.solve(*F, src, 1.0 / n)
    g = (T < 1e9).double() * 0.01
    lam, grads, cl = rfk.backward(T, *F, src, 1.0 / n, g, accumulate=not per_grid)
    ok = True
    acc = None
    for b in range(B):
        Fb = [x[b] for x in F] if per_grid else F
        t1, r1 = rfk.solve(*Fb, src[b], 1.0 / n)
        ok &= torch.equal(t1, T[b])
        l1, g1, _ = rfk.backward(t1, *Fb, src[b], 1.0 / n, g[b])
        ok &= torch.equal(l1, lam[b])
        if per_grid:
            ok &= torch.equal(g1, grads[:, b])
        else:
            acc = g1.clone() if acc is None else acc + g1
    if not per_grid:
        ok &= torch.equal(acc, grads)
    if not ok:
        bad += 1
        print("MISMATCH rep", rep, n, B, per_grid, flush=True)
print("stress_batch bad", bad, flush=True)
