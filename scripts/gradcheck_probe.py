"""Diagnostic: central differences at several eps for chosen (node, channel)
points of the C3 field, next to the adjoint (exact solves)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_00035_b200 as rfk
from paper_2603_00035_b200 import gradcheck, workload as wl
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
drift = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
F = [torch.as_tensor(x).cuda() for x in wl.host_fields(n, 1, drift)]
src = torch.as_tensor(wl.host_point_source(n, n)).cuda()[None]
obs = torch.as_tensor(wl.host_observation_mask(src[0].cpu().numpy())).cuda()[None]
val = torch.zeros((1, n, n), dtype=torch.float64, device="cuda")
h = 1.0 / n
t, rep = rfk.solve(*F, src[0], h, tol=1e-300, max_iters=100)
print("K exact", rep.iterations, "last deltas", rep.max_delta_history[-3:])
g, _, _ = rfk.loss_grad_mse(t, obs[0], val[0])
_, pg, _ = rfk.backward(t, *F, src[0], h, g, tol=1e-6)
pts = [(2508, 471, 0), (3362, 539, 3), (3736, 23, 2), (3868, 2559, 3), (1823, 1958, 2), (2946, 1044, 4)] if n == 4096 else \
      [(n * 3 // 5, n // 7, 0), (n // 3, n * 2 // 3, 3), (n * 4 // 5, n // 2, 2)]
for r, c, ch in pts:
    node = r * n + c
    an = float(pg[ch].view(-1)[node])
    row = []
    for eps in (1e-4, 1e-5, 1e-6, 1e-7):
        pp = [p.clone() for p in F]; pm = [p.clone() for p in F]
        pp[ch].view(-1)[node] += eps; pm[ch].view(-1)[node] -= eps
        dl = gradcheck.loss_difference(pp, pm, src, obs, val, h, tol=1e-300, max_iters=100)
        row.append(dl / (2 * eps))
    print(f"({r},{c}) ch {ch}: adj {an:.10e} fd(1e-4..1e-7) " + " ".join(f"{x:.10e}" for x in row)
          + " rel " + " ".join(f"{abs(x - an) / max(abs(x), abs(an)):.1e}" for x in row), flush=True)
