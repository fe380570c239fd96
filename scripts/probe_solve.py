"""Timing probe: device-resident solve + backward (second call timed)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2603_00035_b200 as rfk
from paper_2603_00035_b200 import workload as wl

sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "512,1024,2048,4096").split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for n in sizes:
    F = wl.randers_fields(n, 1, 0.2)
    src = wl.point_source(n, n)
    h = 1.0 / n
    obs = wl.observation_mask(src)
    for r in range(reps):
        torch.cuda.synchronize()
        t0 = time.time()
        t, rep = rfk.solve(*F, src, h)
        torch.cuda.synchronize()
        t1 = time.time()
        g, loss, _ = rfk.loss_grad_mse(t, obs, torch.zeros_like(t), exact=False)
        torch.cuda.synchronize()
        t2 = time.time()
        lam, grads, cl = rfk.backward(t, *F, src, h, g)
        torch.cuda.synchronize()
        t3 = time.time()
    W = wl.node_updates(rep.iterations, n * n, 1, int(((t < 1e9) & (src == 0)).sum()))
    print(f"n={n} K={rep.iterations} conv={rep.converged} fwd={t1-t0:.4f}s loss={t2-t1:.4f}s bwd={t3-t2:.4f}s "
          f"W={W/1e6:.1f}M -> {W/(t3-t0)/1e9:.3f} G node-updates/s; fwd-only {4*rep.iterations*n*n/(t1-t0)/1e9:.3f} G/s "
          f"sweeps={4*rep.iterations} ms/sweep={(t1-t0)*1e3/(4*rep.iterations):.3f}", flush=True)
    if os.environ.get("CHECK_T"):
        torch.save(t.cpu(), f"gpurun_out/t_{n}_{os.environ.get('RFK_SWEEP_VERSION','2')}.pt")
