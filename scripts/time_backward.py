"""Wall vs device time of the fused backward at n x n (device-resident)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2603_00035_b200 as rfk
from paper_2603_00035_b200 import workload as wl

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
F = wl.randers_fields(n, 1, 0.2)
src = wl.point_source(n, n)
h = 1.0 / n
ctx = rfk.context()
t, rep = rfk.solve(*F, src, h, ctx=ctx)
g, loss, _ = rfk.loss_grad_mse(t, wl.observation_mask(src), torch.zeros_like(t), exact=False, ctx=ctx)
for r in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    lam, grads, cl = rfk.backward(t, *F, src, h, g, want_lambda=False, ctx=ctx)
    e1.record()
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    print(f"rep {r}: wall {1e3*(w1-w0):.2f} ms  events {e0.elapsed_time(e1):.2f} ms", flush=True)

print("-- bench-like step: solve, loss, backward")
obs = wl.observation_mask(src)
vals = torch.zeros((n, n), dtype=torch.float64, device="cuda")
for r in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    t, rep = rfk.solve(*F, src, h, ctx=ctx)
    ev[1].record()
    g, loss, unr = rfk.loss_grad_mse(t, obs, vals, exact=False, ctx=ctx)
    ev[2].record()
    lam, grads, cl = rfk.backward(t, *F, src, h, g, want_lambda=False, ctx=ctx)
    ev[3].record()
    torch.cuda.synchronize()
    print(f"rep {r}: solve {ev[0].elapsed_time(ev[1]):.1f} loss {ev[1].elapsed_time(ev[2]):.1f} "
          f"backward {ev[2].elapsed_time(ev[3]):.1f} ms", flush=True)
