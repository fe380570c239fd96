"""Batched forward solves (K source sets on one metric, or K metrics): wall
time per grid and bitwise agreement with one-at-a-time solves."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_00035_b200 as rfk
from paper_2603_00035_b200 import workload as wl
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
shared = (sys.argv[3] if len(sys.argv) > 3 else "shared") == "shared"
F = wl.randers_fields(n, 1, 0.2)
src = torch.zeros((K, n, n), dtype=torch.uint8, device="cuda")
for k in range(K):
    src[k, (n // 2 + 97 * k) % n, (n // 3 + 61 * k) % n] = 1
if not shared:
    F = [torch.stack([x * (1.0 + 0.01 * k) if i < 3 else x for k in range(K)]) for i, x in enumerate(F)]
for rep in range(3):
    torch.cuda.synchronize(); t = time.time()
    T, r = rfk.solve(*F, src, 1.0 / n)
    torch.cuda.synchronize(); dt = time.time() - t
    print(f"batch n={n} K={K} shared={shared}: {dt:.4f} s, {dt / K:.4f} s/grid, iters {list(np.asarray(r.iterations))}", flush=True)
one = []
torch.cuda.synchronize(); t = time.time()
for k in range(K):
    Fk = [x if shared else x[k] for x in F]
    one.append(rfk.solve(*Fk, src[k], 1.0 / n)[0])
torch.cuda.synchronize(); dt = time.time() - t
print(f"one at a time: {dt:.4f} s, {dt / K:.4f} s/grid", flush=True)
print("bitwise equal:", all(torch.equal(T[k], one[k]) for k in range(K)))
