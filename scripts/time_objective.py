"""K-source objective_and_grad at n x n (device-resident): wall time and the
solve / backward split."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_00035_b200 as rfk
from paper_2603_00035_b200 import workload as wl
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
F = wl.randers_fields(n, 1, 0.2)
src = torch.zeros((K, n, n), dtype=torch.uint8, device="cuda")
for k in range(K):
    src[k, (n // 2 + 97 * k) % n, (n // 3 + 61 * k) % n] = 1
obs = torch.stack([wl.observation_mask(src[k]) for k in range(K)])
vals = torch.zeros((K, n, n), dtype=torch.float64, device="cuda")
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.time()
    T, r = rfk.solve(*F, src, 1.0 / n)
    torch.cuda.synchronize(); t1 = time.time()
    o = rfk.objective_and_grad(*F, src, obs, vals, 1.0 / n, exact=False)
    torch.cuda.synchronize(); t2 = time.time()
    print(f"n={n} K={K}: solve {t1 - t0:.4f} s, objective {t2 - t1:.4f} s (backward+loss ~ {t2 - t1 - (t1 - t0):.4f} s)",
          flush=True)
