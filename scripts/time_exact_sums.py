"""Exact (sequential, reference-order) sums vs tree sums at n x n."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_00035_b200 as rfk
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
g = [torch.randn(n, n, dtype=torch.float64, device="cuda") for _ in range(5)]
for exact in (True, False):
    for rep in range(2):
        x = [p.clone() for p in g]
        torch.cuda.synchronize(); t = time.time()
        nrm = rfk.clip_global_norm(x, 1.0, exact=exact)
        torch.cuda.synchronize()
        print(f"clip_global_norm 5 x {n}^2 exact={exact}: {time.time() - t:.4f} s norm {nrm!r}", flush=True)
