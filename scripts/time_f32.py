"""fp32-mode vs fp64 forward at n x n: wall time and max relative difference."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_00035_b200 as rfk
from paper_2603_00035_b200 import workload as wl
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
F = wl.randers_fields(n, 1, 0.2)
src = wl.point_source(n, n)
for rep in range(3):
    torch.cuda.synchronize(); t = time.time()
    T64, r64 = rfk.solve(*F, src, 1.0 / n)
    torch.cuda.synchronize(); t1 = time.time()
    T32, r32 = rfk.solve_f32(*F, src, 1.0 / n)
    torch.cuda.synchronize(); t2 = time.time()
    m = T64 < 1e9
    rel = ((T32.double() - T64).abs()[m] / T64[m].abs().clamp_min(1e-3)).max().item()
    print(f"n={n}: fp64 {t1 - t:.4f} s (K={r64.iterations}), fp32 {t2 - t1:.4f} s (K={r32.iterations}), max rel {rel:.2e}",
          flush=True)
