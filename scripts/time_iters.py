"""Forward time vs iteration cap (max_iters) on the 4096^2 bench fields:
the per-iteration cost of the sweep as the dirty fraction falls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_00035_b200 as rfk
from paper_2603_00035_b200 import workload as wl
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
F = [torch.as_tensor(x).cuda() for x in wl.host_fields(n, 1, 0.2)]
src = torch.as_tensor(wl.host_point_source(n, n)).cuda()
rfk.solve(*F, src, 1.0 / n)
prev = 0.0
for m in [1, 2, 3, 4, 6, 8, 10, 12, 14, 15, 16]:
    best = 1e9
    for _ in range(2):
        torch.cuda.synchronize(); t = time.time()
        T, rep = rfk.solve(*F, src, 1.0 / n, max_iters=m)
        torch.cuda.synchronize(); best = min(best, time.time() - t)
    print(f"max_iters {m:3d}: {best*1e3:8.2f} ms  (+{(best - prev)*1e3:7.2f} ms)  K={rep.iterations}", flush=True)
    prev = best
