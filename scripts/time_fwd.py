"""Forward solve wall time at n x n (device-resident inputs), 3 repeats."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_00035_b200 as rfk
from paper_2603_00035_b200 import workload as wl
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
F = [torch.as_tensor(x).cuda() for x in wl.host_fields(n, 1, 0.2)]
src = torch.as_tensor(wl.host_point_source(n, n)).cuda()
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    torch.cuda.synchronize()
    t = time.time()
    T, rep = rfk.solve(*F, src, 1.0 / n)
    torch.cuda.synchronize()
    print("fwd", round(time.time() - t, 4), rep.iterations, flush=True)
