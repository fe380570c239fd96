"""One Randers solve (+ loss + backward) at n x n for profiler captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2603_00035_b200 as rfk
from paper_2603_00035_b200 import workload as wl

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
F = [torch.as_tensor(x).cuda() for x in wl.host_fields(n, 1, 0.2)]
src = torch.as_tensor(wl.host_point_source(n, n)).cuda()
t, rep = rfk.solve(*F, src, 1.0 / n)
g, loss, _ = rfk.loss_grad_mse(t, torch.as_tensor(wl.host_observation_mask(src.cpu().numpy())).cuda(), torch.zeros_like(t), exact=False)
lam, grads, cl = rfk.backward(t, *F, src, 1.0 / n, g)
torch.cuda.synchronize()
print("ok", n, rep.iterations, float(loss))
