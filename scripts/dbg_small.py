import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_00035_b200 as rfk
from oracle.pyoracle import Oracle
o = Oracle()
n = int(sys.argv[1]); it = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = np.zeros((5, n, n)); g[0] = g[2] = 1.0
src = np.zeros((n, n), np.uint8); src[n // 2, n // 2] = 1
t0 = time.time()
t, rep = rfk.solve(*g, src, 1.0 / n, max_iters=it)
print("solved", n, rep.iterations, time.time() - t0, flush=True)
r = o.solve(*g, src, 1.0 / n, max_iters=it)
print("match", np.array_equal(t, r.t), np.abs(t - r.t).max(), flush=True)
