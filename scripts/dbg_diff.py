import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_00035_b200 as rfk
from oracle.pyoracle import Oracle
o = Oracle()
n = int(sys.argv[1]); it = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = np.zeros((5, n, n)); g[0] = g[2] = 1.0
src = np.zeros((n, n), np.uint8); src[n // 2, n // 2] = 1
for order in ([0, 1, 2, 3], [0, 0, 0, 0], [1, 1, 1, 1], [2, 2, 2, 2], [3, 3, 3, 3]):
    t, rep = rfk.solve(*g, src, 1.0 / n, max_iters=it, sweep_order=order)
    r = o.solve(*g, src, 1.0 / n, max_iters=it, order=order)
    d = np.argwhere(t != r.t)
    print("order", order, "ndiff", len(d), "first", d[:10].tolist(), flush=True)
    if len(d):
        i, j = d[0]
        print("got", t[i, j], "want", r.t[i, j])
