# Stress check: repeat the 48x40 golden solve and compare T and the max|dT| history with the oracle bit for bit.
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_00035_b200 as rfk
from oracle.pyoracle import Oracle
o = Oracle()
_z = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "randers48x40.npz")); G = {k: _z[k] for k in _z.files}
F = list(G["fields"])
src, h = G["src"], float(G["h"])
for order in ((3, 1, 0, 2), (0, 1, 2, 3), (2, 2, 2, 2), (3, 3, 3, 3)):
    r = o.solve(*F, src, h, tol=float(G['tol_order3102']), max_iters=int(G['maxit_order3102']), order=list(order))
    bad = 0
    for rep_i in range(int(os.environ.get("REPS", "20"))):
        t, rep = rfk.solve(*F, src, h, tol=float(G['tol_order3102']), max_iters=int(G['maxit_order3102']), sweep_order=order)
        okT = np.array_equal(t, r.t)
        okH = np.array_equal(np.asarray(rep.max_delta_history), r.history)
        if not (okT and okH):
            bad += 1
            if bad == 1:
                print(order, "rep", rep_i, "T ok", okT, "hist", list(rep.max_delta_history), "want", list(r.history), flush=True)
    print(order, "bad", bad, "of", os.environ.get("REPS", "20"), flush=True)
