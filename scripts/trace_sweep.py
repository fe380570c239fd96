"""Per-band timing trace of the sweep kernel (RFK_TRACE=1 diagnostics).

The traced kernel is in a diagnostic build only:
    scripts/build_variant.sh trace -DRFK_SWEEP_TRACE_BUILD=1
    RFK_LIBRARY=$PWD/paper_2603_00035_b200/librfk_trace.so python scripts/trace_sweep.py 4096 all
"""
import ctypes as C
import os
import sys

os.environ["RFK_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2603_00035_b200 as rfk
from paper_2603_00035_b200 import workload as wl

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ctx = rfk.context()
F = wl.host_fields(n, 1, 0.2)
src = wl.host_point_source(n, n)
t, rep = rfk.solve(*F, src, 1.0 / n, ctx=ctx)
t, rep = rfk.solve(*F, src, 1.0 / n, ctx=ctx)
BLn = int(os.environ.get("RFK_BAND_LINES", "16"))
nb = (n + BLn - 1) // BLn
TW = 32
buf = np.zeros(4 * 50 * nb * TW + 8, np.uint64)
lib = ctx.lib
lib.rfk_debug_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
lib.rfk_debug_trace.restype = C.c_int64
got = lib.rfk_debug_trace(ctx.handle, buf.ctypes.data, buf.size)
if got <= 8:
    sys.exit("no trace recorded: RFK_LIBRARY must point at a -DRFK_SWEEP_TRACE_BUILD=1 build (see the docstring)")
tr = buf[:got - 8].reshape(-1, nb, TW).astype(np.int64)
npass = 4 * rep.iterations
print(f"n={n} K={rep.iterations} bands={nb}")
S = 2 * (BLn - 1) + n
for p in range(min(npass, 8)) if len(sys.argv) < 3 else range(npass):
    r = tr[p]
    t0 = r[:, 0].min()
    start = (r[:, 0] - t0) / 1e3
    end = (r[:, 1] - t0) / 1e3
    dur = end - start
    first_mb = np.where(r[:, 4] > 0, (r[:, 4] - r[:, 0]) / 1e3, np.nan)
    print(f"pass {p}: span {end.max():8.1f}us band dur mean {dur.mean():7.1f} start lag {np.diff(start).mean():6.2f}us"
          f" | band0 cyc/step {r[0,2]/S:6.0f} wait {r[0,3]/S:6.0f} dirty steps {r[0,6]:5d} cyc/dirty {r[0,5]/max(1,r[0,6]):6.0f}"
          f" | all bands: wait/step {r[:,3].mean()/S:6.0f} dirty steps {r[:,6].mean():6.0f} cyc/dirty {r[:,5].sum()/max(1,r[:,6].sum()):6.0f}"
          f" first_mbox {np.nanmean(first_mb):6.1f}us | skipped {r[:,11].mean():6.0f} decisions {r[:,15].mean():6.0f}"
          f" | wait own/mbox/hoist per step {r[:,17].mean()/S:5.0f}/{r[:,18].mean()/S:5.0f}/{r[:,19].mean()/S:5.0f}"
          f" prod prevpass/step {r[:,20].mean()/S:5.0f} ringfull polls {r[:,21].mean():6.0f}"
          f" tma lat {r[:,22].sum()/max(1,r[:,23].sum()):6.0f}cyc x{r[:,23].mean():5.0f}"
          f" | prod cyc/chunk room(comp/wr) {r[:,24].mean()/max(1,r[:,28].mean()):6.0f}/{r[:,25].mean()/max(1,r[:,28].mean()):6.0f}"
          f" load {r[:,26].mean()/max(1,r[:,28].mean()):6.0f} bits {r[:,27].mean()/max(1,r[:,28].mean()):6.0f}"
          f" | wr batches {r[:,29].mean():5.0f} cyc/batch {r[:,30].mean()/max(1,r[:,29].mean()):6.0f}"
          f" | band0 wait own/mbox/hoist {r[0,17]/S:5.0f}/{r[0,18]/S:5.0f}/{r[0,19]/S:5.0f} skipped {r[0,11]}")

# timeline (us from the solve's first band start): each pass's first band start, band 0's first
# step, last band end -- the second pass of an iteration waits for the previous iteration's decision
g0 = tr[:npass, :, 0][tr[:npass, :, 0] > 0].min()
print("timeline: pass  first-start  band0-step0  last-end")
for p in range(npass):
    r = tr[p]
    print(f"  {p:3d} {(r[:, 0].min() - g0) / 1e3:10.1f} {(r[0, 9] - g0) / 1e3:10.1f} {(r[:, 1].max() - g0) / 1e3:10.1f}")
dsum = tr[:npass, :, 12].sum(axis=1); rsum = tr[:npass, :, 13].sum(axis=1); csum = tr[:npass, :, 14].sum(axis=1)
print("dirty node evaluations per pass:", dsum.tolist())
print("refined-dirty per pass:", rsum.tolist())
print("changed per pass:", csum.tolist())
print("totals: dirty", int(dsum.sum()), "refined", int(rsum.sum()), "changed", int(csum.sum()))
probe = buf[got - 8:got].astype(np.int64)
nd = max(1, int(tr[:npass, :, 6].sum()))
nst = npass * nb * S
names = ["ballot", "loads->s", "->disc", "->t0", "->best", "fold-xchg", "leader", "bar"]
print("probe cycles per dirty step (warp 0 lane 0, all bands):",
      {nm: round(float(probe[i]) / (nd if 0 < i < 7 else nst), 1) for i, nm in enumerate(names)}, "(ballot, bar per step)")
# handoff anatomy for pass 1, bands 1..5: prev band's step-0 compute start, its column-0 mailbox put,
# this band's first mailbox column, this band's step-0 start (us, relative to pass start)
for pa in sorted({1, npass - 4, npass // 2}):
  r = tr[pa]; t0 = r[:, 0].min()
  print(f"-- pass {pa} handoff anatomy (us)")
  for b in list(range(1, 6)) + [100, 101, 200]:
    print(f"  band {b}: start {(r[b,0]-t0)/1e3:8.1f} chunk0 {(r[b,16]-t0)/1e3:8.1f} prev step0 {(r[b-1,9]-t0)/1e3:8.1f} prev last-line col0 done {(r[b-1,10]-t0)/1e3:8.1f} prev mbox col0 put {(r[b-1,8]-t0)/1e3:8.1f} -> mbox col0 seen {(r[b,4]-t0)/1e3:8.1f} -> step0 {(r[b,9]-t0)/1e3:8.1f}")

