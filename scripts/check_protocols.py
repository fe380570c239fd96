"""Protocol-checker stress (the compute-sanitizer stand-in: this pool refuses
compute-sanitizer).  Runs with RFK_LIBRARY pointing at a build with
-DRFK_SWEEP_CHECKED=1 (scripts/build_variant.sh chk): every shared-memory ring
read of the sweep is checked against the slot's position/step tag, and a
violation fails the solve.  Repeats the golden solves in every sweep order,
random grids of many shapes (skinny, tiny, non-square), concurrent batched
grids, and one 4096^2 solve, comparing results with the oracle where cheap.
Prints one summary line per group and a final verdict."""
import glob
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2603_00035_b200 as rfk
from paper_2603_00035_b200 import workload as wl

reps = int(os.environ.get("REPS", "10"))
fails, solves = 0, 0
t0 = time.time()
try:
    from oracle.pyoracle import RefLib
    ref = RefLib()
except Exception:
    ref = None


def run(F, src, h, **kw):
    global fails, solves
    solves += 1
    try:
        return rfk.solve(*F, src, h, **kw)
    except rfk.Error as e:
        fails += 1
        print("VIOLATION:", e, flush=True)
        return None, None


for path in sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "*.npz"))):
    with np.load(path) as z:
        G = {k: z[k] for k in z.files}
    if "fixed_values" in G:
        continue
    F, src, h = list(G["fields"]), G["src"], float(G["h"])
    bad = 0
    for order in ((0, 1, 2, 3), (3, 1, 0, 2), (2, 2, 2, 2)):
        want = ref.solve(*F, src, h, order=list(order)).t if ref else None
        for _ in range(reps):
            t, rep = run(F, src, h, sweep_order=order)
            if t is not None and want is not None and not np.array_equal(t, want):
                bad += 1
    print(f"{os.path.basename(path)}: {3 * reps} solves, {bad} result mismatches", flush=True)
    fails += bad

rng = np.random.default_rng(5)
shapes = [(3, 3), (3, 700), (700, 3), (17, 300), (300, 17), (31, 33), (64, 200), (200, 64), (256, 257)]
for R, C in shapes:
    F = wl.host_fields(R, int(rng.integers(1, 99)), 0.2, cols=C)
    src = np.zeros((R, C), np.uint8)
    src[int(rng.integers(0, R)), int(rng.integers(0, C))] = 1
    want = ref.solve(*F, src, 1.0 / max(R, C), max_iters=200).t if ref else None
    bad = 0
    for _ in range(reps):
        t, rep = run(F, src, 1.0 / max(R, C), max_iters=200)
        if t is not None and want is not None and not np.array_equal(t, want):
            bad += 1
    print(f"random {R}x{C}: {reps} solves, {bad} result mismatches", flush=True)
    fails += bad

import torch
F = [torch.as_tensor(x).cuda() for x in wl.host_fields(512, 3, 0.2)]
src = torch.zeros((6, 512, 512), dtype=torch.uint8, device="cuda")
for b in range(6):
    src[b, (37 * b + 11) % 512, (91 * b + 5) % 512] = 1
for _ in range(3):
    tb, rb = run(F, src, 1.0 / 512)
print("batched 6 x 512^2 (concurrent slots): 3 solves", flush=True)
F = [torch.as_tensor(x).cuda() for x in wl.host_fields(4096, 1, 0.2)]
src = torch.as_tensor(wl.host_point_source(4096, 4096)).cuda()
t, rep = run(F, src, 1.0 / 4096)
print(f"4096^2: K={rep.iterations if rep else None}", flush=True)
lib = os.environ.get("RFK_LIBRARY", "")
kind = "checked solves" if "chk" in os.path.basename(lib) else \
    "solves, results only (RFK_LIBRARY is not a -DRFK_SWEEP_CHECKED build: no tag checks)"
print(f"library: {lib or 'paper_2603_00035_b200/librfk.so'}")
print(f"protocol checker: {solves} {kind}, {fails} violations or mismatches ({time.time() - t0:.0f} s)")
sys.exit(1 if fails else 0)
