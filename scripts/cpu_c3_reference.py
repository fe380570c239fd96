"""Time the reference library's own forward + adjoint (solve, loss_grad_mse,
identify_stencils, solve_adjoint, param_gradients: the body of
adjoint_gradient, src/oracle.cpp:226-247) at C3 -- 4096^2 Randers, the bench's
inputs -- on one host core, once.  ~11 min.  Writes
profiles/r02_cpu_c3_reference.json (test infrastructure / CPU baseline only)."""
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from oracle.pyoracle import RefLib
from paper_2603_00035_b200 import workload as wl

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "r02_cpu_c3_reference.json")
F = wl.host_fields(n, 1, 0.2)
src = wl.host_point_source(n, n)
obs = wl.host_observation_mask(src)
ref = RefLib()
t0 = time.time()
wall, times, K, nrec, conv = ref.pipeline(*F, src, obs, np.zeros((n, n)), 1.0 / n, 1e-6, 50, 1, 1)
W = wl.node_updates(K, n * n, 1, nrec)
model = "unknown"
with open("/proc/cpuinfo") as f:
    for line in f:
        if line.startswith("model name"):
            model = line.split(":", 1)[1].strip()
            break
res = {"grid": f"{n}x{n}", "K": K, "records": nrec, "converged": conv, "node_updates": W,
       "seconds": wall, "phase_seconds": {"solve": times[0], "loss": times[1], "identify": times[2],
                                          "adjoint": times[3], "param_grads": times[4]},
       "node_updates_per_s": W / wall, "cores": 1, "kind": "reference",
       "host": {"nproc": os.cpu_count(), "model": model, "node": platform.node()},
       "input_digest": wl.fields_digest(*F, src, obs),
       "how": "oracle/_ref (the reference's own sources, -O3 -DNDEBUG -ffp-contract=off), one thread"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
