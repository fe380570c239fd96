"""Bit parity at BASELINE.json's own configs (C2 1024^2 Riemannian, one C4
2048^2 Randers scene, C3 4096^2 Randers -- the bench's workload), against
digests of the reference library's own outputs on the same inputs
(tests/golden/gen_large.py ran oracle/_ref once; the planes are too large to
commit, their sha256 digests are in tests/golden/large_hashes.json).

Compared bit for bit: the input planes (regenerated on this host by the
deterministic generator), T, K, converged, the max|dT| history, the stencil
records (type, stencil, donors) and their caches, dL/dT and the loss, the
adjoint lambda, the five parameter-gradient planes and the clamped-diagonal
count (src/sweeper.cpp:133-158, src/adjoint.cpp:10-160).  "Stencil choices
identical" at 4096^2 is the records digest.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR

pytestmark = pytest.mark.gpu

with open(os.path.join(GOLDEN_DIR, "large_hashes.json")) as _f:
    GOLD = json.load(_f)


def _inputs(name):
    from paper_2603_00035_b200 import workload as wl
    g = GOLD[name]
    n = g["n"]
    F = wl.host_fields(n, g["seed"], g["drift"])
    src = wl.host_point_source(n, n)
    obs = wl.host_observation_mask(src)
    assert wl.fields_digest(*F, src, obs) == g["input_digest"], \
        f"{name}: the host generator produced different inputs than the golden's"
    return F, src, obs, g


@pytest.mark.parametrize("name", sorted(GOLD))
def test_fullsize_bitwise_vs_reference(name):
    import paper_2603_00035_b200 as rfk
    from paper_2603_00035_b200 import workload as wl
    F, src, obs, g = _inputs(name)
    h = g["h"]
    for k, r in enumerate(g["runs"]):
        t, rep = rfk.solve(*F, src, h, tol=r["tol"], max_iters=r["max_iters"], sweep_order=tuple(r["order"]))
        assert rep.iterations == r["iterations"], (name, k, rep.iterations, r["iterations"])
        assert rep.converged == r["converged"]
        assert [float(x).hex() for x in rep.max_delta_history] == r["history"], (name, k, "history")
        assert wl.fields_digest(t) == r["t_digest"], f"{name} run {k}: T differs from the reference"
        if "lam_digest" not in r:
            continue
        grad, loss, unr = rfk.loss_grad_mse(t, obs, np.zeros_like(t), exact=True)
        assert wl.fields_digest(grad) == r["loss_grad_digest"]
        assert float(loss).hex() == r["loss"] and unr == r["unreached"]
        rec = rfk.identify_stencils(t, *F, src, h, r["tol"])
        assert [rec.two_point_count, rec.one_point_count] == r["rec_counts"]
        assert wl.fields_digest(rec.type, rec.stencil, rec.donor1, rec.donor2) == r["rec_digest"], \
            f"{name}: stencil choices differ from the reference"
        assert wl.fields_digest(np.ascontiguousarray(rec.c)) == r["rec_c_digest"]
        lam, grads, cl = rfk.backward(t, *F, src, h, grad, r["tol"])
        assert cl == r["clamped"]
        assert wl.fields_digest(lam) == r["lam_digest"], f"{name}: lambda differs from the reference"
        assert wl.fields_digest(grads) == r["grads_digest"], f"{name}: gradients differ from the reference"


def test_c2_live_oracle_1024(reflib):
    """A live comparison at C2's size (the reference library on this host,
    ~10 s): T, K and history, plus the plane-level first mismatch if any."""
    import paper_2603_00035_b200 as rfk
    from conftest import assert_bitwise
    F, src, obs, g = _inputs("c2")
    h = g["h"]
    ref = reflib.solve(*F, src, h, tol=1e-6, max_iters=50)
    t, rep = rfk.solve(*F, src, h, tol=1e-6, max_iters=50)
    assert rep.iterations == ref.iterations
    assert_bitwise(t, ref.t, "C2 T")
    assert_bitwise(rep.max_delta_history, ref.history[:ref.iterations], "C2 history")
