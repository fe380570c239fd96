"""fp32 mode (parity target 1e-4 relative to the fp64
oracle): the same exact wavefront with fp32 storage and arithmetic."""
import numpy as np
import pytest

from conftest import golden_cases, load_golden

pytestmark = pytest.mark.gpu


def _rel_err(t32, t64):
    t32 = np.asarray(t32, np.float64)
    m = t64 < 1e9
    assert np.array_equal(m, t32 < 1e9), "reached sets differ"
    return float(np.max(np.abs(t32[m] - t64[m]) / np.maximum(np.abs(t64[m]), 1e-3)))


@pytest.mark.parametrize("name", [c for c in golden_cases() if c != "fixed36x50"])
def test_fp32_solve_vs_fp64_oracle_golden(name, oracle):
    import paper_2603_00035_b200 as rfk
    G = load_golden(name)
    F, src, h = G["fields"], G["src"], float(G["h"])
    ref = oracle.solve(*F, src, h)
    t32, rep = rfk.solve_f32(*F, src, h)
    assert t32.dtype == np.float32 and rep.converged
    assert _rel_err(t32, ref.t) <= 1e-4


@pytest.mark.parametrize("n,seed,ds", [(256, 3, 0.2), (200, 4, 0.0)])
def test_fp32_random_fields_and_batch(n, seed, ds, reflib):
    import torch

    import paper_2603_00035_b200 as rfk
    F = reflib.random_feasible_fields(n, seed, ds)
    src = np.zeros((3, n, n), np.uint8)
    src[0, n // 2, n // 2] = 1
    src[1, n // 5, n // 3] = 1
    src[2, 7, n - 9] = 1
    t64, _ = rfk.solve(*F, src, 1.0 / n)
    t32, rep = rfk.solve_f32(*F, src, 1.0 / n)
    for b in range(3):
        assert _rel_err(t32[b], t64[b]) <= 1e-4
    # device memory, per-grid metrics (param_stride), concurrent slots
    Fd = [torch.stack([torch.tensor(x, device="cuda") * (1.0 if i > 2 else 1.0 + 0.05 * b) for b in range(3)])
          for i, x in enumerate(F)]
    sd = torch.tensor(src, device="cuda")
    td, _ = rfk.solve_f32(*Fd, sd, 1.0 / n)
    t64d, _ = rfk.solve(*Fd, sd, 1.0 / n)
    for b in range(3):
        assert _rel_err(td[b].cpu().numpy(), t64d[b].cpu().numpy()) <= 1e-4


def test_fp32_4096_vs_reference_digest():
    """fp32 mode at C3's size against the fp64 solution whose bits equal the
    reference library's (tests/golden/large_hashes.json c3, checked here
    through its digest): 1e-4 relative, iteration count within one."""
    import json
    import os

    import torch

    import paper_2603_00035_b200 as rfk
    from conftest import GOLDEN_DIR
    from paper_2603_00035_b200 import workload as wl
    G = json.load(open(os.path.join(GOLDEN_DIR, "large_hashes.json")))["c3"]
    n = G["n"]
    F = [torch.as_tensor(x).cuda() for x in wl.host_fields(n, G["seed"], G["drift"])]
    src = torch.as_tensor(wl.host_point_source(n, n)).cuda()
    t64, rep64 = rfk.solve(*F, src, 1.0 / n)
    assert wl.fields_digest(t64.cpu().numpy()) == G["runs"][0]["t_digest"]
    t32, rep32 = rfk.solve_f32(*F, src, 1.0 / n)
    assert bool(rep32.converged), (rep32.iterations, rep32.max_delta_history)
    # the stopping test max_delta < tol sees fp32 rounding (~1e-7 at T ~ 1):
    # C3's fp64 run stops at 9.5e-7 after 16 passes, the fp32 run saw 1.1e-6
    # there and takes a 17th
    assert abs(int(rep32.iterations) - int(rep64.iterations)) <= 1, (rep32.max_delta_history,
                                                                     rep64.max_delta_history)
    m = t64 < 1e9
    assert torch.equal(m, t32 < 1e9)
    rel = ((t32.double() - t64).abs()[m] / t64[m].abs().clamp_min(1e-3)).max().item()
    assert rel <= 1e-4, rel


@pytest.mark.parametrize("device,accumulate", [(False, False), (True, False), (True, True)])
def test_fp32_backward_is_the_widened_fp64_backward(device, accumulate, reflib):
    """rfk_backward_f32 = round-to-fp32 of rfk_backward on the exactly widened
    fp32 inputs, bit for bit (host and device memory, per-grid and summed
    gradients)."""
    import torch

    import paper_2603_00035_b200 as rfk
    n = 96
    F = [np.asarray(x, np.float32) for x in reflib.random_feasible_fields(n, 11, 0.2)]
    src = np.zeros((3, n, n), np.uint8)
    for b in range(3):
        src[b, (17 + 29 * b) % n, (5 + 41 * b) % n] = 1
    lg = np.random.default_rng(3).standard_normal((3, n, n)).astype(np.float32)
    if device:
        F = [torch.as_tensor(x).cuda() for x in F]
        src, lg = torch.as_tensor(src).cuda(), torch.as_tensor(lg).cuda()
    t32, _ = rfk.solve_f32(*F, src, 1.0 / n)
    g32, cl32 = rfk.backward_f32(t32, *F, src, 1.0 / n, lg, accumulate=accumulate)
    wide = (lambda x: x.double()) if device else (lambda x: np.asarray(x, np.float64))
    _, g64, cl64 = rfk.backward(wide(t32), *(wide(x) for x in F), src, 1.0 / n, wide(lg), accumulate=accumulate,
                                want_lambda=False)
    host = (lambda x: x.cpu().numpy()) if device else np.asarray
    assert host(g32).dtype == np.float32
    assert np.array_equal(host(g32), host(g64).astype(np.float32))
    assert np.array_equal(np.asarray(cl32), np.asarray(cl64))


def test_fp32_gradient_agrees_with_fp64_gradient(reflib):
    """The whole fp32 chain (solve_f32 -> loss -> backward_f32) against the
    fp64 chain on the same fields: 1e-3 relative in the L2 norm of each
    gradient plane (stencil choices at near-ties may differ)."""
    import paper_2603_00035_b200 as rfk
    n = 160
    F = reflib.random_feasible_fields(n, 21, 0.2)
    src = np.zeros((2, n, n), np.uint8)
    src[0, n // 3, n // 2] = 1
    src[1, 9, n - 12] = 1
    obs = (np.random.default_rng(8).random((2, n, n)) < 0.3) & (src == 0)
    t64, _ = rfk.solve(*F, src, 1.0 / n)
    tgt = t64 * 1.05
    lg64 = np.where(obs, 2.0 * (t64 - tgt), 0.0)
    t32, _ = rfk.solve_f32(*F, src, 1.0 / n)
    lg32 = np.where(obs, 2.0 * (np.asarray(t32, np.float64) - tgt), 0.0).astype(np.float32)
    _, g64, _ = rfk.backward(t64, *F, src, 1.0 / n, lg64, accumulate=True, want_lambda=False)
    g32, _ = rfk.backward_f32(t32, *F, src, 1.0 / n, lg32, accumulate=True)
    for k in range(5):
        a, b = np.asarray(g32[k], np.float64), g64[k]
        rel = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
        assert rel <= 1e-3, (k, rel)
