"""Size-independent properties at the benchmark's full size (C3: 4096^2 Randers
with drift, BASELINE.json), where the CPU oracle would need minutes per solve:

* the solve converges and its sources hold 0, every other node a finite,
  positive arrival time;
* the converged field is a fixed point of the reference's own candidate
  evaluation: identify_stencils re-derives every node's value from its
  recorded stencil (InconsistentFixedPoint otherwise), and node_update on a
  sample of nodes cannot improve any of them by tol or more;
* the max|dT| history decreases to below tol;
* a batch of two grids (concurrent slots) equals two single solves bit for bit;
* the fused backward gives finite gradients and zero adjoint at the source.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 4096


@pytest.fixture(scope="module")
def problem():
    import torch

    import paper_2603_00035_b200 as rfk
    from paper_2603_00035_b200 import workload as wl
    F = wl.randers_fields(N, 1, 0.2)
    src = wl.point_source(N, N)
    t, rep = rfk.solve(*F, src, 1.0 / N)
    torch.cuda.synchronize()
    return F, src, t, rep


def test_converged_field(problem):
    import torch
    F, src, t, rep = problem
    assert bool(rep.converged) and 1 <= int(rep.iterations) <= 50
    s = src.bool()
    assert torch.all(t[s] == 0.0)
    rest = t[~s]
    assert torch.all(torch.isfinite(rest)) and torch.all(rest > 0.0) and torch.all(rest < 1e9)
    hist = np.asarray(rep.max_delta_history)
    assert hist[-1] < 1e-6 <= hist[-2]
    assert np.all(np.diff(hist[1:]) <= 0.0) or hist[-1] < 1e-6  # geometric decay after the first sweeps


def test_fixed_point_of_reference_candidates(problem):
    import torch

    import paper_2603_00035_b200 as rfk
    F, src, t, rep = problem
    h = 1.0 / N
    rec = rfk.identify_stencils(t, *F, src, h, 1e-6)  # raises InconsistentFixedPoint if any node disagrees
    assert int(rec.two_point_count) + int(rec.one_point_count) == N * N - 1
    rng = np.random.default_rng(0)
    nodes = rng.choice(N * N, size=1 << 16, replace=False).astype(np.int32)
    nodes = nodes[~src.flatten().cpu().numpy()[nodes].astype(bool)]
    c = rfk.best_candidates(nodes, t, *F, h, node_update=True)
    tv = t.flatten()[torch.as_tensor(nodes, device=t.device, dtype=torch.long)]
    improvement = (tv - c["t0"]).max().item()
    assert improvement < 1e-6


def test_batch_of_two_equals_singles(problem):
    import torch

    import paper_2603_00035_b200 as rfk
    F, src, t, rep = problem
    src2 = torch.zeros((2, N, N), dtype=torch.uint8, device=t.device)
    src2[0] = src
    src2[1, N // 5, (3 * N) // 4] = 1
    tb, rb = rfk.solve(*F, src2, 1.0 / N)
    assert torch.equal(tb[0], t) and int(rb.iterations[0]) == int(rep.iterations)
    t1, _ = rfk.solve(*F, src2[1], 1.0 / N)
    assert torch.equal(tb[1], t1)


def test_backward_full_size(problem):
    import torch

    import paper_2603_00035_b200 as rfk
    from paper_2603_00035_b200 import workload as wl
    F, src, t, rep = problem
    h = 1.0 / N
    g, loss, unreached = rfk.loss_grad_mse(t, wl.observation_mask(src), torch.zeros_like(t), exact=False)
    lam, grads, clamped = rfk.backward(t, *F, src, h, g)
    assert torch.all(torch.isfinite(grads)) and torch.all(torch.isfinite(lam))
    assert torch.all(lam[src.bool()] == 0.0)
    assert int(clamped) < N  # a handful of clamped diagonals at most
    assert float(grads.abs().max()) > 0.0
