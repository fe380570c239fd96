"""C5 training step (training.py): encoder -> projection -> solve -> MSE ->
adjoint -> encoder gradients, under DDP (NCCL, world size 1 here; the
round-end box has one GPU)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _batch(n=24, B=2, seed=0):
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed)
    cov = torch.randn((B, 3, n, n), generator=g).cuda()
    src = torch.zeros((B, n, n), dtype=torch.uint8, device="cuda")
    src[0, n // 2, n // 2] = 1
    src[1, 3, n - 4] = 1
    obs = (torch.rand((B, n, n), generator=g) < 0.3).to(torch.uint8).cuda()
    tgt = torch.rand((B, n, n), generator=g, dtype=torch.float64).cuda()
    return cov, src, obs, tgt


def test_encoder_grads_flow_through_solver_and_projection():
    import torch

    from paper_2603_00035_b200 import training

    torch.manual_seed(0)
    model = training.RandersEncoder().cuda()
    assert 100_000 < sum(p.numel() for p in model.parameters()) < 130_000
    batch = _batch()
    loss = training.c5_loss(model, *batch, 1.0 / 24)
    loss.backward()
    norms = [p.grad.norm().item() for p in model.parameters()]
    assert all(np.isfinite(norms)) and sum(norms) > 0


def test_ddp_train_steps_reduce_loss():
    import torch
    import torch.distributed as dist

    from paper_2603_00035_b200 import training

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        torch.manual_seed(1)
        model = torch.nn.parallel.DistributedDataParallel(training.RandersEncoder().cuda())
        opt = torch.optim.Adam(model.parameters(), lr=3e-3)
        batch = _batch(seed=2)
        losses = [float(training.train_step(model, opt, batch, 1.0 / 24)) for _ in range(6)]
        assert losses[-1] < losses[0], losses
    finally:
        dist.destroy_process_group()


def test_bf16_encoder_matches_fp32_loss_and_trains():
    """bench.py --workload c5 --encoder bf16: the encoder runs under bf16
    autocast with channels-last activations; the solver path stays fp64.  The
    loss is close to the fp32 encoder's and training still reduces it."""
    import torch

    from paper_2603_00035_b200 import training

    torch.manual_seed(3)
    ref = training.RandersEncoder().cuda()
    model = training.prepare_encoder(training.RandersEncoder().cuda(), "bf16")
    model.load_state_dict(ref.state_dict())
    cov, src, obs, tgt = _batch(seed=4)
    l32 = float(training.c5_loss(ref, cov, src, obs, tgt, 1.0 / 24).detach())
    x = training.encoder_input(cov, "bf16")
    l16 = float(training.c5_loss(model, x, src, obs, tgt, 1.0 / 24, precision="bf16").detach())
    assert abs(l16 - l32) <= 0.05 * abs(l32), (l16, l32)
    opt = torch.optim.Adam(model.parameters(), lr=3e-3)
    losses = [float(training.train_step(model, opt, (x, src, obs, tgt), 1.0 / 24, precision="bf16"))
              for _ in range(6)]
    assert losses[-1] < losses[0], losses
