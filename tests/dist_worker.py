"""Worker for tests/test_multirank_gpu.py, launched by torchrun with world
size 2 and the gloo backend on the one GPU of the test box (ranks here run
independent work -- no rank waits on another's kernels -- so sharing a device
is sound; the production backend is NCCL, one rank per GPU).

  mode c4: the C4 data term sharded by scene (sharding.shard_range): each
           rank solves + differentiates its scenes and writes per-scene
           digests of T and of the 5 gradient planes;
  mode c5: one DDP step of the C5 encoder over a batch split across the
           ranks; rank 0 writes the all-reduced encoder gradients.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch
import torch.distributed as dist


def c4(out_dir, n, scenes):
    import paper_2603_00035_b200 as rfk
    from paper_2603_00035_b200 import workload as wl
    from paper_2603_00035_b200.sharding import reduce_step_stats, shard_range
    rank, world = dist.get_rank(), dist.get_world_size()
    lo, hi = shard_range(scenes, rank, world)
    h = 1.0 / n
    res = {}
    units = 0
    for s in range(lo, hi):
        F = [torch.as_tensor(x).cuda() for x in wl.host_fields(n, s, 0.2)]
        src = torch.as_tensor(wl.host_point_source(n, n)).cuda()
        obs = torch.as_tensor(wl.host_observation_mask(src.cpu().numpy(), stream=100 + s)).cuda()
        t, rep = rfk.solve(*F, src, h)
        g, loss, _ = rfk.loss_grad_mse(t, obs, torch.zeros_like(t))
        _, grads, _ = rfk.backward(t, *F, src, h, g)
        res[s] = {"K": int(rep.iterations), "t": wl.fields_digest(t.cpu().numpy()),
                  "grads": wl.fields_digest(grads.cpu().numpy()), "loss": float(loss).hex()}
        units += wl.node_updates(rep.iterations, n * n, 1, int(((t < 1e9) & (src == 0)).sum()))
    t_ms, total = reduce_step_stats(float(rank + 1), float(units))
    with open(os.path.join(out_dir, f"c4_rank{rank}.json"), "w") as f:
        json.dump({"scenes": res, "lo": lo, "hi": hi, "reduced_ms": t_ms, "reduced_units": total,
                   "local_units": units}, f)


def c5(out_dir, n, batch):
    from paper_2603_00035_b200 import training
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.manual_seed(3)
    model = torch.nn.parallel.DistributedDataParallel(training.RandersEncoder().cuda().double())
    g = torch.Generator(device="cpu").manual_seed(11)
    cov = torch.randn((batch, 3, n, n), generator=g, dtype=torch.float64)
    src = torch.zeros((batch, n, n), dtype=torch.uint8)
    for b in range(batch):
        src[b, (5 + 7 * b) % n, (11 + 3 * b) % n] = 1
    obs = (torch.rand((batch, n, n), generator=g) < 0.3).to(torch.uint8)
    tgt = torch.rand((batch, n, n), generator=g, dtype=torch.float64)
    per = batch // world
    sl = slice(rank * per, (rank + 1) * per)
    part = [x[sl].cuda() for x in (cov, src, obs, tgt)]
    loss = training.c5_loss(model, *part, 1.0 / n)
    loss.backward()  # DDP all-reduces (averages) the encoder gradients
    if rank == 0:
        grads = [p.grad.detach().double().cpu().numpy() for p in model.module.parameters()]
        np.savez(os.path.join(out_dir, "c5_ddp_grads.npz"), *grads)


if __name__ == "__main__":
    mode, out_dir = sys.argv[1], sys.argv[2]
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    dist.init_process_group("gloo")
    try:
        if mode == "c4":
            c4(out_dir, int(sys.argv[3]), int(sys.argv[4]))
        else:
            c5(out_dir, int(sys.argv[3]), int(sys.argv[4]))
    finally:
        dist.destroy_process_group()
