"""Batch sharding of independent grids across ranks.

The exact Gauss-Seidel chain of one grid cannot be split across GPUs, so
multi-GPU work is partitioned by scene / sample: rank r of W owns a
contiguous block of the batch.  No data-path collective is needed; the only
collectives are scalar reductions (step time max, loss sum) used for
reporting, and — for the C5 training workload — the encoder gradient
all-reduce.
"""
from __future__ import annotations


def shard_range(n_items: int, rank: int, world: int):
    """Contiguous [lo, hi) block of `n_items` for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def reduce_step_stats(local_ms: float, local_units: float, group=None):
    """(max step time over ranks, total units over ranks) — the bench's
    whole-job aggregate.  Uses whatever backend the process group has
    (NCCL on the GPU box, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return local_ms, local_units
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([local_ms], dtype=torch.float64, device=dev)
    u = torch.tensor([local_units], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(u, op=dist.ReduceOp.SUM, group=group)
    return float(t.item()), float(u.item())
