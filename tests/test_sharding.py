"""Multi-process (gloo, world_size 2) tests of the batch sharding used for
N>1 runs: every scene lands on exactly one rank and the reported aggregate is
max-time / total-units over ranks."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2603_00035_b200.sharding import reduce_step_stats, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 64, 65):
        for w in (1, 2, 3, 8):
            got = []
            for r in range(w):
                lo, hi = shard_range(n, r, w)
                got.extend(range(lo, hi))
                assert hi - lo in (n // w, n // w + 1)
            assert got == list(range(n))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(64, rank, world)
    # pretend each scene costs (index+1) ms and 1000 node-updates
    ms = float(sum(i + 1 for i in range(lo, hi)))
    units = 1000.0 * (hi - lo)
    t, u = reduce_step_stats(ms, units)
    q.put((rank, lo, hi, t, u))
    dist.destroy_process_group()


def test_gloo_two_ranks_aggregate():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, lo0, hi0, t0, u0), (r1, lo1, hi1, t1, u1) = res
    assert (lo0, hi0, lo1, hi1) == (0, 32, 32, 64)
    assert t0 == t1 == float(sum(range(33, 65)))  # max over ranks
    assert u0 == u1 == 64000.0                     # whole-job total
