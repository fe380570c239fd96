"""The sharded paths with more than one rank: torchrun, world
size 2, gloo, on the test box's one GPU (tests/dist_worker.py).

* C4: scenes sharded over the ranks give every scene the same T, loss and
  gradient bits as a single-rank run; the step aggregate is max-time /
  total-units over the ranks.
* C5: one DDP step (fp64 encoder) over a batch split across the ranks gives
  the encoder gradients of a single process on the union batch to 1e-12 (the
  all-reduce averages two partial means in another order).
* bench.py --workload c4/c5 under torchrun (the distributed branches of the
  bench) run and print their JSON line.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _torchrun(args, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={29700 + os.getpid() % 200}"] + args
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    return p


def test_c4_two_ranks_equal_single_rank(tmp_path):
    import torch

    import paper_2603_00035_b200 as rfk
    from paper_2603_00035_b200 import workload as wl
    n, scenes = 192, 5
    _torchrun([os.path.join(ROOT, "tests", "dist_worker.py"), "c4", str(tmp_path), str(n), str(scenes)])
    ranks = [json.load(open(tmp_path / f"c4_rank{r}.json")) for r in range(2)]
    assert [(r["lo"], r["hi"]) for r in ranks] == [(0, 3), (3, 5)]
    got = {int(k): v for r in ranks for k, v in r["scenes"].items()}
    assert sorted(got) == list(range(scenes))
    assert ranks[0]["reduced_ms"] == ranks[1]["reduced_ms"] == 2.0
    assert ranks[0]["reduced_units"] == ranks[1]["reduced_units"] == sum(r["local_units"] for r in ranks)
    h = 1.0 / n
    for s in range(scenes):
        F = [torch.as_tensor(x).cuda() for x in wl.host_fields(n, s, 0.2)]
        src = torch.as_tensor(wl.host_point_source(n, n)).cuda()
        obs = torch.as_tensor(wl.host_observation_mask(src.cpu().numpy(), stream=100 + s)).cuda()
        t, rep = rfk.solve(*F, src, h)
        g, loss, _ = rfk.loss_grad_mse(t, obs, torch.zeros_like(t))
        _, grads, _ = rfk.backward(t, *F, src, h, g)
        assert got[s]["K"] == rep.iterations
        assert got[s]["t"] == wl.fields_digest(t.cpu().numpy()), s
        assert got[s]["grads"] == wl.fields_digest(grads.cpu().numpy()), s
        assert got[s]["loss"] == float(loss).hex()


def test_c5_ddp_two_ranks_equal_union_batch(tmp_path):
    import torch

    from paper_2603_00035_b200 import training
    n, batch = 32, 4
    _torchrun([os.path.join(ROOT, "tests", "dist_worker.py"), "c5", str(tmp_path), str(n), str(batch)])
    with np.load(tmp_path / "c5_ddp_grads.npz") as z:
        ddp = [z[k] for k in z.files]
    torch.manual_seed(3)
    model = training.RandersEncoder().cuda().double()
    g = torch.Generator(device="cpu").manual_seed(11)
    cov = torch.randn((batch, 3, n, n), generator=g, dtype=torch.float64)
    src = torch.zeros((batch, n, n), dtype=torch.uint8)
    for b in range(batch):
        src[b, (5 + 7 * b) % n, (11 + 3 * b) % n] = 1
    obs = (torch.rand((batch, n, n), generator=g) < 0.3).to(torch.uint8)
    tgt = torch.rand((batch, n, n), generator=g, dtype=torch.float64)
    loss = training.c5_loss(model, *(x.cuda() for x in (cov, src, obs, tgt)), 1.0 / n)
    loss.backward()
    single = [p.grad.detach().double().cpu().numpy() for p in model.parameters()]
    assert len(single) == len(ddp)
    for a, b in zip(ddp, single):
        # fp64 encoder: the ranks' partial means are averaged by the all-reduce
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12 * float(np.abs(b).max()))


@pytest.mark.parametrize("workload,extra", [("c4", ["--scenes", "4", "--grid", "256", "--chunk", "2"]),
                                            ("c5", ["--scenes", "4", "--grid", "64", "--chunk", "2"])])
def test_bench_distributed_branches(workload, extra):
    p = _torchrun([os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1",
                   "--workload", workload, "--dist-backend", "gloo"] + extra)
    line = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
