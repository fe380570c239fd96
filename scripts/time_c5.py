"""Stage times of one C5 micro-batch (bench.py --workload c5) on cuda:0.

Times, with CUDA events after warm-up: the encoder forward+backward alone
(per encoder precision), the projection forward, the solve, the adjoint
backward through the solve, and the whole micro-batch loss+backward.
Usage: python scripts/time_c5.py [n] [micro_batch]
"""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_00035_b200 as rfk  # noqa: E402
from paper_2603_00035_b200 import torch_ops, training  # noqa: E402
from paper_2603_00035_b200 import workload as wl  # noqa: E402


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    dev = torch.device("cuda", 0)
    torch.backends.cudnn.benchmark = os.environ.get("CUDNN_BENCH", "0") == "1"
    h = 1.0 / n
    torch.manual_seed(1234)
    truth = training.RandersEncoder().to(dev)
    torch.manual_seed(7)
    src = wl.point_source(n, n, device=dev).expand(B, n, n).contiguous()
    obs = wl.observation_mask(src[0]).expand(B, n, n).contiguous()
    cov = torch.stack([torch.stack([wl.correlated_noise(n, n, 3, 3 * s + k, device=dev) for k in range(3)])
                       for s in range(B)]).float()
    with torch.no_grad():
        tgt, _ = rfk.solve(*training.raw_to_fields(truth(cov)), src, h)
    print(f"n={n} micro_batch={B} cudnn.allow_tf32={torch.backends.cudnn.allow_tf32} "
          f"cudnn.benchmark={torch.backends.cudnn.benchmark}")
    for prec in training.ENCODER_PRECISIONS:
        model = training.RandersEncoder().to(dev)
        training.prepare_encoder(model, prec)
        x = training.encoder_input(cov, prec)

        def enc():
            model.zero_grad(set_to_none=True)
            with training.encoder_autocast(prec):
                out = model(x)
            out.float().square().mean().backward()

        def full():
            model.zero_grad(set_to_none=True)
            training.c5_loss(model, x, src, obs, tgt, h, precision=prec).backward()

        print(f"  {prec:5s}: encoder fwd+bwd {timed(enc):8.2f} ms   micro-batch loss+backward {timed(full):8.2f} ms")
    model = training.RandersEncoder().to(dev)
    with torch.no_grad():
        raw = model(cov)
    fields = [f.detach().requires_grad_(True) for f in training.raw_to_fields(raw)]
    print(f"  raw_to_fields (fp64 + projection)   {timed(lambda: training.raw_to_fields(raw)):8.2f} ms")
    print(f"  solve                                {timed(lambda: rfk.solve(*[f.detach() for f in fields], src, h)):8.2f} ms")

    def solve_bwd():
        t = torch_ops.eikonal_solve(*fields, src, h)
        t.backward(torch.ones_like(t) * obs)

    print(f"  solve + adjoint backward             {timed(solve_bwd):8.2f} ms")


if __name__ == "__main__":
    main()
