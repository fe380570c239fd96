"""Command line front end for the two hot-path subcommands of the reference's
`rfeik` tool (tools/main.cpp): `solve` (cmd_solve, :56-85) and `bench`
(cmd_bench, :304-347), with the same flags, stdout lines, CSV output and exit
codes (0 ok, 2 usage, 3 numerical).  The solves run on the GPU.

    python -m paper_2603_00035_b200 solve --metric g.rfek --drift b.rfek \\
        --sources s.rfek --h 0.01 --out t.rfek
    python -m paper_2603_00035_b200 bench --sizes 50,100,200,400 --out bench.csv
"""
from __future__ import annotations

import argparse
import sys
import time

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_NUMERICAL = 0, 2, 3


def _cmd_solve(a) -> int:
    from . import api, field_io as fio
    g = fio.read_metric(a.metric)
    b = fio.read_drift(a.drift)
    src = fio.read_mask(a.sources)
    if b[0].shape != g[0].shape or src.shape != g[0].shape:
        print("dimension mismatch", file=sys.stderr)
        return EXIT_USAGE
    max_iters = a.max_iters
    if a.solver == "jacobi" and max_iters is None:
        max_iters = api.jacobi_iteration_budget(*g[0].shape)
    if max_iters is None:
        max_iters = 50
    fn = api.solve_jacobi if a.solver == "jacobi" else api.solve
    t, rep = fn(*g, *b, src, a.h, tol=a.tol, max_iters=max_iters)
    fio.write_arrival(a.out, t)
    hist = rep.max_delta_history
    last = float(hist[-1]) if len(hist) else 0.0
    print(f"iters={rep.iterations} max_delta={fio._to_chars(last)}")
    return EXIT_OK if rep.converged else EXIT_NUMERICAL


def _cmd_bench(a) -> int:
    import torch

    from . import api, field_io as fio
    if a.repeat < 1:
        print("repeat must be positive", file=sys.stderr)
        return EXIT_USAGE
    table = np.zeros((len(a.sizes), 3))
    ctx = api.context()
    for i, n in enumerate(a.sizes):
        g = [torch.ones((n, n), dtype=torch.float64, device="cuda"),
             torch.zeros((n, n), dtype=torch.float64, device="cuda"),
             torch.ones((n, n), dtype=torch.float64, device="cuda")]
        b = [torch.zeros((n, n), dtype=torch.float64, device="cuda") for _ in range(2)]
        src = torch.zeros((n, n), dtype=torch.uint8, device="cuda")
        src[n // 2, n // 2] = 1
        max_iters = api.jacobi_iteration_budget(n, n) if a.solver == "jacobi" else 50
        fn = api.solve_jacobi if a.solver == "jacobi" else api.solve
        times, iters = [], 0
        for _ in range(a.repeat):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, rep = fn(*g, *b, src, 1.0 / n, max_iters=max_iters, ctx=ctx)
            torch.cuda.synchronize()
            times.append((time.perf_counter() - t0) * 1e3)
            iters = rep.iterations
        times.sort()
        med = times[len(times) // 2]
        table[i] = (n, iters, med)
        print(f"size={n} iters={iters} median_ms={fio._to_chars(med)}")
    fio.export_csv(table, a.out)
    return EXIT_OK


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="python -m paper_2603_00035_b200",
                                description="Randers eikonal solver (B200 hot path)")
    sub = p.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="forward arrival-time solve")
    s.add_argument("--metric", required=True)
    s.add_argument("--drift", required=True)
    s.add_argument("--sources", required=True)
    s.add_argument("--h", type=float, default=1.0)
    s.add_argument("--out", required=True)
    s.add_argument("--tol", type=float, default=1e-6)
    s.add_argument("--max-iters", type=int, default=None)
    s.add_argument("--solver", choices=["sweep", "jacobi"], default="sweep")
    bch = sub.add_parser("bench", help="solver timing")
    bch.add_argument("--sizes", type=lambda v: [int(x) for x in v.split(",")], default=[50, 100, 200, 400])
    bch.add_argument("--solver", choices=["sweep", "jacobi"], default="sweep")
    bch.add_argument("--repeat", type=int, default=3)
    bch.add_argument("--out", required=True)
    try:
        a = p.parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code else EXIT_OK
    from . import api
    try:
        return _cmd_solve(a) if a.cmd == "solve" else _cmd_bench(a)
    except api.NotConverged as e:
        print(str(e), file=sys.stderr)
        return EXIT_NUMERICAL
    except api.Error as e:
        print(str(e), file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
