"""bench.py keeps the driver's JSON contract (small sizes, one GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_bench_c3_line_keys():
    line = _bench("--n", "256", "--steps", "2", "--warmup", "3", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in line, k
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert line["config"]["node_updates_per_step"] > 0


@pytest.mark.gpu
def test_bench_c4_batch_line():
    line = _bench("--workload", "c4", "--n", "128", "--scenes", "3", "--chunk", "2", "--steps", "1", "--warmup", "3")
    assert line["config"]["scenes"] == 3 and line["config"]["grid"] == "128x128"
    assert line["value"] > 0 and line["gpu_launches"] > 0


@pytest.mark.gpu
def test_bench_c5_training_line():
    line = _bench("--workload", "c5", "--n", "64", "--scenes", "3", "--chunk", "2", "--steps", "1", "--warmup", "3")
    assert line["config"]["samples"] == 3 and line["config"]["grid"] == "64x64"
    assert line["value"] > 0 and line["gpu_launches"] > 0 and line["config"]["node_updates_per_step"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["c3", "c4"])
def test_bench_under_torchrun_one_rank(workload):
    """The driver's multi-GPU launch (torch.distributed.run, NCCL, rank env)
    at one rank: same JSON line, n_gpus from WORLD_SIZE."""
    extra = ["--no-cpu-baseline"] if workload == "c3" else ["--scenes", "2", "--chunk", "2"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", "29613" if workload == "c3" else "29614",
           os.path.join(ROOT, "bench.py"), "--gpus", "1", "--workload", workload, "--grid", "256",
           "--steps", "1", "--warmup", "3", *extra]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["gpu_launches"] > 0


@pytest.mark.gpu
def test_reference_arm_under_torchrun_one_rank():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", "29615", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "1", "--steps", "1", "--warmup", "3"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0


def test_reference_arm_line_on_cpu():
    """The reference arm needs no GPU: the reference library (oracle/_ref) on
    row strips of the C3 fields, one per host thread (small grid here)."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libranders_ref.so")):
        pytest.skip("oracle/_ref not built")
    line = _bench("--impl", "reference", "--n", "256", "--steps", "2", "--warmup", "1")
    assert line["impl"] == "reference" and line["value"] > 0 and line["steps"] == 2 and line["warmup"] == 1
    for k in ("metric", "unit", "ms_per_step", "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["config"]["grid"] == "256x256"
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
