"""Build librfk.so in-tree for sm_100a (nvcc; no JIT cache, so the .so
travels with the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["rfk_solve.cu", "rfk_sweep.cu", "rfk_sweep_f32.cu", "rfk_backward.cu", "rfk_project.cu", "rfk_inverse.cu", "rfk_capi.cu", "rfk_capi_inverse.cu"]
OUT = os.path.join(HERE, "librfk.so")

# --fmad=false: no FMA contraction (bit parity with the reference's non-FMA
# x86-64 build); fp64 '/' and sqrt are IEEE by default.
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(HERE, "..", "include", "rfk.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


# Diagnostic variant built alongside: the sweep with its shared-memory ring
# protocol checks (RFK_SWEEP_CHECKED, rfk_sweep.cu), loaded only through
# RFK_LIBRARY by scripts/check_protocols.py / tests/test_protocol_checker_gpu.py.
CHECKED_OUT = os.path.join(HERE, "librfk_chk.so")


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return OUT
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    cmd = [nvcc()] + NVCC_FLAGS + ["-o", OUT + ".tmp"] + srcs
    chk = [nvcc()] + NVCC_FLAGS + ["-DRFK_SWEEP_CHECKED=1", "-o", CHECKED_OUT + ".tmp"] + srcs
    if verbose:
        cmd += ["-Xptxas", "-v"]
        print(" ".join(cmd), file=sys.stderr)
    procs = [subprocess.Popen(c) for c in (cmd, chk)]
    for p, c in zip(procs, (cmd, chk)):
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, c)
    os.replace(OUT + ".tmp", OUT)
    os.replace(CHECKED_OUT + ".tmp", CHECKED_OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
