"""Synthetic workloads of BASELINE.json's configs, generated
on the device.

The reference generates fields with libstdc++'s std::normal_distribution
(correlated_noise, src/oracle.cpp:496-542), which cannot be reproduced off
that library; the recipe is kept (two separable radius-3 box-blur passes with
edge renormalisation, unit-variance normalisation, g = 1 + 0.35 e, g12 =
0.2 e, b = s e, projected with eps 0.5 / lambda_max 2.5 / tau = min(0.95, 2s)
as in tests/helpers.hpp:67-90) with torch's RNG.  Parity never depends on
this: tests compare the CUDA path and the oracle on the same inputs.
"""
from __future__ import annotations

import numpy as np


def _box_blur_1d(x, radius: int, dim: int):
    import torch

    n = x.shape[dim]
    pad = [0, 0, 0, 0]
    # cumulative-sum box filter with per-position counts (edges renormalised)
    c = torch.cumsum(x, dim=dim)
    zero_shape = list(x.shape)
    zero_shape[dim] = 1
    c = torch.cat([torch.zeros(zero_shape, dtype=x.dtype, device=x.device), c], dim=dim)
    idx = torch.arange(n, device=x.device)
    hi = torch.clamp(idx + radius + 1, max=n)
    lo = torch.clamp(idx - radius, min=0)
    cnt = (hi - lo).to(x.dtype)
    s = c.index_select(dim, hi) - c.index_select(dim, lo)
    shape = [1, 1]
    shape[dim] = n
    del pad
    return s / cnt.view(shape)


def correlated_noise(rows: int, cols: int, radius: int, seed: int, device="cuda"):
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    f = torch.randn((rows, cols), generator=g, dtype=torch.float64, device=device)
    for _ in range(2):
        f = _box_blur_1d(f, radius, 1)
        f = _box_blur_1d(f, radius, 0)
    f = f - f.mean()
    sd = torch.sqrt((f * f).mean())
    return f / sd if float(sd) > 0 else f


def randers_fields(n: int, seed: int, drift_scale: float = 0.2, device="cuda", cols: int = None):
    """(g11, g12, g22, b1, b2) device tensors of an n x cols feasible field."""
    import torch

    from . import api

    cols = cols or n
    e = [correlated_noise(n, cols, 3, seed * 5 + k, device) for k in range(1, 6)]
    g11 = 1.0 + 0.35 * e[0]
    g12 = 0.2 * e[1]
    g22 = 1.0 + 0.35 * e[2]
    g11, g12, g22 = api.project_spd(g11, g12, g22, 0.5, 2.5)
    if drift_scale > 0:
        b1, b2 = api.project_drift(drift_scale * e[3], drift_scale * e[4], g11, g12, g22,
                                   min(0.95, 2.0 * drift_scale))
    else:
        b1 = torch.zeros_like(g11)
        b2 = torch.zeros_like(g11)
    return g11, g12, g22, b1, b2


def point_source(rows: int, cols: int, device="cuda"):
    import torch

    s = torch.zeros((rows, cols), dtype=torch.uint8, device=device)
    s[rows // 2, cols // 2] = 1
    return s


def observation_mask(src, frac: float = 0.3, seed: int = 2024):
    """30% observed mask, no sources (tests/acceptance_main.cpp:57-68 recipe)."""
    import torch

    g = torch.Generator(device=src.device)
    g.manual_seed(seed)
    u = torch.rand(src.shape, generator=g, dtype=torch.float64, device=src.device)
    return ((u < frac) & (src == 0)).to(torch.uint8)


def node_updates(iterations: int, n_nodes: int, n_sources: int, n_records: int) -> int:
    """Algorithmic work unit of SURVEY.md §8d: W = 4 K (N^2 - |S|) + n_records."""
    return 4 * int(iterations) * (int(n_nodes) - int(n_sources)) + int(n_records)


def numpy_fields(n: int, seed: int, drift_scale: float = 0.2):
    """Host copy of randers_fields for CPU-side baselines."""
    return [x.cpu().numpy() for x in randers_fields(n, seed, drift_scale)]


__all__ = ["correlated_noise", "randers_fields", "point_source", "observation_mask", "node_updates",
           "numpy_fields", "np"]
