"""Synthetic workloads of BASELINE.json's configs.

Two generators:

* ``host_fields`` (the bench and the full-size parity goldens): a
  deterministic host recipe built only from integer hashing, IEEE +, *, /
  and sqrt (no transcendental functions, no reductions whose order depends
  on the CPU's SIMD width), so the same seed gives the same bits on every
  x86-64 host.  The oracle's golden dumps at 1024^2 / 2048^2 / 4096^2
  (tests/golden/gen_large.py) are computed on exactly these inputs, and the
  GPU tests regenerate them on the box and check an input hash first.
* ``randers_fields`` (older tests, batch stress): generated on the device
  with torch's RNG.

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


# ---- deterministic host generator -------------------------------------------
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def _splitmix64(ctr):
    z = ctr * _GOLD
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def host_uniform(n: int, stream: int):
    """n uniforms in [0, 1) (53-bit), counter-based: value i of stream s is
    splitmix64(s * 2^40 + i + 1) >> 11, scaled by 2^-53."""
    ctr = np.arange(n, dtype=np.uint64) + ((np.uint64(stream) << np.uint64(40)) + np.uint64(1))
    return (_splitmix64(ctr) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def _seq_sum(x):
    # sequential (cumulative) sum: its order does not depend on the CPU
    return float(np.cumsum(x, dtype=np.float64)[-1])


def _box_blur_host(x, radius: int, axis: int):
    """Box filter of width 2r+1 along `axis`, edges renormalised by the number
    of in-range terms: s_i = C[min(i+r+1, n)] - C[max(i-r, 0)] over the
    exclusive prefix sums C (sequential, so host-independent)."""
    x = np.moveaxis(x, axis, -1)
    n = x.shape[-1]
    c = np.empty(x.shape[:-1] + (n + 1,), np.float64)
    c[..., 0] = 0.0
    np.cumsum(x, axis=-1, out=c[..., 1:])
    r = radius
    s = np.empty_like(x)
    # interior i in [r, n-r-1]: C[i+r+1] - C[i-r]
    if n > 2 * r:
        s[..., r:n - r] = c[..., 2 * r + 1:] - c[..., :n - 2 * r]
        edges = list(range(r)) + list(range(n - r, n))
    else:
        edges = range(n)
    for i in edges:
        s[..., i] = c[..., min(i + r + 1, n)] - c[..., max(i - r, 0)]
    cnt = (np.minimum(np.arange(n) + r + 1, n) - np.maximum(np.arange(n) - r, 0)).astype(np.float64)
    s /= cnt
    return np.ascontiguousarray(np.moveaxis(s, -1, axis))


def host_noise(rows: int, cols: int, radius: int, stream: int):
    """Unit-variance correlated noise: triangular white noise (u1 + u2 - 1)
    * sqrt(6), two separable radius-`radius` box blurs with edge
    renormalisation (the recipe of correlated_noise, src/oracle.cpp:496-542,
    without libstdc++'s normal_distribution)."""
    u = host_uniform(2 * rows * cols, stream).reshape(2, rows, cols)
    f = (u[0] + u[1] - 1.0) * np.sqrt(6.0)
    del u
    for _ in range(2):
        f = _box_blur_host(f, radius, 1)
        f = _box_blur_host(f, radius, 0)
    n = float(rows * cols)
    f = f - _seq_sum(f) / n
    sd = np.sqrt(_seq_sum(f * f) / n)
    return f / sd if sd > 0 else f


def host_project_spd(a, b, c, lo: float, hi: float):
    """Eigenvalue clamp of [[a, b], [b, c]] to [lo, hi] without trigonometry
    (spectral projectors; the inputs generator's own projection, not the
    reference's project_spd)."""
    m = 0.5 * (a + c)
    d = 0.5 * (a - c)
    r = np.sqrt(d * d + b * b)
    l1, l2 = m + r, m - r
    ok = (l2 >= lo) & (l1 <= hi)
    c1, c2 = np.clip(l1, lo, hi), np.clip(l2, lo, hi)
    rs = np.where(r > 0, r, 1.0)
    # G = l1 P1 + l2 P2 with P1 = (G - l2 I) / (l1 - l2), P2 = I - P1
    p11 = np.where(r > 0, (a - l2) / (2.0 * rs), 0.5)
    p12 = np.where(r > 0, b / (2.0 * rs), 0.0)
    p22 = np.where(r > 0, (c - l2) / (2.0 * rs), 0.5)
    na = c1 * p11 + c2 * (1.0 - p11)
    nb = (c1 - c2) * p12
    nc = c1 * p22 + c2 * (1.0 - p22)
    return np.where(ok, a, na), np.where(ok, b, nb), np.where(ok, c, nc)


def host_project_drift(b1, b2, g11, g12, g22, tau: float, euclid_cap: float = 10.0):
    """Euclidean pre-clip, then |b|_{G^-1} <= tau (the recipe of
    project_drift, src/feasibility.cpp:51-72)."""
    e = np.sqrt(b1 * b1 + b2 * b2)
    s = np.where(e > euclid_cap, euclid_cap / np.where(e > 0, e, 1.0), 1.0)
    b1, b2 = b1 * s, b2 * s
    det = g11 * g22 - g12 * g12
    nsq = (b1 * b1 * g22 - 2.0 * b1 * b2 * g12 + b2 * b2 * g11) / det
    nrm = np.sqrt(np.maximum(nsq, 0.0))
    s = np.where(nrm > tau, tau / np.where(nrm > 0, nrm, 1.0), 1.0)
    return b1 * s, b2 * s


def host_fields(n: int, seed: int, drift_scale: float = 0.2, cols: int = None):
    """(g11, g12, g22, b1, b2) float64 numpy planes of an n x cols feasible
    field (tests/helpers.hpp:67-90 recipe: g = 1 + 0.35 e, g12 = 0.2 e,
    b = s e; eigenvalues clamped to [0.5, 2.5], drift capped at
    tau = min(0.95, 2 s)), bit-identical on every host."""
    cols = cols or n
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(5) as ex:  # numpy releases the GIL; results do not depend on the threads
        e = list(ex.map(lambda k: host_noise(n, cols, 3, 5 * seed + k), range(1, 6)))
    g11, g12, g22 = host_project_spd(1.0 + 0.35 * e[0], 0.2 * e[1], 1.0 + 0.35 * e[2], 0.5, 2.5)
    if drift_scale > 0:
        b1, b2 = host_project_drift(drift_scale * e[3], drift_scale * e[4], g11, g12, g22,
                                    min(0.95, 2.0 * drift_scale))
    else:
        b1 = np.zeros_like(g11)
        b2 = np.zeros_like(g11)
    return tuple(np.ascontiguousarray(x) for x in (g11, g12, g22, b1, b2))


def host_point_source(rows: int, cols: int):
    s = np.zeros((rows, cols), np.uint8)
    s[rows // 2, cols // 2] = 1
    return s


def host_observation_mask(src, frac: float = 0.3, stream: int = 2024):
    """`frac` observed mask, never on a source (acceptance_main.cpp:57-68 recipe)."""
    u = host_uniform(src.size, stream).reshape(src.shape)
    return ((u < frac) & (src == 0)).astype(np.uint8)


def fields_digest(*planes) -> str:
    """sha256 over the raw bytes of the given arrays (inputs / outputs of the
    full-size parity goldens)."""
    import hashlib

    h = hashlib.sha256()
    for p in planes:
        a = np.ascontiguousarray(p)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


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


__all__ = ["correlated_noise", "randers_fields", "host_fields", "host_point_source", "host_observation_mask",
           "host_noise", "host_uniform", "fields_digest", "point_source", "observation_mask", "node_updates",
           "numpy_fields", "np"]
