"""Projection VJP: the backward through project_spd /
project_drift that the reference lacks.  The numpy restatement in
oracle/pyoracle.py is pinned by central finite differences of the oracle's
own forward projections (CPU); the device VJP (rfk_project_*_vjp through the
C ABI) must match it to rounding (GPU)."""
import numpy as np
import pytest

from oracle import pyoracle as po

EPS, LMAX, TAU, CAP = 0.05, 4.0, 0.6, 1.5


def _inputs(n, seed):
    """Metrics whose eigenvalues straddle [EPS, LMAX] and drifts straddling
    both caps, with nodes near a kink (FD-unsafe) dropped by the caller."""
    rng = np.random.default_rng(seed)
    th = rng.uniform(0, np.pi, n)
    l1 = rng.uniform(-0.5, 6.0, n)
    l2 = rng.uniform(0.01, 3.0, n)
    c, s = np.cos(th), np.sin(th)
    g11 = l1 * c * c + l2 * s * s
    g12 = (l1 - l2) * c * s
    g22 = l1 * s * s + l2 * c * c
    r = rng.uniform(0.0, 2.5, n)
    ph = rng.uniform(0, 2 * np.pi, n)
    return g11, g12, g22, r * np.cos(ph), r * np.sin(ph)


def _kink_free(g11, g12, g22, b1, b2, margin=1e-3):
    hi, lo, _, _ = po._eig_frame(g11, g12, g22)
    ok = (np.abs(hi - EPS) > margin) & (np.abs(lo - EPS) > margin) & (np.abs(hi - LMAX) > margin)
    ok &= (np.abs(lo - LMAX) > margin) & (np.abs(hi - lo) > margin)
    p11, p12, p22 = po.project_spd_forward_np(g11, g12, g22, EPS, LMAX)
    en = np.hypot(b1, b2)
    ok &= np.abs(en - CAP) > margin
    f = np.where(en > CAP, CAP / np.maximum(en, 1e-300), 1.0)
    x, y = b1 * f, b2 * f
    det = p11 * p22 - p12 * p12
    gn = np.sqrt((x * x * p22 - 2 * x * y * p12 + y * y * p11) / det)
    ok &= np.abs(gn - TAU) > margin
    return ok


def _joint_forward(oracle, g11, g12, g22, b1, b2):
    p11, p12, p22 = oracle.project_spd(g11, g12, g22, EPS, LMAX)
    x, y = oracle.project_drift(b1, b2, p11, p12, p22, TAU, CAP)
    return np.stack([p11, p12, p22, x, y])


def test_spd_forward_restatement_matches_oracle(oracle):
    g = _inputs(4000, 1)
    want = oracle.project_spd(g[0], g[1], g[2], EPS, LMAX)
    got = po.project_spd_forward_np(g[0], g[1], g[2], EPS, LMAX)
    for a, b in zip(got, want):
        np.testing.assert_allclose(a, b, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("seed", [3, 4])
def test_joint_vjp_reference_pinned_by_central_fd(oracle, seed):
    g = np.stack(_inputs(3000, seed))
    keep = _kink_free(*g)
    g = g[:, keep]
    rng = np.random.default_rng(seed + 100)
    cot = rng.normal(size=g.shape)
    vjp = np.stack(po.project_joint_vjp_np(*g, *cot, EPS, LMAX, TAU, CAP))
    h = 1e-6
    for j in range(5):  # nodewise map: one central difference per input channel
        gp, gm = g.copy(), g.copy()
        gp[j] += h
        gm[j] -= h
        fd = ((_joint_forward(oracle, *gp) - _joint_forward(oracle, *gm)) / (2 * h) * cot).sum(axis=0)
        np.testing.assert_allclose(vjp[j], fd, rtol=1e-5, atol=1e-6, err_msg=f"channel {j}")


def test_drift_vjp_metric_cotangent_matches_fd(oracle):
    g11, g12, g22, b1, b2 = _inputs(3000, 9)
    p = po.project_spd_forward_np(g11, g12, g22, EPS, LMAX)  # a feasible metric
    keep = _kink_free(g11, g12, g22, b1, b2)
    p = [x[keep] for x in p]
    b1, b2 = b1[keep], b2[keep]
    rng = np.random.default_rng(5)
    dx, dy = rng.normal(size=(2, b1.size))
    got = po.project_drift_vjp_np(b1, b2, *p, dx, dy, TAU, CAP)
    h = 1e-6
    for j in range(3):
        pp, pm = [x.copy() for x in p], [x.copy() for x in p]
        pp[j] += h
        pm[j] -= h
        xp, yp = oracle.project_drift(b1, b2, *pp, TAU, CAP)
        xm, ym = oracle.project_drift(b1, b2, *pm, TAU, CAP)
        fd = ((xp - xm) * dx + (yp - ym) * dy) / (2 * h)
        np.testing.assert_allclose(got[2 + j], fd, rtol=1e-5, atol=1e-6)


@pytest.mark.gpu
def test_device_joint_vjp_matches_reference():
    import paper_2603_00035_b200 as rfk

    g = np.stack(_inputs(20000, 11))
    rng = np.random.default_rng(12)
    cot = rng.normal(size=g.shape)
    got = np.stack(rfk.project_vjp(*g, *cot, EPS, LMAX, TAU, CAP))
    want = np.stack(po.project_joint_vjp_np(*g, *cot, EPS, LMAX, TAU, CAP))
    # device atan2/sincos vs glibc at clamped nodes: agreement to rounding
    np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-12)


@pytest.mark.gpu
def test_device_spd_and_drift_vjp_match_reference():
    import paper_2603_00035_b200 as rfk

    g11, g12, g22, b1, b2 = _inputs(20000, 13)
    rng = np.random.default_rng(14)
    d = rng.normal(size=(5, g11.size))
    got = rfk.project_spd_vjp(g11, g12, g22, d[0], d[1], d[2], EPS, LMAX)
    want = po.project_spd_vjp_np(g11, g12, g22, d[0], d[1], d[2], EPS, LMAX)
    for a, b in zip(got, want):
        np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-12)
    p = po.project_spd_forward_np(g11, g12, g22, EPS, LMAX)
    got = rfk.project_drift_vjp(b1, b2, *p, d[3], d[4], TAU, CAP)
    want = po.project_drift_vjp_np(b1, b2, *p, d[3], d[4], TAU, CAP)
    for a, b in zip(got, want):
        np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-12)
    # DriftOnly parameterization: no metric cotangent
    got2 = rfk.project_drift_vjp(b1, b2, *p, d[3], d[4], TAU, CAP, metric_grad=False)
    np.testing.assert_array_equal(got2[0], got[0])


@pytest.mark.gpu
def test_device_vjp_device_memory_and_validation():
    import torch

    import paper_2603_00035_b200 as rfk

    g = [torch.tensor(x, device="cuda") for x in _inputs(5000, 15)]
    cot = [torch.randn(5000, dtype=torch.float64, device="cuda") for _ in range(5)]
    got = rfk.project_vjp(*g, *cot, EPS, LMAX, TAU, CAP)
    want = po.project_joint_vjp_np(*(x.cpu().numpy() for x in g), *(x.cpu().numpy() for x in cot),
                                   EPS, LMAX, TAU, CAP)
    for a, b in zip(got, want):
        np.testing.assert_allclose(a.cpu().numpy(), b, rtol=1e-10, atol=1e-12)
    with pytest.raises(rfk.InvalidArgument):
        rfk.project_vjp(*g, *cot, 1.0, 0.5, TAU, CAP)
    with pytest.raises(rfk.InvalidArgument):
        rfk.project_vjp(*g, *cot, EPS, LMAX, 1.5, CAP)
