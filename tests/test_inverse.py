"""The recovery loop around the solver: TV / Tikhonov
regularizers (feasibility.cpp:106-196), clip_global_norm, adam_step, gd_step,
relative_error, objective_and_grad with its regularizers, recover and
generate_observations (inversion.cpp) — the device versions against the
reference library itself (oracle/_ref), bit for bit where the reference is
deterministic (exact_sum replays its sequential sums)."""
import numpy as np
import pytest

from conftest import assert_bitwise


def _fields(reflib, n=20, m=18, seed=5, drift=0.2):
    return reflib.random_feasible_fields(max(n, m), seed, drift)[:, :n, :m].copy()


def _sources(n, m, K=2):
    src = np.zeros((K, n, m), np.uint8)
    src[0, n // 2, m // 3] = 1
    if K > 1:
        src[1, n // 4, (2 * m) // 3] = 1
    return src


# ---- CPU: the reference-side bindings (pins the checker) ---------------------------
def test_reference_bindings_run(reflib):
    F = _fields(reflib)
    v, g = reflib.tv_value_grad([F[0], F[1], F[2]], 0)
    assert v > 0 and len(g) == 3
    # spatially constant fields score exactly zero (feasibility.hpp:50-52)
    v0, g0 = reflib.tv_value_grad([np.full((5, 6), 2.0)], 0)
    assert v0 == 0.0 and not np.any(g0[0])
    src = _sources(20, 18)
    obs, val = reflib.generate_observations(F, src, 1.0 / 20, 0.3, 0.0, 7)
    assert obs.shape == (2, 20, 18) and obs.sum() > 0
    from paper_2603_00035_b200.inverse import InverseConfig
    r = reflib.recover(src, obs, val, 1.0 / 20, InverseConfig(iters=3).to_reference())
    assert r["iterations"] == 3 and np.all(np.isfinite(r["loss_history"]))


def test_inverse_config_defaults_match_reference_header():
    from paper_2603_00035_b200.inverse import InverseConfig
    c = InverseConfig()
    # inversion.hpp:15-37, feasibility.hpp:9-13
    assert (c.step_g, c.step_b, c.beta1, c.beta2, c.adam_eps, c.grad_clip_norm) == (1e-2, 5e-3, 0.9, 0.999, 1e-8, 1.0)
    assert (c.iters, c.plateau_window, c.plateau_factor, c.unreached_penalty_cap) == (300, 25, 0.5, 1e4)
    assert (c.eps_min, c.lambda_max, c.tau, c.euclid_cap) == (1e-3, 1e3, 0.95, 10.0)


# ---- GPU parity -------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("nch,variant", [(1, 0), (2, 2), (3, 0), (3, 2)])
def test_tv_bitwise(reflib, nch, variant):
    from paper_2603_00035_b200 import inverse as inv
    F = _fields(reflib, 23, 17)
    ch = [F[k] for k in range(nch)] if variant != 2 or nch != 2 else [F[3], F[4]]
    v, g = reflib.tv_value_grad(ch, variant)
    gv, gg = inv.tv_value_grad(ch, inv.TvVariant(variant), exact=True)
    assert gv == v
    assert_bitwise(np.stack(gg), np.stack(g))
    tv, _ = inv.tv_value_grad(ch, inv.TvVariant(variant), exact=False)
    assert abs(tv - v) <= 1e-12 * abs(v)


@pytest.mark.gpu
def test_tv_log_euclidean(reflib):
    from paper_2603_00035_b200 import inverse as inv
    F = _fields(reflib, 16, 15)
    v, g = reflib.tv_value_grad([F[0], F[1], F[2]], 1)
    gv, gg = inv.tv_value_grad([F[0], F[1], F[2]], inv.TvVariant.LogEuclidean, exact=True)
    # device atan2/cos/sin/log vs glibc: ulp-level differences only
    assert abs(gv - v) <= 1e-12 * abs(v)
    np.testing.assert_allclose(np.stack(gg), np.stack(g), rtol=1e-9, atol=1e-12)


@pytest.mark.gpu
def test_tv_errors(reflib):
    from paper_2603_00035_b200 import api, inverse as inv
    F = _fields(reflib, 8, 8)
    with pytest.raises(api.InvalidArgument):
        inv.tv_value_grad([F[0], F[1]], inv.TvVariant.LogEuclidean)
    with pytest.raises(api.InvalidArgument):
        inv.tv_value_grad([F[0]], inv.TvVariant.Frobenius, eps_tv=0.0)
    bad = [F[0].copy(), F[1].copy(), F[2].copy()]
    bad[0][3, 3] = -1.0  # not SPD
    with pytest.raises(api.NonSpdInput):
        inv.tv_value_grad(bad, inv.TvVariant.LogEuclidean)


@pytest.mark.gpu
def test_tikhonov_clip_relative_error_bitwise(reflib):
    from paper_2603_00035_b200 import inverse as inv
    F = _fields(reflib, 19, 21)
    planes = [F[k] for k in range(5)]
    v, g = reflib.tikhonov_value_grad(planes, 0.37)
    gv, gg = inv.tikhonov_value_grad(planes, 0.37, exact=True)
    assert gv == v
    assert_bitwise(np.stack(gg), np.stack(g))
    for max_norm in (1.0, 1e6):  # clipped / untouched
        want_norm, want = reflib.clip_global_norm(planes, max_norm)
        got = [p.copy() for p in planes]
        norm = inv.clip_global_norm(got, max_norm, exact=True)
        assert norm == want_norm
        assert_bitwise(np.stack(got), np.stack(want))
    truth = [p + 0.01 * np.sin(p) for p in planes]
    assert inv.relative_error(planes, truth, exact=True) == reflib.relative_error(planes, truth)


@pytest.mark.gpu
def test_adam_and_gd_steps_bitwise(reflib):
    from paper_2603_00035_b200 import inverse as inv
    F = _fields(reflib, 15, 14)
    params = [F[0].copy(), F[2].copy()]
    rng = np.random.default_rng(1)
    st = inv.AdamState()
    P, M, V, t = [p.copy() for p in params], None, None, 0
    for step in range(4):
        grads = [rng.standard_normal(p.shape) * (3.0 if step == 0 else 0.05) for p in params]
        P, M, V, t = reflib.adam_step(P, M, V, t, grads, [0.01, 0.02])
        inv.adam_step(st, params, grads, [0.01, 0.02], exact=True)
        assert st.t == t
        assert_bitwise(np.stack(params), np.stack(P))
        assert_bitwise(np.stack(st.m), np.stack(M))
        assert_bitwise(np.stack(st.v), np.stack(V))
    gp = [F[3].copy(), F[4].copy()]
    grads = [rng.standard_normal(p.shape) for p in gp]
    want = reflib.gd_step(gp, grads, [0.1, 0.2])
    inv.gd_step(gp, grads, [0.1, 0.2], exact=True)
    assert_bitwise(np.stack(gp), np.stack(want))


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_objective_with_regularizers(reflib, variant):
    from paper_2603_00035_b200 import inverse as inv
    n, m = 22, 20
    F = _fields(reflib, n, m)
    src = _sources(n, m)
    obs, val = reflib.generate_observations(F, src, 1.0 / n, 0.3, 0.0, 11)
    G = _fields(reflib, n, m, seed=9, drift=0.1)  # evaluate away from the truth
    cfg = inv.InverseConfig(lambda_g=0.05, lambda_b=0.02, tv_variant=inv.TvVariant(variant), exact_sum=True)
    l, dl, rl, un, grads = reflib.objective(list(G), src, obs, val, 1.0 / n, cfg.to_reference())
    o = inv.objective(*G, src, obs, val, 1.0 / n, cfg)
    assert o.data_loss == dl and o.unreached_observed == un
    if variant == 0:
        assert o.reg_loss == rl and o.loss == l
        assert_bitwise(o.grad, np.stack(grads))
    else:
        assert abs(o.reg_loss - rl) <= 1e-12 * abs(rl)
        np.testing.assert_allclose(o.grad, np.stack(grads), rtol=1e-9, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("param,opt", [(0, 0), (1, 0), (2, 0), (3, 0), (4, 0), (4, 1)])
def test_recover_bitwise(reflib, param, opt):
    """The whole projected loop against randers::recover: fields, loss and error
    histories bit for bit with exact sums."""
    from paper_2603_00035_b200 import inverse as inv
    n, m = 20, 18
    truth = _fields(reflib, n, m)
    src = _sources(n, m)
    obs, val = reflib.generate_observations(truth, src, 1.0 / n, 0.3, 0.0, 3)
    cfg = inv.InverseConfig(param=inv.Parameterization(param), optimizer=inv.OptimizerKind(opt), iters=6,
                            lambda_g=0.01 if param != 3 else 0.0, lambda_b=0.01 if param >= 3 else 0.0,
                            plateau_window=2, exact_sum=True)
    init = [np.ones((n, m)), np.zeros((n, m)), np.ones((n, m)), np.zeros((n, m)), np.zeros((n, m))]
    if param == 3:  # drift-only recovers b on the true metric
        init[:3] = [truth[0], truth[1], truth[2]]
    tm = (truth[0], truth[1], truth[2]) if param != 3 else None
    td = (truth[3], truth[4]) if param >= 3 else None
    want = reflib.recover(src, obs, val, 1.0 / n, cfg.to_reference(), init=init, truth_metric=tm, truth_drift=td)
    got = inv.recover(src, obs, val, 1.0 / n, cfg, init_metric=tuple(init[:3]), init_drift=tuple(init[3:]),
                      truth_metric=tm, truth_drift=td)
    assert got.iterations == want["iterations"] == 6
    assert_bitwise(got.loss_history, want["loss_history"])
    assert_bitwise(got.error_history, want["error_history"])
    assert got.final_error == want["final_error"]
    assert got.unreached_observed_total == want["unreached_observed_total"]
    assert_bitwise(np.stack(got.metric + got.drift), np.stack(want["fields"]))
    if param == 0:
        assert_bitwise(got.iso_g, want["iso_g"])


@pytest.mark.gpu
def test_recover_default_init_and_device_memory(reflib):
    import torch

    from paper_2603_00035_b200 import inverse as inv
    n, m = 18, 18
    truth = _fields(reflib, n, m)
    src = _sources(n, m, K=1)
    obs, val = reflib.generate_observations(truth, src, 1.0 / n, 0.4, 0.0, 5)
    cfg = inv.InverseConfig(param=inv.Parameterization.Full, iters=4, exact_sum=True)
    want = reflib.recover(src, obs, val, 1.0 / n, cfg.to_reference())
    dev = [torch.tensor(x, device="cuda") for x in (src, obs, val)]
    got = inv.recover(*dev, 1.0 / n, cfg)
    assert_bitwise(got.loss_history, want["loss_history"])
    assert_bitwise(torch.stack(got.metric + got.drift).cpu().numpy(), np.stack(want["fields"]))
    assert got.final_error == -1.0


@pytest.mark.gpu
@pytest.mark.parametrize("noise", [0.0, 0.05])
def test_generate_observations_bitwise(reflib, noise):
    from paper_2603_00035_b200 import inverse as inv
    n, m = 24, 21
    F = _fields(reflib, n, m)
    src = _sources(n, m)
    want_obs, want_val = reflib.generate_observations(F, src, 1.0 / n, 0.25, noise, 42)
    obs, val = inv.generate_observations(*F, src, 1.0 / n, 0.25, noise, 42)
    assert np.array_equal(obs, want_obs)
    assert_bitwise(val, want_val)


@pytest.mark.gpu
def test_recover_errors(reflib):
    from paper_2603_00035_b200 import api, inverse as inv
    n = 10
    src = _sources(n, n, K=1)
    obs = np.zeros_like(src)
    val = np.zeros((1, n, n))
    with pytest.raises(api.InvalidArgument):
        inv.recover(src, obs, val, 0.1, inv.InverseConfig(step_g=0.0))
    with pytest.raises(api.InvalidArgument):
        inv.recover(src, obs, val, 0.1, inv.InverseConfig(iters=0))
    with pytest.raises(api.ZeroDimension):
        inv.recover(src[:, :2, :], obs[:, :2, :], val[:, :2, :], 0.1, inv.InverseConfig(iters=1))
    with pytest.raises(api.InvalidArgument):  # truth metric missing for a metric mode
        inv.recover(src, obs, val, 0.1, inv.InverseConfig(iters=1), truth_drift=(val[0], val[0]))


@pytest.mark.gpu
def test_multi_source_recover_bitwise(reflib):
    from paper_2603_00035_b200 import inverse as inv
    cfg = inv.InverseConfig(iters=5, lambda_g=1e-3, exact_sum=True)
    want = reflib.multi_source_recover([1, 3, 2], 0.07, cfg.to_reference(), 24, 42)
    got = inv.multi_source_recover([1, 3, 2], 0.07, cfg, 24, 42)
    assert [(r.k, r.total_observations, r.error) for r in got] == want
