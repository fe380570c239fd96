// rfk_capi_inverse.cu — C ABI of the recovery loop around the solver
// (include/rfk.h, "regularizers", "optimizer steps", "the recovery loop"):
// tv_value_grad / tikhonov_value_grad (feasibility.cpp:106-196),
// objective_and_grad with its TV terms, clip_global_norm, adam_step, gd_step,
// relative_error, recover and generate_observations (inversion.cpp).
//
// The parameters, Adam moments and gradients of `recover` stay on the device
// for the whole loop; the host only sees one objective value per iteration
// (the plateau schedule and the divergence test branch on it, as in the
// reference).  Host-side scalar arithmetic (bias corrections, the clip factor,
// loss bookkeeping) is the reference's own expressions on the same doubles.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "rfk_capi_internal.h"

namespace {

using rfk::SumArgs;

double read_scalar(rfk_context* ctx, const double* d) {
    double h = 0.0;
    cuda_check(ctx, cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
    return h;
}

// Sum over planes (see rfk::SumArgs for the modes); exact = node order.
double sum_planes(rfk_context* ctx, int mode, bool exact, int64_t n, int planes, const double* const* x,
                  const double* const* y, double scale, double init) {
    if (planes > 5) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "at most 5 planes");
    SumArgs a{};
    a.n = n;
    a.planes = planes;
    for (int p = 0; p < planes; ++p) {
        a.x[p] = x[p];
        a.y[p] = y ? y[p] : nullptr;
    }
    a.scale = scale;
    a.init = init;
    double* partial = tbuf<double>(ctx, "inv:partial", 1024);
    double* out = tbuf<double>(ctx, "inv:sum", 1);
    launched(ctx, rfk::launch_sum(a, mode, exact, partial, out, ctx->stream), "sum", exact ? 1 : 2);
    return read_scalar(ctx, out);
}

// tv_value_grad on device planes (feasibility.cpp:137-182)
double tv_device(rfk_context* ctx, int R, int C, int nch, rfk_tv_variant variant, double eps,
                 const double* const* ch, double* const* grad, bool exact) {
    if (nch < 1 || nch > 3) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "tv_value_grad: need 1..3 channels");
    if (!(eps > 0.0)) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "tv_value_grad: eps_tv must be positive");
    const int64_t n = static_cast<int64_t>(R) * C;
    rfk::TvArgs a{};
    a.R = R;
    a.C = C;
    a.nch = nch;
    a.w[0] = a.w[1] = a.w[2] = 1.0;
    if (nch == 3 && variant != RFK_TV_DRIFT) a.w[1] = 2.0;  // off-diagonal counts twice (:147)
    a.eps = eps;
    a.term = tbuf<double>(ctx, "tv:term", n);
    if (variant != RFK_TV_LOG_EUCLIDEAN) {
        for (int k = 0; k < nch; ++k) {
            a.ch[k] = ch[k];
            a.grad[k] = grad[k];
        }
        launched(ctx, rfk::launch_tv(a, ctx->stream), "tv");
        const double* t = a.term;
        return sum_planes(ctx, 0, exact, n, 1, &t, nullptr, 0.0, 0.0);
    }
    if (nch != 3) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "tv_value_grad: log-Euclidean variant needs 3 channels");
    double* logs[3] = {tbuf<double>(ctx, "tv:l0", n), tbuf<double>(ctx, "tv:l1", n), tbuf<double>(ctx, "tv:l2", n)};
    double* lgrad[3] = {tbuf<double>(ctx, "tv:lg0", n), tbuf<double>(ctx, "tv:lg1", n),
                        tbuf<double>(ctx, "tv:lg2", n)};
    int* non_spd = tbuf<int>(ctx, "tv:nonspd", 1);
    cuda_check(ctx, cudaMemsetAsync(non_spd, 0, sizeof(int), ctx->stream), "memset");
    launched(ctx, rfk::launch_log_spd(n, ch[0], ch[1], ch[2], logs[0], logs[1], logs[2], non_spd, ctx->stream),
             "log_spd");
    int bad = 0;
    cuda_check(ctx, cudaMemcpyAsync(&bad, non_spd, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
    if (bad) fail(ctx, RFK_ERR_NON_SPD_INPUT, "tv_value_grad: log-Euclidean variant needs SPD input");
    for (int k = 0; k < 3; ++k) {
        a.ch[k] = logs[k];
        a.grad[k] = lgrad[k];
    }
    launched(ctx, rfk::launch_tv(a, ctx->stream), "tv");
    const double* t = a.term;
    const double value = sum_planes(ctx, 0, exact, n, 1, &t, nullptr, 0.0, 0.0);
    const double* lg[3] = {lgrad[0], lgrad[1], lgrad[2]};
    double* out[3] = {grad[0], grad[1], grad[2]};
    launched(ctx, rfk::launch_dlog_chain(n, ch[0], ch[1], ch[2], lg, out, ctx->stream), "dlog_chain");
    return value;
}

// clip_global_norm on device planes (inversion.cpp:75-88)
double clip_device(rfk_context* ctx, int64_t n, int np, double* const* g, double max_norm, bool exact) {
    std::vector<const double*> x(g, g + np);
    const double sq = sum_planes(ctx, 1, exact, n, np, x.data(), nullptr, 0.0, 0.0);
    const double norm = std::sqrt(sq);
    if (norm > max_norm && norm > 0.0) {
        const double f = max_norm / norm;
        for (int k = 0; k < np; ++k) launched(ctx, rfk::launch_scale(n, f, g[k], ctx->stream), "scale");
    }
    return norm;
}

// adam_step after the clip (inversion.cpp:90-116); grads are clipped in place
void adam_device(rfk_context* ctx, int64_t n, int np, double* const* p, double* const* m, double* const* v,
                 int64_t& t, double* const* g, const double* steps, double beta1, double beta2, double eps,
                 double clip, bool exact) {
    clip_device(ctx, n, np, g, clip, exact);
    ++t;
    const double bc1 = 1.0 - std::pow(beta1, static_cast<double>(t));
    const double bc2 = 1.0 - std::pow(beta2, static_cast<double>(t));
    for (int k = 0; k < np; ++k)
        launched(ctx, rfk::launch_adam(n, p[k], m[k], v[k], g[k], steps[k], beta1, beta2, bc1, bc2, eps, ctx->stream),
                 "adam");
}

void gd_device(rfk_context* ctx, int64_t n, int np, double* const* p, double* const* g, const double* steps,
               double clip, bool exact) {
    clip_device(ctx, n, np, g, clip, exact);
    for (int k = 0; k < np; ++k) launched(ctx, rfk::launch_gd(n, p[k], g[k], steps[k], ctx->stream), "gd");
}

double relative_error_device(rfk_context* ctx, int64_t n, int np, const double* const* est,
                             const double* const* truth, bool exact) {
    const double num = sum_planes(ctx, 3, exact, n, np, est, truth, 0.0, 0.0);
    const double den = sum_planes(ctx, 1, exact, n, np, truth, nullptr, 0.0, 0.0);
    return den > 0.0 ? std::sqrt(num / den) : std::sqrt(num);
}

void validate_projection_cfg(rfk_context* ctx, const rfk_inverse_config* c) {
    if (!(c->eps_min > 0.0) || !(c->eps_min < c->lambda_max))
        fail(ctx, RFK_ERR_INVALID_ARGUMENT, "ProjectionConfig: need 0 < eps_min < lambda_max");
    if (!(c->tau > 0.0) || !(c->tau < 1.0)) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "ProjectionConfig: need 0 < tau < 1");
}

// objective_and_grad with the regularizers, device pointers (inversion.cpp:25-73)
void objective_device(rfk_context* ctx, const rfk_fields* fd, const rfk_observations* od,
                      const rfk_inverse_config* cfg, rfk_objective_value* out, double* const* grads) {
    rfk_objective_options o{cfg->solve_tol, cfg->solve_max_iters, cfg->unreached_penalty_cap, cfg->exact_sum};
    double dl = 0.0;
    int32_t unr = 0;
    const rfk_status s = rfk_objective_and_grad(ctx, RFK_MEM_DEVICE, fd, od, &o, &dl, &unr, grads[0], grads[1],
                                                grads[2], grads[3], grads[4]);
    if (s != RFK_OK) throw Fail{s};
    const int64_t n = static_cast<int64_t>(fd->rows) * fd->cols;
    const bool exact = cfg->exact_sum != 0;
    double reg = 0.0;
    double* tg[3] = {tbuf<double>(ctx, "reg:g0", n), tbuf<double>(ctx, "reg:g1", n), tbuf<double>(ctx, "reg:g2", n)};
    if (cfg->lambda_g != 0.0) {
        const double* ch[3] = {fd->g11, fd->g12, fd->g22};
        const double v = tv_device(ctx, fd->rows, fd->cols, 3, cfg->tv_variant, 1e-8, ch, tg, exact);
        reg += cfg->lambda_g * v;
        for (int k = 0; k < 3; ++k)
            launched(ctx, rfk::launch_axpy(n, cfg->lambda_g, tg[k], grads[k], ctx->stream), "axpy");
    }
    if (cfg->lambda_b != 0.0) {
        const double* ch[2] = {fd->b1, fd->b2};
        const double v = tv_device(ctx, fd->rows, fd->cols, 2, RFK_TV_DRIFT, 1e-8, ch, tg, exact);
        reg += cfg->lambda_b * v;
        for (int k = 0; k < 2; ++k)
            launched(ctx, rfk::launch_axpy(n, cfg->lambda_b, tg[k], grads[3 + k], ctx->stream), "axpy");
    }
    out->data_loss = dl;
    out->reg_loss = reg;
    out->unreached_observed = unr;
    out->loss = out->data_loss + out->reg_loss;
}


}  // namespace

extern "C" {

RFK_API void rfk_inverse_config_default(rfk_inverse_config* c) {
    if (!c) return;
    c->param = RFK_PARAM_ISOTROPIC;
    c->optimizer = RFK_OPT_ADAM;
    c->step_g = 1e-2;
    c->step_b = 5e-3;
    c->beta1 = 0.9;
    c->beta2 = 0.999;
    c->adam_eps = 1e-8;
    c->grad_clip_norm = 1.0;
    c->lambda_g = 0.0;
    c->lambda_b = 0.0;
    c->tv_variant = RFK_TV_FROBENIUS;
    c->iters = 300;
    c->eps_min = 1e-3;
    c->lambda_max = 1e3;
    c->tau = 0.95;
    c->euclid_cap = 10.0;
    c->solve_tol = 1e-6;
    c->solve_max_iters = 50;
    c->plateau_window = 25;
    c->plateau_factor = 0.5;
    c->unreached_penalty_cap = 1e4;
    c->exact_sum = 0;
}

RFK_API rfk_status rfk_tv_value_grad(rfk_context* ctx, rfk_memory mem, int32_t rows, int32_t cols, int32_t nch,
                                     rfk_tv_variant variant, double eps_tv, const double* const* channels,
                                     double* const* grad, double* value, int32_t exact_sum) {
    return guarded(ctx, [&] {
        if (!channels || !grad || !value) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null argument");
        if (nch < 1 || nch > 3) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "tv_value_grad: need 1..3 channels");
        if (rows < 1 || cols < 1) fail(ctx, RFK_ERR_DIMENSION_MISMATCH, "tv_value_grad: channel shapes");
        const int64_t n = static_cast<int64_t>(rows) * cols;
        Stage st{ctx, mem, {}};
        const double* ch[3] = {nullptr, nullptr, nullptr};
        double* g[3] = {nullptr, nullptr, nullptr};
        for (int k = 0; k < nch; ++k) {
            if (!channels[k] || !grad[k]) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null plane");
            ch[k] = st.in("tv" + std::to_string(k), channels[k], n);
            g[k] = st.out("tvg" + std::to_string(k), grad[k], n);
        }
        *value = tv_device(ctx, rows, cols, nch, variant, eps_tv, ch, g, exact_sum != 0);
        st.finish();
    });
}

RFK_API rfk_status rfk_tikhonov_value_grad(rfk_context* ctx, rfk_memory mem, int64_t n, int32_t nch, double weight,
                                           const double* const* channels, double* const* grad, double* value,
                                           int32_t exact_sum) {
    return guarded(ctx, [&] {
        if (!channels || !grad || !value) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null argument");
        if (nch < 0 || nch > 5) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "tikhonov_value_grad: at most 5 channels");
        Stage st{ctx, mem, {}};
        std::vector<const double*> ch(nch);
        for (int k = 0; k < nch; ++k) {
            ch[k] = st.in("tk" + std::to_string(k), channels[k], n);
            double* g = st.out("tkg" + std::to_string(k), grad[k], n);
            launched(ctx, rfk::launch_weighted_copy(n, weight, ch[k], g, ctx->stream), "tikhonov");
        }
        *value = nch ? sum_planes(ctx, 2, exact_sum != 0, n, nch, ch.data(), nullptr, weight, 0.0) : 0.0;
        st.finish();
    });
}

RFK_API rfk_status rfk_clip_global_norm(rfk_context* ctx, rfk_memory mem, int64_t n, int32_t nplanes,
                                        double* const* grads, double max_norm, double* norm, int32_t exact_sum) {
    return guarded(ctx, [&] {
        if (!grads || nplanes < 0 || nplanes > 5) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "clip_global_norm: 0..5 planes");
        Stage st{ctx, mem, {}};
        std::vector<double*> g(nplanes);
        for (int k = 0; k < nplanes; ++k) g[k] = st.inout("clip" + std::to_string(k), grads[k], n);
        const double v = clip_device(ctx, n, nplanes, g.data(), max_norm, exact_sum != 0);
        if (norm) *norm = v;
        st.finish();
    });
}

RFK_API rfk_status rfk_adam_step(rfk_context* ctx, rfk_memory mem, int64_t n, int32_t nplanes, double* const* params,
                                 double* const* m, double* const* v, int64_t* t, const double* const* grads,
                                 const double* steps, double beta1, double beta2, double adam_eps,
                                 double grad_clip_norm, int32_t exact_sum) {
    return guarded(ctx, [&] {
        if (!params || !m || !v || !t || !grads || !steps || nplanes < 1 || nplanes > 5)
            fail(ctx, RFK_ERR_INVALID_ARGUMENT, "adam_step: bad arguments");
        Stage st{ctx, mem, {}};
        std::vector<double*> p(nplanes), mm(nplanes), vv(nplanes), g(nplanes);
        for (int k = 0; k < nplanes; ++k) {
            const std::string s = std::to_string(k);
            p[k] = st.inout("adp" + s, params[k], n);
            mm[k] = st.inout("adm" + s, m[k], n);
            vv[k] = st.inout("adv" + s, v[k], n);
            // grads are taken by value (inversion.cpp:91): clip a copy
            g[k] = tbuf<double>(ctx, "adg" + s, n);
            cuda_check(ctx,
                       cudaMemcpyAsync(g[k], grads[k], n * sizeof(double),
                                       mem == RFK_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                       ctx->stream),
                       "copy grads");
        }
        adam_device(ctx, n, nplanes, p.data(), mm.data(), vv.data(), *t, g.data(), steps, beta1, beta2, adam_eps,
                    grad_clip_norm, exact_sum != 0);
        st.finish();
    });
}

RFK_API rfk_status rfk_gd_step(rfk_context* ctx, rfk_memory mem, int64_t n, int32_t nplanes, double* const* params,
                               const double* const* grads, const double* steps, double grad_clip_norm,
                               int32_t exact_sum) {
    return guarded(ctx, [&] {
        if (!params || !grads || !steps || nplanes < 1 || nplanes > 5)
            fail(ctx, RFK_ERR_INVALID_ARGUMENT, "gd_step: bad arguments");
        Stage st{ctx, mem, {}};
        std::vector<double*> p(nplanes), g(nplanes);
        for (int k = 0; k < nplanes; ++k) {
            const std::string s = std::to_string(k);
            p[k] = st.inout("gdp" + s, params[k], n);
            g[k] = tbuf<double>(ctx, "gdg" + s, n);
            cuda_check(ctx,
                       cudaMemcpyAsync(g[k], grads[k], n * sizeof(double),
                                       mem == RFK_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                       ctx->stream),
                       "copy grads");
        }
        gd_device(ctx, n, nplanes, p.data(), g.data(), steps, grad_clip_norm, exact_sum != 0);
        st.finish();
    });
}

RFK_API rfk_status rfk_relative_error(rfk_context* ctx, rfk_memory mem, int64_t n, int32_t nplanes,
                                      const double* const* est, const double* const* truth, double* out,
                                      int32_t exact_sum) {
    return guarded(ctx, [&] {
        if (!est || !truth || !out || nplanes < 1 || nplanes > 5)
            fail(ctx, RFK_ERR_INVALID_ARGUMENT, "relative_error: bad arguments");
        Stage st{ctx, mem, {}};
        std::vector<const double*> e(nplanes), t(nplanes);
        for (int k = 0; k < nplanes; ++k) {
            e[k] = st.in("ree" + std::to_string(k), est[k], n);
            t[k] = st.in("ret" + std::to_string(k), truth[k], n);
        }
        *out = relative_error_device(ctx, n, nplanes, e.data(), t.data(), exact_sum != 0);
        st.finish();
    });
}

RFK_API rfk_status rfk_objective(rfk_context* ctx, rfk_memory mem, const rfk_fields* f, const rfk_observations* obs,
                                 const rfk_inverse_config* cfg, rfk_objective_value* out, double* d_g11,
                                 double* d_g12, double* d_g22, double* d_b1, double* d_b2) {
    return guarded(ctx, [&] {
        if (!f || !obs || !cfg || !out) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null argument");
        if (f->batch != 1) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "objective: one parameter set");
        if (obs->count < 1 || !obs->sources || !obs->observed || !obs->values)
            fail(ctx, RFK_ERR_INVALID_ARGUMENT, "objective_and_grad: needs at least one observation set");
        if (!d_g11 || !d_g12 || !d_g22 || !d_b1 || !d_b2) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null output");
        const int64_t n = static_cast<int64_t>(f->rows) * f->cols;
        const size_t nk = static_cast<size_t>(n) * obs->count;
        Stage st{ctx, mem, {}};
        rfk_fields fd = *f;
        fd.g11 = st.in("og11", f->g11, n);
        fd.g12 = st.in("og12", f->g12, n);
        fd.g22 = st.in("og22", f->g22, n);
        fd.b1 = st.in("ob1", f->b1, n);
        fd.b2 = st.in("ob2", f->b2, n);
        rfk_observations od = *obs;
        od.sources = st.in("osrc", obs->sources, nk);
        od.observed = st.in("oobs", obs->observed, nk);
        od.values = st.in("oval", obs->values, nk);
        double* g[5] = {st.out("odg11", d_g11, n), st.out("odg12", d_g12, n), st.out("odg22", d_g22, n),
                        st.out("odb1", d_b1, n), st.out("odb2", d_b2, n)};
        objective_device(ctx, &fd, &od, cfg, out, g);
        st.finish();
    });
}

RFK_API rfk_status rfk_recover(rfk_context* ctx, rfk_memory mem, int32_t rows, int32_t cols, double h,
                               const rfk_observations* obs, const rfk_inverse_config* cfg,
                               const double* const* init_metric, const double* const* init_drift,
                               const double* const* truth_metric, const double* const* truth_drift,
                               rfk_recovery* out) {
    return guarded(ctx, [&] {
        if (!obs || !cfg || !out || !out->loss_history) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null argument");
        // InverseConfig::validate, GridSpec::validate (inversion.hpp:38-42, grid.hpp:61-65)
        if (!(cfg->step_g > 0.0) || !(cfg->step_b > 0.0))
            fail(ctx, RFK_ERR_INVALID_ARGUMENT, "InverseConfig: steps must be positive");
        if (cfg->iters < 1) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "InverseConfig: iters must be >= 1");
        if (rows < 3 || cols < 3) fail(ctx, RFK_ERR_ZERO_DIMENSION, "GridSpec: rows and cols must be at least 3");
        if (!(h > 0.0)) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "GridSpec: h must be positive");
        if (obs->count < 1 || !obs->sources || !obs->observed || !obs->values)
            fail(ctx, RFK_ERR_INVALID_ARGUMENT, "recover: need at least one observation set");
        const int64_t n = static_cast<int64_t>(rows) * cols;
        const size_t nk = static_cast<size_t>(n) * obs->count;
        const bool exact = cfg->exact_sum != 0;
        const cudaMemcpyKind in_kind = mem == RFK_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        Stage st{ctx, mem, {}};
        rfk_observations od = *obs;
        od.sources = st.in("rsrc", obs->sources, nk);
        od.observed = st.in("robs", obs->observed, nk);
        od.values = st.in("rval", obs->values, nk);

        // full fields: initial values g = I, b = 0 unless given (ParamView::make, inversion.cpp:150-152)
        const char* names[5] = {"rec:g11", "rec:g12", "rec:g22", "rec:b1", "rec:b2"};
        double* F[5];
        for (int k = 0; k < 5; ++k) F[k] = tbuf<double>(ctx, names[k], n);
        auto fill = [&](double* d, double v) {
            std::vector<double> hv(static_cast<size_t>(n), v);
            cuda_check(ctx, cudaMemcpyAsync(d, hv.data(), n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream),
                       "H2D");
            cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "sync");
        };
        for (int k = 0; k < 3; ++k) {
            if (init_metric && init_metric[k])
                cuda_check(ctx, cudaMemcpyAsync(F[k], init_metric[k], n * sizeof(double), in_kind, ctx->stream), "init");
            else
                fill(F[k], k == 1 ? 0.0 : 1.0);
        }
        for (int k = 0; k < 2; ++k) {
            if (init_drift && init_drift[k])
                cuda_check(ctx, cudaMemcpyAsync(F[3 + k], init_drift[k], n * sizeof(double), in_kind, ctx->stream),
                           "init");
            else
                fill(F[3 + k], 0.0);
        }
        // the optimized channels (ParamView::channels) alias the full planes
        // they expand into, except the isotropic g22 (a copy of g11) and g12 = 0
        const rfk_parameterization mode = cfg->param;
        std::vector<int> chan;  // indices into F
        switch (mode) {
            case RFK_PARAM_ISOTROPIC: chan = {0}; break;
            case RFK_PARAM_DIAGONAL: chan = {0, 2}; break;
            case RFK_PARAM_FULL: chan = {0, 1, 2}; break;
            case RFK_PARAM_DRIFT_ONLY: chan = {3, 4}; break;
            case RFK_PARAM_JOINT: chan = {0, 1, 2, 3, 4}; break;
            default: fail(ctx, RFK_ERR_INVALID_ARGUMENT, "recover: unknown parameterization");
        }
        const int np = static_cast<int>(chan.size());
        auto project = [&]() {  // ParamView::project (inversion.cpp:261-281)
            switch (mode) {
                case RFK_PARAM_ISOTROPIC:
                case RFK_PARAM_DIAGONAL:
                    for (int k : chan)
                        launched(ctx, rfk::launch_clamp(n, F[k], cfg->eps_min, cfg->lambda_max, ctx->stream), "clamp");
                    break;
                case RFK_PARAM_FULL:
                    validate_projection_cfg(ctx, cfg);
                    launched(ctx, rfk::launch_project_spd(n, F[0], F[1], F[2], cfg->eps_min, cfg->lambda_max, ctx->stream),
                             "project_spd");
                    break;
                case RFK_PARAM_DRIFT_ONLY:
                    validate_projection_cfg(ctx, cfg);
                    launched(ctx,
                             rfk::launch_project_drift(n, F[3], F[4], F[0], F[1], F[2], cfg->tau, cfg->euclid_cap,
                                                       ctx->stream),
                             "project_drift");
                    break;
                case RFK_PARAM_JOINT:
                    validate_projection_cfg(ctx, cfg);
                    launched(ctx, rfk::launch_project_spd(n, F[0], F[1], F[2], cfg->eps_min, cfg->lambda_max, ctx->stream),
                             "project_spd");
                    launched(ctx,
                             rfk::launch_project_drift(n, F[3], F[4], F[0], F[1], F[2], cfg->tau, cfg->euclid_cap,
                                                       ctx->stream),
                             "project_drift");
                    break;
            }
        };
        auto expand = [&]() {  // ParamView::expand (inversion.cpp:174-206)
            if (mode == RFK_PARAM_ISOTROPIC) {
                cuda_check(ctx, cudaMemcpyAsync(F[2], F[0], n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream),
                           "expand");
                cuda_check(ctx, cudaMemsetAsync(F[1], 0, n * sizeof(double), ctx->stream), "expand");
            } else if (mode == RFK_PARAM_DIAGONAL) {
                cuda_check(ctx, cudaMemsetAsync(F[1], 0, n * sizeof(double), ctx->stream), "expand");
            }
        };
        // truth planes in the mode's channel order (ParamView::error_vs, inversion.cpp:289-323)
        const bool has_truth = truth_metric || truth_drift;
        std::vector<const double*> tru;
        if (has_truth) {
            const bool need_g = mode != RFK_PARAM_DRIFT_ONLY, need_b = mode == RFK_PARAM_DRIFT_ONLY ||
                                                                       mode == RFK_PARAM_JOINT;
            if (need_g && !truth_metric) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "recover: truth metric missing");
            if (need_b && !truth_drift) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "recover: truth drift missing");
            for (int k : chan) {
                const double* src = k < 3 ? truth_metric[k] : truth_drift[k - 3];
                tru.push_back(st.in("rtru" + std::to_string(k), src, n));
            }
        }
        auto error_vs = [&]() {
            std::vector<const double*> est;
            for (int k : chan) est.push_back(F[k]);
            return relative_error_device(ctx, n, np, est.data(), tru.data(), exact);
        };
        // Adam moments (AdamState, zero-initialized on the first step)
        double *M[5] = {nullptr}, *V[5] = {nullptr};
        for (int k = 0; k < np; ++k) {
            M[k] = tbuf<double>(ctx, "rec:m" + std::to_string(k), n);
            V[k] = tbuf<double>(ctx, "rec:v" + std::to_string(k), n);
            cuda_check(ctx, cudaMemsetAsync(M[k], 0, n * sizeof(double), ctx->stream), "memset");
            cuda_check(ctx, cudaMemsetAsync(V[k], 0, n * sizeof(double), ctx->stream), "memset");
        }
        int64_t adam_t = 0;
        double* G[5];
        for (int k = 0; k < 5; ++k) G[k] = tbuf<double>(ctx, "rec:d" + std::to_string(k), n);
        double* gsum = tbuf<double>(ctx, "rec:gsum", n);

        project();
        rfk_fields fd{};
        fd.batch = 1;
        fd.rows = rows;
        fd.cols = cols;
        fd.h = h;
        fd.g11 = F[0];
        fd.g12 = F[1];
        fd.g22 = F[2];
        fd.b1 = F[3];
        fd.b2 = F[4];
        fd.src = od.sources;
        std::vector<double> loss_hist, err_hist;
        int32_t unreached_total = 0;
        double lr_scale = 1.0;
        double best_loss = std::numeric_limits<double>::infinity();
        double window_best = std::numeric_limits<double>::infinity();
        double initial_loss = -1.0;
        int window_fill = 0;
        int iterations = 0;
        for (int it = 0; it < cfg->iters; ++it) {
            expand();
            rfk_objective_value obj{};
            objective_device(ctx, &fd, &od, cfg, &obj, G);
            loss_hist.push_back(obj.loss);
            unreached_total += obj.unreached_observed;
            if (has_truth) err_hist.push_back(error_vs());
            if (initial_loss < 0.0)
                initial_loss = obj.loss;
            else if (obj.loss > 1e6 * std::max(initial_loss, 1e-12))
                fail(ctx, RFK_ERR_DIVERGED_LOSS, "recover: loss exploded at iteration " + std::to_string(it));
            // halve the step only when a whole window brings no new low (inversion.cpp:360-368)
            window_best = std::min(window_best, obj.loss);
            if (++window_fill >= cfg->plateau_window) {
                if (window_best >= best_loss * (1.0 - 1e-6) && lr_scale > 1.0 / 256.0) lr_scale *= cfg->plateau_factor;
                best_loss = std::min(best_loss, window_best);
                window_best = std::numeric_limits<double>::infinity();
                window_fill = 0;
            }
            // ParamView::map_gradient and step_sizes (inversion.cpp:208-259)
            std::vector<double*> grads;
            switch (mode) {
                case RFK_PARAM_ISOTROPIC:
                    launched(ctx, rfk::launch_add2(n, G[0], G[2], gsum, ctx->stream), "add2");
                    grads = {gsum};
                    break;
                case RFK_PARAM_DIAGONAL: grads = {G[0], G[2]}; break;
                case RFK_PARAM_FULL: grads = {G[0], G[1], G[2]}; break;
                case RFK_PARAM_DRIFT_ONLY: grads = {G[3], G[4]}; break;
                case RFK_PARAM_JOINT: grads = {G[0], G[1], G[2], G[3], G[4]}; break;
            }
            const double sg = cfg->step_g * lr_scale, sb = cfg->step_b * lr_scale;
            std::vector<double> steps;
            for (int k : chan) steps.push_back(k < 3 ? sg : sb);
            std::vector<double*> params;
            for (int k : chan) params.push_back(F[k]);
            if (cfg->optimizer == RFK_OPT_ADAM)
                adam_device(ctx, n, np, params.data(), M, V, adam_t, grads.data(), steps.data(), cfg->beta1,
                            cfg->beta2, cfg->adam_eps, cfg->grad_clip_norm, exact);
            else
                gd_device(ctx, n, np, params.data(), grads.data(), steps.data(), cfg->grad_clip_norm, exact);
            project();
            iterations = it + 1;
        }
        expand();
        double* outs[5] = {out->g11, out->g12, out->g22, out->b1, out->b2};
        const cudaMemcpyKind out_kind = mem == RFK_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        for (int k = 0; k < 5; ++k)
            if (outs[k])
                cuda_check(ctx, cudaMemcpyAsync(outs[k], F[k], n * sizeof(double), out_kind, ctx->stream), "out");
        if (mode == RFK_PARAM_ISOTROPIC && out->iso_g)
            cuda_check(ctx, cudaMemcpyAsync(out->iso_g, F[0], n * sizeof(double), out_kind, ctx->stream), "out");
        out->final_error = has_truth ? error_vs() : -1.0;
        st.finish();
        std::copy(loss_hist.begin(), loss_hist.end(), out->loss_history);
        if (out->error_history) std::copy(err_hist.begin(), err_hist.end(), out->error_history);
        out->iterations = iterations;
        out->unreached_observed_total = unreached_total;
    });
}

RFK_API rfk_status rfk_generate_observations(rfk_context* ctx, rfk_memory mem, const rfk_fields* f, int32_t count,
                                             const uint8_t* sources, double density, double noise_level,
                                             uint64_t seed, uint8_t* observed, double* values) {
    return guarded(ctx, [&] {
        if (!f || !sources || !observed || !values || count < 1) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null argument");
        // inversion.cpp:391-394
        if (!(density > 0.0) || density > 1.0)
            fail(ctx, RFK_ERR_INVALID_ARGUMENT, "generate_observations: density must be in (0, 1]");
        if (noise_level < 0.0) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "generate_observations: noise_level must be >= 0");
        const int64_t n = static_cast<int64_t>(f->rows) * f->cols;
        const size_t nk = static_cast<size_t>(n) * count;
        rfk_fields fb = *f;
        fb.batch = count;
        fb.param_stride = 0;
        fb.src = sources;
        fb.src_stride = n;
        fb.fixed_values = nullptr;
        // the count solves run as one batch on the device; T comes back to the host
        std::vector<double> T(nk);
        std::vector<int32_t> its(count), conv(count);
        std::vector<uint8_t> hsrc(nk);
        if (mem == RFK_MEM_DEVICE) {
            double* td = tbuf<double>(ctx, "gen:t", nk);
            int32_t* itd = tbuf<int32_t>(ctx, "gen:it", count);
            int32_t* cvd = tbuf<int32_t>(ctx, "gen:cv", count);
            const rfk_status s = rfk_solve(ctx, RFK_MEM_DEVICE, &fb, nullptr, td, itd, cvd, nullptr);
            if (s != RFK_OK) throw Fail{s};
            cuda_check(ctx, cudaMemcpy(T.data(), td, nk * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
            cuda_check(ctx, cudaMemcpy(conv.data(), cvd, count * sizeof(int32_t), cudaMemcpyDeviceToHost), "D2H");
            cuda_check(ctx, cudaMemcpy(hsrc.data(), sources, nk, cudaMemcpyDeviceToHost), "D2H");
        } else {
            const rfk_status s = rfk_solve(ctx, RFK_MEM_HOST, &fb, nullptr, T.data(), its.data(), conv.data(), nullptr);
            if (s != RFK_OK) throw Fail{s};
            std::copy(sources, sources + nk, hsrc.begin());
        }
        std::vector<uint8_t> hobs(nk, 0);
        std::vector<double> hval(nk, 0.0);
        for (int si = 0; si < count; ++si) {
            if (!conv[si]) fail(ctx, RFK_ERR_NOT_CONVERGED, "generate_observations: solve did not converge");
            const double* t = T.data() + static_cast<size_t>(si) * n;
            const uint8_t* src = hsrc.data() + static_cast<size_t>(si) * n;
            // inversion.cpp:404-433, the reference's own sampling
            std::vector<int> candidates;
            for (int i = 0; i < static_cast<int>(n); ++i)
                if (!src[i] && t[i] < 1e9) candidates.push_back(i);
            std::mt19937_64 rng(seed ^ (0x9e3779b97f4a7c15ULL * (static_cast<uint64_t>(si) + 1)));
            std::shuffle(candidates.begin(), candidates.end(), rng);
            const size_t cnt = static_cast<size_t>(density * candidates.size());
            double mean = 0.0, sq = 0.0;
            for (size_t k = 0; k < cnt; ++k) mean += t[candidates[k]];
            if (cnt > 0) mean /= static_cast<double>(cnt);
            for (size_t k = 0; k < cnt; ++k) {
                const double d = t[candidates[k]] - mean;
                sq += d * d;
            }
            const double sd = cnt > 1 ? std::sqrt(sq / static_cast<double>(cnt)) : 0.0;
            std::normal_distribution<double> noise(0.0, 1.0);
            uint8_t* ob = hobs.data() + static_cast<size_t>(si) * n;
            double* va = hval.data() + static_cast<size_t>(si) * n;
            for (size_t k = 0; k < cnt; ++k) {
                const int i = candidates[k];
                ob[i] = 1;
                double v = t[i];
                if (noise_level > 0.0) v += noise_level * sd * noise(rng);
                va[i] = std::max(v, 0.0);
            }
        }
        const cudaMemcpyKind kind = mem == RFK_MEM_DEVICE ? cudaMemcpyHostToDevice : cudaMemcpyHostToHost;
        cuda_check(ctx, cudaMemcpy(observed, hobs.data(), nk, kind), "out");
        cuda_check(ctx, cudaMemcpy(values, hval.data(), nk * sizeof(double), kind), "out");
    });
}

RFK_API rfk_status rfk_multi_source_recover(rfk_context* ctx, const int32_t* ks, int32_t nks, double density,
                                            const rfk_inverse_config* cfg, int32_t grid_size, uint64_t seed,
                                            rfk_multi_source_row* rows) {
    return guarded(ctx, [&] {
        if (!ks || nks < 1 || !cfg || !rows) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "null argument");
        for (int i = 0; i < nks; ++i)
            if (ks[i] < 1) fail(ctx, RFK_ERR_INVALID_ARGUMENT, "multi_source_recover: k must be >= 1");
        const int n = grid_size;
        const double h = 1.0 / n;
        const size_t nn = static_cast<size_t>(n) * n;
        // two-region isotropic medium, interface down the middle (inversion.cpp:447-454)
        std::vector<double> g11(nn, 1.0), g12(nn, 0.0), zero(nn, 0.0);
        for (int r = 0; r < n; ++r)
            for (int c = n / 2; c < n; ++c) g11[static_cast<size_t>(r) * n + c] = 2.0;
        // nested source layouts (inversion.cpp:456-477), the reference's own sampling
        const int kmax = *std::max_element(ks, ks + nks);
        std::mt19937_64 rng(seed);
        std::uniform_int_distribution<int> pick(n / 8, n - 1 - n / 8);
        std::vector<std::pair<int, int>> pts;
        double min_sep = n / 4.0;
        int attempts = 0;
        while (static_cast<int>(pts.size()) < kmax) {
            const int r = pick(rng), c = pick(rng);
            bool ok = true;
            for (auto [pr, pc] : pts) {
                const double d = std::hypot(double(r - pr), double(c - pc));
                if (d < min_sep) {
                    ok = false;
                    break;
                }
            }
            if (ok) pts.emplace_back(r, c);
            if (++attempts > 2000) {
                min_sep *= 0.9;
                attempts = 0;
            }
        }
        const double* truth_g[3] = {g11.data(), g12.data(), g11.data()};
        rfk_inverse_config c2 = *cfg;
        c2.param = RFK_PARAM_ISOTROPIC;
        std::vector<double> loss_hist(static_cast<size_t>(std::max(1, c2.iters)));
        for (int i = 0; i < nks; ++i) {
            const int k = ks[i];
            std::vector<uint8_t> src(nn * k, 0), obs(nn * k);
            std::vector<double> val(nn * k);
            for (int j = 0; j < k; ++j) src[nn * j + static_cast<size_t>(pts[j].first) * n + pts[j].second] = 1;
            rfk_fields f{};
            f.batch = 1;
            f.rows = f.cols = n;
            f.h = h;
            f.g11 = g11.data();
            f.g12 = g12.data();
            f.g22 = g11.data();
            f.b1 = zero.data();
            f.b2 = zero.data();
            f.src = src.data();
            rfk_status s = rfk_generate_observations(ctx, RFK_MEM_HOST, &f, k, src.data(), density, 0.0, seed,
                                                     obs.data(), val.data());
            if (s != RFK_OK) throw Fail{s};
            int total = 0;
            for (uint8_t o : obs) total += o ? 1 : 0;
            rfk_observations od{k, src.data(), obs.data(), val.data()};
            rfk_recovery res{};
            res.loss_history = loss_hist.data();
            s = rfk_recover(ctx, RFK_MEM_HOST, n, n, h, &od, &c2, nullptr, nullptr, truth_g, nullptr, &res);
            if (s != RFK_OK) throw Fail{s};
            rows[i].k = k;
            rows[i].total_observations = total;
            rows[i].error = res.final_error;
        }
    });
}

}  // extern "C"
