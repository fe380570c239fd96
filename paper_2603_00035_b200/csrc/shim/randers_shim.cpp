// randers_shim.cpp — the link-level drop-in for the reference's hot path.
//
// Exports the exact randers:: symbols of the reference translation units
// src/stencil.cpp, src/sweeper.cpp, src/adjoint.cpp and the projections and
// regularizers of src/feasibility.cpp, implemented on top of the C ABI in
// include/rfk.h.  Compiled against the reference's own public headers
// (-I proj/include), so reference callers — objective_and_grad, recover,
// the validation oracles, the acceptance gate — link against it unchanged.
// Every computation runs on the GPU through librfk.so; the shim only
// converts randers:: containers to planes and status codes to exceptions.
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "randers/adjoint.hpp"
#include "randers/feasibility.hpp"
#include "randers/stencil.hpp"
#include "randers/sweeper.hpp"
#include "rfk.h"

namespace {

// One rfk_context per calling thread.  A context owns mutable state (the
// named device workspaces, the error string, the epoch counters), so sharing
// one across threads would race; the reference functions this shim replaces
// are reentrant, and a caller that runs independent
// problems on several threads stays correct: each thread gets its own
// workspaces, and the calls, which are synchronous, serialise on the device.
struct ThreadContext {
    rfk_context* c = nullptr;
    bool tried = false;
    ~ThreadContext() {
        if (c) rfk_destroy(c);
    }
};

rfk_context* ctx() {
    static thread_local ThreadContext tc;
    if (!tc.tried) {
        tc.tried = true;
        if (rfk_create(&tc.c, 0) != RFK_OK) tc.c = nullptr;
    }
    if (!tc.c) throw randers::Error("randers (B200): no CUDA device available — there is no CPU fallback");
    return tc.c;
}

// rfk_status -> the reference's exception types (errors.hpp:8-50)
void check(rfk_status st) {
    if (st == RFK_OK) return;
    const std::string msg = rfk_last_error(ctx());
    switch (st) {
        case RFK_ERR_DIMENSION_MISMATCH: throw randers::DimensionMismatch(msg);
        case RFK_ERR_ZERO_DIMENSION: throw randers::ZeroDimension(msg);
        case RFK_ERR_INVALID_ARGUMENT: throw randers::InvalidArgument(msg);
        case RFK_ERR_INCONSISTENT_FIXED_POINT: throw randers::InconsistentFixedPoint(msg);
        case RFK_ERR_NOT_CONVERGED: throw randers::NotConverged(msg);
        case RFK_ERR_NON_SPD_INPUT: throw randers::NonSpdInput(msg);
        case RFK_ERR_DIVERGED_LOSS: throw randers::DivergedLoss(msg);
        default: throw randers::Error("randers (B200): " + msg);
    }
}

// check_dims (sweeper.cpp:76-84): GridSpec first, then shapes, then sources.
void check_dims(const randers::MetricField& g, const randers::DriftField& b, const randers::SourceMask& src,
                const randers::GridSpec& spec) {
    spec.validate();
    auto same = [&](const auto& p) { return p.same_shape(spec.rows, spec.cols); };
    if (!same(g.g11) || !same(g.g12) || !same(g.g22) || !same(b.b1) || !same(b.b2) || !same(src.mask))
        throw randers::DimensionMismatch("solve: field dimensions disagree with grid spec");
}

rfk_fields fields(const randers::MetricField& g, const randers::DriftField& b, const randers::SourceMask& src,
                  const randers::GridSpec& spec, const double* fixed_values) {
    rfk_fields f{};
    f.batch = 1;
    f.rows = spec.rows;
    f.cols = spec.cols;
    f.h = spec.h;
    f.g11 = g.g11.data();
    f.g12 = g.g12.data();
    f.g22 = g.g22.data();
    f.b1 = b.b1.data();
    f.b2 = b.b2.data();
    f.src = src.mask.data();
    f.fixed_values = fixed_values;
    return f;
}

std::pair<randers::ArrivalField, randers::SolveReport> run(const randers::MetricField& g,
                                                           const randers::DriftField& b,
                                                           const randers::SourceMask& src,
                                                           const randers::Grid2D<double>* values,
                                                           const randers::GridSpec& spec,
                                                           const randers::SolveOptions& opt, bool jacobi) {
    check_dims(g, b, src, spec);
    if (values && !values->same_shape(spec.rows, spec.cols))
        throw randers::DimensionMismatch("solve: field dimensions disagree with grid spec");
    const rfk_fields f = fields(g, b, src, spec, values ? values->data() : nullptr);
    rfk_solve_options o{opt.tol, opt.max_iters, {opt.sweep_order[0], opt.sweep_order[1], opt.sweep_order[2],
                                                 opt.sweep_order[3]}};
    randers::ArrivalField out(spec.rows, spec.cols);
    std::vector<double> hist(opt.max_iters > 0 ? opt.max_iters : 1);
    int32_t it = 0, conv = 0;
    check(jacobi ? rfk_solve_jacobi(ctx(), RFK_MEM_HOST, &f, &o, out.t.data(), &it, &conv, hist.data())
                 : rfk_solve(ctx(), RFK_MEM_HOST, &f, &o, out.t.data(), &it, &conv, hist.data()));
    randers::SolveReport rep;
    rep.iterations = it;
    rep.converged = conv != 0;
    rep.max_delta_history.assign(hist.begin(), hist.begin() + it);
    return {std::move(out), rep};
}

randers::NodeCandidate candidate(int r, int c, const randers::Grid2D<double>& t, const randers::MetricField& g,
                                 const randers::DriftField& b, double h, bool update) {
    rfk_fields f{};
    f.batch = 1;
    f.rows = t.rows();
    f.cols = t.cols();
    f.h = h;
    f.g11 = g.g11.data();
    f.g12 = g.g12.data();
    f.g22 = g.g22.data();
    f.b1 = b.b1.data();
    f.b2 = b.b2.data();
    const int32_t node = t.index(r, c);
    double t0, l1, l2;
    int8_t ty, st, d1, d2, fd;
    check(rfk_best_candidate(ctx(), RFK_MEM_HOST, &f, t.data(), 1, &node, update ? 1 : 0, &t0, &ty, &st, &d1, &d2,
                             &l1, &l2, &fd));
    randers::NodeCandidate nc;
    nc.t0 = t0;
    nc.type = ty == RFK_TWO_POINT ? randers::UpdateType::TwoPoint : randers::UpdateType::OnePoint;
    nc.stencil = st;
    nc.donor1 = d1;
    nc.donor2 = d2;
    nc.lam1 = l1;
    nc.lam2 = l2;
    nc.found = fd != 0;
    return nc;
}

int neighbour_id(int cols, int node, int donor) {
    const int dr = donor / cols - node / cols, dc = donor % cols - node % cols;
    for (int k = 0; k < 8; ++k)
        if (randers::StencilTable::dr[k] == dr && randers::StencilTable::dc[k] == dc) return k;
    throw randers::InvalidArgument("stencil record: donor is not a Moore neighbour");
}

struct Planes {
    std::vector<int8_t> type, stencil, donor1, donor2;
    std::vector<double> c[5];
    rfk_records view() {
        rfk_records r{};
        r.type = type.data();
        r.stencil = stencil.data();
        r.donor1 = donor1.data();
        r.donor2 = donor2.data();
        for (int k = 0; k < 5; ++k) r.c[k] = c[k].data();
        return r;
    }
};

Planes to_planes(const randers::StencilRecordSet& set, int rows, int cols) {
    const size_t n = static_cast<size_t>(rows) * cols;
    Planes p;
    p.type.assign(n, -1);
    p.stencil.assign(n, -1);
    p.donor1.assign(n, -1);
    p.donor2.assign(n, -1);
    for (auto& v : p.c) v.assign(n, 0.0);
    for (const randers::StencilRecord& rec : set.records) {
        const size_t i = static_cast<size_t>(rec.node);
        const bool two = rec.type == randers::UpdateType::TwoPoint;
        p.type[i] = two ? RFK_TWO_POINT : RFK_ONE_POINT;
        p.stencil[i] = rec.stencil;
        p.donor1[i] = static_cast<int8_t>(neighbour_id(cols, rec.node, rec.donor[0]));
        if (two) {
            p.donor2[i] = static_cast<int8_t>(neighbour_id(cols, rec.node, rec.donor[1]));
            p.c[0][i] = rec.q11;
            p.c[1][i] = rec.q12;
            p.c[2][i] = rec.q22;
            p.c[3][i] = rec.u1;
            p.c[4][i] = rec.u2;
        } else {
            p.c[0][i] = rec.r_edge;
            p.c[1][i] = rec.e_edge;
        }
    }
    return p;
}

}  // namespace

namespace randers {

// ---- src/stencil.cpp ---------------------------------------------------------
TwoPointResult two_point_update(double t1, double t2, const Vec2& m1, const Vec2& m2, const Sym2& g,
                                const Vec2& b) {
    double t0, l1, l2;
    int8_t valid;
    check(rfk_two_point_update(ctx(), RFK_MEM_HOST, 1, &t1, &t2, &m1.x, &m1.y, &m2.x, &m2.y, &g.a11, &g.a12, &g.a22,
                               &b.x, &b.y, &t0, &l1, &l2, &valid));
    TwoPointResult r;
    r.t0 = t0;
    r.lam1 = l1;
    r.lam2 = l2;
    r.valid = valid != 0;
    return r;
}

// ---- src/sweeper.cpp ---------------------------------------------------------
NodeCandidate best_candidate(int r, int c, const Grid2D<double>& t, const MetricField& g, const DriftField& b,
                             double h) {
    return candidate(r, c, t, g, b, h, false);
}

NodeCandidate node_update(int r, int c, const Grid2D<double>& t, const MetricField& g, const DriftField& b,
                          double h) {
    return candidate(r, c, t, g, b, h, true);
}

std::pair<ArrivalField, SolveReport> solve(const MetricField& g, const DriftField& b, const SourceMask& src,
                                           const GridSpec& spec, const SolveOptions& opt) {
    return run(g, b, src, nullptr, spec, opt, false);
}

std::pair<ArrivalField, SolveReport> solve_from_values(const MetricField& g, const DriftField& b,
                                                       const SourceMask& fixed, const Grid2D<double>& fixed_values,
                                                       const GridSpec& spec, const SolveOptions& opt) {
    return run(g, b, fixed, &fixed_values, spec, opt, false);
}

std::pair<ArrivalField, SolveReport> solve_jacobi(const MetricField& g, const DriftField& b, const SourceMask& src,
                                                  const GridSpec& spec, const SolveOptions& opt) {
    return run(g, b, src, nullptr, spec, opt, true);
}

// ---- src/adjoint.cpp ---------------------------------------------------------
StencilRecordSet identify_stencils(const ArrivalField& t, const MetricField& g, const DriftField& b,
                                   const SourceMask& src, const GridSpec& spec, double tol) {
    check_dims(g, b, src, spec);
    const int rows = spec.rows, cols = spec.cols;
    const size_t n = static_cast<size_t>(rows) * cols;
    Planes p;
    p.type.resize(n);
    p.stencil.resize(n);
    p.donor1.resize(n);
    p.donor2.resize(n);
    for (auto& v : p.c) v.resize(n);
    rfk_records rv = p.view();
    const rfk_fields f = fields(g, b, src, spec, nullptr);
    int32_t n2 = 0, n1 = 0;
    int64_t bad = -1;
    check(rfk_identify(ctx(), RFK_MEM_HOST, &f, t.t.data(), tol, &rv, &n2, &n1, &bad));
    StencilRecordSet set;
    set.record_index = Grid2D<int>(rows, cols, -1);
    set.records.reserve(static_cast<size_t>(n2) + n1);
    for (size_t i = 0; i < n; ++i) {
        if (p.type[i] < 0) continue;
        StencilRecord rec;
        const int node = static_cast<int>(i), r = node / cols, c = node % cols;
        rec.node = node;
        rec.type = p.type[i] == RFK_TWO_POINT ? UpdateType::TwoPoint : UpdateType::OnePoint;
        rec.stencil = p.stencil[i];
        const auto o1 = StencilTable::offset(p.donor1[i]);
        rec.donor[0] = t.t.index(r + o1[0], c + o1[1]);
        rec.m1 = StencilTable::displacement(p.donor1[i], spec.h);
        if (rec.type == UpdateType::TwoPoint) {
            const auto o2 = StencilTable::offset(p.donor2[i]);
            rec.donor[1] = t.t.index(r + o2[0], c + o2[1]);
            rec.m2 = StencilTable::displacement(p.donor2[i], spec.h);
            rec.q11 = p.c[0][i];
            rec.q12 = p.c[1][i];
            rec.q22 = p.c[2][i];
            rec.u1 = p.c[3][i];
            rec.u2 = p.c[4][i];
        } else {
            rec.r_edge = p.c[0][i];
            rec.e_edge = p.c[1][i];
        }
        set.record_index[i] = static_cast<int>(set.records.size());
        set.records.push_back(rec);
    }
    set.two_point_count = n2;
    set.one_point_count = n1;
    return set;
}

JacobianEntries jacobian_entries(const StencilRecord& rec) {
    const int8_t ty = rec.type == UpdateType::TwoPoint ? RFK_TWO_POINT : RFK_ONE_POINT;
    const double c0 = ty == RFK_TWO_POINT ? rec.q11 : rec.r_edge;
    const double c1 = ty == RFK_TWO_POINT ? rec.q12 : rec.e_edge;
    const double c2 = rec.q22, c3 = rec.u1, c4 = rec.u2;
    double d, j0, j1;
    int8_t cl;
    check(rfk_jacobian_entries(ctx(), RFK_MEM_HOST, 1, &ty, &c0, &c1, &c2, &c3, &c4, &d, &j0, &j1, &cl));
    JacobianEntries out;
    out.diag = d;
    out.donor[0] = j0;
    out.donor[1] = j1;
    out.clamped = cl != 0;
    return out;
}

AdjointField solve_adjoint(const StencilRecordSet& records, const ArrivalField& t, const Grid2D<double>& loss_grad) {
    const int rows = t.rows(), cols = t.cols();
    Planes p = to_planes(records, rows, cols);
    rfk_records rv = p.view();
    AdjointField out;
    out.lambda = Grid2D<double>(rows, cols, 0.0);
    int32_t cl = 0;
    check(rfk_solve_adjoint(ctx(), RFK_MEM_HOST, 1, rows, cols, t.t.data(), &rv, loss_grad.data(), out.lambda.data(),
                            &cl));
    out.clamped_diagonals = cl;
    return out;
}

ParamGradients param_gradients(const StencilRecordSet& records, const AdjointField& adj) {
    const int rows = adj.lambda.rows(), cols = adj.lambda.cols();
    ParamGradients out(rows, cols);
    if (records.records.empty()) return out;
    // the grid spacing is the records' own displacement length (stencil.hpp:24)
    const Vec2& m = records.records.front().m1;
    const double h = std::fabs(m.x) > 0.0 ? std::fabs(m.x) : std::fabs(m.y);
    Planes p = to_planes(records, rows, cols);
    rfk_records rv = p.view();
    check(rfk_param_gradients(ctx(), RFK_MEM_HOST, 1, rows, cols, h, &rv, adj.lambda.data(), out.g11.data(),
                              out.g12.data(), out.g22.data(), out.b1.data(), out.b2.data()));
    return out;
}

LossGrad loss_grad_mse(const ArrivalField& t, const ObservationSet& obs) {
    LossGrad out;
    out.grad = Grid2D<double>(t.rows(), t.cols(), 0.0);
    double loss = 0.0;
    int32_t unr = 0;
    check(rfk_loss_grad_mse(ctx(), RFK_MEM_HOST, 1, static_cast<int64_t>(t.t.size()), t.t.data(),
                            obs.observed.data(), obs.values.data(), out.grad.data(), &loss, &unr, 1));
    out.loss = loss;
    out.unreached_observed = unr;
    return out;
}

// ---- src/feasibility.cpp (projections) ----------------------------------------
void project_spd(Grid2D<double>& g11, Grid2D<double>& g12, Grid2D<double>& g22, const ProjectionConfig& cfg) {
    cfg.validate();
    check(rfk_project_spd(ctx(), RFK_MEM_HOST, static_cast<int64_t>(g11.size()), g11.data(), g12.data(), g22.data(),
                          cfg.eps_min, cfg.lambda_max));
}

void project_drift(Grid2D<double>& b1, Grid2D<double>& b2, const Grid2D<double>& g11, const Grid2D<double>& g12,
                   const Grid2D<double>& g22, const ProjectionConfig& cfg) {
    cfg.validate();
    check(rfk_project_drift(ctx(), RFK_MEM_HOST, static_cast<int64_t>(b1.size()), b1.data(), b2.data(), g11.data(),
                            g12.data(), g22.data(), cfg.tau, cfg.euclid_cap));
}

double drift_norm_sq(double b1, double b2, double g11, double g12, double g22) {
    double out = 0.0;
    check(rfk_drift_norm_sq(ctx(), RFK_MEM_HOST, 1, &b1, &b2, &g11, &g12, &g22, &out));
    return out;
}

// ---- src/feasibility.cpp (regularizers, feasibility.cpp:137-196) ----------------
// The sums run in the reference's node order (exact_sum), so values and
// gradients are the reference's bits (Frobenius/Drift; Log-Euclidean goes
// through the device atan2/cos/sin/log).
TvResult tv_value_grad(const std::vector<Grid2D<double>>& channels, TvVariant variant, double eps_tv) {
    if (channels.empty() || channels.size() > 3) throw InvalidArgument("tv_value_grad: need 1..3 channels");
    if (!(eps_tv > 0.0)) throw InvalidArgument("tv_value_grad: eps_tv must be positive");
    const int rows = channels[0].rows(), cols = channels[0].cols();
    for (const auto& ch : channels)
        if (!ch.same_shape(rows, cols)) throw DimensionMismatch("tv_value_grad: channel shapes");
    TvResult out;
    out.grad.assign(channels.size(), Grid2D<double>(rows, cols, 0.0));
    const double* ch[3] = {nullptr, nullptr, nullptr};
    double* g[3] = {nullptr, nullptr, nullptr};
    for (size_t k = 0; k < channels.size(); ++k) {
        ch[k] = channels[k].data();
        g[k] = out.grad[k].data();
    }
    check(rfk_tv_value_grad(ctx(), RFK_MEM_HOST, rows, cols, static_cast<int32_t>(channels.size()),
                            static_cast<rfk_tv_variant>(static_cast<int>(variant)), eps_tv, ch, g, &out.value, 1));
    return out;
}

TikhonovResult tikhonov_value_grad(const std::vector<Grid2D<double>>& channels, double weight) {
    TikhonovResult out;
    std::vector<const double*> ch;
    for (const auto& c : channels) {
        out.grad.emplace_back(c.rows(), c.cols(), 0.0);
        ch.push_back(c.data());
    }
    if (channels.empty()) return out;
    std::vector<double*> g;
    for (auto& x : out.grad) g.push_back(x.data());
    check(rfk_tikhonov_value_grad(ctx(), RFK_MEM_HOST, static_cast<int64_t>(channels[0].size()),
                                  static_cast<int32_t>(channels.size()), weight, ch.data(), g.data(), &out.value, 1));
    return out;
}

}  // namespace randers
