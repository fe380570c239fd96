// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin C ABI over the *unmodified* reference library (/root/reference/proj),
// compiled by oracle/Makefile from the reference's own sources into
// oracle/_ref/libranders_ref.so.  It lets the Python tests and bench.py's
// CPU-baseline / reference arm call the reference's public API
// (proj/include/randers/*.hpp) on plain arrays:
//   - golden fixture generation (tests/golden/gen_golden.py),
//   - pinning the C restatement in oracle/oracle.c against the real thing,
//   - timing the reference's own CPU path (`bench.py --impl reference`).
// Every function here only marshals arrays into randers:: types and calls the
// reference; no arithmetic of the path is restated.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <random>
#include <thread>
#include <vector>

#include "randers/adjoint.hpp"
#include "randers/feasibility.hpp"
#include "randers/field_io.hpp"
#include "randers/inversion.hpp"
#include "randers/oracle.hpp"
#include "randers/sweeper.hpp"

using namespace randers;

namespace {

enum {
    REF_OK = 0,
    REF_DIM_MISMATCH = 1,
    REF_ZERO_DIM = 2,
    REF_INVALID_ARG = 3,
    REF_INCONSISTENT = 4,
    REF_NOT_CONVERGED = 8,
    REF_NON_SPD = 9,
    REF_DIVERGED = 10,
    REF_OTHER = 99,
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return REF_OK;
    } catch (const DimensionMismatch&) {
        return REF_DIM_MISMATCH;
    } catch (const ZeroDimension&) {
        return REF_ZERO_DIM;
    } catch (const InvalidArgument&) {
        return REF_INVALID_ARG;
    } catch (const InconsistentFixedPoint&) {
        return REF_INCONSISTENT;
    } catch (const NotConverged&) {
        return REF_NOT_CONVERGED;
    } catch (const NonSpdInput&) {
        return REF_NON_SPD;
    } catch (const DivergedLoss&) {
        return REF_DIVERGED;
    } catch (...) {
        return REF_OTHER;
    }
}

Grid2D<double> plane(int rows, int cols, const double* p) {
    Grid2D<double> g(rows, cols, 0.0);
    std::memcpy(g.data(), p, sizeof(double) * g.size());
    return g;
}

MetricField metric(int rows, int cols, const double* g11, const double* g12, const double* g22) {
    MetricField g(rows, cols);
    g.g11 = plane(rows, cols, g11);
    g.g12 = plane(rows, cols, g12);
    g.g22 = plane(rows, cols, g22);
    return g;
}

DriftField drift(int rows, int cols, const double* b1, const double* b2) {
    DriftField b(rows, cols);
    b.b1 = plane(rows, cols, b1);
    b.b2 = plane(rows, cols, b2);
    return b;
}

SourceMask mask(int rows, int cols, const uint8_t* m) {
    SourceMask s(rows, cols);
    std::memcpy(s.mask.data(), m, s.mask.size());
    return s;
}

void out_plane(const Grid2D<double>& g, double* out) {
    std::memcpy(out, g.data(), sizeof(double) * g.size());
}

struct Problem {
    GridSpec spec;
    MetricField g;
    DriftField b;
    SourceMask src;
};

Problem problem(int rows, int cols, double h, const double* g11, const double* g12,
                const double* g22, const double* b1, const double* b2, const uint8_t* src) {
    return Problem{GridSpec{rows, cols, h}, metric(rows, cols, g11, g12, g22),
                   drift(rows, cols, b1, b2), mask(rows, cols, src)};
}

}  // namespace

extern "C" {

// mode: 0 = solve, 1 = solve_jacobi, 2 = solve_from_values (fixed_values != NULL)
int ref_solve(int rows, int cols, double h, const double* g11, const double* g12,
              const double* g22, const double* b1, const double* b2, const uint8_t* src,
              const double* fixed_values, int mode, double tol, int max_iters,
              const int* sweep_order, double* t_out, int* iterations, int* converged,
              double* history) {
    return guarded([&] {
        Problem p = problem(rows, cols, h, g11, g12, g22, b1, b2, src);
        SolveOptions opt;
        opt.tol = tol;
        opt.max_iters = max_iters;
        if (sweep_order)
            for (int i = 0; i < 4; ++i) opt.sweep_order[i] = sweep_order[i];
        std::pair<ArrivalField, SolveReport> res;
        if (mode == 1) {
            res = solve_jacobi(p.g, p.b, p.src, p.spec, opt);
        } else if (mode == 2) {
            const Grid2D<double> fv = plane(rows, cols, fixed_values);
            res = solve_from_values(p.g, p.b, p.src, fv, p.spec, opt);
        } else {
            res = solve(p.g, p.b, p.src, p.spec, opt);
        }
        out_plane(res.first.t, t_out);
        *iterations = res.second.iterations;
        *converged = res.second.converged ? 1 : 0;
        if (history)
            for (size_t i = 0; i < res.second.max_delta_history.size(); ++i)
                history[i] = res.second.max_delta_history[i];
    });
}

// Per-node best_candidate for a list of nodes.
int ref_best_candidate(int rows, int cols, double h, const double* t, const double* g11,
                       const double* g12, const double* g22, const double* b1, const double* b2,
                       int n, const int* nodes, int node_update, double* t0, int8_t* type,
                       int8_t* stencil, int8_t* donor1, int8_t* donor2, double* lam1,
                       double* lam2, int8_t* found) {
    return guarded([&] {
        const MetricField g = metric(rows, cols, g11, g12, g22);
        const DriftField b = drift(rows, cols, b1, b2);
        const Grid2D<double> tt = plane(rows, cols, t);
        for (int i = 0; i < n; ++i) {
            const int r = nodes[i] / cols, c = nodes[i] % cols;
            const NodeCandidate nc = node_update ? randers::node_update(r, c, tt, g, b, h)
                                                 : best_candidate(r, c, tt, g, b, h);
            t0[i] = nc.t0;
            type[i] = static_cast<int8_t>(nc.type);
            stencil[i] = nc.stencil;
            donor1[i] = nc.donor1;
            donor2[i] = nc.donor2;
            lam1[i] = nc.lam1;
            lam2[i] = nc.lam2;
            found[i] = nc.found ? 1 : 0;
        }
    });
}

int ref_two_point_update(int n, const double* t1, const double* t2, const double* m1x,
                         const double* m1y, const double* m2x, const double* m2y,
                         const double* g11, const double* g12, const double* g22,
                         const double* b1, const double* b2, double* t0, double* lam1,
                         double* lam2, int8_t* valid) {
    return guarded([&] {
        for (int i = 0; i < n; ++i) {
            const TwoPointResult r =
                two_point_update(t1[i], t2[i], Vec2{m1x[i], m1y[i]}, Vec2{m2x[i], m2y[i]},
                                 Sym2{g11[i], g12[i], g22[i]}, Vec2{b1[i], b2[i]});
            t0[i] = r.t0;
            lam1[i] = r.lam1;
            lam2[i] = r.lam2;
            valid[i] = r.valid ? 1 : 0;
        }
    });
}

// identify_stencils expanded into per-node planes (row-major node index):
// type -1 = no record; two-point caches in c0..c4 = (q11, q12, q22, u1, u2);
// one-point caches c0, c1 = (r_edge, e_edge).  donor ids are neighbour
// indices 0..7 recovered from the linear donor nodes.
int ref_identify(int rows, int cols, double h, const double* t, const double* g11,
                 const double* g12, const double* g22, const double* b1, const double* b2,
                 const uint8_t* src, double tol, int8_t* type, int8_t* stencil, int8_t* donor1,
                 int8_t* donor2, double* c0, double* c1, double* c2, double* c3, double* c4,
                 int* two_point_count, int* one_point_count, int* record_index) {
    return guarded([&] {
        Problem p = problem(rows, cols, h, g11, g12, g22, b1, b2, src);
        ArrivalField at(rows, cols);
        at.t = plane(rows, cols, t);
        const StencilRecordSet set = identify_stencils(at, p.g, p.b, p.src, p.spec, tol);
        const size_t n = static_cast<size_t>(rows) * cols;
        for (size_t i = 0; i < n; ++i) {
            type[i] = -1;
            stencil[i] = donor1[i] = donor2[i] = -1;
            c0[i] = c1[i] = c2[i] = c3[i] = c4[i] = 0.0;
            record_index[i] = set.record_index[i];
        }
        auto neighbour_of = [&](int node, int donor) {
            const int dr = donor / cols - node / cols, dc = donor % cols - node % cols;
            for (int k = 0; k < 8; ++k)
                if (StencilTable::dr[k] == dr && StencilTable::dc[k] == dc) return k;
            return -1;
        };
        for (const StencilRecord& rec : set.records) {
            const int i = rec.node;
            type[i] = static_cast<int8_t>(rec.type);
            stencil[i] = rec.stencil;
            donor1[i] = static_cast<int8_t>(neighbour_of(i, rec.donor[0]));
            if (rec.type == UpdateType::TwoPoint) {
                donor2[i] = static_cast<int8_t>(neighbour_of(i, rec.donor[1]));
                c0[i] = rec.q11;
                c1[i] = rec.q12;
                c2[i] = rec.q22;
                c3[i] = rec.u1;
                c4[i] = rec.u2;
            } else {
                c0[i] = rec.r_edge;
                c1[i] = rec.e_edge;
            }
        }
        *two_point_count = set.two_point_count;
        *one_point_count = set.one_point_count;
    });
}

// identify_stencils -> solve_adjoint -> param_gradients on one converged field.
int ref_backward(int rows, int cols, double h, const double* t, const double* g11,
                 const double* g12, const double* g22, const double* b1, const double* b2,
                 const uint8_t* src, double tol, const double* loss_grad, double* lambda,
                 double* d_g11, double* d_g12, double* d_g22, double* d_b1, double* d_b2,
                 int* clamped) {
    return guarded([&] {
        Problem p = problem(rows, cols, h, g11, g12, g22, b1, b2, src);
        ArrivalField at(rows, cols);
        at.t = plane(rows, cols, t);
        const StencilRecordSet set = identify_stencils(at, p.g, p.b, p.src, p.spec, tol);
        const AdjointField adj = solve_adjoint(set, at, plane(rows, cols, loss_grad));
        const ParamGradients pg = param_gradients(set, adj);
        out_plane(adj.lambda, lambda);
        out_plane(pg.g11, d_g11);
        out_plane(pg.g12, d_g12);
        out_plane(pg.g22, d_g22);
        out_plane(pg.b1, d_b1);
        out_plane(pg.b2, d_b2);
        *clamped = adj.clamped_diagonals;
    });
}

int ref_jacobian_entries(int n, const int8_t* type, const double* c0, const double* c1,
                         const double* c2, const double* c3, const double* c4, double* diag,
                         double* j0, double* j1, int8_t* clamped) {
    return guarded([&] {
        for (int i = 0; i < n; ++i) {
            StencilRecord rec;
            rec.type = type[i] == 0 ? UpdateType::TwoPoint : UpdateType::OnePoint;
            if (rec.type == UpdateType::TwoPoint) {
                rec.q11 = c0[i];
                rec.q12 = c1[i];
                rec.q22 = c2[i];
                rec.u1 = c3[i];
                rec.u2 = c4[i];
            } else {
                rec.r_edge = c0[i];
                rec.e_edge = c1[i];
            }
            const JacobianEntries je = jacobian_entries(rec);
            diag[i] = je.diag;
            j0[i] = je.donor[0];
            j1[i] = je.donor[1];
            clamped[i] = je.clamped ? 1 : 0;
        }
    });
}

int ref_loss_grad_mse(int rows, int cols, const double* t, const uint8_t* observed,
                      const double* values, double* grad, double* loss, int* unreached) {
    return guarded([&] {
        ArrivalField at(rows, cols);
        at.t = plane(rows, cols, t);
        ObservationSet obs;
        obs.observed = Grid2D<uint8_t>(rows, cols, 0);
        std::memcpy(obs.observed.data(), observed, obs.observed.size());
        obs.values = plane(rows, cols, values);
        const LossGrad lg = loss_grad_mse(at, obs);
        out_plane(lg.grad, grad);
        *loss = lg.loss;
        *unreached = lg.unreached_observed;
    });
}

int ref_project_spd(int n, double* g11, double* g12, double* g22, double eps_min,
                    double lambda_max) {
    return guarded([&] {
        Grid2D<double> a = plane(1, n, g11), b = plane(1, n, g12), c = plane(1, n, g22);
        ProjectionConfig cfg;
        cfg.eps_min = eps_min;
        cfg.lambda_max = lambda_max;
        project_spd(a, b, c, cfg);
        out_plane(a, g11);
        out_plane(b, g12);
        out_plane(c, g22);
    });
}

int ref_project_drift(int n, double* b1, double* b2, const double* g11, const double* g12,
                      const double* g22, double tau, double euclid_cap) {
    return guarded([&] {
        Grid2D<double> x = plane(1, n, b1), y = plane(1, n, b2);
        ProjectionConfig cfg;
        cfg.tau = tau;
        cfg.euclid_cap = euclid_cap;
        project_drift(x, y, plane(1, n, g11), plane(1, n, g12), plane(1, n, g22), cfg);
        out_plane(x, b1);
        out_plane(y, b2);
    });
}

double ref_drift_norm_sq(double b1, double b2, double g11, double g12, double g22) {
    return drift_norm_sq(b1, b2, g11, g12, g22);
}

int ref_correlated_noise(int rows, int cols, int radius, uint64_t seed, int normalize,
                         double* out) {
    return guarded([&] { out_plane(correlated_noise(rows, cols, radius, seed, normalize != 0), out); });
}

// The unit-test helper random_feasible_fields (proj/tests/helpers.hpp:67-90),
// driven through the reference library: correlated noise, then the
// reference's own projections.
int ref_random_feasible_fields(int n, uint64_t seed, double drift_scale, double* g11,
                               double* g12, double* g22, double* b1, double* b2) {
    return guarded([&] {
        MetricField g(n, n, 1.0);
        DriftField b(n, n);
        const Grid2D<double> e1 = correlated_noise(n, n, 3, seed * 5 + 1);
        const Grid2D<double> e2 = correlated_noise(n, n, 3, seed * 5 + 2);
        const Grid2D<double> e3 = correlated_noise(n, n, 3, seed * 5 + 3);
        const Grid2D<double> e4 = correlated_noise(n, n, 3, seed * 5 + 4);
        const Grid2D<double> e5 = correlated_noise(n, n, 3, seed * 5 + 5);
        for (size_t i = 0; i < g.g11.size(); ++i) {
            g.g11[i] = 1.0 + 0.35 * e1[i];
            g.g12[i] = 0.2 * e2[i];
            g.g22[i] = 1.0 + 0.35 * e3[i];
            b.b1[i] = drift_scale * e4[i];
            b.b2[i] = drift_scale * e5[i];
        }
        ProjectionConfig cfg;
        cfg.eps_min = 0.5;
        cfg.lambda_max = 2.5;
        cfg.tau = std::min(0.95, 2.0 * drift_scale);
        project_spd(g, cfg);
        project_drift(b, g, cfg);
        out_plane(g.g11, g11);
        out_plane(g.g12, g12);
        out_plane(g.g22, g22);
        out_plane(b.b1, b1);
        out_plane(b.b2, b2);
    });
}

// 30% observation mask of tests/acceptance_main.cpp:57-68 (reference_loss).
int ref_observation_mask(int rows, int cols, const uint8_t* src, uint64_t seed, double frac,
                         uint8_t* observed) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> uni(0.0, 1.0);
        for (int i = 0; i < rows * cols; ++i) {
            observed[i] = 0;
            if (!src[i] && uni(rng) < frac) observed[i] = 1;
        }
    });
}

// ---------------------------------------------------------------------------
// CPU baseline: the body of adjoint_gradient (src/oracle.cpp:226-247) —
// solve -> loss_grad_mse -> identify_stencils -> solve_adjoint ->
// param_gradients — on `nprob` independent problems, one std::thread per
// problem (the reference has no intra-problem parallelism).  All problems
// share the same fields.  times[0..4] = per-phase seconds summed over
// problems; iterations = K of problem 0; records = records of problem 0.
// The reference arm's bounded sample at the bench config: nprob independent
// forward solves (problem i = planes + i*rows*cols), one std::thread each,
// all started together; wall time of the whole batch.  Forward only
// (max_iters may stop a solve early, so no adjoint follows).
int ref_solve_batch(int nprob, int rows, int cols, double h, const double* g11, const double* g12,
                    const double* g22, const double* b1, const double* b2, const uint8_t* src, double tol,
                    int max_iters, double* wall_seconds, int* iterations) {
    return guarded([&] {
        const size_t n = static_cast<size_t>(rows) * cols;
        std::vector<Problem> ps;
        ps.reserve(nprob);
        for (int i = 0; i < nprob; ++i)
            ps.push_back(problem(rows, cols, h, g11 + i * n, g12 + i * n, g22 + i * n, b1 + i * n, b2 + i * n,
                                 src + i * n));
        SolveOptions opt;
        opt.tol = tol;
        opt.max_iters = max_iters;
        std::vector<int> k(nprob, 0);
        auto w0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int i = 0; i < nprob; ++i)
            pool.emplace_back([&, i] { k[i] = solve(ps[i].g, ps[i].b, ps[i].src, ps[i].spec, opt).second.iterations; });
        for (auto& th : pool) th.join();
        *wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
        for (int i = 0; i < nprob; ++i) iterations[i] = k[i];
    });
}

int ref_pipeline(int rows, int cols, double h, const double* g11, const double* g12,
                 const double* g22, const double* b1, const double* b2, const uint8_t* src,
                 const uint8_t* observed, const double* values, double tol, int max_iters,
                 int nprob, int nthreads, double* wall_seconds, double* times, int* iterations,
                 int* records, int* converged) {
    return guarded([&] {
        Problem p = problem(rows, cols, h, g11, g12, g22, b1, b2, src);
        ObservationSet obs;
        obs.sources = p.src;
        obs.observed = Grid2D<uint8_t>(rows, cols, 0);
        std::memcpy(obs.observed.data(), observed, obs.observed.size());
        obs.values = plane(rows, cols, values);
        SolveOptions opt;
        opt.tol = tol;
        opt.max_iters = max_iters;

        std::vector<double> t_phase(5 * nprob, 0.0);
        std::vector<int> k(nprob, 0), nrec(nprob, 0), conv(nprob, 0);
        auto work = [&](int i) {
            using C = std::chrono::steady_clock;
            auto t0 = C::now();
            auto [t, rep] = solve(p.g, p.b, p.src, p.spec, opt);
            auto t1 = C::now();
            const LossGrad lg = loss_grad_mse(t, obs);
            auto t2 = C::now();
            const StencilRecordSet rs = identify_stencils(t, p.g, p.b, p.src, p.spec, tol);
            auto t3 = C::now();
            const AdjointField adj = solve_adjoint(rs, t, lg.grad);
            auto t4 = C::now();
            const ParamGradients pg = param_gradients(rs, adj);
            auto t5 = C::now();
            auto s = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
            t_phase[5 * i + 0] = s(t0, t1);
            t_phase[5 * i + 1] = s(t1, t2);
            t_phase[5 * i + 2] = s(t2, t3);
            t_phase[5 * i + 3] = s(t3, t4);
            t_phase[5 * i + 4] = s(t4, t5);
            k[i] = rep.iterations;
            conv[i] = rep.converged ? 1 : 0;
            nrec[i] = static_cast<int>(rs.records.size());
            (void)pg;
        };
        auto w0 = std::chrono::steady_clock::now();
        int next = 0;
        while (next < nprob) {
            std::vector<std::thread> pool;
            for (int j = 0; j < nthreads && next < nprob; ++j, ++next) pool.emplace_back(work, next);
            for (auto& th : pool) th.join();
        }
        *wall_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
        for (int f = 0; f < 5; ++f) {
            times[f] = 0.0;
            for (int i = 0; i < nprob; ++i) times[f] += t_phase[5 * i + f];
        }
        *iterations = k[0];
        *records = nrec[0];
        *converged = conv[0];
    });
}

// objective_and_grad (inversion.cpp:25-73) over `count` observation sets,
// regularizers off (lambda_g = lambda_b = 0).
int ref_objective_and_grad(int rows, int cols, double h, const double* g11, const double* g12,
                           const double* g22, const double* b1, const double* b2, int count,
                           const uint8_t* sources, const uint8_t* observed, const double* values,
                           double solve_tol, int solve_max_iters, double penalty_cap,
                           double* data_loss, int* unreached, double* d_g11, double* d_g12,
                           double* d_g22, double* d_b1, double* d_b2) {
    return guarded([&] {
        const size_t n = static_cast<size_t>(rows) * cols;
        const MetricField g = metric(rows, cols, g11, g12, g22);
        const DriftField b = drift(rows, cols, b1, b2);
        std::vector<ObservationSet> obs(count);
        for (int k = 0; k < count; ++k) {
            obs[k].sources = mask(rows, cols, sources + n * k);
            obs[k].observed = Grid2D<uint8_t>(rows, cols, 0);
            std::memcpy(obs[k].observed.data(), observed + n * k, n);
            obs[k].values = plane(rows, cols, values + n * k);
        }
        InverseConfig cfg;
        cfg.solve_tol = solve_tol;
        cfg.solve_max_iters = solve_max_iters;
        cfg.unreached_penalty_cap = penalty_cap;
        const Objective o = objective_and_grad(g, b, obs, GridSpec{rows, cols, h}, cfg);
        *data_loss = o.data_loss;
        *unreached = o.unreached_observed;
        out_plane(o.grad.g11, d_g11);
        out_plane(o.grad.g12, d_g12);
        out_plane(o.grad.g22, d_g22);
        out_plane(o.grad.b1, d_b1);
        out_plane(o.grad.b2, d_b2);
    });
}

// ---- recovery loop pieces (feasibility.cpp:106-196, inversion.cpp) ----------
static std::vector<Grid2D<double>> planes_of(int rows, int cols, int k, const double* const* p) {
    std::vector<Grid2D<double>> v;
    for (int i = 0; i < k; ++i) v.push_back(plane(rows, cols, p[i]));
    return v;
}

int ref_tv_value_grad(int rows, int cols, int nch, int variant, double eps_tv, const double* const* ch,
                      double* const* grad, double* value) {
    return guarded([&] {
        const TvResult r = tv_value_grad(planes_of(rows, cols, nch, ch), static_cast<TvVariant>(variant), eps_tv);
        *value = r.value;
        for (int k = 0; k < nch; ++k) out_plane(r.grad[k], grad[k]);
    });
}

int ref_tikhonov_value_grad(int rows, int cols, int nch, double weight, const double* const* ch,
                            double* const* grad, double* value) {
    return guarded([&] {
        const TikhonovResult r = tikhonov_value_grad(planes_of(rows, cols, nch, ch), weight);
        *value = r.value;
        for (int k = 0; k < nch; ++k) out_plane(r.grad[k], grad[k]);
    });
}

int ref_clip_global_norm(int rows, int cols, int np, double* const* g, double max_norm, double* norm) {
    return guarded([&] {
        std::vector<Grid2D<double>> v = planes_of(rows, cols, np, g);
        std::vector<Grid2D<double>*> p;
        for (auto& x : v) p.push_back(&x);
        *norm = clip_global_norm(p, max_norm);
        for (int k = 0; k < np; ++k) out_plane(v[k], g[k]);
    });
}

// one Adam step from a state (m, v, t); m, v, params updated in place
int ref_adam_step(int rows, int cols, int np, double* const* params, double* const* m, double* const* v, long* t,
                  const double* const* grads, const double* steps, double beta1, double beta2, double adam_eps,
                  double clip) {
    return guarded([&] {
        std::vector<Grid2D<double>> P = planes_of(rows, cols, np, params);
        std::vector<Grid2D<double>*> pp;
        for (auto& x : P) pp.push_back(&x);
        AdamState st;
        if (*t > 0) {
            st.m = planes_of(rows, cols, np, m);
            st.v = planes_of(rows, cols, np, v);
        }
        st.t = *t;
        InverseConfig cfg;
        cfg.beta1 = beta1;
        cfg.beta2 = beta2;
        cfg.adam_eps = adam_eps;
        cfg.grad_clip_norm = clip;
        adam_step(st, pp, planes_of(rows, cols, np, grads), std::vector<double>(steps, steps + np), cfg);
        for (int k = 0; k < np; ++k) {
            out_plane(P[k], params[k]);
            out_plane(st.m[k], m[k]);
            out_plane(st.v[k], v[k]);
        }
        *t = st.t;
    });
}

int ref_gd_step(int rows, int cols, int np, double* const* params, const double* const* grads, const double* steps,
                double clip) {
    return guarded([&] {
        std::vector<Grid2D<double>> P = planes_of(rows, cols, np, params);
        std::vector<Grid2D<double>*> pp;
        for (auto& x : P) pp.push_back(&x);
        InverseConfig cfg;
        cfg.grad_clip_norm = clip;
        gd_step(pp, planes_of(rows, cols, np, grads), std::vector<double>(steps, steps + np), cfg);
        for (int k = 0; k < np; ++k) out_plane(P[k], params[k]);
    });
}

int ref_relative_error(int rows, int cols, int np, const double* const* est, const double* const* truth,
                       double* out) {
    return guarded([&] {
        std::vector<Grid2D<double>> E = planes_of(rows, cols, np, est), T = planes_of(rows, cols, np, truth);
        std::vector<const Grid2D<double>*> e, t;
        for (int k = 0; k < np; ++k) {
            e.push_back(&E[k]);
            t.push_back(&T[k]);
        }
        *out = relative_error(e, t);
    });
}

// InverseConfig as a flat array of doubles (the order of rfk_inverse_config):
// param, optimizer, step_g, step_b, beta1, beta2, adam_eps, grad_clip_norm,
// lambda_g, lambda_b, tv_variant, iters, eps_min, lambda_max, tau, euclid_cap,
// solve_tol, solve_max_iters, plateau_window, plateau_factor, unreached_penalty_cap
static InverseConfig config_of(const double* c) {
    InverseConfig cfg;
    cfg.param = static_cast<Parameterization>(static_cast<int>(c[0]));
    cfg.optimizer = static_cast<OptimizerKind>(static_cast<int>(c[1]));
    cfg.step_g = c[2];
    cfg.step_b = c[3];
    cfg.beta1 = c[4];
    cfg.beta2 = c[5];
    cfg.adam_eps = c[6];
    cfg.grad_clip_norm = c[7];
    cfg.lambda_g = c[8];
    cfg.lambda_b = c[9];
    cfg.tv_variant = static_cast<TvVariant>(static_cast<int>(c[10]));
    cfg.iters = static_cast<int>(c[11]);
    cfg.projection.eps_min = c[12];
    cfg.projection.lambda_max = c[13];
    cfg.projection.tau = c[14];
    cfg.projection.euclid_cap = c[15];
    cfg.solve_tol = c[16];
    cfg.solve_max_iters = static_cast<int>(c[17]);
    cfg.plateau_window = static_cast<int>(c[18]);
    cfg.plateau_factor = c[19];
    cfg.unreached_penalty_cap = c[20];
    return cfg;
}

static std::vector<ObservationSet> obs_of(int rows, int cols, int count, const uint8_t* sources,
                                          const uint8_t* observed, const double* values) {
    const size_t n = static_cast<size_t>(rows) * cols;
    std::vector<ObservationSet> obs(count);
    for (int k = 0; k < count; ++k) {
        obs[k].sources = mask(rows, cols, sources + n * k);
        obs[k].observed = Grid2D<uint8_t>(rows, cols, 0);
        std::memcpy(obs[k].observed.data(), observed + n * k, n);
        obs[k].values = plane(rows, cols, values + n * k);
    }
    return obs;
}

// objective_and_grad with the full config (regularizers included)
int ref_objective(int rows, int cols, double h, const double* const* fields, int count, const uint8_t* sources,
                  const uint8_t* observed, const double* values, const double* cfgv, double* loss, double* data_loss,
                  double* reg_loss, int* unreached, double* const* grads) {
    return guarded([&] {
        const MetricField g = metric(rows, cols, fields[0], fields[1], fields[2]);
        const DriftField b = drift(rows, cols, fields[3], fields[4]);
        const Objective o = objective_and_grad(g, b, obs_of(rows, cols, count, sources, observed, values),
                                               GridSpec{rows, cols, h}, config_of(cfgv));
        *loss = o.loss;
        *data_loss = o.data_loss;
        *reg_loss = o.reg_loss;
        *unreached = o.unreached_observed;
        const Grid2D<double>* gp[5] = {&o.grad.g11, &o.grad.g12, &o.grad.g22, &o.grad.b1, &o.grad.b2};
        for (int k = 0; k < 5; ++k) out_plane(*gp[k], grads[k]);
    });
}

// recover (inversion.cpp:327-385).  init / truth: 5 planes or null
// (truth_mask bit 0: metric present, bit 1: drift present).
int ref_recover(int rows, int cols, double h, int count, const uint8_t* sources, const uint8_t* observed,
                const double* values, const double* cfgv, const double* const* init, const double* const* truth,
                int truth_mask, double* const* out_fields, double* iso_g, double* loss_history,
                double* error_history, int* iterations, double* final_error, int* unreached_total) {
    return guarded([&] {
        std::optional<MetricField> im;
        std::optional<DriftField> id;
        if (init) {
            im = metric(rows, cols, init[0], init[1], init[2]);
            id = drift(rows, cols, init[3], init[4]);
        }
        TruthFields tf;
        if (truth && (truth_mask & 1)) tf.metric = metric(rows, cols, truth[0], truth[1], truth[2]);
        if (truth && (truth_mask & 2)) tf.drift = drift(rows, cols, truth[3], truth[4]);
        const RecoveryResult r = recover(obs_of(rows, cols, count, sources, observed, values),
                                         GridSpec{rows, cols, h}, config_of(cfgv), im, id, truth ? &tf : nullptr);
        const Grid2D<double>* fp[5] = {&r.metric.g11, &r.metric.g12, &r.metric.g22, &r.drift.b1, &r.drift.b2};
        for (int k = 0; k < 5; ++k) out_plane(*fp[k], out_fields[k]);
        if (iso_g && r.iso_g.size()) out_plane(r.iso_g, iso_g);
        std::copy(r.loss_history.begin(), r.loss_history.end(), loss_history);
        if (error_history) std::copy(r.error_history.begin(), r.error_history.end(), error_history);
        *iterations = r.iterations;
        *final_error = r.final_error;
        *unreached_total = r.unreached_observed_total;
    });
}

int ref_generate_observations(int rows, int cols, double h, const double* const* fields, int count,
                              const uint8_t* sources, double density, double noise_level, unsigned long long seed,
                              uint8_t* observed, double* values) {
    return guarded([&] {
        const size_t n = static_cast<size_t>(rows) * cols;
        std::vector<SourceMask> src;
        for (int k = 0; k < count; ++k) src.push_back(mask(rows, cols, sources + n * k));
        const auto obs = generate_observations(metric(rows, cols, fields[0], fields[1], fields[2]),
                                               drift(rows, cols, fields[3], fields[4]), src,
                                               GridSpec{rows, cols, h}, density, noise_level, seed);
        for (int k = 0; k < count; ++k) {
            std::memcpy(observed + n * k, obs[k].observed.data(), n);
            std::memcpy(values + n * k, obs[k].values.data(), n * sizeof(double));
        }
    });
}

int ref_multi_source_recover(const int* ks, int nks, double density, const double* cfgv, int grid_size,
                             unsigned long long seed, int* out_k, int* out_total, double* out_err) {
    return guarded([&] {
        const auto rows = multi_source_recover(std::vector<int>(ks, ks + nks), density, config_of(cfgv), grid_size,
                                               seed);
        for (size_t i = 0; i < rows.size(); ++i) {
            out_k[i] = rows[i].k;
            out_total[i] = rows[i].total_observations;
            out_err[i] = rows[i].error;
        }
    });
}

// field_io (field_io.cpp): write `channels` planes / export one as CSV.
int ref_write_field(const char* path, int rows, int cols, int channels, const double* planes) {
    return guarded([&] {
        std::vector<Grid2D<double>> ch;
        for (int k = 0; k < channels; ++k)
            ch.push_back(plane(rows, cols, planes + static_cast<size_t>(rows) * cols * k));
        write_field(path, ch);
    });
}
int ref_read_field_dims(const char* path, int* rows, int* cols, int* channels) {
    return guarded([&] {
        const FieldData d = read_field(path);
        *rows = d.rows();
        *cols = d.cols();
        *channels = d.channel_count();
    });
}
int ref_read_field(const char* path, double* planes) {
    return guarded([&] {
        const FieldData d = read_field(path);
        for (int k = 0; k < d.channel_count(); ++k)
            out_plane(d.channels[k], planes + static_cast<size_t>(d.rows()) * d.cols() * k);
    });
}
int ref_export_csv(const char* path, int rows, int cols, const double* p) {
    return guarded([&] { export_csv(plane(rows, cols, p), path); });
}

}  // extern "C"
