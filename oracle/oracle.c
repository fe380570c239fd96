/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
 *
 * Plain C, compiled with -O2 -ffp-contract=off (no FMA contraction, no
 * -march) so every double operation rounds exactly like the reference's
 * g++ -O3 build.  Each function cites the reference line it
 * restates; operation order (association of every +,*) is kept literally,
 * because it fixes the bits.  Pinned bit-for-bit against the reference
 * library (oracle/_ref) and the golden fixtures by tests/test_oracle.py.
 *
 * Used only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg.  The product never links it. */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define UNREACHED 1e10          /* grid.hpp:14 */
#define UNREACHED_THRESHOLD 1e9 /* grid.hpp:15 */

/* Moore ring (stencil.hpp:17-18): UL, W, LL, S, LR, E, UR, N. */
static const int RING_DR[8] = {-1, 0, 1, 1, 1, 0, -1, -1};
static const int RING_DC[8] = {-1, -1, -1, 0, 1, 1, 1, 0};

static int reached(double t) { return t < UNREACHED_THRESHOLD; } /* grid.hpp:17 */
/* std::max / std::min / std::clamp as libstdc++ defines them. */
static double smax(double a, double b) { return (a < b) ? b : a; }
static double smin(double a, double b) { return (b < a) ? b : a; }
static double sclamp(double v, double lo, double hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

/* displacement(k, h) = (dc*h, dr*h), int*double (stencil.hpp:24). */
static void disp(int k, double h, double* x, double* y) {
    *x = (double)RING_DC[k] * h;
    *y = (double)RING_DR[k] * h;
}
/* Vec2::dot, Sym2::mul, Sym2::quad (mat2.hpp:17,32,33). */
static double dot2(double ax, double ay, double bx, double by) { return ax * bx + ay * by; }
static void mul2(double g11, double g12, double g22, double vx, double vy, double* ox, double* oy) {
    *ox = g11 * vx + g12 * vy;
    *oy = g12 * vx + g22 * vy;
}
static double quad2(double g11, double g12, double g22, double vx, double vy) {
    double gx, gy;
    mul2(g11, g12, g22, vx, vy, &gx, &gy);
    return dot2(vx, vy, gx, gy);
}

/* two_point_update, src/stencil.cpp:7-43. */
void orc_two_point_update(double t1, double t2, double m1x, double m1y, double m2x, double m2y,
                          double g11, double g12, double g22, double b1, double b2,
                          double* t0_out, double* lam1_out, double* lam2_out, int* valid_out) {
    double gm1x, gm1y, gm2x, gm2y;
    *t0_out = 0.0;
    *lam1_out = 0.0;
    *lam2_out = 0.0;
    *valid_out = 0;
    mul2(g11, g12, g22, m1x, m1y, &gm1x, &gm1y);
    const double e11 = dot2(m1x, m1y, gm1x, gm1y);
    const double e12 = dot2(m2x, m2y, gm1x, gm1y);
    mul2(g11, g12, g22, m2x, m2y, &gm2x, &gm2y);
    const double e22 = dot2(m2x, m2y, gm2x, gm2y);
    const double det = e11 * e22 - e12 * e12;
    if (!(det > 1e-14 * smax(e11 * e22, e12 * e12))) return; /* :17-18 */
    const double q11 = e22 / det;
    const double q12 = -e12 / det;
    const double q22 = e11 / det;
    const double s1 = t1 + dot2(m1x, m1y, b1, b2);
    const double s2 = t2 + dot2(m2x, m2y, b1, b2);
    const double a = q11 + 2.0 * q12 + q22;
    const double bq = (q11 + q12) * s1 + (q12 + q22) * s2;
    const double c = q11 * s1 * s1 + 2.0 * q12 * s1 * s2 + q22 * s2 * s2 - 1.0;
    const double disc = bq * bq - a * c;
    if (disc < 0.0 || a <= 0.0) return; /* :32-33 */
    const double t0 = (bq + sqrt(disc)) / a;
    const double d1 = t0 - s1;
    const double d2 = t0 - s2;
    *t0_out = t0;
    *lam1_out = q11 * d1 + q12 * d2;
    *lam2_out = q12 * d1 + q22 * d2;
    *valid_out = t0 > smax(t1, t2) && *lam1_out >= 0.0 && *lam2_out >= 0.0; /* :41 */
}

/* best_candidate, src/sweeper.cpp:8-61. */
orc_candidate orc_best_candidate(int r, int c, int rows, int cols, double h, const double* t,
                                 const double* g11, const double* g12, const double* g22,
                                 const double* b1, const double* b2) {
    orc_candidate best = {UNREACHED, 1, -1, -1, -1, 0.0, 0.0, 0};
    const size_t node = (size_t)r * cols + c;
    const double G11 = g11[node], G12 = g12[node], G22 = g22[node];
    const double B1 = b1[node], B2 = b2[node];
    double tn[8];
    int in[8];
    for (int k = 0; k < 8; ++k) {
        const int nr = r + RING_DR[k], nc = c + RING_DC[k];
        in[k] = nr >= 0 && nr < rows && nc >= 0 && nc < cols;
        tn[k] = in[k] ? t[(size_t)nr * cols + nc] : UNREACHED;
    }
    for (int k = 0; k < 8; ++k) {
        const int k2 = (k + 1) % 8;
        if (in[k] && in[k2] && reached(tn[k]) && reached(tn[k2])) {
            double m1x, m1y, m2x, m2y, t0, l1, l2;
            int valid;
            disp(k, h, &m1x, &m1y);
            disp(k2, h, &m2x, &m2y);
            orc_two_point_update(tn[k], tn[k2], m1x, m1y, m2x, m2y, G11, G12, G22, B1, B2, &t0,
                                 &l1, &l2, &valid);
            if (valid) {
                if (!best.found || t0 < best.t0) { /* :44 */
                    best.found = 1;
                    best.t0 = t0;
                    best.type = 0;
                    best.stencil = k;
                    best.donor1 = k;
                    best.donor2 = k2;
                    best.lam1 = l1;
                    best.lam2 = l2;
                }
                continue; /* :54 */
            }
        }
        /* one-point fallbacks from k then k2 (:24-36, :57-58) */
        for (int j = 0; j < 2; ++j) {
            const int d = j == 0 ? k : k2;
            double mx, my;
            if (!in[d] || !reached(tn[d])) continue;
            disp(d, h, &mx, &my);
            /* one_point_update, stencil.hpp:43-45 */
            const double t0 = tn[d] + dot2(mx, my, B1, B2) + sqrt(quad2(G11, G12, G22, mx, my));
            if (best.found && !(t0 < best.t0)) continue; /* :27 */
            best.found = 1;
            best.t0 = t0;
            best.type = 1;
            best.stencil = k;
            best.donor1 = d;
            best.donor2 = -1;
            best.lam1 = best.lam2 = 0.0;
        }
    }
    return best;
}

/* check_dims + GridSpec::validate + SourceMask::validate (sweeper.cpp:76-84,
 * grid.hpp:61-65, :124-126). */
static int validate(int rows, int cols, double h, const uint8_t* src) {
    if (rows < 3 || cols < 3) return 2;
    if (!(h > 0.0)) return 3;
    size_t n = (size_t)rows * cols, cnt = 0;
    for (size_t i = 0; i < n; ++i) cnt += src[i] ? 1 : 0;
    if (cnt == 0) return 3;
    return 0;
}

/* Sweeper::relax + sweep (sweeper.cpp:92-121). */
static void relax(int r, int c, int rows, int cols, double h, double* t, const uint8_t* fixed,
                  const double* g11, const double* g12, const double* g22, const double* b1,
                  const double* b2) {
    const size_t i = (size_t)r * cols + c;
    if (fixed[i]) return;
    const orc_candidate cand = orc_best_candidate(r, c, rows, cols, h, t, g11, g12, g22, b1, b2);
    if (cand.found && cand.t0 < t[i]) t[i] = cand.t0;
}

static void sweep(int dir, int rows, int cols, double h, double* t, const uint8_t* fixed,
                  const double* g11, const double* g12, const double* g22, const double* b1,
                  const double* b2) {
    int r, c;
    switch (dir) {
        case 0: /* columns left to right, rows top to bottom */
            for (c = 0; c < cols; ++c)
                for (r = 0; r < rows; ++r) relax(r, c, rows, cols, h, t, fixed, g11, g12, g22, b1, b2);
            break;
        case 1: /* rows top to bottom, columns right to left */
            for (r = 0; r < rows; ++r)
                for (c = cols - 1; c >= 0; --c)
                    relax(r, c, rows, cols, h, t, fixed, g11, g12, g22, b1, b2);
            break;
        case 2: /* columns right to left, rows bottom to top */
            for (c = cols - 1; c >= 0; --c)
                for (r = rows - 1; r >= 0; --r)
                    relax(r, c, rows, cols, h, t, fixed, g11, g12, g22, b1, b2);
            break;
        default: /* rows bottom to top, columns left to right */
            for (r = rows - 1; r >= 0; --r)
                for (c = 0; c < cols; ++c) relax(r, c, rows, cols, h, t, fixed, g11, g12, g22, b1, b2);
            break;
    }
}

/* run_sweeping (sweeper.cpp:133-158), solve_from_values (:168-174),
 * solve_jacobi (:176-205). */
int orc_solve(int rows, int cols, double h, const double* g11, const double* g12,
              const double* g22, const double* b1, const double* b2, const uint8_t* src,
              const double* fixed_values, int mode, double tol, int max_iters,
              const int* sweep_order, double* t, int* iterations, int* converged,
              double* history) {
    const int st = validate(rows, cols, h, src);
    if (st) return st;
    const size_t n = (size_t)rows * cols;
    static const int default_order[4] = {0, 1, 2, 3};
    const int* order = sweep_order ? sweep_order : default_order;
    for (size_t i = 0; i < n; ++i) /* initial_field :124-131 */
        t[i] = src[i] ? ((mode == 2 && fixed_values) ? fixed_values[i] : 0.0) : UNREACHED;
    double* other = (double*)malloc(n * sizeof(double));
    memcpy(other, t, n * sizeof(double));
    *iterations = 0;
    *converged = 0;
    for (int it = 0; it < max_iters; ++it) {
        double max_delta = 0.0;
        if (mode == 1) {
            /* Jacobi: other := relaxed copy of t, then swap roles. */
            for (int r = 0; r < rows; ++r)
                for (int c = 0; c < cols; ++c) {
                    const size_t i = (size_t)r * cols + c;
                    if (src[i]) continue;
                    const orc_candidate cand =
                        orc_best_candidate(r, c, rows, cols, h, t, g11, g12, g22, b1, b2);
                    const double cur = t[i];
                    const double v = cand.found ? smin(cur, cand.t0) : cur;
                    other[i] = v;
                    max_delta = smax(max_delta, fabs(v - cur));
                }
            memcpy(t, other, n * sizeof(double));
        } else {
            /* `other` holds prev */
            for (int d = 0; d < 4; ++d) sweep(order[d], rows, cols, h, t, src, g11, g12, g22, b1, b2);
            for (size_t i = 0; i < n; ++i) max_delta = smax(max_delta, fabs(t[i] - other[i]));
        }
        if (history) history[it] = max_delta;
        *iterations = it + 1;
        if (max_delta < tol) {
            *converged = 1;
            break;
        }
        if (mode != 1) memcpy(other, t, n * sizeof(double));
    }
    free(other);
    return 0;
}

/* identify_stencils, src/adjoint.cpp:10-67. */
int orc_identify(int rows, int cols, double h, const double* t, const double* g11,
                 const double* g12, const double* g22, const double* b1, const double* b2,
                 const uint8_t* src, double tol, int8_t* type, int8_t* stencil, int8_t* donor1,
                 int8_t* donor2, double* c0, double* c1, double* c2, double* c3, double* c4,
                 int* two_point_count, int* one_point_count, int* bad_node) {
    int n2 = 0, n1 = 0;
    *bad_node = -1;
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            const size_t i = (size_t)r * cols + c;
            type[i] = stencil[i] = donor1[i] = donor2[i] = -1;
            c0[i] = c1[i] = c2[i] = c3[i] = c4[i] = 0.0;
            if (src[i] || !reached(t[i])) continue;
            const orc_candidate cand =
                orc_best_candidate(r, c, rows, cols, h, t, g11, g12, g22, b1, b2);
            const double stored = t[i];
            if (!cand.found || fabs(cand.t0 - stored) > 100.0 * tol) { /* :22-25 */
                if (*bad_node < 0) *bad_node = (int)i;
                continue;
            }
            const double G11 = g11[i], G12 = g12[i], G22 = g22[i], B1 = b1[i], B2 = b2[i];
            type[i] = (int8_t)cand.type;
            stencil[i] = (int8_t)cand.stencil;
            donor1[i] = (int8_t)cand.donor1;
            const size_t d0 = (size_t)(r + RING_DR[cand.donor1]) * cols + (c + RING_DC[cand.donor1]);
            double m1x, m1y;
            disp(cand.donor1, h, &m1x, &m1y);
            if (cand.type == 0) { /* :34-53 */
                double m2x, m2y, gx, gy;
                donor2[i] = (int8_t)cand.donor2;
                const size_t d1 =
                    (size_t)(r + RING_DR[cand.donor2]) * cols + (c + RING_DC[cand.donor2]);
                disp(cand.donor2, h, &m2x, &m2y);
                mul2(G11, G12, G22, m1x, m1y, &gx, &gy);
                const double e11 = dot2(m1x, m1y, gx, gy);
                const double e12 = dot2(m2x, m2y, gx, gy);
                const double e22 = quad2(G11, G12, G22, m2x, m2y);
                const double det = e11 * e22 - e12 * e12;
                c0[i] = e22 / det;
                c1[i] = -e12 / det;
                c2[i] = e11 / det;
                const double s1 = t[d0] + dot2(m1x, m1y, B1, B2);
                const double s2 = t[d1] + dot2(m2x, m2y, B1, B2);
                c3[i] = s1 - stored;
                c4[i] = s2 - stored;
                ++n2;
            } else { /* :54-61 */
                c0[i] = t[d0] + dot2(m1x, m1y, B1, B2) - stored;
                c1[i] = quad2(G11, G12, G22, m1x, m1y);
                ++n1;
            }
        }
    *two_point_count = n2;
    *one_point_count = n1;
    return *bad_node >= 0 ? 4 : 0;
}

/* jacobian_entries, src/adjoint.cpp:69-89. */
void orc_jacobian_entries(int type, double c0, double c1, double c2, double c3, double c4,
                          double* diag, double* j0, double* j1, int* clamped) {
    if (type == 0) {
        const double qu1 = c0 * c3 + c1 * c4;
        const double qu2 = c1 * c3 + c2 * c4;
        *diag = -2.0 * (qu1 + qu2);
        *j0 = 2.0 * qu1;
        *j1 = 2.0 * qu2;
    } else {
        *diag = -2.0 * c0;
        *j0 = 2.0 * c0;
        *j1 = 0.0;
    }
    const double scale = smax(fabs(*j0) + fabs(*j1), 1.0);
    const double floor_ = 1e-12 * scale;
    *clamped = 0;
    if (fabs(*diag) < floor_) {
        *diag = copysign(floor_, *diag == 0.0 ? 1.0 : *diag);
        *clamped = 1;
    }
}

static const double* g_sort_t;
static int by_time_desc(const void* pa, const void* pb) { /* adjoint.cpp:96-103 */
    const int a = *(const int*)pa, b = *(const int*)pb;
    const double ta = g_sort_t[a], tb = g_sort_t[b];
    if (ta != tb) return ta > tb ? -1 : 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* solve_adjoint, src/adjoint.cpp:91-117: sort by T desc / node asc, then
 * scatter back-substitution. */
int orc_adjoint(int rows, int cols, const double* t, const int8_t* type, const int8_t* donor1,
                const int8_t* donor2, const double* c0, const double* c1, const double* c2,
                const double* c3, const double* c4, const double* loss_grad, double* lambda,
                int* clamped) {
    const size_t n = (size_t)rows * cols;
    int* order = (int*)malloc(n * sizeof(int));
    double* acc = (double*)malloc(n * sizeof(double));
    size_t m = 0;
    for (size_t i = 0; i < n; ++i) {
        lambda[i] = 0.0;
        acc[i] = loss_grad[i];
        if (type[i] >= 0) order[m++] = (int)i;
    }
    g_sort_t = t;
    qsort(order, m, sizeof(int), by_time_desc);
    int nclamp = 0;
    for (size_t k = 0; k < m; ++k) {
        const int i = order[k];
        double diag, j0, j1;
        int cl;
        orc_jacobian_entries(type[i], c0[i], c1[i], c2[i], c3[i], c4[i], &diag, &j0, &j1, &cl);
        nclamp += cl;
        const double lam = acc[i] / diag;
        lambda[i] = lam;
        const int r = i / cols, c = i % cols;
        acc[(r + RING_DR[donor1[i]]) * cols + (c + RING_DC[donor1[i]])] -= j0 * lam;
        if (type[i] == 0) acc[(r + RING_DR[donor2[i]]) * cols + (c + RING_DC[donor2[i]])] -= j1 * lam;
    }
    *clamped = nclamp;
    free(order);
    free(acc);
    return 0;
}

/* param_gradients, src/adjoint.cpp:119-144. */
void orc_param_gradients(int rows, int cols, double h, const int8_t* type, const int8_t* donor1,
                         const int8_t* donor2, const double* c0, const double* c1,
                         const double* c2, const double* c3, const double* c4,
                         const double* lambda, double* d_g11, double* d_g12, double* d_g22,
                         double* d_b1, double* d_b2) {
    const size_t n = (size_t)rows * cols;
    for (size_t i = 0; i < n; ++i) {
        d_g11[i] = d_g12[i] = d_g22[i] = d_b1[i] = d_b2[i] = 0.0;
        if (type[i] < 0) continue;
        const double lam = lambda[i];
        if (lam == 0.0) continue; /* :123 */
        double m1x, m1y;
        disp(donor1[i], h, &m1x, &m1y);
        if (type[i] == 0) {
            double m2x, m2y;
            disp(donor2[i], h, &m2x, &m2y);
            const double qu1 = c0[i] * c3[i] + c1[i] * c4[i];
            const double qu2 = c1[i] * c3[i] + c2[i] * c4[i];
            const double wx = m1x * qu1 + m2x * qu2; /* M Q u */
            const double wy = m1y * qu1 + m2y * qu2;
            d_b1[i] = -lam * 2.0 * wx;
            d_b2[i] = -lam * 2.0 * wy;
            d_g11[i] = lam * wx * wx;
            d_g12[i] = lam * 2.0 * wx * wy;
            d_g22[i] = lam * wy * wy;
        } else {
            d_b1[i] = -lam * 2.0 * c0[i] * m1x;
            d_b2[i] = -lam * 2.0 * c0[i] * m1y;
            d_g11[i] = lam * m1x * m1x;
            d_g12[i] = lam * 2.0 * m1x * m1y;
            d_g22[i] = lam * m1y * m1y;
        }
    }
    (void)rows;
    (void)cols;
}

/* loss_grad_mse, src/adjoint.cpp:146-160. */
void orc_loss_grad_mse(int n, const double* t, const uint8_t* observed, const double* values,
                       double* grad, double* loss, int* unreached) {
    double l = 0.0;
    int u = 0;
    for (int i = 0; i < n; ++i) {
        grad[i] = 0.0;
        if (!observed[i]) continue;
        if (!reached(t[i])) {
            ++u;
            continue;
        }
        const double diff = t[i] - values[i];
        grad[i] = diff;
        l += 0.5 * diff * diff;
    }
    *loss = l;
    *unreached = u;
}

/* ProjectionConfig::validate, feasibility.hpp:15-20. */
static int validate_projection(double eps_min, double lambda_max, double tau) {
    if (!(eps_min > 0.0) || !(eps_min < lambda_max)) return 3;
    if (!(tau > 0.0) || !(tau < 1.0)) return 3;
    return 0;
}

/* project_spd with decompose/recompose, src/feasibility.cpp:15-44 and
 * sym2_eigenvalues mat2.hpp:44-49. */
int orc_project_spd(int n, double* g11, double* g12, double* g22, double eps_min,
                    double lambda_max) {
    const int st = validate_projection(eps_min, lambda_max, 0.95);
    if (st) return st;
    for (int i = 0; i < n; ++i) {
        const double a = g11[i], b = g12[i], c = g22[i];
        const double half_tr = 0.5 * (a + c);
        const double disc = sqrt(0.25 * (a - c) * (a - c) + b * b);
        const double hi = half_tr + disc, lo = half_tr - disc;
        const double theta = 0.5 * atan2(2.0 * b, a - c);
        const double cs = cos(theta), sn = sin(theta);
        if (lo >= eps_min && hi <= lambda_max) continue;
        const double H = sclamp(hi, eps_min, lambda_max);
        const double L = sclamp(lo, eps_min, lambda_max);
        g11[i] = H * cs * cs + L * sn * sn;
        g12[i] = (H - L) * cs * sn;
        g22[i] = H * sn * sn + L * cs * cs;
    }
    return 0;
}

/* drift_norm_sq, src/feasibility.cpp:46-49. */
double orc_drift_norm_sq(double b1, double b2, double g11, double g12, double g22) {
    const double det = g11 * g22 - g12 * g12;
    return (b1 * b1 * g22 - 2.0 * b1 * b2 * g12 + b2 * b2 * g11) / det;
}

/* project_drift, src/feasibility.cpp:51-72. */
int orc_project_drift(int n, double* b1, double* b2, const double* g11, const double* g12,
                      const double* g22, double tau, double euclid_cap) {
    const int st = validate_projection(1e-3, 1e3, tau);
    if (st) return st;
    for (int i = 0; i < n; ++i) {
        double x = b1[i], y = b2[i];
        const double en = sqrt(x * x + y * y);
        if (en > euclid_cap) {
            const double f = euclid_cap / en;
            x *= f;
            y *= f;
        }
        const double gn = sqrt(orc_drift_norm_sq(x, y, g11[i], g12[i], g22[i]));
        if (gn > tau) {
            const double f = tau / gn;
            x *= f;
            y *= f;
        }
        b1[i] = x;
        b2[i] = y;
    }
    return 0;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

int orc_pipeline(int rows, int cols, double h, const double* g11, const double* g12,
                 const double* g22, const double* b1, const double* b2, const uint8_t* src,
                 const uint8_t* observed, const double* values, double tol, int max_iters,
                 double* times, int* iterations, int* records) {
    const size_t n = (size_t)rows * cols;
    double* t = (double*)malloc(n * sizeof(double));
    double* grad = (double*)malloc(n * sizeof(double));
    double* lam = (double*)malloc(n * sizeof(double));
    double* cc = (double*)malloc(5 * n * sizeof(double));
    double* dg = (double*)malloc(5 * n * sizeof(double));
    int8_t* codes = (int8_t*)malloc(4 * n);
    int conv, n2, n1, bad, cl, st;
    double loss;
    int unr;
    double t0 = now_s();
    st = orc_solve(rows, cols, h, g11, g12, g22, b1, b2, src, NULL, 0, tol, max_iters, NULL, t,
                   iterations, &conv, NULL);
    double t1 = now_s();
    if (!st) {
        orc_loss_grad_mse((int)n, t, observed, values, grad, &loss, &unr);
    }
    double t2 = now_s();
    if (!st)
        st = orc_identify(rows, cols, h, t, g11, g12, g22, b1, b2, src, tol, codes, codes + n,
                          codes + 2 * n, codes + 3 * n, cc, cc + n, cc + 2 * n, cc + 3 * n,
                          cc + 4 * n, &n2, &n1, &bad);
    double t3 = now_s();
    if (!st)
        orc_adjoint(rows, cols, t, codes, codes + 2 * n, codes + 3 * n, cc, cc + n, cc + 2 * n,
                    cc + 3 * n, cc + 4 * n, grad, lam, &cl);
    double t4 = now_s();
    if (!st)
        orc_param_gradients(rows, cols, h, codes, codes + 2 * n, codes + 3 * n, cc, cc + n,
                            cc + 2 * n, cc + 3 * n, cc + 4 * n, lam, dg, dg + n, dg + 2 * n,
                            dg + 3 * n, dg + 4 * n);
    double t5 = now_s();
    times[0] = t1 - t0;
    times[1] = t2 - t1;
    times[2] = t3 - t2;
    times[3] = t4 - t3;
    times[4] = t5 - t4;
    *records = st ? 0 : n2 + n1;
    free(t);
    free(grad);
    free(lam);
    free(cc);
    free(dg);
    free(codes);
    return st;
}
