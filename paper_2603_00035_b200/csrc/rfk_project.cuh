// rfk_project.cuh — the metric-feasibility projections and their VJP as
// per-node device functions, shared by the elementwise projection kernels
// (rfk_project.cu), the projecting hoist of the sweep (rfk_sweep.cu) and the
// projecting parameter-gradient pass of the backward (rfk_backward.cu), so
// the fused and unfused paths run the same operations.
//
// Reference: project_spd with decompose/recompose (src/feasibility.cpp:15-44,
// sym2_eigenvalues mat2.hpp:44-49), drift_norm_sq (:46-49), project_drift
// (:51-72).  project_drift and every pass-through node of project_spd are
// bit-identical to the reference; at nodes that need an eigenvalue clamp the
// recomposition uses the device atan2/cos/sin, which may differ from glibc by
// an ulp.
#pragma once

#include "rfk_numerics.cuh"

namespace rfk {
namespace proj {

__device__ __forceinline__ double sclamp(double v, double lo, double hi) {
    return (v < lo) ? lo : (hi < v) ? hi : v;  // std::clamp
}

// project_spd at one node (feasibility.cpp:15-44); returns false on the
// pass-through branch (:36), where the outputs equal the inputs.
__device__ __forceinline__ bool spd_node(double a, double b, double c, double eps_min, double lambda_max,
                                         double& o11, double& o12, double& o22) {
    const double half_tr = mul(0.5, add(a, c));
    const double amc = sub(a, c);
    const double disc = sqrt(add(mul(mul(0.25, amc), amc), mul(b, b)));
    const double hi = add(half_tr, disc), lo = sub(half_tr, disc);
    o11 = a;
    o12 = b;
    o22 = c;
    if (lo >= eps_min && hi <= lambda_max) return false;
    const double theta = mul(0.5, atan2(mul(2.0, b), amc));
    double sn, cs;
    sincos(theta, &sn, &cs);
    const double H = sclamp(hi, eps_min, lambda_max);
    const double L = sclamp(lo, eps_min, lambda_max);
    o11 = add(mul(mul(H, cs), cs), mul(mul(L, sn), sn));
    o12 = mul(mul(sub(H, L), cs), sn);
    o22 = add(mul(mul(H, sn), sn), mul(mul(L, cs), cs));
    return true;
}

__device__ __forceinline__ double drift_norm_sq(double b1, double b2, double g11, double g12, double g22) {
    const double det = sub(mul(g11, g22), mul(g12, g12));
    return add(sub(mul(mul(b1, b1), g22), mul(mul(mul(2.0, b1), b2), g12)), mul(mul(b2, b2), g11)) / det;
}

// ---- projection VJP (absent in the reference) ----------
//
// The paper's "differentiable projection layers".  The
// cotangents of the three metric channels are (d11, d12, d22) with g12 one
// channel feeding both off-diagonal entries, i.e. the matrix cotangent is
// [[d11, d12/2], [d12/2, d22]].
//
// project_spd = V f(Lambda) V^T with f = clamp(., eps_min, lambda_max):
// Daleckii-Krein, dG = V (F o (V^T Gbar V)) V^T with F_ii = f'(l_i) and
// F_12 = (f(hi) - f(lo)) / (hi - lo) (f'(hi) at a tie).  Pass-through nodes
// (:36) have the identity Jacobian.
__device__ __forceinline__ void spd_vjp_node(double a, double b, double c, double eps_min, double lambda_max, double& d11,
                             double& d12, double& d22) {
    const double half_tr = 0.5 * (a + c);
    const double amc = a - c;
    const double disc = sqrt(0.25 * amc * amc + b * b);
    const double hi = half_tr + disc, lo = half_tr - disc;
    if (lo >= eps_min && hi <= lambda_max) return;  // identity
    const double theta = 0.5 * atan2(2.0 * b, amc);
    double sn, cs;
    sincos(theta, &sn, &cs);
    // eigenvectors: v = (cs, sn) for hi, w = (-sn, cs) for lo
    const double Fh = (hi > eps_min && hi < lambda_max) ? 1.0 : 0.0;
    const double Fl = (lo > eps_min && lo < lambda_max) ? 1.0 : 0.0;
    const double fh = sclamp(hi, eps_min, lambda_max), fl = sclamp(lo, eps_min, lambda_max);
    const double F12 = (hi > lo) ? (fh - fl) / (hi - lo) : Fh;
    // Gbar in the eigenbasis: P = V^T Gbar V
    const double g11 = d11, g12 = 0.5 * d12, g22 = d22;
    const double pvv = cs * cs * g11 + 2.0 * cs * sn * g12 + sn * sn * g22;
    const double pww = sn * sn * g11 - 2.0 * cs * sn * g12 + cs * cs * g22;
    const double pvw = -cs * sn * g11 + (cs * cs - sn * sn) * g12 + cs * sn * g22;
    const double qvv = Fh * pvv, qww = Fl * pww, qvw = F12 * pvw;
    // back to the grid basis: V Q V^T
    const double r11 = cs * cs * qvv - 2.0 * cs * sn * qvw + sn * sn * qww;
    const double r22 = sn * sn * qvv + 2.0 * cs * sn * qvw + cs * cs * qww;
    const double r12 = cs * sn * qvv + (cs * cs - sn * sn) * qvw - cs * sn * qww;
    d11 = r11;
    d12 = 2.0 * r12;
    d22 = r22;
}

// project_drift (feasibility.cpp:51-72): b1 = cap*b/|b| if |b| > cap, then
// b' = tau*b1/n with n = ||b1||_{G^-1} if n > tau.  In: (db1, db2) = d/db';
// out: d/db, and d/dG through n accumulated into (dg11, dg12, dg22).
__device__ __forceinline__ void drift_vjp_node(double x, double y, double g11, double g12, double g22, double tau, double cap,
                               double& dx, double& dy, double& dg11, double& dg12, double& dg22) {
    const double en = sqrt(x * x + y * y);
    double x1 = x, y1 = y, f1 = 1.0;
    const bool c1 = en > cap;
    if (c1) {
        f1 = cap / en;
        x1 = x * f1;
        y1 = y * f1;
    }
    const double det = g11 * g22 - g12 * g12;
    const double mx = (g22 * x1 - g12 * y1) / det, my = (g11 * y1 - g12 * x1) / det;  // G^-1 b1
    const double gn = sqrt(x1 * mx + y1 * my);
    if (gn > tau) {
        const double dot = dx * x1 + dy * y1;
        const double k = tau * dot / (gn * gn * gn);
        // d(n^2)/dG = -(G^-1 b)(G^-1 b)^T; channel g12 feeds both off-diagonals
        dg11 += 0.5 * k * mx * mx;
        dg22 += 0.5 * k * my * my;
        dg12 += k * mx * my;
        const double s = tau / gn;
        dx = s * dx - k * mx;
        dy = s * dy - k * my;
    }
    if (c1) {
        const double dot = (x * dx + y * dy) / (en * en);
        dx = f1 * (dx - x * dot);
        dy = f1 * (dy - y * dot);
    }
}

// project_drift at one node (feasibility.cpp:51-72): Euclidean pre-clip to
// `cap`, then scale to tau if ||b||_{G^-1} > tau.
__device__ __forceinline__ void drift_node(double& x, double& y, double g11, double g12, double g22, double tau,
                                           double cap) {
    const double en = sqrt(add(mul(x, x), mul(y, y)));
    if (en > cap) {
        const double f = cap / en;
        x = mul(x, f);
        y = mul(y, f);
    }
    const double gn = sqrt(drift_norm_sq(x, y, g11, g12, g22));
    if (gn > tau) {
        const double f = tau / gn;
        x = mul(x, f);
        y = mul(y, f);
    }
}

// ParamView::project for mode 1 (project_spd), 2 (project_drift against the
// metric as given) or 3 (both: spd, then drift against the projected metric,
// inversion.cpp:276-279), one node, in place.
__device__ __forceinline__ void project_node(int mode, double eps_min, double lambda_max, double tau, double cap,
                                             double& g11, double& g12, double& g22, double& b1, double& b2) {
    if (mode & 1) {
        double o11, o12, o22;
        if (spd_node(g11, g12, g22, eps_min, lambda_max, o11, o12, o22)) {
            g11 = o11;
            g12 = o12;
            g22 = o22;
        }
    }
    if (mode & 2) drift_node(b1, b2, g11, g12, g22, tau, cap);
}

// The VJP of project_node (the ParamView::project backward): cotangents of
// the projected channels in (d*), of the raw channels out; raw inputs.
__device__ __forceinline__ void project_vjp_node(int mode, double eps_min, double lambda_max, double tau, double cap,
                                                 double a, double b, double c, double x, double y, double& d11,
                                                 double& d12, double& d22, double& dx, double& dy) {
    if (mode & 2) {
        double pa = a, pb = b, pc = c;
        if (mode & 1) spd_node(a, b, c, eps_min, lambda_max, pa, pb, pc);
        drift_vjp_node(x, y, pa, pb, pc, tau, cap, dx, dy, d11, d12, d22);
    }
    if (mode & 1) spd_vjp_node(a, b, c, eps_min, lambda_max, d11, d12, d22);
}

}  // namespace proj
}  // namespace rfk
