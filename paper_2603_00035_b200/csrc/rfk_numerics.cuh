// rfk_numerics.cuh — bit-exact device arithmetic of the Randers local update.
//
// Every function replays the reference's operation order exactly
// (include/randers/mat2.hpp:14-35, src/stencil.cpp:7-43,
// include/randers/stencil.hpp:43-45, src/sweeper.cpp:8-61).  The whole
// library is compiled with --fmad=false: no a*b+c is ever contracted into an
// FMA, so each * and + rounds exactly like the reference's SSE2 build.  fp64
// '/' and sqrt are IEEE correctly rounded on the device, as on the host.
//
// Evaluation layout: one node is evaluated by an aligned group of 8 lanes;
// lane k owns triangular stencil k (neighbours k and (k+1)%8) and its two
// one-point fallbacks, so the 8 stencils run concurrently and the
// sequential "first-found, strictly smaller wins" fold of best_candidate
// becomes an order-preserving 3-level shuffle reduction.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rfk {

constexpr int RFK_TWO_POINT_T = 0;  // UpdateType::TwoPoint (sweeper.hpp:14)
constexpr int RFK_ONE_POINT_T = 1;  // UpdateType::OnePoint
constexpr double kUnreached = 1e10;          // grid.hpp:14
constexpr double kUnreachedThreshold = 1e9;  // grid.hpp:15

__device__ __forceinline__ bool reached(double t) { return t < kUnreachedThreshold; }

// Moore ring (stencil.hpp:17-18): UL, W, LL, S, LR, E, UR, N.
__device__ __forceinline__ int ring_dr(int k) { return (k == 0 || k >= 6) ? -1 : (k == 1 || k == 5) ? 0 : 1; }
__device__ __forceinline__ int ring_dc(int k) { return (k <= 2) ? -1 : (k == 3 || k == 7) ? 0 : 1; }

// libstdc++ std::max / std::min / std::clamp semantics (NaN-sensitive).
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }

// All arithmetic goes through these so no compiler transformation can fuse
// or reorder (belt and braces on top of --fmad=false).
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

struct Metric {
    double g11, g12, g22, b1, b2;
};

// StencilTable::displacement (stencil.hpp:24): (dc*h, dr*h), int*double.
__device__ __forceinline__ void displacement(int k, double h, double& x, double& y) {
    x = mul(static_cast<double>(ring_dc(k)), h);
    y = mul(static_cast<double>(ring_dr(k)), h);
}

// Vec2::dot (mat2.hpp:17), Sym2::mul (:32), Sym2::quad (:33).
__device__ __forceinline__ double dot2(double ax, double ay, double bx, double by) {
    return add(mul(ax, bx), mul(ay, by));
}
__device__ __forceinline__ void gmul(const Metric& g, double vx, double vy, double& ox, double& oy) {
    ox = add(mul(g.g11, vx), mul(g.g12, vy));
    oy = add(mul(g.g12, vx), mul(g.g22, vy));
}
__device__ __forceinline__ double quad(const Metric& g, double vx, double vy) {
    double gx, gy;
    gmul(g, vx, vy, gx, gy);
    return dot2(vx, vy, gx, gy);
}

struct TwoPoint {
    double t0, lam1, lam2;
    bool valid;
};

// two_point_update, src/stencil.cpp:7-43, operation for operation.
__device__ __forceinline__ TwoPoint two_point_update(double t1, double t2, double m1x, double m1y,
                                                     double m2x, double m2y, const Metric& g) {
    TwoPoint res{0.0, 0.0, 0.0, false};
    double gm1x, gm1y;
    gmul(g, m1x, m1y, gm1x, gm1y);
    const double e11 = dot2(m1x, m1y, gm1x, gm1y);
    const double e12 = dot2(m2x, m2y, gm1x, gm1y);
    const double e22 = quad(g, m2x, m2y);
    const double det = sub(mul(e11, e22), mul(e12, e12));
    if (!(det > mul(1e-14, smax(mul(e11, e22), mul(e12, e12))))) return res;  // :17-18
    const double q11 = e22 / det;
    const double q12 = -e12 / det;
    const double q22 = e11 / det;
    const double s1 = add(t1, dot2(m1x, m1y, g.b1, g.b2));
    const double s2 = add(t2, dot2(m2x, m2y, g.b1, g.b2));
    const double a = add(add(q11, mul(2.0, q12)), q22);
    const double bq = add(mul(add(q11, q12), s1), mul(add(q12, q22), s2));
    const double c = sub(add(add(mul(mul(q11, s1), s1), mul(mul(mul(2.0, q12), s1), s2)),
                             mul(mul(q22, s2), s2)),
                         1.0);
    const double disc = sub(mul(bq, bq), mul(a, c));
    if (disc < 0.0 || a <= 0.0) return res;  // :32-33
    const double t0 = add(bq, sqrt(disc)) / a;
    const double d1 = sub(t0, s1);
    const double d2 = sub(t0, s2);
    res.t0 = t0;
    res.lam1 = add(mul(q11, d1), mul(q12, d2));
    res.lam2 = add(mul(q12, d1), mul(q22, d2));
    res.valid = t0 > smax(t1, t2) && res.lam1 >= 0.0 && res.lam2 >= 0.0;  // :41
    return res;
}

// one_point_update, stencil.hpp:43-45: (ti + mi.b) + sqrt(mi'G mi).
__device__ __forceinline__ double one_point_update(double ti, double mx, double my, const Metric& g) {
    return add(add(ti, dot2(mx, my, g.b1, g.b2)), sqrt(quad(g, mx, my)));
}

// ---------------------------------------------------------------------------
// Per-lane candidate of stencil k, folded in the reference's enumeration
// order (sweeper.cpp:37-59): the valid two-point update of stencil k if any,
// otherwise the one-point updates from donor k then donor k2.
//
// Summary kept for the cross-lane fold:
//   found      any candidate found
//   first_nan  the first found candidate (in order) is NaN
//   best       minimum over non-NaN candidates, earliest on ties
//              (+inf when none) — with `which` = 0 two-point, 1 one-point k,
//              2 one-point k2 identifying it.
// The sequential fold "take if !found || t0 < best" (two-point) and
// "skip if found && !(t0 < best)" (one-point) equals: NaN if the first found
// candidate is NaN, else the earliest argmin over non-NaN candidates.
struct LaneCand {
    double best;
    double lam1, lam2;
    int which;
    int first_which;  // which of the first found candidate (for the NaN case)
    bool found, first_nan;
};

__device__ __forceinline__ void lane_take(LaneCand& lc, double t0, int which) {
    const bool nan = t0 != t0;
    if (!lc.found) {
        lc.found = true;
        lc.first_nan = nan;
        lc.first_which = which;
    }
    if (!nan && t0 < lc.best) {
        lc.best = t0;
        lc.which = which;
    }
}

// tk, tk2: neighbour values (out of bounds == unreached, which the reference
// treats identically: both need in[] && reached, sweeper.cpp:39,109).
template <bool kWantLambda>
__device__ __forceinline__ LaneCand lane_candidate(int k, double tk, double tk2, const Metric& g,
                                                   double h) {
    LaneCand lc;
    lc.best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    lc.lam1 = lc.lam2 = 0.0;
    lc.which = lc.first_which = -1;
    lc.found = lc.first_nan = false;
    const int k2 = (k + 1) & 7;
    const bool r1 = reached(tk), r2 = reached(tk2);
    double m1x, m1y, m2x, m2y;
    displacement(k, h, m1x, m1y);
    displacement(k2, h, m2x, m2y);
    if (r1 && r2) {
        const TwoPoint tp = two_point_update(tk, tk2, m1x, m1y, m2x, m2y, g);
        if (tp.valid) {
            lc.found = true;
            lc.best = tp.t0;  // valid => t0 > max(t1,t2): never NaN
            lc.which = lc.first_which = 0;
            if (kWantLambda) {
                lc.lam1 = tp.lam1;
                lc.lam2 = tp.lam2;
            }
            return lc;
        }
    }
    if (r1) lane_take(lc, one_point_update(tk, m1x, m1y, g), 1);
    if (r2) lane_take(lc, one_point_update(tk2, m2x, m2y, g), 2);
    return lc;
}

// Order-preserving reduction across the aligned 8-lane group.  Returns, in
// every lane of the group: found, the winning value (NaN when the first found
// candidate is NaN) and the winning candidate id (lane*4 + which) when
// found and not NaN.
struct GroupResult {
    double t0;
    int id;  // lane*4 + which, -1 if none
    bool found;
};

__device__ __forceinline__ GroupResult group_reduce(const LaneCand& lc) {
    const unsigned lane = threadIdx.x & 31u;
    const unsigned gbase = lane & ~7u;
    const unsigned fmask = (__ballot_sync(0xffffffffu, lc.found) >> gbase) & 0xffu;
    const unsigned nmask = (__ballot_sync(0xffffffffu, lc.first_nan) >> gbase) & 0xffu;
    double v = lc.best;
    int id = lc.which < 0 ? -1 : static_cast<int>((lane & 7u) * 4u + lc.which);
#pragma unroll
    for (int off = 1; off < 8; off <<= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, off);
        const int oid = __shfl_xor_sync(0xffffffffu, id, off);
        // lower lane = earlier in enumeration order; take later only if strictly smaller
        const bool i_am_lower = (lane & off) == 0;
        const double lo_v = i_am_lower ? v : ov, hi_v = i_am_lower ? ov : v;
        const int lo_id = i_am_lower ? id : oid, hi_id = i_am_lower ? oid : id;
        const bool take_hi = hi_v < lo_v;
        v = take_hi ? hi_v : lo_v;
        id = take_hi ? hi_id : lo_id;
    }
    const int first_lane = fmask ? __ffs(fmask) - 1 : 0;
    const int first_which = __shfl_sync(0xffffffffu, lc.first_which, gbase + first_lane);
    GroupResult r;
    r.found = fmask != 0u;
    if (r.found && ((nmask >> first_lane) & 1u)) {
        // The first found candidate is NaN: the sequential fold keeps it.
        r.t0 = __longlong_as_double(0x7ff8000000000000ll);
        r.id = first_lane * 4 + first_which;
    } else {
        r.t0 = v;
        r.id = id;
    }
    return r;
}

}  // namespace rfk
