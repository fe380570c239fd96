// rfk_backward.cu — implicit-differentiation backward pass on sm_100a.
//
// Reference: identify_stencils / jacobian_entries / solve_adjoint /
// param_gradients / loss_grad_mse (src/adjoint.cpp:10-160), plus the
// per-node helpers best_candidate / node_update / two_point_update
// (src/sweeper.cpp:8-72, src/stencil.cpp:7-43).
//
// Adjoint in gather form.  The reference back-substitutes in the order
// (T desc, node asc), scattering acc[donor] -= J*lambda.  Node i's final
// accumulator is therefore g_i minus the contributions of exactly those
// dependents j (records whose donor is i) that precede i in that order,
// subtracted in that order.  Here every node gathers its <= 8 dependents,
// sorts their contributions by rank and subtracts them in the same order:
// the same floating-point operations, bit for bit, with no fp atomics.
// Scheduling is dataflow over the radix-sorted order: warps take tickets of
// 32 consecutive ranks, each lane waits (acquire) on its dependents' done
// flags, computes lambda and releases its own flag.  Every dependency points
// to a smaller rank held by a running warp, so the schedule cannot deadlock.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cstdint>

#include "rfk_common.cuh"
#include "rfk_internal.h"
#include "rfk_numerics.cuh"
#include "rfk_project.cuh"

namespace rfk {

namespace {

__device__ __forceinline__ LaneCand empty_lane() {
    LaneCand lc;
    lc.best = __longlong_as_double(0x7ff0000000000000ll);
    lc.lam1 = lc.lam2 = 0.0;
    lc.which = lc.first_which = -1;
    lc.found = lc.first_nan = false;
    return lc;
}

// Full NodeCandidate (sweeper.hpp:20-29) of the group's node, valid in every
// lane of the group.
struct FullCand {
    double t0, lam1, lam2;
    int type, stencil, donor1, donor2;
    bool found;
};

__device__ __forceinline__ FullCand group_full_candidate(const LaneCand& lc, const GroupResult& gr) {
    const unsigned gbase = (threadIdx.x & 31u) & ~7u;
    FullCand f;
    f.found = gr.found;
    f.t0 = kUnreached;
    f.lam1 = f.lam2 = 0.0;
    f.type = RFK_ONE_POINT_T;
    f.stencil = f.donor1 = f.donor2 = -1;
    const int id = gr.found ? gr.id : 0;
    const int wl = id >> 2, which = id & 3;
    const double l1 = __shfl_sync(0xffffffffu, lc.lam1, gbase + wl);
    const double l2 = __shfl_sync(0xffffffffu, lc.lam2, gbase + wl);
    if (gr.found && gr.id >= 0) {
        f.t0 = gr.t0;
        f.stencil = wl;
        if (which == 0) {
            f.type = RFK_TWO_POINT_T;
            f.donor1 = wl;
            f.donor2 = (wl + 1) & 7;
            f.lam1 = l1;
            f.lam2 = l2;
        } else {
            f.donor1 = which == 1 ? wl : ((wl + 1) & 7);
        }
    } else if (gr.found) {  // found but only +inf candidates: value without identity
        f.t0 = gr.t0;
    }
    return f;
}

__device__ __forceinline__ LaneCand eval_lane_global(int k, int r, int c, int R, int C, const double* T,
                                                     const Metric& m, double h) {
    const int k2 = (k + 1) & 7;
    const int r1 = r + ring_dr(k), c1 = c + ring_dc(k);
    const int r2 = r + ring_dr(k2), c2 = c + ring_dc(k2);
    const double tk = (r1 >= 0 && r1 < R && c1 >= 0 && c1 < C) ? __ldg(T + static_cast<int64_t>(r1) * C + c1)
                                                               : kUnreached;
    const double tk2 = (r2 >= 0 && r2 < R && c2 >= 0 && c2 < C) ? __ldg(T + static_cast<int64_t>(r2) * C + c2)
                                                                : kUnreached;
    return lane_candidate<true>(k, tk, tk2, m, h);
}

// ---- best_candidate / node_update at a node list ------------------------------
__global__ void __launch_bounds__(256) best_candidate_kernel(CandidateArgs a) {
    const int k = threadIdx.x & 7;
    const int64_t warp = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5) * 4;
    for (int64_t base = warp * 4; base < a.n_nodes; base += stride) {
        const int64_t q = base + ((threadIdx.x >> 3) & 3);
        const bool active = q < a.n_nodes;
        LaneCand lc = empty_lane();
        int node = 0;
        if (active) {
            node = a.nodes[q];
            const int r = node / a.C, c = node % a.C;
            const Metric m{__ldg(a.g11 + node), __ldg(a.g12 + node), __ldg(a.g22 + node),
                           __ldg(a.b1 + node), __ldg(a.b2 + node)};
            lc = eval_lane_global(k, r, c, a.R, a.C, a.T, m, a.h);
        }
        const GroupResult gr = group_reduce(lc);
        FullCand f = group_full_candidate(lc, gr);
        if (active && k == 0) {
            if (a.node_update) {  // sweeper.cpp:63-72
                const double cur = __ldg(a.T + node);
                if (!f.found || !(f.t0 < cur)) {
                    f.found = false;
                    f.t0 = cur;
                    f.type = RFK_ONE_POINT_T;
                    f.stencil = f.donor1 = f.donor2 = -1;
                    f.lam1 = f.lam2 = 0.0;
                }
            }
            a.t0[q] = f.t0;
            a.type[q] = static_cast<int8_t>(f.type);
            a.stencil[q] = static_cast<int8_t>(f.stencil);
            a.donor1[q] = static_cast<int8_t>(f.donor1);
            a.donor2[q] = static_cast<int8_t>(f.donor2);
            a.lam1[q] = f.lam1;
            a.lam2[q] = f.lam2;
            a.found[q] = f.found ? 1 : 0;
        }
    }
}

__global__ void two_point_kernel(TwoPointArgs a) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const Metric m{a.g11[i], a.g12[i], a.g22[i], a.b1[i], a.b2[i]};
        const TwoPoint tp = two_point_update(a.t1[i], a.t2[i], a.m1x[i], a.m1y[i], a.m2x[i], a.m2y[i], m);
        a.t0[i] = tp.t0;
        a.lam1[i] = tp.lam1;
        a.lam2[i] = tp.lam2;
        a.valid[i] = tp.valid ? 1 : 0;
    }
}

// ---- identify_stencils (adjoint.cpp:10-67) -------------------------------------
__global__ void __launch_bounds__(256) identify_kernel(IdentifyArgs a) {
    __shared__ int cnt2[8], cnt1[8];
    const int k = threadIdx.x & 7;
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    const int64_t warp = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5) * 4;
    int my2 = 0, my1 = 0;
    for (int64_t base = warp * 4; base < n; base += stride) {
        const int64_t node = base + ((threadIdx.x >> 3) & 3);
        bool active = node < n;
        double stored = kUnreached;
        Metric m{0, 0, 0, 0, 0};
        int r = 0, c = 0;
        if (active) {
            stored = __ldg(a.T + node);
            active = __ldg(a.src + node) == 0 && reached(stored);
        }
        LaneCand lc = empty_lane();
        if (active) {
            r = static_cast<int>(node / a.C);
            c = static_cast<int>(node % a.C);
            m = Metric{__ldg(a.g11 + node), __ldg(a.g12 + node), __ldg(a.g22 + node), __ldg(a.b1 + node),
                       __ldg(a.b2 + node)};
            lc = eval_lane_global(k, r, c, a.R, a.C, a.T, m, a.h);
        }
        const GroupResult gr = group_reduce(lc);
        const FullCand f = group_full_candidate(lc, gr);
        if (k != 0 || node >= n) continue;
        int8_t ty = -1, st = -1, d1 = -1, d2 = -1;
        double c0 = 0.0, c1v = 0.0, c2 = 0.0, c3 = 0.0, c4 = 0.0;
        if (active) {
            if (!f.found || fabs(f.t0 - stored) > mul(100.0, a.tol)) {  // :22-25
                atomicMin(a.bad_node, static_cast<unsigned long long>(node));
            } else {
                ty = static_cast<int8_t>(f.type);
                st = static_cast<int8_t>(f.stencil);
                d1 = static_cast<int8_t>(f.donor1);
                double m1x, m1y;
                displacement(f.donor1, a.h, m1x, m1y);
                const double td1 = __ldg(a.T + static_cast<int64_t>(r + ring_dr(f.donor1)) * a.C +
                                         (c + ring_dc(f.donor1)));
                if (f.type == RFK_TWO_POINT_T) {  // :34-53
                    d2 = static_cast<int8_t>(f.donor2);
                    double m2x, m2y, gx, gy;
                    displacement(f.donor2, a.h, m2x, m2y);
                    gmul(m, m1x, m1y, gx, gy);
                    const double e11 = dot2(m1x, m1y, gx, gy);
                    const double e12 = dot2(m2x, m2y, gx, gy);
                    const double e22 = quad(m, m2x, m2y);
                    const double det = sub(mul(e11, e22), mul(e12, e12));
                    c0 = e22 / det;
                    c1v = -e12 / det;
                    c2 = e11 / det;
                    const double td2 = __ldg(a.T + static_cast<int64_t>(r + ring_dr(f.donor2)) * a.C +
                                             (c + ring_dc(f.donor2)));
                    const double s1 = add(td1, dot2(m1x, m1y, m.b1, m.b2));
                    const double s2 = add(td2, dot2(m2x, m2y, m.b1, m.b2));
                    c3 = sub(s1, stored);
                    c4 = sub(s2, stored);
                    ++my2;
                } else {  // :54-61
                    c0 = sub(add(td1, dot2(m1x, m1y, m.b1, m.b2)), stored);
                    c1v = quad(m, m1x, m1y);
                    ++my1;
                }
            }
        }
        a.rec.type[node] = ty;
        a.rec.stencil[node] = st;
        a.rec.donor1[node] = d1;
        a.rec.donor2[node] = d2;
        a.rec.c[0][node] = c0;
        a.rec.c[1][node] = c1v;
        a.rec.c[2][node] = c2;
        a.rec.c[3][node] = c3;
        a.rec.c[4][node] = c4;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        my2 += __shfl_xor_sync(0xffffffffu, my2, off);
        my1 += __shfl_xor_sync(0xffffffffu, my1, off);
    }
    if ((threadIdx.x & 31) == 0) {
        cnt2[threadIdx.x >> 5] = my2;
        cnt1[threadIdx.x >> 5] = my1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int s2 = 0, s1 = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            s2 += cnt2[w];
            s1 += cnt1[w];
        }
        if (s2) atomicAdd(a.two_point_count, s2);
        if (s1) atomicAdd(a.one_point_count, s1);
    }
}

// ---- identify_stencils from the hoisted stencil records ----------------------
// The same records as identify_kernel, with each lane's candidate evaluated in
// the sweep's form from the T-independent record of the node (hoist_kernel,
// rfk_sweep.cu: Q = E^-1, sqrt(m'Gm), m.b and RN(1/a) per stencil class):
// no E/det/Q divisions per lane.  The candidate arithmetic is the sweep's
// compute role operation for operation (bit-exact with the reference's
// two_point_update / one_point_update, which the sweep's parity tests pin),
// and a two-point record's Q entries are the record's own (the hoist computes
// them with identify_kernel's expressions).
namespace hid {
constexpr int kRecH = 24;  // doubles per hoisted record (rfk_sweep.cu kRec)
__device__ __forceinline__ bool exp_in(double v, int p) {
    const unsigned e = static_cast<unsigned>(__double_as_longlong(v) >> 52) & 0x7ffu;
    return e - static_cast<unsigned>(1023 - p) < static_cast<unsigned>(2 * p);
}
// rfk_sweep.cu slow_update (the IEEE division and the exact lambda tie test)
__device__ __noinline__ double slow_update(double x, double a, double s1, double s2, double q11, double q12,
                                           double q22) {
    const double t0 = x / a;
    const double d1 = sub(t0, s1), d2 = sub(t0, s2);
    const double a1 = mul(q11, d1), b1 = mul(q12, d2), a2 = mul(q12, d1), b2 = mul(q22, d2);
    const auto ex = [](double v) { return static_cast<unsigned>(__double_as_longlong(v) >> 52) & 0x7ffu; };
    const bool tie_ok = ((a1 != -b1) | (ex(a1) != 0x7ffu)) & ((a2 != -b2) | (ex(a2) != 0x7ffu));
    return tie_ok ? t0 : __longlong_as_double(0x7ff8000000000000ll);
}
__device__ __forceinline__ double flip(double v, bool neg) {
    return neg ? __longlong_as_double(__double_as_longlong(v) ^ static_cast<long long>(0x8000000000000000ull)) : v;
}
// lane k's candidate (lane_candidate's contract) from the node's record
__device__ __forceinline__ LaneCand lane_candidate(int k, double tk, double tk2, const double* __restrict__ rec) {
    LaneCand lc;
    lc.best = __longlong_as_double(0x7ff0000000000000ll);
    lc.lam1 = lc.lam2 = 0.0;
    lc.which = lc.first_which = -1;
    lc.found = lc.first_nan = false;
    const int k2 = (k + 1) & 7, c = k & 3, c2 = k2 & 3;
    const double q11 = __ldg(rec + 3 * c), q12 = __ldg(rec + 3 * c + 1), q22 = __ldg(rec + 3 * c + 2);
    const double sq1 = __ldg(rec + 12 + c), sq2 = __ldg(rec + 12 + c2);
    const double mb1 = flip(__ldg(rec + 16 + c), k >= 4), mb2 = flip(__ldg(rec + 16 + c2), k2 >= 4);
    const bool r1 = reached(tk), r2 = reached(tk2);
    const double s1 = add(tk, mb1), s2 = add(tk2, mb2);
    if (r1 && r2) {
        const double ap = add(add(q11, mul(2.0, q12)), q22);  // stencil.cpp:28
        if (ap > 0.0) {
            const double qa = add(q11, q12), qb = add(q12, q22);
            const double bq = add(mul(qa, s1), mul(qb, s2));
            const double cc = sub(add(add(mul(mul(q11, s1), s1), mul(mul(mul(2.0, q12), s1), s2)), mul(mul(q22, s2), s2)),
                                  1.0);
            const double disc = sub(mul(bq, bq), mul(ap, cc));
            if (!(disc < 0.0)) {
                const double y = __ldg(rec + 20 + c);
                const double x = add(bq, sqrt(disc));
                double t0;
                if (y == 0.0 || !exp_in(x, 900)) {
                    t0 = slow_update(x, ap, s1, s2, q11, q12, q22);
                } else {
                    const double q = mul(x, y);
                    t0 = fma(fma(-ap, q, x), y, q);
                }
                const double d1 = sub(t0, s1), d2 = sub(t0, s2);
                const double a1 = mul(q11, d1), b1 = mul(q12, d2), a2 = mul(q12, d1), b2 = mul(q22, d2);
                if (t0 > smax(tk, tk2) && a1 >= -b1 && a2 >= -b2) {
                    lc.found = true;
                    lc.best = t0;
                    lc.which = lc.first_which = 0;
                    return lc;
                }
            }
        }
    }
    if (r1) lane_take(lc, add(s1, sq1), 1);
    if (r2) lane_take(lc, add(s2, sq2), 2);
    return lc;
}
}  // namespace hid

__global__ void __launch_bounds__(256) identify_hoisted_kernel(IdentifyArgs a, const double* __restrict__ hoisted) {
    __shared__ int cnt2[8], cnt1[8];
    const int k = threadIdx.x & 7;
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    const int64_t warp = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5) * 4;
    int my2 = 0, my1 = 0;
    for (int64_t base = warp * 4; base < n; base += stride) {
        const int64_t node = base + ((threadIdx.x >> 3) & 3);
        bool active = node < n;
        double stored = kUnreached;
        int r = 0, c = 0;
        if (active) {
            stored = __ldg(a.T + node);
            active = __ldg(a.src + node) == 0 && reached(stored);
        }
        LaneCand lc = empty_lane();
        const double* rec = hoisted + node * hid::kRecH;
        if (active) {
            r = static_cast<int>(node / a.C);
            c = static_cast<int>(node % a.C);
            const int k2 = (k + 1) & 7;
            const int r1 = r + ring_dr(k), c1 = c + ring_dc(k), r2 = r + ring_dr(k2), c2 = c + ring_dc(k2);
            const double tk = (r1 >= 0 && r1 < a.R && c1 >= 0 && c1 < a.C)
                                  ? __ldg(a.T + static_cast<int64_t>(r1) * a.C + c1) : kUnreached;
            const double tk2 = (r2 >= 0 && r2 < a.R && c2 >= 0 && c2 < a.C)
                                   ? __ldg(a.T + static_cast<int64_t>(r2) * a.C + c2) : kUnreached;
            lc = hid::lane_candidate(k, tk, tk2, rec);
        }
        const GroupResult gr = group_reduce(lc);
        const FullCand f = group_full_candidate(lc, gr);
        if (k != 0 || node >= n) continue;
        int8_t ty = -1, st = -1, d1 = -1, d2 = -1;
        double c0 = 0.0, c1v = 0.0, c2 = 0.0, c3 = 0.0, c4 = 0.0;
        if (active) {
            if (!f.found || fabs(f.t0 - stored) > mul(100.0, a.tol)) {  // :22-25
                atomicMin(a.bad_node, static_cast<unsigned long long>(node));
            } else {
                ty = static_cast<int8_t>(f.type);
                st = static_cast<int8_t>(f.stencil);
                d1 = static_cast<int8_t>(f.donor1);
                const double td1 = __ldg(a.T + static_cast<int64_t>(r + ring_dr(f.donor1)) * a.C +
                                         (c + ring_dc(f.donor1)));
                const double s1 = add(td1, hid::flip(__ldg(rec + 16 + (f.donor1 & 3)), f.donor1 >= 4));
                if (f.type == RFK_TWO_POINT_T) {  // :34-53: Q = E^-1 of the stencil, from the record
                    d2 = static_cast<int8_t>(f.donor2);
                    const int cl = f.stencil & 3;
                    c0 = __ldg(rec + 3 * cl);
                    c1v = __ldg(rec + 3 * cl + 1);
                    c2 = __ldg(rec + 3 * cl + 2);
                    const double td2 = __ldg(a.T + static_cast<int64_t>(r + ring_dr(f.donor2)) * a.C +
                                             (c + ring_dc(f.donor2)));
                    const double s2 = add(td2, hid::flip(__ldg(rec + 16 + (f.donor2 & 3)), f.donor2 >= 4));
                    c3 = sub(s1, stored);
                    c4 = sub(s2, stored);
                    ++my2;
                } else {  // :54-61
                    double m1x, m1y;
                    displacement(f.donor1, a.h, m1x, m1y);
                    const Metric m{__ldg(a.g11 + node), __ldg(a.g12 + node), __ldg(a.g22 + node), 0.0, 0.0};
                    c0 = sub(s1, stored);
                    c1v = quad(m, m1x, m1y);
                    ++my1;
                }
            }
        }
        a.rec.type[node] = ty;
        a.rec.stencil[node] = st;
        a.rec.donor1[node] = d1;
        a.rec.donor2[node] = d2;
        a.rec.c[0][node] = c0;
        a.rec.c[1][node] = c1v;
        a.rec.c[2][node] = c2;
        a.rec.c[3][node] = c3;
        a.rec.c[4][node] = c4;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        my2 += __shfl_xor_sync(0xffffffffu, my2, off);
        my1 += __shfl_xor_sync(0xffffffffu, my1, off);
    }
    if ((threadIdx.x & 31) == 0) {
        cnt2[threadIdx.x >> 5] = my2;
        cnt1[threadIdx.x >> 5] = my1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int s2 = 0, s1 = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            s2 += cnt2[w];
            s1 += cnt1[w];
        }
        if (s2) atomicAdd(a.two_point_count, s2);
        if (s1) atomicAdd(a.one_point_count, s1);
    }
}

// ---- jacobian_entries (adjoint.cpp:69-89) --------------------------------------
struct Jac {
    double diag, j0, j1;
    bool clamped;
};

__device__ __forceinline__ Jac jacobian_entries(int type, double c0, double c1, double c2, double c3,
                                                double c4) {
    Jac o;
    if (type == RFK_TWO_POINT_T) {
        const double qu1 = add(mul(c0, c3), mul(c1, c4));
        const double qu2 = add(mul(c1, c3), mul(c2, c4));
        o.diag = mul(-2.0, add(qu1, qu2));
        o.j0 = mul(2.0, qu1);
        o.j1 = mul(2.0, qu2);
    } else {
        o.diag = mul(-2.0, c0);
        o.j0 = mul(2.0, c0);
        o.j1 = 0.0;
    }
    const double scale = smax(add(fabs(o.j0), fabs(o.j1)), 1.0);
    const double fl = mul(1e-12, scale);
    o.clamped = false;
    if (fabs(o.diag) < fl) {
        o.diag = copysign(fl, o.diag == 0.0 ? 1.0 : o.diag);
        o.clamped = true;
    }
    return o;
}

__global__ void jacobian_kernel(JacobianArgs a) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const Jac j = jacobian_entries(a.type[i], a.c[0][i], a.c[1][i], a.c[2][i], a.c[3][i], a.c[4][i]);
        a.diag[i] = j.diag;
        a.j0[i] = j.j0;
        a.j1[i] = j.j1;
        a.clamped[i] = j.clamped ? 1 : 0;
    }
}

// ---- param_gradients (adjoint.cpp:119-144), one node --------------------------
__device__ __forceinline__ void node_param_grads(int type, int dn1, int dn2, double c0, double c1,
                                                 double c2, double c3, double c4, double lam, double h,
                                                 double& g11, double& g12, double& g22, double& b1,
                                                 double& b2) {
    g11 = g12 = g22 = b1 = b2 = 0.0;
    if (lam == 0.0) return;  // :123
    double m1x, m1y;
    displacement(dn1, h, m1x, m1y);
    if (type == RFK_TWO_POINT_T) {
        double m2x, m2y;
        displacement(dn2, h, m2x, m2y);
        const double qu1 = add(mul(c0, c3), mul(c1, c4));
        const double qu2 = add(mul(c1, c3), mul(c2, c4));
        const double wx = add(mul(m1x, qu1), mul(m2x, qu2));
        const double wy = add(mul(m1y, qu1), mul(m2y, qu2));
        b1 = mul(mul(-lam, 2.0), wx);
        b2 = mul(mul(-lam, 2.0), wy);
        g11 = mul(mul(lam, wx), wx);
        g12 = mul(mul(mul(lam, 2.0), wx), wy);
        g22 = mul(mul(lam, wy), wy);
    } else {
        b1 = mul(mul(mul(-lam, 2.0), c0), m1x);
        b2 = mul(mul(mul(-lam, 2.0), c0), m1y);
        g11 = mul(mul(lam, m1x), m1x);
        g12 = mul(mul(mul(lam, 2.0), m1x), m1y);
        g22 = mul(mul(lam, m1y), m1y);
    }
}

__global__ void param_grad_kernel(ParamGradArgs a) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double g11 = 0, g12 = 0, g22 = 0, b1 = 0, b2 = 0;
        const int ty = a.rec.type[i];
        if (ty >= 0)
            node_param_grads(ty, a.rec.donor1[i], a.rec.donor2[i], a.rec.c[0][i], a.rec.c[1][i],
                             a.rec.c[2][i], a.rec.c[3][i], a.rec.c[4][i], a.lambda[i], a.h, g11, g12,
                             g22, b1, b2);
        a.d_g11[i] = g11;
        a.d_g12[i] = g12;
        a.d_g22[i] = g22;
        a.d_b1[i] = b1;
        a.d_b2[i] = b2;
    }
}

// ---- adjoint -------------------------------------------------------------------
// Orderable key: descending T, ties broken by the (stable) index order.
__device__ __forceinline__ unsigned long long desc_key(double t) {
    if (t == 0.0) t = 0.0;  // -0.0 ties +0.0 in the reference's comparator
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(t));
    const unsigned long long ord = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
    return ~ord;
}

__global__ void adjoint_prepare_kernel(AdjointArgs a) {
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    int cl = 0, nr = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int ty = a.rec.type[i];
        unsigned long long key = ~0ull;
        if (ty >= 0) {
            const Jac j = jacobian_entries(ty, a.rec.c[0][i], a.rec.c[1][i], a.rec.c[2][i], a.rec.c[3][i],
                                           a.rec.c[4][i]);
            a.diag[i] = j.diag;
            a.j0[i] = j.j0;
            a.j1[i] = j.j1;
            cl += j.clamped ? 1 : 0;
            ++nr;
            key = desc_key(a.T[i]);
            if (key == ~0ull) key = ~0ull - 1;
        }
        if (!a.order_src) {
            a.keys[i] = key;
            a.order[i] = static_cast<int32_t>(i);
        }
        a.lambda[i] = 0.0;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        cl += __shfl_xor_sync(0xffffffffu, cl, off);
        nr += __shfl_xor_sync(0xffffffffu, nr, off);
    }
    if ((threadIdx.x & 31) == 0) {
        if (cl) atomicAdd(a.clamped, cl);
        if (nr) atomicAdd(a.nrec, nr);
    }
}

// Split mode: the sort keys from T and the source mask (identify's "active"
// predicate, identify_kernel), the same keys prepare derives from the records
// when identification succeeds.
__global__ void adjoint_keys_kernel(const double* __restrict__ T, const uint8_t* __restrict__ src, int64_t n,
                                    unsigned long long* keys, int32_t* order) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double t = __ldg(T + i);
        unsigned long long key = ~0ull;
        if (__ldg(src + i) == 0 && reached(t)) {
            key = desc_key(t);
            if (key == ~0ull) key = ~0ull - 1;
        }
        keys[i] = key;
        order[i] = static_cast<int32_t>(i);
    }
}

__global__ void rank_kernel(const int32_t* sorted, int32_t* rank, int64_t n) {
    for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x)
        rank[sorted[p]] = static_cast<int32_t>(p);
}

// lambda hand-off word pair: {tag | lo32, tag | hi32}, tag = epoch << 32,
// written by one 16-byte store, so a single 16-byte load both detects
// completion and returns the value (no separate flag round trip).
__device__ __forceinline__ void ll_put(unsigned long long* slot, unsigned epoch, double v) {
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
    const unsigned long long tag = static_cast<unsigned long long>(epoch) << 32;
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(slot), "l"(tag | (bits & 0xffffffffull)),
                 "l"(tag | (bits >> 32))
                 : "memory");
}

// Gather preparation, fully parallel in rank order: the record of rank p
// (node i = sorted[p]) collects its dependents (the records that use i as a
// donor and precede it in the reference's order, adjoint.cpp:106-115),
// sorted by that order, and writes them at p so the dataflow reads them
// coalesced.  Walking ranks rather than nodes makes every store coalesced;
// the neighbourhood loads it scatters instead stay local (consecutive ranks
// lie along one arrival-time front).
__global__ void adjoint_gather_prep_kernel(AdjointArgs a, const int32_t* sorted) {
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    if (a.bad && *a.bad != ~0ull) return;  // identification failed: the call fails
    const int64_t nrec = *a.nrec;
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < nrec;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = sorted[q];
        const int p = static_cast<int>(q);
        const int r = i / a.C, c = i % a.C;
        // the 8 candidate dependents, in registers (fully unrolled, constant indices)
        bool ok[8];
        int jn[8], rk[8];
        double co[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            ok[k] = false;
            jn[k] = 0;
            rk[k] = 0;
            co[k] = 0.0;
            const int nr = r + ring_dr(k), nc = c + ring_dc(k);
            if (nr < 0 || nr >= a.R || nc < 0 || nc >= a.C) continue;
            const int j = nr * a.C + nc;
            const int tj = a.rec.type[j];
            if (tj < 0) continue;
            const int opp = (k + 4) & 7;
            double coef;
            if (a.rec.donor1[j] == opp) coef = a.j0[j];
            else if (tj == RFK_TWO_POINT_T && a.rec.donor2[j] == opp) coef = a.j1[j];
            else continue;
            const int rj = a.rank[j];
            if (rj > p) continue;  // processed after i in the reference: no contribution
            ok[k] = true;
            jn[k] = j;
            rk[k] = rj;
            co[k] = coef;
        }
        // slot of each dependent = its position in the reference's processing
        // order (ranks are distinct: a permutation)
        const int64_t nn = n;
        int cnt = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (!ok[k]) continue;
            ++cnt;
            int pos = 0;
#pragma unroll
            for (int m = 0; m < 8; ++m) pos += (ok[m] && rk[m] < rk[k]) ? 1 : 0;
            a.dep_j[pos * nn + p] = jn[k];
            a.dep_c[pos * nn + p] = co[k];
        }
        a.dep_n[p] = static_cast<int8_t>(cnt);
        a.self_g[p] = a.loss_grad[i];
        a.self_d[p] = a.diag[i];
    }
}

// The back-substitution as a dataflow over ranks: warps take tickets of 32
// consecutive ranks; a node waits for all of its dependents' lambdas at once
// (one 16-byte epoch-tagged word each: value and completion in one load),
// subtracts them in the reference's order, divides by the diagonal and
// publishes its own lambda.
#ifndef RFK_DF_SLEEP
#define RFK_DF_SLEEP 0  // ns between unsuccessful poll rounds of the dataflow adjoint (0: spin)
#endif
template <bool FUSED>
__global__ void __launch_bounds__(256) adjoint_dataflow_kernel(AdjointArgs a, const int32_t* sorted) {
    const int lane = threadIdx.x & 31;
    if (a.bad && *a.bad != ~0ull) return;  // identification failed: the call fails
    const long long nrec = *a.nrec;
    const int64_t nn = static_cast<int64_t>(a.R) * a.C;
    while (true) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(a.ticket, 32ull);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= static_cast<unsigned long long>(nrec)) break;
        const long long p = static_cast<long long>(base) + lane;
        if (p >= nrec) continue;
        const int i = sorted[p];
        int jn_[8], cnt;
        double co[8], v[8], g, dg;
        if constexpr (FUSED) {
            // The node's dependents (records whose donor is i, processed before it
            // in the reference's order), found here instead of by a separate gather
            // pass: the loads overlap the wait for the dependents' lambdas.  Sorted
            // by rank with a fixed 8-element network (register arrays, constant
            // indices), so the subtraction below runs in the reference's order.
            int rk_[8];
            {
                const int r = i / a.C, c = i % a.C;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    jn_[k] = 0;
                    rk_[k] = 0x7fffffff;
                    co[k] = 0.0;
                    const int nr = r + ring_dr(k), nc = c + ring_dc(k);
                    if (nr < 0 || nr >= a.R || nc < 0 || nc >= a.C) continue;
                    const int j = nr * a.C + nc;
                    const int tj = a.rec.type[j];
                    if (tj < 0) continue;
                    const int opp = (k + 4) & 7;
                    double coef;
                    if (a.rec.donor1[j] == opp) coef = a.j0[j];
                    else if (tj == RFK_TWO_POINT_T && a.rec.donor2[j] == opp) coef = a.j1[j];
                    else continue;
                    const int rj = a.rank[j];
                    if (rj > p) continue;  // processed after i in the reference: no contribution
                    jn_[k] = j;
                    rk_[k] = rj;
                    co[k] = coef;
                }
                // Batcher's odd-even merge sort of 8 (19 compare-exchanges), by rank
                auto cx = [&](int x, int y) {
                    const bool sw = rk_[y] < rk_[x];
                    const int r0 = rk_[x], j0 = jn_[x];
                    const double c0 = co[x];
                    rk_[x] = sw ? rk_[y] : r0;
                    jn_[x] = sw ? jn_[y] : j0;
                    co[x] = sw ? co[y] : c0;
                    rk_[y] = sw ? r0 : rk_[y];
                    jn_[y] = sw ? j0 : jn_[y];
                    co[y] = sw ? c0 : co[y];
                };
                cx(0, 1); cx(2, 3); cx(4, 5); cx(6, 7);
                cx(0, 2); cx(1, 3); cx(4, 6); cx(5, 7);
                cx(1, 2); cx(5, 6);
                cx(0, 4); cx(1, 5); cx(2, 6); cx(3, 7);
                cx(2, 4); cx(3, 5);
                cx(1, 2); cx(3, 4); cx(5, 6);
            }
            cnt = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) cnt += rk_[k] != 0x7fffffff ? 1 : 0;
            g = a.loss_grad[i];
            dg = a.diag[i];
        } else {
            cnt = a.dep_n[p];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q < cnt) {
                    jn_[q] = a.dep_j[q * nn + p];
                    co[q] = a.dep_c[q * nn + p];
                }
            }
            g = a.self_g[p];
            dg = a.self_d[p];
        }
        unsigned pending = (1u << cnt) - 1u;
        // One poll round = one L2 round trip: every pending dependent's word is
        // loaded by a predicated load (no branch between the loads, so they
        // issue back to back), then all are tested.
        const unsigned long long* slot[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) slot[q] = a.ll + 2 * static_cast<size_t>(q < cnt ? jn_[q] : 0);
        while (pending) {
            // all loads first, each into its own registers (uninitialised
            // outputs of predicated loads: no zeroing that would make the
            // register allocator recycle one set and serialise the round)
            unsigned long long w0[8], w1[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.u32 p, %3, 0;\n"
                    " @p ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n}\n"
                    : "=l"(w0[q]), "=l"(w1[q])
                    : "l"(slot[q]), "r"((pending >> q) & 1u));
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const bool got = ((pending >> q) & 1u) && static_cast<unsigned>(w0[q] >> 32) == a.epoch &&
                                 static_cast<unsigned>(w1[q] >> 32) == a.epoch;
                if (got) {
                    v[q] = mul(co[q], __longlong_as_double(static_cast<long long>((w1[q] << 32) |
                                                                                   (w0[q] & 0xffffffffull))));
                    pending &= ~(1u << q);
                }
            }
#if RFK_DF_SLEEP
            if (pending) __nanosleep(RFK_DF_SLEEP);  // back off: waiting lanes poll L2 less often
#endif
        }

        double acc = g;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (q < cnt) acc = sub(acc, v[q]);
        const double lam = acc / dg;
        ll_put(a.ll + 2 * static_cast<size_t>(i), a.epoch, lam);
        st_l2(a.lambda + i, lam);
    }
}

// param_gradients fused into the backward as a parallel pass over nodes
// (adjoint.cpp:119-144).
__global__ void adjoint_param_grad_kernel(AdjointArgs a) {
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double g11 = 0.0, g12 = 0.0, g22 = 0.0, b1 = 0.0, b2 = 0.0;
        const int ty = a.rec.type[i];
        if (ty >= 0)
            node_param_grads(ty, a.rec.donor1[i], a.rec.donor2[i], a.rec.c[0][i], a.rec.c[1][i], a.rec.c[2][i],
                             a.rec.c[3][i], a.rec.c[4][i], a.lambda[i], a.h, g11, g12, g22, b1, b2);
        if (a.proj.mode)  // the projection's VJP, fused into the gradient pass (rfk_project.cuh)
            proj::project_vjp_node(a.proj.mode, a.proj.eps_min, a.proj.lambda_max, a.proj.tau, a.proj.cap,
                                   a.raw[0][i], a.raw[1][i], a.raw[2][i], a.raw[3][i], a.raw[4][i], g11, g12, g22,
                                   b1, b2);
        a.d_g11[i] = g11;
        a.d_g12[i] = g12;
        a.d_g22[i] = g22;
        a.d_b1[i] = b1;
        a.d_b2[i] = b2;
    }
}

// ---- loss_grad_mse (adjoint.cpp:146-160) --------------------------------------
__global__ void loss_grad_kernel(LossArgs a) {
    __shared__ double sh[256];
    __shared__ int shu[256];
    double part = 0.0;
    int unr = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double g = 0.0;
        if (a.observed[i]) {
            const double t = a.T[i];
            if (!reached(t)) {
                ++unr;
            } else {
                const double diff = sub(t, a.values[i]);
                g = diff;
                part = add(part, mul(mul(0.5, diff), diff));
            }
        }
        a.grad[i] = g;
    }
    sh[threadIdx.x] = part;
    shu[threadIdx.x] = unr;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            sh[threadIdx.x] = add(sh[threadIdx.x], sh[threadIdx.x + s]);
            shu[threadIdx.x] += shu[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.partial[blockIdx.x] = sh[0];
        if (shu[0]) atomicAdd(a.unreached, shu[0]);
    }
}

__global__ void loss_final_kernel(LossArgs a, int nparts) {
    __shared__ double sh[1024];
    double v = 0.0;
    if (threadIdx.x < nparts) v = a.partial[threadIdx.x];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = add(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *a.loss = sh[0];
}

// Sequential sums in node order, bit-identical to the reference's loops
// (adjoint.cpp:146-160 loss, inversion.cpp:42-47 unreached penalty).  One
// block: warps 1..7 stage the next chunk's terms in shared memory while thread
// 0 adds the current chunk in order.  Nodes that contribute nothing add +0.0,
// an identity here: every partial sum is >= +0.
constexpr int kSeqChunk = 2048;
template <class Term>
__device__ void seq_sum_block(int64_t n, double init, Term term, double* out) {
    __shared__ double buf[2][kSeqChunk];
    const int64_t nchunks = (n + kSeqChunk - 1) / kSeqChunk;
    for (int e = threadIdx.x; e < kSeqChunk; e += blockDim.x) buf[0][e] = e < n ? term(e) : 0.0;
    __syncthreads();
    double acc = init;
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        if (threadIdx.x == 0) {
            const double* cur = buf[ch & 1];
            const int cnt = static_cast<int>(n - ch * kSeqChunk < kSeqChunk ? n - ch * kSeqChunk : kSeqChunk);
            for (int e = 0; e < cnt; ++e) acc = add(acc, cur[e]);
        } else if (threadIdx.x >= 32 && ch + 1 < nchunks) {
            const int64_t base = (ch + 1) * kSeqChunk;
            double* dst = buf[(ch + 1) & 1];
            for (int e = threadIdx.x - 32; e < kSeqChunk; e += blockDim.x - 32)
                dst[e] = base + e < n ? term(base + e) : 0.0;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = acc;
}

__global__ void __launch_bounds__(256) loss_exact_kernel(LossArgs a) {
    seq_sum_block(
        a.n, 0.0,
        [&](int64_t i) {
            if (!a.observed[i]) return 0.0;
            const double t = a.T[i];
            if (!reached(t)) return 0.0;
            const double diff = sub(t, a.values[i]);
            return mul(mul(0.5, diff), diff);
        },
        a.loss);
}

__global__ void __launch_bounds__(256) unreached_penalty_kernel(int64_t n, const double* T, const uint8_t* observed,
                                                                const double* values, double cap, double* acc) {
    const double init = *acc;
    __syncthreads();  // every thread has read *acc before thread 0 overwrites it
    seq_sum_block(
        n, init,
        [&](int64_t i) {
            if (!observed[i] || reached(T[i])) return 0.0;
            const double d = sub(cap, values[i]);
            return mul(mul(0.5, d), d);
        },
        acc);
}

__global__ void accumulate5_kernel(int64_t n, double* a0, double* a1, double* a2, double* a3, double* a4,
                                   const double* b0, const double* b1, const double* b2, const double* b3,
                                   const double* b4) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        a0[i] = add(a0[i], b0[i]);
        a1[i] = add(a1[i], b1[i]);
        a2[i] = add(a2[i], b2[i]);
        a3[i] = add(a3[i], b3[i]);
        a4[i] = add(a4[i], b4[i]);
    }
}

int grid_for(int64_t n, int threads, int cap = 8192) {
    int64_t g = (n + threads - 1) / threads;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return static_cast<int>(g);
}

}  // namespace

cudaError_t launch_best_candidate(const CandidateArgs& a, cudaStream_t stream) {
    best_candidate_kernel<<<grid_for((a.n_nodes + 3) / 4 * 32, 256), 256, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_two_point(const TwoPointArgs& a, cudaStream_t stream) {
    two_point_kernel<<<grid_for(a.n, 256), 256, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_identify(const IdentifyArgs& a, cudaStream_t stream) {
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    identify_kernel<<<grid_for((n + 3) / 4 * 32, 256, 148 * 16), 256, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_identify_hoisted(const IdentifyArgs& a, const double* hoisted, cudaStream_t stream) {
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    identify_hoisted_kernel<<<grid_for((n + 3) / 4 * 32, 256, 148 * 16), 256, 0, stream>>>(a, hoisted);
    return cudaGetLastError();
}

cudaError_t launch_jacobian(const JacobianArgs& a, cudaStream_t stream) {
    jacobian_kernel<<<grid_for(a.n, 256), 256, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_param_gradients(const ParamGradArgs& a, cudaStream_t stream) {
    param_grad_kernel<<<grid_for(a.n, 256), 256, 0, stream>>>(a);
    return cudaGetLastError();
}

size_t adjoint_sort_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const unsigned long long*>(nullptr),
                                    static_cast<unsigned long long*>(nullptr),
                                    static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                    static_cast<int>(n));
    return bytes;
}

cudaError_t launch_adjoint_prepare(const AdjointArgs& a, cudaStream_t stream) {
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    cudaError_t e;
    if ((e = cudaMemsetAsync(a.clamped, 0, sizeof(int), stream)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(a.nrec, 0, sizeof(int), stream)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(a.ticket, 0, sizeof(unsigned long long), stream)) != cudaSuccess) return e;
    adjoint_prepare_kernel<<<grid_for(n, 256), 256, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_adjoint_order(const AdjointArgs& a, cudaStream_t stream) {
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    cudaError_t e;
    if (a.order_src) {
        adjoint_keys_kernel<<<grid_for(n, 256), 256, 0, stream>>>(a.T, a.order_src, n, a.keys, a.order);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    size_t bytes = a.sort_temp_bytes;
    e = cub::DeviceRadixSort::SortPairs(a.sort_temp, bytes, a.keys, a.keys_alt, a.order, a.order_alt,
                                        static_cast<int>(n), 0, 64, stream);
    if (e != cudaSuccess) return e;
    rank_kernel<<<grid_for(n, 256), 256, 0, stream>>>(a.order_alt, a.rank, n);
    return cudaGetLastError();
}

cudaError_t launch_adjoint_solve(const AdjointArgs& a, cudaStream_t stream) {
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    cudaError_t e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (a.fused_prep)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, adjoint_dataflow_kernel<true>, 256, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, adjoint_dataflow_kernel<false>, 256, 0);
    if (per_sm < 1) per_sm = 1;
    if (!a.fused_prep) {
        adjoint_gather_prep_kernel<<<grid_for(n, 256), 256, 0, stream>>>(a, a.order_alt);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    int df_grid = sms * per_sm;
    if (a.max_ctas > 0 && df_grid > a.max_ctas * per_sm) df_grid = a.max_ctas * per_sm;
    if (a.fused_prep)
        adjoint_dataflow_kernel<true><<<df_grid, 256, 0, stream>>>(a, a.order_alt);
    else
        adjoint_dataflow_kernel<false><<<df_grid, 256, 0, stream>>>(a, a.order_alt);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (a.d_g11) adjoint_param_grad_kernel<<<grid_for(n, 256), 256, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_adjoint(const AdjointArgs& a, cudaStream_t stream) {
    cudaError_t e;
    if ((e = launch_adjoint_prepare(a, stream)) != cudaSuccess) return e;
    if ((e = launch_adjoint_order(a, stream)) != cudaSuccess) return e;
    return launch_adjoint_solve(a, stream);
}

cudaError_t launch_loss_grad(const LossArgs& a, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(a.unreached, 0, sizeof(int), stream);
    if (e != cudaSuccess) return e;
    const int parts = grid_for(a.n, 256, 1024);
    loss_grad_kernel<<<parts, 256, 0, stream>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (a.exact)
        loss_exact_kernel<<<1, 256, 0, stream>>>(a);
    else
        loss_final_kernel<<<1, 1024, 0, stream>>>(a, parts);
    return cudaGetLastError();
}

cudaError_t launch_unreached_penalty(int64_t n, const double* T, const uint8_t* observed, const double* values,
                                     double cap, double* acc, cudaStream_t stream) {
    unreached_penalty_kernel<<<1, 256, 0, stream>>>(n, T, observed, values, cap, acc);
    return cudaGetLastError();
}

cudaError_t launch_accumulate5(int64_t n, double* const acc[5], const double* const add_[5],
                               cudaStream_t stream) {
    accumulate5_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, acc[0], acc[1], acc[2], acc[3], acc[4],
                                                             add_[0], add_[1], add_[2], add_[3], add_[4]);
    return cudaGetLastError();
}

}  // namespace rfk
