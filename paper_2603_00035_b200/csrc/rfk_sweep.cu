// rfk_sweep.cu — the exact Gauss-Seidel fast sweep on sm_100a (v2).
//
// Reference: run_sweeping / solve / solve_from_values, src/sweeper.cpp:
// 86-174 (relax :92-96, the four loop orders :101-121, max|dT| < tol stop
// :146-151).
//
// Schedule (bit-exact): node (L, W) of a directional pass (line L, position
// W in the reference's loop order) runs at hyperplane step s = 2L + W.  That
// order honours every RAW edge (new values of line L-1 and of (L, W-1)) and
// every WAR edge (old values of (L, W+1) and of line L+1) of the sequential
// sweep, and nodes of one step are never neighbours.
//
// CTA layout (warp-specialised, persistent, cooperative launch):
//   * BL/4 compute warps walk one band of BL consecutive lines in lockstep
//     (named barrier per step).  A node is evaluated by 8 lanes, one per
//     triangular stencil; the stencil fold of best_candidate is an
//     order-preserving shuffle reduction (rfk_numerics.cuh).
//   * 1 producer warp stages, ahead of the compute warps, each position
//     column of the band into shared-memory rings: T and sweep stamps of
//     lines L0-1 .. L0+BL, the five metric planes and the fixed mask of the
//     own lines, and the iteration-start values for the max|dT| test.
//   * Band-to-band handoff: the last line of band b is published per
//     position into a mailbox of 8-byte words that each carry 32 data bits
//     and a 32-bit sweep tag (the NCCL "LL" idea), so the consumer polls the
//     data itself: no fence, no flag round trip on the critical path.
//
// Work reduction (both exact):
//   * T-independent terms of every stencil (E = M'GM, Q = E^-1, a, the
//     drift projections m.b, the edge costs sqrt(m'Gm)) are computed once
//     per node visit, for the next node while the current node's dependent
//     chain runs; the dependent chain is ~15 fp64 ops + 1 sqrt + 1 div.
//   * Skip-unchanged: a node none of whose 8 neighbours changed in this or
//     the previous pass evaluates to the same candidate it produced last
//     time, which cannot lower it again; such nodes are not evaluated.
//     Changes are tracked with an 8-bit pass stamp per node.
#include <cuda_runtime.h>

#include <cstdint>

#include "rfk_common.cuh"
#include "rfk_internal.h"
#include "rfk_numerics.cuh"

namespace rfk {

namespace {

__device__ __forceinline__ int sweep_dir(int o) { return (o == 0 || o == 1 || o == 2) ? o : 3; }

template <int BL>
struct Cfg {
    static constexpr int NCW = BL / 4;  // compute warps (4 nodes per warp)
    static constexpr int THREADS = (NCW + 1) * 32;
    // position ring: a column lives 2*BL steps; the rest is producer lookahead
    static constexpr int P = (BL <= 16) ? 128 : 256;
    static constexpr int MASK = P - 1;
    static constexpr int CH = (BL <= 16) ? 16 : 8;              // producer chunk (columns per round)
    static constexpr int MAXE = (CH * (BL + 1) + 31) / 32;      // staged elements per producer lane
    // shared memory carve-up (bytes)
    static constexpr size_t T_OFF = 0;
    static constexpr size_t P_OFF = T_OFF + sizeof(double) * (BL + 2) * P;      // prev (last pass)
    static constexpr size_t G_OFF = P_OFF + sizeof(double) * BL * P;            // 5 metric planes
    static constexpr size_t S_OFF = G_OFF + sizeof(double) * 5 * BL * P;        // stamps
    static constexpr size_t F_OFF = S_OFF + (BL + 2) * P;                       // fixed mask
    static constexpr size_t C_OFF = (F_OFF + BL * P + 15) / 16 * 16;            // control words
    static constexpr size_t BYTES = C_OFF + 64;
};

struct Smem {
    double* T;
    double* Pv;
    double* G;
    uint8_t* St;
    uint8_t* Fx;
    volatile int* loaded;    // columns [0, loaded) staged
    volatile int* computed;  // steps [0, computed) finished
};

// T-independent part of stencil k at one node (hoisted out of the
// dependent chain).  Bit-identical to two_point_update's own arithmetic
// (src/stencil.cpp:12-30) and one_point_update's edge cost.
struct Hoist {
    double q11, q12, q22, q12x2, a, qa, qb;
    double mb1, mb2, sq1, sq2;
    bool tp_ok;  // E well conditioned and a > 0 (else the two-point is invalid)
};

__device__ __forceinline__ Hoist hoist_stencil(const Metric& g, double m1x, double m1y, double m2x,
                                               double m2y, unsigned partner) {
    Hoist z;
    double gx, gy;
    gmul(g, m1x, m1y, gx, gy);
    const double e11 = dot2(m1x, m1y, gx, gy);  // = quad(m1), stencil.cpp:13
    const double e12 = dot2(m2x, m2y, gx, gy);  // :14
    z.mb1 = dot2(m1x, m1y, g.b1, g.b2);         // m1.b (:24)
    z.sq1 = sqrt(e11);                           // one-point edge cost sqrt(m'Gm)
    // stencil k's second donor is stencil k2's first: its quad form, drift
    // projection and edge cost come from that lane (same operations).
    const double e22 = __shfl_sync(0xffffffffu, e11, partner);
    z.sq2 = __shfl_sync(0xffffffffu, z.sq1, partner);
    z.mb2 = __shfl_sync(0xffffffffu, z.mb1, partner);
    const double p = mul(e11, e22), q = mul(e12, e12);
    const double det = sub(p, q);
    z.tp_ok = det > mul(1e-14, smax(p, q));  // :17-18
    if (z.tp_ok) {
        z.q11 = e22 / det;
        z.q12 = -e12 / det;
        z.q22 = e11 / det;
    } else {
        z.q11 = z.q12 = z.q22 = 0.0;
    }
    z.q12x2 = mul(2.0, z.q12);
    z.a = add(add(z.q11, z.q12x2), z.q22);  // :28
    z.qa = add(z.q11, z.q12);
    z.qb = add(z.q12, z.q22);
    z.tp_ok = z.tp_ok && !(z.a <= 0.0);  // :33 (a part; disc part below)
    return z;
}

// Dependent chain of stencil k given the hoisted terms (stencil.cpp:24-41,
// stencil.hpp:43-45, folded like sweeper.cpp:37-59).
__device__ __forceinline__ LaneCand lane_eval(const Hoist& z, double t1, double t2) {
    LaneCand lc;
    lc.best = __longlong_as_double(0x7ff0000000000000ll);
    lc.lam1 = lc.lam2 = 0.0;
    lc.which = lc.first_which = -1;
    lc.found = lc.first_nan = false;
    const bool r1 = reached(t1), r2 = reached(t2);
    const double s1 = add(t1, z.mb1);
    const double s2 = add(t2, z.mb2);
    if (r1 && r2 && z.tp_ok) {
        const double bq = add(mul(z.qa, s1), mul(z.qb, s2));
        const double c = sub(add(add(mul(mul(z.q11, s1), s1), mul(mul(z.q12x2, s1), s2)), mul(mul(z.q22, s2), s2)),
                             1.0);
        const double disc = sub(mul(bq, bq), mul(z.a, c));
        if (!(disc < 0.0)) {
            const double t0 = add(bq, sqrt(disc)) / z.a;
            const double d1 = sub(t0, s1), d2 = sub(t0, s2);
            const double l1 = add(mul(z.q11, d1), mul(z.q12, d2));
            const double l2 = add(mul(z.q12, d1), mul(z.q22, d2));
            if (t0 > smax(t1, t2) && l1 >= 0.0 && l2 >= 0.0) {
                lc.found = true;
                lc.best = t0;
                lc.which = lc.first_which = 0;
                return lc;
            }
        }
    }
    if (r1) lane_take(lc, add(s1, z.sq1), 1);
    if (r2) lane_take(lc, add(s2, z.sq2), 2);
    return lc;
}

// ---- mailbox: {lo32 | tag32} and {hi32 | tag32}, tag = (epoch<<1)|changed ----
__device__ __forceinline__ void mailbox_put(unsigned long long* slot, unsigned epoch, double v, bool changed) {
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
    const unsigned long long tag = static_cast<unsigned long long>((epoch << 1) | (changed ? 1u : 0u)) << 32;
    const unsigned long long w0 = tag | (bits & 0xffffffffull);
    const unsigned long long w1 = tag | (bits >> 32);
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(slot), "l"(w0), "l"(w1) : "memory");
}

__device__ __forceinline__ bool mailbox_get(const unsigned long long* slot, unsigned epoch, double& v,
                                            bool& changed) {
    unsigned long long w0, w1;
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(slot) : "memory");
    const unsigned e = epoch & 0x7fffffffu;
    if (static_cast<unsigned>(w0 >> 33) != e || static_cast<unsigned>(w1 >> 33) != e) return false;
    v = __longlong_as_double(static_cast<long long>((w1 << 32) | (w0 & 0xffffffffull)));
    changed = (w0 >> 32) & 1ull;
    return true;
}

__device__ __forceinline__ bool stamp_dirty(uint8_t st, unsigned S) {
    return ((S - st) & 0xffu) <= 1u;  // changed in this pass or the previous one
}

// ---------------------------------------------------------------------------
template <int BL>
__device__ void produce_band(const SweepArgs& a, const SweepGeom& geo, int bi, bool first_pass, bool last_pass,
                             unsigned epoch, unsigned S, Smem sm) {
    using K = Cfg<BL>;
    const int lane = threadIdx.x & 31;
    const int L0 = bi * BL;
    const int nl = min(BL, geo.NL - L0);
    const int NW = geo.NW;
    const bool has_prev = L0 > 0;
    const bool has_next = L0 + nl < geo.NL;
    const unsigned long long* mbox = a.mailbox + static_cast<size_t>(bi - 1) * a.mailbox_stride;
    int own_upto = 0;
    int prev_upto = has_prev ? 0 : NW;
    int published = 0;
    while (published < NW) {
        bool progress = false;
        const int comp = *sm.computed;
        const int limit = min(NW, comp + K::P - 2 * nl);
        if (own_upto < limit) {
            const int X0 = own_upto, X1 = min(limit, X0 + K::CH);
            const int ncol = X1 - X0;
            // rows 1..nl+1 of the T/stamp ring (own lines + next band's first line):
            // issue every load of the chunk first (memory-level parallelism),
            // then write shared memory.
            double v[K::MAXE], pv[K::MAXE], gp[K::MAXE][5];
            uint8_t st[K::MAXE], fx[K::MAXE];
            const double* planes[5] = {a.g11, a.g12, a.g22, a.b1, a.b2};
#pragma unroll
            for (int u = 0; u < K::MAXE; ++u) {
                const int e = lane + 32 * u;
                const int X = X0 + e / (nl + 1), j = e % (nl + 1);  // j: 0..nl-1 own, nl next
                v[u] = kUnreached;
                pv[u] = 0.0;
                st[u] = static_cast<uint8_t>(S - 2);
                fx[u] = 1;
                if (e < ncol * (nl + 1) && (j < nl || has_next)) {
                    const int64_t node = geo.node(L0 + j, X);
                    v[u] = ld_l2(a.T + node);
                    st[u] = a.stamp[node];
                    if (j < nl) {
#pragma unroll
                        for (int c = 0; c < 5; ++c) gp[u][c] = __ldg(planes[c] + node);
                        fx[u] = __ldg(a.src + node);
                        if (last_pass) pv[u] = ld_l2(a.prev + node);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < K::MAXE; ++u) {
                const int e = lane + 32 * u;
                if (e >= ncol * (nl + 1)) continue;
                const int X = X0 + e / (nl + 1), j = e % (nl + 1);
                const int slot = X & K::MASK;
                sm.T[(j + 1) * K::P + slot] = v[u];
                sm.St[(j + 1) * K::P + slot] = st[u];
                if (j < nl) {
#pragma unroll
                    for (int c = 0; c < 5; ++c) sm.G[(c * BL + j) * K::P + slot] = gp[u][c];
                    sm.Fx[j * K::P + slot] = fx[u];
                    if (last_pass) sm.Pv[j * K::P + slot] = pv[u];
                    if (first_pass) st_l2(a.prev + geo.node(L0 + j, X), v[u]);
                }
            }
            if (!has_prev) {
                for (int X = X0 + lane; X < X1; X += 32) {
                    sm.T[X & K::MASK] = kUnreached;
                    sm.St[X & K::MASK] = static_cast<uint8_t>(S - 2);
                }
            }
            own_upto = X1;
            progress = true;
        }
        if (prev_upto < own_upto) {
            // line L0-1 from band b-1's mailbox: lane i polls column prev_upto+i
            const int X = prev_upto + lane;
            double v = 0.0;
            bool ch = false, ok = false;
            if (X < own_upto) ok = mailbox_get(mbox + 2 * static_cast<size_t>(X), epoch, v, ch);
            const unsigned ready = __ballot_sync(0xffffffffu, ok);
            const int cnt = (~ready == 0u) ? 32 : (__ffs(~ready) - 1);
            if (lane < cnt) {
                const int slot = X & K::MASK;
                sm.T[slot] = v;
                uint8_t st = a.stamp[geo.node(L0 - 1, X)];
                if (ch) st = static_cast<uint8_t>(S);
                sm.St[slot] = st;
            }
            prev_upto += cnt;
            progress = progress || cnt > 0;
        }
        if (progress) {
            __syncwarp();
            __threadfence_block();
            const int up = min(own_upto, prev_upto);
            if (lane == 0) *sm.loaded = up;
            published = up;
        } else {
            __nanosleep(40);
        }
    }
}

template <int BL>
__device__ void compute_band(const SweepArgs& a, const SweepGeom& geo, int bi, bool last_pass, unsigned epoch,
                             unsigned S, Smem sm, double& my_delta) {
    using K = Cfg<BL>;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int k = lane & 7;
    const int l = warp * 4 + (lane >> 3);
    const unsigned partner = (lane & ~7u) | ((k + 1) & 7);
    const int L0 = bi * BL;
    const int nl = min(BL, geo.NL - L0);
    const int NW = geo.NW;
    const int nsteps = 2 * (nl - 1) + NW;
    unsigned long long* my_mbox = a.mailbox + static_cast<size_t>(bi) * a.mailbox_stride;

    double m1x, m1y, m2x, m2y;
    displacement(k, a.h, m1x, m1y);
    displacement((k + 1) & 7, a.h, m2x, m2y);
    int dl1, dw1, dl2, dw2;
    geo.ring_lw(k, ring_dr(k), ring_dc(k), dl1, dw1);
    geo.ring_lw((k + 1) & 7, ring_dr((k + 1) & 7), ring_dc((k + 1) & 7), dl2, dw2);

    auto load_metric = [&](int W) {
        const int slot = W & K::MASK;
        return Metric{sm.G[(0 * BL + l) * K::P + slot], sm.G[(1 * BL + l) * K::P + slot],
                      sm.G[(2 * BL + l) * K::P + slot], sm.G[(3 * BL + l) * K::P + slot],
                      sm.G[(4 * BL + l) * K::P + slot]};
    };

    Hoist hz;
    bool hz_ready = false;
    for (int s = 0; s < nsteps; ++s) {
        const int need = min(s + 2, NW);
        if (lane == 0)
            while (*sm.loaded < need) {
            }
        __syncwarp();
        __threadfence_block();

        const int W = s - 2 * l;
        const bool active = l < nl && W >= 0 && W < NW;
        const int slot = W & K::MASK;
        bool fixed = true;
        double t1 = kUnreached, t2 = kUnreached;
        bool ndirty = false;
        if (active) {
            fixed = sm.Fx[l * K::P + slot] != 0;
            const int W1 = W + dw1, W2 = W + dw2;
            if (W1 >= 0 && W1 < NW) {
                const int i1 = (l + 1 + dl1) * K::P + (W1 & K::MASK);
                t1 = sm.T[i1];
                ndirty = stamp_dirty(sm.St[i1], S);
            }
            if (W2 >= 0 && W2 < NW) t2 = sm.T[(l + 1 + dl2) * K::P + (W2 & K::MASK)];
        }
        const unsigned gbit = __ballot_sync(0xffffffffu, ndirty);
        const bool gdirty = active && !fixed && ((gbit >> (lane & ~7u)) & 0xffu) != 0u;
        const bool wdirty = __any_sync(0xffffffffu, gdirty);

        double tnew = 0.0;
        bool changed = false;
        if (wdirty) {
            if (!hz_ready) hz = hoist_stencil(active ? load_metric(W) : Metric{1, 0, 1, 0, 0}, m1x, m1y, m2x, m2y, partner);
            LaneCand lc = lane_eval(hz, t1, t2);
            if (!gdirty) {
                lc.found = false;
                lc.which = -1;
                lc.best = __longlong_as_double(0x7ff0000000000000ll);
            }
            const GroupResult gr = group_reduce(lc);
            if (gdirty && k == 0) {
                const double t = sm.T[(l + 1) * K::P + slot];
                if (gr.found && gr.t0 < t) {  // Sweeper::relax, sweeper.cpp:95
                    tnew = gr.t0;
                    changed = true;
                }
            }
            // hoist the next node's T-independent terms while the pipe is warm
            const int Wn = W + 1;
            const bool nact = l < nl && Wn >= 0 && Wn < NW;
            hz = hoist_stencil(nact ? load_metric(Wn) : Metric{1, 0, 1, 0, 0}, m1x, m1y, m2x, m2y, partner);
            hz_ready = true;
        } else {
            hz_ready = false;
        }
        if (active && k == 0) {
            const int self = (l + 1) * K::P + slot;
            const int64_t node = geo.node(L0 + l, W);
            double t = sm.T[self];
            if (changed) {
                t = tnew;
                sm.T[self] = t;
                sm.St[self] = static_cast<uint8_t>(S);
                st_l2(a.T + node, t);
                a.stamp[node] = static_cast<uint8_t>(S);
            }
            if (l == nl - 1) mailbox_put(my_mbox + 2 * static_cast<size_t>(W), epoch, t, changed);
            if (last_pass) my_delta = smax(my_delta, fabs(t - sm.Pv[l * K::P + slot]));
        }
        asm volatile("bar.sync 1, %0;" ::"r"(K::NCW * 32) : "memory");
        if (threadIdx.x == 0) {
            __threadfence_block();
            *sm.computed = s + 1;
        }
    }
}

template <int BL>
__global__ void __launch_bounds__(Cfg<BL>::THREADS, 1) sweep_kernel(SweepArgs a) {
    using K = Cfg<BL>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem sm{reinterpret_cast<double*>(smem_raw + K::T_OFF), reinterpret_cast<double*>(smem_raw + K::P_OFF),
            reinterpret_cast<double*>(smem_raw + K::G_OFF), smem_raw + K::S_OFF, smem_raw + K::F_OFF,
            reinterpret_cast<volatile int*>(smem_raw + K::C_OFF),
            reinterpret_cast<volatile int*>(smem_raw + K::C_OFF + 16)};
    __shared__ double red[K::NCW + 1];
    const bool producer = (threadIdx.x >> 5) == K::NCW;

    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *a.iterations = 0;
        *a.converged = 0;
    }
    unsigned epoch = a.epoch_base;
    unsigned S = 0;  // pass counter for the 8-bit change stamps (init kernel set 255/254)
    for (int it = 0; it < a.max_iters; ++it) {
        double my_delta = 0.0;
        for (int q = 0; q < 4; ++q, ++epoch, ++S) {
            const SweepGeom geo = SweepGeom::make(sweep_dir(a.order[q]), a.R, a.C);
            const int nbands = (geo.NL + BL - 1) / BL;
            for (int bi = blockIdx.x; bi < nbands; bi += gridDim.x) {
                if (threadIdx.x == 0) {
                    *sm.loaded = 0;
                    *sm.computed = 0;
                }
                __syncthreads();
                if (producer)
                    produce_band<BL>(a, geo, bi, q == 0, q == 3, epoch, S, sm);
                else
                    compute_band<BL>(a, geo, bi, q == 3, epoch, S, sm, my_delta);
                __syncthreads();
            }
            if (q == 3) {
                double v = my_delta;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v = smax(v, __shfl_xor_sync(0xffffffffu, v, off));
                if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
                __syncthreads();
                if (threadIdx.x == 0) {
                    double b = 0.0;
                    for (int w = 0; w <= K::NCW; ++w) b = smax(b, red[w]);
                    atomic_max_nonneg(a.maxdelta + it, b);
                }
            }
            grid_sync(a.bar);
        }
        const double md = __longlong_as_double(static_cast<long long>(ld_acquire(a.maxdelta + it)));
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (a.history) a.history[it] = md;
            *a.iterations = it + 1;
            if (md < a.tol) *a.converged = 1;
        }
        if (md < a.tol) break;  // sweeper.cpp:151 (strict)
    }
}

__global__ void init_stamps_kernel(uint8_t* stamp, const uint8_t* src, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        stamp[i] = src[i] ? 255 : 254;  // pass -1 = "changed" (sources), -2 = clean
}

template <int BL>
cudaError_t launch_bl(const SweepArgs& a, int max_ctas, cudaStream_t stream, int* used) {
    using K = Cfg<BL>;
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<BL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(K::BYTES));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<BL>, K::THREADS, K::BYTES);
    if (e != cudaSuccess) return e;
    if (per_sm > 1) per_sm = 1;  // one band per SM: the FP64 pipe belongs to it
    const int max_bands = ((a.R > a.C ? a.R : a.C) + BL - 1) / BL;
    int grid = per_sm * sms;
    if (grid > max_bands) grid = max_bands;
    if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
    if (grid < 1) grid = 1;
    *used = grid;
    void* args[] = {const_cast<SweepArgs*>(&a)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(sweep_kernel<BL>), dim3(grid), dim3(K::THREADS),
                                       args, K::BYTES, stream);
}

}  // namespace

size_t sweep_mailbox_words(int R, int C, int band_lines) {
    const int mx = R > C ? R : C;
    const int nb = (mx + band_lines - 1) / band_lines;
    return static_cast<size_t>(nb) * mx * 2;  // 2 words per position
}

cudaError_t launch_init_stamps(uint8_t* stamp, const uint8_t* src, int64_t n, cudaStream_t stream) {
    int grid = static_cast<int>((n + 255) / 256);
    if (grid > 4096) grid = 4096;
    if (grid < 1) grid = 1;
    init_stamps_kernel<<<grid, 256, 0, stream>>>(stamp, src, n);
    return cudaGetLastError();
}

cudaError_t launch_sweep(const SweepArgs& a, int band_lines, int max_ctas, cudaStream_t stream, int* used) {
    switch (band_lines) {
        case 32: return launch_bl<32>(a, max_ctas, stream, used);
        default: return launch_bl<16>(a, max_ctas, stream, used);
    }
}

}  // namespace rfk
