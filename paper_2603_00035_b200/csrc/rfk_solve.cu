// rfk_solve.cu — forward fast-sweeping solver on sm_100a.
//
// Reference: run_sweeping / solve / solve_from_values (src/sweeper.cpp:
// 124-174) and solve_jacobi (:176-205).
//
// Exact Gauss-Seidel replay.  A directional pass relaxes node (L, W) (line L,
// position W in the reference's loop order) reading NEW values of lines L-1
// and of (L, W-1) and OLD values of (L, W+1) and line L+1.  Scheduling node
// (L, W) at hyperplane step s = 2L + W satisfies every read-after-write and
// write-after-read edge of that order, and nodes of one step are never
// neighbours, so relaxing a whole step at once reproduces the sequential
// sweep bit for bit.
//
// Kernel shape: one persistent cooperative kernel per solve.  The lines of a
// pass are cut into bands of BL lines; a CTA owns one band at a time and
// walks its private hyperplane (2(BL-1) + NW steps), 8 lanes per node
// (one per triangular stencil).  The band's lines live in a shared-memory
// ring of positions; band b reads the last line of band b-1 through L2
// after an acquire on b-1's progress flag, and publishes its own last line
// with a release.  Passes are separated by a grid barrier; the iteration's
// max|dT| is reduced on the device and tested against tol without any host
// round trip (report.iterations / converged / max_delta_history written by
// the kernel).
#include <cuda_runtime.h>

#include <cstdint>

#include "rfk_common.cuh"
#include "rfk_internal.h"
#include "rfk_numerics.cuh"

namespace rfk {

namespace {

__device__ __forceinline__ unsigned long long progress_tag(unsigned long long epoch, int pos) {
    return (epoch << 32) | static_cast<unsigned long long>(pos + 1);
}

__device__ __forceinline__ int sweep_dir(int o) { return (o == 0 || o == 1 || o == 2) ? o : 3; }

struct BandSmem {
    double* Ts;  // [(BL+2) * P]  line j = L0-1+j
    double* Ps;  // [BL * P]      iteration-start values of own lines (last pass)
};

template <int BL, int P>
__device__ void process_band(const SolveArgs& a, const SweepGeom& geo, int bi, bool first_pass,
                             bool last_pass, unsigned long long epoch, BandSmem sm,
                             double& my_delta) {
    constexpr int MASK = P - 1;
    const int tid = threadIdx.x;
    const int l = tid >> 3;  // local line of this 8-lane group
    const int k = tid & 7;   // stencil owned by this lane
    const int L0 = bi * BL;
    const int nl = min(BL, geo.NL - L0);
    const int NW = geo.NW;
    const int nsteps = 2 * (nl - 1) + NW;
    const unsigned long long* prev_band = bi > 0 ? a.progress + (bi - 1) : nullptr;
    unsigned long long* my_band = a.progress + bi;

    // Column loader role: thread j < nl+2 owns line L0-1+j of the ring.
    const int j = tid;
    const bool loader = j < nl + 2;
    const int line = L0 - 1 + j;
    const bool line_exists = loader && line >= 0 && line < geo.NL;
    const bool own_line = loader && j >= 1 && j <= nl;

    auto fetch = [&](int X, double& v, double& pv) {
        v = kUnreached;
        pv = 0.0;
        if (!line_exists || X >= NW) return;
        if (j == 0) {  // last line of the previous band: wait for it to pass X
            const unsigned long long need = progress_tag(epoch, X);
            while (ld_acquire(prev_band) < need) {
            }
        }
        const int64_t node = geo.node(line, X);
        v = ld_l2(a.T + node);
        if (own_line && last_pass) pv = ld_l2(a.prev + node);
    };
    auto stage = [&](int X, double v, double pv) {
        if (!loader || X >= NW) return;
        sm.Ts[j * P + (X & MASK)] = v;
        if (own_line) {
            if (first_pass) st_l2(a.prev + geo.node(line, X), v);
            if (last_pass) sm.Ps[(j - 1) * P + (X & MASK)] = pv;
        }
    };

    // Per-node inputs of the group's next node, prefetched one step ahead.
    Metric nm{0, 0, 0, 0, 0};
    bool nfixed = true;
    auto fetch_params = [&](int s) {
        const int W = s - 2 * l;
        if (l < nl && W >= 0 && W < NW) {
            const int64_t node = geo.node(L0 + l, W);
            nm.g11 = __ldg(a.g11 + node);
            nm.g12 = __ldg(a.g12 + node);
            nm.g22 = __ldg(a.g22 + node);
            nm.b1 = __ldg(a.b1 + node);
            nm.b2 = __ldg(a.b2 + node);
            nfixed = __ldg(a.src + node) != 0;
        }
    };

    // Ring neighbour offsets in (line, position) space for this lane's two donors.
    int dl1, dw1, dl2, dw2;
    geo.ring_lw(k, ring_dr(k), ring_dc(k), dl1, dw1);
    geo.ring_lw((k + 1) & 7, ring_dr((k + 1) & 7), ring_dc((k + 1) & 7), dl2, dw2);

    {
        double v, pv;
        fetch(0, v, pv);
        stage(0, v, pv);
    }
    double nv, npv;
    fetch(1, nv, npv);
    fetch_params(0);
    __syncthreads();

    for (int s = 0; s < nsteps; ++s) {
        stage(s + 1, nv, npv);
        const Metric m = nm;
        const bool fixed = nfixed;
        fetch(s + 2, nv, npv);
        fetch_params(s + 1);
        __syncthreads();

        const int W = s - 2 * l;
        const bool active = l < nl && W >= 0 && W < NW;
        LaneCand lc;
        lc.best = __longlong_as_double(0x7ff0000000000000ll);
        lc.which = lc.first_which = -1;
        lc.found = lc.first_nan = false;
        if (active && !fixed) {
            const int W1 = W + dw1, W2 = W + dw2;
            const double tk = (W1 >= 0 && W1 < NW) ? sm.Ts[(l + 1 + dl1) * P + (W1 & MASK)] : kUnreached;
            const double tk2 = (W2 >= 0 && W2 < NW) ? sm.Ts[(l + 1 + dl2) * P + (W2 & MASK)] : kUnreached;
            lc = lane_candidate<false>(k, tk, tk2, m, a.h);
        }
        const GroupResult gr = group_reduce(lc);
        if (active && k == 0) {
            double* self = sm.Ts + (l + 1) * P + (W & MASK);
            double t = *self;
            const int64_t node = geo.node(L0 + l, W);
            if (!fixed && gr.found && gr.t0 < t) {  // Sweeper::relax, sweeper.cpp:95
                t = gr.t0;
                *self = t;
                st_l2(a.T + node, t);
            }
            if (last_pass) my_delta = smax(my_delta, fabs(t - sm.Ps[l * P + (W & MASK)]));
            if (l == nl - 1) st_release(my_band, progress_tag(epoch, W));
        }
        __syncthreads();
    }
}

template <int BL>
__global__ void __launch_bounds__(BL * 8) sweep_solve_kernel(SolveArgs a) {
    constexpr int P = SweepSmem<BL>::P;
    extern __shared__ double smem[];
    BandSmem sm{smem, smem + (BL + 2) * P};
    __shared__ double red[BL * 8 / 32];

    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *a.iterations = 0;
        *a.converged = 0;
    }
    unsigned long long epoch = a.epoch_base;
    for (int it = 0; it < a.max_iters; ++it) {
        double my_delta = 0.0;
        for (int q = 0; q < 4; ++q) {
            const SweepGeom geo = SweepGeom::make(sweep_dir(a.order[q]), a.R, a.C);
            const int nbands = (geo.NL + BL - 1) / BL;
            for (int bi = blockIdx.x; bi < nbands; bi += gridDim.x)
                process_band<BL, P>(a, geo, bi, q == 0, q == 3, epoch, sm, my_delta);
            ++epoch;
            if (q == 3) {
                // block max -> one atomic per CTA
                double v = my_delta;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v = smax(v, __shfl_xor_sync(0xffffffffu, v, off));
                if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
                __syncthreads();
                if (threadIdx.x == 0) {
                    double b = 0.0;
                    for (int w = 0; w < BL * 8 / 32; ++w) b = smax(b, red[w]);
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

// ---- Jacobi (solve_jacobi, sweeper.cpp:176-205) --------------------------------
__global__ void __launch_bounds__(256) jacobi_kernel(JacobiArgs a) {
    __shared__ double red[8];
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    const int k = threadIdx.x & 7;
    const int64_t warp = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5) * 4;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *a.iterations = 0;
        *a.converged = 0;
    }
    double* cur = a.T;
    double* nxt = a.T2;
    for (int it = 0; it < a.max_iters; ++it) {
        double my = 0.0;
        // warp-uniform trip count so the group shuffles stay converged
        for (int64_t base = warp * 4; base < n; base += stride) {
            const int64_t node = base + ((threadIdx.x >> 3) & 3);
            const bool active = node < n && __ldg(a.src + node) == 0;
            LaneCand lc;
            lc.best = __longlong_as_double(0x7ff0000000000000ll);
            lc.which = lc.first_which = -1;
            lc.found = lc.first_nan = false;
            double curv = 0.0;
            if (active) {
                const int r = static_cast<int>(node / a.C), c = static_cast<int>(node % a.C);
                const Metric m{__ldg(a.g11 + node), __ldg(a.g12 + node), __ldg(a.g22 + node),
                               __ldg(a.b1 + node), __ldg(a.b2 + node)};
                const int k2 = (k + 1) & 7;
                const int r1 = r + ring_dr(k), c1 = c + ring_dc(k);
                const int r2 = r + ring_dr(k2), c2 = c + ring_dc(k2);
                const double tk = (r1 >= 0 && r1 < a.R && c1 >= 0 && c1 < a.C)
                                      ? ld_l2(cur + static_cast<int64_t>(r1) * a.C + c1)
                                      : kUnreached;
                const double tk2 = (r2 >= 0 && r2 < a.R && c2 >= 0 && c2 < a.C)
                                       ? ld_l2(cur + static_cast<int64_t>(r2) * a.C + c2)
                                       : kUnreached;
                lc = lane_candidate<false>(k, tk, tk2, m, a.h);
                curv = ld_l2(cur + node);
            }
            const GroupResult gr = group_reduce(lc);
            if (active && k == 0) {
                const double v = gr.found ? smin(curv, gr.t0) : curv;
                st_l2(nxt + node, v);
                my = smax(my, fabs(v - curv));
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) my = smax(my, __shfl_xor_sync(0xffffffffu, my, off));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = my;
        __syncthreads();
        if (threadIdx.x == 0) {
            double b = 0.0;
            for (int w = 0; w < 8; ++w) b = smax(b, red[w]);
            atomic_max_nonneg(a.maxdelta + it, b);
        }
        grid_sync(a.bar);
        double* t = cur;
        cur = nxt;
        nxt = t;
        const double md = __longlong_as_double(static_cast<long long>(ld_acquire(a.maxdelta + it)));
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (a.history) a.history[it] = md;
            *a.iterations = it + 1;
            if (md < a.tol) *a.converged = 1;
        }
        if (md < a.tol) break;
    }
    // result lives in `cur`; make a.T hold it
    if (cur != a.T) {
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            a.T[i] = ld_l2(cur + i);
    }
}

// initial_field (sweeper.cpp:124-131) + source count for SourceMask::validate.
__global__ void init_field_kernel(double* t, double* t2, const uint8_t* src, const double* fixed_values,
                                  int64_t n, unsigned long long* source_count) {
    unsigned cnt = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const bool s = src[i] != 0;
        const double v = s ? (fixed_values ? fixed_values[i] : 0.0) : kUnreached;
        t[i] = v;
        if (t2) t2[i] = v;
        cnt += s ? 1u : 0u;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(source_count, static_cast<unsigned long long>(cnt));
}

}  // namespace

// ---- host launchers -------------------------------------------------------------
template <int BL>
static cudaError_t launch_sweep_bl(const SolveArgs& a, int max_ctas, cudaStream_t stream,
                                   int* used_ctas) {
    constexpr int threads = BL * 8;
    const size_t smem = SweepSmem<BL>::bytes;
    cudaError_t e = cudaFuncSetAttribute(sweep_solve_kernel<BL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_solve_kernel<BL>, threads, smem);
    if (e != cudaSuccess) return e;
    const int max_bands = ((a.R > a.C ? a.R : a.C) + BL - 1) / BL;
    int grid = per_sm * sms;
    if (grid > max_bands) grid = max_bands;
    if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
    if (grid < 1) grid = 1;
    *used_ctas = grid;
    void* args[] = {const_cast<SolveArgs*>(&a)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(sweep_solve_kernel<BL>), dim3(grid),
                                       dim3(threads), args, smem, stream);
}

cudaError_t launch_sweep_solve(const SolveArgs& a, int band_lines, int max_ctas,
                               cudaStream_t stream, int* used_ctas) {
    switch (band_lines) {
        case 16: return launch_sweep_bl<16>(a, max_ctas, stream, used_ctas);
        case 64: return launch_sweep_bl<64>(a, max_ctas, stream, used_ctas);
        default: return launch_sweep_bl<32>(a, max_ctas, stream, used_ctas);
    }
}

cudaError_t launch_jacobi(const JacobiArgs& a, cudaStream_t stream) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_kernel, 256, 0);
    if (e != cudaSuccess) return e;
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    int64_t need = (n + 31) / 32;
    int grid = per_sm * sms;
    if (need < grid) grid = static_cast<int>(need);
    if (grid < 1) grid = 1;
    void* args[] = {const_cast<JacobiArgs*>(&a)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(jacobi_kernel), dim3(grid), dim3(256),
                                       args, 0, stream);
}

cudaError_t launch_init_field(double* t, double* t2, const uint8_t* src, const double* fixed_values,
                              int64_t n, unsigned long long* source_count, cudaStream_t stream) {
    int grid = static_cast<int>((n + 255) / 256);
    if (grid > 4096) grid = 4096;
    if (grid < 1) grid = 1;
    init_field_kernel<<<grid, 256, 0, stream>>>(t, t2, src, fixed_values, n, source_count);
    return cudaGetLastError();
}

}  // namespace rfk
