// rfk_solve.cu — solve_jacobi (src/sweeper.cpp:176-205) on sm_100a, a
// bit-exact parallel baseline, and the field initialisation of
// run_sweeping (:124-131).  The Gauss-Seidel sweep itself is rfk_sweep.cu.
#include <cuda_runtime.h>

#include <cstdint>

#include "rfk_common.cuh"
#include "rfk_internal.h"
#include "rfk_numerics.cuh"

namespace rfk {

namespace {

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
