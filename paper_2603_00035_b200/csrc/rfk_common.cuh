// rfk_common.cuh — device helpers shared by the kernels: memory-model
// primitives, the persistent-kernel grid barrier and the sweep-direction
// geometry.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rfk {

// ---- memory model -----------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Loads of data another SM may have written during this kernel: bypass L1
// (which is not coherent across SMs).
__device__ __forceinline__ int ld_acquire_int(const int* p) {
    return static_cast<int>(ld_acquire(reinterpret_cast<const unsigned*>(p)));
}
__device__ __forceinline__ void st_release_int(int* p, int v) {
    st_release(reinterpret_cast<unsigned*>(p), static_cast<unsigned>(v));
}
__device__ __forceinline__ double ld_l2(const double* p) { return __ldcg(p); }
__device__ __forceinline__ void st_l2(double* p, double v) { __stcg(p, v); }

// Non-negative doubles order like their bit patterns: max via integer atomics.
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* p, double v) {
    atomicMax(p, static_cast<unsigned long long>(__double_as_longlong(v)));
}

// ---- grid barrier (all CTAs co-resident: cooperative launch) ---------------
// B: any struct with `unsigned* count, *generation` (count starts at 0).
template <class B>
__device__ __forceinline__ void grid_sync(const B& b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = ld_acquire(b.generation);
        __threadfence();
        if (atomicAdd(b.count, 1u) == gridDim.x - 1) {
            *b.count = 0u;
            __threadfence();
            st_release(b.generation, gen + 1u);
        } else {
            while (ld_acquire(b.generation) == gen) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// ---- sweep geometry -----------------------------------------------------------
// Directional pass d visits lines L (outer loop) and positions W (inner loop)
// in the reference's order (sweeper.cpp:104-119):
//   d0: c↑ r↑  L=c      W=r          d1: r↑ c↓  L=r      W=C-1-c
//   d2: c↓ r↓  L=C-1-c  W=R-1-r      d3: r↓ c↑  L=R-1-r  W=c
struct SweepGeom {
    int dir, R, C, NL, NW;

    __device__ __forceinline__ static SweepGeom make(int dir, int R, int C) {
        SweepGeom g;
        g.dir = dir;
        g.R = R;
        g.C = C;
        const bool cols_are_lines = (dir & 1) == 0;
        g.NL = cols_are_lines ? C : R;
        g.NW = cols_are_lines ? R : C;
        return g;
    }
    __device__ __forceinline__ int64_t node(int L, int W) const {
        int r, c;
        switch (dir) {
            case 0: r = W; c = L; break;
            case 1: r = L; c = C - 1 - W; break;
            case 2: r = R - 1 - W; c = C - 1 - L; break;
            default: r = R - 1 - L; c = W; break;
        }
        return static_cast<int64_t>(r) * C + c;
    }
    // Ring neighbour k (dr, dc) expressed as a (line, position) offset.
    __device__ __forceinline__ void ring_lw(int k, int dr, int dc, int& dl, int& dw) const {
        (void)k;
        switch (dir) {
            case 0: dl = dc; dw = dr; break;
            case 1: dl = dr; dw = -dc; break;
            case 2: dl = -dc; dw = -dr; break;
            default: dl = -dr; dw = dc; break;
        }
    }
};

}  // namespace rfk
