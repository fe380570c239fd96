// Latency microbenchmarks for the sweep's per-step building blocks (B200).
#include <cstdio>
#include <cuda_runtime.h>

#define N 1024
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }

__global__ void k_dadd(double* out, double x, long long* cyc) {
    double a = x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = xadd(a, 1e-300);
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dmul(double* out, double x, long long* cyc) {
    double a = x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = xmul(a, 1.0000001);
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_ddiv(double* out, double x, long long* cyc) {
    double a = x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = 1.7 / a;
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dsqrt(double* out, double x, long long* cyc) {
    double a = x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = sqrt(a) + 1.5;
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl(double* out, double x, long long* cyc) {
    double a = x + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = __shfl_xor_sync(0xffffffffu, a, 1);
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_bar(double* out, double x, long long* cyc) {
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) asm volatile("bar.sync 1, 128;" ::: "memory");
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_acq(double* out, double x, long long* cyc) {
    __shared__ int f[4];
    if (threadIdx.x == 0) f[0] = 1;
    __syncthreads();
    int s = 0;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        int v;
        asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(f)) : "memory");
        s += v;
    }
    long long t1 = clock64();
    out[threadIdx.x] = s; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_rel(double* out, double x, long long* cyc) {
    __shared__ int f[4];
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i)
        asm volatile("st.release.cta.shared.b32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(f)), "r"(i) : "memory");
    long long t1 = clock64();
    out[threadIdx.x] = f[0]; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds(double* out, double x, long long* cyc) {
    __shared__ int f[64];
    f[threadIdx.x & 63] = (threadIdx.x + 1) & 63;
    __syncthreads();
    int p = threadIdx.x & 63;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) p = f[p];
    long long t1 = clock64();
    out[threadIdx.x] = p; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}


__global__ void k_dmin(double* out, double x, long long* cyc) {
    double a = x, b = x * 0.5 + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { double c = __dadd_rn(b, 0.0); a = (c < a) ? c : a; b = a; }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dsel(double* out, double x, long long* cyc) {
    double a = x, b = x * 0.5 + threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < 4; ++i) b = b * 1.01;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { a = (b < a) ? b : a; b = a + 0.0 * i; }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_kmin(double* out, double x, long long* cyc) {
    unsigned long long a = __double_as_longlong(x), b = a ^ threadIdx.x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { a = (b < a) ? b : a; b = a ^ (unsigned long long)(i & 1); }
    long long t1 = clock64();
    out[threadIdx.x] = (double)a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_redux(double* out, double x, long long* cyc) {
    unsigned a = threadIdx.x * 7u + (unsigned)x;
    const unsigned m = 0xffu << (threadIdx.x & 24);
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = __reduce_min_sync(m, a) + threadIdx.x;
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_vote(double* out, double x, long long* cyc) {
    int a = threadIdx.x & (int)x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = __any_sync(0xffffffffu, a == (int)threadIdx.x) + i;
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_ballot(double* out, double x, long long* cyc) {
    unsigned a = threadIdx.x & (int)x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = __ballot_sync(0xffffffffu, (a >> (threadIdx.x & 7)) & 1) + i;
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_smemx(double* out, double x, long long* cyc) {
    __shared__ double sm[32];
    double a = x + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        sm[threadIdx.x] = a;
        __syncwarp();
        a = sm[(threadIdx.x & ~7) + 7 - (threadIdx.x & 7)];
        __syncwarp();
    }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dfma(double* out, double x, long long* cyc) {
    double a = x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = __fma_rn(a, 1.0000001, 1e-300);
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dsqrt_only(double* out, double x, long long* cyc) {
    double a = x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) a = __dsqrt_rn(a) ;
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double* out; long long* cyc; long long h;
    cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
    auto run = [&](const char* name, void (*k)(double*, double, long long*), int threads) {
        k<<<1, threads>>>(out, 1.2345, cyc);
        k<<<1, threads>>>(out, 1.2345, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-10s %6.1f cycles/op (threads=%d)\n", name, (double)h / N, threads);
    };
    run("dadd", k_dadd, 32); run("dmul", k_dmul, 32); run("ddiv", k_ddiv, 32); run("dsqrt+add", k_dsqrt, 32);
    run("shfl.f64", k_shfl, 32); run("bar128", k_bar, 128); run("ld.acq", k_acq, 32); run("st.rel", k_rel, 32);
    run("lds-chase", k_lds, 32);
    run("dadd x4w", k_dadd, 128); run("ddiv x4w", k_ddiv, 128);
    run("dmin(add)", k_dmin, 32); run("dsel", k_dsel, 32); run("kmin64", k_kmin, 32); run("redux8", k_redux, 32);
    run("vote.any", k_vote, 32); run("ballot", k_ballot, 32); run("sts/lds x", k_smemx, 32); run("dfma", k_dfma, 32);
    run("dsqrt", k_dsqrt_only, 32);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
