// Per-step latency of the sweep's dirty-node evaluation, isolated: one warp,
// each iteration's neighbour value depends on the previous iteration's result.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2603_00035_b200/csrc/rfk_numerics.cuh"
using namespace rfk;

__device__ __forceinline__ unsigned long long order_key(double v) {
    unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v));
    if (u == 0x8000000000000000ull) u = 0ull;
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

template <int MODE>
__global__ void k_step(const double* hq, double* out, long long* cyc, int iters) {
    const int lane = threadIdx.x & 31, k = lane & 7, c = k & 3, k2 = (k + 1) & 7;
    const unsigned gbase = lane & ~7u;
    const double q11 = hq[0], q12 = hq[1], q22 = hq[2], a = hq[3], qa = hq[4], qb = hq[5];
    const double mb1 = hq[6 + k], mb2 = hq[6 + k2], sq1 = hq[14 + c], sq2 = hq[14 + (k2 & 3)];
    double t1 = 0.5 + 0.01 * k, t2 = 0.5 + 0.011 * k2, tself = 1.0;
    double acc = 0.0;
    long long t0c = clock64();
    for (int it = 0; it < iters; ++it) {
        const bool r1 = t1 < 1e9, r2 = t2 < 1e9;
        const double s1 = add(t1, mb1), s2 = add(t2, mb2);
        double best;
        bool found = true, first_nan = false;
        if (MODE == 2) {
            best = s1 + s2;  // reduce-only baseline
        } else {
            const double bq = add(mul(qa, s1), mul(qb, s2));
            const double cc = sub(add(add(mul(mul(q11, s1), s1), mul(mul(mul(2.0, q12), s1), s2)), mul(mul(q22, s2), s2)), 1.0);
            const double disc = sub(mul(bq, bq), mul(a, cc));
            const double t0 = add(bq, sqrt(disc)) / a;
            const double d1 = sub(t0, s1), d2 = sub(t0, s2);
            const double l1 = add(mul(q11, d1), mul(q12, d2));
            const double l2 = add(mul(q12, d1), mul(q22, d2));
            const bool valid = r1 && r2 && !(disc < 0.0) && t0 > smax(t1, t2) && l1 >= 0.0 && l2 >= 0.0;
            const double o1 = add(s1, sq1), o2 = add(s2, sq2);
            const bool n1 = o1 != o1, n2 = o2 != o2;
            found = valid || r1 || r2;
            first_nan = !valid && (r1 ? n1 : (r2 && n2));
            best = valid ? t0 : __longlong_as_double(0x7ff0000000000000ll);
            if (!valid) {
                const double c1 = (r1 && !n1) ? o1 : best;
                const double c2 = (r2 && !n2) ? o2 : best;
                best = (c2 < c1) ? c2 : c1;
            }
        }
        double res = best;
        if (MODE != 1) {
            const unsigned fmask = (__ballot_sync(0xffffffffu, found) >> gbase) & 0xffu;
            const unsigned nmask = (__ballot_sync(0xffffffffu, first_nan) >> gbase) & 0xffu;
            unsigned long long key = order_key(best);
            int id = k;
#pragma unroll
            for (int off = 1; off < 8; off <<= 1) {
                const unsigned long long okey = __shfl_xor_sync(0xffffffffu, key, off);
                const int oid = __shfl_xor_sync(0xffffffffu, id, off);
                const bool lower = (lane & off) == 0;
                const bool take = lower ? (okey < key) : !(key < okey);
                key = take ? okey : key;
                id = take ? oid : id;
            }
            const bool nan_first = fmask && ((nmask >> (__ffs(fmask) - 1)) & 1u);
            res = (!nan_first && key < order_key(tself)) ? __longlong_as_double(key & 0x7fffffffffffffffull) : tself;
        }
        // feed the result back as the next step's fresh neighbour
        t1 = add(mul(res, 1e-3), 0.5 + 0.01 * k);
        acc = add(acc, res);
    }
    long long t1c = clock64();
    out[threadIdx.x] = acc + t1;
    if (threadIdx.x == 0) cyc[0] = t1c - t0c;
}

int main() {
    double h[32];
    h[0] = 1.2; h[1] = 0.1; h[2] = 1.1; h[3] = 1.2 + 0.2 + 1.1; h[4] = 1.3; h[5] = 1.2;
    for (int i = 0; i < 8; ++i) h[6 + i] = 0.01 * (i - 3);
    for (int i = 0; i < 4; ++i) h[14 + i] = 0.7 + 0.1 * i;
    double *dq, *out; long long* cyc; long long c;
    cudaMalloc(&dq, 256); cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8);
    cudaMemcpy(dq, h, sizeof(h), cudaMemcpyHostToDevice);
    const int iters = 4096;
    const char* names[3] = {"full (chain+fold)", "chain only", "fold only"};
    for (int w : {32, 128}) {
        k_step<0><<<1, w>>>(dq, out, cyc, iters); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("%-20s warps=%d %7.1f cyc/step\n", names[0], w / 32, (double)c / iters);
        k_step<1><<<1, w>>>(dq, out, cyc, iters); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("%-20s warps=%d %7.1f cyc/step\n", names[1], w / 32, (double)c / iters);
        k_step<2><<<1, w>>>(dq, out, cyc, iters); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("%-20s warps=%d %7.1f cyc/step\n", names[2], w / 32, (double)c / iters);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
