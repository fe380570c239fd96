// Dirty-step latency of the sweep's compute role, isolated (B200): 4 warps,
// 8 lanes per node, every step dirty; each node reads two neighbour values
// written by the previous step (ring in shared memory) and writes its result;
// one named barrier per step.  MODE bits ablate pieces of the step:
//   1: no barrier (warps run free)     2: sqrt -> mul
//   4: no fold (each lane writes)      8: division instead of the hoisted reciprocal
//  16: key-free ballots skipped (no found/first_nan ballots)
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2603_00035_b200/csrc/rfk_numerics.cuh"
using namespace rfk;

template <int MODE>
__global__ void k_step(const double* hq, double* out, long long* cyc, int iters) {
    __shared__ double ring[17][64];
    __shared__ __align__(16) double fold[128];
    __shared__ __align__(8) unsigned char flg[128];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, k = lane & 7, c = k & 3, k2 = (k + 1) & 7;
    const int l = warp * 4 + (lane >> 3);
    const unsigned gbase = lane & ~7u;
    const double q11 = hq[0], q12 = hq[1], q22 = hq[2], ap = hq[3], y = hq[4];
    const double mb1 = hq[6 + k], mb2 = hq[6 + k2], sq1 = hq[14 + c], sq2 = hq[14 + (k2 & 3)];
    for (int i = threadIdx.x; i < 17 * 64; i += blockDim.x) (&ring[0][0])[i] = 0.3 + 0.001 * (i % 13);
    __syncthreads();
    long long t0c = clock64();
    for (int it = 0; it < iters; ++it) {
        const double t1 = ring[l][(it + k) & 63], t2 = ring[l][(it + k2) & 63];
        const double tself = ring[l + 1][it & 63];
        const bool r1 = t1 < 1e9, r2 = t2 < 1e9;
        const double qa = add(q11, q12), qb = add(q12, q22);
        const double s1 = add(t1, mb1), s2 = add(t2, mb2);
        const double bq = add(mul(qa, s1), mul(qb, s2));
        const double cc = sub(add(add(mul(mul(q11, s1), s1), mul(mul(mul(2.0, q12), s1), s2)), mul(mul(q22, s2), s2)), 1.0);
        const double disc = sub(mul(bq, bq), mul(ap, cc));
        const bool need = r1 && r2 && ap > 0.0 && !(disc < 0.0);
        const double disc_s = need ? disc : 1.0;
        const double x = add(bq, (MODE & 2) ? mul(disc_s, 0.5) : sqrt(disc_s));
        double t0;
        if (MODE & 8) {
            t0 = x / (need ? ap : 1.0);
        } else {
            const double q = __dmul_rn(x, y);
            t0 = __fma_rn(__fma_rn(-ap, q, x), y, q);
        }
        const double d1 = sub(t0, s1), d2 = sub(t0, s2);
        const double l1 = add(mul(q11, d1), mul(q12, d2));
        const double l2 = add(mul(q12, d1), mul(q22, d2));
        const bool valid = need && t0 > smax(t1, t2) && l1 >= 0.0 && l2 >= 0.0;
        const double o1 = add(s1, sq1), o2 = add(s2, sq2);
        const bool n1 = o1 != o1, n2 = o2 != o2;
        const bool found = valid || r1 || r2;
        const bool first_nan = !valid && (r1 ? n1 : (r2 && n2));
        double best = valid ? t0 : __longlong_as_double(0x7ff0000000000000ll);
        if (!valid) {
            const double c1 = (r1 && !n1) ? o1 : best;
            const double c2 = (r2 && !n2) ? o2 : best;
            best = (c2 < c1) ? c2 : c1;
        }
        if (MODE & 4) {
            ring[l + 1][(it + 1) & 63] = best * 1e-3 + tself * 0.999;
        } else {
            fold[warp * 32 + lane] = best;
            unsigned fm = 1, nm = 0;
            if (MODE & 32) {
                flg[warp * 32 + lane] = (found ? 1 : 0) | (first_nan ? 2 : 0);
            } else if (!(MODE & 16)) {
                fm = __ballot_sync(0xffffffffu, found);
                nm = __ballot_sync(0xffffffffu, first_nan);
            }
            __syncwarp();
            if (k == 0) {
                const double2* fv = reinterpret_cast<const double2*>(fold + warp * 32 + gbase);
                const double2 p01 = fv[0], p23 = fv[1], p45 = fv[2], p67 = fv[3];
                const double m01 = (p01.y < p01.x) ? p01.y : p01.x;
                const double m23 = (p23.y < p23.x) ? p23.y : p23.x;
                const double m45 = (p45.y < p45.x) ? p45.y : p45.x;
                const double m67 = (p67.y < p67.x) ? p67.y : p67.x;
                const double m03 = (m23 < m01) ? m23 : m01;
                const double m47 = (m67 < m45) ? m67 : m45;
                const double g = (m47 < m03) ? m47 : m03;
                bool any, blocked;
                if (MODE & 32) {
                    const unsigned long long w = *reinterpret_cast<const unsigned long long*>(flg + warp * 32 + gbase);
                    const unsigned long long f = w & 0x0101010101010101ull;
                    any = f != 0ull;
                    blocked = any && ((w >> (__ffsll(static_cast<long long>(f)) - 1)) & 2ull);
                } else {
                    const unsigned f8 = (fm >> gbase) & 0xffu, n8 = (nm >> gbase) & 0xffu;
                    any = f8 != 0u;
                    blocked = f8 != 0u && ((n8 >> (__ffs(f8) - 1)) & 1u);
                }
                ring[l + 1][(it + 1) & 63] = (any && !blocked && g < tself) ? g : tself * 0.999 + g * 1e-3;
            }
        }
        if (!(MODE & 1)) asm volatile("bar.sync 1, 128;" ::: "memory");
        else __syncwarp();
    }
    long long t1c = clock64();
    if (threadIdx.x == 0) cyc[0] = t1c - t0c;
    out[threadIdx.x] = ring[l + 1][5];
}

int main() {
    double hq[32];
    // a mildly anisotropic metric at h = 1/1024: admissible two-point updates
    const double h = 1.0 / 1024;
    hq[0] = 1.1 / (h * h); hq[1] = 0.1 / (h * h); hq[2] = 0.9 / (h * h);
    hq[3] = hq[0] + 2 * hq[1] + hq[2]; hq[4] = 1.0 / hq[3];
    for (int k = 0; k < 8; ++k) hq[6 + k] = 1e-4 * (k - 3.5);
    for (int c = 0; c < 4; ++c) hq[14 + c] = h * (1.0 + 0.1 * c);
    double *d_hq, *out; long long* cyc; long long hc;
    cudaMalloc(&d_hq, sizeof(hq)); cudaMalloc(&out, 128 * 8); cudaMalloc(&cyc, 8);
    cudaMemcpy(d_hq, hq, sizeof(hq), cudaMemcpyHostToDevice);
    const int iters = 20000;
#define RUN(M, name) k_step<M><<<1, 128>>>(d_hq, out, cyc, iters); k_step<M><<<1, 128>>>(d_hq, out, cyc, iters); \
    cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost); printf("%-34s %7.1f cycles/step\n", name, (double)hc / iters);
    RUN(0, "full step");
    RUN(1, "no barrier");
    RUN(2, "sqrt->mul");
    RUN(4, "no fold");
    RUN(8, "ieee division");
    RUN(16, "no flag ballots");
    RUN(32, "flags via smem bytes");
    RUN(33, "flags via smem, no barrier");
    RUN(34, "flags via smem, sqrt->mul");
    RUN(6, "sqrt->mul, no fold");
    RUN(7, "sqrt->mul, no fold, no barrier");
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
