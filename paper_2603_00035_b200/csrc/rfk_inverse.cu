// rfk_inverse.cu — device kernels of the recovery loop around the solver:
// the smoothed-TV and Tikhonov regularizers (feasibility.cpp:106-196), the
// global-norm clip and the Adam / gradient-descent steps (inversion.cpp:75-127),
// the isotropic/diagonal clamp projection (inversion.cpp:263-272) and the
// relative error (inversion.cpp:129-138).
//
// Everything is elementwise or a stencil of forward differences, so HBM-bound.
// Results are bit-identical to the reference where it is deterministic:
//  * TV gradients are evaluated in gather form.  The reference scatters
//    (tv_core: grad(r,c) -= fx+fy; grad(r,c+1) += fx; grad(r+1,c) += fy, in
//    row-major order), so node (r,c) receives +fy of (r-1,c), then +fx of
//    (r,c-1), then -(fx+fy) of itself: replayed here in that order.
//  * Sums the reference takes sequentially (TV value, Tikhonov value, the clip
//    norm, relative error) have two modes: `exact` replays the sequential sum
//    in node order (one block: staged chunks, one adding thread; bit for bit,
//    bound by the dependent DADD chain), otherwise a tree reduction (fast,
//    last-bit differences).
//  * The Log-Euclidean variant goes through atan2/cos/sin/log, whose device
//    versions may differ from glibc by an ulp.
#include <cuda_runtime.h>

#include <cstdint>

#include "rfk_internal.h"
#include "rfk_numerics.cuh"

namespace rfk {

namespace {

int grid_for(int64_t n, int threads, int cap = 8192) {
    int64_t g = (n + threads - 1) / threads;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return static_cast<int>(g);
}

__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// tv_core's per-node quantities (feasibility.cpp:113-124): forward
// differences with zero flux at the far edges, s = eps^2 + sum w_k (dx^2+dy^2).
__device__ __forceinline__ double tv_node(const TvArgs& a, int r, int c, double fx[3], double fy[3]) {
    const int64_t i = static_cast<int64_t>(r) * a.C + c;
    double dx[3] = {0.0, 0.0, 0.0}, dy[3] = {0.0, 0.0, 0.0};
    double s = mul(a.eps, a.eps);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (k >= a.nch) break;
        const double v = a.ch[k][i];
        if (c + 1 < a.C) dx[k] = sub(a.ch[k][i + 1], v);
        if (r + 1 < a.R) dy[k] = sub(a.ch[k][i + a.C], v);
        s = add(s, mul(a.w[k], add(mul(dx[k], dx[k]), mul(dy[k], dy[k]))));
    }
    const double root = __dsqrt_rn(s);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (k >= a.nch) break;
        fx[k] = ddiv(mul(a.w[k], dx[k]), root);
        fy[k] = ddiv(mul(a.w[k], dy[k]), root);
    }
    return root;
}

__global__ void tv_kernel(TvArgs a) {
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / a.C), c = static_cast<int>(i - static_cast<int64_t>(r) * a.C);
        double fx[3], fy[3], ux[3], uy[3], lx[3], ly[3];
        const double root = tv_node(a, r, c, fx, fy);
        a.term[i] = sub(root, a.eps);  // value += root - eps (:120)
        if (r > 0) tv_node(a, r - 1, c, ux, uy);
        if (c > 0) tv_node(a, r, c - 1, lx, ly);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (k >= a.nch) break;
            double g = 0.0;
            if (r > 0) g = add(g, uy[k]);   // grad(r+1,c) += fy of the node above (:126)
            if (c > 0) g = add(g, lx[k]);   // grad(r,c+1) += fx of the node to the left (:125)
            g = sub(g, add(fx[k], fy[k]));  // grad(r,c) -= fx + fy (:124)
            a.grad[k][i] = g;
        }
    }
}

// ---- Log-Euclidean variant (feasibility.cpp:74-104, :156-178) --------------
struct Eig {
    double hi, lo, c, s;
};

__device__ __forceinline__ Eig decompose(double g11, double g12, double g22) {
    Eig d;
    const double half_tr = mul(0.5, add(g11, g22));
    const double amc = sub(g11, g22);
    const double disc = __dsqrt_rn(add(mul(mul(0.25, amc), amc), mul(g12, g12)));
    d.hi = add(half_tr, disc);
    d.lo = sub(half_tr, disc);
    const double theta = mul(0.5, atan2(mul(2.0, g12), amc));
    sincos(theta, &d.s, &d.c);
    return d;
}

__global__ void log_spd_kernel(int64_t n, const double* g11, const double* g12, const double* g22, double* l11,
                               double* l12, double* l22, int* non_spd) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const Eig d = decompose(g11[i], g12[i], g22[i]);
        if (!(d.lo > 0.0)) {
            atomicExch(non_spd, 1);
            l11[i] = l12[i] = l22[i] = 0.0;
            continue;
        }
        const double H = log(d.hi), L = log(d.lo);
        // recompose(d, log hi, log lo) (:24-27)
        l11[i] = add(mul(mul(H, d.c), d.c), mul(mul(L, d.s), d.s));
        l12[i] = mul(mul(sub(H, L), d.c), d.s);
        l22[i] = add(mul(mul(H, d.s), d.s), mul(mul(L, d.c), d.c));
    }
}

// out[k] = lgrad . dlog_apply(d, e_k) (:170-177)
__global__ void dlog_chain_kernel(int64_t n, const double* g11, const double* g12, const double* g22,
                                  const double* lg0, const double* lg1, const double* lg2, double* o0, double* o1,
                                  double* o2) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const Eig d = decompose(g11[i], g12[i], g22[i]);
        const double c1 = d.c, s1 = d.s;
        const double phi11 = ddiv(1.0, d.hi), phi22 = ddiv(1.0, d.lo);
        const double phi12 = fabs(sub(d.hi, d.lo)) > mul(1e-12, d.hi)
                                 ? ddiv(sub(log(d.hi), log(d.lo)), sub(d.hi, d.lo))
                                 : ddiv(1.0, d.hi);
        double* outs[3] = {o0, o1, o2};
        const double l0 = lg0[i], l1 = lg1[i], l2 = lg2[i];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double ma = k == 0 ? 1.0 : 0.0, mb = k == 1 ? 1.0 : 0.0, mc = k == 2 ? 1.0 : 0.0;
            // m.mul(v) = (a v.x + b v.y, b v.x + c v.y); v1 = (c1, s1), v2 = (-s1, c1)
            const double p1x = add(mul(ma, c1), mul(mb, s1)), p1y = add(mul(mb, c1), mul(mc, s1));
            const double p2x = add(mul(ma, -s1), mul(mb, c1)), p2y = add(mul(mb, -s1), mul(mc, c1));
            const double m11 = add(mul(c1, p1x), mul(s1, p1y));
            const double m12 = add(mul(c1, p2x), mul(s1, p2y));
            const double m22 = add(mul(-s1, p2x), mul(c1, p2y));
            const double a = mul(m11, phi11), b = mul(m12, phi12), c = mul(m22, phi22);
            const double r11 = add(sub(mul(mul(a, c1), c1), mul(mul(mul(2.0, b), c1), s1)), mul(mul(c, s1), s1));
            const double r12 =
                sub(add(mul(mul(a, c1), s1), mul(b, sub(mul(c1, c1), mul(s1, s1)))), mul(mul(c, c1), s1));
            const double r22 = add(add(mul(mul(a, s1), s1), mul(mul(mul(2.0, b), c1), s1)), mul(mul(c, c1), c1));
            outs[k][i] = add(add(mul(l0, r11), mul(l1, r12)), mul(l2, r22));
        }
    }
}

// ---- sums --------------------------------------------------------------------
// Sequential: acc = acc + f(x_i) for i in order (see seq_sum_kernel).
template <int MODE>
__device__ __forceinline__ double term_of(const SumArgs& a, int p, int64_t i) {
    const double x = a.x[p][i];
    if (MODE == 0) return x;                                     // plain values
    if (MODE == 1) return mul(x, x);                             // squares (clip norm)
    if (MODE == 2) return mul(mul(mul(0.5, a.scale), x), x);     // 0.5*w*x*x (Tikhonov)
    const double d = sub(x, a.y[p][i]);                          // MODE 3: (est - truth)^2
    return mul(d, d);
}

// One block: the other threads stage the next chunk's terms in shared memory
// (coalesced loads) while thread 0 adds the current chunk in order, so the
// cost is the dependent DADD chain, not memory latency.
constexpr int kSeqChunk = 2048;
template <int MODE>
__global__ void __launch_bounds__(256) seq_sum_kernel(SumArgs a, double* out) {
    __shared__ double buf[2][kSeqChunk];
    const int64_t total = a.n * a.planes;
    const int64_t nchunks = (total + kSeqChunk - 1) / kSeqChunk;
    auto stage = [&](int64_t ch, double* dst) {
        const int64_t base = ch * kSeqChunk;
        for (int e = threadIdx.x; e < kSeqChunk; e += blockDim.x) {
            const int64_t g = base + e;
            double v = 0.0;
            if (g < total) {
                const int p = static_cast<int>(g / a.n);
                v = term_of<MODE>(a, p, g - static_cast<int64_t>(p) * a.n);
            }
            dst[e] = v;
        }
    };
    double acc = a.init;
    if (nchunks > 0) stage(0, buf[0]);
    __syncthreads();
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        const double* cur = buf[ch & 1];
        if (threadIdx.x == 0) {
            const int cnt = static_cast<int>(total - ch * kSeqChunk < kSeqChunk ? total - ch * kSeqChunk : kSeqChunk);
            for (int e = 0; e < cnt; ++e) acc = add(acc, cur[e]);  // in index order (bit for bit)
        } else if (ch + 1 < nchunks) {
            // warps other than thread 0's stage the next chunk meanwhile
            if (threadIdx.x >= 32) {
                const int64_t base = (ch + 1) * kSeqChunk;
                double* dst = buf[(ch + 1) & 1];
                for (int e = threadIdx.x - 32; e < kSeqChunk; e += blockDim.x - 32) {
                    const int64_t g = base + e;
                    double v = 0.0;
                    if (g < total) {
                        const int p = static_cast<int>(g / a.n);
                        v = term_of<MODE>(a, p, g - static_cast<int64_t>(p) * a.n);
                    }
                    dst[e] = v;
                }
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = acc;
}

template <int MODE>
__global__ void tree_sum_kernel(SumArgs a, double* partial) {
    __shared__ double sh[256];
    double part = 0.0;
    for (int p = 0; p < a.planes; ++p)
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            part = add(part, term_of<MODE>(a, p, i));
    sh[threadIdx.x] = part;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = add(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void tree_final_kernel(const double* partial, int nparts, double init, double* out) {
    __shared__ double sh[1024];
    sh[threadIdx.x] = threadIdx.x < nparts ? partial[threadIdx.x] : 0.0;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = add(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = add(init, sh[0]);
}

// ---- elementwise ----------------------------------------------------------------
__global__ void axpy_kernel(int64_t n, double alpha, const double* x, double* y) {
    // y[i] += alpha * x[i]   (inversion.cpp:57-59, :66-67)
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        y[i] = add(y[i], mul(alpha, x[i]));
}

__global__ void scale_kernel(int64_t n, double f, double* x, double w, const double* src) {
    // src == null: x *= f (clip_global_norm :84-85); else x = w * src (Tikhonov grad :190)
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = src ? mul(w, src[i]) : mul(x[i], f);
}

__global__ void add2_kernel(int64_t n, const double* a, const double* b, double* out) {
    // ParamView::map_gradient, isotropic: g11 + g22 (inversion.cpp:222-226)
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = add(a[i], b[i]);
}

__global__ void clamp_kernel(int64_t n, double* x, double lo, double hi) {
    // std::clamp (inversion.cpp:265-272)
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = x[i];
        x[i] = (v < lo) ? lo : (hi < v) ? hi : v;
    }
}

__global__ void adam_kernel(int64_t n, double* p, double* m, double* v, const double* g, double step, double b1,
                            double b2, double bc1, double bc2, double eps) {
    // adam_step (inversion.cpp:110-115)
    const double c1 = sub(1.0, b1), c2 = sub(1.0, b2);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double gi = g[i];
        const double mi = add(mul(b1, m[i]), mul(c1, gi));
        const double vi = add(mul(b2, v[i]), mul(mul(c2, gi), gi));
        m[i] = mi;
        v[i] = vi;
        p[i] = sub(p[i], ddiv(mul(step, ddiv(mi, bc1)), add(__dsqrt_rn(ddiv(vi, bc2)), eps)));
    }
}

__global__ void gd_kernel(int64_t n, double* p, const double* g, double step) {
    // gd_step (inversion.cpp:124-126)
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = sub(p[i], mul(step, g[i]));
}

}  // namespace

cudaError_t launch_tv(const TvArgs& a, cudaStream_t stream) {
    const int64_t n = static_cast<int64_t>(a.R) * a.C;
    tv_kernel<<<grid_for(n, 256), 256, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_log_spd(int64_t n, const double* g11, const double* g12, const double* g22, double* l11,
                           double* l12, double* l22, int* non_spd, cudaStream_t stream) {
    log_spd_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, g11, g12, g22, l11, l12, l22, non_spd);
    return cudaGetLastError();
}

cudaError_t launch_dlog_chain(int64_t n, const double* g11, const double* g12, const double* g22,
                              const double* const lg[3], double* const out[3], cudaStream_t stream) {
    dlog_chain_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, g11, g12, g22, lg[0], lg[1], lg[2], out[0], out[1],
                                                            out[2]);
    return cudaGetLastError();
}

cudaError_t launch_sum(const SumArgs& a, int mode, bool exact, double* partial, double* out, cudaStream_t stream) {
    if (exact) {
        switch (mode) {
            case 0: seq_sum_kernel<0><<<1, 256, 0, stream>>>(a, out); break;
            case 1: seq_sum_kernel<1><<<1, 256, 0, stream>>>(a, out); break;
            case 2: seq_sum_kernel<2><<<1, 256, 0, stream>>>(a, out); break;
            default: seq_sum_kernel<3><<<1, 256, 0, stream>>>(a, out); break;
        }
        return cudaGetLastError();
    }
    const int parts = grid_for(a.n, 256, 1024);
    switch (mode) {
        case 0: tree_sum_kernel<0><<<parts, 256, 0, stream>>>(a, partial); break;
        case 1: tree_sum_kernel<1><<<parts, 256, 0, stream>>>(a, partial); break;
        case 2: tree_sum_kernel<2><<<parts, 256, 0, stream>>>(a, partial); break;
        default: tree_sum_kernel<3><<<parts, 256, 0, stream>>>(a, partial); break;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    tree_final_kernel<<<1, 1024, 0, stream>>>(partial, parts, a.init, out);
    return cudaGetLastError();
}

cudaError_t launch_axpy(int64_t n, double alpha, const double* x, double* y, cudaStream_t stream) {
    axpy_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, alpha, x, y);
    return cudaGetLastError();
}

cudaError_t launch_scale(int64_t n, double f, double* x, cudaStream_t stream) {
    scale_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, f, x, 0.0, nullptr);
    return cudaGetLastError();
}

cudaError_t launch_weighted_copy(int64_t n, double w, const double* src, double* out, cudaStream_t stream) {
    scale_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, 1.0, out, w, src);
    return cudaGetLastError();
}

cudaError_t launch_add2(int64_t n, const double* a, const double* b, double* out, cudaStream_t stream) {
    add2_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, a, b, out);
    return cudaGetLastError();
}

cudaError_t launch_clamp(int64_t n, double* x, double lo, double hi, cudaStream_t stream) {
    clamp_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, x, lo, hi);
    return cudaGetLastError();
}

cudaError_t launch_adam(int64_t n, double* p, double* m, double* v, const double* g, double step, double b1,
                        double b2, double bc1, double bc2, double eps, cudaStream_t stream) {
    adam_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, p, m, v, g, step, b1, b2, bc1, bc2, eps);
    return cudaGetLastError();
}

cudaError_t launch_gd(int64_t n, double* p, const double* g, double step, cudaStream_t stream) {
    gd_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, p, g, step);
    return cudaGetLastError();
}

}  // namespace rfk
