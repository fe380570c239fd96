// rfk_project.cu — metric-feasibility projections on sm_100a.
//
// Reference: project_spd with decompose/recompose (src/feasibility.cpp:15-44,
// sym2_eigenvalues mat2.hpp:44-49), drift_norm_sq (:46-49), project_drift
// (:51-72).  Elementwise, HBM-bound.  project_drift and every pass-through
// node of project_spd are bit-identical to the reference; at nodes that need
// an eigenvalue clamp the recomposition uses the device atan2/cos/sin, which
// may differ from glibc by an ulp.
#include <cuda_runtime.h>

#include <cstdint>

#include "rfk_internal.h"
#include "rfk_numerics.cuh"

namespace rfk {

namespace {

__device__ __forceinline__ double sclamp(double v, double lo, double hi) {
    return (v < lo) ? lo : (hi < v) ? hi : v;  // std::clamp
}

__global__ void project_spd_kernel(int64_t n, double* g11, double* g12, double* g22, double eps_min,
                                   double lambda_max) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double a = g11[i], b = g12[i], c = g22[i];
        const double half_tr = mul(0.5, add(a, c));
        const double amc = sub(a, c);
        const double disc = sqrt(add(mul(mul(0.25, amc), amc), mul(b, b)));
        const double hi = add(half_tr, disc), lo = sub(half_tr, disc);
        if (lo >= eps_min && hi <= lambda_max) continue;  // :36 pass-through
        const double theta = mul(0.5, atan2(mul(2.0, b), amc));
        double sn, cs;
        sincos(theta, &sn, &cs);
        const double H = sclamp(hi, eps_min, lambda_max);
        const double L = sclamp(lo, eps_min, lambda_max);
        g11[i] = add(mul(mul(H, cs), cs), mul(mul(L, sn), sn));
        g12[i] = mul(mul(sub(H, L), cs), sn);
        g22[i] = add(mul(mul(H, sn), sn), mul(mul(L, cs), cs));
    }
}

__device__ __forceinline__ double drift_norm_sq(double b1, double b2, double g11, double g12, double g22) {
    const double det = sub(mul(g11, g22), mul(g12, g12));
    return add(sub(mul(mul(b1, b1), g22), mul(mul(mul(2.0, b1), b2), g12)), mul(mul(b2, b2), g11)) / det;
}

__global__ void project_drift_kernel(int64_t n, double* b1, double* b2, const double* g11,
                                     const double* g12, const double* g22, double tau, double cap) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double x = b1[i], y = b2[i];
        const double en = sqrt(add(mul(x, x), mul(y, y)));
        if (en > cap) {
            const double f = cap / en;
            x = mul(x, f);
            y = mul(y, f);
        }
        const double gn = sqrt(drift_norm_sq(x, y, g11[i], g12[i], g22[i]));
        if (gn > tau) {
            const double f = tau / gn;
            x = mul(x, f);
            y = mul(y, f);
        }
        b1[i] = x;
        b2[i] = y;
    }
}

__global__ void drift_norm_sq_kernel(int64_t n, const double* b1, const double* b2, const double* g11,
                                     const double* g12, const double* g22, double* out) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = drift_norm_sq(b1[i], b2[i], g11[i], g12[i], g22[i]);
}

int grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 32) g = 148 * 32;
    return g < 1 ? 1 : static_cast<int>(g);
}

}  // namespace

cudaError_t launch_project_spd(int64_t n, double* g11, double* g12, double* g22, double eps_min,
                               double lambda_max, cudaStream_t stream) {
    project_spd_kernel<<<grid_for(n), 256, 0, stream>>>(n, g11, g12, g22, eps_min, lambda_max);
    return cudaGetLastError();
}

cudaError_t launch_project_drift(int64_t n, double* b1, double* b2, const double* g11,
                                 const double* g12, const double* g22, double tau,
                                 double euclid_cap, cudaStream_t stream) {
    project_drift_kernel<<<grid_for(n), 256, 0, stream>>>(n, b1, b2, g11, g12, g22, tau, euclid_cap);
    return cudaGetLastError();
}

cudaError_t launch_drift_norm_sq(int64_t n, const double* b1, const double* b2, const double* g11,
                                 const double* g12, const double* g22, double* out,
                                 cudaStream_t stream) {
    drift_norm_sq_kernel<<<grid_for(n), 256, 0, stream>>>(n, b1, b2, g11, g12, g22, out);
    return cudaGetLastError();
}

}  // namespace rfk
