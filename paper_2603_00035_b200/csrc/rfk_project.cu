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
#include "rfk_project.cuh"

namespace rfk {

namespace {

using namespace proj;

__global__ void project_spd_kernel(int64_t n, double* g11, double* g12, double* g22, double eps_min,
                                   double lambda_max) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double o11, o12, o22;
        if (spd_node(g11[i], g12[i], g22[i], eps_min, lambda_max, o11, o12, o22)) {
            g11[i] = o11;
            g12[i] = o12;
            g22[i] = o22;
        }
    }
}

__global__ void project_drift_kernel(int64_t n, double* b1, double* b2, const double* g11,
                                     const double* g12, const double* g22, double tau, double cap) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double x = b1[i], y = b2[i];
        drift_node(x, y, g11[i], g12[i], g22[i], tau, cap);
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

// mode 1: project_spd only; 2: project_drift only (metric fixed, its
// cotangent accumulated if dg11 != nullptr); 3: ParamView::project for the
// Joint parameterization (inversion.cpp:276-279): spd, then drift against the
// projected metric.
__global__ void project_vjp_kernel(int mode, int64_t n, const double* g11, const double* g12, const double* g22,
                                   const double* b1, const double* b2, double eps_min, double lambda_max,
                                   double tau, double cap, double* dg11, double* dg12, double* dg22, double* db1,
                                   double* db2) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double a = g11[i], b = g12[i], c = g22[i];
        double d11 = dg11 ? dg11[i] : 0.0, d12 = dg12 ? dg12[i] : 0.0, d22 = dg22 ? dg22[i] : 0.0;
        double dx = (mode & 2) ? db1[i] : 0.0, dy = (mode & 2) ? db2[i] : 0.0;
        project_vjp_node(mode, eps_min, lambda_max, tau, cap, a, b, c, (mode & 2) ? b1[i] : 0.0,
                         (mode & 2) ? b2[i] : 0.0, d11, d12, d22, dx, dy);
        if (mode & 2) {
            db1[i] = dx;
            db2[i] = dy;
        }
        if (dg11) {
            dg11[i] = d11;
            dg12[i] = d12;
            dg22[i] = d22;
        }
    }
}

__global__ void widen_kernel(int64_t n, const float* in, double* out) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<double>(in[i]);
}

__global__ void narrow_kernel(int64_t n, const double* in, float* out) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<float>(in[i]);
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

cudaError_t launch_project_vjp(int mode, int64_t n, const double* g11, const double* g12, const double* g22,
                               const double* b1, const double* b2, double eps_min, double lambda_max, double tau,
                               double euclid_cap, double* dg11, double* dg12, double* dg22, double* db1,
                               double* db2, cudaStream_t stream) {
    project_vjp_kernel<<<grid_for(n), 256, 0, stream>>>(mode, n, g11, g12, g22, b1, b2, eps_min, lambda_max, tau,
                                                        euclid_cap, dg11, dg12, dg22, db1, db2);
    return cudaGetLastError();
}

cudaError_t launch_widen_f32(int64_t n, const float* in, double* out, cudaStream_t stream) {
    widen_kernel<<<grid_for(n), 256, 0, stream>>>(n, in, out);
    return cudaGetLastError();
}

cudaError_t launch_narrow_f64(int64_t n, const double* in, float* out, cudaStream_t stream) {
    narrow_kernel<<<grid_for(n), 256, 0, stream>>>(n, in, out);
    return cudaGetLastError();
}

}  // namespace rfk
