// FP64 pipe throughput on this B200 (the second roofline of the sweep, SURVEY
// §8d): DFMA, DADD, DMUL issued from every SM with 8 independent chains per
// thread, timed with CUDA events.  Prints one JSON object:
//   {"dfma_tops": thread-level DFMA per second / 1e12, "dadd_tops": ...,
//    "dmul_tops": ..., "fp64_tflops": 2 * dfma_tops, "sm_count": ...,
//    "warp_inst_per_s": warp-level FP64 instructions per second (DFMA)}
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

template <int OP>
__global__ void __launch_bounds__(256) k_pipe(double* out, double x) {
    double a[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] = x + threadIdx.x + i;
    const double m = 1.0000000001, c = 1e-300;
#pragma unroll 1
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) {
            if (OP == 0) a[i] = __fma_rn(a[i], m, c);
            if (OP == 1) a[i] = __dadd_rn(a[i], c);
            if (OP == 2) a[i] = __dmul_rn(a[i], m);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kChains; ++i) s += a[i];
    if (s == 12345.0) out[threadIdx.x] = s;  // keep the chains live
}

template <int OP>
double run(int sms) {
    double* out;
    cudaMalloc(&out, 1024 * sizeof(double));
    const int blocks = sms * 8, threads = 256;
    k_pipe<OP><<<blocks, threads>>>(out, 1.0);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_pipe<OP><<<blocks, threads>>>(out, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFree(out);
    const double ops = static_cast<double>(blocks) * threads * kIters * kChains;
    return ops / (best * 1e-3);
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const double fma = run<0>(sms), add = run<1>(sms), mul = run<2>(sms);
    printf("{\"dfma_tops\": %.4f, \"dadd_tops\": %.4f, \"dmul_tops\": %.4f, \"fp64_tflops\": %.4f, "
           "\"warp_inst_per_s\": %.4e, \"sm_count\": %d, \"clock_khz_attr\": %d, "
           "\"per_sm_per_clk_at_attr\": %.2f}\n",
           fma / 1e12, add / 1e12, mul / 1e12, 2 * fma / 1e12, fma / 32, sms, clk,
           fma / sms / (clk * 1e3));
    return 0;
}
