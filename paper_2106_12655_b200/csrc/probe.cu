// FP64 pipe microbenchmarks (roofline denominator; BASELINE.md §3 asks for a
// measured DFMA peak because MEASURED_PEAKS.json carries none).
#include "common.cuh"

namespace lc {
namespace {

// 8 independent DFMA chains per thread, `iters` x 8 x 2 flops per thread.
__global__ void __launch_bounds__(256) dfma_chain_kernel(double *out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 12345.678) out[0] = s;   // never true; keeps the chains alive
}

__device__ __forceinline__ void dmma_m8n8k4(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// 4 independent FP64 tensor-core MMA chains per warp (m8n8k4: 256 FMA = 512 FLOP each).
__global__ void __launch_bounds__(256) dmma_chain_kernel(double *out, int iters, double a, double b) {
    double m0[4], m1[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        m0[k] = k + threadIdx.x * 1e-9;
        m1[k] = k + 0.5;
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int k = 0; k < 4; ++k) dmma_m8n8k4(m0[k], m1[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s += m0[k] + m1[k];
    if (s == 12345.678) out[0] = s;
}

}  // namespace

// FP64 tensor-core (DMMA) throughput: the FP64 datapath's other peak (shared with DFMA).
double probe_dmma_flops(cudaStream_t s, float *elapsed_ms) {
    int sms = 0, dev = 0;
    LC_CUDA(cudaGetDevice(&dev));
    LC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double *out = nullptr;
    LC_CUDA(cudaMallocAsync(&out, sizeof(double), s));
    const int blocks = sms * 8, threads = 256, iters = 1024;
    dmma_chain_kernel<<<blocks, threads, 0, s>>>(out, 16, 0.999999, 1e-7);   // warm-up
    LC_CHECK_LAUNCH();
    cudaEvent_t e0, e1;
    LC_CUDA(cudaEventCreate(&e0));
    LC_CUDA(cudaEventCreate(&e1));
    LC_CUDA(cudaEventRecord(e0, s));
    const int reps = 3;
    for (int r = 0; r < reps; ++r) dmma_chain_kernel<<<blocks, threads, 0, s>>>(out, iters, 0.999999, 1e-7);
    LC_CHECK_LAUNCH();
    LC_CUDA(cudaEventRecord(e1, s));
    LC_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    LC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    LC_CUDA(cudaFreeAsync(out, s));
    if (elapsed_ms) *elapsed_ms = ms;
    const double warps = (double)reps * blocks * (threads / 32) * iters;
    return warps * 4 * 4 * 512.0 / (ms * 1e-3);
}

// Returns achieved FP64 FLOP/s of a pure DFMA kernel over `ms_target` ms.
double probe_dfma_flops(cudaStream_t s, float *elapsed_ms) {
    int sms = 0, dev = 0;
    LC_CUDA(cudaGetDevice(&dev));
    LC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double *out = nullptr;
    LC_CUDA(cudaMallocAsync(&out, sizeof(double), s));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    dfma_chain_kernel<<<blocks, threads, 0, s>>>(out, 64, 0.999999, 1e-7);   // warm-up
    LC_CHECK_LAUNCH();
    cudaEvent_t e0, e1;
    LC_CUDA(cudaEventCreate(&e0));
    LC_CUDA(cudaEventCreate(&e1));
    LC_CUDA(cudaEventRecord(e0, s));
    const int reps = 5;
    for (int r = 0; r < reps; ++r) dfma_chain_kernel<<<blocks, threads, 0, s>>>(out, iters, 0.999999, 1e-7);
    LC_CHECK_LAUNCH();
    LC_CUDA(cudaEventRecord(e1, s));
    LC_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    LC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    LC_CUDA(cudaFreeAsync(out, s));
    if (elapsed_ms) *elapsed_ms = ms;
    const double flops = (double)reps * blocks * threads * (double)iters * 4 * 8 * 2;
    return flops / (ms * 1e-3);
}

}  // namespace lc
