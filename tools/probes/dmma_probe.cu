// FP64 pipe question for the Gauss kernel design: does the FP64 tensor-core MMA
// (mma.sync m8n8k4 f64) add throughput beside vector DFMA on sm_100a?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probes/dmma_probe.cu -o tools/probes/dmma_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NF, int NM>
__global__ void __launch_bounds__(256) mix_kernel(double *out, int iters, double a, double b) {
    double f[8], m0[4], m1[4];
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = threadIdx.x * 1e-9 + k;
#pragma unroll
    for (int k = 0; k < 4; ++k) { m0[k] = k; m1[k] = k + 0.5; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < NF; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) f[k] = fma(f[k], a, b);
#pragma unroll
        for (int u = 0; u < NM; ++u)
#pragma unroll
            for (int k = 0; k < 4; ++k) dmma(m0[k], m1[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += f[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) s += m0[k] + m1[k];
    if (s == 12345.678) out[0] = s;
}

template <int NF, int NM>
void run(const char *name, int sms) {
    double *out;
    cudaMalloc(&out, 8);
    const int blocks = sms * 8, threads = 256, iters = 2048;
    mix_kernel<NF, NM><<<blocks, threads>>>(out, 16, 0.999999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) mix_kernel<NF, NM><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double thr = (double)3 * blocks * threads * iters;
    const double fma_flops = thr * NF * 8 * 2;                 // per thread
    const double mma_flops = thr / 32 * NM * 4 * 8 * 8 * 4 * 2;  // per warp instruction: 256 FMA
    printf("%-10s %8.3f ms  DFMA %7.2f TF/s  DMMA %7.2f TF/s  total %7.2f TF/s\n", name, ms,
           fma_flops / ms / 1e9, mma_flops / ms / 1e9, (fma_flops + mma_flops) / ms / 1e9);
    cudaFree(out);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<4, 0>("dfma", sms);
    run<0, 4>("dmma", sms);
    run<4, 4>("mix 1:1", sms);
    run<4, 1>("mix 4:1", sms);
    run<1, 4>("mix 1:4", sms);
    return 0;
}
