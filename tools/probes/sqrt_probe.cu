// Accuracy of the branch-free FP64 sqrt variants of the Gauss kernel vs the
// correctly rounded __dsqrt_rn, and of the MUFU rsqrt.approx.f64 seed.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probes/sqrt_probe.cu -o /tmp/sqrt_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsq(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ double sqrt7(double x) {   // coupled Goldschmidt, 2 iterations (round-1 kernel)
    double y = rsq(x);
    double g = x * y, hh = 0.5 * y;
    double r = fma(-g, hh, 0.5);
    g = fma(g, r, g);
    hh = fma(hh, r, hh);
    r = fma(-g, hh, 0.5);
    return fma(g, r, g);
}
__device__ __forceinline__ double sqrt5(double x) {   // one step with the 2nd-order correction
    double y = rsq(x);
    double t = x * y;
    double e = fma(-t, y, 1.0);
    double q = e * fma(e, 0.375, 0.5);
    return fma(t, q, t);
}
__device__ __forceinline__ double sqrt6(double x) {   // one step with the 3rd-order correction
    double y = rsq(x);
    double t = x * y;
    double e = fma(-t, y, 1.0);
    double q = e * fma(e, fma(e, 0.3125, 0.375), 0.5);
    return fma(t, q, t);
}
__device__ __forceinline__ uint64_t rng(uint64_t &s) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s;
}
__global__ void probe(int n, unsigned long long *maxulp, double *maxseed, long long *hist) {
    uint64_t s = 0x9E3779B97F4A7C15ull ^ (blockIdx.x * 1315423911ull + threadIdx.x * 2654435761ull);
    unsigned long long m7 = 0, m5 = 0, m6 = 0;
    double ms = 0;
    for (int i = 0; i < n; ++i) {
        // random positive doubles over a wide exponent range and every mantissa
        uint64_t bits = (rng(s) & 0x000FFFFFFFFFFFFFull) | ((uint64_t)(900 + rng(s) % 250) << 52);
        double x = __longlong_as_double((long long)bits);
        double r = __dsqrt_rn(x);
        long long rb = __double_as_longlong(r);
        long long d7 = __double_as_longlong(sqrt7(x)) - rb, d5 = __double_as_longlong(sqrt5(x)) - rb,
                  d6 = __double_as_longlong(sqrt6(x)) - rb;
        d7 = d7 < 0 ? -d7 : d7; d5 = d5 < 0 ? -d5 : d5; d6 = d6 < 0 ? -d6 : d6;
        m7 = d7 > m7 ? d7 : m7; m5 = d5 > m5 ? d5 : m5; m6 = d6 > m6 ? d6 : m6;
        if (d5 < 4) atomicAdd((unsigned long long *)&hist[d5], 1ull); else atomicAdd((unsigned long long *)&hist[4], 1ull);
        double e = fabs(rsq(x) * r - 1.0);
        ms = e > ms ? e : ms;
    }
    atomicMax(&maxulp[0], m7);
    atomicMax(&maxulp[1], m5);
    atomicMax(&maxulp[2], m6);
    atomicMax((unsigned long long *)maxseed, (unsigned long long)__double_as_longlong(ms));
}
int main() {
    unsigned long long *mu; double *msd; long long *h;
    cudaMallocManaged(&mu, 3 * 8); cudaMallocManaged(&msd, 8); cudaMallocManaged(&h, 5 * 8);
    for (int k = 0; k < 3; ++k) mu[k] = 0;
    *msd = 0; for (int k = 0; k < 5; ++k) h[k] = 0;
    probe<<<148 * 4, 256>>>(2000, mu, msd, h);
    cudaDeviceSynchronize();
    printf("samples %lld\n", 148LL * 4 * 256 * 2000);
    printf("max ulp vs __dsqrt_rn: sqrt7 (Goldschmidt x2) %llu, sqrt5 (1 step + e^2) %llu, sqrt6 (+e^3) %llu\n",
           mu[0], mu[1], mu[2]);
    printf("rsqrt.approx.f64 seed max rel error %.3e (2^%.1f)\n", *msd, __builtin_log2(*msd));
    printf("sqrt5 ulp histogram 0:%lld 1:%lld 2:%lld 3:%lld >=4:%lld\n", h[0], h[1], h[2], h[3], h[4]);
    return 0;
}
