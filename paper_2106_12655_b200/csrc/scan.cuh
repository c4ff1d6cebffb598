// Exclusive int64 scans of the pipeline's small index arrays (cell counts,
// per-row pair counts, items per pair).  Up to kSmallScanMax elements one
// 1024-thread block walks the array in 16k tiles (a block scan per tile plus
// a running carry): one launch, no tile-status initialisation — the cost of
// CUB's decoupled look-back (init + scan kernels) is pure latency at these
// sizes.  Larger arrays go to cub::DeviceScan.  In place is allowed.
#pragma once
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace lc {

constexpr int kSmallScanThreads = 1024;
constexpr int kSmallScanItems = 16;
constexpr int64_t kSmallScanMax = 0;   // single-block path disabled: its strided loads measured 50 us / scan (CUB: 9 us)

template <int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS) small_exclusive_scan_kernel(const int64_t *in, int64_t *out, int64_t n) {
    using BlockScan = cub::BlockScan<long long, THREADS>;
    __shared__ typename BlockScan::TempStorage tmp;
    long long carry = 0;
    for (int64_t base = 0; base < n; base += (int64_t)THREADS * ITEMS) {
        const int64_t b = base + (int64_t)threadIdx.x * ITEMS;
        long long v[ITEMS], sum = 0;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            v[k] = b + k < n ? (long long)in[b + k] : 0;
            sum += v[k];
        }
        long long pre, total;
        BlockScan(tmp).ExclusiveSum(sum, pre, total);
        __syncthreads();   // every thread read its tile before anyone writes (in place) / tmp reuse
        long long run = carry + pre;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            if (b + k < n) out[b + k] = run;
            run += v[k];
        }
        carry += total;
    }
}

// Temporary bytes the CUB fallback needs for n elements (0 on the small path).
inline size_t exclusive_scan_i64_tmp_bytes(int64_t n) {
    if (n <= kSmallScanMax) return 0;
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int64_t *)nullptr, (int64_t *)nullptr, (int)n);
    return bytes;
}

inline void exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, void *tmp, size_t tmp_bytes,
                               cudaStream_t s) {
    if (n <= 0) return;
    if (n <= kSmallScanMax) {
        small_exclusive_scan_kernel<kSmallScanThreads, kSmallScanItems><<<1, kSmallScanThreads, 0, s>>>(in, out, n);
        LC_CHECK_LAUNCH();
        return;
    }
    size_t bytes = tmp_bytes;
    LC_CUB(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int)n, s));
}

}  // namespace lc
