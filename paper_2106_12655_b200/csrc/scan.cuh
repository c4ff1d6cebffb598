// Exclusive int64 scans of the pipeline's index arrays (cell counts, per-row
// pair counts, items per pair): cub::DeviceScan (decoupled look-back).  A
// single-block tiled scan (50 us: strided loads) and a one-kernel cooperative
// scan (grid barrier; no faster than CUB's init + scan at 14k-300k elements)
// were measured and dropped.  In place is allowed.
#pragma once
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace lc {

inline size_t exclusive_scan_i64_tmp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int64_t *)nullptr, (int64_t *)nullptr, (int)(n > 0 ? n : 1));
    return bytes;
}

inline void exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, void *tmp, size_t tmp_bytes,
                               cudaStream_t s) {
    if (n <= 0) return;
    size_t bytes = tmp_bytes;
    LC_CUB(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int)n, s));
}

}  // namespace lc
