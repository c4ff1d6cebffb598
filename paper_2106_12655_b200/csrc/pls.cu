// Device potential-link search: tight segment boxes -> loop AABBs ->
// sort-and-sweep -> sorted unique (i<j) loop pairs.
//
// Reference: linkcert/pls.py:48-73 (loop_boxes, potential_link_search),
// bvh.py:93-98 (closed-interval overlap), bvh.py:227-243 (the broad phase it
// replaces; only the resulting SET matters, the caller sorts).  The pair set
// is exact: the sweep visits every pair whose sweep-axis intervals overlap
// (for two overlapping closed intervals, one lower end lies inside the
// other interval) and then applies the full 3-axis closed test.
#include <climits>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "geom.cuh"
#include "pls.cuh"

namespace lc {
namespace {

__global__ void seg_boxes_kernel(const double *__restrict__ coeffs, const double *__restrict__ t,
                                 const int64_t *__restrict__ loff, int64_t L, int64_t M, double min_diam,
                                 double *__restrict__ box, int32_t *__restrict__ seg_loop, int *zero_loop) {
    const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= M) return;
    int64_t lo = 0, hi = L;   // loop: largest l with loff[l] <= m
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (loff[mid] <= m) lo = mid; else hi = mid;
    }
    seg_loop[m] = (int32_t)lo;
    double bl[3], bh[3];
    tight_box(coeffs + 12 * m, t[2 * m], t[2 * m + 1], bl, bh);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        box[d * M + m] = bl[d];
        box[(3 + d) * M + m] = bh[d];
    }
    if (diag_norm(bl, bh) < min_diam) atomicMin(zero_loop, (int)lo);
}

__global__ void loop_boxes_kernel(const double *__restrict__ box, int64_t M, const int64_t *__restrict__ loff,
                                  int64_t L, double *__restrict__ lbox) {
    const int64_t l = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (l >= L) return;
    double v[6];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        v[d] = CUDART_INF;
        v[3 + d] = -CUDART_INF;
    }
    for (int64_t m = loff[l] + lane; m < loff[l + 1]; m += 32) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            v[d] = np_min(v[d], box[d * M + m]);
            v[3 + d] = np_max(v[3 + d], box[(3 + d) * M + m]);
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            v[d] = np_min(v[d], __shfl_xor_sync(0xffffffffu, v[d], off));
            v[3 + d] = np_max(v[3 + d], __shfl_xor_sync(0xffffffffu, v[3 + d], off));
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < 6; ++d) lbox[d * L + l] = v[d];
    }
}

// One block: axis of the largest model extent -> *axis; keys[l] = lo_axis[l], idx[l] = l.
__global__ void sweep_axis_kernel(const double *__restrict__ lbox, int64_t L, int *axis, double *keys,
                                  int32_t *idx) {
    __shared__ double red[6][32];
    double v[6] = {CUDART_INF, CUDART_INF, CUDART_INF, -CUDART_INF, -CUDART_INF, -CUDART_INF};
    for (int64_t l = threadIdx.x; l < L; l += blockDim.x) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            v[d] = fmin(v[d], lbox[d * L + l]);
            v[3 + d] = fmax(v[3 + d], lbox[(3 + d) * L + l]);
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            v[d] = fmin(v[d], __shfl_xor_sync(0xffffffffu, v[d], off));
            v[3 + d] = fmax(v[3 + d], __shfl_xor_sync(0xffffffffu, v[3 + d], off));
        }
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0)
        for (int d = 0; d < 6; ++d) red[d][w] = v[d];
    __syncthreads();
    __shared__ int s_axis;
    if (threadIdx.x == 0) {
        for (int k = 1; k < nw; ++k)
            for (int d = 0; d < 3; ++d) {
                red[d][0] = fmin(red[d][0], red[d][k]);
                red[3 + d][0] = fmax(red[3 + d][0], red[3 + d][k]);
            }
        int a = 0;
        double best = red[3][0] - red[0][0];
        for (int d = 1; d < 3; ++d) {
            const double e = red[3 + d][0] - red[d][0];
            if (e > best) { best = e; a = d; }
        }
        s_axis = a;
        *axis = a;
    }
    __syncthreads();
    const int a = s_axis;
    for (int64_t l = threadIdx.x; l < L; l += blockDim.x) {
        keys[l] = lbox[a * L + l];
        idx[l] = (int32_t)l;
    }
}

__device__ __forceinline__ bool boxes_overlap(const double *__restrict__ b, int64_t n, int64_t i, int64_t j) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        // alo > bhi or blo > ahi -> disjoint (bvh.py:93-98)
        if (b[d * n + i] > b[(3 + d) * n + j] || b[d * n + j] > b[(3 + d) * n + i]) return false;
    }
    return true;
}

__device__ __forceinline__ bool is_excluded(const uint64_t *__restrict__ ex, int64_t n, uint64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const uint64_t v = ex[mid];
        if (v == key) return true;
        if (v < key) lo = mid + 1; else hi = mid;
    }
    return false;
}

template <bool WRITE>
__global__ void sweep_kernel(const double *__restrict__ lbox, int64_t L, const int *__restrict__ axis,
                             const double *__restrict__ skeys, const int32_t *__restrict__ perm,
                             const uint64_t *__restrict__ excl, int64_t n_excl, int64_t *__restrict__ counts,
                             const int64_t *__restrict__ offs, uint64_t *__restrict__ out) {
    const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= L) return;
    const int ax = *axis;
    const int64_t ia = perm[a];
    const double hia = lbox[(3 + ax) * L + ia];
    int64_t c = 0;
    int64_t w = WRITE ? offs[a] : 0;
    for (int64_t b = a + 1; b < L && skeys[b] <= hia; ++b) {
        const int64_t ib = perm[b];
        if (!boxes_overlap(lbox, L, ia, ib)) continue;
        const uint64_t i = ia < ib ? ia : ib, j = ia < ib ? ib : ia;
        const uint64_t key = (i << 32) | j;
        if (n_excl && is_excluded(excl, n_excl, key)) continue;
        if (WRITE) out[w++] = key;
        else ++c;
    }
    if (!WRITE) counts[a] = c;
}

__global__ void unpack_pairs_kernel(const uint64_t *__restrict__ keys, int64_t P, int32_t *__restrict__ pairs) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    const uint64_t k = keys[p];
    pairs[2 * p] = (int32_t)(k >> 32);
    pairs[2 * p + 1] = (int32_t)(k & 0xffffffffu);
}

}  // namespace

void launch_seg_boxes(const double *coeffs, const double *t, const int64_t *loff, int64_t L, int64_t M,
                      double min_diam, double *seg_box, int32_t *seg_loop, int *zero_loop, cudaStream_t s) {
    const int init = INT_MAX;
    LC_CUDA(cudaMemcpyAsync(zero_loop, &init, sizeof(int), cudaMemcpyHostToDevice, s));
    if (M == 0) return;
    seg_boxes_kernel<<<(unsigned)ceil_div(M, 128), 128, 0, s>>>(coeffs, t, loff, L, M, min_diam, seg_box,
                                                                   seg_loop, zero_loop);
    LC_CHECK_LAUNCH();
}

void launch_loop_boxes(const double *seg_box, int64_t M, const int64_t *loff, int64_t L, double *loop_box,
                       cudaStream_t s) {
    if (L == 0) return;
    loop_boxes_kernel<<<(unsigned)ceil_div(L * 32, 256), 256, 0, s>>>(seg_box, M, loff, L, loop_box);
    LC_CHECK_LAUNCH();
}

int64_t run_pls(const double *loop_box, int64_t L, const uint64_t *h_excl, int64_t n_excl, PlsScratch &sc,
                DevBuf &pairs, cudaStream_t s) {
    if (L < 2) return 0;
    sc.keys.reserve(sizeof(double) * L, s);
    sc.keys_sorted.reserve(sizeof(double) * L, s);
    sc.idx.reserve(sizeof(int32_t) * L, s);
    sc.perm.reserve(sizeof(int32_t) * L, s);
    sc.counts.reserve(sizeof(int64_t) * (L + 1), s);
    sc.offs.reserve(sizeof(int64_t) * (L + 1), s);
    sc.axis.reserve(sizeof(int), s);
    sc.excl.reserve(sizeof(uint64_t) * (n_excl > 0 ? n_excl : 1), s);
    if (n_excl > 0)
        LC_CUDA(cudaMemcpyAsync(sc.excl.ptr, h_excl, sizeof(uint64_t) * n_excl, cudaMemcpyHostToDevice, s));

    sweep_axis_kernel<<<1, 1024, 0, s>>>(loop_box, L, sc.axis.as<int>(), sc.keys.as<double>(), sc.idx.as<int32_t>());
    LC_CHECK_LAUNCH();
    size_t b1 = 0, b2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b1, (double *)nullptr, (double *)nullptr, (int32_t *)nullptr,
                                    (int32_t *)nullptr, (int)L);
    cub::DeviceScan::ExclusiveSum(nullptr, b2, (int64_t *)nullptr, (int64_t *)nullptr, (int)(L + 1));
    sc.cub_tmp.reserve(b1 > b2 ? b1 : b2, s);
    size_t bytes = sc.cub_tmp.bytes;
    LC_CUB(cub::DeviceRadixSort::SortPairs(sc.cub_tmp.ptr, bytes, sc.keys.as<double>(), sc.keys_sorted.as<double>(),
                                            sc.idx.as<int32_t>(), sc.perm.as<int32_t>(), (int)L, 0, 64, s));
    const unsigned grid = (unsigned)ceil_div(L, 128);
    LC_CUDA(cudaMemsetAsync(sc.counts.as<int64_t>() + L, 0, sizeof(int64_t), s));
    sweep_kernel<false><<<grid, 128, 0, s>>>(loop_box, L, sc.axis.as<int>(), sc.keys_sorted.as<double>(),
                                             sc.perm.as<int32_t>(), sc.excl.as<uint64_t>(), n_excl,
                                             sc.counts.as<int64_t>(), nullptr, nullptr);
    LC_CHECK_LAUNCH();
    bytes = sc.cub_tmp.bytes;
    LC_CUB(cub::DeviceScan::ExclusiveSum(sc.cub_tmp.ptr, bytes, sc.counts.as<int64_t>(), sc.offs.as<int64_t>(),
                                          (int)(L + 1), s));
    int64_t P = 0;
    LC_CUDA(cudaMemcpyAsync(&P, sc.offs.as<int64_t>() + L, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
    if (P == 0) return 0;
    sc.pair_keys.reserve(sizeof(uint64_t) * P, s);
    sc.pair_keys_sorted.reserve(sizeof(uint64_t) * P, s);
    sweep_kernel<true><<<grid, 128, 0, s>>>(loop_box, L, sc.axis.as<int>(), sc.keys_sorted.as<double>(),
                                            sc.perm.as<int32_t>(), sc.excl.as<uint64_t>(), n_excl, nullptr,
                                            sc.offs.as<int64_t>(), sc.pair_keys.as<uint64_t>());
    LC_CHECK_LAUNCH();
    size_t b3 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b3, (uint64_t *)nullptr, (uint64_t *)nullptr, (int)P);
    sc.cub_tmp.reserve(b3, s);
    bytes = sc.cub_tmp.bytes;
    LC_CUB(cub::DeviceRadixSort::SortKeys(sc.cub_tmp.ptr, bytes, sc.pair_keys.as<uint64_t>(),
                                           sc.pair_keys_sorted.as<uint64_t>(), (int)P, 0, 64, s));
    pairs.reserve(sizeof(int32_t) * 2 * P, s);
    unpack_pairs_kernel<<<(unsigned)ceil_div(P, 256), 256, 0, s>>>(sc.pair_keys_sorted.as<uint64_t>(), P,
                                                                     pairs.as<int32_t>());
    LC_CHECK_LAUNCH();
    return P;
}

}  // namespace lc
