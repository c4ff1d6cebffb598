// Device-resident pipeline state: PLS -> discretize -> Gauss sum -> rounding.
#pragma once
#include "gauss.cuh"

namespace lc {

// Pinned host staging buffer (grow-only).
struct PinnedBuf {
    void *ptr = nullptr;
    size_t bytes = 0;
    void reserve(size_t n) {
        if (n <= bytes) return;
        if (ptr) cudaFreeHost(ptr);
        size_t want = n < 4096 ? 4096 : n + n / 4;
        LC_CUDA(cudaHostAlloc(&ptr, want, cudaHostAllocDefault));
        bytes = want;
    }
    void release() {
        if (ptr) cudaFreeHost(ptr);
        ptr = nullptr;
        bytes = 0;
    }
    template <class T> T *as() const { return static_cast<T *>(ptr); }
};

struct Pipeline {
    cudaStream_t s = nullptr;

    // Gauss input: closed SoA polylines, scaled by 2^-e (exact).
    DevBuf d_aos, d_in_off, d_voff, d_X, d_Y, d_Z, d_exp;
    int64_t L = 0, V = 0, Vc = 0;
    std::vector<int64_t> h_voff;

    // Pair list (i < j), int32 x 2.
    DevBuf d_pairs;
    int64_t P = 0;

    // Work items and results.
    DevBuf d_pg, d_item_off, d_scan, d_counter, d_partials, d_raw, d_lk, d_flags, d_quads, d_qout;
    int64_t n_items = 0;

    PinnedBuf h_stage;

    void init(cudaStream_t st);
    void set_stream(cudaStream_t st) { s = st; }
    void release();

    void upload_polylines(const double *verts, const int64_t *vert_off, int64_t nloops);
    void upload_pairs(const int32_t *pairs, int64_t npairs);
    void build_gauss_items();
    void run_gauss(int mode, int64_t item_begin, int64_t item_end, double *partials_ext, cudaEvent_t ev0,
                   cudaEvent_t ev1);
    void reduce_pairs(const double *partials_ext);
    void download_results(double *raw, int64_t *lk, uint8_t *flags);
    void segment_pair_lambda(const double *quads, int64_t n, double *out);
};

}  // namespace lc
