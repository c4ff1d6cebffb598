// Device-resident pipeline state: PLS -> discretize -> Gauss sum -> rounding.
#pragma once
#include <vector>

#include "discretize.cuh"
#include "gauss.cuh"
#include "pls.cuh"

namespace lc {

enum StageEvent : int { EV_BEGIN = 0, EV_PLS, EV_DISC, EV_GAUSS0, EV_GAUSS1, EV_END, EV_COUNT };

struct Pipeline {
    cudaStream_t s = nullptr;
    cudaEvent_t ev[EV_COUNT] = {};

    // Model: packed monomial cubics (linkcert LoopGeometry arrays, geometry.py:206-296).
    DevBuf d_coeffs, d_t, d_loff, d_seg_box, d_seg_loop, d_loop_box, d_min_diag, d_model_exp, d_verts_in;
    int64_t L = 0, M = 0;
    bool model_ready = false;

    PlsScratch pls_sc;
    DiscScratch disc_sc;
    DiscOutput dout;
    DiscError derr;

    // Gauss input (closed SoA, scaled by 2^-e): from discretize() or upload_polylines().
    const double *gX = nullptr, *gY = nullptr, *gZ = nullptr;
    const int64_t *gvoff = nullptr;
    bool polylines_ready = false;
    bool polylines_from_model = false;

    // upload_polylines() buffers
    DevBuf d_aos, d_in_off, d_voff, d_X, d_Y, d_Z, d_exp, d_tmp_aos;
    int64_t V = 0, Vc = 0;
    std::vector<int64_t> h_voff;

    // Pair list (i < j), int32 x 2.
    DevBuf d_pairs;
    int64_t P = 0;

    // Work items and results.
    DevBuf d_pg, d_item_off, d_item_pair, d_scan, d_counter, d_partials, d_raw, d_lk, d_flags, d_quads, d_qout;
    int64_t n_items = 0;

    void init(cudaStream_t st);
    void set_stream(cudaStream_t st) { s = st; }
    void release();

    // model + stages
    void upload_model(const double *coeffs, const double *t, const int64_t *loff, int64_t nloops);
    // closed polylines given as vertices only (a0 = v_k, a1 = v_k+1 - v_k, a2 = a3 = 0, t = [0, 1])
    void upload_model_polylines(const double *verts, const int64_t *loff, int64_t nloops);
    int64_t potential_link_search(const uint64_t *excl_keys, int64_t n_excl);   // -> d_pairs, P
    bool discretize(const DiscParams &prm);                                      // -> dout = gauss input
    void download_loop_boxes(double *lo, double *hi);
    void download_polylines(double *verts, int64_t *vert_off);

    // gauss
    void upload_polylines(const double *verts, const int64_t *vert_off, int64_t nloops);
    void upload_pairs(const int32_t *pairs, int64_t npairs);
    void download_pairs(int32_t *pairs);
    void build_gauss_items();
    // build items and read back n_items together with a deferred discretize
    // validation result (one sync); false + derr on a ValidationError
    bool build_gauss_items_checked();
    void run_gauss(int mode, int64_t item_begin, int64_t item_end, double *partials_ext, cudaEvent_t ev0,
                   cudaEvent_t ev1);
    void reduce_pairs(const double *partials_ext);
    void download_results(double *raw, int64_t *lk, uint8_t *flags);
    // pairs | raw | lk | flags of the last reduce into pinned host memory (one sync)
    void download_results_pinned();
    PinnedBuf h_res;
    int64_t h_res_P = -1;
    void segment_pair_lambda(const double *quads, int64_t n, double *out);

    float stage_ms(int e0, int e1);

  private:
    void model_boxes();
    void finish_items();
};

}  // namespace lc
