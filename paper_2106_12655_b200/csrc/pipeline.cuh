// Device-resident pipeline state: PLS -> discretize -> Gauss sum -> rounding.
#pragma once
#include <vector>

#include "discretize.cuh"
#include "gauss.cuh"
#include "pls.cuh"

namespace lc {

// Device-written summary of a fused run (lives at the head of the pinned result buffer).
struct FastStatus {
    int64_t P, n_items;
    int max_row, zero_loop, n_unpaired, n_large;
    unsigned long long marked;
    int val_err[2];
    unsigned long long first_fail;   // early exit: place of the first failing pair (~0: none)
    unsigned long long n_eval;       // early exit: pairs evaluated
};

enum FastResult : int { FAST_OK = 0, FAST_FALLBACK = 1, FAST_INVALID = 2, FAST_PENDING = 3 };

enum StageEvent : int { EV_BEGIN = 0, EV_PLS, EV_DISC, EV_GAUSS0, EV_GAUSS1, EV_END, EV_COUNT };

struct Pipeline {
    cudaStream_t s = nullptr;
    cudaEvent_t ev[EV_COUNT] = {};
    // fused run: side branches (chord write || PLS; pass-1 checks || items + Gauss sum)
    cudaStream_t side[2] = {};
    cudaEvent_t ev_fork = nullptr, ev_chords = nullptr, ev_pairs = nullptr, ev_checks = nullptr;
    cudaStream_t crit = nullptr;                          // fused run's critical path (highest priority)
    cudaEvent_t ev_enter = nullptr, ev_leave = nullptr;   // caller stream <-> crit joins

    // Model: packed monomial cubics (linkcert LoopGeometry arrays, geometry.py:206-296).
    DevBuf d_coeffs, d_t, d_loff, d_seg_box, d_seg_fbox, d_seg_sub, d_loop_keys, d_seg_loop, d_loop_box, d_min_diag, d_model_exp, d_verts_in;
    int64_t L = 0, M = 0;
    int64_t max_loop = -1;       // most segments in one loop (host-known at upload)
    bool model_ready = false;
    bool model_poly = false;     // uploaded as closed-polyline vertices (d_verts_in)
    bool coeffs_ready = false;   // d_coeffs/d_t hold the model (polyline models: formed on demand)
    bool derived = false;        // segment/loop boxes of the current model
    bool derived_in_run = false; // derive() ran during the current lc_run_pipeline

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
    DevBuf d_tot, d_pg, d_item_off, d_item_pair, d_scan, d_counter, d_partials, d_raw, d_lk, d_flags, d_quads, d_qout;
    int64_t n_items = 0;

    void init(cudaStream_t st);
    void set_stream(cudaStream_t st) { s = st; }
    void release();

    // model + stages
    // Segment boxes, loop boxes, min diagonals and the coordinate exponent from
    // the resident model (records EV_BEGIN first).  Every lc_run_pipeline runs it.
    void derive();
    void ensure_derived() {
        if (!derived) derive();
    }
    void ensure_coeffs();
    void reserve_derived();   // the derive() outputs' buffers (the fused path derives in two halves)
    void upload_model(const double *coeffs, const double *t, const int64_t *loff, int64_t nloops);
    // closed polylines given as vertices only (a0 = v_k, a1 = v_k+1 - v_k, a2 = a3 = 0, t = [0, 1])
    void upload_model_polylines(const double *verts, const int64_t *loff, int64_t nloops);
    // the same from one vertex array per loop: gathered on host threads into a
    // library-owned pinned staging buffer and copied asynchronously (no host sync;
    // the next gather waits only for the previous copy)
    void upload_model_polyline_ptrs(const double *const *loop_verts, const int64_t *loff, int64_t nloops);
    PinnedBuf h_stage;
    cudaEvent_t ev_stage = nullptr;
    bool stage_pending = false;
    // -> d_pairs, P; in_run: EV_BEGIN already recorded by derive() of this run
    int64_t potential_link_search(const uint64_t *excl_keys, int64_t n_excl, bool in_run = false);
    bool discretize(const DiscParams &prm);                                      // -> dout = gauss input
    void download_loop_boxes(double *lo, double *hi);
    void download_polylines(double *verts, int64_t *vert_off);

    // gauss
    void upload_polylines(const double *verts, const int64_t *vert_off, int64_t nloops);
    void upload_pairs(const int32_t *pairs, int64_t npairs);
    void download_pairs(int32_t *pairs);
    // items for Gauss mode `mode` (the sequential anglesum mode has its own tiling)
    void build_gauss_items(int mode = GAUSS_PHASE);
    // build items and read back n_items together with a deferred discretize
    // validation result (one sync); false + derr on a ValidationError
    bool build_gauss_items_checked(int mode = GAUSS_PHASE);
    // Device early exit of verify(early_exit=True): the certificate's sorted keys and values
    DevBuf d_ref_keys, d_ref_lk, d_posv, d_want, d_ee;
    int64_t n_ref = 0;
    bool ee_on = false;
    // fused runs record only the Gauss-stage events unless stage_detail (or the env
    // LINKCERT_STAGE_TIMES=1): an external event-record node costs ~0.8 us of graph
    // launch; last_detail = the last run recorded every stage event
    bool stage_detail = false, last_detail = true;
    int64_t ee_first_fail = -1, ee_n_eval = -1;   // last fused run (-1: not an early-exit run)
    void set_early_exit(const uint64_t *keys, const int64_t *lk, int64_t n, bool enable);
    bool items_seq = false;   // the current items are whole-row (sequential-mode) items
    bool items_ready = false; // d_item_pair holds the item records of the current pairs
    void run_gauss(int mode, int64_t item_begin, int64_t item_end, double *partials_ext, cudaEvent_t ev0,
                   cudaEvent_t ev1);
    void reduce_pairs(const double *partials_ext);
    void download_results(double *raw, int64_t *lk, uint8_t *flags);
    // pairs | raw | lk | flags of the last reduce into pinned host memory (one sync)
    void download_results_pinned();
    PinnedBuf h_res;
    int64_t h_res_P = -1;
    bool fused_shard_pending = false;   // run_fast(shards > 1) left res_* for shard_reduce to fill
    char *res_pairs = nullptr, *res_raw = nullptr, *res_lk = nullptr, *res_flags = nullptr;

    // Fused pipeline: PLS -> discretize (no-refinement case) -> items -> Gauss
    // sum -> rounding -> results into pinned memory with one host sync.  Sizes
    // stay on the device (capacity-bounded grids); the summary decides whether
    // the run was the reference's: FAST_OK (results in h_res), FAST_INVALID
    // (PolylineLoop ValidationError in derr), FAST_FALLBACK (the model needs
    // refinement / the sweep path / larger buffers: run the staged pipeline).
    // shards > 1 (or force_sharded): the Gauss kernel evaluates only the
    // cost-balanced item range of `shard` (launch_shard_bounds) into d_partials at
    // absolute item ids and the sums wait for the exchange + shard_finish().
    // async: enqueue the run and return FAST_PENDING without a
    // host sync; the item partials not owned by this shard hold the bits of -0.0
    // (INT64_MIN), so an int64 MAX all-reduce of d_partials assembles every
    // shard's items exactly; shard_finish() then reduces, exports and syncs once.
    int run_fast(const uint64_t *excl_keys, int64_t n_excl, const DiscParams &prm, int mode, int shard = 0,
                 int shards = 1, bool async = false, bool force_sharded = false);
    int shard_finish();
    int gather_share = 1;         // ranks sharing this host (host gather threads / rank)
    void prefill_partials_neg_zero(int64_t n);   // d_partials[0, n) <- bits of -0.0 (staged sharded path)
    int64_t part_cap = 0;   // d_partials entries of the last run (item capacity)
    DevBuf d_bounds;        // cost-balanced shard boundaries of the item list (shards + 1)
    // staged path: cost-balanced bounds of the current items (device d_bounds; out: host copy, may be null)
    void shard_bounds(int shards, int64_t *out);
    int64_t items_cap = 0;
    int64_t pairs_seen = 0;   // largest pair count of a fused run (sizes the next run's capacity)
    // The fused sequence is replayed as a CUDA graph once a run with the same
    // shape (FastKey) and the same buffer generation has completed uncaptured.
    struct FastKey {
        int64_t L, M, pcap, icap, n_excl;
        int mode, model_poly, shard, shards;
        double min_diam, poly_thr;
        unsigned long long gen;
        int64_t n_ref;   // early-exit certificate size (-1: off)
        bool detail;     // every stage event recorded
        bool operator==(const FastKey &o) const {
            return L == o.L && M == o.M && pcap == o.pcap && icap == o.icap && n_excl == o.n_excl &&
                   mode == o.mode && model_poly == o.model_poly && shard == o.shard && shards == o.shards &&
                   min_diam == o.min_diam && poly_thr == o.poly_thr && gen == o.gen && n_ref == o.n_ref &&
                   detail == o.detail;
        }
    };
    FastKey fast_seen{}, graph_key{};
    // state of an enqueued fused run between run_fast and finish_fast
    struct Pending {
        bool on = false;
        FastKey key{};
        int64_t pcap = 0, icap = 0;
        int shards = 1;
        bool sharded = false;
        FastStatus *st = nullptr;
        char *hp = nullptr, *hr = nullptr, *hl = nullptr, *hf = nullptr;
    } pend;
    int finish_fast();
    bool fast_seen_valid = false;
    cudaGraphExec_t graph_exec = nullptr;
    long long graph_launches = 0;   // kernels inside the captured graph (lc_launch_count)
    PinnedBuf h_excl;               // excluded keys staged for the graph's H2D copy
    bool last_fast_graph = false;
    void segment_pair_lambda(const double *quads, int64_t n, double *out);
    void retile_few_items();   // build_gauss_items*: more, shorter items when there are very few
    // link_direct of two open-vertex loops (direct.py:149-161): closed scaled SoA and the
    // pair's work items built on the host, one H2D copy, the items kernel, the fixed-order
    // reduction, one D2H of the raw sum; the resident model is left untouched
    double link_direct(const double *loop1, int64_t n1, const double *loop2, int64_t n2, int mode,
                       cudaEvent_t ev0, cudaEvent_t ev1);
    PinnedBuf h_ld;
    DevBuf d_ld, d_ld_out;

    float stage_ms(int e0, int e1);
    void record(int e, cudaStream_t st = nullptr);

  private:
    void finish_items();
};

}  // namespace lc
