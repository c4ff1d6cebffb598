/*
 * linkcert_b200 — C-ABI of the B200-native direct-summation Gauss linking
 * number path (arXiv 2106.12655; reference package `linkcert`).
 *
 * Conventions
 *   - Every int-returning call returns 0 (LC_OK) on success or an LC_ERR_*
 *     code; lc_last_error() then holds a thread-local message.
 *   - Host pointers are caller-owned and only read/written during the call.
 *     Calls marked [device] take device pointers and are stream-ordered on
 *     the context's stream.
 *   - Vertex buffers are float64 AoS (n, 3), C order, WITHOUT the closing
 *     vertex (the library closes every loop, linkcert/direct.py:164-166).
 *     vert_off has L+1 entries, vert_off[0] == 0; loop v owns rows
 *     [vert_off[v], vert_off[v+1]).
 *   - Pair lists are int32 (P, 2) rows (i, j), i < j — linkcert PairList
 *     (pls.py:17-45).  For pair (i, j) the sum is link_direct(loop i, loop j)
 *     (certify.py:114): loop i is the inner loop `l`, loop j the outer `k`.
 *   - Results are deterministic: bitwise identical run to run and for any
 *     split of the work-item range across GPUs.
 *   - Calls on one context are serialized; contexts are independent.
 */
#ifndef LINKCERT_B200_H
#define LINKCERT_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define LC_API __attribute__((visibility("default")))
#else
#define LC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define LC_ABI_VERSION 2

enum {
    LC_OK = 0,
    LC_ERR_CUDA = 1,
    LC_ERR_ARG = 2,
    LC_ERR_STATE = 3,
    LC_ERR_DISCRETIZE = 4,
    LC_ERR_VALIDATION = 5
};

/* Arithmetic variant of the Gauss-sum kernel (all FP64). */
enum {
    LC_GAUSS_PHASE = 0, /* default: shared corner terms + turn-counted phase product */
    LC_GAUSS_ATAN = 1,  /* shared corner terms + one fused atan2 per segment pair   */
    LC_GAUSS_REF = 2,   /* reference formula per pair, no FMA, two atan2            */
    LC_GAUSS_ANGLESUM = 3 /* the reference's "anglesum" variant (direct.py:75-134):
                             lane per outer segment, phase product over the inner
                             segments in order, one atan2 per outer segment;
                             its work items differ (lc_prepare_gauss(mode))      */
};

/* Per-pair result flags (lc_evaluate_pairs flags_out). */
#define LC_FLAG_NAN 1u       /* raw is NaN: round() raises ValueError (kernels.py:68) */
#define LC_FLAG_AMBIGUOUS 2u /* |raw - rint(raw)| > 0.25 (kernels.py:19-20,69-72)     */

typedef struct lc_ctx lc_ctx;

LC_API int lc_abi_version(void);
LC_API const char *lc_last_error(void);
LC_API int lc_device_count(int *count);

/* One context per device; owns a non-blocking stream and cached device buffers. */
LC_API lc_ctx *lc_create(int device);
LC_API void lc_destroy(lc_ctx *ctx);
/* Use a caller stream (e.g. torch.cuda.current_stream().cuda_stream); NULL = own stream. */
LC_API int lc_set_stream(lc_ctx *ctx, void *cuda_stream);
LC_API int lc_synchronize(lc_ctx *ctx);

/* ---- Gauss sum (replaces linkcert/direct.py + certify._evaluate_pairs) ---- */

/* Batched drop-in for certify._evaluate_pairs (certify.py:108-127) with the
 * DS branch of kernels.compute_link (kernels.py:45-73): raw[p] = link_direct
 * of pair p, lk[p] = half-to-even rounding, flags[p] = LC_FLAG_*. */
LC_API int lc_evaluate_pairs(lc_ctx *ctx, const double *verts, const int64_t *vert_off, int64_t L,
                      const int32_t *pairs, int64_t P, int mode, double *raw, int64_t *lk,
                      uint8_t *flags);

/* Drop-in for direct.link_direct(loop1, loop2, "atan") (direct.py:149-161). */
LC_API int lc_link_direct(lc_ctx *ctx, const double *loop1, int64_t n1, const double *loop2, int64_t n2,
                   int mode, double *raw);

/* Drop-in for direct.segment_pair_lambda (direct.py:137-146), batched:
 * quads (n, 12) = (l_j, l_j1, k_i, k_i1) rows; out (n,). */
LC_API int lc_segment_pair_lambda(lc_ctx *ctx, const double *quads, int64_t n, double *out);

/* Duration (CUDA events on the context stream) of the last Gauss-sum kernel. */
LC_API int lc_last_gauss_ms(lc_ctx *ctx, float *ms);

/* Device-resident staging for repeated / sharded evaluation.
 * lc_stage_polylines uploads polylines + pairs and builds the work items.
 * lc_gauss_run evaluates items [item_begin, item_end) [device] into
 * partials_dev (NULL = internal buffer of n_items doubles; an external
 * buffer must hold n_items doubles and is indexed by absolute item id).
 * lc_gauss_reduce reduces all n_items partials per pair in fixed order and
 * copies raw/lk/flags (P each; any may be NULL) to the host. */
LC_API int lc_stage_polylines(lc_ctx *ctx, const double *verts, const int64_t *vert_off, int64_t L,
                       const int32_t *pairs, int64_t P, int mode, int64_t *n_items);
LC_API int lc_gauss_run(lc_ctx *ctx, int mode, int64_t item_begin, int64_t item_end, double *partials_dev);
LC_API int lc_gauss_reduce(lc_ctx *ctx, const double *partials_dev, double *raw, int64_t *lk, uint8_t *flags);
/* The fused path's pair-claiming Gauss kernel over the staged pairs (their raw sums
 * into the library's partials buffer; timing A/B against lc_gauss_run — read the
 * time with lc_gauss_event_ms). */
LC_API int lc_gauss_run_pairs(lc_ctx *ctx, int mode);
/* Duration of the last lc_gauss_run kernel (waits for it). */
LC_API int lc_gauss_event_ms(lc_ctx *ctx, float *ms);

/* ---- Model pipeline: PLS -> discretize -> Gauss sum, device resident ----
 *
 * Model = packed monomial cubics, the arrays of linkcert LoopGeometry
 * (geometry.py:206-296): coeffs (M, 4, 3) float64 (a0..a3 rows), t (M, 2)
 * parameter domains, loop_off (L+1) segment offsets per loop. */
LC_API int lc_model_upload(lc_ctx *ctx, const double *coeffs, const double *t, const int64_t *loop_off,
                           int64_t L);
/* Same model when every loop is a plain closed polyline (LoopGeometry.from_polyline,
 * geometry.py:269-283): only the vertices (M, 3) travel; the device builds
 * a0 = v_k, a1 = v_{k+1} - v_k, a2 = a3 = 0, t = [0, 1] (bitwise the host arrays). */
LC_API int lc_model_upload_polylines(lc_ctx *ctx, const double *verts, const int64_t *loop_off, int64_t L);
/* Same model from one vertex array per loop (loop_verts[l] -> (n_l, 3) rows,
 * n_l = loop_off[l+1] - loop_off[l]) — the arrays of L separate
 * LoopGeometry.from_polyline loops, no host-side packing by the caller: the
 * library gathers them on host threads into its own pinned staging buffer and
 * copies asynchronously (returns before the copy ends; the caller's arrays are
 * no longer read after return). */
LC_API int lc_model_upload_polyline_ptrs(lc_ctx *ctx, const double *const *loop_verts, const int64_t *loop_off,
                                         int64_t L);
/* Drop-in for geometry.tight_boxes (geometry.py:113-152): coeffs (m,4,3),
 * t (m,2) domains -> lo, hi (m,3).  Independent of the uploaded model. */
LC_API int lc_tight_boxes(lc_ctx *ctx, const double *coeffs, const double *t, int64_t m, double *lo,
                          double *hi);
/* Loop AABBs, unions of tight segment boxes (pls.py:48-56): lo, hi (L, 3). */
LC_API int lc_loop_boxes(lc_ctx *ctx, double *lo, double *hi);
/* Drop-in for pls.potential_link_search (pls.py:59-73): closed-interval box
 * overlap, i < j, minus excluded keys ((min<<32)|max, sorted unique),
 * sorted.  The pair list stays on the device; lc_get_pairs copies it out. */
LC_API int lc_potential_link_search(lc_ctx *ctx, const uint64_t *excluded_keys, int64_t n_excl,
                                    int64_t *n_pairs);
LC_API int lc_get_pairs(lc_ctx *ctx, int32_t *pairs);
/* Replace the device pair list (a caller-built PairList for lc_discretize). */
LC_API int lc_set_pairs(lc_ctx *ctx, const int32_t *pairs, int64_t P);

/* Discretization error kinds (lc_discretize_error). */
enum {
    LC_DISC_OK = 0,
    LC_DISC_ZERO_LENGTH = 1,      /* ZeroLengthInput, loops = (idx,)                 */
    LC_DISC_CURVES_INTERSECT = 2, /* CurvesIntersect, loops = (a, b)                  */
    LC_DISC_SUBSEG_BUDGET = 3,    /* PassLimitExceeded, loops = (i,) max_subsegments  */
    LC_DISC_PASS_BUDGET = 4,      /* PassLimitExceeded, loops = busy, max_passes      */
    LC_DISC_INVALID_POLYLINE = 5  /* ValidationError from PolylineLoop, detail = 1 <3 vertices,
                                     2 non-finite, 3 zero-length segment            */
};
/* Drop-in for discretize.discretize (discretize.py:112-191) over the device
 * model and pair list.  Returns LC_ERR_DISCRETIZE or LC_ERR_VALIDATION for
 * the reference's DiscretizationError / ValidationError; details from
 * lc_discretize_error.  Output polylines stay on the device (they are the
 * Gauss-sum input); lc_get_polylines copies them out (AoS (V,3) + (L+1)). */
LC_API int lc_discretize(lc_ctx *ctx, double xi, double epsilon, int max_passes, int64_t max_subsegments,
                         int64_t *n_vertices, int *passes);
LC_API int lc_discretize_error(lc_ctx *ctx, int *kind, int *detail, int64_t *loops, int64_t cap,
                               int64_t *n_loops);
LC_API int lc_get_polylines(lc_ctx *ctx, double *verts, int64_t *vert_off);
/* Build the Gauss-sum work items of Gauss mode `mode` for the device polylines + pair list. */
LC_API int lc_prepare_gauss(lc_ctx *ctx, int mode, int64_t *n_items);
/* Gauss sum over the device polylines and pair list; results to the host. */
LC_API int lc_evaluate_staged(lc_ctx *ctx, int mode, double *raw, int64_t *lk, uint8_t *flags);
/* Whole device path on the resident model: PLS -> discretize -> items ->
 * Gauss sum -> rounding (certify._prepare + _evaluate_pairs, certify.py:108-138).
 * Results stay on the device; lc_get_pairs / lc_get_results copy them out,
 * lc_result_views exposes them in pinned memory.  Runs the fused single-sync
 * path first (no-refinement models) and the staged path otherwise;
 * LINKCERT_FUSED=0 in the environment forces the staged path. */
LC_API int lc_run_pipeline(lc_ctx *ctx, const uint64_t *excluded_keys, int64_t n_excl, double xi,
                           double epsilon, int max_passes, int64_t max_subsegments, int mode,
                           int64_t *n_pairs);
LC_API int lc_get_results(lc_ctx *ctx, double *raw, int64_t *lk, uint8_t *flags);
/* Zero-copy views of the last lc_run_pipeline results in library-owned pinned
 * memory: pairs int32 (P,2), raw f64 (P), lk int64 (P), flags u8 (P).  Valid
 * until the next pipeline call on this context. */
LC_API int lc_result_views(lc_ctx *ctx, void **pairs, void **raw, void **lk, void **flags, int64_t *n_pairs);
/* ---- Multi-GPU: one process per GPU, all ranks on the same model ----
 * The reference has no distribution (certify.py:117-119 fans pairs over a
 * GIL-bound thread pool); this is the B200 replacement of that fan-out, the
 * multi-device contract of SURVEY §8(b)/(e).  The work-item list is split by
 * COST (segment pairs, lc_shard_bounds) over the ranks; the small per-item
 * partials vector is exchanged in place by an NCCL int64 MAX all-reduce (items
 * of other ranks hold the bits of -0.0) and reduced per pair in a fixed order,
 * so results are bitwise those of one GPU for any world size.
 *
 * Library-owned communicator (no torch.distributed needed):
 *   rank 0: lc_comm_unique_id(id)  -> move the 128 bytes to every rank
 *   every rank: lc_comm_init(ctx, id, world, rank) on its own device's context
 *   every step: lc_model_upload* + lc_run_pipeline_sharded -> lc_result_views
 * NCCL is loaded at run time (the copy already in the process, else
 * libnccl.so.2).  lc_nccl_version: the loaded NCCL's version code, 0 if none. */
LC_API int lc_nccl_version(void);
LC_API int lc_comm_unique_id(char *id_out /* 128 bytes */);
LC_API int lc_comm_init(lc_ctx *ctx, const char *id /* 128 bytes */, int world, int rank);
LC_API int lc_comm_destroy(lc_ctx *ctx);
/* lc_run_pipeline over the communicator: fused single-sync run of this rank's
 * item range with the exchange enqueued behind it on the context stream, or
 * (refinement / sweep PLS / anglesum) the staged path with the same split.
 * Every rank gets the full results (lc_result_views); same return codes. */
LC_API int lc_run_pipeline_sharded(lc_ctx *ctx, const uint64_t *excluded_keys, int64_t n_excl, double xi,
                                   double epsilon, int max_passes, int64_t max_subsegments, int mode,
                                   int64_t *n_pairs);
/* Cost-balanced item ranges of the current work items (after lc_prepare_gauss /
 * lc_stage_polylines): bounds[0..shards], rank r owns [bounds[r], bounds[r+1]),
 * each range's segment-pair cost within one item of total / shards. */
LC_API int lc_shard_bounds(lc_ctx *ctx, int shards, int64_t *bounds);
/* The same exchange with a caller-owned collective (e.g. torch.distributed):
 * lc_run_pipeline_shard_async enqueues the fused run of shard `shard` of
 * `shards` (>= 1, cost-balanced ranges) on the context stream and returns at
 * once with the library's item-partials buffer (*part_cap int64 words;
 * *part_cap = 0: the model needs the staged path).  The caller enqueues an
 * in-place int64 MAX all-reduce of that buffer on the context stream
 * (lc_get_stream); lc_shard_finish then enqueues the fixed-order reduction and
 * the export and syncs once; *fused = 1: results ready (lc_result_views), 0:
 * run the staged path; LC_ERR_VALIDATION as lc_run_pipeline. */
LC_API int lc_run_pipeline_shard_async(lc_ctx *ctx, const uint64_t *excluded_keys, int64_t n_excl, double xi,
                                       double epsilon, int max_passes, int64_t max_subsegments, int mode, int shard,
                                       int shards, double **partials_dev, int64_t *part_cap);
LC_API int lc_shard_finish(lc_ctx *ctx, int *fused);
LC_API int lc_get_stream(lc_ctx *ctx, void **stream);
/* Device early exit for verify(..., early_exit=True) (certify.py:195-216).
 * lc_set_early_exit hands the library the reference certificate — keys
 * (i << 32 | j) sorted unique, values lk (nonzero) — and, enable != 0, makes the
 * next single-GPU fused runs evaluate the candidate pairs against it in the
 * reference's order (certificate pairs, then the other candidates, each in key
 * order): the first pair whose value differs (or is NaN / ambiguous) ends the
 * evaluation and every pair after it in that order is cancelled.  Pairs before it
 * are all evaluated, so the caller replays the reference's report from the
 * results.  lc_early_exit_stats: that pair's place (-1: none) and the number of
 * pairs evaluated (-1: the last run was not a device early-exit run). */
LC_API int lc_set_early_exit(lc_ctx *ctx, const uint64_t *ref_keys, const int64_t *ref_lk, int64_t n_ref,
                             int enable);
LC_API int lc_early_exit_stats(lc_ctx *ctx, int64_t *first_fail_place, int64_t *n_evaluated);
/* Path of the last lc_run_pipeline: 0 staged, 1 fused, 2 fused replayed from
 * the captured CUDA graph (same shape as the previous run, no reallocation). */
LC_API int lc_last_run_fused(lc_ctx *ctx);
/* Device times (ms) of the last pipeline: [derive + PLS, discretize, Gauss kernel, reduce,
 * first stage start -> reduce end] (ms must hold 5 floats); -1 for the stages a
 * fused run without stage detail did not time (it records only the Gauss stage). */
LC_API int lc_stage_times(lc_ctx *ctx, float *ms);
/* Fused runs record every stage event (on) or only the Gauss stage's (off, the
 * default: each event-record node adds ~0.8 us to the graph launch).  The env
 * LINKCERT_STAGE_TIMES=1 forces detail on. */
LC_API int lc_set_stage_detail(lc_ctx *ctx, int on);

/* ---- Canonical model serialization (host, multithreaded) ----
 * Bytes of json.dumps(model_to_dict(model), sort_keys=True,
 * separators=(",", ":")) (model_io.py:122-172) for a packed model; the
 * caller hashes them (SHA-256) to obtain model_digest.  closed: one byte per
 * loop (NULL = all closed).  Returns the length, -1 for a non-finite
 * coordinate, -2 if cap is too small (size with lc_model_json_bound). */
LC_API int64_t lc_model_json_bound(const int64_t *loop_off, int64_t L);
LC_API int64_t lc_model_json(const double *coeffs, const double *t, const int64_t *loop_off,
                             const uint8_t *closed, int64_t L, int nthreads, char *out, int64_t cap);
/* Drop-in for model_io.model_digest (model_io.py:169-172): SHA-256 hex (65
 * bytes incl. NUL) of the canonical JSON, formatted on nthreads workers and
 * hashed in stream order (SHA-NI when available).  -1: non-finite coordinate. */
LC_API int lc_model_digest(const double *coeffs, const double *t, const int64_t *loop_off,
                           const uint8_t *closed, int64_t L, int nthreads, char *hex_out);
/* model_digest of a model whose loops are all closed LoopGeometry.from_polyline
 * loops, from one vertex array per loop (as lc_model_upload_polyline_ptrs):
 * the canonical "points" are the vertices (model_io.py:126-133), so no packed
 * coefficient array is needed.  -1: non-finite coordinate, -2: null pointer. */
LC_API int lc_model_digest_polylines(const double *const *loop_verts, const int64_t *loop_off, int64_t L,
                                     int nthreads, char *hex_out);
/* lc_model_digest_polylines over input that is still being written: the caller
 * fills loop_verts[l] and loop_off[l + 1] in loop order and publishes progress
 * by storing the count of filled loops into *ready (release order; x86 stores),
 * so hashing starts before the caller has walked every loop.  *ready < 0 aborts
 * (-3: e.g. a loop turned out not to be a closed polyline); the caller must
 * eventually store L or a negative value.  -1 non-finite, -2 null pointer. */
LC_API int lc_model_digest_polylines_stream(const double *const *loop_verts, const int64_t *loop_off, int64_t L,
                                            const int64_t *ready, int nthreads, char *hex_out);
/* SHA-256 hex of a buffer (test hook; force_portable skips SHA-NI); returns 1 if SHA-NI exists. */
LC_API int lc_sha256_hex(const void *data, int64_t n, int force_portable, char *hex_out);
/* Page-locked host memory for model arrays (the per-call H2D copies of verify
 * then run at DMA speed).  NULL when no CUDA device is usable. */
LC_API void *lc_host_alloc(int64_t bytes);
LC_API void lc_host_free(void *p);
/* CPython float.__repr__ of x into out (>= 32 bytes); returns the length. */
LC_API int lc_float_repr(double x, char *out);
/* Test hook: repr of n doubles, each followed by '\n', into out (cap >= 26 n);
 * use_tochars selects the std::to_chars cross-check formatter.  Returns bytes. */
LC_API int64_t lc_float_repr_many(const double *x, int64_t n, int use_tochars, char *out, int64_t cap);

/* Kernel launches issued by the library so far, all contexts (own kernels
 * exactly; each CUB device-algorithm call counted once). */
LC_API long long lc_launch_count(void);

/* ---- Barnes-Hut (reference: linkcert/barneshut.py, tree: linkcert/bvh.py) ----
 * A forest is the moment trees (leaf size 1, the reference's median split and
 * node numbering) of L closed polylines, device-resident, owned by ctx.
 * lc_bh_forest_build replaces MomentTree.__init__ (barneshut.py:298-312):
 *   verts (M, 3) row-major, loop t = rows [loop_off[t], loop_off[t+1]), closed
 *   implicitly (segment i ends at the next vertex of its loop, np.roll).
 * lc_bh_forest_sizes: trees, segments, nodes, levels (max depth + 1).
 * lc_bh_forest_nodes copies node data to the host in the reference's per-tree
 *   numbering (bvh.BvhTree fields + barneshut moment arrays; any pointer may be
 *   NULL): node_off (L+1), left/right (-1 = leaf), start/end, prim_order (M),
 *   node_lo/node_hi/center (N,3), radius (N), cm (N,3), cd (N,3,3), cq (N,3,3,3),
 *   ncm/ncd/ncq (N).  Node ids / positions are relative to each tree.
 * lc_bh_far_field replaces barneshut._far_field via far_field_eval
 *   (barneshut.py:330-345); node ids are forest-global (node_off[t] + local).
 * lc_bh_eval replaces barneshut._dual_eval (barneshut.py:175-240) for P tree
 *   pairs at once: pairs (P, 2) = (tree in a, tree in b), beta (P) opening
 *   parameters; lam/e_est (P) out; visits = node pairs visited (may be NULL). */
typedef struct lc_bh_forest lc_bh_forest;
LC_API int lc_bh_forest_build(lc_ctx *ctx, const double *verts, const int64_t *loop_off, int64_t L,
                              lc_bh_forest **out);
LC_API int lc_bh_forest_free(lc_ctx *ctx, lc_bh_forest *f);
LC_API int lc_bh_forest_sizes(const lc_bh_forest *f, int64_t *L, int64_t *M, int64_t *N, int *levels);
LC_API int lc_bh_forest_nodes(lc_ctx *ctx, const lc_bh_forest *f, int64_t *node_off, int64_t *left, int64_t *right,
                              int64_t *start, int64_t *end, int64_t *prim_order, double *node_lo, double *node_hi,
                              double *center, double *radius, double *cm, double *cd, double *cq, double *ncm,
                              double *ncd, double *ncq);
LC_API int lc_bh_far_field(lc_ctx *ctx, const lc_bh_forest *a, int64_t node_a, const lc_bh_forest *b, int64_t node_b,
                           int quadrupole, double *out);
LC_API int lc_bh_eval(lc_ctx *ctx, const lc_bh_forest *a, const lc_bh_forest *b, const int32_t *pairs, int64_t P,
                      const double *beta, int quadrupole, double k_const, double *lam, double *e_est, int64_t *visits);

/* FP64 DFMA-chain throughput probe (roofline denominator), FLOP/s. */
LC_API int lc_probe_fp64_peak(lc_ctx *ctx, double *flops, float *ms);
/* FP64 tensor-core (mma.sync m8n8k4 f64) throughput probe, FLOP/s: the FP64
 * datapath's other peak (DFMA and DMMA share it; the roofline takes the max). */
LC_API int lc_probe_fp64_dmma_peak(lc_ctx *ctx, double *flops, float *ms);

#ifdef __cplusplus
}
#endif

#endif /* LINKCERT_B200_H */
