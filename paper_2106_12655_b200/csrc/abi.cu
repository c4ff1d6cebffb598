// extern "C" boundary of liblinkcert_b200.so — see include/linkcert_b200.h.
//
// Every entry point returns 0 on success or an lc::Code; no C++ exception
// crosses the ABI.  The library owns device buffers (grow-only, cached in the
// context); callers own every host buffer they pass.  Calls on one context
// are serialized by its mutex.
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "bh.cuh"
#include "comm.cuh"
#include "gauss.cuh"
#include "pipeline.cuh"

namespace lc {
double probe_dfma_flops(cudaStream_t s, float *elapsed_ms);
double probe_dmma_flops(cudaStream_t s, float *elapsed_ms);
}

using namespace lc;

static thread_local std::string g_last_error;

struct lc_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::mutex mu;
    Pipeline pipe;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    float last_gauss_ms = 0.f;
    int last_fused = 0;   // last lc_run_pipeline: 0 staged, 1 fused, 2 fused replayed as a CUDA graph
    DevBuf tb_coeffs, tb_t, tb_box, tb_loop, tb_off, tb_flag;   // lc_tight_boxes scratch
    BhScratch bh;                                                // Barnes-Hut traversal scratch
    Comm comm;                                                   // multi-GPU communicator (lc_comm_init)
};

struct lc_bh_forest {
    lc::BhForest f;
    lc_ctx *owner = nullptr;
};

template <class F>
static int guarded(lc_ctx *ctx, F &&f) {
    try {
        if (!ctx) throw Error(LC_ERR_ARG, "null context");
        std::lock_guard<std::mutex> lock(ctx->mu);
        LC_CUDA(cudaSetDevice(ctx->device));
        f();
        return LC_OK;
    } catch (const Error &e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception &e) {
        g_last_error = e.what();
        return LC_ERR_STATE;
    } catch (...) {
        g_last_error = "unknown error";
        return LC_ERR_STATE;
    }
}

extern "C" {

int lc_abi_version(void) { return LC_ABI_VERSION; }

const char *lc_last_error(void) { return g_last_error.c_str(); }

int lc_device_count(int *count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        g_last_error = cudaGetErrorString(e);
        *count = 0;
        return LC_ERR_CUDA;
    }
    *count = n;
    return LC_OK;
}

lc_ctx *lc_create(int device) {
    lc_ctx *ctx = new lc_ctx();
    ctx->device = device;
    try {
        LC_CUDA(cudaSetDevice(device));
        // stream-ordered frees stay in the device pool (no OS round trip when a
        // moment forest or a scratch buffer is rebuilt at the same size)
        cudaMemPool_t pool;
        LC_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = ~0ull;
        LC_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        LC_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
        LC_CUDA(cudaEventCreate(&ctx->ev0));
        LC_CUDA(cudaEventCreate(&ctx->ev1));
        ctx->pipe.init(ctx->stream);
    } catch (const std::exception &e) {
        g_last_error = e.what();
        delete ctx;
        return nullptr;
    }
    return ctx;
}

void lc_destroy(lc_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    ctx->pipe.release();
    BhScratch &b = ctx->bh;   // the context's other device buffers (Barnes-Hut, tight-box scratch)
    for (DevBuf *x : {&b.fr[0], &b.fr[1], &b.val, &b.cnt, &b.off, &b.key, &b.uniq, &b.agg, &b.nruns, &b.tmp, &b.tot,
                      &b.beta, &b.pairs, &b.leaves, &ctx->tb_coeffs, &ctx->tb_t, &ctx->tb_box, &ctx->tb_loop,
                      &ctx->tb_off, &ctx->tb_flag})
        x->release(ctx->stream);
    b.host.release();
    try {
        comm_destroy(ctx->comm);
    } catch (...) {
    }
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->own_stream && ctx->stream) {
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
    }
    delete ctx;
}

int lc_set_stream(lc_ctx *ctx, void *stream) {
    return guarded(ctx, [&] {
        LC_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        ctx->own_stream = stream == nullptr;
        if (stream) ctx->stream = (cudaStream_t)stream;
        else LC_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->pipe.set_stream(ctx->stream);
    });
}

int lc_synchronize(lc_ctx *ctx) {
    return guarded(ctx, [&] { LC_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

// ---------------------------------------------------------------- Gauss sum

int lc_evaluate_pairs(lc_ctx *ctx, const double *verts, const int64_t *vert_off, int64_t L,
                      const int32_t *pairs, int64_t P, int mode, double *raw, int64_t *lk,
                      uint8_t *flags) {
    return guarded(ctx, [&] {
        if (L < 0 || P < 0 || (L > 0 && (!verts || !vert_off)) || (P > 0 && !pairs))
            throw Error(LC_ERR_ARG, "lc_evaluate_pairs: bad arguments");
        ctx->pipe.upload_polylines(verts, vert_off, L);
        ctx->pipe.upload_pairs(pairs, P);
        ctx->pipe.build_gauss_items(mode);
        ctx->pipe.run_gauss(mode, 0, ctx->pipe.n_items, nullptr, ctx->ev0, ctx->ev1);
        ctx->pipe.reduce_pairs(nullptr);
        ctx->pipe.download_results(raw, lk, flags);
        LC_CUDA(cudaEventElapsedTime(&ctx->last_gauss_ms, ctx->ev0, ctx->ev1));
    });
}

int lc_link_direct(lc_ctx *ctx, const double *loop1, int64_t n1, const double *loop2, int64_t n2,
                   int mode, double *raw) {
    return guarded(ctx, [&] {
        if (!loop1 || !loop2 || n1 < 1 || n2 < 1) throw Error(LC_ERR_ARG, "lc_link_direct: bad arguments");
        *raw = ctx->pipe.link_direct(loop1, n1, loop2, n2, mode, ctx->ev0, ctx->ev1);
        LC_CUDA(cudaEventElapsedTime(&ctx->last_gauss_ms, ctx->ev0, ctx->ev1));
    });
}

int lc_segment_pair_lambda(lc_ctx *ctx, const double *quads, int64_t n, double *out) {
    return guarded(ctx, [&] {
        if (n < 0 || (n > 0 && (!quads || !out))) throw Error(LC_ERR_ARG, "lc_segment_pair_lambda: bad arguments");
        ctx->pipe.segment_pair_lambda(quads, n, out);
    });
}

int lc_last_gauss_ms(lc_ctx *ctx, float *ms) {
    return guarded(ctx, [&] { *ms = ctx->last_gauss_ms; });
}

// Device-resident staging (bench / multi-GPU): upload once, run many times.
int lc_stage_polylines(lc_ctx *ctx, const double *verts, const int64_t *vert_off, int64_t L,
                       const int32_t *pairs, int64_t P, int mode, int64_t *n_items) {
    return guarded(ctx, [&] {
        ctx->pipe.upload_polylines(verts, vert_off, L);
        ctx->pipe.upload_pairs(pairs, P);
        ctx->pipe.build_gauss_items(mode);
        *n_items = ctx->pipe.n_items;
    });
}

int lc_gauss_run(lc_ctx *ctx, int mode, int64_t item_begin, int64_t item_end, double *partials_dev) {
    return guarded(ctx, [&] {
        if (item_begin < 0 || item_end > ctx->pipe.n_items || item_begin > item_end)
            throw Error(LC_ERR_ARG, "lc_gauss_run: item range out of bounds");
        ctx->pipe.run_gauss(mode, item_begin, item_end, partials_dev, ctx->ev0, ctx->ev1);
    });
}

int lc_gauss_run_pairs(lc_ctx *ctx, int mode) {
    return guarded(ctx, [&] {
        Pipeline &p = ctx->pipe;
        if (!p.items_ready || p.items_seq) throw Error(LC_ERR_STATE, "no tile work items built (lc_prepare_gauss)");
        p.d_tot.reserve(4 * sizeof(int64_t), ctx->stream);
        p.d_counter.reserve(2 * sizeof(unsigned long long), ctx->stream);
        p.d_partials.reserve(sizeof(double) * (size_t)(p.P > 0 ? p.P : 1), ctx->stream);
        LC_CUDA(cudaMemcpyAsync(p.d_tot.ptr, &p.P, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        LC_CUDA(cudaMemsetAsync(p.d_counter.ptr, 0, sizeof(unsigned long long), ctx->stream));
        LC_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
        launch_gauss_pairs(mode, p.gX, p.gY, p.gZ, p.d_pg.as<PairGeom>(), p.d_tot.as<int64_t>(), p.P,
                           p.d_counter.as<unsigned long long>(), nullptr, nullptr, 0, p.d_partials.as<double>(),
                           nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, ctx->stream);
        LC_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
        LC_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int lc_gauss_reduce(lc_ctx *ctx, const double *partials_dev, double *raw, int64_t *lk, uint8_t *flags) {
    return guarded(ctx, [&] {
        ctx->pipe.reduce_pairs(partials_dev);
        ctx->pipe.download_results(raw, lk, flags);
    });
}

int lc_gauss_event_ms(lc_ctx *ctx, float *ms) {
    return guarded(ctx, [&] {
        LC_CUDA(cudaEventSynchronize(ctx->ev1));
        LC_CUDA(cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1));
    });
}

// ------------------------------------------------------- model pipeline

int lc_tight_boxes(lc_ctx *ctx, const double *coeffs, const double *t, int64_t m, double *lo, double *hi) {
    return guarded(ctx, [&] {
        if (m < 0 || (m > 0 && (!coeffs || !t || !lo || !hi))) throw Error(LC_ERR_ARG, "lc_tight_boxes: bad arguments");
        if (m == 0) return;
        cudaStream_t s = ctx->stream;
        ctx->tb_coeffs.reserve(sizeof(double) * 12 * m, s);
        ctx->tb_t.reserve(sizeof(double) * 2 * m, s);
        ctx->tb_box.reserve(sizeof(double) * 6 * m, s);
        ctx->tb_loop.reserve(sizeof(int32_t) * m, s);
        ctx->tb_off.reserve(sizeof(int64_t) * 2, s);
        ctx->tb_flag.reserve(sizeof(int), s);
        const int64_t off[2] = {0, m};
        LC_CUDA(cudaMemcpyAsync(ctx->tb_coeffs.ptr, coeffs, sizeof(double) * 12 * m, cudaMemcpyHostToDevice, s));
        LC_CUDA(cudaMemcpyAsync(ctx->tb_t.ptr, t, sizeof(double) * 2 * m, cudaMemcpyHostToDevice, s));
        LC_CUDA(cudaMemcpyAsync(ctx->tb_off.ptr, off, sizeof off, cudaMemcpyHostToDevice, s));
        launch_seg_boxes(ctx->tb_coeffs.as<double>(), ctx->tb_t.as<double>(), nullptr, ctx->tb_off.as<int64_t>(), 1, m,
                         ctx->tb_box.as<double>(), ctx->tb_loop.as<int32_t>(), nullptr, nullptr, s);
        std::vector<double> b((size_t)6 * m);
        LC_CUDA(cudaMemcpyAsync(b.data(), ctx->tb_box.ptr, sizeof(double) * 6 * m, cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaStreamSynchronize(s));
        for (int64_t k = 0; k < m; ++k)
            for (int d = 0; d < 3; ++d) {
                lo[3 * k + d] = b[d * m + k];
                hi[3 * k + d] = b[(3 + d) * m + k];
            }
    });
}

int lc_model_upload(lc_ctx *ctx, const double *coeffs, const double *t, const int64_t *loop_off, int64_t L) {
    return guarded(ctx, [&] {
        if (L < 0 || !loop_off || (L > 0 && loop_off[L] > 0 && (!coeffs || !t)))
            throw Error(LC_ERR_ARG, "lc_model_upload: bad arguments");
        ctx->pipe.upload_model(coeffs, t, loop_off, L);
    });
}

int lc_model_upload_polylines(lc_ctx *ctx, const double *verts, const int64_t *loop_off, int64_t L) {
    return guarded(ctx, [&] {
        if (L < 0 || !loop_off || (L > 0 && loop_off[L] > 0 && !verts))
            throw Error(LC_ERR_ARG, "lc_model_upload_polylines: bad arguments");
        ctx->pipe.upload_model_polylines(verts, loop_off, L);
    });
}

int lc_model_upload_polyline_ptrs(lc_ctx *ctx, const double *const *loop_verts, const int64_t *loop_off,
                                  int64_t L) {
    return guarded(ctx, [&] {
        if (L < 0 || !loop_off || (L > 0 && !loop_verts))
            throw Error(LC_ERR_ARG, "lc_model_upload_polyline_ptrs: bad arguments");
        ctx->pipe.upload_model_polyline_ptrs(loop_verts, loop_off, L);
    });
}

int lc_loop_boxes(lc_ctx *ctx, double *lo, double *hi) {
    return guarded(ctx, [&] { ctx->pipe.download_loop_boxes(lo, hi); });
}

static int pls_abi(lc_ctx *ctx, const uint64_t *excluded_keys, int64_t n_excl, int64_t *n_pairs, bool in_run) {
    return guarded(ctx, [&] {
        if (n_excl < 0 || (n_excl > 0 && !excluded_keys)) throw Error(LC_ERR_ARG, "bad excluded keys");
        for (int64_t k = 1; k < n_excl; ++k)
            if (excluded_keys[k] <= excluded_keys[k - 1]) throw Error(LC_ERR_ARG, "excluded keys must be sorted unique");
        *n_pairs = ctx->pipe.potential_link_search(excluded_keys, n_excl, in_run);
    });
}

int lc_potential_link_search(lc_ctx *ctx, const uint64_t *excluded_keys, int64_t n_excl, int64_t *n_pairs) {
    return pls_abi(ctx, excluded_keys, n_excl, n_pairs, false);
}

int lc_get_pairs(lc_ctx *ctx, int32_t *pairs) {
    return guarded(ctx, [&] { ctx->pipe.download_pairs(pairs); });
}

int lc_set_pairs(lc_ctx *ctx, const int32_t *pairs, int64_t P) {
    return guarded(ctx, [&] {
        if (P < 0 || (P > 0 && !pairs)) throw Error(LC_ERR_ARG, "bad pair list");
        ctx->pipe.upload_pairs(pairs, P);
    });
}

static int run_discretize_abi(lc_ctx *ctx, double xi, double epsilon, int max_passes, int64_t max_subsegments,
                              int64_t *n_vertices, int *passes, bool defer_validation = false) {
    int rc = LC_OK;
    int g = guarded(ctx, [&] {
        DiscParams prm;
        prm.xi = xi;
        prm.epsilon = epsilon;
        prm.max_passes = max_passes;
        prm.max_subsegments = max_subsegments;
        prm.defer_validation = defer_validation;
        const bool ok = ctx->pipe.discretize(prm);
        if (passes) *passes = ctx->pipe.dout.passes;
        if (!ok) {
            rc = ctx->pipe.derr.kind == DISC_INVALID_POLYLINE ? LC_ERR_VALIDATION : LC_ERR_DISCRETIZE;
            return;
        }
        if (n_vertices) *n_vertices = ctx->pipe.V;
    });
    if (g != LC_OK) return g;
    if (rc != LC_OK) g_last_error = "discretization failed (see lc_discretize_error)";
    return rc;
}

int lc_discretize(lc_ctx *ctx, double xi, double epsilon, int max_passes, int64_t max_subsegments,
                  int64_t *n_vertices, int *passes) {
    return run_discretize_abi(ctx, xi, epsilon, max_passes, max_subsegments, n_vertices, passes);
}

int lc_discretize_error(lc_ctx *ctx, int *kind, int *detail, int64_t *loops, int64_t cap, int64_t *n_loops) {
    return guarded(ctx, [&] {
        const DiscError &e = ctx->pipe.derr;
        *kind = e.kind;
        *detail = e.detail;
        *n_loops = (int64_t)e.loops.size();
        for (int64_t k = 0; k < cap && k < (int64_t)e.loops.size(); ++k) loops[k] = e.loops[k];
    });
}

int lc_get_polylines(lc_ctx *ctx, double *verts, int64_t *vert_off) {
    return guarded(ctx, [&] { ctx->pipe.download_polylines(verts, vert_off); });
}

int lc_prepare_gauss(lc_ctx *ctx, int mode, int64_t *n_items) {
    return guarded(ctx, [&] {
        ctx->pipe.build_gauss_items(mode);
        *n_items = ctx->pipe.n_items;
    });
}

int lc_evaluate_staged(lc_ctx *ctx, int mode, double *raw, int64_t *lk, uint8_t *flags) {
    return guarded(ctx, [&] {
        ctx->pipe.build_gauss_items(mode);
        ctx->pipe.run_gauss(mode, 0, ctx->pipe.n_items, nullptr, nullptr, nullptr);
        ctx->pipe.reduce_pairs(nullptr);
        ctx->pipe.download_results(raw, lk, flags);
        ctx->last_gauss_ms = ctx->pipe.stage_ms(EV_GAUSS0, EV_GAUSS1);
    });
}

int lc_run_pipeline(lc_ctx *ctx, const uint64_t *excluded_keys, int64_t n_excl, double xi, double epsilon,
                    int max_passes, int64_t max_subsegments, int mode, int64_t *n_pairs) {
    // Fused single-sync run first (LINKCERT_FUSED=0 disables it); it reports
    // FAST_FALLBACK for the models it does not cover (refinement passes, the
    // sweep path, PLS row overflow) and the staged pipeline below runs them.
    const char *fz = getenv("LINKCERT_FUSED");
    ctx->last_fused = 0;
    ctx->pipe.derived_in_run = false;
    const int gd = guarded(ctx, [&] {
        if (n_excl < 0 || (n_excl > 0 && !excluded_keys)) throw Error(LC_ERR_ARG, "bad excluded keys");
        for (int64_t k = 1; k < n_excl; ++k)
            if (excluded_keys[k] <= excluded_keys[k - 1]) throw Error(LC_ERR_ARG, "excluded keys must be sorted unique");
    });
    if (gd != LC_OK) return gd;
    if (!(fz && fz[0] == '0')) {
        int fr = FAST_FALLBACK;
        const int g = guarded(ctx, [&] {
            DiscParams prm;
            prm.xi = xi;
            prm.epsilon = epsilon;
            prm.max_passes = max_passes;
            prm.max_subsegments = max_subsegments;
            fr = ctx->pipe.run_fast(excluded_keys, n_excl, prm, mode);
            if (n_pairs) *n_pairs = ctx->pipe.P;
        });
        if (g != LC_OK) return g;
        ctx->last_fused = fr == FAST_FALLBACK ? 0 : (ctx->pipe.last_fast_graph ? 2 : 1);
        if (fr == FAST_OK) return LC_OK;
        if (fr == FAST_INVALID) {
            g_last_error = "discretization failed (see lc_discretize_error)";
            return LC_ERR_VALIDATION;
        }
    }
    // staged path: derive the boxes unless the fused attempt just did
    if (!ctx->pipe.derived_in_run) {
        const int g2 = guarded(ctx, [&] { ctx->pipe.derive(); });
        if (g2 != LC_OK) return g2;
    }
    int rc = pls_abi(ctx, excluded_keys, n_excl, n_pairs, true);
    if (rc != LC_OK) return rc;
    int64_t nv = 0;
    int passes = 0;
    rc = run_discretize_abi(ctx, xi, epsilon, max_passes, max_subsegments, &nv, &passes, true);
    if (rc != LC_OK) return rc;
    bool valid = true;
    rc = guarded(ctx, [&] { valid = ctx->pipe.build_gauss_items_checked(mode); });
    if (rc != LC_OK) return rc;
    if (!valid) {   // deferred PolylineLoop validation failed (read back with n_items)
        g_last_error = "discretization failed (see lc_discretize_error)";
        return LC_ERR_VALIDATION;
    }
    return guarded(ctx, [&] {
        ctx->pipe.run_gauss(mode, 0, ctx->pipe.n_items, nullptr, nullptr, nullptr);
        ctx->pipe.reduce_pairs(nullptr);
        ctx->pipe.download_results_pinned();
    });
}

int lc_run_pipeline_shard_async(lc_ctx *ctx, const uint64_t *excluded_keys, int64_t n_excl, double xi,
                                double epsilon, int max_passes, int64_t max_subsegments, int mode, int shard,
                                int shards, double **partials_dev, int64_t *part_cap) {
    if (part_cap) *part_cap = 0;
    ctx->last_fused = 0;
    ctx->pipe.derived_in_run = false;
    return guarded(ctx, [&] {
        if (!partials_dev || !part_cap || shards < 1) throw Error(LC_ERR_ARG, "lc_run_pipeline_shard_async: bad arguments");
        if (n_excl < 0 || (n_excl > 0 && !excluded_keys)) throw Error(LC_ERR_ARG, "bad excluded keys");
        for (int64_t k = 1; k < n_excl; ++k)
            if (excluded_keys[k] <= excluded_keys[k - 1]) throw Error(LC_ERR_ARG, "excluded keys must be sorted unique");
        DiscParams prm;
        prm.xi = xi;
        prm.epsilon = epsilon;
        prm.max_passes = max_passes;
        prm.max_subsegments = max_subsegments;
        const int fr = ctx->pipe.run_fast(excluded_keys, n_excl, prm, mode, shard, shards, true);
        if (fr == FAST_PENDING) {
            *partials_dev = ctx->pipe.d_partials.as<double>();
            *part_cap = ctx->pipe.part_cap;
        }
    });
}

// ---------------------------------------------------- multi-GPU (NCCL)

int lc_nccl_version(void) { return nccl_version(); }

int lc_comm_unique_id(char *id_out) {
    try {
        if (!id_out) throw Error(LC_ERR_ARG, "null id buffer");
        ncclUniqueId id;
        comm_unique_id(&id);
        std::memcpy(id_out, id.internal, sizeof id.internal);
        return LC_OK;
    } catch (const Error &e) {
        g_last_error = e.what();
        return e.code;
    }
}

int lc_comm_init(lc_ctx *ctx, const char *id, int world, int rank) {
    return guarded(ctx, [&] {
        if (!id) throw Error(LC_ERR_ARG, "null id");
        ncclUniqueId u;
        std::memcpy(u.internal, id, sizeof u.internal);
        comm_init(ctx->comm, u, world, rank);
        ctx->pipe.gather_share = world;
    });
}

int lc_comm_destroy(lc_ctx *ctx) {
    return guarded(ctx, [&] {
        comm_destroy(ctx->comm);
        ctx->pipe.gather_share = 1;
    });
}

int lc_shard_bounds(lc_ctx *ctx, int shards, int64_t *bounds) {
    return guarded(ctx, [&] {
        if (!bounds) throw Error(LC_ERR_ARG, "null bounds");
        ctx->pipe.shard_bounds(shards, bounds);
    });
}

int lc_run_pipeline_sharded(lc_ctx *ctx, const uint64_t *excluded_keys, int64_t n_excl, double xi, double epsilon,
                            int max_passes, int64_t max_subsegments, int mode, int64_t *n_pairs) {
    ctx->last_fused = 0;
    ctx->pipe.derived_in_run = false;
    int world = 1, rank = 0;
    const int gd = guarded(ctx, [&] {
        if (!ctx->comm.ready()) throw Error(LC_ERR_STATE, "lc_run_pipeline_sharded needs lc_comm_init");
        if (n_excl < 0 || (n_excl > 0 && !excluded_keys)) throw Error(LC_ERR_ARG, "bad excluded keys");
        for (int64_t k = 1; k < n_excl; ++k)
            if (excluded_keys[k] <= excluded_keys[k - 1]) throw Error(LC_ERR_ARG, "excluded keys must be sorted unique");
        world = ctx->comm.world;
        rank = ctx->comm.rank;
    });
    if (gd != LC_OK) return gd;
    // fused single-sync run, this rank's cost-balanced item range; the partials
    // exchange is enqueued right behind it on the same stream (no host round trip)
    const char *fz = getenv("LINKCERT_FUSED");
    if (!(fz && fz[0] == '0')) {
        int fr = FAST_FALLBACK;
        const int g = guarded(ctx, [&] {
            DiscParams prm;
            prm.xi = xi;
            prm.epsilon = epsilon;
            prm.max_passes = max_passes;
            prm.max_subsegments = max_subsegments;
            fr = ctx->pipe.run_fast(excluded_keys, n_excl, prm, mode, rank, world, true, true);
            if (fr == FAST_PENDING) {
                comm_allreduce_max_i64(ctx->comm, ctx->pipe.d_partials.ptr, (size_t)ctx->pipe.part_cap,
                                       ctx->stream);
                fr = ctx->pipe.shard_finish();
            }
            if (n_pairs) *n_pairs = ctx->pipe.P;
        });
        if (g != LC_OK) return g;
        ctx->last_fused = fr == FAST_FALLBACK ? 0 : (ctx->pipe.last_fast_graph ? 2 : 1);
        if (fr == FAST_OK) return LC_OK;
        if (fr == FAST_INVALID) {
            g_last_error = "discretization failed (see lc_discretize_error)";
            return LC_ERR_VALIDATION;
        }
    }
    // staged path (refinement, the sweep PLS, anglesum): every rank runs the same
    // front end; the Gauss sum covers this rank's cost-balanced item range
    if (!ctx->pipe.derived_in_run) {
        const int g2 = guarded(ctx, [&] { ctx->pipe.derive(); });
        if (g2 != LC_OK) return g2;
    }
    int rc = pls_abi(ctx, excluded_keys, n_excl, n_pairs, true);
    if (rc != LC_OK) return rc;
    int64_t nv = 0;
    int passes = 0;
    rc = run_discretize_abi(ctx, xi, epsilon, max_passes, max_subsegments, &nv, &passes, true);
    if (rc != LC_OK) return rc;
    bool valid = true;
    rc = guarded(ctx, [&] { valid = ctx->pipe.build_gauss_items_checked(mode); });
    if (rc != LC_OK) return rc;
    if (!valid) {
        g_last_error = "discretization failed (see lc_discretize_error)";
        return LC_ERR_VALIDATION;
    }
    return guarded(ctx, [&] {
        Pipeline &p = ctx->pipe;
        std::vector<int64_t> b((size_t)world + 1);
        p.shard_bounds(world, b.data());
        p.prefill_partials_neg_zero(p.n_items);
        p.run_gauss(mode, b[rank], b[rank + 1], nullptr, nullptr, nullptr);
        comm_allreduce_max_i64(ctx->comm, p.d_partials.ptr, (size_t)p.n_items, ctx->stream);
        p.reduce_pairs(nullptr);
        p.download_results_pinned();
    });
}

int lc_set_early_exit(lc_ctx *ctx, const uint64_t *ref_keys, const int64_t *ref_lk, int64_t n_ref, int enable) {
    return guarded(ctx, [&] { ctx->pipe.set_early_exit(ref_keys, ref_lk, n_ref, enable != 0); });
}

int lc_early_exit_stats(lc_ctx *ctx, int64_t *first_fail_place, int64_t *n_evaluated) {
    return guarded(ctx, [&] {
        if (first_fail_place) *first_fail_place = ctx->pipe.ee_first_fail;
        if (n_evaluated) *n_evaluated = ctx->pipe.ee_n_eval;
    });
}

int lc_shard_finish(lc_ctx *ctx, int *fused) {
    if (fused) *fused = 0;
    int fr = FAST_FALLBACK;
    const int g = guarded(ctx, [&] { fr = ctx->pipe.shard_finish(); });
    if (g != LC_OK) return g;
    ctx->last_fused = fr == FAST_FALLBACK ? 0 : (ctx->pipe.last_fast_graph ? 2 : 1);
    if (fused) *fused = fr == FAST_OK ? 1 : 0;
    if (fr == FAST_INVALID) {
        g_last_error = "discretization failed (see lc_discretize_error)";
        return LC_ERR_VALIDATION;
    }
    return LC_OK;
}

int lc_get_stream(lc_ctx *ctx, void **stream) {
    return guarded(ctx, [&] {
        if (!stream) throw Error(LC_ERR_ARG, "null stream pointer");
        *stream = (void *)ctx->stream;
    });
}


int lc_result_views(lc_ctx *ctx, void **pairs, void **raw, void **lk, void **flags, int64_t *n_pairs) {
    return guarded(ctx, [&] {
        Pipeline &p = ctx->pipe;
        if (p.h_res_P < 0) throw Error(LC_ERR_STATE, "no pipeline results");
        *pairs = p.res_pairs;
        *raw = p.res_raw;
        *lk = p.res_lk;
        *flags = p.res_flags;
        *n_pairs = p.h_res_P;
    });
}

int lc_get_results(lc_ctx *ctx, double *raw, int64_t *lk, uint8_t *flags) {
    return guarded(ctx, [&] { ctx->pipe.download_results(raw, lk, flags); });
}

int lc_stage_times(lc_ctx *ctx, float *ms) {
    return guarded(ctx, [&] {
        Pipeline &p = ctx->pipe;
        // a fused run without stage detail records only the Gauss-stage events
        const bool all = ctx->last_fused == 0 || p.last_detail;
        ms[0] = all ? p.stage_ms(EV_BEGIN, EV_PLS) : -1.f;
        ms[1] = all ? p.stage_ms(EV_PLS, EV_DISC) : -1.f;
        ms[2] = p.stage_ms(EV_GAUSS0, EV_GAUSS1);
        ms[3] = all ? p.stage_ms(EV_GAUSS1, EV_END) : -1.f;
        ms[4] = all ? p.stage_ms(EV_BEGIN, EV_END) : -1.f;
    });
}

int lc_set_stage_detail(lc_ctx *ctx, int on) {
    return guarded(ctx, [&] { ctx->pipe.stage_detail = on != 0; });
}

void *lc_host_alloc(int64_t bytes) {
    void *p = nullptr;
    if (bytes <= 0 || cudaHostAlloc(&p, (size_t)bytes, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();   // clear the sticky-free error of a failed allocation
        return nullptr;
    }
    return p;
}

void lc_host_free(void *p) {
    if (p) cudaFreeHost(p);
}

int lc_last_run_fused(lc_ctx *ctx) { return ctx ? ctx->last_fused : 0; }

long long lc_launch_count(void) { return launch_counter().load(); }

int lc_bh_forest_build(lc_ctx *ctx, const double *verts, const int64_t *loop_off, int64_t L, lc_bh_forest **out) {
    if (out) *out = nullptr;
    return guarded(ctx, [&] {
        if (!out || !loop_off || L < 1 || (!verts && loop_off[L] > 0)) throw Error(LC_ERR_ARG, "lc_bh_forest_build: bad arguments");
        for (int64_t t = 0; t < L; ++t)
            if (loop_off[t + 1] <= loop_off[t]) throw Error(LC_ERR_ARG, "lc_bh_forest_build: empty loop or bad offsets");
        auto *h = new lc_bh_forest;
        h->owner = ctx;
        try {
            bh_build(h->f, verts, loop_off, L, ctx->stream);
        } catch (...) {
            h->f.release(ctx->stream);
            delete h;
            throw;
        }
        *out = h;
    });
}

int lc_bh_forest_free(lc_ctx *ctx, lc_bh_forest *f) {
    if (!f) return LC_OK;
    return guarded(ctx, [&] {
        if (f->owner != ctx) throw Error(LC_ERR_ARG, "forest belongs to another context");
        f->f.release(ctx->stream);
        delete f;
    });
}

int lc_bh_forest_sizes(const lc_bh_forest *f, int64_t *L, int64_t *M, int64_t *N, int *levels) {
    if (!f) {
        g_last_error = "null forest";
        return LC_ERR_ARG;
    }
    if (L) *L = f->f.L;
    if (M) *M = f->f.M;
    if (N) *N = f->f.N;
    if (levels) *levels = f->f.levels;
    return LC_OK;
}

int lc_bh_forest_nodes(lc_ctx *ctx, const lc_bh_forest *f, int64_t *node_off, int64_t *left, int64_t *right,
                       int64_t *start, int64_t *end, int64_t *prim_order, double *node_lo, double *node_hi,
                       double *center, double *radius, double *cm, double *cd, double *cq, double *ncm, double *ncd,
                       double *ncq) {
    return guarded(ctx, [&] {
        if (!f || f->owner != ctx) throw Error(LC_ERR_ARG, "lc_bh_forest_nodes: bad forest");
        bh_download(f->f, node_off, left, right, start, end, prim_order, node_lo, node_hi, center, radius, cm, cd, cq,
                    ncm, ncd, ncq, ctx->stream);
    });
}

int lc_bh_far_field(lc_ctx *ctx, const lc_bh_forest *a, int64_t node_a, const lc_bh_forest *b, int64_t node_b,
                    int quadrupole, double *out) {
    return guarded(ctx, [&] {
        if (!a || !b || !out || a->owner != ctx || b->owner != ctx) throw Error(LC_ERR_ARG, "lc_bh_far_field: bad arguments");
        *out = bh_far_field(a->f, node_a, b->f, node_b, quadrupole != 0, ctx->bh, ctx->stream);
    });
}

int lc_bh_eval(lc_ctx *ctx, const lc_bh_forest *a, const lc_bh_forest *b, const int32_t *pairs, int64_t P,
               const double *beta, int quadrupole, double k_const, double *lam, double *e_est, int64_t *visits) {
    return guarded(ctx, [&] {
        if (!a || !b || a->owner != ctx || b->owner != ctx || P < 0 || (P > 0 && (!pairs || !beta)))
            throw Error(LC_ERR_ARG, "lc_bh_eval: bad arguments");
        bh_eval(a->f, b->f, pairs, P, beta, quadrupole != 0, k_const, lam, e_est, visits, ctx->bh, ctx->stream);
    });
}

int lc_probe_fp64_peak(lc_ctx *ctx, double *flops, float *ms) {
    return guarded(ctx, [&] { *flops = probe_dfma_flops(ctx->stream, ms); });
}

int lc_probe_fp64_dmma_peak(lc_ctx *ctx, double *flops, float *ms) {
    return guarded(ctx, [&] {
        const double f = probe_dmma_flops(ctx->stream, ms);
        if (flops) *flops = f;
    });
}

}  // extern "C"
