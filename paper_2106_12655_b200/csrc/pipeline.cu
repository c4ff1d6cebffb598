// Pipeline stage orchestration on one device/stream (host side of the C-ABI).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cstring>
#include <thread>
#include <vector>

#include "pipeline.cuh"

#include <cstddef>

namespace lc {

#ifndef LC_BRUTE_PDL
#define LC_BRUTE_PDL 1
#endif
constexpr bool kBrutePdl = LC_BRUTE_PDL;
#ifndef LC_CHAIN_PDL
#define LC_CHAIN_PDL 1   // programmatic dependent launch along the PLS chain of the fused run
#endif
constexpr bool kChainPdl = LC_CHAIN_PDL;
#ifndef LC_PASS1_GROUPS
#define LC_PASS1_GROUPS 1   // fused pass-1 check through 8-segment group boxes (brute_any_pair_sub)
#endif
constexpr bool kPass1Groups = LC_PASS1_GROUPS;

namespace {

// Closed polylines from vertices: exactly LoopGeometry.from_polyline's arrays
// (geometry.py:269-283): a0 = v_k, a1 = v_{k+1} - v_k, a2 = a3 = 0, t = [0, 1].
__global__ void polyline_coeffs_kernel(const double *__restrict__ v, const int64_t *__restrict__ loff, int64_t L,
                                       int64_t M, double *__restrict__ coeffs, double *__restrict__ t) {
    const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= M) return;
    int64_t lo = 0, hi = L;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (loff[mid] <= m) lo = mid; else hi = mid;
    }
    const int64_t nx = m + 1 < loff[lo + 1] ? m + 1 : loff[lo];
    double *c = coeffs + 12 * m;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        c[d] = v[3 * m + d];
        c[3 + d] = v[3 * nx + d] - v[3 * m + d];
        c[6 + d] = 0.0;
        c[9 + d] = 0.0;
    }
    t[2 * m] = 0.0;
    t[2 * m + 1] = 1.0;
}

__global__ void fill_bits_kernel(unsigned long long *__restrict__ p, int64_t n, unsigned long long v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void export_results_kernel(const int64_t *__restrict__ dP, int64_t cap, const int64_t *__restrict__ d_items,
                                      const int *__restrict__ d_max_row, const PreCounters *__restrict__ ctr,
                                      const int *__restrict__ val_err, const int2 *__restrict__ pairs,
                                      const double *__restrict__ raw, const int64_t *__restrict__ lk,
                                      const uint8_t *__restrict__ flags, FastStatus *__restrict__ st,
                                      int2 *__restrict__ h_pairs, double *__restrict__ h_raw,
                                      int64_t *__restrict__ h_lk, uint8_t *__restrict__ h_flags,
                                      const unsigned long long *__restrict__ ee = nullptr) {
    LC_PDL_WAIT();   // launched as the sum's programmatic dependent (LC_EXPORT_PDL); else a no-op
    const int64_t P = *dP < cap ? *dP : cap;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += stride) {
        if (pairs) h_pairs[i] = pairs[i];
        if (raw) {   // sharded runs export the sums after the partials exchange
            h_raw[i] = raw[i];
            h_lk[i] = lk[i];
            h_flags[i] = flags[i];
        }
    }
    if (st && blockIdx.x == 0 && threadIdx.x == 0) {
        FastStatus f;
        f.P = dP[2];          // the real counts (dP[0], dP[1] are 0 for an unusable run)
        f.n_items = dP[3];
        f.max_row = *d_max_row;
        f.zero_loop = ctr->zero_loop;
        f.n_unpaired = ctr->n_unpaired;
        f.n_large = ctr->n_large;
        f.marked = ctr->marked;
        f.val_err[0] = val_err[0];
        f.val_err[1] = val_err[1];
        f.first_fail = ee ? ee[0] : ~0ULL;
        f.n_eval = ee ? ee[1] : ~0ULL;
        *st = f;
    }
}

// The per-pair reduction (warp_pair_sum, the order of reduce_pairs_kernel) fused
// with the export: each block sums 64 pairs into shared memory (8 warps x 8
// pairs), then 64 threads write raw / lk / flags to pinned host memory in
// coalesced runs; block 0 also writes the status record.
#ifndef LC_EXPORT_CHUNK
#define LC_EXPORT_CHUNK 64   // pairs per block (A/B builds: -DLC_EXPORT_CHUNK=n, a multiple of 8)
#endif
constexpr int kExportChunk = LC_EXPORT_CHUNK;
constexpr int kPairsPerWarp = kExportChunk / 8;
// 8 warps x kPairsPerWarp pairs per block; lane j + 1 carries pair j's end offset
static_assert(kExportChunk % 8 == 0 && kPairsPerWarp >= 1 && kPairsPerWarp < 32,
              "LC_EXPORT_CHUNK must be a multiple of 8 below 256");
__global__ void __launch_bounds__(256) reduce_export_kernel(
    const double *__restrict__ partials, const int64_t *__restrict__ item_off, const int64_t *__restrict__ dP,
    int64_t cap, const int64_t *__restrict__ d_items, const int *__restrict__ d_max_row,
    const PreCounters *__restrict__ ctr, const int *__restrict__ val_err, FastStatus *__restrict__ st,
    double *__restrict__ raw, int64_t *__restrict__ lk, uint8_t *__restrict__ flags, double *__restrict__ h_raw,
    int64_t *__restrict__ h_lk, uint8_t *__restrict__ h_flags) {
    __shared__ double sraw[kExportChunk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t P = *dP < cap ? *dP : cap;
    for (int64_t c0 = (int64_t)blockIdx.x * kExportChunk; c0 < P; c0 += (int64_t)gridDim.x * kExportChunk) {
        // warp w sums pairs pb .. pb+7 in warp_pair_sum's order (lane strides,
        // then the xor butterfly: bitwise equal to reduce_pairs_kernel), with the
        // 9 offsets in one load and the pairs' first partials loaded side by side
        const int64_t pb = c0 + warp * kPairsPerWarp;
        // item_off null: one partial per pair (the pair-claiming Gauss kernel's sums)
        const int64_t off = lane <= kPairsPerWarp && pb + lane <= P ? (item_off ? item_off[pb + lane] : pb + lane) : 0;
        double v[kPairsPerWarp];
        int64_t b[kPairsPerWarp], e[kPairsPerWarp];
#pragma unroll
        for (int j = 0; j < kPairsPerWarp; ++j) {
            b[j] = __shfl_sync(0xffffffffu, off, j);
            e[j] = __shfl_sync(0xffffffffu, off, j + 1);
            if (pb + j >= P) e[j] = b[j];
        }
#pragma unroll
        for (int j = 0; j < kPairsPerWarp; ++j) {
            v[j] = 0.0;
            if (b[j] + lane < e[j]) v[j] += partials[b[j] + lane];
        }
#pragma unroll
        for (int j = 0; j < kPairsPerWarp; ++j)   // pairs of more than 32 items
            for (int64_t k = b[j] + lane + 32; k < e[j]; k += 32) v[j] += partials[k];
#pragma unroll
        for (int j = 0; j < kPairsPerWarp; ++j) {
#pragma unroll
            for (int o = 16; o; o >>= 1) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
            if (lane == 0) sraw[warp * kPairsPerWarp + j] = v[j];
        }
        __syncthreads();
        if (threadIdx.x < kExportChunk && c0 + threadIdx.x < P) {
            const int64_t p = c0 + threadIdx.x;
            const double v = sraw[threadIdx.x];
            int64_t r;
            const uint8_t f = round_link(v, r);
            raw[p] = v;   // the device copies serve lc_get_results
            lk[p] = r;
            flags[p] = f;
            h_raw[p] = v;
            h_lk[p] = r;
            h_flags[p] = f;
        }
        __syncthreads();
    }
    if (st && blockIdx.x == 0 && threadIdx.x == 0) {
        FastStatus f;
        f.P = dP[2];
        f.n_items = dP[3];
        f.max_row = *d_max_row;
        f.zero_loop = ctr->zero_loop;
        f.n_unpaired = ctr->n_unpaired;
        f.n_large = ctr->n_large;
        f.marked = ctr->marked;
        f.val_err[0] = val_err[0];
        f.val_err[1] = val_err[1];
        f.first_fail = ~0ULL;
        f.n_eval = ~0ULL;
        *st = f;
    }
}

void launch_reduce_export(const double *partials, const int64_t *item_off, const int64_t *dP, int64_t cap,
                          const int64_t *d_items, const int *d_max_row, const PreCounters *ctr, const int *val_err,
                          FastStatus *st, double *raw, int64_t *lk, uint8_t *flags, double *h_raw, int64_t *h_lk,
                          uint8_t *h_flags, cudaStream_t s) {
    int64_t blocks = ceil_div(cap > 0 ? cap : 1, kExportChunk);
    if (blocks > 148 * 8) blocks = 148 * 8;
    reduce_export_kernel<<<(unsigned)blocks, 256, 0, s>>>(partials, item_off, dP, cap, d_items, d_max_row, ctr,
                                                          val_err, st, raw, lk, flags, h_raw, h_lk, h_flags);
    LC_CHECK_LAUNCH();
}

}  // namespace

void Pipeline::init(cudaStream_t st) {
    s = st;
    for (auto &e : ev) LC_CUDA(cudaEventCreate(&e));
    // the checks branch runs at the highest priority: its blocks are dispatched ahead
    // of the Gauss kernel's persistent CTAs when both become ready after the PLS
    int prio_lo = 0, prio_hi = 0;
    LC_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    LC_CUDA(cudaStreamCreateWithPriority(&side[0], cudaStreamNonBlocking, prio_lo));
    LC_CUDA(cudaStreamCreateWithPriority(&side[1], cudaStreamNonBlocking, prio_hi));
    // the fused run's critical path (derive -> PLS -> Gauss sum) at the highest priority:
    // its small latency-bound kernels are dispatched ahead of the chord branch's blocks
    LC_CUDA(cudaStreamCreateWithPriority(&crit, cudaStreamNonBlocking, prio_hi));
    for (cudaEvent_t *e : {&ev_fork, &ev_chords, &ev_pairs, &ev_checks, &ev_stage, &ev_enter, &ev_leave})
        LC_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
}

void Pipeline::release() {
    DevBuf *bufs[] = {&d_ref_keys, &d_ref_lk, &d_posv, &d_want, &d_ee, &d_bounds, &d_tot, &d_coeffs, &d_t, &d_loff, &d_seg_box, &d_seg_fbox, &d_seg_sub, &d_loop_keys, &d_seg_loop, &d_loop_box, &d_min_diag, &d_model_exp,
                      &d_verts_in, &d_aos, &d_in_off, &d_voff, &d_X, &d_Y, &d_Z, &d_exp, &d_tmp_aos, &d_pairs,
                      &d_pg, &d_item_off, &d_item_pair, &d_scan, &d_counter, &d_partials, &d_raw, &d_lk, &d_flags,
                      &d_quads, &d_qout, &dout.X, &dout.Y, &dout.Z, &dout.voff, &dout.vert_off};
    for (DevBuf *b : bufs) b->release(s);
    DevBuf *pb[] = {&pls_sc.keys, &pls_sc.keys_sorted, &pls_sc.idx, &pls_sc.perm, &pls_sc.sbox, &pls_sc.counter,
                    &pls_sc.cub_tmp, &pls_sc.pair_keys, &pls_sc.pair_keys_sorted, &pls_sc.axis, &pls_sc.excl,
                    &pls_sc.counts, &pls_sc.offs, &pls_sc.lcell, &pls_sc.lrank, &pls_sc.acc};
    for (DevBuf *b : pb) b->release(s);
    pls_sc.acc_ready = nullptr;   // a new acc buffer gets its identity keys again
    DiscScratch &d = disc_sc;
    DevBuf *db[] = {&d.paired, &d.act_seg, &d.act_loop, &d.act_tlo, &d.act_thi, &d.act_off, &d.nxt_seg,
                    &d.nxt_loop, &d.nxt_tlo, &d.nxt_thi, &d.nxt_off, &d.nxt_partner, &d.box, &d.nxt_box,
                    &d.skey[0], &d.skey[1], &d.skey[2], &d.sperm[0], &d.sperm[1], &d.sperm[2], &d.iota,
                    &d.pair_axis, &d.sweep_off, &d.mark, &d.first_pair, &d.mark_scan, &d.done_seg, &d.done_tlo,
                    &d.done_seg2, &d.done_tlo2, &d.sort_idx, &d.sort_idx2, &d.done_cnt, &d.done_off,
                    &d.bad_first, &d.counters, &d.cub_tmp, &d.loop_err, &d.val_flags, &d.ucnt, &d.tmp_aos,
                    &d.prectr};
    for (DevBuf *b : db) b->release(s);
    if (s) cudaStreamSynchronize(s);
    h_res.release();
    h_excl.release();
    h_stage.release();
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    graph_exec = nullptr;
    for (auto &e : ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {ev_fork, ev_chords, ev_pairs, ev_checks, ev_stage, ev_enter, ev_leave})
        if (e) cudaEventDestroy(e);
    for (auto &x : side)
        if (x) cudaStreamDestroy(x);
    if (crit) cudaStreamDestroy(crit);
}

// Stage event on the stream; inside a stream capture it must become an
// external event-record node to stay usable for timing after graph replays.
void Pipeline::record(int e, cudaStream_t st) {
    if (!st) st = s;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    LC_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusActive)
        LC_CUDA(cudaEventRecordWithFlags(ev[e], st, cudaEventRecordExternal));
    else
        LC_CUDA(cudaEventRecord(ev[e], st));
}

float Pipeline::stage_ms(int e0, int e1) {
    float ms = 0.f;
    LC_CUDA(cudaEventSynchronize(ev[e1]));
    LC_CUDA(cudaEventElapsedTime(&ms, ev[e0], ev[e1]));
    return ms;
}

// ------------------------------------------------------------------ model

void Pipeline::reserve_derived() {
    d_seg_box.reserve(sizeof(double) * 6 * (M > 0 ? M : 1), s);
    d_seg_fbox.reserve(sizeof(float) * 6 * (M > 0 ? M : 1), s);
    if (kPass1Groups) d_seg_sub.reserve(sizeof(float) * 6 * pass1_group_stride(M, L), s);
    d_seg_loop.reserve(sizeof(int32_t) * (M > 0 ? M : 1), s);
    d_loop_box.reserve(sizeof(double) * 6 * (L > 0 ? L : 1), s);
    d_min_diag.reserve(sizeof(unsigned long long) * (L > 0 ? L : 1), s);
    d_model_exp.reserve(sizeof(int), s);
    d_loop_keys.reserve(sizeof(unsigned long long) * 6 * (L > 0 ? L : 1), s);
}

void Pipeline::derive() {
    if (!model_ready) throw Error(LC_ERR_STATE, "no model uploaded");
    record(EV_BEGIN);
    d_seg_box.reserve(sizeof(double) * 6 * (M > 0 ? M : 1), s);
    d_seg_fbox.reserve(sizeof(float) * 6 * (M > 0 ? M : 1), s);
    d_seg_loop.reserve(sizeof(int32_t) * (M > 0 ? M : 1), s);
    d_loop_box.reserve(sizeof(double) * 6 * (L > 0 ? L : 1), s);
    d_min_diag.reserve(sizeof(unsigned long long) * (L > 0 ? L : 1), s);
    d_model_exp.reserve(sizeof(int), s);
    // tight segment boxes, per-loop min diagonals, coordinate exponent, loop boxes
    d_loop_keys.reserve(sizeof(unsigned long long) * 6 * (L > 0 ? L : 1), s);
    launch_seg_boxes(model_poly ? nullptr : d_coeffs.as<double>(), model_poly ? nullptr : d_t.as<double>(),
                     model_poly ? d_verts_in.as<double>() : nullptr, d_loff.as<int64_t>(), L, M,
                     d_seg_box.as<double>(), d_seg_loop.as<int32_t>(), d_min_diag.as<unsigned long long>(),
                     d_model_exp.as<int>(), s, d_seg_fbox.as<float>(), d_loop_keys.as<unsigned long long>(),
                     d_loop_box.as<double>(), max_loop);
    derived = true;
    derived_in_run = true;
}

// The from_polyline coefficient arrays of a polyline model, for the stages that
// evaluate cubics (refinement passes, chord writes of the staged path).
void Pipeline::ensure_coeffs() {
    if (coeffs_ready) return;
    d_coeffs.reserve(sizeof(double) * 12 * (M > 0 ? M : 1), s);
    d_t.reserve(sizeof(double) * 2 * (M > 0 ? M : 1), s);
    if (M > 0) {
        polyline_coeffs_kernel<<<(unsigned)ceil_div(M, 256), 256, 0, s>>>(d_verts_in.as<double>(), d_loff.as<int64_t>(),
                                                                           L, M, d_coeffs.as<double>(), d_t.as<double>());
        LC_CHECK_LAUNCH();
    }
    coeffs_ready = true;
}

void Pipeline::upload_model(const double *coeffs, const double *t, const int64_t *loff, int64_t nloops) {
    L = nloops;
    M = L > 0 ? loff[L] : 0;
    if (L > 0 && loff[0] != 0) throw Error(LC_ERR_ARG, "loop offsets must start at 0");
    max_loop = 0;
    for (int64_t l = 0; l < L; ++l) {
        if (loff[l + 1] < loff[l]) throw Error(LC_ERR_ARG, "loop offsets must be non-decreasing");
        if (loff[l + 1] - loff[l] > max_loop) max_loop = loff[l + 1] - loff[l];
    }
    d_coeffs.reserve(sizeof(double) * 12 * (M > 0 ? M : 1), s);
    d_t.reserve(sizeof(double) * 2 * (M > 0 ? M : 1), s);
    d_loff.reserve(sizeof(int64_t) * (L + 1), s);
    if (M > 0) {
        LC_CUDA(cudaMemcpyAsync(d_coeffs.ptr, coeffs, sizeof(double) * 12 * M, cudaMemcpyHostToDevice, s));
        LC_CUDA(cudaMemcpyAsync(d_t.ptr, t, sizeof(double) * 2 * M, cudaMemcpyHostToDevice, s));
    }
    LC_CUDA(cudaMemcpyAsync(d_loff.ptr, loff, sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice, s));
    model_ready = true;
    model_poly = false;
    coeffs_ready = true;
    derived = false;
    polylines_ready = false;
    P = 0;
    LC_CUDA(cudaStreamSynchronize(s));   // the caller's host buffers may be released after return
}

void Pipeline::upload_model_polylines(const double *verts, const int64_t *loff, int64_t nloops) {
    L = nloops;
    M = L > 0 ? loff[L] : 0;
    if (L > 0 && loff[0] != 0) throw Error(LC_ERR_ARG, "loop offsets must start at 0");
    max_loop = 0;
    for (int64_t l = 0; l < L; ++l) {
        if (loff[l + 1] - loff[l] < 1) throw Error(LC_ERR_ARG, "every loop needs at least one vertex");
        if (loff[l + 1] - loff[l] > max_loop) max_loop = loff[l + 1] - loff[l];
    }
    d_loff.reserve(sizeof(int64_t) * (L + 1), s);
    d_verts_in.reserve(sizeof(double) * 3 * (M > 0 ? M : 1), s);
    if (M > 0) LC_CUDA(cudaMemcpyAsync(d_verts_in.ptr, verts, sizeof(double) * 3 * M, cudaMemcpyHostToDevice, s));
    LC_CUDA(cudaMemcpyAsync(d_loff.ptr, loff, sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice, s));
    model_ready = true;
    model_poly = true;
    coeffs_ready = false;
    derived = false;
    polylines_ready = false;
    P = 0;
    LC_CUDA(cudaStreamSynchronize(s));
}

namespace {

// Copy loop rows [l0, l1) of a per-loop pointer table into dst (row_bytes each).
void gather_loops(char *dst, const double *const *src, const int64_t *loff, int64_t l0, int64_t l1,
                  size_t row_bytes) {
    for (int64_t l = l0; l < l1; ++l) {
        const int64_t m = loff[l + 1] - loff[l];
        if (m > 0) std::memcpy(dst + (size_t)loff[l] * row_bytes, src[l], (size_t)m * row_bytes);
    }
}

}  // namespace

void Pipeline::upload_model_polyline_ptrs(const double *const *loop_verts, const int64_t *loff, int64_t nloops) {
    if (nloops > 0 && loff[0] != 0) throw Error(LC_ERR_ARG, "loop offsets must start at 0");
    int64_t mx = 0;
    for (int64_t l = 0; l < nloops; ++l) {
        const int64_t m = loff[l + 1] - loff[l];
        if (m < 1) throw Error(LC_ERR_ARG, "every loop needs at least one vertex");
        if (!loop_verts[l]) throw Error(LC_ERR_ARG, "null loop vertex pointer");
        if (m > mx) mx = m;
    }
    const int64_t nM = nloops > 0 ? loff[nloops] : 0;
    const size_t vbytes = sizeof(double) * 3 * (size_t)nM, obytes = sizeof(int64_t) * (size_t)(nloops + 1);
    if (stage_pending) {   // the previous upload's copy still reads the staging buffer
        LC_CUDA(cudaEventSynchronize(ev_stage));
        stage_pending = false;
    }
    h_stage.reserve(vbytes + obytes);
    char *st = static_cast<char *>(h_stage.ptr);
    // loops split into ~equal-byte ranges, one per thread (the caller's thread takes the first)
    const int64_t per_thread = 1 << 18;   // rows (6 MiB) per thread at least
    int nt = (int)std::min<int64_t>(8, std::max<int64_t>(1, nM / per_thread));
    const unsigned hw = std::thread::hardware_concurrency();
    const int share = gather_share > 1 ? gather_share : 1;   // ranks of one host split its cores
    if (hw > 0 && (unsigned)nt > hw / (2 * share)) nt = std::max(1, (int)hw / (2 * share));
    std::vector<int64_t> cut(nt + 1, nloops);
    cut[0] = 0;
    for (int k = 1, l = 0; k < nt; ++k) {
        const int64_t want = nM * k / nt;
        while (l < nloops && loff[l] < want) ++l;
        cut[k] = l;
    }
    std::vector<std::thread> th;
    for (int k = 1; k < nt; ++k)
        th.emplace_back(gather_loops, st, loop_verts, loff, cut[k], cut[k + 1], sizeof(double) * 3);
    gather_loops(st, loop_verts, loff, cut[0], cut[1], sizeof(double) * 3);
    std::memcpy(st + vbytes, loff, obytes);
    for (auto &x : th) x.join();
    L = nloops;
    M = nM;
    max_loop = mx;
    d_loff.reserve(obytes, s);
    d_verts_in.reserve(sizeof(double) * 3 * (M > 0 ? M : 1), s);
    if (M > 0) LC_CUDA(cudaMemcpyAsync(d_verts_in.ptr, st, vbytes, cudaMemcpyHostToDevice, s));
    LC_CUDA(cudaMemcpyAsync(d_loff.ptr, st + vbytes, obytes, cudaMemcpyHostToDevice, s));
    LC_CUDA(cudaEventRecord(ev_stage, s));
    stage_pending = true;
    model_ready = true;
    model_poly = true;
    coeffs_ready = false;
    derived = false;
    polylines_ready = false;
    P = 0;
}

int64_t Pipeline::potential_link_search(const uint64_t *excl_keys, int64_t n_excl, bool in_run) {
    if (!model_ready) throw Error(LC_ERR_STATE, "no model uploaded");
    if (!derived) derive();
    else if (!in_run) record(EV_BEGIN);
    // LINKCERT_PLS_SWEEP=1 selects the sort-and-sweep PLS instead of grid culling — tests cover both
    static const bool force_sweep = [] {
        const char *e = getenv("LINKCERT_PLS_SWEEP");
        return e && e[0] == '1';
    }();
    P = run_pls(d_loop_box.as<double>(), L, excl_keys, n_excl, pls_sc, d_pairs, s, force_sweep);
    record(EV_PLS);
    return P;
}

bool Pipeline::discretize(const DiscParams &prm) {
    if (!model_ready) throw Error(LC_ERR_STATE, "no model uploaded");
    ensure_derived();
    ensure_coeffs();
    DiscInput in{d_coeffs.as<double>(), d_t.as<double>(), d_loff.as<int64_t>(), d_seg_loop.as<int32_t>(),
                 d_seg_box.as<double>(), d_loop_box.as<double>(), d_min_diag.as<unsigned long long>(),
                 d_model_exp.as<int>(), L, M, d_pairs.as<int32_t>(), P};
    in.verts = model_poly ? d_verts_in.as<double>() : nullptr;
    in.seg_fbox = d_seg_fbox.as<float>();
    derr = DiscError();
    polylines_ready = false;
    if (!run_discretize(in, prm, disc_sc, dout, &derr, s)) return false;
    V = dout.V;
    Vc = dout.Vc;
    gX = dout.X.as<double>();
    gY = dout.Y.as<double>();
    gZ = dout.Z.as<double>();
    gvoff = dout.voff.as<int64_t>();
    polylines_ready = true;
    polylines_from_model = true;
    record(EV_DISC);
    return true;
}

void Pipeline::download_loop_boxes(double *lo, double *hi) {
    if (!model_ready) throw Error(LC_ERR_STATE, "no model uploaded");
    ensure_derived();
    std::vector<double> b((size_t)6 * L);
    if (L > 0)
        LC_CUDA(cudaMemcpyAsync(b.data(), d_loop_box.ptr, sizeof(double) * 6 * L, cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
    for (int64_t l = 0; l < L; ++l)
        for (int d = 0; d < 3; ++d) {
            lo[3 * l + d] = b[d * L + l];
            hi[3 * l + d] = b[(3 + d) * L + l];
        }
}

void Pipeline::download_polylines(double *verts, int64_t *vert_off) {
    if (!polylines_ready || !polylines_from_model) throw Error(LC_ERR_STATE, "no discretized polylines");
    if (V > 0 && verts) {
        d_tmp_aos.reserve(sizeof(double) * 3 * V, s);
        unpack_polylines(dout, L, d_model_exp.as<int>(), d_tmp_aos.as<double>(), s);
        LC_CUDA(cudaMemcpyAsync(verts, d_tmp_aos.ptr, sizeof(double) * 3 * V, cudaMemcpyDeviceToHost, s));
    }
    if (vert_off)
        LC_CUDA(cudaMemcpyAsync(vert_off, dout.vert_off.ptr, sizeof(int64_t) * (L + 1), cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ gauss

// Host AoS polylines (no closing vertex; loop v = rows [vert_off[v], vert_off[v+1]))
// -> device closed SoA with vertex 0 repeated at the end of every loop
// (direct.py:164-166 _closed), scaled by an exact power of two.
void Pipeline::upload_polylines(const double *verts, const int64_t *vert_off, int64_t nloops) {
    L = nloops;
    model_ready = false;
    V = L > 0 ? vert_off[L] - vert_off[0] : 0;
    if (L > 0 && vert_off[0] != 0) throw Error(LC_ERR_ARG, "vert_off[0] must be 0");
    for (int64_t l = 0; l < L; ++l)
        if (vert_off[l + 1] < vert_off[l]) throw Error(LC_ERR_ARG, "vert_off must be non-decreasing");
    h_voff.resize((size_t)L + 1);
    for (int64_t v = 0; v <= L; ++v) h_voff[v] = (L > 0 ? vert_off[v] : 0) + v;
    Vc = V + L;
    d_aos.reserve(sizeof(double) * 3 * (size_t)(V > 0 ? V : 1), s);
    d_in_off.reserve(sizeof(int64_t) * (size_t)(L + 1), s);
    d_voff.reserve(sizeof(int64_t) * (size_t)(L + 1), s);
    d_X.reserve(sizeof(double) * (size_t)(Vc + 1), s);
    d_Y.reserve(sizeof(double) * (size_t)(Vc + 1), s);
    d_Z.reserve(sizeof(double) * (size_t)(Vc + 1), s);
    d_exp.reserve(sizeof(int) * 2, s);
    if (V > 0) LC_CUDA(cudaMemcpyAsync(d_aos.ptr, verts, sizeof(double) * 3 * V, cudaMemcpyHostToDevice, s));
    if (L > 0) {
        LC_CUDA(cudaMemcpyAsync(d_in_off.ptr, vert_off, sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice, s));
        LC_CUDA(cudaMemcpyAsync(d_voff.ptr, h_voff.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice, s));
    }
    LC_CUDA(cudaMemsetAsync(d_exp.ptr, 0, sizeof(int), s));
    launch_max_exponent(d_aos.as<double>(), 3 * V, d_exp.as<int>(), s);
    launch_pack_closed_soa(d_aos.as<double>(), d_in_off.as<int64_t>(), d_voff.as<int64_t>(), L, Vc,
                           d_exp.as<int>(), d_X.as<double>(), d_Y.as<double>(), d_Z.as<double>(), s);
    gX = d_X.as<double>();
    gY = d_Y.as<double>();
    gZ = d_Z.as<double>();
    gvoff = d_voff.as<int64_t>();
    polylines_ready = true;
    polylines_from_model = false;
    LC_CUDA(cudaStreamSynchronize(s));
}

double Pipeline::link_direct(const double *loop1, int64_t n1, const double *loop2, int64_t n2, int mode,
                             cudaEvent_t ev0, cudaEvent_t ev1) {
    if (!gauss_mode_valid(mode)) throw Error(LC_ERR_ARG, "unknown Gauss-sum mode");
    const int64_t Vc = n1 + n2 + 2;   // both loops closed (their first vertex repeated)
    // the exact power-of-two scale of upload_polylines (largest exponent field of any coordinate)
    int emax = 0;
    for (int k = 0; k < 2; ++k) {
        const double *a = k ? loop2 : loop1;
        const int64_t n = 3 * (k ? n2 : n1);
        for (int64_t q = 0; q < n; ++q) {
            uint64_t b;
            std::memcpy(&b, a + q, 8);
            const int e = (int)((b >> 52) & 0x7ff);
            emax = e > emax ? e : emax;
        }
    }
    int e = emax - 1023;
    e = e < -1022 ? -1022 : (e > 1022 ? 1022 : e);
    double scale;
    const uint64_t sbits = (uint64_t)(1023 - e) << 52;
    std::memcpy(&scale, &sbits, 8);
    // pair (0, 1): loop 1 = columns ("l"), loop 2 = rows ("k"), as the staged path tiles it
    const bool seq = gauss_mode_sequential(mode);
    PairGeom g = make_pair_geom(0, n1 + 1, (int)n1, (int)n2, seq);
    // one pair alone: shorter column strips until there are ~8 items per SM (a 1024 x 1024
    // pair is otherwise 8 items — 8 warps on the whole GPU)
    for (int cl = g.cl; !seq && (int64_t)g.items_r * g.items_c < 8 * (int64_t)num_sms() && cl > 16;) {
        cl = cl / 2 > 16 ? cl / 2 : 16;
        g = make_pair_geom(0, n1 + 1, (int)n1, (int)n2, false, cl);
    }
    const int64_t items = (int64_t)g.items_r * g.items_c;
    // staging layout: X | Y | Z (Vc each, padded to 8 doubles) | items | item_off[2]
    const int64_t cv = (Vc + 7) & ~int64_t(7);
    const size_t bytes = sizeof(double) * 3 * cv + sizeof(ItemRec) * (items > 0 ? items : 1) + 2 * sizeof(int64_t);
    h_ld.reserve(bytes);
    d_ld.reserve(bytes, s);
    d_ld_out.reserve(sizeof(double) * (items > 0 ? items : 1) + 64, s);
    d_counter.reserve(sizeof(unsigned long long), s);
    char *h = static_cast<char *>(h_ld.ptr);   // (the previous call's copies completed with its sync)
    double *X = reinterpret_cast<double *>(h), *Y = X + cv, *Z = Y + cv;
    int64_t v = 0;
    for (int k = 0; k < 2; ++k) {
        const double *a = k ? loop2 : loop1;
        const int64_t n = k ? n2 : n1;
        for (int64_t q = 0; q <= n; ++q, ++v) {
            const int64_t src = q < n ? q : 0;
            X[v] = a[3 * src] * scale;
            Y[v] = a[3 * src + 1] * scale;
            Z[v] = a[3 * src + 2] * scale;
        }
    }
    ItemRec *it = reinterpret_cast<ItemRec *>(h + sizeof(double) * 3 * cv);
    for (int64_t k = 0; k < items; ++k) {
        it[k].g = g;
        it[k].ir = (int32_t)(k / g.items_c);
        it[k].ic = (int32_t)(k % g.items_c);
    }
    int64_t *ioff = reinterpret_cast<int64_t *>(reinterpret_cast<char *>(it) + sizeof(ItemRec) * (items > 0 ? items : 1));
    ioff[0] = 0;
    ioff[1] = items;
    LC_CUDA(cudaMemcpyAsync(d_ld.ptr, h, bytes, cudaMemcpyHostToDevice, s));
    char *d = static_cast<char *>(d_ld.ptr);
    const double *dX = reinterpret_cast<const double *>(d), *dY = dX + cv, *dZ = dY + cv;
    const ItemRec *dit = reinterpret_cast<const ItemRec *>(d + sizeof(double) * 3 * cv);
    const int64_t *dioff =
        reinterpret_cast<const int64_t *>(d + sizeof(double) * 3 * cv + sizeof(ItemRec) * (items > 0 ? items : 1));
    double *partials = d_ld_out.as<double>();
    double *raw = reinterpret_cast<double *>(reinterpret_cast<char *>(partials) + sizeof(double) * (items > 0 ? items : 1));
    int64_t *lk = reinterpret_cast<int64_t *>(raw + 1);
    uint8_t *fl = reinterpret_cast<uint8_t *>(lk + 1);
    LC_CUDA(cudaEventRecord(ev0, s));
    launch_gauss_items(mode, dX, dY, dZ, dit, 0, items, d_counter.as<unsigned long long>(), partials, s);
    LC_CUDA(cudaEventRecord(ev1, s));
    launch_reduce_pairs(partials, dioff, 1, raw, lk, fl, s);
    double out = 0.0;
    LC_CUDA(cudaMemcpyAsync(h, raw, sizeof(double), cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
    std::memcpy(&out, h, sizeof(double));
    return out;
}

void Pipeline::upload_pairs(const int32_t *pairs, int64_t npairs) {
    P = npairs;
    d_pairs.reserve(sizeof(int32_t) * 2 * (size_t)(P > 0 ? P : 1), s);
    for (int64_t p = 0; p < P; ++p) {
        const int32_t i = pairs[2 * p], j = pairs[2 * p + 1];
        if (i < 0 || j < 0 || i >= L || j >= L) throw Error(LC_ERR_ARG, "pair index out of range");
    }
    if (P > 0) LC_CUDA(cudaMemcpyAsync(d_pairs.ptr, pairs, sizeof(int32_t) * 2 * P, cudaMemcpyHostToDevice, s));
    LC_CUDA(cudaStreamSynchronize(s));
}

void Pipeline::download_pairs(int32_t *pairs) {
    if (P > 0) LC_CUDA(cudaMemcpyAsync(pairs, d_pairs.ptr, sizeof(int32_t) * 2 * P, cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
}

void Pipeline::build_gauss_items(int mode) {
    if (!polylines_ready) throw Error(LC_ERR_STATE, "no polylines staged");
    if (!gauss_mode_valid(mode)) throw Error(LC_ERR_ARG, "unknown Gauss-sum mode");
    items_seq = gauss_mode_sequential(mode);
    d_pg.reserve(sizeof(PairGeom) * (size_t)(P > 0 ? P : 1), s);
    d_item_off.reserve(sizeof(int64_t) * (size_t)(P + 1), s);
    const size_t scan_bytes = build_items_scan_bytes(P > 0 ? P : 1);
    d_scan.reserve(scan_bytes, s);
    d_counter.reserve(sizeof(unsigned long long), s);
    n_items = build_items(d_pairs.as<int32_t>(), P, gvoff, d_pg.as<PairGeom>(), d_item_off.as<int64_t>(), d_scan.ptr,
                          d_scan.bytes, s, true, nullptr, items_seq);
    retile_few_items();
    finish_items();
}

// Few work items (a pair or two of long loops: a lone 1024 x 1024 pair is 8 items,
// 8 warps on the GPU): rebuild with shorter column strips for ~8 items per SM.  Only
// where no fused run of the same model exists to stay bitwise equal to — polylines
// staged directly, or a model with a loop the fused path does not take (> 256 segments).
void Pipeline::retile_few_items() {
    const int64_t target = 8 * (int64_t)num_sms();
    if (items_seq || n_items <= 0 || n_items >= target || (polylines_from_model && max_loop <= 256)) return;
    int max_cl = kMaxColsPerLane;
    for (int64_t est = n_items; est < target && max_cl > 16; est *= 2) max_cl /= 2;
    n_items = build_items(d_pairs.as<int32_t>(), P, gvoff, d_pg.as<PairGeom>(), d_item_off.as<int64_t>(), d_scan.ptr,
                          d_scan.bytes, s, true, nullptr, false, max_cl);
}

bool Pipeline::build_gauss_items_checked(int mode) {
    if (!polylines_ready) throw Error(LC_ERR_STATE, "no polylines staged");
    if (!gauss_mode_valid(mode)) throw Error(LC_ERR_ARG, "unknown Gauss-sum mode");
    items_seq = gauss_mode_sequential(mode);
    d_pg.reserve(sizeof(PairGeom) * (size_t)(P > 0 ? P : 1), s);
    d_item_off.reserve(sizeof(int64_t) * (size_t)(P + 1), s);
    const size_t scan_bytes = build_items_scan_bytes(P > 0 ? P : 1);
    d_scan.reserve(scan_bytes, s);
    d_counter.reserve(sizeof(unsigned long long), s);
    build_items(d_pairs.as<int32_t>(), P, gvoff, d_pg.as<PairGeom>(), d_item_off.as<int64_t>(), d_scan.ptr,
                d_scan.bytes, s, false, nullptr, items_seq);
    int ve[2] = {INT_MAX, INT_MAX};
    n_items = 0;
    LC_CUDA(cudaMemcpyAsync(&n_items, d_item_off.as<int64_t>() + P, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    if (dout.validation_pending && dout.d_val_err)
        LC_CUDA(cudaMemcpyAsync(ve, dout.d_val_err, sizeof ve, cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
    if (dout.validation_pending) {
        dout.validation_pending = false;
        if (validation_error(ve, &derr)) {
            polylines_ready = false;
            return false;
        }
    }
    retile_few_items();
    finish_items();
    return true;
}

void Pipeline::finish_items() {
    items_ready = true;
    d_partials.reserve(sizeof(double) * (size_t)(n_items > 0 ? n_items : 1), s);
    d_item_pair.reserve(sizeof(ItemRec) * (size_t)(n_items > 0 ? n_items : 1), s);
    launch_item_pairs(d_item_off.as<int64_t>(), d_pg.as<PairGeom>(), P, n_items, d_item_pair.as<ItemRec>(), s);
    d_raw.reserve(sizeof(double) * (size_t)(P > 0 ? P : 1), s);
    d_lk.reserve(sizeof(int64_t) * (size_t)(P > 0 ? P : 1), s);
    d_flags.reserve((size_t)(P > 0 ? P : 1), s);
}

void Pipeline::run_gauss(int mode, int64_t item_begin, int64_t item_end, double *partials_ext,
                         cudaEvent_t ev0, cudaEvent_t ev1) {
    if (!gauss_mode_valid(mode)) throw Error(LC_ERR_ARG, "unknown Gauss-sum mode");
    if (!items_ready) throw Error(LC_ERR_STATE, "no work items built (lc_prepare_gauss)");
    if (gauss_mode_sequential(mode) != items_seq)
        throw Error(LC_ERR_STATE, "the work items were built for another Gauss-sum mode");
    double *out = partials_ext ? partials_ext : d_partials.as<double>();
    LC_CUDA(cudaEventRecord(ev0 ? ev0 : ev[EV_GAUSS0], s));
    launch_gauss_items(mode, gX, gY, gZ, d_item_pair.as<ItemRec>(),
                       item_begin, item_end, d_counter.as<unsigned long long>(), out, s);
    LC_CUDA(cudaEventRecord(ev1 ? ev1 : ev[EV_GAUSS1], s));
}

void Pipeline::reduce_pairs(const double *partials_ext) {
    const double *in = partials_ext ? partials_ext : d_partials.as<double>();
    launch_reduce_pairs(in, d_item_off.as<int64_t>(), P, d_raw.as<double>(), d_lk.as<int64_t>(),
                        d_flags.as<uint8_t>(), s);
    record(EV_END);
}

void Pipeline::download_results(double *raw, int64_t *lk, uint8_t *flags) {
    if (P > 0) {
        if (raw) LC_CUDA(cudaMemcpyAsync(raw, d_raw.ptr, sizeof(double) * P, cudaMemcpyDeviceToHost, s));
        if (lk) LC_CUDA(cudaMemcpyAsync(lk, d_lk.ptr, sizeof(int64_t) * P, cudaMemcpyDeviceToHost, s));
        if (flags) LC_CUDA(cudaMemcpyAsync(flags, d_flags.ptr, (size_t)P, cudaMemcpyDeviceToHost, s));
    }
    LC_CUDA(cudaStreamSynchronize(s));
}

void Pipeline::download_results_pinned() {
    const size_t n = (size_t)(P > 0 ? P : 0);
    h_res.reserve(n * (8 + 8 + 8 + 1) + 64);
    char *h = static_cast<char *>(h_res.ptr);
    res_pairs = h;
    res_raw = h + 8 * n;
    res_lk = h + 16 * n;
    res_flags = h + 24 * n;
    if (n > 0) {
        LC_CUDA(cudaMemcpyAsync(h, d_pairs.ptr, 8 * n, cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaMemcpyAsync(h + 8 * n, d_raw.ptr, 8 * n, cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaMemcpyAsync(h + 16 * n, d_lk.ptr, 8 * n, cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaMemcpyAsync(h + 24 * n, d_flags.ptr, n, cudaMemcpyDeviceToHost, s));
    }
    LC_CUDA(cudaStreamSynchronize(s));
    h_res_P = (int64_t)n;
}

int Pipeline::run_fast(const uint64_t *excl_keys, int64_t n_excl, const DiscParams &prm, int mode, int shard,
                       int shards, bool async, bool force_sharded) {
    pend.on = false;
    if (shards < 1 || shard < 0 || shard >= shards) throw Error(LC_ERR_ARG, "bad shard");
    // sharded: the partials are exchanged (all-reduce) before the per-pair sums —
    // every run of a multi-GPU communicator, including world size 1
    const bool sharded = shards > 1 || force_sharded;
    // loops longer than the brute-force side limit make every pair they are in a
    // large (sweep) pair: the staged path handles those models directly
    if (!model_ready || L < 2 || M == 0 || prm.max_passes < 1 || max_loop > 256 ||
        (int64_t)kRowSlots * L >= (int64_t(1) << 24))   // the packed row scan holds P in 24 bits
        return FAST_FALLBACK;
    if (!gauss_mode_valid(mode)) throw Error(LC_ERR_ARG, "unknown Gauss-sum mode");
    if (gauss_mode_sequential(mode)) return FAST_FALLBACK;   // the anglesum variant: staged path (own item tiling)
    // pair capacity: the grid PLS bound (16 per row) until a run has shown the
    // model's pair count; then that plus headroom (smaller grids and scans)
    int64_t pcap = (int64_t)kRowSlots * L;
    if (pairs_seen > 0 && pairs_seen + pairs_seen / 4 + 1024 < pcap) pcap = pairs_seen + pairs_seen / 4 + 1024;
    const int64_t icap = items_cap > pcap ? items_cap : pcap;
    h_res_P = -1;
    fused_shard_pending = false;
    polylines_ready = false;
    // every buffer sized up front from host-known capacities
    pls_sc.excl.reserve(sizeof(uint64_t) * (n_excl > 0 ? n_excl : 1), s);
    h_excl.reserve(sizeof(uint64_t) * (n_excl > 0 ? n_excl : 1));
    d_pairs.reserve(sizeof(int32_t) * 2 * pcap, s);
    d_pg.reserve(sizeof(PairGeom) * pcap, s);
    d_item_off.reserve(sizeof(int64_t) * (pcap + 1), s);
    d_scan.reserve(build_items_scan_bytes(pcap), s);
    d_counter.reserve(sizeof(unsigned long long), s);
    reserve_pls_grid(L, pls_sc, s);   // prezeroed by the run's first kernel
    d_tot.reserve(4 * sizeof(int64_t), s);
    part_cap = pcap;   // pair partials (sharded); a shard writes only its cost-balanced pair range
    const bool ee = ee_on && !sharded;   // device early exit (single GPU; sharded runs replay it on the host)
    if (ee) {
        d_posv.reserve(sizeof(int64_t) * pcap, s);
        d_want.reserve(sizeof(int64_t) * pcap, s);
        d_ee.reserve(2 * sizeof(unsigned long long), s);
    }
    d_partials.reserve(sizeof(double) * part_cap, s);
    d_bounds.reserve(sizeof(int64_t) * (shards + 1), s);
    d_item_pair.reserve(sizeof(ItemRec) * icap, s);
    d_raw.reserve(sizeof(double) * pcap, s);
    d_lk.reserve(sizeof(int64_t) * pcap, s);
    d_flags.reserve((size_t)pcap, s);
    const size_t head = 128;
    h_res.reserve(head + (size_t)pcap * 25);
    char *h = static_cast<char *>(h_res.ptr);
    FastStatus *st = reinterpret_cast<FastStatus *>(h);
    char *hp = h + head, *hr = hp + 8 * pcap, *hl = hr + 8 * pcap, *hf = hl + 8 * pcap;
    if (n_excl > 0) std::memcpy(h_excl.ptr, excl_keys, sizeof(uint64_t) * n_excl);

    const PreCounters *ctr = nullptr;
    // The whole device sequence; stream-capturable (no allocation once the
    // buffers are sized, no host-pageable copies, no host syncs).
    const bool split = seg_boxes_split_ok(L, max_loop);
    if (split) reserve_derived();
    static const bool env_detail = [] {
        const char *e = getenv("LINKCERT_STAGE_TIMES");
        return e && e[0] == '1';
    }();
    const bool detail = stage_detail || env_detail;
    auto enqueue = [&]() {
        // the whole sequence runs on the high-priority critical stream, joined to the
        // caller's stream at both ends (captured with it into the graph)
        cudaStream_t caller = s;
        LC_CUDA(cudaEventRecord(ev_enter, caller));
        LC_CUDA(cudaStreamWaitEvent(crit, ev_enter, 0));
        s = crit;
        struct Restore {
            cudaStream_t &ref, val;
            ~Restore() { ref = val; }
        } restore{s, caller};
        tl_reset();
        if (split) {   // the loop half of derive on the critical path, the segment half on the chord branch
            if (detail) record(EV_BEGIN);
            derived = true;
            derived_in_run = true;
        } else {
            derive();   // records EV_BEGIN; (re)sizes the box buffers read below
        }
        DiscInput in{d_coeffs.as<double>(), d_t.as<double>(), d_loff.as<int64_t>(), d_seg_loop.as<int32_t>(),
                     d_seg_box.as<double>(), d_loop_box.as<double>(), d_min_diag.as<unsigned long long>(),
                     d_model_exp.as<int>(), L, M, d_pairs.as<int32_t>(), pcap};
        in.verts = model_poly ? d_verts_in.as<double>() : nullptr;
        in.seg_fbox = d_seg_fbox.as<float>();
        in.seg_sub = split && kPass1Groups ? d_seg_sub.as<float>() : nullptr;   // written by the segment half
        reserve_discretize_fast(in, disc_sc, dout, s);
        // every initial value of the run — the pass-1 counters + abort flag and
        // validation slots (launch_discretize_init's values, before any branch reads
        // them), the grid PLS memsets, the Gauss claim counter — written by the run's
        // first kernel: the loop-box kernel on the split path, else one prezero node
        static_assert(sizeof(PreCounters) == 32 && offsetof(PreCounters, marked) == 16 &&
                          offsetof(PreCounters, err_loop) == 24,
                      "prezero word layout of PreCounters");
        unsigned *pc = disc_sc.prectr.as<unsigned>();
        const ZeroRange extra[] = {
            {pc, 1, (unsigned)INT_MAX},                   // zero_loop
            {pc + 1, 5, 0u},                              // n_unpaired, n_large, abort, marked
            {pc + 6, 1, (unsigned)INT_MAX},               // err_loop
            {pc + 7, 1, 0u},                              // pad
            {disc_sc.val_err2.ptr, 2, (unsigned)INT_MAX}, // validation: first bad loop / pair
            {d_counter.ptr, 2, 0u},                       // Gauss item claim counter
            {d_model_exp.ptr, 1, 0u},                     // coordinate exponent (atomicMax)
            {ee ? d_ee.ptr : nullptr, ee ? 2 : 0, ~0u},  // early exit: first failure (~0)
            {ee ? static_cast<unsigned *>(d_ee.ptr) + 2 : nullptr, ee ? 2 : 0, 0u},   // pairs evaluated
            {disc_sc.val_flags.ptr, L > 0 ? L : 1, 0u},                 // chords: PolylineLoop flags
            {disc_sc.paired.ptr, (L + 3) / 4 > 0 ? (L + 3) / 4 : 1, 0u}, // checks: paired-loop bytes
        };
        const int n_extra = (int)(sizeof extra / sizeof extra[0]);
        if (!split) {
            launch_grid_prezero(L, pls_sc, extra, n_extra, s);
            tl_mark("prezero", s);
        }
        // branch 1: the chords need only the model — they run beside the PLS; the
        // segment half of derive goes with them, after the loop half (which it
        // would otherwise slow down by sharing the HBM bandwidth on the critical path)
        if (split) {
            const double *vp = model_poly ? d_verts_in.as<double>() : nullptr;
            const double *cp = model_poly ? nullptr : d_coeffs.as<double>(), *tp = model_poly ? nullptr : d_t.as<double>();
            // loop boxes + minimum diagonals with the PLS grid reduction folded in, and the initial values
            launch_loop_grid(cp, tp, vp, d_loff.as<int64_t>(), L, d_min_diag.as<unsigned long long>(),
                             d_loop_box.as<double>(), pls_sc, s, kChainPdl && !timeline().on, extra, n_extra);
            tl_mark("loop_boxes", s);
        }
        LC_CUDA(cudaEventRecord(ev_fork, s));
        LC_CUDA(cudaStreamWaitEvent(side[0], ev_fork, 0));
        if (split) {
            const double *vp = model_poly ? d_verts_in.as<double>() : nullptr;
            const double *cp = model_poly ? nullptr : d_coeffs.as<double>(), *tp = model_poly ? nullptr : d_t.as<double>();
            launch_seg_boxes_split(cp, tp, vp, d_loff.as<int64_t>(), L, M, false, d_seg_box.as<double>(),
                                   d_seg_fbox.as<float>(), d_seg_loop.as<int32_t>(), d_model_exp.as<int>(), nullptr,
                                   nullptr, side[0], const_cast<float *>(in.seg_sub));
            tl_mark("S0:seg_boxes", side[0]);
        }
        launch_discretize_chords(in, prm, disc_sc, dout, side[0], /*prezeroed=*/true);
        tl_mark("S0:chords", side[0]);
        LC_CUDA(cudaEventRecord(ev_chords, side[0]));
        if (n_excl > 0)
            LC_CUDA(cudaMemcpyAsync(pls_sc.excl.ptr, h_excl.ptr, sizeof(uint64_t) * n_excl, cudaMemcpyHostToDevice,
                                    s));
        const int *dmx = nullptr;
        launch_pls_grid(d_loop_box.as<double>(), L, n_excl, pls_sc, d_pairs.as<int32_t>(), pcap, d_loff.as<int64_t>(),
                        d_pg.as<PairGeom>(), d_item_off.as<int64_t>(), d_tot.as<int64_t>(), icap, s, &dmx,
                        /*prezeroed=*/true, /*grid_ready=*/split, kChainPdl && !timeline().on);
        const int64_t *dP = d_tot.as<int64_t>(), *d_items = d_tot.as<int64_t>() + 1;
        if (detail) record(EV_PLS);
        // branch 2: pass-1 detection + validation only feed the status — they run
        // beside the work items and the Gauss sum
        LC_CUDA(cudaEventRecord(ev_pairs, s));
        LC_CUDA(cudaStreamWaitEvent(side[1], ev_pairs, 0));
        // the pass-1 pair check goes on the critical stream right before the sum, which
        // starts beside it as its programmatic dependent; the rest of the checks stay on
        // this branch (measured: the check inside the Gauss kernel, 0.49 ms per Kusari
        // step, or starved on this branch behind the persistent sum, 0.47 ms)
        launch_discretize_checks(in, dP, prm, disc_sc, dout, side[1], ev_chords, &ctr, kBrutePdl,
                                 /*prezeroed=*/true);
        tl_mark("S1:checks", side[1]);
        if (detail) record(EV_DISC, side[1]);
        // the pair list is final: the copy engine moves the whole capacity to pinned
        // memory while the sums run (no SM time; the host reads the first P)
        LC_CUDA(cudaMemcpyAsync(hp, d_pairs.ptr, sizeof(int32_t) * 2 * pcap, cudaMemcpyDeviceToHost, side[1]));
        LC_CUDA(cudaEventRecord(ev_checks, side[1]));
        tl_mark("pls_items", s);
        if (sharded) {   // pairs of other shards: the bits of -0.0 (the int64 MAX all-reduce identity)
            fill_bits_kernel<<<(unsigned)ceil_div(part_cap, 256), 256, 0, s>>>(
                reinterpret_cast<unsigned long long *>(d_partials.ptr), part_cap, 0x8000000000000000ull);
            LC_CHECK_LAUNCH();
            launch_shard_bounds(d_pg.as<PairGeom>(), nullptr, pcap, dP, shards, d_bounds.as<int64_t>(), s);
        }
        EarlyExitArgs eea;
        if (ee) {   // the certificate's ordering of the candidates, and certificate pairs no longer candidates
            launch_early_exit_order(d_pairs.as<int32_t>(), dP, pcap, d_ref_keys.as<uint64_t>(),
                                    d_ref_lk.as<int64_t>(), n_ref, d_posv.as<int64_t>(), d_want.as<int64_t>(),
                                    d_ee.as<unsigned long long>(), s);
            eea.posv = d_posv.as<int64_t>();
            eea.want = d_want.as<int64_t>();
            eea.first_fail = d_ee.as<unsigned long long>();
            eea.n_eval = d_ee.as<unsigned long long>() + 1;
        }
        LC_CUDA(cudaStreamWaitEvent(s, ev_chords, 0));   // the sum reads the chords (the check, the segment boxes)
        tl_mark("chords_joined", s);
        record(EV_GAUSS0);
#ifndef LC_AB_NO_PASS1   // (A/B measurement builds only: without the pass-1 check the fused result is unchecked)
        if (kBrutePdl) launch_pass1_brute(in, dP, disc_sc, s);   // immediately before the sum: its PDL primary
#endif
        // warps claim whole pairs; unsharded, each pair's raw / lk / flags go straight to
        // the pinned result arrays as it completes (no reduce / export pass after the sum)
        launch_gauss_pairs(mode, dout.X.as<double>(), dout.Y.as<double>(), dout.Z.as<double>(), d_pg.as<PairGeom>(), dP,
                           pcap, d_counter.as<unsigned long long>(), &disc_sc.prectr.as<PreCounters>()->abort,
                           sharded ? d_bounds.as<int64_t>() : nullptr, shard,
                           sharded ? d_partials.as<double>() : nullptr, d_raw.as<double>(), d_lk.as<int64_t>(),
                           d_flags.as<uint8_t>(), reinterpret_cast<double *>(hr), reinterpret_cast<int64_t *>(hl),
                           reinterpret_cast<uint8_t *>(hf), s, eea, kBrutePdl);
#if LC_EXPORT_PDL
        // the status export as the sum's programmatic dependent (no event node between them)
        LC_CUDA(cudaStreamWaitEvent(s, ev_checks, 0));
        launch_pdl(export_results_kernel, dim3(1), dim3(32), s, !timeline().on, dP, pcap, d_items, dmx, ctr,
                   (const int *)dout.d_val_err, (const int2 *)nullptr, (const double *)nullptr,
                   (const int64_t *)nullptr, (const uint8_t *)nullptr, st, (int2 *)nullptr, (double *)nullptr,
                   (int64_t *)nullptr, (uint8_t *)nullptr,
                   (const unsigned long long *)(ee ? d_ee.as<unsigned long long>() : nullptr));
        record(EV_GAUSS1);
        tl_mark("gauss", s);
#else
        record(EV_GAUSS1);
        tl_mark("gauss", s);
        LC_CUDA(cudaStreamWaitEvent(s, ev_checks, 0));
        // the run's status record (sharded: lc_shard_finish reduces after the exchange)
        export_results_kernel<<<1, 32, 0, s>>>(dP, pcap, d_items, dmx, ctr, dout.d_val_err, nullptr, nullptr, nullptr,
                                               nullptr, st, nullptr, nullptr, nullptr, nullptr,
                                               ee ? d_ee.as<unsigned long long>() : nullptr);
#endif
        LC_CHECK_LAUNCH();
        if (detail) record(EV_END);   // "reduce" = Gauss end -> status in pinned memory
        tl_mark("export", s);
        LC_CUDA(cudaEventRecord(ev_leave, crit));
        LC_CUDA(cudaStreamWaitEvent(caller, ev_leave, 0));
    };

    static const bool no_graph = [] {
        const char *e = getenv("LINKCERT_NO_GRAPH");
        return e && e[0] == '1';
    }();
    FastKey key{L, M, pcap, icap, n_excl, mode, model_poly ? 1 : 0, shard, sharded ? shards : 0, prm.epsilon * prm.xi,
                2.220446049250313e-16 * prm.xi, alloc_generation().load(), ee ? n_ref : -1, detail};
    last_fast_graph = false;
    if (!no_graph && graph_exec && key == graph_key) {
        static const bool ginfo = [] {
            const char *e = getenv("LINKCERT_GRAPH_INFO");
            return e && e[0] == '1';
        }();
        const auto t0 = std::chrono::steady_clock::now();
        LC_CUDA(cudaGraphLaunch(graph_exec, s));
        if (ginfo) {
            const auto t1 = std::chrono::steady_clock::now();
            cudaStreamSynchronize(s);
            const auto t2 = std::chrono::steady_clock::now();
            fprintf(stderr, "[graph] launch call %.2f us, to sync return %.2f us\n",
                    std::chrono::duration<double, std::micro>(t1 - t0).count(),
                    std::chrono::duration<double, std::micro>(t2 - t0).count());
        }
        launch_counter().fetch_add(graph_launches, std::memory_order_relaxed);
        last_fast_graph = true;
        derived = true;
        derived_in_run = true;
        // host-side results of the captured launch helpers (device pointers are fixed)
        ctr = disc_sc.prectr.as<PreCounters>();
        dout.passes = 1;
        dout.splits = 0;
        dout.V = M;
        dout.Vc = M + L;
        dout.d_val_err = disc_sc.val_err2.as<int>();
    } else if (!no_graph && fast_seen_valid && key == fast_seen) {
        // same shape as the last completed run and nothing reallocated since: capture
        if (graph_exec) {
            cudaGraphExecDestroy(graph_exec);
            graph_exec = nullptr;
        }
        const long long n0 = launch_counter().load();
        cudaGraph_t g = nullptr;
        LC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue();
        } catch (...) {
            cudaStreamEndCapture(s, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        LC_CUDA(cudaStreamEndCapture(s, &g));
        graph_launches = launch_counter().load() - n0;
        if (const char *gi = getenv("LINKCERT_GRAPH_INFO"); gi && gi[0] == '1') {   // debug: node census
            size_t nn = 0;
            LC_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
            std::vector<cudaGraphNode_t> nodes(nn);
            LC_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
            int by_type[32] = {};
            for (auto n : nodes) {
                cudaGraphNodeType t;
                LC_CUDA(cudaGraphNodeGetType(n, &t));
                by_type[(int)t & 31]++;
            }
            fprintf(stderr, "[graph] %zu nodes:", nn);
            for (int t = 0; t < 32; ++t)
                if (by_type[t]) fprintf(stderr, " type%d=%d", t, by_type[t]);
            fprintf(stderr, "\n");
        }
        const bool same_gen = alloc_generation().load() == key.gen;
        if (same_gen) {
            // honour the captured per-node priorities (critical path / checks high, chords low)
            LC_CUDA(cudaGraphInstantiateWithFlags(&graph_exec, g, cudaGraphInstantiateFlagUseNodePriority));
            graph_key = key;
        }
        if (same_gen) {
            LC_CUDA(cudaGraphLaunch(graph_exec, s));
            last_fast_graph = true;
        }
        LC_CUDA(cudaGraphDestroy(g));
        if (!same_gen) {   // something allocated during capture: run it plainly (next call recaptures)
            launch_counter().fetch_sub(graph_launches, std::memory_order_relaxed);
            enqueue();
        }
    } else {
        enqueue();
    }
    last_detail = detail;
    pend.on = true;
    pend.key = key;
    pend.pcap = pcap;
    pend.icap = icap;
    pend.shards = shards;
    pend.sharded = sharded;
    pend.st = st;
    pend.hp = hp;
    pend.hr = hr;
    pend.hl = hl;
    pend.hf = hf;
    if (async) return FAST_PENDING;
    return finish_fast();
}

// Host side of a fused run: the one sync, then the device summary decides.
int Pipeline::finish_fast() {
    if (!pend.on) throw Error(LC_ERR_STATE, "no enqueued fused run");
    pend.on = false;
    const FastKey key = pend.key;
    const int64_t pcap = pend.pcap, icap = pend.icap;
    const bool pend_sharded = pend.sharded;
    char *hp = pend.hp, *hr = pend.hr, *hl = pend.hl, *hf = pend.hf;
    LC_CUDA(cudaStreamSynchronize(s));
    tl_print(last_fast_graph ? "fused graph" : "fused");
    fast_seen = key;
    fast_seen.gen = alloc_generation().load();
    fast_seen_valid = true;

    const FastStatus f = *pend.st;
    ee_first_fail = f.first_fail == ~0ULL ? -1 : (int64_t)f.first_fail;
    ee_n_eval = f.n_eval == ~0ULL ? -1 : (int64_t)f.n_eval;
    if (f.n_items > items_cap) items_cap = f.n_items;
    if (f.P > pairs_seen) pairs_seen = f.P;
    if (f.max_row > kRowSlots || f.P > pcap || f.zero_loop != INT_MAX || f.n_large != 0 || f.marked != 0 ||
        f.n_items > icap)
        return FAST_FALLBACK;
    // the run was the reference's: adopt its sizes as the pipeline state
    P = f.P;
    n_items = f.n_items;
    items_seq = false;
    items_ready = false;   // the fused run claims pairs: no item records (lc_prepare_gauss builds them)
    V = dout.V;
    Vc = dout.Vc;
    gX = dout.X.as<double>();
    gY = dout.Y.as<double>();
    gZ = dout.Z.as<double>();
    gvoff = dout.voff.as<int64_t>();
    dout.validation_pending = false;
    derr = DiscError();
    if (validation_error(f.val_err, &derr)) return FAST_INVALID;
    polylines_ready = true;
    polylines_from_model = true;
    res_pairs = hp;
    res_raw = hr;
    res_lk = hl;
    res_flags = hf;
    h_res_P = pend_sharded ? -1 : P;   // sharded: lc_shard_finish completes the results
    fused_shard_pending = pend_sharded;
    return FAST_OK;
}

// After an async sharded run and the in-place all-reduce of d_partials: the
// fixed-order per-pair reduction and the results into pinned memory, sized on
// the device (no host count needed), then the run's single host sync.
int Pipeline::shard_finish() {
    if (!pend.on) throw Error(LC_ERR_STATE, "no pending sharded run");
    const int64_t *dP = d_tot.as<int64_t>();
    launch_reduce_export(d_partials.as<double>(), nullptr, dP, pend.pcap, nullptr, nullptr, nullptr,
                         nullptr, nullptr, d_raw.as<double>(), d_lk.as<int64_t>(), d_flags.as<uint8_t>(),
                         reinterpret_cast<double *>(pend.hr), reinterpret_cast<int64_t *>(pend.hl),
                         reinterpret_cast<uint8_t *>(pend.hf), s);
    const int r = finish_fast();
    if (r == FAST_OK) {
        h_res_P = P;
        fused_shard_pending = false;
    }
    return r;
}

void Pipeline::set_early_exit(const uint64_t *keys, const int64_t *lk, int64_t n, bool enable) {
    ee_on = enable;
    if (!enable) return;
    if (n < 0 || (n > 0 && (!keys || !lk))) throw Error(LC_ERR_ARG, "bad certificate arrays");
    for (int64_t k = 1; k < n; ++k)
        if (keys[k] <= keys[k - 1]) throw Error(LC_ERR_ARG, "certificate keys must be sorted unique");
    n_ref = n;
    d_ref_keys.reserve(sizeof(uint64_t) * (n > 0 ? n : 1), s);
    d_ref_lk.reserve(sizeof(int64_t) * (n > 0 ? n : 1), s);
    d_ee.reserve(2 * sizeof(unsigned long long), s);
    if (n > 0) {
        LC_CUDA(cudaMemcpyAsync(d_ref_keys.ptr, keys, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, s));
        LC_CUDA(cudaMemcpyAsync(d_ref_lk.ptr, lk, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    }
    LC_CUDA(cudaStreamSynchronize(s));   // the caller's arrays may go after return
}

void Pipeline::prefill_partials_neg_zero(int64_t n) {
    d_partials.reserve(sizeof(double) * (size_t)(n > 0 ? n : 1), s);
    if (n == 0) return;
    fill_bits_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(reinterpret_cast<unsigned long long *>(d_partials.ptr),
                                                                n, 0x8000000000000000ull);
    LC_CHECK_LAUNCH();
}

void Pipeline::shard_bounds(int shards, int64_t *out) {
    if (!polylines_ready) throw Error(LC_ERR_STATE, "no work items built");
    if (shards < 1) throw Error(LC_ERR_ARG, "shards must be >= 1");
    d_bounds.reserve(sizeof(int64_t) * (shards + 1), s);
    launch_shard_bounds(d_pg.as<PairGeom>(), d_item_off.as<int64_t>(), P, nullptr, shards, d_bounds.as<int64_t>(), s,
                        items_seq);
    if (out) {
        LC_CUDA(cudaMemcpyAsync(out, d_bounds.ptr, sizeof(int64_t) * (shards + 1), cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaStreamSynchronize(s));
    }
}

void Pipeline::segment_pair_lambda(const double *quads, int64_t n, double *out) {
    if (n == 0) return;
    d_quads.reserve(sizeof(double) * 12 * (size_t)n, s);
    d_qout.reserve(sizeof(double) * (size_t)n, s);
    LC_CUDA(cudaMemcpyAsync(d_quads.ptr, quads, sizeof(double) * 12 * n, cudaMemcpyHostToDevice, s));
    launch_segment_pairs(d_quads.as<double>(), n, d_qout.as<double>(), s);
    LC_CUDA(cudaMemcpyAsync(out, d_qout.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
}

}  // namespace lc
