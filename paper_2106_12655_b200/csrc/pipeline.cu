// Pipeline stage orchestration on one device/stream (host side of the C-ABI).
#include <cstring>
#include <vector>

#include "pipeline.cuh"

namespace lc {

void Pipeline::init(cudaStream_t st) { s = st; }

void Pipeline::release() {
    DevBuf *bufs[] = {&d_aos, &d_in_off, &d_voff, &d_X, &d_Y, &d_Z, &d_exp, &d_pairs, &d_pg,
                      &d_item_off, &d_scan, &d_counter, &d_partials, &d_raw, &d_lk, &d_flags,
                      &d_quads, &d_qout};
    for (DevBuf *b : bufs) b->release(s);
    if (s) cudaStreamSynchronize(s);
    h_stage.release();
}

// Host AoS polylines (no closing vertex; loop v = rows [vert_off[v], vert_off[v+1]))
// -> device closed SoA with vertex 0 repeated at the end of every loop
// (direct.py:164-166 _closed), scaled by an exact power of two.
void Pipeline::upload_polylines(const double *verts, const int64_t *vert_off, int64_t nloops) {
    L = nloops;
    V = L > 0 ? vert_off[L] - vert_off[0] : 0;
    if (L > 0 && vert_off[0] != 0) throw Error(LC_ERR_ARG, "vert_off[0] must be 0");
    h_voff.resize((size_t)L + 1);
    for (int64_t v = 0; v <= L; ++v) h_voff[v] = (L > 0 ? vert_off[v] : 0) + v;
    Vc = V + L;
    d_aos.reserve(sizeof(double) * 3 * (size_t)(V > 0 ? V : 1), s);
    d_in_off.reserve(sizeof(int64_t) * (size_t)(L + 1), s);
    d_voff.reserve(sizeof(int64_t) * (size_t)(L + 1), s);
    d_X.reserve(sizeof(double) * (size_t)(Vc + 1), s);
    d_Y.reserve(sizeof(double) * (size_t)(Vc + 1), s);
    d_Z.reserve(sizeof(double) * (size_t)(Vc + 1), s);
    d_exp.reserve(sizeof(int), s);
    if (V > 0) LC_CUDA(cudaMemcpyAsync(d_aos.ptr, verts, sizeof(double) * 3 * V, cudaMemcpyHostToDevice, s));
    if (L > 0) {
        LC_CUDA(cudaMemcpyAsync(d_in_off.ptr, vert_off, sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice, s));
        LC_CUDA(cudaMemcpyAsync(d_voff.ptr, h_voff.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice, s));
    }
    LC_CUDA(cudaMemsetAsync(d_exp.ptr, 0, sizeof(int), s));
    launch_max_exponent(d_aos.as<double>(), 3 * V, d_exp.as<int>(), s);
    launch_pack_closed_soa(d_aos.as<double>(), d_in_off.as<int64_t>(), d_voff.as<int64_t>(), L, Vc,
                           d_exp.as<int>(), d_X.as<double>(), d_Y.as<double>(), d_Z.as<double>(), s);
    // the caller's host buffers may be released after return
    LC_CUDA(cudaStreamSynchronize(s));
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

void Pipeline::build_gauss_items() {
    d_pg.reserve(sizeof(PairGeom) * (size_t)(P > 0 ? P : 1), s);
    d_item_off.reserve(sizeof(int64_t) * (size_t)(P + 1), s);
    const size_t scan_bytes = build_items_scan_bytes(P > 0 ? P : 1);
    d_scan.reserve(scan_bytes, s);
    d_counter.reserve(sizeof(unsigned long long), s);
    n_items = build_items(d_pairs.as<int32_t>(), P, d_voff.as<int64_t>(), d_pg.as<PairGeom>(),
                          d_item_off.as<int64_t>(), d_scan.ptr, d_scan.bytes, s);
    d_partials.reserve(sizeof(double) * (size_t)(n_items > 0 ? n_items : 1), s);
    d_raw.reserve(sizeof(double) * (size_t)(P > 0 ? P : 1), s);
    d_lk.reserve(sizeof(int64_t) * (size_t)(P > 0 ? P : 1), s);
    d_flags.reserve((size_t)(P > 0 ? P : 1), s);
}

void Pipeline::run_gauss(int mode, int64_t item_begin, int64_t item_end, double *partials_ext,
                         cudaEvent_t ev0, cudaEvent_t ev1) {
    if (mode < GAUSS_PHASE || mode > GAUSS_REF) throw Error(LC_ERR_ARG, "unknown Gauss-sum mode");
    double *out = partials_ext ? partials_ext : d_partials.as<double>();
    if (ev0) LC_CUDA(cudaEventRecord(ev0, s));
    launch_gauss_items(mode, d_X.as<double>(), d_Y.as<double>(), d_Z.as<double>(), d_pg.as<PairGeom>(),
                       d_item_off.as<int64_t>(), P, item_begin, item_end,
                       d_counter.as<unsigned long long>(), out, s);
    if (ev1) LC_CUDA(cudaEventRecord(ev1, s));
}

void Pipeline::reduce_pairs(const double *partials_ext) {
    const double *in = partials_ext ? partials_ext : d_partials.as<double>();
    launch_reduce_pairs(in, d_item_off.as<int64_t>(), P, d_raw.as<double>(), d_lk.as<int64_t>(),
                        d_flags.as<uint8_t>(), s);
}

void Pipeline::download_results(double *raw, int64_t *lk, uint8_t *flags) {
    if (P > 0) {
        if (raw) LC_CUDA(cudaMemcpyAsync(raw, d_raw.ptr, sizeof(double) * P, cudaMemcpyDeviceToHost, s));
        if (lk) LC_CUDA(cudaMemcpyAsync(lk, d_lk.ptr, sizeof(int64_t) * P, cudaMemcpyDeviceToHost, s));
        if (flags) LC_CUDA(cudaMemcpyAsync(flags, d_flags.ptr, (size_t)P, cudaMemcpyDeviceToHost, s));
    }
    LC_CUDA(cudaStreamSynchronize(s));
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
