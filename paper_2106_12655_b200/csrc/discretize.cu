// Device discretization: refine paired loops until the tight boxes of their
// subsegments are pairwise disjoint across every PLS pair, then emit chords.
//
// Reference: linkcert/discretize.py:112-191 with _LoopState (:52-105).  The
// per-pass state is a loop-major SoA list of active subsegments (segment id,
// t_lo, t_hi) whose within-loop order reproduces the reference's list order
// exactly ([left halves..., right halves...] after every split, :91-98), so
// the first-bad-child error report (:170-174) names the same loops.
//
// Pass structure (one host sync per pass):
//   boxes (computed when the list was formed)
//   -> per-loop sorted lower bounds on 3 axes (CUB segmented sort)
//   -> per pair, per subsegment of either loop: binary search + sweep of the
//      other loop's sorted list on the pair's axis, closed 3-axis test;
//      hits set mark[] and the first marking pair via atomicMin (pairs are
//      processed in PairList order in the reference, so "first partner" is
//      the smallest pair index that hits the subsegment, :77-80,151-159)
//   -> scan of marks: unmarked -> done list, marked -> two children
//   -> children boxes, CurvesIntersect / max_subsegments checks per loop.
// Final: stable sort of done chords by (segment, t_lo) (the lexsort of
// :104), start points via eval_cubics (:89), validation as PolylineLoop
// (geometry.py:333-340).
#include <climits>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "discretize.cuh"
#include "geom.cuh"

namespace lc {
namespace {

constexpr double kMachineEps = 2.220446049250313e-16;
// "no index yet" sentinel of atomicMin slots initialized by cudaMemset(0x7f)
constexpr int32_t kNoIndex = 0x7f7f7f7f;

struct PassCounters {
    int64_t total_marked;
    int err_loop;
    int pad;
};

__global__ void mark_paired_kernel(const int32_t *__restrict__ pairs, int64_t P, uint8_t *__restrict__ paired) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    paired[pairs[2 * p]] = 1;
    paired[pairs[2 * p + 1]] = 1;
}

__global__ void init_counts_kernel(const int64_t *__restrict__ loff, const uint8_t *__restrict__ paired, int64_t L,
                                   int64_t *__restrict__ cnt) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l < L) cnt[l] = paired[l] ? loff[l + 1] - loff[l] : 0;
    else if (l == L) cnt[L] = 0;
}

__global__ void init_active_kernel(int64_t M, const int32_t *__restrict__ seg_loop, const int64_t *__restrict__ loff,
                                   const uint8_t *__restrict__ paired, const double *__restrict__ t,
                                   const double *__restrict__ seg_box, const int64_t *__restrict__ act_off,
                                   int64_t stride, int32_t *__restrict__ act_seg, int32_t *__restrict__ act_loop,
                                   double *__restrict__ tlo, double *__restrict__ thi, double *__restrict__ box) {
    const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= M) return;
    const int l = seg_loop[m];
    if (!paired[l]) return;
    const int64_t e = act_off[l] + (m - loff[l]);
    act_seg[e] = (int32_t)m;
    act_loop[e] = l;
    tlo[e] = t[2 * m];
    thi[e] = t[2 * m + 1];
#pragma unroll
    for (int d = 0; d < 6; ++d) box[d * stride + e] = seg_box[d * M + m];
}

// Sweep axis per pair: the axis along which the two loop boxes' intersection is longest.
__global__ void pair_axis_kernel(const int32_t *__restrict__ pairs, int64_t P, const double *__restrict__ lbox,
                                 int64_t L, int8_t *__restrict__ axis) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int i = pairs[2 * p], j = pairs[2 * p + 1];
    int a = 0;
    double best = -CUDART_INF;
    for (int d = 0; d < 3; ++d) {
        const double e = fmin(lbox[(3 + d) * L + i], lbox[(3 + d) * L + j]) - fmax(lbox[d * L + i], lbox[d * L + j]);
        if (e > best) { best = e; a = d; }
    }
    axis[p] = (int8_t)a;
}

__global__ void copy_lo_kernel(const double *__restrict__ box, int64_t stride, int64_t n, int axis,
                               double *__restrict__ key, int32_t *__restrict__ iota) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n) return;
    key[e] = box[axis * stride + e];
    if (iota) iota[e] = (int32_t)e;
}

__global__ void sweep_counts_kernel(const int32_t *__restrict__ pairs, int64_t P, const int64_t *__restrict__ act_off,
                                    int64_t *__restrict__ cnt) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < P) {
        const int i = pairs[2 * p], j = pairs[2 * p + 1];
        cnt[p] = (act_off[i + 1] - act_off[i]) + (act_off[j + 1] - act_off[j]);
    } else if (p == P) {
        cnt[P] = 0;
    }
}

__device__ __forceinline__ int64_t upper_index(const int64_t *__restrict__ off, int64_t n, int64_t k) {
    int64_t lo = 0, hi = n;   // largest idx in [0, n) with off[idx] <= k  (off[0] == 0)
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (off[mid] <= k) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void sweep_kernel(const int32_t *__restrict__ pairs, int64_t P, const int8_t *__restrict__ axis,
                             const int64_t *__restrict__ sweep_off, const int64_t *__restrict__ act_off,
                             const double *__restrict__ box, int64_t stride, const double *__restrict__ k0,
                             const double *__restrict__ k1, const double *__restrict__ k2,
                             const int32_t *__restrict__ p0, const int32_t *__restrict__ p1,
                             const int32_t *__restrict__ p2, uint8_t *__restrict__ mark,
                             int32_t *__restrict__ first_pair) {
    const int64_t total = sweep_off[P];
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = upper_index(sweep_off, P, k);
        const int i = pairs[2 * p], j = pairs[2 * p + 1];
        const int64_t ni = act_off[i + 1] - act_off[i];
        const int64_t local = k - sweep_off[p];
        const int A = local < ni ? i : j, B = local < ni ? j : i;
        const int64_t e = act_off[A] + (local < ni ? local : local - ni);
        const int a = axis[p];
        const double *keys = a == 0 ? k0 : (a == 1 ? k1 : k2);
        const int32_t *perm = a == 0 ? p0 : (a == 1 ? p1 : p2);
        double el[3], eh[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            el[d] = box[d * stride + e];
            eh[d] = box[(3 + d) * stride + e];
        }
        const double lo_a = el[a], hi_a = eh[a];
        int64_t lo = act_off[B], hi = act_off[B + 1];
        const int64_t end = hi;
        while (lo < hi) {   // first q with keys[q] >= lo_a
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < lo_a) lo = mid + 1; else hi = mid;
        }
        bool hit_any = false;
        for (int64_t q = lo; q < end && keys[q] <= hi_a; ++q) {
            const int64_t tt = perm[q];
            bool ov = true;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                if (el[d] > box[(3 + d) * stride + tt] || box[d * stride + tt] > eh[d]) ov = false;
            }
            if (ov) {
                hit_any = true;
                mark[tt] = 1;
                atomicMin(first_pair + tt, (int32_t)p);
            }
        }
        if (hit_any) {
            mark[e] = 1;
            atomicMin(first_pair + e, (int32_t)p);
        }
    }
}

__global__ void mark_to_i64_kernel(const uint8_t *__restrict__ mark, int64_t n, int64_t *__restrict__ out) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < n) out[e] = mark[e];
    else if (e == n) out[n] = 0;
}

__global__ void finish_kernel(int64_t n_act, const int32_t *__restrict__ pairs, const uint8_t *__restrict__ mark,
                              const int64_t *__restrict__ mscan, const int32_t *__restrict__ first_pair,
                              const int64_t *__restrict__ act_off, const int32_t *__restrict__ act_seg,
                              const int32_t *__restrict__ act_loop, const double *__restrict__ act_tlo,
                              const double *__restrict__ act_thi, int32_t *__restrict__ nxt_seg,
                              int32_t *__restrict__ nxt_loop, double *__restrict__ nxt_tlo,
                              double *__restrict__ nxt_thi, int32_t *__restrict__ nxt_partner, int64_t n_done,
                              int32_t *__restrict__ done_seg, double *__restrict__ done_tlo) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_act) return;
    const int64_t r = mscan[e];
    const int l = act_loop[e];
    const int32_t seg = act_seg[e];
    const double tlo = act_tlo[e], thi = act_thi[e];
    if (mark[e]) {
        const int64_t base = mscan[act_off[l]];
        const int64_t cnt = mscan[act_off[l + 1]] - base;
        const int64_t k = r - base, no = 2 * base;
        const double tm = __dmul_rn(0.5, __dadd_rn(tlo, thi));   // 0.5 * (tlo + thi)  (:95)
        const int32_t pp = first_pair[e];
        const int32_t partner = pairs[2 * pp] == l ? pairs[2 * pp + 1] : pairs[2 * pp];
        nxt_seg[no + k] = seg;       nxt_loop[no + k] = l;
        nxt_tlo[no + k] = tlo;       nxt_thi[no + k] = tm;       nxt_partner[no + k] = partner;
        nxt_seg[no + cnt + k] = seg; nxt_loop[no + cnt + k] = l;
        nxt_tlo[no + cnt + k] = tm;  nxt_thi[no + cnt + k] = thi; nxt_partner[no + cnt + k] = partner;
    } else {
        const int64_t d = n_done + (e - r);
        done_seg[d] = seg;
        done_tlo[d] = tlo;
    }
}

__global__ void next_off_kernel(const int64_t *__restrict__ act_off, const int64_t *__restrict__ mscan, int64_t L,
                                int64_t *__restrict__ nxt_off) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l <= L) nxt_off[l] = 2 * mscan[act_off[l]];
}

__global__ void child_boxes_kernel(int64_t n, const double *__restrict__ coeffs, const int32_t *__restrict__ seg,
                                   const int32_t *__restrict__ loop, const double *__restrict__ tlo,
                                   const double *__restrict__ thi, const int64_t *__restrict__ off, int64_t stride,
                                   double min_diam, double *__restrict__ box, int32_t *__restrict__ bad_first) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n) return;
    double bl[3], bh[3];
    tight_box(coeffs + 12 * (int64_t)seg[e], tlo[e], thi[e], bl, bh);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        box[d * stride + e] = bl[d];
        box[(3 + d) * stride + e] = bh[d];
    }
    if (diag_norm(bl, bh) < min_diam) {
        const int l = loop[e];
        atomicMin(bad_first + l, (int32_t)(e - off[l]));
    }
}

__global__ void pass_errors_kernel(const int64_t *__restrict__ nxt_off, const int32_t *__restrict__ bad_first,
                                   int64_t L, int64_t max_sub, const int64_t *__restrict__ mscan, int64_t n_act,
                                   PassCounters *__restrict__ ctr) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l == 0) ctr->total_marked = mscan[n_act];
    if (l >= L) return;
    const int64_t c = nxt_off[l + 1] - nxt_off[l];
    if (c > 0 && (bad_first[l] != kNoIndex || c > max_sub)) atomicMin(&ctr->err_loop, (int)l);
}

__global__ void gather_seg_kernel(const int32_t *__restrict__ idx, int64_t n, const int32_t *__restrict__ seg,
                                  int32_t *__restrict__ out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) out[k] = seg[idx[k]];
}

__global__ void done_hist_kernel(const int32_t *__restrict__ seg, int64_t n, const int32_t *__restrict__ seg_loop,
                                 unsigned long long *__restrict__ cnt) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) atomicAdd(cnt + seg_loop[seg[k]], 1ULL);
}

__global__ void out_counts_kernel(const unsigned long long *__restrict__ dcnt, const uint8_t *__restrict__ paired,
                                  const int64_t *__restrict__ loff, int64_t L, int64_t *__restrict__ ocnt,
                                  int64_t *__restrict__ dcnt64) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l < L) {
        ocnt[l] = paired[l] ? (int64_t)dcnt[l] : loff[l + 1] - loff[l];
        dcnt64[l] = (int64_t)dcnt[l];
    } else if (l == L) {
        ocnt[L] = 0;
        dcnt64[L] = 0;
    }
}

// Start points of the given (segment, t) list into AoS at out_off[loop] + local.
__global__ void write_done_kernel(int64_t n, const int32_t *__restrict__ seg, const double *__restrict__ tlo,
                                  const int32_t *__restrict__ idx, const int32_t *__restrict__ seg_loop,
                                  const double *__restrict__ coeffs, const int64_t *__restrict__ out_off,
                                  const int64_t *__restrict__ done_off, double *__restrict__ verts) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int32_t s = seg[k];
    const double t = idx ? tlo[idx[k]] : tlo[k];
    const int l = seg_loop[s];
    const int64_t pos = out_off[l] + (k - done_off[l]);
    double p[3];
    eval_point(coeffs + 12 * (int64_t)s, t, p);
    verts[3 * pos] = p[0];
    verts[3 * pos + 1] = p[1];
    verts[3 * pos + 2] = p[2];
}

// Unpaired loops: chords through the segment start points (_chord_loop, :108-109).
__global__ void write_unpaired_kernel(int64_t M, const int32_t *__restrict__ seg_loop, const uint8_t *__restrict__ paired,
                                      const int64_t *__restrict__ loff, const double *__restrict__ coeffs,
                                      const double *__restrict__ t, const int64_t *__restrict__ out_off,
                                      double *__restrict__ verts) {
    const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= M) return;
    const int l = seg_loop[m];
    if (paired && paired[l]) return;
    const int64_t pos = (out_off ? out_off[l] : loff[l]) + (m - loff[l]);
    double p[3];
    eval_point(coeffs + 12 * m, t[2 * m], p);
    verts[3 * pos] = p[0];
    verts[3 * pos + 1] = p[1];
    verts[3 * pos + 2] = p[2];
}

// PolylineLoop validation (geometry.py:333-340) of loops with want(l):
// flags bit0 non-finite vertex, bit1 segment length <= eps*scale.
__global__ void validate_vertices_kernel(const double *__restrict__ v, const int64_t *__restrict__ off, int64_t L,
                                         int64_t n, const uint8_t *__restrict__ paired, int want_paired,
                                         double thr, unsigned *__restrict__ flags) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t l = upper_index(off, L, k);
    if (paired && (int)paired[l] != want_paired) return;
    const int64_t b = off[l], e = off[l + 1];
    const int64_t nx = (k + 1 < e) ? k + 1 : b;
    const double x = v[3 * k], y = v[3 * k + 1], z = v[3 * k + 2];
    unsigned f = 0;
    if (!(isfinite(x) && isfinite(y) && isfinite(z))) f |= 1;
    const double dx = __dsub_rn(v[3 * nx], x), dy = __dsub_rn(v[3 * nx + 1], y), dz = __dsub_rn(v[3 * nx + 2], z);
    const double len = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    if (len <= thr) f |= 2;
    if (f) atomicOr(flags + l, f);
}

__global__ void validate_loops_kernel(const int64_t *__restrict__ off, int64_t L, const uint8_t *__restrict__ paired,
                                      int want_paired, const unsigned *__restrict__ flags, int *__restrict__ err) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= L) return;
    if (paired && (int)paired[l] != want_paired) return;
    const int64_t n = off[l + 1] - off[l];
    int kind = PL_OK;
    if (n < 3) kind = PL_TOO_FEW;
    else if (flags[l] & 1) kind = PL_NONFINITE;
    else if (flags[l] & 2) kind = PL_ZERO_SEGMENT;
    if (kind) atomicMin(err, (int)(l * 4 + kind));
}

__global__ void zero_length_kernel(const double *__restrict__ box, int64_t M, const int32_t *__restrict__ seg_loop,
                                   double min_diam, int *__restrict__ zl) {
    const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= M) return;
    double bl[3], bh[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        bl[d] = box[d * M + m];
        bh[d] = box[(3 + d) * M + m];
    }
    if (diag_norm(bl, bh) < min_diam) atomicMin(zl, (int)seg_loop[m]);
}

inline unsigned grid_for(int64_t n, int threads = 256) { return (unsigned)(n > 0 ? ceil_div(n, threads) : 1); }

template <class T> T d2h(const void *p, cudaStream_t s) {
    T v;
    LC_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
    return v;
}

// Validate loops selected by paired==want; returns loop*4+kind or INT_MAX.
int validate(const double *verts, const int64_t *off, int64_t L, int64_t n, const uint8_t *paired, int want,
             double thr, DiscScratch &sc, cudaStream_t s) {
    sc.val_flags.reserve(sizeof(unsigned) * (L > 0 ? L : 1), s);
    sc.loop_err.reserve(sizeof(int), s);
    LC_CUDA(cudaMemsetAsync(sc.val_flags.ptr, 0, sizeof(unsigned) * L, s));
    const int init = INT_MAX;
    LC_CUDA(cudaMemcpyAsync(sc.loop_err.ptr, &init, sizeof(int), cudaMemcpyHostToDevice, s));
    if (n > 0) {
        validate_vertices_kernel<<<grid_for(n), 256, 0, s>>>(verts, off, L, n, paired, want, thr,
                                                             sc.val_flags.as<unsigned>());
        LC_CHECK_LAUNCH();
    }
    validate_loops_kernel<<<grid_for(L), 256, 0, s>>>(off, L, paired, want, sc.val_flags.as<unsigned>(),
                                                      sc.loop_err.as<int>());
    LC_CHECK_LAUNCH();
    return d2h<int>(sc.loop_err.ptr, s);
}

void scan_i64(const int64_t *in, int64_t *out, int64_t n, DiscScratch &sc, cudaStream_t s) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n);
    sc.cub_tmp.reserve(bytes, s);
    bytes = sc.cub_tmp.bytes;
    LC_CUB(cub::DeviceScan::ExclusiveSum(sc.cub_tmp.ptr, bytes, in, out, (int)n, s));
}

}  // namespace

bool run_discretize(const DiscInput &in, const DiscParams &prm, DiscScratch &sc, DiscOutput &out,
                    DiscError *err, cudaStream_t s) {
    const int64_t L = in.L, M = in.M, P = in.P;
    const double min_diam = prm.epsilon * prm.xi;      // discretize.py:122
    const double poly_thr = kMachineEps * prm.xi;       // PolylineLoop(xi_hint=xi), geometry.py:338-340
    out.passes = 0;
    out.splits = 0;

    // (1) ZeroLengthInput over all loops in order (:124-129).
    sc.loop_err.reserve(sizeof(int), s);
    {
        const int init = INT_MAX;
        LC_CUDA(cudaMemcpyAsync(sc.loop_err.ptr, &init, sizeof(int), cudaMemcpyHostToDevice, s));
        if (M > 0)
            zero_length_kernel<<<grid_for(M), 256, 0, s>>>(in.seg_box, M, in.seg_loop, min_diam, sc.loop_err.as<int>());
        LC_CHECK_LAUNCH();
    }
    const int zl = d2h<int>(sc.loop_err.ptr, s);
    if (zl != INT_MAX) {
        err->kind = DISC_ZERO_LENGTH;
        err->loops = {zl};
        return false;
    }

    // (2) paired loops; unpaired loops become control chords, validated now (:131-142).
    sc.paired.reserve(L > 0 ? L : 1, s);
    LC_CUDA(cudaMemsetAsync(sc.paired.ptr, 0, L, s));
    if (P > 0) mark_paired_kernel<<<grid_for(P), 256, 0, s>>>(in.pairs, P, sc.paired.as<uint8_t>());
    LC_CHECK_LAUNCH();
    // unpaired start points into a temporary AoS in original segment layout (reuse out.verts)
    out.verts.reserve(sizeof(double) * 3 * (M > 0 ? M : 1), s);
    if (M > 0)
        write_unpaired_kernel<<<grid_for(M), 256, 0, s>>>(M, in.seg_loop, sc.paired.as<uint8_t>(), in.loff, in.coeffs,
                                                          in.t, nullptr, out.verts.as<double>());
    LC_CHECK_LAUNCH();
    {
        const int ve = validate(out.verts.as<double>(), in.loff, L, M, sc.paired.as<uint8_t>(), 0, poly_thr, sc, s);
        if (ve != INT_MAX) {
            err->kind = DISC_INVALID_POLYLINE;
            err->detail = ve & 3;
            err->loops = {ve >> 2};
            return false;
        }
    }

    // (3) initial active list: all segments of paired loops, loop-major.
    sc.act_off.reserve(sizeof(int64_t) * (L + 1), s);
    sc.nxt_off.reserve(sizeof(int64_t) * (L + 1), s);
    sc.counters.reserve(sizeof(int64_t) * (L + 2), s);   // temp counts
    init_counts_kernel<<<grid_for(L + 1), 256, 0, s>>>(in.loff, sc.paired.as<uint8_t>(), L, sc.counters.as<int64_t>());
    LC_CHECK_LAUNCH();
    scan_i64(sc.counters.as<int64_t>(), sc.act_off.as<int64_t>(), L + 1, sc, s);
    int64_t n_act = d2h<int64_t>(sc.act_off.as<int64_t>() + L, s);
    int64_t stride = n_act > 0 ? n_act : 1;
    auto reserve_list = [&](DevBuf &seg, DevBuf &loop, DevBuf &tlo, DevBuf &thi, DevBuf &box, int64_t cap) {
        seg.reserve(sizeof(int32_t) * cap, s);
        loop.reserve(sizeof(int32_t) * cap, s);
        tlo.reserve(sizeof(double) * cap, s);
        thi.reserve(sizeof(double) * cap, s);
        box.reserve(sizeof(double) * 6 * cap, s);
    };
    reserve_list(sc.act_seg, sc.act_loop, sc.act_tlo, sc.act_thi, sc.box, stride);
    if (M > 0)
        init_active_kernel<<<grid_for(M), 256, 0, s>>>(M, in.seg_loop, in.loff, sc.paired.as<uint8_t>(), in.t, in.seg_box,
                                                       sc.act_off.as<int64_t>(), stride, sc.act_seg.as<int32_t>(),
                                                       sc.act_loop.as<int32_t>(), sc.act_tlo.as<double>(),
                                                       sc.act_thi.as<double>(), sc.box.as<double>());
    LC_CHECK_LAUNCH();
    sc.pair_axis.reserve(P > 0 ? P : 1, s);
    if (P > 0) pair_axis_kernel<<<grid_for(P), 256, 0, s>>>(in.pairs, P, in.loop_box, L, sc.pair_axis.as<int8_t>());
    LC_CHECK_LAUNCH();
    sc.sweep_off.reserve(sizeof(int64_t) * (P + 1), s);
    sc.bad_first.reserve(sizeof(int32_t) * (L > 0 ? L : 1), s);

    int64_t n_done = 0;
    const int nsm = 148;
    int pass = 0;
    for (; pass < prm.max_passes; ++pass) {
        if (n_act == 0) break;
        out.passes = pass + 1;
        // per-loop sorted lower bounds on each axis
        sc.iota.reserve(sizeof(int32_t) * n_act, s);
        for (int a = 0; a < 3; ++a) {
            sc.skey[a].reserve(sizeof(double) * n_act, s);
            sc.sperm[a].reserve(sizeof(int32_t) * n_act, s);
        }
        DevBuf &tmpkey = sc.done_tlo2;   // scratch: unsorted keys
        tmpkey.reserve(sizeof(double) * n_act, s);
        for (int a = 0; a < 3; ++a) {
            copy_lo_kernel<<<grid_for(n_act), 256, 0, s>>>(sc.box.as<double>(), stride, n_act, a, tmpkey.as<double>(),
                                                          a == 0 ? sc.iota.as<int32_t>() : nullptr);
            LC_CHECK_LAUNCH();
            size_t bytes = 0;
            cub::DeviceSegmentedSort::SortPairs(nullptr, bytes, tmpkey.as<double>(), sc.skey[a].as<double>(),
                                                sc.iota.as<int32_t>(), sc.sperm[a].as<int32_t>(), (int)n_act, (int)L,
                                                sc.act_off.as<int64_t>(), sc.act_off.as<int64_t>() + 1);
            sc.cub_tmp.reserve(bytes, s);
            bytes = sc.cub_tmp.bytes;
            LC_CUB(cub::DeviceSegmentedSort::SortPairs(sc.cub_tmp.ptr, bytes, tmpkey.as<double>(),
                                                        sc.skey[a].as<double>(), sc.iota.as<int32_t>(),
                                                        sc.sperm[a].as<int32_t>(), (int)n_act, (int)L,
                                                        sc.act_off.as<int64_t>(), sc.act_off.as<int64_t>() + 1, s));
        }
        // sweep over pairs
        sc.mark.reserve(n_act, s);
        sc.first_pair.reserve(sizeof(int32_t) * n_act, s);
        LC_CUDA(cudaMemsetAsync(sc.mark.ptr, 0, n_act, s));
        LC_CUDA(cudaMemsetAsync(sc.first_pair.ptr, 0x7f, sizeof(int32_t) * n_act, s));
        if (P > 0) {
            sc.counters.reserve(sizeof(int64_t) * (P + 1), s);
            sweep_counts_kernel<<<grid_for(P + 1), 256, 0, s>>>(in.pairs, P, sc.act_off.as<int64_t>(),
                                                               sc.counters.as<int64_t>());
            LC_CHECK_LAUNCH();
            scan_i64(sc.counters.as<int64_t>(), sc.sweep_off.as<int64_t>(), P + 1, sc, s);
            sweep_kernel<<<nsm * 8, 256, 0, s>>>(in.pairs, P, sc.pair_axis.as<int8_t>(), sc.sweep_off.as<int64_t>(),
                                                 sc.act_off.as<int64_t>(), sc.box.as<double>(), stride,
                                                 sc.skey[0].as<double>(), sc.skey[1].as<double>(),
                                                 sc.skey[2].as<double>(), sc.sperm[0].as<int32_t>(),
                                                 sc.sperm[1].as<int32_t>(), sc.sperm[2].as<int32_t>(),
                                                 sc.mark.as<uint8_t>(), sc.first_pair.as<int32_t>());
            LC_CHECK_LAUNCH();
        }
        // ranks of marked entries
        sc.mark_scan.reserve(sizeof(int64_t) * (n_act + 1), s);
        sc.counters.reserve(sizeof(int64_t) * (n_act + 1), s);
        mark_to_i64_kernel<<<grid_for(n_act + 1), 256, 0, s>>>(sc.mark.as<uint8_t>(), n_act, sc.counters.as<int64_t>());
        LC_CHECK_LAUNCH();
        scan_i64(sc.counters.as<int64_t>(), sc.mark_scan.as<int64_t>(), n_act + 1, sc, s);
        // capacity: children <= 2 n_act, done <= n_done + n_act
        const int64_t nstride = 2 * n_act;
        reserve_list(sc.nxt_seg, sc.nxt_loop, sc.nxt_tlo, sc.nxt_thi, sc.nxt_box, nstride);
        sc.nxt_partner.reserve(sizeof(int32_t) * nstride, s);
        if (n_done + n_act > sc.cap_done) {
            // grow preserving contents
            const int64_t cap = (n_done + n_act) * 2;
            DevBuf ns, nt;
            ns.reserve(sizeof(int32_t) * cap, s);
            nt.reserve(sizeof(double) * cap, s);
            if (n_done) {
                LC_CUDA(cudaMemcpyAsync(ns.ptr, sc.done_seg.ptr, sizeof(int32_t) * n_done, cudaMemcpyDeviceToDevice, s));
                LC_CUDA(cudaMemcpyAsync(nt.ptr, sc.done_tlo.ptr, sizeof(double) * n_done, cudaMemcpyDeviceToDevice, s));
            }
            sc.done_seg.release(s);
            sc.done_tlo.release(s);
            sc.done_seg = ns;
            sc.done_tlo = nt;
            sc.cap_done = cap;
        }
        finish_kernel<<<grid_for(n_act), 256, 0, s>>>(
            n_act, in.pairs, sc.mark.as<uint8_t>(), sc.mark_scan.as<int64_t>(), sc.first_pair.as<int32_t>(),
            sc.act_off.as<int64_t>(), sc.act_seg.as<int32_t>(), sc.act_loop.as<int32_t>(), sc.act_tlo.as<double>(),
            sc.act_thi.as<double>(), sc.nxt_seg.as<int32_t>(), sc.nxt_loop.as<int32_t>(), sc.nxt_tlo.as<double>(),
            sc.nxt_thi.as<double>(), sc.nxt_partner.as<int32_t>(), n_done, sc.done_seg.as<int32_t>(),
            sc.done_tlo.as<double>());
        LC_CHECK_LAUNCH();
        next_off_kernel<<<grid_for(L + 1), 256, 0, s>>>(sc.act_off.as<int64_t>(), sc.mark_scan.as<int64_t>(), L,
                                                        sc.nxt_off.as<int64_t>());
        LC_CHECK_LAUNCH();
        // children boxes + error checks (:166-180); n_new unknown on host: bound by 2 n_act via mark_scan
        LC_CUDA(cudaMemsetAsync(sc.bad_first.ptr, 0x7f, sizeof(int32_t) * L, s));
        PassCounters init{0, INT_MAX, 0};
        DevBuf &ctr = sc.ucnt;
        ctr.reserve(sizeof(PassCounters), s);
        LC_CUDA(cudaMemcpyAsync(ctr.ptr, &init, sizeof init, cudaMemcpyHostToDevice, s));
        // total marked needed for the child grid: read it (sync 1)
        const int64_t marked = d2h<int64_t>(sc.mark_scan.as<int64_t>() + n_act, s);
        const int64_t n_new = 2 * marked;
        if (n_new > 0)
            child_boxes_kernel<<<grid_for(n_new), 256, 0, s>>>(n_new, in.coeffs, sc.nxt_seg.as<int32_t>(),
                                                               sc.nxt_loop.as<int32_t>(), sc.nxt_tlo.as<double>(),
                                                               sc.nxt_thi.as<double>(), sc.nxt_off.as<int64_t>(),
                                                               nstride, min_diam, sc.nxt_box.as<double>(),
                                                               sc.bad_first.as<int32_t>());
        LC_CHECK_LAUNCH();
        pass_errors_kernel<<<grid_for(L > 0 ? L : 1), 256, 0, s>>>(sc.nxt_off.as<int64_t>(), sc.bad_first.as<int32_t>(), L,
                                                                   prm.max_subsegments, sc.mark_scan.as<int64_t>(),
                                                                   n_act, ctr.as<PassCounters>());
        LC_CHECK_LAUNCH();
        const PassCounters pc = d2h<PassCounters>(ctr.ptr, s);
        n_done += n_act - marked;
        out.splits += marked;
        if (pc.err_loop != INT_MAX) {
            const int l = pc.err_loop;
            const int32_t bf = d2h<int32_t>(sc.bad_first.as<int32_t>() + l, s);
            if (bf != kNoIndex) {
                const int64_t o = d2h<int64_t>(sc.nxt_off.as<int64_t>() + l, s);
                const int32_t partner = d2h<int32_t>(sc.nxt_partner.as<int32_t>() + o + bf, s);
                err->kind = DISC_CURVES_INTERSECT;
                err->loops = {l < partner ? l : partner, l < partner ? partner : l};
            } else {
                err->kind = DISC_SUBSEG_BUDGET;
                err->loops = {l};
            }
            return false;
        }
        // swap lists
        std::swap(sc.act_seg, sc.nxt_seg);
        std::swap(sc.act_loop, sc.nxt_loop);
        std::swap(sc.act_tlo, sc.nxt_tlo);
        std::swap(sc.act_thi, sc.nxt_thi);
        std::swap(sc.box, sc.nxt_box);
        std::swap(sc.act_off, sc.nxt_off);
        stride = nstride > 0 ? nstride : 1;
        n_act = n_new;
    }
    if (n_act > 0) {   // for-else of :144,181-187
        std::vector<int64_t> off(L + 1);
        LC_CUDA(cudaMemcpyAsync(off.data(), sc.act_off.ptr, sizeof(int64_t) * (L + 1), cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaStreamSynchronize(s));
        err->kind = DISC_PASS_BUDGET;
        err->loops.clear();
        for (int64_t l = 0; l < L; ++l)
            if (off[l + 1] > off[l]) err->loops.push_back(l);
        return false;
    }

    // (4) chords: done entries sorted by (seg, tlo) (:100-105)
    const int32_t *seg_sorted = sc.done_seg.as<int32_t>();
    const int32_t *t_idx = nullptr;
    if (out.splits > 0 && n_done > 0) {
        sc.sort_idx.reserve(sizeof(int32_t) * n_done, s);
        sc.sort_idx2.reserve(sizeof(int32_t) * n_done, s);
        sc.done_tlo2.reserve(sizeof(double) * n_done, s);
        sc.done_seg2.reserve(sizeof(int32_t) * n_done, s);
        sc.iota.reserve(sizeof(int32_t) * n_done, s);
        copy_lo_kernel<<<grid_for(n_done), 256, 0, s>>>(sc.done_tlo.as<double>(), 0, n_done, 0, sc.done_tlo2.as<double>(),
                                                        sc.iota.as<int32_t>());
        LC_CHECK_LAUNCH();
        size_t b1 = 0, b2 = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, b1, (double *)nullptr, (double *)nullptr, (int32_t *)nullptr,
                                        (int32_t *)nullptr, (int)n_done);
        cub::DeviceRadixSort::SortPairs(nullptr, b2, (int32_t *)nullptr, (int32_t *)nullptr, (int32_t *)nullptr,
                                        (int32_t *)nullptr, (int)n_done);
        sc.cub_tmp.reserve(b1 > b2 ? b1 : b2, s);
        size_t bytes = sc.cub_tmp.bytes;
        // by tlo (scratch key copy in done_tlo2 -> sorted into skey[0])
        sc.skey[0].reserve(sizeof(double) * n_done, s);
        LC_CUB(cub::DeviceRadixSort::SortPairs(sc.cub_tmp.ptr, bytes, sc.done_tlo2.as<double>(), sc.skey[0].as<double>(),
                                                sc.iota.as<int32_t>(), sc.sort_idx.as<int32_t>(), (int)n_done, 0, 64, s));
        gather_seg_kernel<<<grid_for(n_done), 256, 0, s>>>(sc.sort_idx.as<int32_t>(), n_done, sc.done_seg.as<int32_t>(),
                                                          sc.done_seg2.as<int32_t>());
        LC_CHECK_LAUNCH();
        sc.sperm[0].reserve(sizeof(int32_t) * n_done, s);
        bytes = sc.cub_tmp.bytes;
        LC_CUB(cub::DeviceRadixSort::SortPairs(sc.cub_tmp.ptr, bytes, sc.done_seg2.as<int32_t>(),
                                                sc.sperm[0].as<int32_t>(), sc.sort_idx.as<int32_t>(),
                                                sc.sort_idx2.as<int32_t>(), (int)n_done, 0, 32, s));
        seg_sorted = sc.sperm[0].as<int32_t>();
        t_idx = sc.sort_idx2.as<int32_t>();
    }
    // per-loop output counts and offsets
    sc.done_cnt.reserve(sizeof(unsigned long long) * (L + 1), s);
    LC_CUDA(cudaMemsetAsync(sc.done_cnt.ptr, 0, sizeof(unsigned long long) * (L + 1), s));
    if (n_done > 0) {
        done_hist_kernel<<<grid_for(n_done), 256, 0, s>>>(seg_sorted, n_done, in.seg_loop,
                                                          sc.done_cnt.as<unsigned long long>());
        LC_CHECK_LAUNCH();
    }
    sc.counters.reserve(sizeof(int64_t) * 2 * (L + 1), s);
    int64_t *ocnt = sc.counters.as<int64_t>(), *dcnt = ocnt + (L + 1);
    out_counts_kernel<<<grid_for(L + 1), 256, 0, s>>>(sc.done_cnt.as<unsigned long long>(), sc.paired.as<uint8_t>(),
                                                      in.loff, L, ocnt, dcnt);
    LC_CHECK_LAUNCH();
    out.vert_off.reserve(sizeof(int64_t) * (L + 1), s);
    sc.done_off.reserve(sizeof(int64_t) * (L + 1), s);
    scan_i64(ocnt, out.vert_off.as<int64_t>(), L + 1, sc, s);
    scan_i64(dcnt, sc.done_off.as<int64_t>(), L + 1, sc, s);
    out.V = d2h<int64_t>(out.vert_off.as<int64_t>() + L, s);
    out.verts.reserve(sizeof(double) * 3 * (out.V > 0 ? out.V : 1), s);
    if (n_done > 0)
        write_done_kernel<<<grid_for(n_done), 256, 0, s>>>(n_done, seg_sorted, sc.done_tlo.as<double>(), t_idx, in.seg_loop,
                                                           in.coeffs, out.vert_off.as<int64_t>(), sc.done_off.as<int64_t>(),
                                                           out.verts.as<double>());
    if (n_done > 0) LC_CHECK_LAUNCH();
    if (M > 0)
        write_unpaired_kernel<<<grid_for(M), 256, 0, s>>>(M, in.seg_loop, sc.paired.as<uint8_t>(), in.loff, in.coeffs, in.t,
                                                          out.vert_off.as<int64_t>(), out.verts.as<double>());
    LC_CHECK_LAUNCH();
    // (5) paired loops become PolylineLoops (:189-191) -> validation
    const int ve = validate(out.verts.as<double>(), out.vert_off.as<int64_t>(), L, out.V, sc.paired.as<uint8_t>(), 1,
                            poly_thr, sc, s);
    if (ve != INT_MAX) {
        err->kind = DISC_INVALID_POLYLINE;
        err->detail = ve & 3;
        err->loops = {ve >> 2};
        return false;
    }
    return true;
}

}  // namespace lc
