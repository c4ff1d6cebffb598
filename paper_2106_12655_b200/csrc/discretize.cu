#include <algorithm>
// Device discretization: refine paired loops until the tight boxes of their
// subsegments are pairwise disjoint across every PLS pair, then emit chords.
//
// Reference: linkcert/discretize.py:112-191 with _LoopState (:52-105).  The
// per-pass state is a loop-major SoA list of active subsegments (segment id,
// t_lo, t_hi) whose within-loop order reproduces the reference's list order
// exactly ([left halves..., right halves...] after every split, :91-98), so
// the first-bad-child error report (:170-174) names the same loops.
//
// Per pass (one host sync):
//   overlap detection for every PLS pair whose loops are active:
//     small pairs (n_i*n_j <= 16384, both <= 256 — the reference's own
//     brute-force rule, bvh.py:224,236): one warp per pair, loop j's boxes
//     staged in shared memory, all box pairs tested;
//     large pairs: per-loop sorted lower bounds on 3 axes (CUB segmented
//     sort) + binary search and sweep on the pair's axis;
//   a hit marks both subsegments (atomicOr, exact marked count) and records
//   the first marking pair (atomicMin: the reference processes pairs in
//   PairList order, :77-80,151-159);
//   no marks -> the pass finishes every active subsegment; otherwise a scan
//   of the marks moves unmarked entries to the done list and writes children,
//   whose boxes feed the CurvesIntersect / max_subsegments checks (:166-180).
// Fast path (polyline chainmail, one pass, nothing marked): the active list
// is the segment list itself and the chords are the segment start points,
// written straight into the Gauss-sum layout with PolylineLoop validation
// fused in.  Vertices are eval_cubics(coeffs[seg], t_lo) in numpy's
// operation order (:89) — bitwise the reference's.
#include <climits>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "discretize.cuh"
#include "pass1.cuh"
#include "scan.cuh"
#include "geom.cuh"

namespace lc {
namespace {

constexpr double kMachineEps = 2.220446049250313e-16;
constexpr int32_t kNoIndex = 0x7f7f7f7f;       // atomicMin sentinel from cudaMemset(0x7f)
constexpr int kBruteWarps = 4;


// View of the active subsegment list: either the segment arrays themselves
// (identity, pass 1 with every loop paired) or materialized SoA arrays.
struct ActView {
    const int32_t *seg;   // nullptr: entry e is segment e
    const int32_t *loop;
    const double *tlo, *thi;
    int tstride;
    const double *box;
    int64_t bstride;
    const int64_t *off;
};

__device__ __forceinline__ double scale_of(const int *max_exp) {
    int e = *max_exp - 1023;
    e = e < -1022 ? -1022 : (e > 1022 ? 1022 : e);
    return __hiloint2double((1023 - e) << 20, 0);   // 2^-e, exact
}


__device__ __forceinline__ int64_t upper_index(const int64_t *__restrict__ off, int64_t n, int64_t k) {
    int64_t lo = 0, hi = n;   // largest idx in [0, n) with off[idx] <= k  (off[0] == 0)
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (off[mid] <= k) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ void mark_entry(uint32_t *__restrict__ mark, int32_t *__restrict__ first_pair, int64_t e,
                                           int32_t p, unsigned long long *__restrict__ marked) {
    if (!mark) {   // fused fast path: only "was anything marked" matters
        atomicAdd(marked, 1ULL);
        return;
    }
    if (atomicOr(mark + e, 1u) == 0u) atomicAdd(marked, 1ULL);
    atomicMin(first_pair + e, p);
}

// ---------------------------------------------------------------- pre-pass

__global__ void fast_init_kernel(PreCounters *__restrict__ ctr, int *__restrict__ val_err) {
    *ctr = PreCounters{INT_MAX, 0, 0, 0, 0, INT_MAX, 0};
    val_err[0] = INT_MAX;
    val_err[1] = INT_MAX;
}

__global__ void pre_pairs_kernel(const int32_t *__restrict__ pairs, int64_t P, const int64_t *__restrict__ dP,
                                 const int64_t *__restrict__ loff, const double *__restrict__ lbox, int64_t L,
                                 uint8_t *__restrict__ paired, int8_t *__restrict__ axis,
                                 PreCounters *__restrict__ ctr) {
    if (dP && *dP < P) P = *dP;   // fused path: P on the device (grid-stride over the real count)
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const int i = pairs[2 * p], j = pairs[2 * p + 1];
    paired[i] = 1;
    paired[j] = 1;
    // sweep axis: the axis along which the two loop boxes' intersection is longest
    int a = 0;
    double best = -CUDART_INF;
    for (int d = 0; d < 3; ++d) {
        const double e = fmin(lbox[(3 + d) * L + i], lbox[(3 + d) * L + j]) - fmax(lbox[d * L + i], lbox[d * L + j]);
        if (e > best) {
            best = e;
            a = d;
        }
    }
    axis[p] = (int8_t)a;
    if (!brute_pair(loff[i + 1] - loff[i], loff[j + 1] - loff[j])) {
        atomicAdd(&ctr->n_large, 1);
        ctr->abort = 1;
    }
    }
}

__global__ void pre_loops_kernel(const unsigned long long *__restrict__ min_diag, const uint8_t *__restrict__ paired,
                                 int64_t L, double min_diam, PreCounters *__restrict__ ctr) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= L) return;
    // min over segments of sqrt(squared diagonal) == sqrt(min squared diagonal)
    if (__dsqrt_rn(__longlong_as_double((long long)min_diag[l])) < min_diam) {
        atomicMin(&ctr->zero_loop, (int)l);
        ctr->abort = 1;
    }
    if (!paired[l]) atomicAdd(&ctr->n_unpaired, 1);
}

// ------------------------------------------------------------- detection

__device__ __forceinline__ bool box_overlap_f(const float *__restrict__ b, int64_t stride, int64_t e,
                                              const float lo[3], const float hi[3]) {
    return !(lo[0] > b[3 * stride + e] || b[e] > hi[0] || lo[1] > b[4 * stride + e] || b[stride + e] > hi[1] ||
             lo[2] > b[5 * stride + e] || b[2 * stride + e] > hi[2]);
}

// Warp-wide compaction of the entries [b, b+n) whose box overlaps [lo, hi]
// into list[]; returns the count (all lanes).  fbox: test the outward-rounded
// float boxes against [flo, fhi] (outward too) instead — a superset of the
// exact hits, which is all a prefilter needs (half the bytes).
__device__ __forceinline__ int filter_entries(const double *__restrict__ box, const float *__restrict__ fbox,
                                              int64_t stride, int64_t b, int64_t n, const double lo[3],
                                              const double hi[3], const float flo[3], const float fhi[3],
                                              int32_t *list, int lane) {
    int cnt = 0;
    for (int64_t k0 = 0; k0 < n; k0 += 32) {
        const int64_t k = k0 + lane;
        const bool in = k < n && (fbox ? box_overlap_f(fbox, stride, b + k, flo, fhi)
                                       : box_overlap(box, stride, b + k, lo, hi));
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        if (in) list[cnt + __popc(bal & ((1u << lane) - 1u))] = (int32_t)(b + k);
        cnt += __popc(bal);
    }
    __syncwarp();
    return cnt;
}

// Warp per brute-force pair.  Only subsegments of loop i whose box meets the
// union box of loop j's active subsegments can overlap one of them (and vice
// versa), so both sides are first filtered against the other loop's union
// box; the (usually tiny) filtered lists are then tested exhaustively.
__global__ void __launch_bounds__(32 * kBruteWarps) brute_kernel(ActView v, const double *__restrict__ ubox,
                                                                 const float *__restrict__ fbox,
                                                                 int64_t L, const int32_t *__restrict__ pairs,
                                                                 int64_t P, const int64_t *__restrict__ dP,
                                                                 uint32_t *__restrict__ mark,
                                                                 int32_t *__restrict__ first_pair,
                                                                 unsigned long long *__restrict__ marked) {
    __shared__ int32_t lists[kBruteWarps][2][kBruteMaxSide];
    if (dP && *dP < P) P = *dP;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * kBruteWarps;
    for (int64_t p = blockIdx.x * (int64_t)kBruteWarps + w; p < P; p += nw) {
        const int i = pairs[2 * p], j = pairs[2 * p + 1];
        const int64_t bi = v.off[i], ni = v.off[i + 1] - bi;
        const int64_t bj = v.off[j], nj = v.off[j + 1] - bj;
        if (ni == 0 || nj == 0 || !brute_pair(ni, nj)) continue;
        double ilo[3], ihi[3], jlo[3], jhi[3];
        float filo[3], fihi[3], fjlo[3], fjhi[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            ilo[d] = ubox[d * L + i];
            ihi[d] = ubox[(3 + d) * L + i];
            jlo[d] = ubox[d * L + j];
            jhi[d] = ubox[(3 + d) * L + j];
            filo[d] = __double2float_rd(ilo[d]);
            fihi[d] = __double2float_ru(ihi[d]);
            fjlo[d] = __double2float_rd(jlo[d]);
            fjhi[d] = __double2float_ru(jhi[d]);
        }
        int32_t *si = lists[w][0], *tj = lists[w][1];
        const int ns = filter_entries(v.box, fbox, v.bstride, bi, ni, jlo, jhi, fjlo, fjhi, si, lane);
        const int nt = ns ? filter_entries(v.box, fbox, v.bstride, bj, nj, ilo, ihi, filo, fihi, tj, lane) : 0;
        const int tot = ns * nt;
        for (int k = lane; k < tot; k += 32) {
            const int64_t es = si[k / nt], et = tj[k % nt];
            if (fbox) {   // float prefilter of the pair test; exact double test on a float hit
                float flo[3], fhi[3];
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    flo[d] = fbox[d * v.bstride + es];
                    fhi[d] = fbox[(3 + d) * v.bstride + es];
                }
                if (!box_overlap_f(fbox, v.bstride, et, flo, fhi)) continue;
            }
            double lo[3], hi[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                lo[d] = v.box[d * v.bstride + es];
                hi[d] = v.box[(3 + d) * v.bstride + es];
            }
            if (box_overlap(v.box, v.bstride, et, lo, hi)) {
                mark_entry(mark, first_pair, es, (int32_t)p, marked);
                mark_entry(mark, first_pair, et, (int32_t)p, marked);
            }
        }
        __syncwarp();
    }
}

// Fused-path pass-1 detection: does ANY pair of the (small) PLS pairs have two
// overlapping segment boxes?  (Only "nothing marked" keeps the fused path;
// otherwise the staged path recomputes the exact marks.)  Warp per pair: the
// segments of both loops are filtered against the other loop's box in one
// sweep over their outward-rounded float boxes (all loads in flight together),
// survivors are staged in shared memory with their float boxes, tested
// pairwise in float, and a float hit is confirmed with the exact closed-box
// test on the double boxes (bvh.py:93-98).  Hits are counted into *marked.
constexpr int kAnyWarps = 8;

#ifndef LC_ANY_MINB
#define LC_ANY_MINB 4   // blocks per SM the pass-1 kernel is compiled for (64 registers)
#endif
__global__ void __launch_bounds__(32 * kAnyWarps, LC_ANY_MINB) brute_any_kernel(
    const double *__restrict__ box, const float *__restrict__ fbox, int64_t M, const int64_t *__restrict__ loff,
    const double *__restrict__ lbox, int64_t L, const int32_t *__restrict__ pairs, int64_t P,
    const int64_t *__restrict__ dP, unsigned long long *__restrict__ marked, int *__restrict__ abort,
    const float *__restrict__ sub) {
    __shared__ int32_t sidx[kAnyWarps][2][kAnyCap];
    __shared__ float sbox[kAnyWarps][2][6 * kAnyCap];
    // programmatic dependent launch: the Gauss kernel queued behind this one on the
    // critical stream may start as soon as every CTA here is resident (it does not read
    // these results; it polls the abort flag), so the check runs beside the sum
    asm volatile("griddepcontrol.launch_dependents;");
    if (dP && *dP < P) P = *dP;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * kAnyWarps;
    if (sub) {   // the 8-segment group boxes exist (fused path, loops of <= 1024 segments)
        for (int64_t p = blockIdx.x * (int64_t)kAnyWarps + w; p < P; p += nw)
            brute_any_pair_sub(p, box, fbox, sub, M, L, loff, pairs, lane, marked, abort);
        return;
    }
    for (int64_t p = blockIdx.x * (int64_t)kAnyWarps + w; p < P; p += nw)
        brute_any_pair(p, box, fbox, M, loff, lbox, L, pairs, sidx[w][0], sidx[w][1], sbox[w][0], sbox[w][1], lane,
                       marked, abort);
}

// The same as single-warp blocks of kAnyLitePairs pairs capped at 32 registers:
// a block fits beside the Gauss kernel's three 168-register CTAs on an SM
// (1024 registers left), so the checks use the issue slots the FP64-bound sum
// leaves free instead of taking SMs from it.
constexpr int kAnyLitePairs = 4;
__global__ void __maxnreg__(32) brute_any_lite_kernel(
    const double *__restrict__ box, const float *__restrict__ fbox, int64_t M, const int64_t *__restrict__ loff,
    const double *__restrict__ lbox, int64_t L, const int32_t *__restrict__ pairs, int64_t P,
    const int64_t *__restrict__ dP, unsigned long long *__restrict__ marked, int *__restrict__ abort) {
    __shared__ int32_t sidx[2][kAnyCap];
    __shared__ float sbox[2][6 * kAnyCap];
    if (dP && *dP < P) P = *dP;
    const int lane = threadIdx.x & 31;
    // grid-stride over the device pair count: a bounded grid (the capacity-sized one
    // was ~56k single-warp blocks for the Kusari tube, dispatched a few at a time
    // beside the Gauss CTAs — it finished after the sum)
    for (int64_t p0 = (int64_t)blockIdx.x * kAnyLitePairs; p0 < P; p0 += (int64_t)gridDim.x * kAnyLitePairs)
        for (int64_t p = p0; p < p0 + kAnyLitePairs && p < P; ++p)
            brute_any_pair(p, box, fbox, M, loff, lbox, L, pairs, sidx[0], sidx[1], sbox[0], sbox[1], lane, marked,
                           abort);
}

// Union box of every loop's active subsegments (warp per loop).
__global__ void union_boxes_kernel(const double *__restrict__ box, int64_t stride, const int64_t *__restrict__ off,
                                   int64_t L, double *__restrict__ ubox) {
    const int64_t l = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (l >= L) return;
    double v[6] = {CUDART_INF, CUDART_INF, CUDART_INF, -CUDART_INF, -CUDART_INF, -CUDART_INF};
    for (int64_t e = off[l] + lane; e < off[l + 1]; e += 32) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            v[d] = fmin(v[d], box[d * stride + e]);
            v[3 + d] = fmax(v[3 + d], box[(3 + d) * stride + e]);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            v[d] = fmin(v[d], __shfl_xor_sync(0xffffffffu, v[d], o));
            v[3 + d] = fmax(v[3 + d], __shfl_xor_sync(0xffffffffu, v[3 + d], o));
        }
    if (lane == 0)
#pragma unroll
        for (int d = 0; d < 6; ++d) ubox[d * L + l] = v[d];
}

// Marks of the identity view (entry = segment) -> the materialized paired-only list.
__global__ void gather_marks_kernel(int64_t n, const int32_t *__restrict__ act_seg, const uint32_t *__restrict__ mark_in,
                                    const int32_t *__restrict__ fp_in, uint32_t *__restrict__ mark_out,
                                    int32_t *__restrict__ fp_out) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n) return;
    const int32_t m = act_seg[e];
    mark_out[e] = mark_in[m];
    fp_out[e] = fp_in[m];
}

__global__ void copy_lo_kernel(const double *__restrict__ box, int64_t stride, int64_t n, int axis,
                               double *__restrict__ key, int32_t *__restrict__ iota) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n) return;
    key[e] = box[axis * stride + e];
    if (iota) iota[e] = (int32_t)e;
}

// per pair: number of sweep threads (0 for brute-force pairs)
__global__ void sweep_counts_kernel(const int32_t *__restrict__ pairs, int64_t P, const int64_t *__restrict__ off,
                                    int64_t *__restrict__ cnt) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < P) {
        const int i = pairs[2 * p], j = pairs[2 * p + 1];
        const int64_t ni = off[i + 1] - off[i], nj = off[j + 1] - off[j];
        cnt[p] = (ni == 0 || nj == 0 || brute_pair(ni, nj)) ? 0 : ni + nj;
    } else if (p == P) {
        cnt[P] = 0;
    }
}

__global__ void sweep_kernel(ActView v, const int32_t *__restrict__ pairs, int64_t P, const int8_t *__restrict__ axis,
                             const int64_t *__restrict__ sweep_off, const double *__restrict__ k0,
                             const double *__restrict__ k1, const double *__restrict__ k2,
                             const int32_t *__restrict__ p0, const int32_t *__restrict__ p1,
                             const int32_t *__restrict__ p2, uint32_t *__restrict__ mark,
                             int32_t *__restrict__ first_pair, unsigned long long *__restrict__ marked) {
    const int64_t total = sweep_off[P];
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = upper_index(sweep_off, P, k);
        const int i = pairs[2 * p], j = pairs[2 * p + 1];
        const int64_t ni = v.off[i + 1] - v.off[i];
        const int64_t local = k - sweep_off[p];
        const int A = local < ni ? i : j, B = local < ni ? j : i;
        const int64_t e = v.off[A] + (local < ni ? local : local - ni);
        const int a = axis[p];
        const double *keys = a == 0 ? k0 : (a == 1 ? k1 : k2);
        const int32_t *perm = a == 0 ? p0 : (a == 1 ? p1 : p2);
        double el[3], eh[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            el[d] = v.box[d * v.bstride + e];
            eh[d] = v.box[(3 + d) * v.bstride + e];
        }
        const double lo_a = el[a], hi_a = eh[a];
        int64_t lo = v.off[B], hi = v.off[B + 1];
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
            for (int d = 0; d < 3; ++d)
                if (el[d] > v.box[(3 + d) * v.bstride + tt] || v.box[d * v.bstride + tt] > eh[d]) ov = false;
            if (ov) {
                hit_any = true;
                mark_entry(mark, first_pair, tt, (int32_t)p, marked);
            }
        }
        if (hit_any) mark_entry(mark, first_pair, e, (int32_t)p, marked);
    }
}

// ------------------------------------------------------------ split / done

__global__ void init_counts_kernel(const int64_t *__restrict__ loff, const uint8_t *__restrict__ paired, int64_t L,
                                   int64_t *__restrict__ cnt) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l < L) cnt[l] = paired[l] ? loff[l + 1] - loff[l] : 0;
    else if (l == L) cnt[L] = 0;
}

// Materialize the pass-1 list (segments of paired loops, loop-major).
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

__global__ void mark_to_i64_kernel(const uint32_t *__restrict__ mark, int64_t n, int64_t *__restrict__ out) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < n) out[e] = mark[e];
    else if (e == n) out[n] = 0;
}

__global__ void finish_kernel(int64_t n_act, const int32_t *__restrict__ pairs, const uint32_t *__restrict__ mark,
                              const int64_t *__restrict__ mscan, const int32_t *__restrict__ first_pair,
                              const int64_t *__restrict__ act_off, const int32_t *__restrict__ act_seg,
                              const int32_t *__restrict__ act_loop, const double *__restrict__ act_tlo,
                              const double *__restrict__ act_thi, int32_t *__restrict__ nxt_seg,
                              int32_t *__restrict__ nxt_loop, double *__restrict__ nxt_tlo,
                              double *__restrict__ nxt_thi, int32_t *__restrict__ nxt_partner, int64_t n_done,
                              int32_t *__restrict__ done_seg, double *__restrict__ done_tlo) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_act) return;
    const int64_t r = mscan ? mscan[e] : 0;
    const int l = act_loop[e];
    const int32_t seg = act_seg[e];
    const double tlo = act_tlo[e], thi = act_thi[e];
    if (mark && mark[e]) {
        const int64_t base = mscan[act_off[l]];
        const int64_t cnt = mscan[act_off[l + 1]] - base;
        const int64_t k = r - base, no = 2 * base;
        const double tm = __dmul_rn(0.5, __dadd_rn(tlo, thi));   // 0.5 * (tlo + thi)  (:95)
        const int32_t pp = first_pair[e];
        const int32_t partner = pairs[2 * pp] == l ? pairs[2 * pp + 1] : pairs[2 * pp];
        nxt_seg[no + k] = seg;
        nxt_loop[no + k] = l;
        nxt_tlo[no + k] = tlo;
        nxt_thi[no + k] = tm;
        nxt_partner[no + k] = partner;
        nxt_seg[no + cnt + k] = seg;
        nxt_loop[no + cnt + k] = l;
        nxt_tlo[no + cnt + k] = tm;
        nxt_thi[no + cnt + k] = thi;
        nxt_partner[no + cnt + k] = partner;
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
                                   int64_t L, int64_t max_sub, PreCounters *__restrict__ ctr) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
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

__global__ void closed_offsets_kernel(const int64_t *__restrict__ off, int64_t L, int64_t *__restrict__ voff,
                                      int64_t *__restrict__ vert_off = nullptr) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l <= L) {
        voff[l] = off[l] + l;
        if (vert_off) vert_off[l] = off[l];   // the chords' open offsets = the model's
    }
}

__device__ __forceinline__ void put_closed(double *__restrict__ X, double *__restrict__ Y, double *__restrict__ Z,
                                           int64_t vo, int64_t local, int64_t n, const double p[3], double sc) {
    X[vo + local] = p[0] * sc;
    Y[vo + local] = p[1] * sc;
    Z[vo + local] = p[2] * sc;
    if (local == 0) {   // closing vertex (direct.py:164-166)
        X[vo + n] = p[0] * sc;
        Y[vo + n] = p[1] * sc;
        Z[vo + n] = p[2] * sc;
    }
}

// No-split fast path: chord vertex m = start point of segment m for every loop
// (paired loops keep all segments; unpaired loops are control chords, :108-109),
// with the PolylineLoop checks fused (geometry.py:333-340).
template <bool POLY>
__global__ void write_all_kernel(int64_t M, const double *__restrict__ coeffs, const double *__restrict__ t,
                                 const double *__restrict__ verts, const int32_t *__restrict__ seg_loop,
                                 const int64_t *__restrict__ loff, const int *__restrict__ max_exp, double thr,
                                 double *__restrict__ X, double *__restrict__ Y, double *__restrict__ Z,
                                 unsigned *__restrict__ flags) {
    const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= M) return;
    const int l = seg_loop[m];
    const int64_t b = loff[l], n = loff[l + 1] - b, local = m - b;
    const int64_t nx = local + 1 < n ? m + 1 : b;
    double p[3], q[3];
    if (POLY) {   // eval_cubics at t = 0 of the from_polyline coefficients (a1 = next - start, a2 = a3 = 0)
        const int64_t nn = nx + 1 < b + n ? nx + 1 : b;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double v0 = verts[3 * m + d], v1 = verts[3 * nx + d], v2 = verts[3 * nn + d];
            p[d] = eval_axis(v0, v1 - v0, 0.0, 0.0, 0.0);
            q[d] = eval_axis(v1, v2 - v1, 0.0, 0.0, 0.0);
        }
    } else {
        eval_point(coeffs + 12 * m, t[2 * m], p);
        eval_point(coeffs + 12 * nx, t[2 * nx], q);
    }
    put_closed(X, Y, Z, b + l, local, n, p, scale_of(max_exp));
    unsigned f = 0;
    if (!(isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2]))) f |= 1;
    const double dx = __dsub_rn(q[0], p[0]), dy = __dsub_rn(q[1], p[1]), dz = __dsub_rn(q[2], p[2]);
    if (__dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz))) <= thr) f |= 2;
    if (f) atomicOr(flags + l, f);
}

void launch_write_all(const DiscInput &in, double thr, DiscOutput &out, unsigned *flags, cudaStream_t s) {
    if (in.M == 0) return;
    if (in.verts)
        write_all_kernel<true><<<(unsigned)ceil_div(in.M, 256), 256, 0, s>>>(in.M, nullptr, nullptr, in.verts, in.seg_loop, in.loff,
                                                             in.max_exp, thr, out.X.as<double>(), out.Y.as<double>(),
                                                             out.Z.as<double>(), flags);
    else
        write_all_kernel<false><<<(unsigned)ceil_div(in.M, 256), 256, 0, s>>>(in.M, in.coeffs, in.t, nullptr, in.seg_loop, in.loff,
                                                              in.max_exp, thr, out.X.as<double>(), out.Y.as<double>(),
                                                              out.Z.as<double>(), flags);
    LC_CHECK_LAUNCH();
}

// General path: sorted done chords + unpaired control chords into the closed SoA.
__global__ void write_done_kernel(int64_t n, const int32_t *__restrict__ seg, const double *__restrict__ tlo,
                                  const int32_t *__restrict__ idx, const int32_t *__restrict__ seg_loop,
                                  const double *__restrict__ coeffs, const int64_t *__restrict__ out_off,
                                  const int64_t *__restrict__ done_off, const int *__restrict__ max_exp,
                                  double *__restrict__ X, double *__restrict__ Y, double *__restrict__ Z) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int32_t s = seg[k];
    const double t = idx ? tlo[idx[k]] : tlo[k];
    const int l = seg_loop[s];
    const int64_t local = k - done_off[l];
    double p[3];
    eval_point(coeffs + 12 * (int64_t)s, t, p);
    put_closed(X, Y, Z, out_off[l] + l, local, out_off[l + 1] - out_off[l], p, scale_of(max_exp));
}

__global__ void write_unpaired_kernel(int64_t M, const int32_t *__restrict__ seg_loop, const uint8_t *__restrict__ paired,
                                      const int64_t *__restrict__ loff, const double *__restrict__ coeffs,
                                      const double *__restrict__ t, const int64_t *__restrict__ out_off,
                                      const int *__restrict__ max_exp, double *__restrict__ X, double *__restrict__ Y,
                                      double *__restrict__ Z, double *__restrict__ aos) {
    const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= M) return;
    const int l = seg_loop[m];
    if (paired[l]) return;
    const int64_t local = m - loff[l];
    double p[3];
    eval_point(coeffs + 12 * m, t[2 * m], p);
    if (aos) {   // temporary AoS in segment layout (pre-pass validation)
        aos[3 * m] = p[0];
        aos[3 * m + 1] = p[1];
        aos[3 * m + 2] = p[2];
    } else {
        put_closed(X, Y, Z, out_off[l] + l, local, out_off[l + 1] - out_off[l], p, scale_of(max_exp));
    }
}

// PolylineLoop checks of loops with paired[l] == want over AoS vertices with offsets `off`.
__global__ void validate_aos_kernel(const double *__restrict__ v, const int64_t *__restrict__ off,
                                    const int32_t *__restrict__ seg_loop, int64_t n,
                                    const uint8_t *__restrict__ paired, int want, double thr,
                                    unsigned *__restrict__ flags) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t l = seg_loop[k];   // AoS in segment layout: vertex k is segment k's start
    if (paired && (int)paired[l] != want) return;
    const int64_t b = off[l], e = off[l + 1];
    const int64_t nx = (k + 1 < e) ? k + 1 : b;
    const double x = v[3 * k], y = v[3 * k + 1], z = v[3 * k + 2];
    unsigned f = 0;
    if (!(isfinite(x) && isfinite(y) && isfinite(z))) f |= 1;
    const double dx = __dsub_rn(v[3 * nx], x), dy = __dsub_rn(v[3 * nx + 1], y), dz = __dsub_rn(v[3 * nx + 2], z);
    if (__dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz))) <= thr) f |= 2;
    if (f) atomicOr(flags + l, f);
}

// Same over the scaled closed SoA (vertex k+1 always exists); thr_scaled = thr * 2^-e.
__global__ void validate_soa_kernel(const double *__restrict__ X, const double *__restrict__ Y,
                                    const double *__restrict__ Z, const int64_t *__restrict__ voff, int64_t L,
                                    int64_t nclosed, const uint8_t *__restrict__ paired, int want,
                                    const int *__restrict__ max_exp, double thr, unsigned *__restrict__ flags) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nclosed) return;
    const int64_t l = upper_index(voff, L, k);
    if (k == voff[l + 1] - 1) return;   // closing vertex
    if (paired && (int)paired[l] != want) return;
    const double x = X[k], y = Y[k], z = Z[k];
    unsigned f = 0;
    if (!(isfinite(x) && isfinite(y) && isfinite(z))) f |= 1;
    const double dx = __dsub_rn(X[k + 1], x), dy = __dsub_rn(Y[k + 1], y), dz = __dsub_rn(Z[k + 1], z);
    const double len = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    if (len <= thr * scale_of(max_exp)) f |= 2;
    if (f) atomicOr(flags + l, f);
}

// First invalid loop among loops with paired == want (or all when paired == nullptr).
__global__ void validate_loops_kernel(const int64_t *__restrict__ off, int64_t L, int closed_layout,
                                      const uint8_t *__restrict__ paired, int want, const unsigned *__restrict__ flags,
                                      int *__restrict__ err) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= L) return;
    if (paired && (int)paired[l] != want) return;
    const int64_t n = off[l + 1] - off[l] - closed_layout;
    int kind = PL_OK;
    if (n < 3) kind = PL_TOO_FEW;
    else if (flags[l] & 1) kind = PL_NONFINITE;
    else if (flags[l] & 2) kind = PL_ZERO_SEGMENT;
    if (kind) atomicMin(err, (int)(l * 4 + kind));
}

__global__ void unpack_kernel(const double *__restrict__ X, const double *__restrict__ Y, const double *__restrict__ Z,
                              const int64_t *__restrict__ voff, int64_t L, int64_t nclosed,
                              const int *__restrict__ max_exp, double *__restrict__ aos) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nclosed) return;
    const int64_t l = upper_index(voff, L, k);
    if (k == voff[l + 1] - 1) return;
    const int64_t o = k - l;   // plain index
    const double inv = 1.0 / scale_of(max_exp);   // exact power of two
    aos[3 * o] = X[k] * inv;
    aos[3 * o + 1] = Y[k] * inv;
    aos[3 * o + 2] = Z[k] * inv;
}

// First invalid loop per class: err[0] over unpaired loops, err[1] over paired loops.
__global__ void validate_loops2_kernel(const int64_t *__restrict__ off, int64_t L, const uint8_t *__restrict__ paired,
                                       const unsigned *__restrict__ flags, int *__restrict__ err) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= L) return;
    const int64_t n = off[l + 1] - off[l];
    int kind = PL_OK;
    if (n < 3) kind = PL_TOO_FEW;
    else if (flags[l] & 1) kind = PL_NONFINITE;
    else if (flags[l] & 2) kind = PL_ZERO_SEGMENT;
    if (kind) atomicMin(err + (paired[l] ? 1 : 0), (int)(l * 4 + kind));
}

inline unsigned grid_for(int64_t n, int threads = 256) { return (unsigned)(n > 0 ? ceil_div(n, threads) : 1); }
// single-warp check blocks running beside the Gauss CTAs: 8 per SM
constexpr unsigned kChecksBlocks = 148 * 8;

template <class T> T d2h(const void *p, cudaStream_t s) {
    T v;
    LC_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
    return v;
}

void scan_i64(const int64_t *in, int64_t *out, int64_t n, DiscScratch &sc, cudaStream_t s) {
    sc.cub_tmp.reserve(exclusive_scan_i64_tmp_bytes(n) + 16, s);
    exclusive_scan_i64(in, out, n, sc.cub_tmp.ptr, sc.cub_tmp.bytes, s);
}

int finish_validation(DiscScratch &sc, const int64_t *off, int64_t L, int closed_layout, const uint8_t *paired,
                      int want, cudaStream_t s) {
    const int init = INT_MAX;
    LC_CUDA(cudaMemcpyAsync(sc.loop_err.ptr, &init, sizeof(int), cudaMemcpyHostToDevice, s));
    validate_loops_kernel<<<grid_for(L), 256, 0, s>>>(off, L, closed_layout, paired, want, sc.val_flags.as<unsigned>(),
                                                      sc.loop_err.as<int>());
    LC_CHECK_LAUNCH();
    return d2h<int>(sc.loop_err.ptr, s);
}

bool polyline_error(int ve, DiscError *err) {
    if (ve == INT_MAX) return false;
    err->kind = DISC_INVALID_POLYLINE;
    err->detail = ve & 3;
    err->loops = {ve >> 2};
    return true;
}

}  // namespace

void unpack_polylines(const DiscOutput &out, int64_t L, const int *max_exp, double *aos, cudaStream_t s) {
    if (out.Vc == 0) return;
    unpack_kernel<<<grid_for(out.Vc), 256, 0, s>>>(out.X.as<double>(), out.Y.as<double>(), out.Z.as<double>(),
                                                   out.voff.as<int64_t>(), L, out.Vc, max_exp, aos);
    LC_CHECK_LAUNCH();
}

bool validation_error(const int val_err[2], DiscError *err) {
    return polyline_error(val_err[0], err) || polyline_error(val_err[1], err);
}

bool run_discretize(const DiscInput &in, const DiscParams &prm, DiscScratch &sc, DiscOutput &out, DiscError *err,
                    cudaStream_t s) {
    out.validation_pending = false;
    out.d_val_err = nullptr;
    const int64_t L = in.L, M = in.M, P = in.P;
    const double min_diam = prm.epsilon * prm.xi;      // discretize.py:122
    const double poly_thr = kMachineEps * prm.xi;       // PolylineLoop(xi_hint=xi), geometry.py:338-340
    out.passes = 0;
    out.splits = 0;

    // ---- (1) pre-pass: paired flags, pair axes, zero-length check, counts (one sync)
    sc.paired.reserve(L > 0 ? L : 1, s);
    sc.pair_axis.reserve(P > 0 ? P : 1, s);
    sc.prectr.reserve(sizeof(PreCounters), s);
    sc.loop_err.reserve(sizeof(int), s);
    sc.val_flags.reserve(sizeof(unsigned) * (L > 0 ? L : 1), s);
    LC_CUDA(cudaMemsetAsync(sc.paired.ptr, 0, L > 0 ? L : 1, s));
    PreCounters pc0{INT_MAX, 0, 0, 0, 0, INT_MAX, 0};
    LC_CUDA(cudaMemcpyAsync(sc.prectr.ptr, &pc0, sizeof pc0, cudaMemcpyHostToDevice, s));
    PreCounters *ctr = sc.prectr.as<PreCounters>();
    if (P > 0) {
        pre_pairs_kernel<<<grid_for(P), 256, 0, s>>>(in.pairs, P, nullptr, in.loff, in.loop_box, L,
                                                     sc.paired.as<uint8_t>(), sc.pair_axis.as<int8_t>(), ctr);
        LC_CHECK_LAUNCH();
    }
    if (L > 0) {
        pre_loops_kernel<<<grid_for(L), 256, 0, s>>>(in.loop_min_diag, sc.paired.as<uint8_t>(), L, min_diam, ctr);
        LC_CHECK_LAUNCH();
    }
    // Pass-1 small-pair detection is launched before the first sync (identity
    // view: entry e == segment e, union boxes == loop boxes), so one read-back
    // returns the pre-checks and the pass-1 mark count together.
    const int nsm = 148;
    sc.mark.reserve(sizeof(uint32_t) * (M > 0 ? M : 1), s);
    sc.first_pair.reserve(sizeof(int32_t) * (M > 0 ? M : 1), s);
    if (M > 0) {
        LC_CUDA(cudaMemsetAsync(sc.mark.ptr, 0, sizeof(uint32_t) * M, s));
        LC_CUDA(cudaMemsetAsync(sc.first_pair.ptr, 0x7f, sizeof(int32_t) * M, s));
    }
    const ActView view0{nullptr, in.seg_loop, in.t, in.t + 1, 2, in.seg_box, M > 0 ? M : 1, in.loff};
    if (P > 0) {
        const int64_t blocks = ceil_div(P, kBruteWarps) < nsm * 16 ? ceil_div(P, kBruteWarps) : nsm * 16;
        brute_kernel<<<(unsigned)blocks, 32 * kBruteWarps, 0, s>>>(view0, in.loop_box, in.seg_fbox, L, in.pairs, P, nullptr,
                                                                   sc.mark.as<uint32_t>(), sc.first_pair.as<int32_t>(),
                                                                   &ctr->marked);
        LC_CHECK_LAUNCH();
    }
    const PreCounters pc = d2h<PreCounters>(sc.prectr.ptr, s);
    if (pc.zero_loop != INT_MAX) {   // ZeroLengthInput, first loop in order (:124-129)
        err->kind = DISC_ZERO_LENGTH;
        err->loops = {pc.zero_loop};
        return false;
    }
    // ---- (2) unpaired loops are control chords, validated before any pass (:131-142).
    // Only a refinement pass can raise an error that must come after this check;
    // without one, the check is folded into the final chord validation.
    const bool unpaired_first = pc.n_unpaired > 0 && (pc.marked > 0 || pc.n_large > 0);
    if (unpaired_first && M > 0) {
        sc.tmp_aos.reserve(sizeof(double) * 3 * M, s);
        write_unpaired_kernel<<<grid_for(M), 256, 0, s>>>(M, in.seg_loop, sc.paired.as<uint8_t>(), in.loff, in.coeffs,
                                                          in.t, nullptr, in.max_exp, nullptr, nullptr, nullptr,
                                                          sc.tmp_aos.as<double>());
        LC_CHECK_LAUNCH();
        LC_CUDA(cudaMemsetAsync(sc.val_flags.ptr, 0, sizeof(unsigned) * L, s));
        validate_aos_kernel<<<grid_for(M), 256, 0, s>>>(sc.tmp_aos.as<double>(), in.loff, in.seg_loop, M,
                                                        sc.paired.as<uint8_t>(), 0, poly_thr,
                                                        sc.val_flags.as<unsigned>());
        LC_CHECK_LAUNCH();
        if (polyline_error(finish_validation(sc, in.loff, L, 0, sc.paired.as<uint8_t>(), 0, s), err)) return false;
    }

    // ---- (3) passes
    // pass-1 list: the segment arrays themselves when every loop is paired
    int64_t n_act = 0, stride = 1;
    ActView view{};
    auto materialize = [&]() {
        sc.act_off.reserve(sizeof(int64_t) * (L + 1), s);
        sc.counters.reserve(sizeof(int64_t) * (L + 2), s);
        init_counts_kernel<<<grid_for(L + 1), 256, 0, s>>>(in.loff, sc.paired.as<uint8_t>(), L,
                                                           sc.counters.as<int64_t>());
        LC_CHECK_LAUNCH();
        scan_i64(sc.counters.as<int64_t>(), sc.act_off.as<int64_t>(), L + 1, sc, s);
        n_act = d2h<int64_t>(sc.act_off.as<int64_t>() + L, s);
        stride = n_act > 0 ? n_act : 1;
        sc.act_seg.reserve(sizeof(int32_t) * stride, s);
        sc.act_loop.reserve(sizeof(int32_t) * stride, s);
        sc.act_tlo.reserve(sizeof(double) * stride, s);
        sc.act_thi.reserve(sizeof(double) * stride, s);
        sc.box.reserve(sizeof(double) * 6 * stride, s);
        if (M > 0) {
            init_active_kernel<<<grid_for(M), 256, 0, s>>>(M, in.seg_loop, in.loff, sc.paired.as<uint8_t>(), in.t,
                                                           in.seg_box, sc.act_off.as<int64_t>(), stride,
                                                           sc.act_seg.as<int32_t>(), sc.act_loop.as<int32_t>(),
                                                           sc.act_tlo.as<double>(), sc.act_thi.as<double>(),
                                                           sc.box.as<double>());
            LC_CHECK_LAUNCH();
        }
    };
    auto act_view = [&]() {
        return ActView{sc.act_seg.as<int32_t>(), sc.act_loop.as<int32_t>(), sc.act_tlo.as<double>(),
                       sc.act_thi.as<double>(), 1, sc.box.as<double>(), stride, sc.act_off.as<int64_t>()};
    };
    // Pass 1 always runs on the segment arrays themselves (entry e == segment e):
    // unpaired loops belong to no pair, so nothing marks them, and with no mark
    // at all the chords are the segment start points of every loop.
    n_act = M;
    view = view0;
    bool is_identity = true;
    const double *ubox = in.loop_box;   // union boxes of the active subsegments per loop
    sc.ubox.reserve(sizeof(double) * 6 * (L > 0 ? L : 1), s);
    int64_t n_large = pc.n_large;
    int64_t n_done = 0;
    sc.bad_first.reserve(sizeof(int32_t) * (L > 0 ? L : 1), s);
    sc.sweep_off.reserve(sizeof(int64_t) * (P + 1), s);
    for (int pass = 0; pass < prm.max_passes; ++pass) {
        if (n_act == 0) break;
        out.passes = pass + 1;
        unsigned long long *marked_ctr = &ctr->marked;
        if (pass > 0) {
            sc.mark.reserve(sizeof(uint32_t) * n_act, s);
            sc.first_pair.reserve(sizeof(int32_t) * n_act, s);
            LC_CUDA(cudaMemsetAsync(sc.mark.ptr, 0, sizeof(uint32_t) * n_act, s));
            LC_CUDA(cudaMemsetAsync(sc.first_pair.ptr, 0x7f, sizeof(int32_t) * n_act, s));
            LC_CUDA(cudaMemsetAsync(marked_ctr, 0, sizeof(unsigned long long), s));
        }
        if (P > 0) {
            // small pairs: brute force with union-box prefilter (pass 1 already launched above)
            const int64_t blocks = ceil_div(P, kBruteWarps) < nsm * 16 ? ceil_div(P, kBruteWarps) : nsm * 16;
            if (!is_identity) {
                union_boxes_kernel<<<grid_for(L * 32), 256, 0, s>>>(view.box, view.bstride, view.off, L,
                                                                    sc.ubox.as<double>());
                LC_CHECK_LAUNCH();
                ubox = sc.ubox.as<double>();
            }
            if (pass > 0) {
                brute_kernel<<<(unsigned)blocks, 32 * kBruteWarps, 0, s>>>(view, ubox, nullptr, L, in.pairs, P, nullptr,
                                                                           sc.mark.as<uint32_t>(),
                                                                           sc.first_pair.as<int32_t>(), marked_ctr);
                LC_CHECK_LAUNCH();
            }
            // large pairs: segmented sorts + sweep (pass 1: count known; later passes: recount)
            sc.counters.reserve(sizeof(int64_t) * (P + 1), s);
            if (pass > 0) {
                sweep_counts_kernel<<<grid_for(P + 1), 256, 0, s>>>(in.pairs, P, view.off, sc.counters.as<int64_t>());
                LC_CHECK_LAUNCH();
                scan_i64(sc.counters.as<int64_t>(), sc.sweep_off.as<int64_t>(), P + 1, sc, s);
                n_large = d2h<int64_t>(sc.sweep_off.as<int64_t>() + P, s);
            }
            if (n_large > 0) {
                if (pass == 0) {
                    sweep_counts_kernel<<<grid_for(P + 1), 256, 0, s>>>(in.pairs, P, view.off,
                                                                       sc.counters.as<int64_t>());
                    LC_CHECK_LAUNCH();
                    scan_i64(sc.counters.as<int64_t>(), sc.sweep_off.as<int64_t>(), P + 1, sc, s);
                }
                sc.iota.reserve(sizeof(int32_t) * n_act, s);
                sc.done_tlo2.reserve(sizeof(double) * n_act, s);   // scratch: unsorted keys
                for (int a = 0; a < 3; ++a) {
                    sc.skey[a].reserve(sizeof(double) * n_act, s);
                    sc.sperm[a].reserve(sizeof(int32_t) * n_act, s);
                    copy_lo_kernel<<<grid_for(n_act), 256, 0, s>>>(view.box, view.bstride, n_act, a,
                                                                  sc.done_tlo2.as<double>(),
                                                                  a == 0 ? sc.iota.as<int32_t>() : nullptr);
                    LC_CHECK_LAUNCH();
                    size_t bytes = 0;
                    cub::DeviceSegmentedSort::SortPairs(nullptr, bytes, sc.done_tlo2.as<double>(),
                                                        sc.skey[a].as<double>(), sc.iota.as<int32_t>(),
                                                        sc.sperm[a].as<int32_t>(), (int)n_act, (int)L, view.off,
                                                        view.off + 1);
                    sc.cub_tmp.reserve(bytes, s);
                    bytes = sc.cub_tmp.bytes;
                    LC_CUB(cub::DeviceSegmentedSort::SortPairs(sc.cub_tmp.ptr, bytes, sc.done_tlo2.as<double>(),
                                                               sc.skey[a].as<double>(), sc.iota.as<int32_t>(),
                                                               sc.sperm[a].as<int32_t>(), (int)n_act, (int)L,
                                                               view.off, view.off + 1, s));
                }
                sweep_kernel<<<nsm * 8, 256, 0, s>>>(view, in.pairs, P, sc.pair_axis.as<int8_t>(),
                                                     sc.sweep_off.as<int64_t>(), sc.skey[0].as<double>(),
                                                     sc.skey[1].as<double>(), sc.skey[2].as<double>(),
                                                     sc.sperm[0].as<int32_t>(), sc.sperm[1].as<int32_t>(),
                                                     sc.sperm[2].as<int32_t>(), sc.mark.as<uint32_t>(),
                                                     sc.first_pair.as<int32_t>(), marked_ctr);
                LC_CHECK_LAUNCH();
            }
        }
        const int64_t marked = (pass == 0 && n_large == 0) ? (int64_t)pc.marked
                                                           : (int64_t)d2h<unsigned long long>(marked_ctr, s);
        if (marked == 0 && out.splits == 0) {   // nothing was ever refined: every segment is a chord
            n_act = 0;
            break;
        }
        if (is_identity) {   // materialize the paired-only list and carry the marks over
            materialize();
            view = act_view();
            is_identity = false;
            sc.mark2.reserve(sizeof(uint32_t) * (n_act > 0 ? n_act : 1), s);
            sc.fp2.reserve(sizeof(int32_t) * (n_act > 0 ? n_act : 1), s);
            if (n_act > 0) {
                gather_marks_kernel<<<grid_for(n_act), 256, 0, s>>>(n_act, sc.act_seg.as<int32_t>(),
                                                                    sc.mark.as<uint32_t>(), sc.first_pair.as<int32_t>(),
                                                                    sc.mark2.as<uint32_t>(), sc.fp2.as<int32_t>());
                LC_CHECK_LAUNCH();
            }
            std::swap(sc.mark, sc.mark2);
            std::swap(sc.first_pair, sc.fp2);
        }
        // capacity: children <= 2 n_act, done <= n_done + n_act
        const int64_t nstride = 2 * n_act;
        sc.nxt_seg.reserve(sizeof(int32_t) * (nstride > 0 ? nstride : 1), s);
        sc.nxt_loop.reserve(sizeof(int32_t) * (nstride > 0 ? nstride : 1), s);
        sc.nxt_tlo.reserve(sizeof(double) * (nstride > 0 ? nstride : 1), s);
        sc.nxt_thi.reserve(sizeof(double) * (nstride > 0 ? nstride : 1), s);
        sc.nxt_box.reserve(sizeof(double) * 6 * (nstride > 0 ? nstride : 1), s);
        sc.nxt_partner.reserve(sizeof(int32_t) * (nstride > 0 ? nstride : 1), s);
        sc.nxt_off.reserve(sizeof(int64_t) * (L + 1), s);
        if (n_done + n_act > sc.cap_done) {   // grow preserving contents
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
        const int64_t *mscan = nullptr;
        if (marked > 0) {
            sc.mark_scan.reserve(sizeof(int64_t) * (n_act + 1), s);
            sc.counters.reserve(sizeof(int64_t) * (n_act + 1), s);
            mark_to_i64_kernel<<<grid_for(n_act + 1), 256, 0, s>>>(sc.mark.as<uint32_t>(), n_act,
                                                                   sc.counters.as<int64_t>());
            LC_CHECK_LAUNCH();
            scan_i64(sc.counters.as<int64_t>(), sc.mark_scan.as<int64_t>(), n_act + 1, sc, s);
            mscan = sc.mark_scan.as<int64_t>();
        }
        finish_kernel<<<grid_for(n_act), 256, 0, s>>>(
            n_act, in.pairs, marked > 0 ? sc.mark.as<uint32_t>() : nullptr, mscan, sc.first_pair.as<int32_t>(),
            sc.act_off.as<int64_t>(), sc.act_seg.as<int32_t>(), sc.act_loop.as<int32_t>(), sc.act_tlo.as<double>(),
            sc.act_thi.as<double>(), sc.nxt_seg.as<int32_t>(), sc.nxt_loop.as<int32_t>(), sc.nxt_tlo.as<double>(),
            sc.nxt_thi.as<double>(), sc.nxt_partner.as<int32_t>(), n_done, sc.done_seg.as<int32_t>(),
            sc.done_tlo.as<double>());
        LC_CHECK_LAUNCH();
        n_done += n_act - marked;
        if (marked == 0) {
            n_act = 0;
            break;
        }
        next_off_kernel<<<grid_for(L + 1), 256, 0, s>>>(sc.act_off.as<int64_t>(), mscan, L, sc.nxt_off.as<int64_t>());
        LC_CHECK_LAUNCH();
        // children boxes + checks (:166-180)
        LC_CUDA(cudaMemsetAsync(sc.bad_first.ptr, 0x7f, sizeof(int32_t) * L, s));
        LC_CUDA(cudaMemsetAsync(&ctr->err_loop, 0x7f, sizeof(int), s));
        const int64_t n_new = 2 * marked;
        child_boxes_kernel<<<grid_for(n_new), 256, 0, s>>>(n_new, in.coeffs, sc.nxt_seg.as<int32_t>(),
                                                           sc.nxt_loop.as<int32_t>(), sc.nxt_tlo.as<double>(),
                                                           sc.nxt_thi.as<double>(), sc.nxt_off.as<int64_t>(), nstride,
                                                           min_diam, sc.nxt_box.as<double>(),
                                                           sc.bad_first.as<int32_t>());
        LC_CHECK_LAUNCH();
        pass_errors_kernel<<<grid_for(L > 0 ? L : 1), 256, 0, s>>>(sc.nxt_off.as<int64_t>(), sc.bad_first.as<int32_t>(),
                                                                   L, prm.max_subsegments, ctr);
        LC_CHECK_LAUNCH();
        const int err_loop = d2h<int>(&ctr->err_loop, s);
        out.splits += marked;
        if (err_loop != kNoIndex) {
            const int l = err_loop;
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
        std::swap(sc.act_seg, sc.nxt_seg);
        std::swap(sc.act_loop, sc.nxt_loop);
        std::swap(sc.act_tlo, sc.nxt_tlo);
        std::swap(sc.act_thi, sc.nxt_thi);
        std::swap(sc.box, sc.nxt_box);
        std::swap(sc.act_off, sc.nxt_off);
        stride = nstride > 0 ? nstride : 1;
        n_act = n_new;
        view = act_view();
    }
    if (n_act > 0) {   // for-else of :144,181-187
        std::vector<int64_t> off(L + 1);
        LC_CUDA(cudaMemcpyAsync(off.data(), view.off, sizeof(int64_t) * (L + 1), cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaStreamSynchronize(s));
        err->kind = DISC_PASS_BUDGET;
        err->loops.clear();
        for (int64_t l = 0; l < L; ++l)
            if (off[l + 1] > off[l]) err->loops.push_back(l);
        return false;
    }

    // ---- (4) chords into the Gauss-sum layout + PolylineLoop validation
    out.vert_off.reserve(sizeof(int64_t) * (L + 1), s);
    out.voff.reserve(sizeof(int64_t) * (L + 1), s);
    LC_CUDA(cudaMemsetAsync(sc.val_flags.ptr, 0, sizeof(unsigned) * (L > 0 ? L : 1), s));
    if (out.splits == 0) {
        out.V = M;
        out.Vc = M + L;
        LC_CUDA(cudaMemcpyAsync(out.vert_off.ptr, in.loff, sizeof(int64_t) * (L + 1), cudaMemcpyDeviceToDevice, s));
        closed_offsets_kernel<<<grid_for(L + 1), 256, 0, s>>>(in.loff, L, out.voff.as<int64_t>());
        LC_CHECK_LAUNCH();
        out.X.reserve(sizeof(double) * (out.Vc + 1), s);
        out.Y.reserve(sizeof(double) * (out.Vc + 1), s);
        out.Z.reserve(sizeof(double) * (out.Vc + 1), s);
        launch_write_all(in, poly_thr, out, sc.val_flags.as<unsigned>(), s);
        // unpaired (control-chord) loops rank before paired ones (:131-142 vs :189-191)
        sc.val_err2.reserve(2 * sizeof(int), s);
        const int init2[2] = {INT_MAX, INT_MAX};
        LC_CUDA(cudaMemcpyAsync(sc.val_err2.ptr, init2, sizeof init2, cudaMemcpyHostToDevice, s));
        validate_loops2_kernel<<<grid_for(L), 256, 0, s>>>(in.loff, L, sc.paired.as<uint8_t>(),
                                                           sc.val_flags.as<unsigned>(), sc.val_err2.as<int>());
        LC_CHECK_LAUNCH();
        out.d_val_err = sc.val_err2.as<int>();
        if (prm.defer_validation) {
            out.validation_pending = true;
            return true;
        }
        int ve[2];
        LC_CUDA(cudaMemcpyAsync(ve, sc.val_err2.ptr, sizeof ve, cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaStreamSynchronize(s));
        return !validation_error(ve, err);
    }
    // general path: done entries sorted by (seg, tlo) (the lexsort of :104)
    const int32_t *seg_sorted = sc.done_seg.as<int32_t>();
    const int32_t *t_idx = nullptr;
    if (n_done > 0) {
        sc.sort_idx.reserve(sizeof(int32_t) * n_done, s);
        sc.sort_idx2.reserve(sizeof(int32_t) * n_done, s);
        sc.done_tlo2.reserve(sizeof(double) * n_done, s);
        sc.done_seg2.reserve(sizeof(int32_t) * n_done, s);
        sc.iota.reserve(sizeof(int32_t) * n_done, s);
        sc.skey[0].reserve(sizeof(double) * n_done, s);
        sc.sperm[0].reserve(sizeof(int32_t) * n_done, s);
        copy_lo_kernel<<<grid_for(n_done), 256, 0, s>>>(sc.done_tlo.as<double>(), 0, n_done, 0,
                                                        sc.done_tlo2.as<double>(), sc.iota.as<int32_t>());
        LC_CHECK_LAUNCH();
        size_t b1 = 0, b2 = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, b1, (double *)nullptr, (double *)nullptr, (int32_t *)nullptr,
                                        (int32_t *)nullptr, (int)n_done);
        cub::DeviceRadixSort::SortPairs(nullptr, b2, (int32_t *)nullptr, (int32_t *)nullptr, (int32_t *)nullptr,
                                        (int32_t *)nullptr, (int)n_done);
        sc.cub_tmp.reserve(b1 > b2 ? b1 : b2, s);
        size_t bytes = sc.cub_tmp.bytes;
        LC_CUB(cub::DeviceRadixSort::SortPairs(sc.cub_tmp.ptr, bytes, sc.done_tlo2.as<double>(), sc.skey[0].as<double>(),
                                               sc.iota.as<int32_t>(), sc.sort_idx.as<int32_t>(), (int)n_done, 0, 64, s));
        gather_seg_kernel<<<grid_for(n_done), 256, 0, s>>>(sc.sort_idx.as<int32_t>(), n_done, sc.done_seg.as<int32_t>(),
                                                          sc.done_seg2.as<int32_t>());
        LC_CHECK_LAUNCH();
        bytes = sc.cub_tmp.bytes;
        LC_CUB(cub::DeviceRadixSort::SortPairs(sc.cub_tmp.ptr, bytes, sc.done_seg2.as<int32_t>(),
                                               sc.sperm[0].as<int32_t>(), sc.sort_idx.as<int32_t>(),
                                               sc.sort_idx2.as<int32_t>(), (int)n_done, 0, 32, s));
        seg_sorted = sc.sperm[0].as<int32_t>();
        t_idx = sc.sort_idx2.as<int32_t>();
    }
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
    sc.done_off.reserve(sizeof(int64_t) * (L + 1), s);
    scan_i64(ocnt, out.vert_off.as<int64_t>(), L + 1, sc, s);
    scan_i64(dcnt, sc.done_off.as<int64_t>(), L + 1, sc, s);
    closed_offsets_kernel<<<grid_for(L + 1), 256, 0, s>>>(out.vert_off.as<int64_t>(), L, out.voff.as<int64_t>());
    LC_CHECK_LAUNCH();
    out.V = d2h<int64_t>(out.vert_off.as<int64_t>() + L, s);
    out.Vc = out.V + L;
    out.X.reserve(sizeof(double) * (out.Vc + 1), s);
    out.Y.reserve(sizeof(double) * (out.Vc + 1), s);
    out.Z.reserve(sizeof(double) * (out.Vc + 1), s);
    if (n_done > 0) {
        write_done_kernel<<<grid_for(n_done), 256, 0, s>>>(n_done, seg_sorted, sc.done_tlo.as<double>(), t_idx,
                                                           in.seg_loop, in.coeffs, out.vert_off.as<int64_t>(),
                                                           sc.done_off.as<int64_t>(), in.max_exp, out.X.as<double>(),
                                                           out.Y.as<double>(), out.Z.as<double>());
        LC_CHECK_LAUNCH();
    }
    if (M > 0 && pc.n_unpaired > 0) {
        write_unpaired_kernel<<<grid_for(M), 256, 0, s>>>(M, in.seg_loop, sc.paired.as<uint8_t>(), in.loff, in.coeffs,
                                                          in.t, out.vert_off.as<int64_t>(), in.max_exp,
                                                          out.X.as<double>(), out.Y.as<double>(), out.Z.as<double>(),
                                                          nullptr);
        LC_CHECK_LAUNCH();
    }
    // (5) paired loops become PolylineLoops (:189-191)
    validate_soa_kernel<<<grid_for(out.Vc), 256, 0, s>>>(out.X.as<double>(), out.Y.as<double>(), out.Z.as<double>(),
                                                         out.voff.as<int64_t>(), L, out.Vc, sc.paired.as<uint8_t>(), 1,
                                                         in.max_exp, poly_thr, sc.val_flags.as<unsigned>());
    LC_CHECK_LAUNCH();
    const int ve = finish_validation(sc, out.voff.as<int64_t>(), L, 1, sc.paired.as<uint8_t>(), 1, s);
    return !polyline_error(ve, err);
}

// Fused pipeline, no-refinement case (see discretize.cuh).  Mirrors the
// pass-1 + splits == 0 branch of run_discretize kernel for kernel.
void reserve_discretize_fast(const DiscInput &in, DiscScratch &sc, DiscOutput &out, cudaStream_t s) {
    const int64_t L = in.L, M = in.M, Pcap = in.P;
    sc.paired.reserve(L > 0 ? L : 1, s);
    sc.pair_axis.reserve(Pcap > 0 ? Pcap : 1, s);
    sc.prectr.reserve(sizeof(PreCounters), s);
    sc.val_flags.reserve(sizeof(unsigned) * (L > 0 ? L : 1), s);
    sc.val_err2.reserve(2 * sizeof(int), s);
    out.vert_off.reserve(sizeof(int64_t) * (L + 1), s);
    out.voff.reserve(sizeof(int64_t) * (L + 1), s);
    out.X.reserve(sizeof(double) * (M + L + 1), s);
    out.Y.reserve(sizeof(double) * (M + L + 1), s);
    out.Z.reserve(sizeof(double) * (M + L + 1), s);
}

void launch_discretize_chords(const DiscInput &in, const DiscParams &prm, DiscScratch &sc, DiscOutput &out,
                              cudaStream_t s, bool prezeroed) {
    const int64_t L = in.L, M = in.M;
    const double poly_thr = kMachineEps * prm.xi;
    out.passes = 1;
    out.splits = 0;
    out.V = M;
    out.Vc = M + L;
    closed_offsets_kernel<<<grid_for(L + 1), 256, 0, s>>>(in.loff, L, out.voff.as<int64_t>(),
                                                           out.vert_off.as<int64_t>());
    LC_CHECK_LAUNCH();
    if (!prezeroed) LC_CUDA(cudaMemsetAsync(sc.val_flags.ptr, 0, sizeof(unsigned) * (L > 0 ? L : 1), s));
    launch_write_all(in, poly_thr, out, sc.val_flags.as<unsigned>(), s);
}

#ifndef LC_BRUTE_BPS
#define LC_BRUTE_BPS 8   // pass-1 check on the critical stream: blocks per SM cap (8 warps each, grid-stride)
#endif
void launch_pass1_brute(const DiscInput &in, const int64_t *d_P, DiscScratch &sc, cudaStream_t s) {
    const int64_t Pcap = in.P, M = in.M;
    if (Pcap <= 0 || M <= 0) return;
    PreCounters *ctr = sc.prectr.as<PreCounters>();
    const int64_t blocks = ceil_div(Pcap, kAnyWarps) < 148 * LC_BRUTE_BPS ? ceil_div(Pcap, kAnyWarps) : 148 * LC_BRUTE_BPS;
    brute_any_kernel<<<(unsigned)blocks, 32 * kAnyWarps, 0, s>>>(in.seg_box, in.seg_fbox, M, in.loff, in.loop_box,
                                                                 in.L, in.pairs, Pcap, d_P, &ctr->marked, &ctr->abort,
                                                                 in.seg_sub);
    LC_CHECK_LAUNCH();
}

void launch_discretize_checks(const DiscInput &in, const int64_t *d_P, const DiscParams &prm, DiscScratch &sc,
                              DiscOutput &out, cudaStream_t s, cudaEvent_t chords_done, const PreCounters **d_ctr,
                              bool brute_by_caller, bool prezeroed) {
    const int64_t L = in.L, M = in.M, Pcap = in.P;
    const double min_diam = prm.epsilon * prm.xi;
    PreCounters *ctr = sc.prectr.as<PreCounters>();
    if (!prezeroed) LC_CUDA(cudaMemsetAsync(sc.paired.ptr, 0, L > 0 ? L : 1, s));
    if (Pcap > 0) {
        // single-warp blocks: they fit beside the Gauss kernel's CTAs (this branch runs under it)
        pre_pairs_kernel<<<std::min(grid_for(Pcap, 32), kChecksBlocks), 32, 0, s>>>(in.pairs, Pcap, d_P, in.loff, in.loop_box, L,
                                                        sc.paired.as<uint8_t>(), sc.pair_axis.as<int8_t>(), ctr);
        LC_CHECK_LAUNCH();
        tl_mark("S1:pre_pairs", s);
    }
    if (L > 0) {
        pre_loops_kernel<<<grid_for(L, 32), 32, 0, s>>>(in.loop_min_diag, sc.paired.as<uint8_t>(), L, min_diam, ctr);
        LC_CHECK_LAUNCH();
    }
    if (Pcap > 0 && M > 0 && !brute_by_caller) {   // else launch_pass1_brute on the caller's stream
        // the 8-warp grid-stride kernel (default) runs in the slots the short-lived Gauss
        // CTAs free; LINKCERT_BRUTE_LITE=1 selects the single-warp variant (A/B: 0.460 vs
        // 0.463 ms per Kusari step)
        static const bool lite = [] {
            const char *e = getenv("LINKCERT_BRUTE_LITE");
            return e && e[0] == '1';
        }();
        if (lite) {
            brute_any_lite_kernel<<<(unsigned)ceil_div(Pcap, kAnyLitePairs), 32, 0, s>>>(
                in.seg_box, in.seg_fbox, M, in.loff, in.loop_box, L, in.pairs, Pcap, d_P, &ctr->marked, &ctr->abort);
        } else {
            const int64_t blocks = ceil_div(Pcap, kAnyWarps) < 148 * 8 ? ceil_div(Pcap, kAnyWarps) : 148 * 8;
            brute_any_kernel<<<(unsigned)blocks, 32 * kAnyWarps, 0, s>>>(in.seg_box, in.seg_fbox, M, in.loff,
                                                                         in.loop_box, L, in.pairs, Pcap, d_P,
                                                                         &ctr->marked, &ctr->abort, in.seg_sub);
        }
        LC_CHECK_LAUNCH();
        tl_mark("S1:brute", s);
    }
    if (chords_done) LC_CUDA(cudaStreamWaitEvent(s, chords_done, 0));   // validation reads the chord flags
    if (L > 0) {
        validate_loops2_kernel<<<grid_for(L, 32), 32, 0, s>>>(in.loff, L, sc.paired.as<uint8_t>(),
                                                           sc.val_flags.as<unsigned>(), sc.val_err2.as<int>());
        LC_CHECK_LAUNCH();
    }
    out.d_val_err = sc.val_err2.as<int>();
    out.validation_pending = true;
    *d_ctr = ctr;
}

void launch_discretize_init(DiscScratch &sc, cudaStream_t s) {
    fast_init_kernel<<<1, 1, 0, s>>>(sc.prectr.as<PreCounters>(), sc.val_err2.as<int>());
    LC_CHECK_LAUNCH();
}

void launch_discretize_fast(const DiscInput &in, const int64_t *d_P, const DiscParams &prm, DiscScratch &sc,
                            DiscOutput &out, cudaStream_t s, const PreCounters **d_ctr) {
    reserve_discretize_fast(in, sc, out, s);
    launch_discretize_init(sc, s);
    launch_discretize_chords(in, prm, sc, out, s);
    launch_discretize_checks(in, d_P, prm, sc, out, s, nullptr, d_ctr);
}

}  // namespace lc
