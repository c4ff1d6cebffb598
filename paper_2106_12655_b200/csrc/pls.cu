// Device potential-link search: tight segment boxes -> loop AABBs ->
// warp-cooperative sort-and-sweep -> sorted unique (i<j) loop pairs.
//
// Reference: linkcert/pls.py:48-73 (loop_boxes, potential_link_search),
// bvh.py:93-98 (closed-interval overlap), bvh.py:227-243 (the broad phase it
// replaces; only the resulting SET matters, the caller sorts).  The pair set
// is exact: for two overlapping closed intervals one lower end lies inside
// the other interval, so sweeping every loop over the loops that follow it
// in lower-bound order while lo_b <= hi_a visits every overlapping pair; the
// full 3-axis closed test then decides.
#include <climits>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "geom.cuh"
#include "gauss.cuh"
#include "pls.cuh"
#include "scan.cuh"

namespace lc {
namespace {

constexpr int kPackShift = 24;   // fused-path row scan: pair count in the low 24 bits, items above

// The initial values of a fused run (counters, flags, cell counts ...), written by
// the first kernel of the run (grid-stride over every range).
constexpr int kMaxZeroRanges = 16;
struct ZeroList {
    ZeroRange r[kMaxZeroRanges];
    int n;
};
__device__ __forceinline__ void zero_ranges(const ZeroList &zl) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int k = 0; k < zl.n; ++k) {
        unsigned *p = static_cast<unsigned *>(zl.r[k].ptr);
        const unsigned v = zl.r[k].value;
        for (int64_t i = t0; i < zl.r[k].words; i += stride) p[i] = v;
    }
}

// acc = the grid reduction's ordered keys (3 min, 4 max) + its block counter, kept
// at the identity between runs: set once at allocation, restored by the last
// block of every reduction after it has read them.
__device__ __forceinline__ void reset_grid_keys(unsigned long long *acc) {
    for (int q = 0; q < 3; ++q) acc[q] = ~0ULL;
    for (int q = 3; q < 8; ++q) acc[q] = 0ULL;
}

__device__ __forceinline__ int exp_field(double x) { return (__double2hiint(x) >> 20) & 0x7ff; }

// Ordered 64-bit keys of doubles for atomicMin/atomicMax: monotone for
// non-NaN values; NaN gets the extreme key of the reduction direction so it
// propagates like np.min / np.max (min keys: 0, max keys: ~0).
__device__ __forceinline__ unsigned long long min_key(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return x != x ? 0ULL : ((b >> 63) ? ~b : b ^ 0x8000000000000000ULL);
}
__device__ __forceinline__ unsigned long long max_key(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return x != x ? ~0ULL : ((b >> 63) ? ~b : b ^ 0x8000000000000000ULL);
}
__device__ __forceinline__ double key_value(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k ^ 0x8000000000000000ULL) : ~k));
}

// Group minimum of a 64-bit value over the lanes in `grp` (all lanes of a group
// call with the same mask): high word first, then the low word among the
// lanes holding the minimal high word.
__device__ __forceinline__ unsigned long long group_min_u64(unsigned grp, unsigned long long v) {
    const unsigned hi = __reduce_min_sync(grp, (unsigned)(v >> 32));
    const unsigned lo = __reduce_min_sync(grp, (unsigned)(v >> 32) == hi ? (unsigned)v : 0xffffffffu);
    return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ unsigned long long group_max_u64(unsigned grp, unsigned long long v) {
    const unsigned hi = __reduce_max_sync(grp, (unsigned)(v >> 32));
    const unsigned lo = __reduce_max_sync(grp, (unsigned)(v >> 32) == hi ? (unsigned)v : 0u);
    return ((unsigned long long)hi << 32) | lo;
}

// Tight per-segment boxes (geometry.py:113-152) plus, fused: seg_loop, the
// outward-rounded float copy, the per-loop union boxes as ordered keys
// (loop_keys: 3 x L min keys, then 3 x L max keys; decoded by
// loop_keys_decode_kernel), the per-loop minimum squared box diagonal and the
// coordinate exponent.  A loop's segments are contiguous, so the lanes of a
// warp that share a loop form one group: group reductions, one atomic per
// group and value.
// POLY: the model is closed polylines given by their vertices (verts, (M,3));
// segment m's coefficients are LoopGeometry.from_polyline's (a0 = v_m,
// a1 = v_next - v_m, a2 = a3 = 0, t = [0, 1]), formed in registers.
template <bool POLY>
__global__ void seg_boxes_kernel(const double *__restrict__ coeffs, const double *__restrict__ t,
                                 const double *__restrict__ verts, const int64_t *__restrict__ loff, int64_t L,
                                 int64_t M, double *__restrict__ box, float *__restrict__ fbox,
                                 int32_t *__restrict__ seg_loop, unsigned long long *__restrict__ loop_min_diag2,
                                 unsigned long long *__restrict__ loop_keys, int *__restrict__ max_exp) {
    const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    // loop of segment m: one binary search per warp (its first segment), then
    // each lane walks forward (a warp spans few loops)
    const int64_t m0 = m - lane;
    int64_t l0 = 0;
    if (lane == 0 && m0 < M) {
        int64_t lo = 0, hi = L;   // largest l with loff[l] <= m0
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (loff[mid] <= m0) lo = mid; else hi = mid;
        }
        l0 = lo;
    }
    l0 = __shfl_sync(0xffffffffu, l0, 0);
    int e = 0;
    int key = -1 - lane;   // unique when the lane has no segment
    double bl[3] = {0, 0, 0}, bh[3] = {0, 0, 0};
    unsigned long long dg = ~0ULL;
    if (m < M) {
        int64_t lo = l0;
        while (loff[lo + 1] <= m) ++lo;
        seg_loop[m] = (int32_t)lo;
        if (POLY) {
            // tight_box of (a0, a1, 0, 0) over [0, 1]: with a2 = a3 = +0 both root
            // candidates are NaN (qa == 0; q == -0 or NaN), so they clip to t = 0 and
            // the box is np.min/np.max over (v(0), v(1), v(0), v(0)) = over (v(0), v(1)).
            const int64_t nx = m + 1 < loff[lo + 1] ? m + 1 : loff[lo];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const double a0 = verts[3 * m + d], a1 = verts[3 * nx + d] - a0;
                // eval_axis at t = 0 and 1 with a2 = a3 = 0, bitwise: a0 (+0 for -0) and a0 + a1 (+0 for -0)
                const double v0 = __dadd_rn(a0, 0.0), v1 = __dadd_rn(__dadd_rn(a0, a1), 0.0);
                bl[d] = np_min(v0, v1);
                bh[d] = np_max(v0, v1);
            }
        } else {
            tight_box(coeffs + 12 * m, t[2 * m], t[2 * m + 1], bl, bh);
        }
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            box[d * M + m] = bl[d];
            box[(3 + d) * M + m] = bh[d];
            if (fbox) {   // outward-rounded float copy: a conservative prefilter box
                fbox[d * M + m] = __double2float_rd(bl[d]);
                fbox[(3 + d) * M + m] = __double2float_ru(bh[d]);
            }
            const int a = exp_field(bl[d]), b = exp_field(bh[d]);
            e = max(e, max(a, b));
        }
        key = (int)lo;
        // squared diagonal ((dx*dx + dy*dy) + dz*dz); sqrt is monotone, so the
        // loop minimum of the norms (discretize.py:124-129) is sqrt of this minimum.
        // Non-negative doubles order like their bit patterns.
        const double dx = __dsub_rn(bh[0], bl[0]), dy = __dsub_rn(bh[1], bl[1]), dz = __dsub_rn(bh[2], bl[2]);
        dg = (unsigned long long)__double_as_longlong(
            __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    }
    if (loop_min_diag2 || loop_keys) {
        const unsigned grp = __match_any_sync(0xffffffffu, key);
        const bool head = lane == __ffs(grp) - 1 && key >= 0;
        if (loop_min_diag2) {
            const unsigned long long g = group_min_u64(grp, dg);
            if (head) atomicMin(loop_min_diag2 + key, g);
        }
        if (loop_keys) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const unsigned long long kl = group_min_u64(grp, min_key(bl[d]));
                const unsigned long long kh = group_max_u64(grp, max_key(bh[d]));
                if (head) {
                    atomicMin(loop_keys + d * L + key, kl);
                    atomicMax(loop_keys + (3 + d) * L + key, kh);
                }
            }
        }
    }
    if (max_exp) {
        e = __reduce_max_sync(0xffffffffu, e);
        if (lane == 0 && e > 0) atomicMax(max_exp, e);
    }
}

// The same outputs for models whose loops are all short (<= kLoopWarpMax
// segments, e.g. chainmail rings): warp per loop, lanes over its segments —
// no loop lookup, plain warp reductions, direct stores of the loop box and
// minimum diagonal (no keys, no atomics but the exponent).
// SEG_OUT / LOOP_OUT: the fused path splits the outputs over two branches —
// the loop-level ones (loop boxes, minimum diagonals: PLS input, on the critical
// path) and the segment-level ones (boxes, float boxes, segment loop, exponent:
// read only by the chord and pass-1 branches) — so the critical path writes
// ~L x 56 B instead of ~M x 76 B.
constexpr int64_t kLoopWarpMax = 1024;
template <bool POLY, bool SEG_OUT = true, bool LOOP_OUT = true>
__global__ void seg_boxes_loop_kernel(const double *__restrict__ coeffs, const double *__restrict__ t,
                                      const double *__restrict__ verts, const int64_t *__restrict__ loff, int64_t L,
                                      int64_t M, double *__restrict__ box, float *__restrict__ fbox,
                                      int32_t *__restrict__ seg_loop, unsigned long long *__restrict__ loop_min_diag2,
                                      double *__restrict__ lbox, int *__restrict__ max_exp,
                                      float *__restrict__ sub = nullptr) {
    const int lane = threadIdx.x & 31;
    const int64_t l = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (l >= L) return;   // the whole warp
    const int64_t b = loff[l], e = loff[l + 1];
    double v[6] = {CUDART_INF, CUDART_INF, CUDART_INF, -CUDART_INF, -CUDART_INF, -CUDART_INF};
    unsigned long long dg = ~0ULL;
    int ex = 0;
    // whole-warp iterations (the group boxes below reduce over lanes); lanes past the
    // loop's end carry empty boxes
#pragma unroll 2   // both segments' loads of a 64-segment loop in flight together
    for (int64_t k0 = 0; k0 < e - b; k0 += 32) {
        const int64_t m = b + k0 + lane;
        const bool ok = m < e;
        double bl[3] = {CUDART_INF, CUDART_INF, CUDART_INF}, bh[3] = {-CUDART_INF, -CUDART_INF, -CUDART_INF};
        if (ok) {
            if (POLY) {   // see seg_boxes_kernel: the box of a from_polyline segment
                const int64_t nx = m + 1 < e ? m + 1 : b;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const double a0 = verts[3 * m + d], a1 = verts[3 * nx + d] - a0;
                    // eval_axis at t = 0 and 1 with a2 = a3 = 0, bitwise: a0 (+0 for -0) and a0 + a1 (+0 for -0)
                    const double v0 = __dadd_rn(a0, 0.0), v1 = __dadd_rn(__dadd_rn(a0, a1), 0.0);
                    bl[d] = np_min(v0, v1);
                    bh[d] = np_max(v0, v1);
                }
            } else {
                tight_box(coeffs + 12 * m, t[2 * m], t[2 * m + 1], bl, bh);
            }
        }
        if (SEG_OUT && ok) seg_loop[m] = (int32_t)l;
        float fl[6];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            fl[d] = __double2float_rd(bl[d]);
            fl[3 + d] = __double2float_ru(bh[d]);
            if (SEG_OUT && ok) {
                box[d * M + m] = bl[d];
                box[(3 + d) * M + m] = bh[d];
                if (fbox) {
                    fbox[d * M + m] = fl[d];
                    fbox[(3 + d) * M + m] = fl[3 + d];
                }
                ex = max(ex, max(exp_field(bl[d]), exp_field(bh[d])));
            }
            v[d] = np_min(v[d], bl[d]);
            v[3 + d] = np_max(v[3 + d], bh[d]);
        }
        if (LOOP_OUT && ok) {
            const double dx = __dsub_rn(bh[0], bl[0]), dy = __dsub_rn(bh[1], bl[1]), dz = __dsub_rn(bh[2], bl[2]);
            const unsigned long long q = (unsigned long long)__double_as_longlong(
                __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
            dg = q < dg ? q : dg;
        }
        if (SEG_OUT && sub) {
            // float boxes of 8-segment groups (the pass-1 check's first level): 8-lane
            // min / max; a NaN coordinate makes the group unbounded on that axis (the
            // segment-level test then sees the NaN)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                fl[d] = fl[d] != fl[d] ? -CUDART_INF_F : fl[d];
                fl[3 + d] = fl[3 + d] != fl[3 + d] ? CUDART_INF_F : fl[3 + d];
            }
#pragma unroll
            for (int off = 1; off < 8; off <<= 1)
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    fl[d] = fminf(fl[d], __shfl_xor_sync(0xffffffffu, fl[d], off));
                    fl[3 + d] = fmaxf(fl[3 + d], __shfl_xor_sync(0xffffffffu, fl[3 + d], off));
                }
            if ((lane & 7) == 0 && ok) {
                const int64_t slot = pass1_group_slot(m, l), S = pass1_group_stride(M, L);
#pragma unroll
                for (int d = 0; d < 6; ++d) sub[d * S + slot] = fl[d];
            }
        }
    }
    if (!LOOP_OUT) {   // segment outputs only: the exponent is the one loop-level value they need
        ex = __reduce_max_sync(0xffffffffu, ex);
        if (lane == 0 && max_exp && ex > 0) atomicMax(max_exp, ex);
        return;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            v[d] = np_min(v[d], __shfl_xor_sync(0xffffffffu, v[d], off));
            v[3 + d] = np_max(v[3 + d], __shfl_xor_sync(0xffffffffu, v[3 + d], off));
        }
    }
    dg = group_min_u64(0xffffffffu, dg);
    ex = __reduce_max_sync(0xffffffffu, ex);
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < 6; ++d) lbox[d * L + l] = v[d];
        if (loop_min_diag2) loop_min_diag2[l] = dg;
        if (max_exp && ex > 0) atomicMax(max_exp, ex);
    }
}

// Loop AABBs from the ordered keys (empty loop: [+inf, -inf], like the
// reduction identity of loop_boxes_kernel).
__global__ void loop_keys_decode_kernel(const unsigned long long *__restrict__ keys, int64_t L,
                                        double *__restrict__ lbox) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= L) return;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const unsigned long long kl = keys[d * L + l], kh = keys[(3 + d) * L + l];
        lbox[d * L + l] = kl == 0ULL ? CUDART_NAN : (kl == ~0ULL ? CUDART_INF : key_value(kl));
        lbox[(3 + d) * L + l] = kh == ~0ULL ? CUDART_NAN : (kh == 0ULL ? -CUDART_INF : key_value(kh));
    }
}

// One block: axis of the largest model extent -> *axis; keys[l] = lo_axis[l], idx[l] = l.
__global__ void sweep_axis_kernel(const double *__restrict__ lbox, int64_t L, int *axis, double *keys,
                                  int32_t *idx) {
    __shared__ double red[6][32];
    __shared__ int s_axis;
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
            if (e > best) {
                best = e;
                a = d;
            }
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

// Boxes in sweep order (coalesced candidate loads in the sweep).
__global__ void gather_boxes_kernel(const double *__restrict__ lbox, const int32_t *__restrict__ perm, int64_t L,
                                    double *__restrict__ sbox) {
    const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= L) return;
    const int64_t l = perm[a];
#pragma unroll
    for (int d = 0; d < 6; ++d) sbox[d * L + a] = lbox[d * L + l];
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

// Warp per sorted loop a: lanes test the following loops 32 at a time while
// lo_axis(b) <= hi_axis(a); hits are appended (ballot + one atomic per warp).
__global__ void sweep_warp_kernel(const double *__restrict__ sbox, const int32_t *__restrict__ perm, int64_t L,
                                  const int *__restrict__ axis, const uint64_t *__restrict__ excl, int64_t n_excl,
                                  unsigned long long *__restrict__ counter, uint64_t *__restrict__ out, int64_t cap) {
    const int lane = threadIdx.x & 31;
    const int ax = *axis;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t a = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; a < L; a += nwarps) {
        double al[3], ah[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            al[d] = sbox[d * L + a];
            ah[d] = sbox[(3 + d) * L + a];
        }
        const double hia = ah[ax];
        const uint64_t ia = (uint64_t)perm[a];
        for (int64_t b0 = a + 1; b0 < L; b0 += 32) {
            const int64_t b = b0 + lane;
            const bool valid = b < L;
            const double key = valid ? sbox[ax * L + b] : CUDART_INF;
            const bool in = valid && key <= hia;
            bool hit = in;
            if (in) {
#pragma unroll
                for (int d = 0; d < 3; ++d)
                    if (al[d] > sbox[(3 + d) * L + b] || sbox[d * L + b] > ah[d]) hit = false;
            }
            uint64_t k64 = 0;
            if (hit) {
                const uint64_t ib = (uint64_t)perm[b];
                k64 = ia < ib ? (ia << 32) | ib : (ib << 32) | ia;
                if (n_excl && is_excluded(excl, n_excl, k64)) hit = false;
            }
            const unsigned ballot = __ballot_sync(0xffffffffu, hit);
            if (ballot) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(counter, (unsigned long long)__popc(ballot));
                base = __shfl_sync(0xffffffffu, base, 0);
                const int64_t pos = (int64_t)base + __popc(ballot & ((1u << lane) - 1u));
                if (hit && pos < cap) out[pos] = k64;
            }
            // keys are sorted: once lane 31's key exceeds hi_a, no later block can start inside
            if (!__shfl_sync(0xffffffffu, in, 31)) break;
        }
    }
}

// ------------------------------------------------------- uniform-grid PLS
// Exact and sort-free.  Cell size c >= the largest loop-box extent, so a loop b
// overlapping loop a satisfies lo_a - c <= lo_b <= hi_a on every axis: every
// loop is stored once, in the cell of its lower corner, and a query scans the
// cells [cell(lo_a) - 2, cell(hi_a)] per axis (floor((x - o) / c) is monotone
// in x; the extra cell absorbs the rounding of lo_a - c).  A pair is emitted
// only from its smaller index, into per-row slots sorted at compaction, so the
// output is the PairList order without a global sort.


struct GridParams {
    double o[3];
    double c, ic;   // cell size (>= the largest loop extent) and 1 / c
    int dims[3];
    int pad;
};

// (x - o) * (1/c): any monotone map of x works (the query's two-cell margin absorbs
// the rounding) and a multiply replaces an FP64 division per coordinate
__device__ __forceinline__ int cell_coord(double x, double o, double ic, int dim) {
    const double f = floor((x - o) * ic);
    return f < 0.0 ? 0 : (f >= (double)dim ? dim - 1 : (int)f);
}

__device__ __forceinline__ int64_t owner_cell(const double *__restrict__ lbox, int64_t L, int64_t l,
                                              const GridParams &g) {
    const int cx = cell_coord(lbox[l], g.o[0], g.ic, g.dims[0]);
    const int cy = cell_coord(lbox[L + l], g.o[1], g.ic, g.dims[1]);
    const int cz = cell_coord(lbox[2 * L + l], g.o[2], g.ic, g.dims[2]);
    return ((int64_t)cz * g.dims[1] + cy) * g.dims[0] + cx;
}

// cell of each loop's lower corner and the loop's rank within that cell
__global__ void cell_count_kernel(const double *__restrict__ lbox, int64_t L, const GridParams *__restrict__ gp,
                                  int64_t *__restrict__ count, int32_t *__restrict__ lcell, int32_t *__restrict__ lrank) {
    LC_PDL_TRIGGER();
    LC_PDL_WAIT();
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= L) return;
    const GridParams g = *gp;
    const int64_t c = owner_cell(lbox, L, l, g);
    lcell[l] = (int32_t)c;
    lrank[l] = (int32_t)atomicAdd((unsigned long long *)(count + c), 1ULL);
}

// loops in cell order with their boxes alongside (the query reads both at once)
__global__ void cell_scatter_kernel(const double *__restrict__ lbox, int64_t L, const int64_t *__restrict__ cell_off,
                                    const int32_t *__restrict__ lcell, const int32_t *__restrict__ lrank,
                                    int32_t *__restrict__ cell_loops, double *__restrict__ cbox) {
    LC_PDL_TRIGGER();
    LC_PDL_WAIT();
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= L) return;
    const int64_t pos = cell_off[lcell[l]] + lrank[l];
    cell_loops[pos] = (int32_t)l;
#pragma unroll
    for (int d = 0; d < 6; ++d) cbox[d * L + pos] = lbox[d * L + l];
}

// Warp per loop a.  The candidate cells form up to 4 x 4 rows (z, y) of 4
// consecutive x cells, i.e. up to 16 contiguous ranges of the cell-ordered
// loop list: lanes fetch the row ranges at once, scan their lengths, and then
// sweep the concatenated candidates 32 at a time (loop id + box read together),
// so a query costs a few dependent memory round trips instead of ~3 per row.
// Hits (b > a, closed-box overlap, not excluded) are ranked with a ballot.
template <bool SLOTS>
__global__ void grid_query_warp_kernel(const double *__restrict__ lbox, int64_t L, const GridParams *__restrict__ gp,
                                       const int64_t *__restrict__ cell_off, const int32_t *__restrict__ cell_loops,
                                       const double *__restrict__ cbox, const uint64_t *__restrict__ excl,
                                       int64_t n_excl, int *__restrict__ row_count, int32_t *__restrict__ slots,
                                       const int64_t *__restrict__ offs, uint64_t *__restrict__ keys,
                                       int64_t *__restrict__ counts64, int *__restrict__ overflow,
                                       const int64_t *__restrict__ item_loff) {
    LC_PDL_TRIGGER();
    LC_PDL_WAIT();
    const int lane = threadIdx.x & 31;
    const int64_t a = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (a >= L) return;
    const GridParams g = *gp;
    double al[3], ah[3];
    int c0[3], c1[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        al[d] = lbox[d * L + a];
        ah[d] = lbox[(3 + d) * L + a];
        c0[d] = max(cell_coord(al[d], g.o[d], g.ic, g.dims[d]) - 2, 0);
        c1[d] = cell_coord(ah[d], g.o[d], g.ic, g.dims[d]);
    }
    const int ny = c1[1] - c0[1] + 1, nrows_all = ny * (c1[2] - c0[2] + 1);   // <= 25 (cells >= any extent)
    int n = 0;
    int64_t row_items = 0;   // fused path: work items of this row's pairs (the loops' segment counts)
    const int64_t w0 = SLOTS ? 0 : offs[a];
    const int ncols_a = item_loff ? (int)(item_loff[a + 1] - item_loff[a]) : 0;
    for (int rb = 0; rb < nrows_all; rb += 32) {   // one batch unless the grid is degenerate
    const int nrows = nrows_all - rb < 32 ? nrows_all - rb : 32;
    int64_t kb = 0, len = 0;
    if (lane < nrows) {
        const int rr = rb + lane;
        const int cz = c0[2] + rr / ny, cy = c0[1] + rr % ny;
        const int64_t row = ((int64_t)cz * g.dims[1] + cy) * g.dims[0];
        kb = cell_off[row + c0[0]];
        len = cell_off[row + c1[0] + 1] - kb;
    }
    int64_t incl = len;   // inclusive scan of the row lengths
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
    const int64_t excl_start = incl - len;
    for (int64_t f0 = 0; f0 < total; f0 += 32) {
        const int64_t f = f0 + lane;
        // row of flat candidate f: the last row whose start is <= f (rows of length 0 skipped)
        int r = 0;
        for (int q = 1; q < nrows; ++q) {
            const int64_t st = __shfl_sync(0xffffffffu, excl_start, q);
            if (st <= f) r = q;
        }
        const int64_t kr = __shfl_sync(0xffffffffu, kb, r) + (f - __shfl_sync(0xffffffffu, excl_start, r));
        bool hit = false;
        int64_t b = 0;
        if (f < total) {
            b = cell_loops[kr];
            double bl[3], bh[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                bl[d] = cbox[d * L + kr];
                bh[d] = cbox[(3 + d) * L + kr];
            }
            hit = b > a;
#pragma unroll
            for (int d = 0; d < 3; ++d)
                if (al[d] > bh[d] || bl[d] > ah[d]) hit = false;
            if (hit && n_excl && is_excluded(excl, n_excl, ((uint64_t)a << 32) | (uint64_t)b)) hit = false;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        if (SLOTS && item_loff && hit) {
            const PairGeom pgm = make_pair_geom(0, 0, ncols_a, (int)(item_loff[b + 1] - item_loff[b]));
            row_items += (int64_t)pgm.items_r * pgm.items_c;
        }
        if (hit) {
            const int rk = n + __popc(bal & ((1u << lane) - 1u));
            if (SLOTS) {
                if (rk < kRowSlots) slots[a * kRowSlots + rk] = (int32_t)b;
            } else {
                keys[w0 + rk] = ((uint64_t)a << 32) | (uint64_t)b;
            }
        }
        n += __popc(bal);
    }
    }
    if (SLOTS && item_loff) {
#pragma unroll
        for (int o = 16; o; o >>= 1) row_items += __shfl_xor_sync(0xffffffffu, row_items, o);
    }
    if (SLOTS && lane == 0) {
        row_count[a] = n;
        // scanned into the pair offsets (fused path: items << kPackShift | pairs, one scan for both)
        counts64[a] = item_loff ? (row_items << kPackShift) | (int64_t)n : (int64_t)n;
        if (a == L - 1) counts64[L] = 0;
        if (n > kRowSlots) atomicMax(overflow, n);   // rare: the two-pass variant takes over
    }
}

// Ordered-integer images of doubles (monotone): min/max through integer atomics.
__device__ __forceinline__ unsigned long long ord_key(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k));
}

// Stage 2 (one thread): origin, cell size >= max extent, dims with product <= max_cells.
__device__ void grid_finalize(const unsigned long long *acc, int64_t max_cells, GridParams *__restrict__ gp) {
    double span[3], c = ord_val(acc[6]);
    for (int d = 0; d < 3; ++d) {
        gp->o[d] = ord_val(acc[d]);
        span[d] = ord_val(acc[3 + d]) - gp->o[d];
    }
    const double smax = fmax(span[0], fmax(span[1], span[2]));
    if (!(c > 0.0)) c = smax > 0.0 ? smax * 1e-6 : 1.0;
    for (;;) {
        double prod = 1.0;
        for (int d = 0; d < 3; ++d) prod *= floor(span[d] / c) + 1.0;
        if (prod <= (double)max_cells) break;
        c *= 1.25;
    }
    gp->c = c;
    gp->ic = 1.0 / c;
    for (int d = 0; d < 3; ++d) gp->dims[d] = (int)(floor(span[d] / c) + 1.0);
}

// Stage 1 (many blocks): acc[0..2] = min lo, acc[3..5] = max hi, acc[6] = max extent (ordered keys).
// The last block to finish also derives the grid parameters (no second launch).
__global__ void grid_reduce_kernel(const double *__restrict__ lbox, int64_t L, unsigned long long *__restrict__ acc,
                                   unsigned *__restrict__ done, int64_t max_cells, GridParams *__restrict__ gp) {
    double v[7] = {CUDART_INF, CUDART_INF, CUDART_INF, -CUDART_INF, -CUDART_INF, -CUDART_INF, 0.0};
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L; l += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double lo = lbox[d * L + l], hi = lbox[(3 + d) * L + l];
            v[d] = fmin(v[d], lo);
            v[3 + d] = fmax(v[3 + d], hi);
            v[6] = fmax(v[6], hi - lo);
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            v[d] = fmin(v[d], __shfl_xor_sync(0xffffffffu, v[d], off));
            v[3 + d] = fmax(v[3 + d], __shfl_xor_sync(0xffffffffu, v[3 + d], off));
        }
        v[6] = fmax(v[6], __shfl_xor_sync(0xffffffffu, v[6], off));
    }
    if ((threadIdx.x & 31) == 0) {
        for (int d = 0; d < 3; ++d) {
            atomicMin(acc + d, ord_key(v[d]));
            atomicMax(acc + 3 + d, ord_key(v[3 + d]));
        }
        atomicMax(acc + 6, ord_key(v[6]));
    }
    __threadfence();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        unsigned long long a[7];
        for (int k = 0; k < 7; ++k) a[k] = atomicAdd(acc + k, 0ULL);   // L2-coherent reads
        grid_finalize(a, max_cells, gp);
        reset_grid_keys(acc);   // (and the block counter, acc[7]): ready for the next run
    }
}


// The fused path's loop half of derive with the grid reduction folded in:
// grid-stride warps per loop (loops of <= kLoopWarpMax segments) write the loop
// box and minimum squared diagonal; the loop boxes are reduced per block
// (ordered-key warp reductions, then shared memory) into the model box and the
// largest loop extent (one atomic set per block), and the last block derives
// the grid parameters — grid_reduce_kernel's outputs with no second pass.
#ifndef LC_LOOPGRID_WARPS
#define LC_LOOPGRID_WARPS 4   // loop-box kernel: warps per block (one loop per warp per step)
#endif
constexpr int kLgWarps = LC_LOOPGRID_WARPS;
template <bool POLY>
__global__ void __launch_bounds__(32 * kLgWarps) loop_grid_kernel(const double *__restrict__ coeffs, const double *__restrict__ t,
                                                        const double *__restrict__ verts,
                                                        const int64_t *__restrict__ loff, int64_t L,
                                                        unsigned long long *__restrict__ loop_min_diag2,
                                                        double *__restrict__ lbox, unsigned long long *__restrict__ acc,
                                                        unsigned *__restrict__ done, int64_t max_cells,
                                                        GridParams *__restrict__ gp, const ZeroList zl) {
    LC_PDL_TRIGGER();
    LC_PDL_WAIT();
    zero_ranges(zl);   // the run's initial values, read by the kernels after this one
    __shared__ unsigned long long sk[kLgWarps][7];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // block accumulators (ordered keys): min lo x3, max hi x3, max extent
    unsigned long long bk[7] = {~0ULL, ~0ULL, ~0ULL, 0ULL, 0ULL, 0ULL, 0ULL};
    const int64_t nw = (int64_t)gridDim.x * kLgWarps;
    for (int64_t l = (int64_t)blockIdx.x * kLgWarps + warp; l < L; l += nw) {
        const int64_t b = loff[l], e = loff[l + 1];
        double v[6] = {CUDART_INF, CUDART_INF, CUDART_INF, -CUDART_INF, -CUDART_INF, -CUDART_INF};
        unsigned long long dg = ~0ULL;
#pragma unroll 2
        for (int64_t m = b + lane; m < e; m += 32) {
            double bl[3], bh[3];
            if (POLY) {
                const int64_t nx = m + 1 < e ? m + 1 : b;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const double a0 = verts[3 * m + d], a1 = verts[3 * nx + d] - a0;
                    // eval_axis at t = 0 and 1 with a2 = a3 = 0, bitwise: a0 (+0 for -0) and a0 + a1 (+0 for -0)
                const double v0 = __dadd_rn(a0, 0.0), v1 = __dadd_rn(__dadd_rn(a0, a1), 0.0);
                    bl[d] = np_min(v0, v1);
                    bh[d] = np_max(v0, v1);
                }
            } else {
                tight_box(coeffs + 12 * m, t[2 * m], t[2 * m + 1], bl, bh);
            }
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                v[d] = np_min(v[d], bl[d]);
                v[3 + d] = np_max(v[3 + d], bh[d]);
            }
            const double dx = __dsub_rn(bh[0], bl[0]), dy = __dsub_rn(bh[1], bl[1]), dz = __dsub_rn(bh[2], bl[2]);
            const unsigned long long q = (unsigned long long)__double_as_longlong(
                __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
            dg = q < dg ? q : dg;
        }
        // loop box: ordered-key warp reductions (2 redux per value instead of 10 shuffles)
        unsigned long long k[6];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            k[d] = group_min_u64(0xffffffffu, ord_key(v[d]));
            k[3 + d] = group_max_u64(0xffffffffu, ord_key(v[3 + d]));
        }
        dg = group_min_u64(0xffffffffu, dg);
        if (lane == 0) {
            double ext = 0.0;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const double lo = ord_val(k[d]), hi = ord_val(k[3 + d]);
                lbox[d * L + l] = lo;
                lbox[(3 + d) * L + l] = hi;
                ext = fmax(ext, hi - lo);
                bk[d] = k[d] < bk[d] ? k[d] : bk[d];
                bk[3 + d] = k[3 + d] > bk[3 + d] ? k[3 + d] : bk[3 + d];
            }
            const unsigned long long ke = ord_key(ext);
            bk[6] = ke > bk[6] ? ke : bk[6];
            loop_min_diag2[l] = dg;
        }
    }
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 7; ++q) sk[warp][q] = bk[q];
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kLgWarps; ++w) {
            for (int q = 0; q < 3; ++q) bk[q] = sk[w][q] < bk[q] ? sk[w][q] : bk[q];
            for (int q = 3; q < 7; ++q) bk[q] = sk[w][q] > bk[q] ? sk[w][q] : bk[q];
        }
        for (int q = 0; q < 3; ++q) atomicMin(acc + q, bk[q]);
        for (int q = 3; q < 7; ++q) atomicMax(acc + q, bk[q]);
        __threadfence();
        const bool last = atomicAdd(done, 1u) == gridDim.x - 1;
        if (last) {
            __threadfence();
            unsigned long long a[7];
            for (int q = 0; q < 7; ++q) a[q] = atomicAdd(acc + q, 0ULL);   // L2-coherent reads
            grid_finalize(a, max_cells, gp);
            reset_grid_keys(acc);   // (and the block counter)
        }
    }
}

// Row i's slots sorted by j -> pairs[off[i] ...] (insertion sort, <= kRowSlots).
__global__ void slots_compact_kernel(const int *__restrict__ row_count, const int64_t *__restrict__ off, int64_t L,
                                     const int32_t *__restrict__ slots, int32_t *__restrict__ pairs, int64_t cap) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= L) return;
    const int n = row_count[i] < kRowSlots ? row_count[i] : kRowSlots;   // > kRowSlots: caller's fallback
    int32_t v[kRowSlots];
#pragma unroll
    for (int k = 0; k < kRowSlots; ++k) v[k] = k < n ? slots[i * kRowSlots + k] : INT_MAX;
#pragma unroll
    for (int a = 1; a < kRowSlots; ++a)
#pragma unroll
        for (int b = a; b > 0; --b)
            if (v[b] < v[b - 1]) {
                const int32_t t = v[b];
                v[b] = v[b - 1];
                v[b - 1] = t;
            }
    const int64_t o = off[i];
#pragma unroll
    for (int k = 0; k < kRowSlots; ++k)
        if (k < n && o + k < cap) {
            pairs[2 * (o + k)] = (int32_t)i;
            pairs[2 * (o + k) + 1] = v[k];
        }
}

// Fused path: compaction that also lays out the work items — PairGeom and the
// exclusive item offset of every pair — from the packed (items, pairs) row scan;
// the last row stores P and the item total (d_tot[0], d_tot[1]) and item_off[P].
__global__ void slots_compact_items_kernel(const int *__restrict__ row_count, const int64_t *__restrict__ offs,
                                           int64_t L, const int32_t *__restrict__ slots, int32_t *__restrict__ pairs,
                                           int64_t cap, const int64_t *__restrict__ loff, PairGeom *__restrict__ pg,
                                           int64_t *__restrict__ item_off, int64_t *__restrict__ d_tot,
                                           const int *__restrict__ overflow, int64_t item_cap) {
    LC_PDL_TRIGGER();
    LC_PDL_WAIT();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= L) return;
    const int64_t mask = (int64_t(1) << kPackShift) - 1;
    const int n = row_count[i] < kRowSlots ? row_count[i] : kRowSlots;
    int32_t v[kRowSlots];
#pragma unroll
    for (int k = 0; k < kRowSlots; ++k) v[k] = k < n ? slots[i * kRowSlots + k] : INT_MAX;
#pragma unroll
    for (int a = 1; a < kRowSlots; ++a)
#pragma unroll
        for (int b = a; b > 0; --b)
            if (v[b] < v[b - 1]) {
                const int32_t t = v[b];
                v[b] = v[b - 1];
                v[b - 1] = t;
            }
    const int64_t packed = offs[i], o = packed & mask;
    int64_t it = packed >> kPackShift;
    const int64_t ci = loff[i] + i;   // closed-vertex offset of loop i (vertex 0 repeated per loop)
    const int ncols = (int)(loff[i + 1] - loff[i]);
#pragma unroll
    for (int k = 0; k < kRowSlots; ++k)
        if (k < n) {
            const int32_t j = v[k];
            const PairGeom g = make_pair_geom(ci, loff[j] + j, ncols, (int)(loff[j + 1] - loff[j]));
            if (o + k < cap) {
                pairs[2 * (o + k)] = (int32_t)i;
                pairs[2 * (o + k) + 1] = j;
                pg[o + k] = g;
                item_off[o + k] = it;
            }
            it += (int64_t)g.items_r * g.items_c;
        }
    if (i == L - 1) {
        const int64_t tot = offs[L], P = tot & mask, items = tot >> kPackShift;
        // a run that cannot be the reference's (row slots overflowed, or more pairs /
        // items than the capacities) hands 0 pairs to everything downstream; the
        // status reports the real counts and the caller reruns on the staged path
        const bool usable = P <= cap && items <= item_cap && *overflow <= kRowSlots;
        d_tot[0] = usable ? P : 0;
        d_tot[1] = usable ? items : 0;
        d_tot[2] = P;
        d_tot[3] = items;
        if (usable) item_off[P] = items;
        else item_off[0] = 0;
    }
}

__global__ void unpack_pairs_kernel(const uint64_t *__restrict__ keys, int64_t P, int32_t *__restrict__ pairs) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    const uint64_t k = keys[p];
    pairs[2 * p] = (int32_t)(k >> 32);
    pairs[2 * p + 1] = (int32_t)(k & 0xffffffffu);
}

}  // namespace

bool seg_boxes_split_ok(int64_t L, int64_t max_loop_segments) {
    return L > 0 && max_loop_segments >= 0 && max_loop_segments <= kLoopWarpMax;
}

void launch_seg_boxes_split(const double *coeffs, const double *t, const double *verts, const int64_t *loff, int64_t L,
                            int64_t M, bool loop_part, double *seg_box, float *seg_fbox, int32_t *seg_loop,
                            int *max_exp, unsigned long long *loop_min_diag2, double *loop_box, cudaStream_t s,
                            float *seg_sub) {
    const unsigned blocks = (unsigned)ceil_div(L * 32, 128);
    if (loop_part) {
        if (verts)
            seg_boxes_loop_kernel<true, false, true><<<blocks, 128, 0, s>>>(nullptr, nullptr, verts, loff, L, M, nullptr,
                                                                            nullptr, nullptr, loop_min_diag2, loop_box,
                                                                            nullptr);
        else
            seg_boxes_loop_kernel<false, false, true><<<blocks, 128, 0, s>>>(coeffs, t, nullptr, loff, L, M, nullptr,
                                                                             nullptr, nullptr, loop_min_diag2, loop_box,
                                                                             nullptr);
    } else {
        if (verts)
            seg_boxes_loop_kernel<true, true, false><<<blocks, 128, 0, s>>>(nullptr, nullptr, verts, loff, L, M, seg_box,
                                                                            seg_fbox, seg_loop, nullptr, nullptr,
                                                                            max_exp, seg_fbox ? seg_sub : nullptr);
        else
            seg_boxes_loop_kernel<false, true, false><<<blocks, 128, 0, s>>>(coeffs, t, nullptr, loff, L, M, seg_box,
                                                                             seg_fbox, seg_loop, nullptr, nullptr,
                                                                             max_exp, seg_fbox ? seg_sub : nullptr);
    }
    LC_CHECK_LAUNCH();
}

void launch_seg_boxes(const double *coeffs, const double *t, const double *verts, const int64_t *loff, int64_t L,
                      int64_t M, double *seg_box, int32_t *seg_loop, unsigned long long *loop_min_diag2, int *max_exp,
                      cudaStream_t s, float *seg_fbox, unsigned long long *loop_keys, double *loop_box,
                      int64_t max_loop_segments) {
    if (loop_box && L > 0 && max_loop_segments >= 0 && max_loop_segments <= kLoopWarpMax) {
        if (max_exp) LC_CUDA(cudaMemsetAsync(max_exp, 0, sizeof(int), s));
        const unsigned blocks = (unsigned)ceil_div(L * 32, 128);
        if (verts)
            seg_boxes_loop_kernel<true><<<blocks, 128, 0, s>>>(nullptr, nullptr, verts, loff, L, M, seg_box, seg_fbox,
                                                               seg_loop, loop_min_diag2, loop_box, max_exp);
        else
            seg_boxes_loop_kernel<false><<<blocks, 128, 0, s>>>(coeffs, t, nullptr, loff, L, M, seg_box, seg_fbox,
                                                                seg_loop, loop_min_diag2, loop_box, max_exp);
        LC_CHECK_LAUNCH();
        return;
    }
    if (loop_min_diag2)
        LC_CUDA(cudaMemsetAsync(loop_min_diag2, 0xff, sizeof(unsigned long long) * (L > 0 ? L : 1), s));
    if (max_exp) LC_CUDA(cudaMemsetAsync(max_exp, 0, sizeof(int), s));
    if (loop_keys && L > 0) {
        LC_CUDA(cudaMemsetAsync(loop_keys, 0xff, sizeof(unsigned long long) * 3 * L, s));
        LC_CUDA(cudaMemsetAsync(loop_keys + 3 * L, 0, sizeof(unsigned long long) * 3 * L, s));
    }
    if (M > 0) {
        if (verts)
            seg_boxes_kernel<true><<<(unsigned)ceil_div(M, 128), 128, 0, s>>>(
                nullptr, nullptr, verts, loff, L, M, seg_box, seg_fbox, seg_loop, loop_min_diag2, loop_keys, max_exp);
        else
            seg_boxes_kernel<false><<<(unsigned)ceil_div(M, 128), 128, 0, s>>>(
                coeffs, t, nullptr, loff, L, M, seg_box, seg_fbox, seg_loop, loop_min_diag2, loop_keys, max_exp);
        LC_CHECK_LAUNCH();
    }
    if (loop_keys && loop_box && L > 0) {
        loop_keys_decode_kernel<<<(unsigned)ceil_div(L, 256), 256, 0, s>>>(loop_keys, L, loop_box);
        LC_CHECK_LAUNCH();
    }
}


namespace {
__global__ void prezero_kernel(ZeroList zl) {
    LC_PDL_TRIGGER();
    zero_ranges(zl);
}
}  // namespace

int64_t pls_grid_max_cells(int64_t L) {
    return 32 * L + 64;   // cells ~ the largest loop extent for surface-like models (tube: 7x fewer candidates than 4L)
}

void reserve_pls_grid(int64_t L, PlsScratch &sc, cudaStream_t s) {
    const int64_t max_cells = pls_grid_max_cells(L);
    sc.keys.reserve(sizeof(int64_t) * (max_cells + 1), s);
    sc.counter.reserve(sizeof(unsigned long long), s);
    sc.counts.reserve(sizeof(int64_t) * (L + 8 > 8 ? L + 8 : 8), s);
    sc.acc.reserve(8 * sizeof(unsigned long long), s);
    if (sc.acc.ptr != sc.acc_ready) {   // a new buffer: the reductions' keys at the identity, once
        unsigned long long *acc = sc.acc.as<unsigned long long>();
        LC_CUDA(cudaMemsetAsync(acc, 0xff, 3 * sizeof(unsigned long long), s));
        LC_CUDA(cudaMemsetAsync(acc + 3, 0, 5 * sizeof(unsigned long long), s));
        sc.acc_ready = sc.acc.ptr;
    }
}

namespace {
// grid_prefix's memsets (cell counts, largest row count) + the caller's ranges
ZeroList grid_zero_list(int64_t L, PlsScratch &sc, const ZeroRange *extra, int n_extra) {
    const int64_t max_cells = pls_grid_max_cells(L);
    if (n_extra < 0 || n_extra > kMaxZeroRanges - 2) throw Error(LC_ERR_ARG, "too many prezero ranges");
    ZeroList zl{};
    zl.r[0] = ZeroRange{sc.keys.ptr, 2 * (max_cells + 1), 0u};
    zl.r[1] = ZeroRange{sc.counter.ptr, 1, 0u};
    zl.n = 2;
    for (int k = 0; k < n_extra; ++k) zl.r[zl.n++] = extra[k];
    return zl;
}
}  // namespace

void launch_grid_prezero(int64_t L, PlsScratch &sc, const ZeroRange *extra, int n_extra, cudaStream_t s) {
    reserve_pls_grid(L, sc, s);
    prezero_kernel<<<2 * 148, 256, 0, s>>>(grid_zero_list(L, sc, extra, n_extra));
    LC_CHECK_LAUNCH();
}

// Grid culling up to the per-row pair counts and their exclusive scan (no
// host sync): sc.offs[L] = P, *sc.counter = largest row count, slots in
// sc.pair_keys, row counts in sc.idx.  Excluded keys already in sc.excl.
static void grid_prefix(const double *loop_box, int64_t L, int64_t n_excl, PlsScratch &sc, cudaStream_t s,
                        const int64_t *item_loff = nullptr, bool prezeroed = false, bool grid_ready = false,
                        bool pdl = false) {
    const int64_t max_cells = pls_grid_max_cells(L);
    sc.axis.reserve(sizeof(GridParams), s);
    sc.keys.reserve(sizeof(int64_t) * (max_cells + 1), s);         // cell counts
    sc.keys_sorted.reserve(sizeof(int64_t) * (max_cells + 1), s);  // cell offsets
    sc.sbox.reserve(sizeof(double) * 6 * L, s);                      // loop boxes in cell order
    sc.lcell.reserve(sizeof(int32_t) * L, s);
    sc.lrank.reserve(sizeof(int32_t) * L, s);
    sc.perm.reserve(sizeof(int32_t) * L, s);                       // loops in cell order
    sc.idx.reserve(sizeof(int) * L, s);                            // row counts
    sc.pair_keys.reserve(sizeof(int32_t) * kRowSlots * L, s);      // slots
    sc.counts.reserve(sizeof(int64_t) * (L + 1), s);
    sc.offs.reserve(sizeof(int64_t) * (L + 1), s);
    sc.counter.reserve(sizeof(unsigned long long), s);
    GridParams *gp = sc.axis.as<GridParams>();
    int64_t *cnt = sc.keys.as<int64_t>(), *coff = sc.keys_sorted.as<int64_t>();
    int *row_count = sc.idx.as<int>(), *max_count = sc.counter.as<int>();
    sc.counts.reserve(sizeof(int64_t) * (L + 8 > 8 ? L + 8 : 8), s);
    reserve_pls_grid(L, sc, s);
    unsigned long long *acc = sc.acc.as<unsigned long long>();   // 7 ordered keys + block counter, at the identity
    if (!grid_ready) {   // else loop_grid_kernel derived the grid parameters with the loop boxes
        grid_reduce_kernel<<<(unsigned)(ceil_div(L, 256) < 148 ? ceil_div(L, 256) : 148), 256, 0, s>>>(
            loop_box, L, acc, reinterpret_cast<unsigned *>(acc + 7), max_cells, gp);
        LC_CHECK_LAUNCH();
        tl_mark("grid_reduce", s);
    }
    if (!prezeroed) LC_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (max_cells + 1), s));
    // thread-per-loop kernels in 64-thread blocks: the latency chains spread over every SM
    const unsigned gl = (unsigned)ceil_div(L, 64);
    launch_pdl(cell_count_kernel, gl, 64, s, pdl, loop_box, L, gp, cnt, sc.lcell.as<int32_t>(), sc.lrank.as<int32_t>());
    tl_mark("cell_count", s);
    const size_t b = exclusive_scan_i64_tmp_bytes(max_cells + 1), b2 = exclusive_scan_i64_tmp_bytes(L + 1);
    sc.cub_tmp.reserve((b > b2 ? b : b2) + 16, s);
    exclusive_scan_i64(cnt, coff, max_cells + 1, sc.cub_tmp.ptr, sc.cub_tmp.bytes, s);
    tl_mark("cell_scan", s);
    launch_pdl(cell_scatter_kernel, gl, 64, s, pdl, loop_box, L, coff, sc.lcell.as<int32_t>(),
               sc.lrank.as<int32_t>(), sc.perm.as<int32_t>(), sc.sbox.as<double>());
    tl_mark("cell_scatter", s);
    if (!prezeroed) LC_CUDA(cudaMemsetAsync(max_count, 0, sizeof(int), s));
    launch_pdl(grid_query_warp_kernel<true>, (unsigned)ceil_div(L * 32, 256), 256, s, pdl, loop_box, L, gp, coff,
               sc.perm.as<int32_t>(), sc.sbox.as<double>(), sc.excl.as<uint64_t>(), n_excl, row_count,
               sc.pair_keys.as<int32_t>(), nullptr, nullptr, sc.counts.as<int64_t>(), max_count, item_loff);
    tl_mark("query", s);
    // (a single-block scan measured 14 us here vs 8.4 us for DeviceScan's init + scan)
    exclusive_scan_i64(sc.counts.as<int64_t>(), sc.offs.as<int64_t>(), L + 1, sc.cub_tmp.ptr, sc.cub_tmp.bytes, s);
    tl_mark("row_scan", s);
}

int64_t run_pls(const double *loop_box, int64_t L, const uint64_t *h_excl, int64_t n_excl, PlsScratch &sc,
                DevBuf &pairs, cudaStream_t s, bool force_sweep) {
    if (L < 2) return 0;
    sc.excl.reserve(sizeof(uint64_t) * (n_excl > 0 ? n_excl : 1), s);
    if (n_excl > 0)
        LC_CUDA(cudaMemcpyAsync(sc.excl.ptr, h_excl, sizeof(uint64_t) * n_excl, cudaMemcpyHostToDevice, s));
    if (!force_sweep) {
        grid_prefix(loop_box, L, n_excl, sc, s);
        const unsigned gl = (unsigned)ceil_div(L, 256);
        int *row_count = sc.idx.as<int>(), *max_count = sc.counter.as<int>();
        const int64_t *coff = sc.keys_sorted.as<int64_t>();
        const GridParams *gp = sc.axis.as<GridParams>();
        int64_t P = 0;
        int mx = 0;
        LC_CUDA(cudaMemcpyAsync(&P, sc.offs.as<int64_t>() + L, sizeof P, cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaMemcpyAsync(&mx, max_count, sizeof mx, cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaStreamSynchronize(s));
        if (P == 0) return 0;
        pairs.reserve(sizeof(int32_t) * 2 * P, s);
        if (mx <= kRowSlots) {
            slots_compact_kernel<<<gl, 256, 0, s>>>(row_count, sc.offs.as<int64_t>(), L, sc.pair_keys.as<int32_t>(),
                                                     pairs.as<int32_t>(), INT64_MAX);
            LC_CHECK_LAUNCH();
            return P;
        }
        // some loop overlaps more than kRowSlots later loops: write keys at exact offsets, sort
        sc.pair_keys.reserve(sizeof(uint64_t) * P, s);
        sc.pair_keys_sorted.reserve(sizeof(uint64_t) * P, s);
        grid_query_warp_kernel<false><<<(unsigned)ceil_div(L * 32, 256), 256, 0, s>>>(loop_box, L, gp, coff, sc.perm.as<int32_t>(),
                                                    sc.sbox.as<double>(), sc.excl.as<uint64_t>(), n_excl, nullptr, nullptr,
                                                    sc.offs.as<int64_t>(), sc.pair_keys.as<uint64_t>(), nullptr,
                                                    nullptr, nullptr);
        LC_CHECK_LAUNCH();
        size_t b3 = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, b3, (uint64_t *)nullptr, (uint64_t *)nullptr, (int)P);
        sc.cub_tmp.reserve(b3, s);
        b3 = sc.cub_tmp.bytes;
        LC_CUB(cub::DeviceRadixSort::SortKeys(sc.cub_tmp.ptr, b3, sc.pair_keys.as<uint64_t>(),
                                              sc.pair_keys_sorted.as<uint64_t>(), (int)P, 0, 64, s));
        unpack_pairs_kernel<<<(unsigned)ceil_div(P, 256), 256, 0, s>>>(sc.pair_keys_sorted.as<uint64_t>(), P,
                                                                        pairs.as<int32_t>());
        LC_CHECK_LAUNCH();
        return P;
    }
    // sort-and-sweep on the axis of largest extent (LINKCERT_PLS_SWEEP=1)
    sc.keys.reserve(sizeof(double) * L, s);
    sc.keys_sorted.reserve(sizeof(double) * L, s);
    sc.idx.reserve(sizeof(int32_t) * L, s);
    sc.perm.reserve(sizeof(int32_t) * L, s);
    sc.sbox.reserve(sizeof(double) * 6 * L, s);
    sc.axis.reserve(sizeof(int), s);
    sc.counter.reserve(sizeof(unsigned long long), s);

    sweep_axis_kernel<<<1, 1024, 0, s>>>(loop_box, L, sc.axis.as<int>(), sc.keys.as<double>(), sc.idx.as<int32_t>());
    LC_CHECK_LAUNCH();
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (double *)nullptr, (double *)nullptr, (int32_t *)nullptr,
                                    (int32_t *)nullptr, (int)L);
    sc.cub_tmp.reserve(bytes, s);
    bytes = sc.cub_tmp.bytes;
    LC_CUB(cub::DeviceRadixSort::SortPairs(sc.cub_tmp.ptr, bytes, sc.keys.as<double>(), sc.keys_sorted.as<double>(),
                                           sc.idx.as<int32_t>(), sc.perm.as<int32_t>(), (int)L, 0, 64, s));
    gather_boxes_kernel<<<(unsigned)ceil_div(L, 256), 256, 0, s>>>(loop_box, sc.perm.as<int32_t>(), L,
                                                                    sc.sbox.as<double>());
    LC_CHECK_LAUNCH();

    int64_t cap = sc.cap > 0 ? sc.cap : 16 * L + 1024;
    unsigned long long P = 0;
    for (;;) {
        sc.pair_keys.reserve(sizeof(uint64_t) * cap, s);
        LC_CUDA(cudaMemsetAsync(sc.counter.ptr, 0, sizeof(unsigned long long), s));
        const int64_t warps = L < 148 * 64 ? L : 148 * 64;
        sweep_warp_kernel<<<(unsigned)ceil_div(warps * 32, 256), 256, 0, s>>>(
            sc.sbox.as<double>(), sc.perm.as<int32_t>(), L, sc.axis.as<int>(), sc.excl.as<uint64_t>(), n_excl,
            sc.counter.as<unsigned long long>(), sc.pair_keys.as<uint64_t>(), cap);
        LC_CHECK_LAUNCH();
        LC_CUDA(cudaMemcpyAsync(&P, sc.counter.ptr, sizeof P, cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaStreamSynchronize(s));
        if ((int64_t)P <= cap) break;
        cap = (int64_t)P + P / 4 + 1024;   // rare: grow and sweep again
    }
    sc.cap = cap;
    if (P == 0) return 0;
    sc.pair_keys_sorted.reserve(sizeof(uint64_t) * P, s);
    size_t b3 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b3, (uint64_t *)nullptr, (uint64_t *)nullptr, (int)P);
    sc.cub_tmp.reserve(b3, s);
    bytes = sc.cub_tmp.bytes;
    LC_CUB(cub::DeviceRadixSort::SortKeys(sc.cub_tmp.ptr, bytes, sc.pair_keys.as<uint64_t>(),
                                          sc.pair_keys_sorted.as<uint64_t>(), (int)P, 0, 64, s));
    pairs.reserve(sizeof(int32_t) * 2 * P, s);
    unpack_pairs_kernel<<<(unsigned)ceil_div((int64_t)P, 256), 256, 0, s>>>(sc.pair_keys_sorted.as<uint64_t>(),
                                                                              (int64_t)P, pairs.as<int32_t>());
    LC_CHECK_LAUNCH();
    return (int64_t)P;
}

#ifndef LC_LOOPGRID_BPS
#define LC_LOOPGRID_BPS 6   // loop-box kernel: blocks per SM cap (4 warps each, grid-stride over loops)
#endif
void launch_loop_grid(const double *coeffs, const double *t, const double *verts, const int64_t *loff, int64_t L,
                      unsigned long long *loop_min_diag2, double *loop_box, PlsScratch &sc, cudaStream_t s,
                      bool pdl, const ZeroRange *extra, int n_extra) {
    const int64_t max_cells = pls_grid_max_cells(L);
    sc.axis.reserve(sizeof(GridParams), s);
    reserve_pls_grid(L, sc, s);
    unsigned long long *acc = sc.acc.as<unsigned long long>();   // keys + block counter, at the identity
    const ZeroList zl = grid_zero_list(L, sc, extra, n_extra);
    int64_t blocks = ceil_div(L, kLgWarps);
    if (blocks > 148 * LC_LOOPGRID_BPS) blocks = 148 * LC_LOOPGRID_BPS;
    if (verts)
        launch_pdl(loop_grid_kernel<true>, (unsigned)blocks, 32 * kLgWarps, s, pdl, (const double *)nullptr,
                   (const double *)nullptr, verts, loff, L, loop_min_diag2, loop_box, acc,
                   reinterpret_cast<unsigned *>(acc + 7), max_cells, sc.axis.as<GridParams>(), zl);
    else
        launch_pdl(loop_grid_kernel<false>, (unsigned)blocks, 32 * kLgWarps, s, pdl, coeffs, t, (const double *)nullptr, loff, L,
                   loop_min_diag2, loop_box, acc, reinterpret_cast<unsigned *>(acc + 7), max_cells,
                   sc.axis.as<GridParams>(), zl);
}

void launch_pls_grid(const double *loop_box, int64_t L, int64_t n_excl, PlsScratch &sc, int32_t *pairs, int64_t cap,
                     const int64_t *loff, PairGeom *pg, int64_t *item_off, int64_t *d_tot, int64_t item_cap,
                     cudaStream_t s, const int **d_max_row, bool prezeroed, bool grid_ready, bool pdl) {
    grid_prefix(loop_box, L, n_excl, sc, s, loff, prezeroed, grid_ready, pdl);
    launch_pdl(slots_compact_items_kernel, (unsigned)ceil_div(L, 64), 64, s, pdl, sc.idx.as<int>(),
               sc.offs.as<int64_t>(), L, sc.pair_keys.as<int32_t>(), pairs, cap, loff, pg, item_off, d_tot,
               sc.counter.as<int>(), item_cap);
    *d_max_row = sc.counter.as<int>();
}

}  // namespace lc
