// Gauss-sum work-item layer: declarations shared by gauss.cu and abi.cu.
#pragma once
#include "common.cuh"

namespace lc {

// Arithmetic variants of the per-lane strip evaluation (all FP64):
//   GAUSS_PHASE : default. Arai terms with corner vectors/norms/edge dots shared
//                 between neighbouring segment pairs, and the per-pair angles
//                 atan2(p,d1)+atan2(p,d2) accumulated as an exact-turn-counted
//                 complex phase product (one atan2 per lane strip).
//   GAUSS_ATAN  : same sharing, one fused atan2 per segment pair with the
//                 exact full-turn correction (direct.py:120-123 rule).
//   GAUSS_REF   : the reference formula evaluated per pair from scratch with
//                 no FMA contraction and two atan2 (direct.py:19-46); used to
//                 freeze F_pair and as a numerics cross-check.
//   GAUSS_ANGLESUM : the reference's "anglesum" variant (_link_angle_sum,
//                 direct.py:75-134): one lane per outer segment walks every
//                 inner segment in order, accumulating the normalized phase
//                 product with its half-plane crossing counts, one atan2 per
//                 outer segment; reference operation order, no contraction.
//   16..20      : A/B builds of the phase kernel (occupancy / shared-memory
//                 variants; tools/kbench.py), not part of the ABI.
enum GaussMode : int { GAUSS_PHASE = 0, GAUSS_ATAN = 1, GAUSS_REF = 2, GAUSS_ANGLESUM = 3, GAUSS_AB_FIRST = 16,
                       GAUSS_AB_LAST = 20 };

inline bool gauss_mode_valid(int mode) {
    return (mode >= GAUSS_PHASE && mode <= GAUSS_ANGLESUM) || (mode >= GAUSS_AB_FIRST && mode <= GAUSS_AB_LAST);
}
// Modes whose work items are whole outer segments (32 per item, all inner segments in order).
inline bool gauss_mode_sequential(int mode) { return mode == GAUSS_ANGLESUM; }

#ifndef LC_ROWS
#define LC_ROWS 4
#endif
constexpr int kRowsPerLane = LC_ROWS;   // outer-loop (k) segments held per lane (A/B builds: -DLC_ROWS=n)
constexpr int kMaxColsPerLane = 2048;

// Per loop-pair tiling, built on the device from the pair list.
struct PairGeom {
    int64_t row_off;   // first vertex of the row loop (loop j of pair (i,j): "k")
    int64_t col_off;   // first vertex of the column loop (loop i: "l")
    int32_t nrows;     // segments of the row loop
    int32_t ncols;     // segments of the column loop
    int32_t rb_log2;   // lanes of one item split as (1<<rb_log2) row blocks x (32>>rb_log2) column strips
    int32_t cl;        // columns per lane strip
    int32_t items_r;   // item grid of this pair
    int32_t items_c;
};

// One work item, self-contained: the pair's tiling and the item's place in it
// (the Gauss kernel's item prologue is one 48-byte load after the claim).
struct ItemRec {
    PairGeom g;
    int32_t ir, ic;   // row-block group and column-strip group of the item
};

// Tiling of pair (column loop i, row loop j) from the two loops' closed-vertex
// offsets and segment counts (one definition for every path that builds items).
// seq: items of the sequential (anglesum) modes — 32 whole rows per item, one per lane.
// max_cl: a smaller column-strip cap for a lone pair (more, shorter items: link_direct).
__host__ __device__ inline PairGeom make_pair_geom(int64_t col_off, int64_t row_off, int ncols, int nrows,
                                                   bool seq = false, int max_cl = kMaxColsPerLane) {
    PairGeom g;
    g.col_off = col_off;
    g.row_off = row_off;
    g.ncols = ncols;
    g.nrows = nrows;
    if (seq) {
        g.rb_log2 = 5;
        g.cl = ncols > 0 ? ncols : 1;
        g.items_r = (nrows + 31) / 32;
        g.items_c = 1;
        if (nrows <= 0 || ncols <= 0) g.items_r = g.items_c = 0;
        return g;
    }
    const int nb = (nrows + kRowsPerLane - 1) / kRowsPerLane;
    int rbl = 0;
    while ((1 << rbl) < nb && rbl < 5) ++rbl;
    g.rb_log2 = rbl;
    const int cs = 32 >> rbl;
    const int cl = (ncols + cs - 1) / cs;
    g.cl = cl < max_cl ? (cl > 0 ? cl : 1) : max_cl;
    g.items_r = (nrows + (kRowsPerLane << rbl) - 1) / (kRowsPerLane << rbl);
    const int64_t span = (int64_t)cs * g.cl;
    g.items_c = (int)((ncols + span - 1) / span);
    if (nrows <= 0 || ncols <= 0) g.items_r = g.items_c = 0;
    return g;
}

// Builds PairGeom[P] and item_off[P+1] (exclusive prefix of items per pair).
// voff: closed-loop SoA vertex offsets (L+1). Returns total item count (syncs).
// d_P (fused path): P is the capacity, the device count *d_P <= P is used and
// capacity slots past it get no items (item_off[P] is still the total).
int64_t build_items(const int32_t *d_pairs, int64_t P, const int64_t *d_voff, PairGeom *d_pg,
                    int64_t *d_item_off, void *d_scan_tmp, size_t scan_tmp_bytes, cudaStream_t s,
                    bool read_back = true, const int64_t *d_P = nullptr, bool seq = false,
                    int max_cl = kMaxColsPerLane);
size_t build_items_scan_bytes(int64_t P);

// Evaluates items [item_begin, item_end) into partials[item] (absolute index).
// d_end (fused path): the item count n on the device bounds the range.
// d_bounds (sharded fused path): the kernel takes items [d_bounds[shard], d_bounds[shard+1])
// instead (launch_shard_bounds).  abort (fused path): polled per item; nonzero
// stops the sum (the run is redone).
void launch_gauss_items(int mode, const double *X, const double *Y, const double *Z, const ItemRec *items,
                        int64_t item_begin, int64_t item_end, unsigned long long *counter,
                        double *partials, cudaStream_t s, const int64_t *d_end = nullptr, int shard = 0,
                        int shards = 1, const int *abort = nullptr, bool counter_zeroed = false,
                        const int64_t *d_bounds = nullptr);

// Fused path: warps claim whole pairs [0, *d_P) (or [d_bounds[shard], d_bounds[shard+1]) of a
// cost-balanced pair split) and evaluate each pair's items in order; raw is bitwise the
// item path's per-pair sum.  partials == null: raw / lk / flags written to the device
// arrays and to the pinned host arrays; else raw to partials[p] (the sharded exchange).
// Device early exit of verify(early_exit=True) (certify.py:195-216): the pairs are
// evaluated against the reference certificate in the reference's ordering
// (reference pairs in key order, then the other candidates in key order);
// posv[p] is pair p's place in that order (an order-preserving value), want[p] the
// certificate's value (0 if absent).  *first_fail = smallest place whose value
// differs; a pair whose place is past it is skipped (cancelled).
struct EarlyExitArgs {
    const int64_t *posv = nullptr;
    const int64_t *want = nullptr;
    unsigned long long *first_fail = nullptr;
    unsigned long long *n_eval = nullptr;
};
void launch_gauss_pairs(int mode, const double *X, const double *Y, const double *Z, const PairGeom *pg,
                        const int64_t *d_P, int64_t pcap, unsigned long long *counter, const int *abort,
                        const int64_t *d_bounds, int shard, double *partials, double *raw, int64_t *lk, uint8_t *flags,
                        double *h_raw, int64_t *h_lk, uint8_t *h_flags, cudaStream_t s,
                        const EarlyExitArgs &ee = EarlyExitArgs(), bool pdl = false);
// Early-exit preparation after the PLS: posv / want of every candidate pair (binary
// search of its key in the certificate) and *first_fail lowered to the place of every
// certificate pair that is no longer a candidate (its value is 0 there: a failure).
void launch_early_exit_order(const int32_t *pairs, const int64_t *d_P, int64_t pcap, const uint64_t *ref_keys,
                             const int64_t *ref_lk, int64_t n_ref, int64_t *posv, int64_t *want,
                             unsigned long long *first_fail, cudaStream_t s);

// Cost-balanced shard boundaries of the item list (item_off null: of the pair list): bounds[0..shards] (device),
// shard r owns items [bounds[r], bounds[r+1]); each shard's segment-pair cost is
// within one item of total / shards.  d_P: device pair count (<= Pcap) or null.
void launch_shard_bounds(const PairGeom *pg, const int64_t *item_off, int64_t Pcap, const int64_t *d_P, int shards,
                         int64_t *bounds, cudaStream_t s,
                         bool seq = false);

// items[it] = the record of work item `it` (pair tiling + the item's place in it).
void launch_item_pairs(const int64_t *item_off, const PairGeom *pg, int64_t P, int64_t n_items, ItemRec *items,
                       cudaStream_t s);
// Fused path: pair count on the device, item_pair capacity cap_items.
void launch_item_pairs_dev(const int64_t *item_off, const PairGeom *pg, int64_t P_cap, const int64_t *d_P,
                           int64_t cap_items, ItemRec *items, cudaStream_t s);

// raw[p] = fixed-order sum of the pair's item partials; lk = rint(raw);
// flags bit0 = NaN, bit1 = |raw - rint(raw)| > 0.25 (kernels.py:19-20,69-72).
void launch_reduce_pairs(const double *partials, const int64_t *item_off, int64_t P, double *raw,
                         int64_t *lk, uint8_t *flags, cudaStream_t s, const int64_t *d_P = nullptr);

#ifdef __CUDACC__
// One warp: the fixed-order sum of items [b, e) (lane-strided partial sums, then
// the xor butterfly) -- every reduction of pair sums goes through this, so the
// staged, fused and sharded paths agree bitwise.  All lanes return the sum.
__device__ __forceinline__ double warp_pair_sum(const double *__restrict__ partials, int64_t b, int64_t e, int lane) {
    double s = 0.0;
    for (int64_t k = b + lane; k < e; k += 32) s += partials[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    return s;
}

// lk = rint(raw) (half-to-even, like Python round()); flags bit0 = NaN, bit1 =
// |raw - rint(raw)| > 0.25 (kernels.py:19-20,69-72).
__device__ __forceinline__ uint8_t round_link(double s, int64_t &lk) {
    if (isnan(s)) {
        lk = 0;
        return 1;
    }
    const double rr = rint(s);
    lk = (int64_t)rr;
    return fabs(s - rr) > 0.25 ? 2 : 0;
}
#endif

// Writes the closed SoA vertex arrays scaled by an exact power of two from
// an AoS (n,3) buffer with per-loop offsets (no closing vertex in the input).
void launch_pack_closed_soa(const double *aos, const int64_t *in_off, const int64_t *voff, int64_t L,
                            int64_t total_closed, const int *d_exp, double *X, double *Y, double *Z,
                            cudaStream_t s);

// d_exp <- biased exponent field of max |aos[k]| over n doubles (atomicMax;
// caller zeroes d_exp first).  The pack kernel scales by 2^-(field-1023).
void launch_max_exponent(const double *aos, int64_t n, int *d_exp, cudaStream_t s);

// out[k] = reference _pair_lambda of quads[k] = (l_j, l_j1, k_i, k_i1), 12 doubles each.
void launch_segment_pairs(const double *quads, int64_t n, double *out, cudaStream_t s);

int num_sms();

}  // namespace lc
