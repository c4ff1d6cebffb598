// Potential link search on the device (replaces linkcert/pls.py:48-73 and
// the bvh.overlap_pairs_boxes broad phase it calls, bvh.py:227-243).
#pragma once
#include "common.cuh"

namespace lc {

// Boxes are SoA: box[0*n..] lo_x, [1*n] lo_y, [2*n] lo_z, [3*n] hi_x, [4*n] hi_y, [5*n] hi_z.

// Per-segment tight boxes over each segment's own domain (geometry.py:113-152);
// seg_loop[m] = loop of segment m.  Optional outputs: loop_min_diag2[l] =
// bit pattern of the smallest squared segment-box diagonal of loop l (its
// sqrt is the ZeroLengthInput diagonal, discretize.py:124-129); *max_exp =
// largest exponent field of any box coordinate (the exact power-of-two scale
// of the Gauss-sum input); seg_fbox = the boxes rounded outward to float (SoA
// 6 x M, the discretization's prefilter copy); loop_keys (6 x L scratch) +
// loop_box: the loop AABBs (pls.py:48-56) reduced in the same pass.
// verts != nullptr: closed polylines given by their vertices (M,3) instead of
// coeffs/t (the from_polyline arrays are formed in registers).
// max_loop_segments (host-known, >= 0) <= 1024 with loop_box: warp-per-loop
// variant (no loop lookup, no keys); otherwise thread per segment + keys.
// The fused path's derive in two halves on two streams (loops of <= 1024 segments):
// loop_part = loop boxes + minimum squared diagonals; otherwise the segment
// boxes, float boxes, segment loops and the coordinate exponent (max_exp zeroed
// by the caller), and with seg_sub the float boxes of 8-segment groups (the
// pass-1 check's first level; layout: pass1_group_slot).
// Float boxes of 8-segment groups, SoA 6 x pass1_group_stride(M, L): the group of
// loop l starting at segment m (m - loff[l] a multiple of 8) sits at slot m / 8 + l —
// consecutive within a loop, and distinct across loops (a loop adds at most one
// partial 8-block).
__host__ __device__ inline int64_t pass1_group_slot(int64_t m, int64_t l) { return (m >> 3) + l; }
__host__ __device__ inline int64_t pass1_group_stride(int64_t M, int64_t L) { return (M >> 3) + L + 1; }
bool seg_boxes_split_ok(int64_t L, int64_t max_loop_segments);
void launch_seg_boxes_split(const double *coeffs, const double *t, const double *verts, const int64_t *loff, int64_t L,
                            int64_t M, bool loop_part, double *seg_box, float *seg_fbox, int32_t *seg_loop,
                            int *max_exp, unsigned long long *loop_min_diag2, double *loop_box, cudaStream_t s,
                            float *seg_sub = nullptr);
void launch_seg_boxes(const double *coeffs, const double *t, const double *verts, const int64_t *loff, int64_t L,
                      int64_t M, double *seg_box, int32_t *seg_loop, unsigned long long *loop_min_diag2, int *max_exp,
                      cudaStream_t s, float *seg_fbox = nullptr, unsigned long long *loop_keys = nullptr,
                      double *loop_box = nullptr, int64_t max_loop_segments = -1);


struct PlsScratch {
    DevBuf keys, keys_sorted, idx, perm, sbox, counter, cub_tmp, pair_keys, pair_keys_sorted, axis, excl, counts,
        offs, lcell, lrank, acc;
    const void *acc_ready = nullptr;   // the acc buffer whose keys were set to the identity
    int64_t cap = 0;
};

// All (i<j) loop pairs with overlapping closed boxes (bvh.py:93-98) minus the
// excluded keys (sorted uint64 (i<<32|j)), sorted lexicographically.
// Default: exact uniform-grid culling (cells >= the largest loop extent, each
// loop stored in the cell of its lower corner, pairs emitted from the
// smaller index into per-row slots sorted at compaction — no global sort).
// force_sweep: sort-and-sweep on the axis of largest extent + radix sort.
// Writes int32 (P,2) into *pairs (grown as needed) and returns P (one sync).
int64_t run_pls(const double *loop_box, int64_t L, const uint64_t *h_excl, int64_t n_excl, PlsScratch &sc,
                DevBuf &pairs, cudaStream_t s, bool force_sweep = false);

// Grid-culling PLS without any host sync (the fused pipeline), which also lays
// out the Gauss-sum work items of the no-refinement case (chords = segment
// start points, so a pair's tiling follows from the loops' segment counts):
// the excluded keys must already be in sc.excl (n_excl of them); pairs go to
// `pairs` (capacity cap), PairGeom to pg, exclusive item offsets to item_off
// (item_off[P] = total), d_tot[0] = P and d_tot[1] = item total on the device
// — both 0 when the run cannot be exact (row overflow, P > cap, items >
// item_cap: nothing downstream then reads past the capacities) — and
// d_tot[2], d_tot[3] = the real P and item total for the status.
// *d_max_row -> device flag > kRowSlots when some row overflowed its slots
// (then the result is not exact and the caller falls back).  Needs 16 L < 2^24.
constexpr int kRowSlots = 16;
struct PairGeom;
void launch_pls_grid(const double *loop_box, int64_t L, int64_t n_excl, PlsScratch &sc, int32_t *pairs, int64_t cap,
                     const int64_t *loff, PairGeom *pg, int64_t *item_off, int64_t *d_tot, int64_t item_cap,
                     cudaStream_t s, const int **d_max_row, bool prezeroed = false, bool grid_ready = false,
                     bool pdl = false);
// Fused path: loop boxes + minimum squared diagonals with the grid reduction folded
// in (launch_pls_grid(..., grid_ready = true) then skips its reduction), loops of
// <= 1024 segments.  As the run's first kernel it also writes launch_grid_prezero's
// initial values (the grid PLS's and the caller's `extra` ranges; the reduction
// keys stay at the identity between runs).
struct ZeroRange;
void launch_loop_grid(const double *coeffs, const double *t, const double *verts, const int64_t *loff, int64_t L,
                      unsigned long long *loop_min_diag2, double *loop_box, PlsScratch &sc, cudaStream_t s,
                      bool pdl, const ZeroRange *extra, int n_extra);

// Scratch sizes of launch_pls_grid, and one kernel doing the memsets it issues
// (grid-reduce keys, cell counts, largest row count) plus `extra` int ranges —
// the fused pipeline folds its initial memsets into this single graph node and
// passes prezeroed = true.
int64_t pls_grid_max_cells(int64_t L);
void reserve_pls_grid(int64_t L, PlsScratch &sc, cudaStream_t s);
struct ZeroRange {
    void *ptr;
    int64_t words;      // 32-bit words
    unsigned value;     // word pattern
};
void launch_grid_prezero(int64_t L, PlsScratch &sc, const ZeroRange *extra, int n_extra, cudaStream_t s);

}  // namespace lc
