// Potential link search on the device (replaces linkcert/pls.py:48-73 and
// the bvh.overlap_pairs_boxes broad phase it calls, bvh.py:227-243).
#pragma once
#include "common.cuh"

namespace lc {

// Boxes are SoA: box[0*n..] lo_x, [1*n] lo_y, [2*n] lo_z, [3*n] hi_x, [4*n] hi_y, [5*n] hi_z.

// Per-segment tight boxes over each segment's own domain; seg_loop[m] = loop
// of segment m; zero-length check (discretize.py:124-129): *zero_loop =
// min loop index with a segment box diagonal < min_diam (INT_MAX if none).
void launch_seg_boxes(const double *coeffs, const double *t, const int64_t *loff, int64_t L, int64_t M,
                      double min_diam, double *seg_box, int32_t *seg_loop, int *zero_loop, cudaStream_t s);

// Loop AABB = union of its segment boxes (pls.py:48-56).
void launch_loop_boxes(const double *seg_box, int64_t M, const int64_t *loff, int64_t L, double *loop_box,
                       cudaStream_t s);

struct PlsScratch {
    DevBuf keys, keys_sorted, idx, perm, counts, offs, cub_tmp, pair_keys, pair_keys_sorted, axis, excl;
};

// Sort-and-sweep over loop boxes on the axis of largest extent, closed
// intervals (bvh.py:93-98), i<j, minus the excluded keys (sorted uint64
// (i<<32|j)), sorted lexicographically.  Writes int32 (P,2) into *pairs
// (grown as needed) and returns P (one host sync for the count).
int64_t run_pls(const double *loop_box, int64_t L, const uint64_t *h_excl, int64_t n_excl, PlsScratch &sc,
                DevBuf &pairs, cudaStream_t s);

}  // namespace lc
