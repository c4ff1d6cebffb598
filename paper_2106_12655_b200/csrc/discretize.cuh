// Adaptive homotopy-safe discretization on the device (linkcert/discretize.py:112-191).
#pragma once
#include <vector>

#include "common.cuh"

namespace lc {

enum DiscErrKind : int {
    DISC_OK = 0,
    DISC_ZERO_LENGTH = 1,       // ZeroLengthInput, loops = (idx,)
    DISC_CURVES_INTERSECT = 2,  // CurvesIntersect, loops = (a, b) sorted
    DISC_SUBSEG_BUDGET = 3,     // PassLimitExceeded, loops = (i,)   (max_subsegments)
    DISC_PASS_BUDGET = 4,       // PassLimitExceeded, loops = busy   (max_passes)
    DISC_INVALID_POLYLINE = 5,  // ValidationError from PolylineLoop, loops = (idx,), detail = reason
};

enum PolylineInvalid : int { PL_OK = 0, PL_TOO_FEW = 1, PL_NONFINITE = 2, PL_ZERO_SEGMENT = 3 };

struct DiscError {
    int kind = DISC_OK;
    int detail = 0;
    std::vector<int64_t> loops;
};

// Pre-pass / pass counters on the device (read back together in one copy).
struct PreCounters {
    int zero_loop;     // first loop with a zero-length segment box (INT_MAX: none)
    int n_unpaired;
    int n_large;       // pairs handled by the sweep path
    int abort;         // fused path: set with any of the above / a pass-1 hit (the Gauss sum stops early)
    unsigned long long marked;
    int err_loop;
    int pad2;
};

struct DiscParams {
    double xi = 1.0;
    double epsilon = 2.220446049250313e-16;   // discretize.py:27 (MACHINE_EPS)
    int max_passes = 64;
    int64_t max_subsegments = int64_t(1) << 22;
    bool defer_validation = false;   // leave the PolylineLoop check result on the device (DiscOutput)
};

struct DiscScratch {
    DevBuf paired, act_seg, act_loop, act_tlo, act_thi, act_off, nxt_seg, nxt_loop, nxt_tlo, nxt_thi, nxt_off,
        nxt_partner, box, nxt_box, skey[3], sperm[3], iota, pair_axis, sweep_off, mark, first_pair, mark_scan,
        done_seg, done_tlo, done_seg2, done_tlo2, sort_idx, sort_idx2, done_cnt, done_off, bad_first, counters,
        cub_tmp, loop_err, val_flags, ucnt, tmp_aos, prectr, ubox, mark2, fp2, val_err2;
    int64_t cap_done = 0;
};

struct DiscInput {
    const double *coeffs;                   // (M, 12)
    const double *t;                        // (M, 2)
    const int64_t *loff;                    // (L+1)
    const int32_t *seg_loop;                // (M)
    const double *seg_box;                  // SoA 6 x M
    const double *loop_box;                 // SoA 6 x L
    const unsigned long long *loop_min_diag;// (L) bit patterns of min squared segment-box diagonals
    const int *max_exp;                     // exponent field of the largest |box coordinate|
    int64_t L, M;
    const int32_t *pairs;                   // (P, 2), sorted PairList
    int64_t P;
    const float *seg_fbox = nullptr;        // seg_box rounded outward to float (prefilter), optional
    const float *seg_sub = nullptr;         // float boxes of 8-segment groups (SoA 6 x M, at each group's
                                            // first segment; fused split path only), optional
    const double *verts = nullptr;          // closed-polyline model: vertices (M,3) (coeffs are then
                                            // LoopGeometry.from_polyline's); lets the no-split chord
                                            // write read 24 B instead of 112 B per segment
};

// Output: the chord polylines, already in the Gauss-sum layout — closed SoA
// (vertex 0 repeated per loop) scaled by 2^-e, e = exponent of the largest
// coordinate (exact).  vert_off = plain per-loop offsets.
struct DiscOutput {
    DevBuf X, Y, Z, voff, vert_off;
    int64_t V = 0, Vc = 0;
    int passes = 0;
    int64_t splits = 0;
    // defer_validation: d_val_err[0] / [1] = first invalid unpaired / paired loop
    // (loop*4 + PolylineInvalid, INT_MAX if none); the caller reads it back.
    bool validation_pending = false;
    const int *d_val_err = nullptr;
};

// Map a (deferred) validation read-back onto *err; true if it holds an error.
bool validation_error(const int val_err[2], DiscError *err);

// Returns false and fills *err on a reference error (nothing else is thrown
// for input-dependent failures).
bool run_discretize(const DiscInput &in, const DiscParams &prm, DiscScratch &sc, DiscOutput &out,
                    DiscError *err, cudaStream_t s);

// Fused pipeline (no host sync): the discretization of the common case where
// pass 1 marks nothing and every pair is a small (brute-force) pair — then
// the chords are every segment's start point (run_discretize's splits == 0
// branch).  in.P is the pair-buffer capacity, d_P the device pair count.
// The result is the reference's iff, after the stream reaches it,
// (*d_ctr)->zero_loop == INT_MAX, n_large == 0 and marked == 0; validation is
// left pending in out.d_val_err like defer_validation.  Otherwise the caller
// reruns run_discretize.
void launch_discretize_fast(const DiscInput &in, const int64_t *d_P, const DiscParams &prm, DiscScratch &sc,
                            DiscOutput &out, cudaStream_t s, const PreCounters **d_ctr);
// The same as two independent branches (no allocation inside; reserve first):
// chords (needs only the model: closed offsets, chord write + PolylineLoop
// flags) and checks (needs the pairs: pre-pass, pass-1 detection, then —
// after `chords_done` — the validation ranking).
void reserve_discretize_fast(const DiscInput &in, DiscScratch &sc, DiscOutput &out, cudaStream_t s);
void launch_discretize_chords(const DiscInput &in, const DiscParams &prm, DiscScratch &sc, DiscOutput &out,
                              cudaStream_t s, bool prezeroed = false);
void launch_discretize_checks(const DiscInput &in, const int64_t *d_P, const DiscParams &prm, DiscScratch &sc,
                              DiscOutput &out, cudaStream_t s, cudaEvent_t chords_done, const PreCounters **d_ctr,
                              bool brute_by_caller = false, bool prezeroed = false);
// The pass-1 pair check alone (brute_any_kernel, grid-stride over *d_P pairs): on the
// critical stream after the segment boxes, followed by the Gauss sum as its
// programmatic dependent (the kernel triggers its dependents as it starts).
void launch_pass1_brute(const DiscInput &in, const int64_t *d_P, DiscScratch &sc, cudaStream_t s);
// Resets the counters (incl. the abort flag the Gauss kernel polls) — on the
// stream every branch forks from, before the fork.
void launch_discretize_init(DiscScratch &sc, cudaStream_t s);

// Unscaled AoS (V, 3) vertices (no closing vertices) from a DiscOutput.
void unpack_polylines(const DiscOutput &out, int64_t L, const int *max_exp, double *aos, cudaStream_t s);

}  // namespace lc
