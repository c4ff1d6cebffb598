// Pass-1 detection of one loop pair (discretize.py:151-159 marking, only "was
// anything marked"): the fused pipeline's check that a model needs no
// refinement (brute_any_kernel / brute_any_lite_kernel, discretize.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "pls.cuh"

namespace lc {
namespace {

constexpr int64_t kBruteLimit = 16384;         // bvh.py:224 BRUTE_FORCE_LIMIT
constexpr int kBruteMaxSide = 256;             // shared-memory staging of loop j's boxes

__device__ __forceinline__ bool brute_pair(int64_t ni, int64_t nj) {
    return ni * nj <= kBruteLimit && ni <= kBruteMaxSide && nj <= kBruteMaxSide;
}

__device__ __forceinline__ bool box_overlap(const double *__restrict__ b, int64_t stride, int64_t e,
                                            const double lo[3], const double hi[3]) {
    // closed-interval overlap (bvh.py:93-98)
    return !(lo[0] > b[3 * stride + e] || b[e] > hi[0] || lo[1] > b[4 * stride + e] || b[stride + e] > hi[1] ||
             lo[2] > b[5 * stride + e] || b[2 * stride + e] > hi[2]);
}

#ifndef LC_PASS1_LANE_PAIRS
#define LC_PASS1_LANE_PAIRS 1   // group pairs one per lane; 0: a row of groups per step (shuffles; A/B)
#endif

constexpr int kAnyCap = 64;   // staged survivors per side; beyond that the test reads global memory

// One pair: the warp's share of the pass-1 detection (see brute_any_kernel).
__device__ __forceinline__ void brute_any_pair(int64_t p, const double *__restrict__ box, const float *__restrict__ fbox,
                                               int64_t M, const int64_t *__restrict__ loff,
                                               const double *__restrict__ lbox, int64_t L,
                                               const int32_t *__restrict__ pairs, int32_t *sidx0, int32_t *sidx1,
                                               float *sbox0, float *sbox1, int lane,
                                               unsigned long long *__restrict__ marked, int *__restrict__ abort) {
    int32_t *sidx_[2] = {sidx0, sidx1};
    float *sbox_[2] = {sbox0, sbox1};
#define sidx_at(sd, r) sidx_[sd][r]
#define sbox_at(sd, d, r) sbox_[sd][(d) * kAnyCap + (r)]

        const int i = pairs[2 * p], j = pairs[2 * p + 1];
        const int64_t bi = loff[i], ni = loff[i + 1] - bi;
        const int64_t bj = loff[j], nj = loff[j + 1] - bj;
        if (ni == 0 || nj == 0 || !brute_pair(ni, nj)) return;
        float fb[2][6];   // [0]: loop j's box (filters side i), [1]: loop i's box (filters side j)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            fb[0][d] = __double2float_rd(lbox[d * L + j]);
            fb[0][3 + d] = __double2float_ru(lbox[(3 + d) * L + j]);
            fb[1][d] = __double2float_rd(lbox[d * L + i]);
            fb[1][3 + d] = __double2float_ru(lbox[(3 + d) * L + i]);
        }
        // side 0: loop i's segments vs loop j's box; side 1 only if side 0 kept any
        int cnt[2] = {0, 0};
#pragma unroll
        for (int sd = 0; sd < 2; ++sd) {
            if (sd == 1 && cnt[0] == 0) break;   // no survivor on one side: no hit possible
            const float *o = fb[sd];
            const int64_t base = sd ? bj : bi;
            const int n = (int)(sd ? nj : ni);
#pragma unroll 2
            for (int k0 = 0; k0 < n; k0 += 32) {
                const int k = k0 + lane;
                const int64_t e = base + k;
                float v[6];
#pragma unroll
                for (int d = 0; d < 6; ++d) v[d] = k < n ? fbox[d * M + e] : 0.f;
                const bool in = k < n && !(o[0] > v[3] || v[0] > o[3] || o[1] > v[4] || v[1] > o[4] ||
                                           o[2] > v[5] || v[2] > o[5]);
                const unsigned bal = __ballot_sync(0xffffffffu, in);
                if (in) {
                    const int r = cnt[sd] + __popc(bal & ((1u << lane) - 1u));
                    if (r < kAnyCap) {
                        sidx_at(sd, r) = (int32_t)e;
#pragma unroll
                        for (int d = 0; d < 6; ++d) sbox_at(sd, d, r) = v[d];
                    }
                }
                cnt[sd] += __popc(bal);
            }
        }
        __syncwarp();
        const int ns = cnt[0], nt = cnt[1];
        int hits = 0;
        if (ns && nt && ns <= kAnyCap && nt <= kAnyCap) {
            // lanes take the larger survivor list (its float box in registers), the smaller
            // one is read from shared memory as a broadcast: ~n_small iterations, no division
            const int sl = ns >= nt ? 0 : 1, nl = sl ? nt : ns, nq = sl ? ns : nt;
            for (int base = 0; base < nl; base += 32) {
                const int l = base + lane;
                float x[6];
                int64_t el = -1;
                if (l < nl) {
                    el = sidx_at(sl, l);
#pragma unroll
                    for (int d = 0; d < 6; ++d) x[d] = sbox_at(sl, d, l);
                }
                for (int q = 0; q < nq; ++q) {
                    float y[6];
#pragma unroll
                    for (int d = 0; d < 6; ++d) y[d] = sbox_at(sl ^ 1, d, q);
                    if (el < 0 || x[0] > y[3] || y[0] > x[3] || x[1] > y[4] || y[1] > x[4] || x[2] > y[5] ||
                        y[2] > x[5])
                        continue;
                    // a float hit: the exact closed test on the double boxes (bvh.py:93-98)
                    const int64_t eq = sidx_at(sl ^ 1, q);
                    double lo[3], hi[3];
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        lo[d] = box[d * M + el];
                        hi[d] = box[(3 + d) * M + el];
                    }
                    if (box_overlap(box, M, eq, lo, hi)) ++hits;
                }
            }
        } else if (ns && nt) {   // rare: more survivors than staged — every combination from global memory
            for (int k = lane; k < ns * nt; k += 32) {
                const int a = k / nt, b = k % nt;
                int64_t es = -1, et = -1;
                int c = 0;
                for (int64_t q = 0; q < ni && es < 0; ++q) {
                    const float *o = fb[0];
                    float u[6];
#pragma unroll
                    for (int d = 0; d < 6; ++d) u[d] = fbox[d * M + bi + q];
                    if (!(o[0] > u[3] || u[0] > o[3] || o[1] > u[4] || u[1] > o[4] || o[2] > u[5] || u[2] > o[5]) &&
                        c++ == a)
                        es = bi + q;
                }
                c = 0;
                for (int64_t q = 0; q < nj && et < 0; ++q) {
                    const float *o = fb[1];
                    float u[6];
#pragma unroll
                    for (int d = 0; d < 6; ++d) u[d] = fbox[d * M + bj + q];
                    if (!(o[0] > u[3] || u[0] > o[3] || o[1] > u[4] || u[1] > o[4] || o[2] > u[5] || u[2] > o[5]) &&
                        c++ == b)
                        et = bj + q;
                }
                double lo[3], hi[3];
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    lo[d] = box[d * M + es];
                    hi[d] = box[(3 + d) * M + es];
                }
                if (box_overlap(box, M, et, lo, hi)) ++hits;
            }
        }
        if (hits) {
            atomicAdd(marked, (unsigned long long)hits);
            if (abort) *abort = 1;
        }
        __syncwarp();
    #undef sidx_at
#undef sbox_at
}


// brute_any_pair with the 8-segment group boxes of seg_boxes_loop_kernel (`sub`,
// layout pass1_group_slot; float, outward, NaN -> unbounded):
// each lane tests one group pair (<= 32 groups per loop: both loops have <= 256
// segments; 24 % fewer instructions than a row of shuffled groups per step,
// profiles/r02/ab_pass1_lane_pairs.log), and only overlapping group pairs test
// their 8 x 8 segment pairs (float, then the exact closed test on the double boxes).  Same decision as brute_any_pair: a segment
// pair overlaps exactly => its float boxes and its groups overlap.
__device__ __forceinline__ void brute_any_pair_sub(int64_t p, const double *__restrict__ box,
                                                   const float *__restrict__ fbox, const float *__restrict__ sub,
                                                   int64_t M, int64_t L, const int64_t *__restrict__ loff,
                                                   const int32_t *__restrict__ pairs, int lane,
                                                   unsigned long long *__restrict__ marked, int *__restrict__ abort) {
    const int i = pairs[2 * p], j = pairs[2 * p + 1];
    const int64_t bi = loff[i], ni = loff[i + 1] - bi;
    const int64_t bj = loff[j], nj = loff[j + 1] - bj;
    if (ni == 0 || nj == 0 || !brute_pair(ni, nj)) return;
    const int gi = (int)((ni + 7) >> 3), gj = (int)((nj + 7) >> 3);
    const int64_t S = pass1_group_stride(M, L), qi = pass1_group_slot(bi, i), qj = pass1_group_slot(bj, j);
    const int u = lane & 7, w = lane >> 3;   // segment pair (u, w) and (u, w + 4) of a group pair
    int hits = 0;
#if LC_PASS1_LANE_PAIRS
    // lane = one group pair (a, c): c = lane mod 2^sh (2^sh >= gj), a = a0 + lane >> sh;
    // loop j's group box stays in the lane across chunks, loop i's is loaded per chunk
    // (no shuffles: 4 chunk loads instead of 8 rows of 6 shuffles for 64-segment loops)
    const int sh = 32 - __clz(gj - 1);
    const int per = 32 >> sh, cl = lane & ((1 << sh) - 1), da = lane >> sh;
    float sj[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) sj[d] = cl < gj ? sub[d * S + qj + cl] : 0.f;
    for (int a0 = 0; a0 < gi; a0 += per) {
        const int ga = a0 + da;
        const bool valid = cl < gj && ga < gi;
        float o[6];
#pragma unroll
        for (int d = 0; d < 6; ++d) o[d] = valid ? sub[d * S + qi + ga] : 0.f;
        const bool ov = valid && !(o[0] > sj[3] || sj[0] > o[3] || o[1] > sj[4] || sj[1] > o[4] ||
                                   o[2] > sj[5] || sj[2] > o[5]);
        unsigned bal = __ballot_sync(0xffffffffu, ov);
        while (bal) {
            const int bit = __ffs(bal) - 1;
            bal &= bal - 1;
            const int a = a0 + (bit >> sh), c = bit & ((1 << sh) - 1);
#else
    float si[6], sj[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        si[d] = lane < gi ? sub[d * S + qi + lane] : 0.f;
        sj[d] = lane < gj ? sub[d * S + qj + lane] : 0.f;
    }
    for (int a = 0; a < gi; ++a) {
        float o[6];
#pragma unroll
        for (int d = 0; d < 6; ++d) o[d] = __shfl_sync(0xffffffffu, si[d], a);
        const bool ov = lane < gj && !(o[0] > sj[3] || sj[0] > o[3] || o[1] > sj[4] || sj[1] > o[4] ||
                                       o[2] > sj[5] || sj[2] > o[5]);
        unsigned bal = __ballot_sync(0xffffffffu, ov);
        while (bal) {
            const int c = __ffs(bal) - 1;
            bal &= bal - 1;
#endif
            const int64_t ki = 8 * a + u;
            if (ki >= ni) continue;
            const int64_t ei = bi + ki;
            float x[6];
#pragma unroll
            for (int d = 0; d < 6; ++d) x[d] = fbox[d * M + ei];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t kj = 8 * c + w + 4 * h;
                if (kj >= nj) continue;
                const int64_t ej = bj + kj;
                float y[6];
#pragma unroll
                for (int d = 0; d < 6; ++d) y[d] = fbox[d * M + ej];
                if (x[0] > y[3] || y[0] > x[3] || x[1] > y[4] || y[1] > x[4] || x[2] > y[5] || y[2] > x[5]) continue;
                double lo[3], hi[3];   // a float hit: the exact closed test on the double boxes (bvh.py:93-98)
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    lo[d] = box[d * M + ei];
                    hi[d] = box[(3 + d) * M + ei];
                }
                if (box_overlap(box, M, ej, lo, hi)) ++hits;
            }
        }
    }
    if (hits) {
        atomicAdd(marked, (unsigned long long)hits);
        if (abort) *abort = 1;
    }
}

}  // namespace
}  // namespace lc
