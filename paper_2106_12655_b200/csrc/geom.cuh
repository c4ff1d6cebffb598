// Device geometry of monomial cubic segments, in the IEEE operation order of
// the reference's numpy code (no FMA contraction: explicit _rn intrinsics).
//
// Segment layout: 12 doubles a0x a0y a0z a1x a1y a1z a2x a2y a2z a3x a3y a3z
// (the reference's (m, 4, 3) coeffs row, geometry.py:35-37).
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

namespace lc {

constexpr double kTwoPi = 6.283185307179586;          // 2.0 * math.pi (direct.py:16)

// Reference _pair_lambda with the IEEE operation sequence of the numba
// kernel (fastmath=False: no contraction): explicit _rn intrinsics.
__device__ __forceinline__ double ref_pair_lambda(double ljx, double ljy, double ljz, double lj1x,
                                                  double lj1y, double lj1z, double kix, double kiy,
                                                  double kiz, double ki1x, double ki1y, double ki1z) {
#define S_(a, b) __dsub_rn(a, b)
#define A_(a, b) __dadd_rn(a, b)
#define M_(a, b) __dmul_rn(a, b)
    const double ax = S_(ljx, kix), ay = S_(ljy, kiy), az = S_(ljz, kiz);
    const double bx = S_(ljx, ki1x), by = S_(ljy, ki1y), bz = S_(ljz, ki1z);
    const double cx = S_(lj1x, ki1x), cy = S_(lj1y, ki1y), cz = S_(lj1z, ki1z);
    const double dx = S_(lj1x, kix), dy = S_(lj1y, kiy), dz = S_(lj1z, kiz);
    const double an = __dsqrt_rn(A_(A_(M_(ax, ax), M_(ay, ay)), M_(az, az)));
    const double bn = __dsqrt_rn(A_(A_(M_(bx, bx), M_(by, by)), M_(bz, bz)));
    const double cn = __dsqrt_rn(A_(A_(M_(cx, cx), M_(cy, cy)), M_(cz, cz)));
    const double dn = __dsqrt_rn(A_(A_(M_(dx, dx), M_(dy, dy)), M_(dz, dz)));
    const double p = A_(A_(M_(ax, S_(M_(by, cz), M_(bz, cy))), M_(ay, S_(M_(bz, cx), M_(bx, cz)))),
                        M_(az, S_(M_(bx, cy), M_(by, cx))));
    const double ab = A_(A_(M_(ax, bx), M_(ay, by)), M_(az, bz));
    const double bc = A_(A_(M_(bx, cx), M_(by, cy)), M_(bz, cz));
    const double ca = A_(A_(M_(cx, ax), M_(cy, ay)), M_(cz, az));
    const double ad = A_(A_(M_(ax, dx), M_(ay, dy)), M_(az, dz));
    const double dc = A_(A_(M_(dx, cx), M_(dy, cy)), M_(dz, cz));
    const double d1 = A_(A_(A_(M_(M_(an, bn), cn), M_(ab, cn)), M_(bc, an)), M_(ca, bn));
    const double d2 = A_(A_(A_(M_(M_(an, dn), cn), M_(ad, cn)), M_(dc, an)), M_(ca, dn));
    return __ddiv_rn(A_(atan2(p, d1), atan2(p, d2)), kTwoPi);
#undef S_
#undef A_
#undef M_
}

// t**3 as numpy evaluates it on dyadic t (exact): (t*t)*t.  For the derivative
// roots of tight_boxes numpy's SIMD power may differ by an ulp.
__device__ __forceinline__ double cube_rn(double t) { return __dmul_rn(__dmul_rn(t, t), t); }

// a0 + a1*t + a2*t*t + a3*t**3  (geometry.py:107-110): ((a0 + a1 t) + (a2 t) t) + a3 (t^3)
__device__ __forceinline__ double eval_axis(double a0, double a1, double a2, double a3, double t) {
    return __dadd_rn(__dadd_rn(__dadd_rn(a0, __dmul_rn(a1, t)), __dmul_rn(__dmul_rn(a2, t), t)),
                     __dmul_rn(a3, cube_rn(t)));
}

__device__ __forceinline__ void eval_point(const double *__restrict__ c, double t, double p[3]) {
#pragma unroll
    for (int d = 0; d < 3; ++d) p[d] = eval_axis(c[d], c[3 + d], c[6 + d], c[9 + d], t);
}

__device__ __forceinline__ double np_min(double a, double b) {   // NaN-propagating like np.min
    return (a != a) ? a : ((b != b) ? b : (b < a ? b : a));
}
__device__ __forceinline__ double np_max(double a, double b) {
    return (a != a) ? a : ((b != b) ? b : (b > a ? b : a));
}

// Tight AABB of a cubic over [tlo, thi] (geometry.py:113-152): candidates are
// the domain ends and the stable roots of 3 a3 t^2 + 2 a2 t + a1, clipped.
__device__ __forceinline__ void tight_box(const double *__restrict__ c, double tlo, double thi,
                                          double lo[3], double hi[3]) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double a0 = c[d], a1 = c[3 + d], a2 = c[6 + d], a3 = c[9 + d];
        const double qa = __dmul_rn(3.0, a3);
        const double qb = __dmul_rn(2.0, a2);
        const double qc = a1;
        const double disc = __dsub_rn(__dmul_rn(qb, qb), __dmul_rn(__dmul_rn(4.0, qa), qc));
        const double dm = (disc != disc) ? disc : (disc > 0.0 ? disc : 0.0);   // np.maximum(disc, 0)
        const double sq = __dsqrt_rn(dm);
        const double q = __dmul_rn(-0.5, __dadd_rn(qb, copysign(sq, qb)));
        const double r1 = (qa != 0.0 && disc >= 0.0) ? __ddiv_rn(q, qa) : CUDART_NAN;
        const double r2 = (q != 0.0 && disc >= 0.0) ? __ddiv_rn(qc, q) : CUDART_NAN;
        // np.clip(r, tlo, thi) == minimum(maximum(r, tlo), thi)
        const double c2 = (r1 != r1) ? tlo : np_min(np_max(r1, tlo), thi);
        const double c3 = (r2 != r2) ? tlo : np_min(np_max(r2, tlo), thi);
        const double v0 = eval_axis(a0, a1, a2, a3, tlo);
        const double v1 = eval_axis(a0, a1, a2, a3, thi);
        const double v2 = eval_axis(a0, a1, a2, a3, c2);
        const double v3 = eval_axis(a0, a1, a2, a3, c3);
        lo[d] = np_min(np_min(np_min(v0, v1), v2), v3);
        hi[d] = np_max(np_max(np_max(v0, v1), v2), v3);
    }
}

// np.linalg.norm(hi - lo, axis=1) for one row: sqrt((dx*dx + dy*dy) + dz*dz)
__device__ __forceinline__ double diag_norm(const double lo[3], const double hi[3]) {
    const double dx = __dsub_rn(hi[0], lo[0]), dy = __dsub_rn(hi[1], lo[1]), dz = __dsub_rn(hi[2], lo[2]);
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

}  // namespace lc
