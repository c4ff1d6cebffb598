// Device geometry of monomial cubic segments, in the IEEE operation order of
// the reference's numpy code (no FMA contraction: explicit _rn intrinsics).
//
// Segment layout: 12 doubles a0x a0y a0z a1x a1y a1z a2x a2y a2z a3x a3y a3z
// (the reference's (m, 4, 3) coeffs row, geometry.py:35-37).
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

namespace lc {

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
