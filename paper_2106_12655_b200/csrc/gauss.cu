// FP64 direct-summation Gauss linking integral over a loop-pair list (sm_100a).
//
// Reference semantics: linkcert/direct.py:19-65 (_pair_lambda, _link_atan),
// batched as certify.py:108-127 (_evaluate_pairs) with kernels.py:45-73
// rounding.  For pair (i, j), i < j, the reference evaluates
//   link_direct(loop_i, loop_j):  l = loop i (inner, "columns"),
//                                 k = loop j (outer, "rows")
// and sums lambda(l_c, l_c+1, k_r, k_r+1) over all r < N_k, c < N_l.
//
// Work decomposition: every pair is cut into warp items.  A
// warp item covers (1<<rb_log2) row blocks of kRowsPerLane rows times
// (32>>rb_log2) column strips of `cl` columns; each lane owns one
// (row block, column strip) and walks its strip column by column, keeping
// the kRowsPerLane+1 row vertices in registers.  The four corner vectors of
// a segment pair are vertex-pair differences r(c, m) = l_c - k_m, so a
// column step computes one new difference vector, norm and two edge dot
// products per row vertex and reuses the previous column's values — the
// operands the reference formula forms.  Column steps alternate between two
// register sets (no array shifting) and contain no branches.
// Item partials go through a warp butterfly (fixed order) into
// partials[item]; pairs are reduced from their contiguous item range in a
// fixed order, so raw sums are identical run to run and for any split of
// the item range across GPUs.
#include "gauss.cuh"
#include "geom.cuh"

#include "scan.cuh"

namespace lc {

namespace {

constexpr double kInvTwoPi = 0.15915494309189535;     // 1 / (2 pi), correctly rounded
#ifndef LC_GAUSS_CARVEOUT
#define LC_GAUSS_CARVEOUT 10   // % of the unified L1 kept as shared memory beside the Gauss CTAs
#endif
constexpr int kGaussCarveout = LC_GAUSS_CARVEOUT;
#ifndef LC_PAIRS_PREFETCH
#define LC_PAIRS_PREFETCH 1        // persistent pair kernel: prefetch the next claim / pair geometry
#endif
#ifndef LC_MINB
#define LC_MINB 2   // resident CTAs per SM the phase items kernel is compiled for (A/B: -DLC_MINB=n)
#endif
#ifndef LC_PAIRS_MINB
#define LC_PAIRS_MINB LC_MINB   // ... and the phase pair kernel (fused path)
#endif

__device__ __forceinline__ int sbit(double x) { return (int)((unsigned)__double2hiint(x) >> 31); }

// U = A * B counting full turns so that, along a product chain,
//   sum of factor angles = 2*pi*turns + atan2(U.y, U.x)   (atan2 signed-zero semantics).
// Half planes by the sign bit of the imaginary part ("upper": arg in [+0, pi],
// "lower": [-pi, -0]); two factors in the same half whose product lands in the
// other half wrapped by one turn — the full-turn rule of _link_angle_sum
// (direct.py:120-123), exact given the computed product.  With a = sb(A.y),
// b = sb(B.y), c = sb(U.y) the wrap is (a == b) ? c - a : 0.
__device__ __forceinline__ void cmul_w(double ax, double ay, double bx, double by, double &ux, double &uy,
                                       int &turns) {
    ux = fma(ax, bx, -ay * by);
    uy = fma(ax, by, ay * bx);
    const int sa = sbit(ay), sb = sbit(by), su = sbit(uy);
    turns += (sa == sb) ? (su - sa) : 0;
}

// sqrt(x) for x >= 0 without the libdevice special-case branch: MUFU rsqrt
// seed + 2 Newton steps, s = x * y (~2 ulp; the norms only enter the d1/d2
// denominators).  LC_SQRT_HERON adds a Heron correction (<= 1 ulp).
#ifndef LC_SQRT
#define LC_SQRT 5
#endif
template <bool ZERO_SAFE = true>
__device__ __forceinline__ double sqrt_nb(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#if LC_SQRT == 7
    // coupled (Goldschmidt) iteration: g -> sqrt(x), hh -> 1/(2 sqrt(x)); 7 FP64 ops
    double g = x * y, hh = 0.5 * y;
    double r = fma(-g, hh, 0.5);
    g = fma(g, r, g);
    hh = fma(hh, r, hh);
    r = fma(-g, hh, 0.5);
    g = fma(g, r, g);
#else
    // one step from the seed with the series of (1 - e)^(-1/2), e = 1 - x y^2:
    // sqrt(x) = x y (1 + e/2 + 3e^2/8 [+ 5e^3/16]); 5 [6] FP64 ops
    const double t = x * y;
    const double e = fma(-t, y, 1.0);
#if LC_SQRT == 6
    const double q = e * fma(e, fma(e, 0.3125, 0.375), 0.5);
#else
    const double q = e * fma(e, 0.375, 0.5);
#endif
    double g = fma(t, q, t);
#endif
    // x == 0 (coincident vertices) gives NaN without the select; the phase fast
    // path omits it and re-evaluates such (degenerate) strips exactly.
    return ZERO_SAFE ? (x > 0.0 ? g : 0.0) : g;
}

// ------------------------------------------------------------ lane strip

constexpr int R = kRowsPerLane;

struct Col {   // one column: r(c, m) = l_c - k_m, |r(c, m)|, v[m] = r(c,m).r(c,m+1)
    double x[R + 1], y[R + 1], z[R + 1], n[R + 1], v[R];
};

// Row vertices k_m of a lane: in registers (KReg) or in shared memory (KSm,
// re-read every column step with volatile loads to free 30 registers).
struct KReg {
    double x[R + 1], y[R + 1], z[R + 1];
    __device__ __forceinline__ double X(int m) const { return x[m]; }
    __device__ __forceinline__ double Y(int m) const { return y[m]; }
    __device__ __forceinline__ double Z(int m) const { return z[m]; }
    __device__ __forceinline__ void set(int m, double a, double b, double c) { x[m] = a; y[m] = b; z[m] = c; }
};
constexpr int kCtaThreads = 128;
struct KSm {
    double *p;   // this thread's column of a [3*(R+1)][kCtaThreads] shared array
    __device__ __forceinline__ static double ld(const double *q) {
        double v;
        asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "l"(__cvta_generic_to_shared(q)));
        return v;
    }
    __device__ __forceinline__ double X(int m) const { return ld(p + m * kCtaThreads); }
    __device__ __forceinline__ double Y(int m) const { return ld(p + (R + 1 + m) * kCtaThreads); }
    __device__ __forceinline__ double Z(int m) const { return ld(p + (2 * R + 2 + m) * kCtaThreads); }
    __device__ __forceinline__ void set(int m, double a, double b, double c) {
        p[m * kCtaThreads] = a;
        p[(R + 1 + m) * kCtaThreads] = b;
        p[(2 * R + 2 + m) * kCtaThreads] = c;
    }
};

template <bool ZERO_SAFE, class K>
__device__ __forceinline__ void col_fill(Col &B, double lx, double ly, double lz, const K &k) {
#pragma unroll
    for (int m = 0; m <= R; ++m) {
        B.x[m] = lx - k.X(m);
        B.y[m] = ly - k.Y(m);
        B.z[m] = lz - k.Z(m);
        B.n[m] = sqrt_nb<ZERO_SAFE>(fma(B.z[m], B.z[m], fma(B.y[m], B.y[m], B.x[m] * B.x[m])));
    }
#pragma unroll
    for (int m = 0; m < R; ++m) B.v[m] = fma(B.z[m], B.z[m + 1], fma(B.y[m], B.y[m + 1], B.x[m] * B.x[m + 1]));
}

// Arai terms of pair (row m, column c) (direct.py:21-46): corner vectors a = r(c,m),
// b = r(c,m+1), c = r(c+1,m+1), d = r(c+1,m); shared dots ab = A.v[m],
// dc = B.v[m], ad = h[m], bc = h[m+1] with h[m] = r(c,m).r(c+1,m).
// Returns w = (d1 + i p)(d2 + i p) = (xp, yp); its wrap (z1, z2 share the sign
// bit of p) goes to `turns`.  A degenerate w == 0 (p = 0 and d1 or d2 = 0)
// contributes the exact atan2(+-0, d) half turns instead and w := 1.
template <bool FAST>
__device__ __forceinline__ void pair_w(const Col &A, const Col &B, const double *h, int m, double &wx, double &wy,
                                       int &turns, int &halves) {
    const double ax = A.x[m], ay = A.y[m], az = A.z[m];
    const double bx = A.x[m + 1], by = A.y[m + 1], bz = A.z[m + 1];
    const double cx = B.x[m + 1], cy = B.y[m + 1], cz = B.z[m + 1];
    const double an = A.n[m], bn = A.n[m + 1], cn = B.n[m + 1], dn = B.n[m];
    const double ab = A.v[m], dc = B.v[m], ad = h[m], bc = h[m + 1];
    const double ca = fma(cz, az, fma(cy, ay, cx * ax));
    const double p = fma(az, fma(bx, cy, -by * cx), fma(ay, fma(bz, cx, -bx * cz), ax * fma(by, cz, -bz * cy)));
    // d1 = an bn cn + ab cn + bc an + ca bn, d2 = an dn cn + ad cn + dc an + ca dn
    const double t1 = fma(an, cn, ca);
    const double d1 = fma(bn, t1, fma(cn, ab, an * bc));
    const double d2 = fma(dn, t1, fma(cn, ad, an * dc));
    const double xp = fma(d1, d2, -p * p);
    const double yp = p * (d1 + d2);
    if (FAST) {   // degenerate w == 0 is caught by the strip's zero/NaN check instead
        turns += sbit(yp) - sbit(p);
        wx = xp;
        wy = yp;
        return;
    }
    const bool deg = (xp == 0.0) & (yp == 0.0);
    const int sp = sbit(p);
    turns += deg ? 0 : (sbit(yp) - sp);
    const int hs = sbit(d1) + sbit(d2);
    halves += deg ? (sp ? -hs : hs) : 0;
    wx = deg ? 1.0 : xp;
    wy = deg ? 0.0 : yp;
}

struct Acc {
    double sx = 1.0, sy = 0.0;   // GAUSS_PHASE: phase product
    double ang = 0.0;            // GAUSS_ATAN: sum of fused angles (radians)
    int turns = 0, halves = 0;
    int bad = 0;                 // GAUSS_PHASE: re-evaluate the strip exactly
};

template <int MODE, bool FULL, bool RENORM, class K>
__device__ __forceinline__ void col_step(const Col &A, Col &B, double lx, double ly, double lz, const K &k,
                                         const bool *rv, Acc &acc) {
    constexpr bool FAST = MODE == GAUSS_PHASE;
    col_fill<!FAST>(B, lx, ly, lz, k);
    double h[R + 1];
#pragma unroll
    for (int m = 0; m <= R; ++m) h[m] = fma(A.z[m], B.z[m], fma(A.y[m], B.y[m], A.x[m] * B.x[m]));
    double wx[R], wy[R];
    if (FAST) {   // the R pair terms stage by stage: independent chains side by side (+2% over pair_w order)
        double ca[R], p[R], t1[R], d1[R], d2[R];
#pragma unroll
        for (int m = 0; m < R; ++m)
            ca[m] = fma(B.z[m + 1], A.z[m], fma(B.y[m + 1], A.y[m], B.x[m + 1] * A.x[m]));
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const double ax = A.x[m], ay = A.y[m], az = A.z[m];
            const double bx = A.x[m + 1], by = A.y[m + 1], bz = A.z[m + 1];
            const double cx = B.x[m + 1], cy = B.y[m + 1], cz = B.z[m + 1];
            p[m] = fma(az, fma(bx, cy, -by * cx), fma(ay, fma(bz, cx, -bx * cz), ax * fma(by, cz, -bz * cy)));
        }
#pragma unroll
        for (int m = 0; m < R; ++m) t1[m] = fma(A.n[m], B.n[m + 1], ca[m]);
#pragma unroll
        for (int m = 0; m < R; ++m) {
            d1[m] = fma(A.n[m + 1], t1[m], fma(B.n[m + 1], A.v[m], A.n[m] * h[m + 1]));
            d2[m] = fma(B.n[m], t1[m], fma(B.n[m + 1], h[m], A.n[m] * B.v[m]));
        }
#pragma unroll
        for (int m = 0; m < R; ++m) {
            wx[m] = fma(d1[m], d2[m], -p[m] * p[m]);
            wy[m] = p[m] * (d1[m] + d2[m]);
            int t = sbit(wy[m]) - sbit(p[m]);
            if (!FULL && !rv[m]) {
                wx[m] = 1.0;
                wy[m] = 0.0;
                t = 0;
            }
            acc.turns += t;
        }
    } else
#pragma unroll
    for (int m = 0; m < R; ++m) {
        int t = 0, hv = 0;
        pair_w<FAST>(A, B, h, m, wx[m], wy[m], t, hv);
        if (!FULL && !rv[m]) {
            wx[m] = 1.0;
            wy[m] = 0.0;
            t = hv = 0;
        }
        acc.turns += t;
        acc.halves += hv;
    }
    if (MODE == GAUSS_ATAN) {
#pragma unroll
        for (int m = 0; m < R; ++m) acc.ang += atan2(wy[m], wx[m]);
    } else {
        // product tree (w0 w1)(w2 w3), S *= W, then renormalize S by an exact power of two
        double ux, uy, nx, ny;
        if (R == 4) {
            double ax, ay, bx, by;
            cmul_w(wx[0], wy[0], wx[1], wy[1], ax, ay, acc.turns);
            cmul_w(wx[2], wy[2], wx[3], wy[3], bx, by, acc.turns);
            cmul_w(ax, ay, bx, by, ux, uy, acc.turns);
        } else {
            ux = wx[0];
            uy = wy[0];
#pragma unroll
            for (int m = 1; m < R; ++m) {
                double tx, ty;
                cmul_w(ux, uy, wx[m], wy[m], tx, ty, acc.turns);
                ux = tx;
                uy = ty;
            }
        }
        cmul_w(acc.sx, acc.sy, ux, uy, nx, ny, acc.turns);
        if (RENORM) {   // every second step: exact power-of-two rescale of S
            const int ex = __double2hiint(nx) & 0x7ff00000, ey = __double2hiint(ny) & 0x7ff00000;
            const int e = ex > ey ? ex : ey;
            acc.bad |= (e == 0) | (e == 0x7ff00000);   // S underflowed / degenerate / NaN
            const double scale = __hiloint2double(0x7fe00000 - e, 0);
            nx *= scale;
            ny *= scale;
        }
        acc.sx = nx;
        acc.sy = ny;
    }
}

#ifndef LC_ITEMS_PREFETCH
#define LC_ITEMS_PREFETCH 0   // (A/B) items kernel: next claim + record fetched a unit ahead
#endif
#ifndef LC_PAIRS_L1PF
#define LC_PAIRS_L1PF 1   // prefetch the next pair's first-item vertices into L1 (0: off, A/B)
#endif
__device__ __forceinline__ void l1_prefetch(const double *q) { asm volatile("prefetch.global.L1 [%0];" ::"l"(q)); }
// The lines this lane's strip of item (ir, ic) of pair tiling g starts with: its
// R + 1 row vertices and its first column vertex, per coordinate array.
struct NextItem {
    const PairGeom *g;   // nullptr: nothing to prefetch
    int ir, ic;
};
__device__ __forceinline__ void l1_prefetch_item(const double *__restrict__ X, const double *__restrict__ Y,
                                                 const double *__restrict__ Z, const PairGeom &g, int ir, int ic,
                                                 int vl) {
    const int row0 = ((ir << g.rb_log2) + (vl & ((1 << g.rb_log2) - 1))) * R;
    const int64_t c0 = ((int64_t)ic * (32 >> g.rb_log2) + (vl >> g.rb_log2)) * g.cl;
    if (row0 >= g.nrows || c0 >= g.ncols) return;
    const int64_t r0 = g.row_off + row0, r1 = g.row_off + min(row0 + R, g.nrows), cc = g.col_off + c0;
    l1_prefetch(X + r0); l1_prefetch(Y + r0); l1_prefetch(Z + r0);
    l1_prefetch(X + r1); l1_prefetch(Y + r1); l1_prefetch(Z + r1);
    l1_prefetch(X + cc); l1_prefetch(Y + cc); l1_prefetch(Z + cc);
}

// Sum over rows [row0, row0+R) x columns [c0, c1) of one pair, in turns.
template <int MODE, bool FULL, class K>
__device__ double lane_strip(const double *__restrict__ X, const double *__restrict__ Y,
                             const double *__restrict__ Z, int64_t row_off, int nrows, int64_t col_off, int row0,
                             int c0, int c1, K &kv, NextItem pf = {nullptr, 0, 0}, int vl = 0) {
    bool rv[R];
#pragma unroll
    for (int m = 0; m <= R; ++m) {
        const int v = FULL ? row0 + m : min(row0 + m, nrows);   // closing vertex sits at index nrows
        kv.set(m, __ldg(X + row_off + v), __ldg(Y + row_off + v), __ldg(Z + row_off + v));
    }
#pragma unroll
    for (int m = 0; m < R; ++m) rv[m] = FULL || row0 + m < nrows;
    const double *px = X + col_off, *py = Y + col_off, *pz = Z + col_off;
    Col A, B;
    col_fill<MODE != GAUSS_PHASE>(A, __ldg(px + c0), __ldg(py + c0), __ldg(pz + c0), kv);
#if LC_PAIRS_L1PF
    if (pf.g) l1_prefetch_item(X, Y, Z, *pf.g, pf.ir, pf.ic, vl);   // the next unit's rows + first column, a strip ahead
#endif
    Acc acc;
    int c = c0;
#ifdef LC_PREFETCH
    // the next pair of columns is loaded one iteration ahead (column loads off the critical path)
    double n1x = 0, n1y = 0, n1z = 0, n2x = 0, n2y = 0, n2z = 0;
    if (c + 2 <= c1) {
        n1x = __ldg(px + c + 1); n1y = __ldg(py + c + 1); n1z = __ldg(pz + c + 1);
        n2x = __ldg(px + c + 2); n2y = __ldg(py + c + 2); n2z = __ldg(pz + c + 2);
    }
    for (; c + 2 <= c1; c += 2) {
        const double l1x = n1x, l1y = n1y, l1z = n1z, l2x = n2x, l2y = n2y, l2z = n2z;
        if (c + 4 <= c1) {
            n1x = __ldg(px + c + 3); n1y = __ldg(py + c + 3); n1z = __ldg(pz + c + 3);
            n2x = __ldg(px + c + 4); n2y = __ldg(py + c + 4); n2z = __ldg(pz + c + 4);
        }
        col_step<MODE, FULL, false>(A, B, l1x, l1y, l1z, kv, rv, acc);
        col_step<MODE, FULL, true>(B, A, l2x, l2y, l2z, kv, rv, acc);
    }
#else
    for (; c + 2 <= c1; c += 2) {
        const double l1x = __ldg(px + c + 1), l1y = __ldg(py + c + 1), l1z = __ldg(pz + c + 1);
        const double l2x = __ldg(px + c + 2), l2y = __ldg(py + c + 2), l2z = __ldg(pz + c + 2);
        col_step<MODE, FULL, false>(A, B, l1x, l1y, l1z, kv, rv, acc);
        col_step<MODE, FULL, true>(B, A, l2x, l2y, l2z, kv, rv, acc);
    }
#endif
    if (c < c1) col_step<MODE, FULL, true>(A, B, __ldg(px + c + 1), __ldg(py + c + 1), __ldg(pz + c + 1), kv, rv, acc);
    if (MODE == GAUSS_PHASE && (acc.bad || !isfinite(acc.sx) || !isfinite(acc.sy)))
        // coincident vertices, w == 0, underflow or NaN input: the exact per-pair path
        return lane_strip<GAUSS_ATAN, FULL>(X, Y, Z, row_off, nrows, col_off, row0, c0, c1, kv);
    const double frac = MODE == GAUSS_ATAN ? acc.ang * kInvTwoPi : atan2(acc.sy, acc.sx) * kInvTwoPi;
    return (double)acc.turns + 0.5 * (double)acc.halves + frac;
}

// GAUSS_REF: the reference formula per pair from scratch (two atan2, no contraction).
__device__ double lane_strip_ref(const double *__restrict__ X, const double *__restrict__ Y,
                                 const double *__restrict__ Z, int64_t row_off, int nrows, int64_t col_off, int row0,
                                 int c0, int c1) {
    double kx[R + 1], ky[R + 1], kz[R + 1];
#pragma unroll
    for (int m = 0; m <= R; ++m) {
        const int v = min(row0 + m, nrows);
        kx[m] = __ldg(X + row_off + v);
        ky[m] = __ldg(Y + row_off + v);
        kz[m] = __ldg(Z + row_off + v);
    }
    double acc = 0.0;
    double lx = __ldg(X + col_off + c0), ly = __ldg(Y + col_off + c0), lz = __ldg(Z + col_off + c0);
    for (int c = c0; c < c1; ++c) {
        const double nx = __ldg(X + col_off + c + 1), ny = __ldg(Y + col_off + c + 1), nz = __ldg(Z + col_off + c + 1);
#pragma unroll
        for (int m = 0; m < R; ++m) {
            if (row0 + m < nrows)
                acc = __dadd_rn(acc, ref_pair_lambda(lx, ly, lz, nx, ny, nz, kx[m], ky[m], kz[m], kx[m + 1], ky[m + 1],
                                                     kz[m + 1]));
        }
        lx = nx;
        ly = ny;
        lz = nz;
    }
    return acc;
}

// GAUSS_ANGLESUM: outer segment `row` of _link_angle_sum (direct.py:75-134) over
// all inner segments in order, in the reference's operation order (explicit _rn:
// no contraction, like numba fastmath=False).  The coordinates are scaled by an
// exact power of two, which every operation here carries exactly (the crossing
// decisions and the normalized phase are bitwise the unscaled ones).
__device__ __forceinline__ double sgn_rs(double x, double y) {   // _sgn (direct.py:68-72)
    return (y > 0.0 || (y == 0.0 && x < 0.0)) ? 1.0 : -1.0;
}

__device__ double lane_anglesum(const double *__restrict__ X, const double *__restrict__ Y,
                                const double *__restrict__ Z, int64_t row_off, int row, int64_t col_off, int ncols) {
#define S_(a, b) __dsub_rn(a, b)
#define A_(a, b) __dadd_rn(a, b)
#define M_(a, b) __dmul_rn(a, b)
    const double kix = __ldg(X + row_off + row), kiy = __ldg(Y + row_off + row), kiz = __ldg(Z + row_off + row);
    const double ki1x = __ldg(X + row_off + row + 1), ki1y = __ldg(Y + row_off + row + 1),
                 ki1z = __ldg(Z + row_off + row + 1);
    double xs = 1.0, ys = 0.0, s_prev = -1.0, lam = 0.0;
    double ljx = __ldg(X + col_off), ljy = __ldg(Y + col_off), ljz = __ldg(Z + col_off);
    for (int j = 0; j < ncols; ++j) {
        const double lj1x = __ldg(X + col_off + j + 1), lj1y = __ldg(Y + col_off + j + 1),
                     lj1z = __ldg(Z + col_off + j + 1);
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
        const double xp = S_(M_(d1, d2), M_(p, p));
        const double yp = M_(p, A_(d1, d2));
        const double s1 = sgn_rs(d1, p), sw = sgn_rs(xp, yp);
        if (s1 * sgn_rs(d2, p) > 0.0 && s1 * sw < 0.0) lam = A_(lam, s1);
        const double xpp = S_(M_(xs, xp), M_(ys, yp));
        const double ypp = A_(M_(xs, yp), M_(ys, xp));
        const double sn = sgn_rs(xpp, ypp);
        if (sw * s_prev > 0.0 && sn * s_prev < 0.0) lam = A_(lam, s_prev);
        s_prev = sn;
        const double axp = fabs(xpp), ayp = fabs(ypp);
        const double nrm = ayp > axp ? ayp : axp;   // Python max(a, b): b only if b > a
        xs = __ddiv_rn(xpp, nrm);
        ys = __ddiv_rn(ypp, nrm);
        ljx = lj1x;
        ljy = lj1y;
        ljz = lj1z;
    }
    return A_(lam, __ddiv_rn(atan2(ys, xs), kTwoPi));
#undef S_
#undef A_
#undef M_
}

__device__ __forceinline__ int64_t find_pair(const int64_t *__restrict__ item_off, int64_t P, int64_t it) {
    // largest p with item_off[p] <= it
    int64_t lo = 0, hi = P;   // item_off[P] > it
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(item_off + mid) <= it) lo = mid; else hi = mid;
    }
    return lo;
}

// Lane `vl`'s strip of work item (ir, ic) of pair tiling g, before the butterfly:
// row block vl & (2^rb - 1) of row group ir, column strip vl >> rb of column group ic.
template <int MODE, bool KSM>
__device__ __forceinline__ double vlane_value(const double *__restrict__ X, const double *__restrict__ Y,
                                              const double *__restrict__ Z, const PairGeom &g, int ir, int ic, int vl,
                                              double *ksh, NextItem pf = {nullptr, 0, 0}) {
    const int rbm = (1 << g.rb_log2) - 1;
    const int my_rb = vl & rbm, my_cs = vl >> g.rb_log2;
    const int row0 = ((ir << g.rb_log2) + my_rb) * R;
    const int64_t c0l = ((int64_t)ic * (32 >> g.rb_log2) + my_cs) * g.cl;
    const int c0 = (int)(c0l < g.ncols ? c0l : g.ncols);
    const int c1 = min(c0 + g.cl, g.ncols);
    double val = 0.0;
    if constexpr (MODE == GAUSS_ANGLESUM) {   // items of 32 whole rows: lane = row
        const int row = (ir << 5) + vl;
        if (row < g.nrows) val = lane_anglesum(X, Y, Z, g.row_off, row, g.col_off, g.ncols);
    } else if (row0 < g.nrows && c0 < c1) {
        if (MODE == GAUSS_REF) {
            val = lane_strip_ref(X, Y, Z, g.row_off, g.nrows, g.col_off, row0, c0, c1);
        } else if (KSM) {
            KSm kv{ksh + threadIdx.x};
            val = row0 + R <= g.nrows
                      ? lane_strip<MODE, true>(X, Y, Z, g.row_off, g.nrows, g.col_off, row0, c0, c1, kv)
                      : lane_strip<MODE, false>(X, Y, Z, g.row_off, g.nrows, g.col_off, row0, c0, c1, kv);
        } else {
            KReg kv;
            val = row0 + R <= g.nrows
                      ? lane_strip<MODE, true>(X, Y, Z, g.row_off, g.nrows, g.col_off, row0, c0, c1, kv, pf, vl)
                      : lane_strip<MODE, false>(X, Y, Z, g.row_off, g.nrows, g.col_off, row0, c0, c1, kv, pf, vl);
        }
    }
    return val;
}

// One work item (row-block group ir, column-strip group ic of pair tiling g):
// every lane's strip, then the fixed xor butterfly.  Returns the butterfly sum
// (lane 0's value is the item partial of every path).
template <int MODE, bool KSM>
__device__ __forceinline__ double item_value(const double *__restrict__ X, const double *__restrict__ Y,
                                             const double *__restrict__ Z, const PairGeom &g, int ir, int ic, int lane,
                                             double *ksh, NextItem pf = {nullptr, 0, 0}) {
    double val = vlane_value<MODE, KSM>(X, Y, Z, g, ir, ic, lane, ksh, pf);
#pragma unroll
    for (int off = 16; off; off >>= 1) val += __shfl_xor_sync(0xffffffffu, val, off);
    return val;
}

// Claim the next unit of work (item or pair) for the whole warp; the abort flag
// (fused path: the concurrent pass-1 checks found the run unusable, a staged
// rerun follows) is read with the claim so both round trips overlap.  Returns
// false when the warp should leave.
__device__ __forceinline__ bool claim(unsigned long long *counter, const int *abort, int lane, int64_t &k) {
    unsigned long long c = 0;
    int ab = 0;
    if (lane == 0) {
        c = atomicAdd(counter, 1ULL);
        if (abort) ab = *(volatile const int *)abort;
    }
    k = (int64_t)__shfl_sync(0xffffffffu, c, 0);
    return !__shfl_sync(0xffffffffu, ab, 0);
}

template <int MODE, int MINB, bool KSM = false>
__global__ void __launch_bounds__(kCtaThreads, MINB) gauss_items_kernel(
    const double *__restrict__ X, const double *__restrict__ Y, const double *__restrict__ Z,
    const ItemRec *__restrict__ items, int64_t item_begin, int64_t item_end, unsigned long long *__restrict__ counter,
    double *__restrict__ partials, const int64_t *__restrict__ d_end, int shard, int shards,
    const int *__restrict__ abort, const int64_t *__restrict__ d_bounds) {
    __shared__ double ksh[KSM ? 3 * (R + 1) * kCtaThreads : 1];
    const int lane = threadIdx.x & 31;
    if (d_bounds) {   // sharded: this shard's cost-balanced item range (shard_bounds_kernel)
        item_begin = d_bounds[shard];
        item_end = d_bounds[shard + 1];
    } else if (d_end) {   // item count on the device
        const int64_t n = *d_end;
        if (n < item_end) item_end = n;
    }
#if LC_ITEMS_PREFETCH
    // the next claim and its record are fetched while the current item is summed, and
    // its first vertex lines are prefetched into L1 (LC_PAIRS_L1PF)
    int64_t k1;
    bool ok1 = claim(counter, abort, lane, k1);
    ItemRec r1 = {};
    if (ok1 && item_begin + k1 < item_end) r1 = items[item_begin + k1];
    for (;;) {
        if (!ok1) break;
        const int64_t it = item_begin + k1;
        if (it >= item_end) break;
        const ItemRec rec = r1;
        ok1 = claim(counter, abort, lane, k1);
        const bool nx = ok1 && item_begin + k1 < item_end;
        if (nx) r1 = items[item_begin + k1];
        const NextItem pf{(LC_PAIRS_L1PF && nx) ? &r1.g : nullptr, r1.ir, r1.ic};
        const double val = item_value<MODE, KSM>(X, Y, Z, rec.g, rec.ir, rec.ic, lane, ksh, pf);
        if (lane == 0) partials[it] = val;
    }
#else
    for (;;) {
        int64_t k;
        if (!claim(counter, abort, lane, k)) break;
        const int64_t it = item_begin + k;
        if (it >= item_end) break;
        const ItemRec rec = items[it];
        const double val = item_value<MODE, KSM>(X, Y, Z, rec.g, rec.ir, rec.ic, lane, ksh);
        if (lane == 0) partials[it] = val;
    }
#endif
}

// Fused path: warps claim whole PAIRS (loops of <= 256 segments: 1-2 items each)
// and evaluate the pair's items in order, so no per-item records are built.
// The pair sum is formed exactly as warp_pair_sum forms it from the item
// partials (item k's partial — lane 0's butterfly value — added into lane k mod
// 32, then the xor butterfly), so raw is bitwise the staged path's.  Unsharded:
// raw / lk / flags go to the device arrays and straight into the pinned result
// arrays (zero-copy writes spread over the kernel: no export pass after it).
// Sharded: raw goes to partials[p] (the exchange buffer) for the pairs of this
// shard's cost-balanced range.
template <int MODE, int MINB>
__global__ void __launch_bounds__(kCtaThreads, MINB) gauss_pairs_kernel(
    const double *__restrict__ X, const double *__restrict__ Y, const double *__restrict__ Z,
    const PairGeom *__restrict__ pg, const int64_t *__restrict__ dP, int64_t pcap,
    unsigned long long *__restrict__ counter, const int *__restrict__ abort, const int64_t *__restrict__ d_bounds,
    int shard, double *__restrict__ partials, double *__restrict__ raw, int64_t *__restrict__ lk,
    uint8_t *__restrict__ flags, double *__restrict__ h_raw, int64_t *__restrict__ h_lk,
    uint8_t *__restrict__ h_flags, const EarlyExitArgs ee) {
#if LC_EXPORT_PDL
    LC_PDL_TRIGGER();   // the status export after the sum may become resident (it waits for the sum)
#endif
    const int lane = threadIdx.x & 31;
    int64_t b = 0, e = *dP < pcap ? *dP : pcap;
    if (d_bounds) {
        b = d_bounds[shard];
        e = d_bounds[shard + 1];
    }
#if LC_PAIRS_PREFETCH
    // two-stage software pipeline of the per-pair prologue: the claim of pair n+2 and the
    // PairGeom load of pair n+1 are issued while pair n is summed, so a pair starts with
    // its vertex loads instead of claim -> geometry -> vertices (three dependent round trips)
    int64_t k1, k2;
    bool ok1 = claim(counter, abort, lane, k1);
    bool ok2 = ok1 && claim(counter, abort, lane, k2);
    PairGeom g1 = {};
    if (ok1 && b + k1 < e) g1 = pg[b + k1];
    for (;;) {
        if (!ok1) break;
        const int64_t p = b + k1;
        if (p >= e) break;
        const PairGeom g = g1;
        ok1 = ok2;
        k1 = k2;
        if (ok1 && b + k1 < e) g1 = pg[b + k1];
        if (ok1) ok2 = claim(counter, abort, lane, k2);
#else
    for (;;) {
        int64_t k;
        if (!claim(counter, abort, lane, k)) break;
        const int64_t p = b + k;
        if (p >= e) break;
        const PairGeom g = pg[p];
#endif
        if (ee.posv) {   // early exit: a pair past the first failure found so far is cancelled
            if ((unsigned long long)ee.posv[p] > *(volatile unsigned long long *)ee.first_fail) continue;
            if (lane == 0) atomicAdd(ee.n_eval, 1ULL);
        }
        const int n = g.items_r * g.items_c;
        double s = 0.0;
        for (int it = 0; it < n; ++it) {
#if LC_PAIRS_L1PF && LC_PAIRS_PREFETCH
            const NextItem pf{(it == 0 && ok1 && b + k1 < e) ? &g1 : nullptr, 0, 0};   // the next pair's item 0
#else
            const NextItem pf{nullptr, 0, 0};
#endif
            const double v = __shfl_sync(0xffffffffu, item_value<MODE, false>(X, Y, Z, g, it / g.items_c,
                                                                                it % g.items_c, lane, nullptr, pf), 0);
            if (lane == (it & 31)) s += v;
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) {
            if (partials) {
                partials[p] = s;
            } else {
                int64_t r;
                const uint8_t f = round_link(s, r);
                raw[p] = s;
                lk[p] = r;
                flags[p] = f;
#ifndef LC_AB_NO_HOSTW
                h_raw[p] = s;
                h_lk[p] = r;
                h_flags[p] = f;
#endif
                // NaN / ambiguous raw: compute_link raises there (kernels.py:68-73), which ends the
                // reference's evaluation order too
                if (ee.posv && (r != ee.want[p] || f)) atomicMin(ee.first_fail, (unsigned long long)ee.posv[p]);
            }
        }
    }
}

__global__ void pair_geom_kernel(const int32_t *__restrict__ pairs, int64_t P, const int64_t *__restrict__ dP,
                                 const int64_t *__restrict__ voff, PairGeom *__restrict__ pg,
                                 int64_t *__restrict__ nitems, bool seq, int max_cl) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    if (dP && p >= *dP) {   // fused path: capacity slots beyond the device pair count hold no items
        nitems[p] = 0;
        return;
    }
    const int i = pairs[2 * p], j = pairs[2 * p + 1];
    const PairGeom g = make_pair_geom(voff[i], voff[j], (int)(voff[i + 1] - voff[i] - 1),
                                      (int)(voff[j + 1] - voff[j] - 1), seq, max_cl);
    pg[p] = g;
    nitems[p] = (int64_t)g.items_r * g.items_c;
}

__global__ void reduce_pairs_kernel(const double *__restrict__ partials, const int64_t *__restrict__ item_off,
                                    int64_t P, const int64_t *__restrict__ dP, double *__restrict__ raw,
                                    int64_t *__restrict__ lk, uint8_t *__restrict__ flags) {
    const int lane = threadIdx.x & 31;
    if (dP && *dP < P) P = *dP;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; p < P; p += nwarps) {
        const double s = warp_pair_sum(partials, item_off[p], item_off[p + 1], lane);
        if (lane == 0) {
            raw[p] = s;
            int64_t r;
            flags[p] = round_link(s, r);
            lk[p] = r;
        }
    }
}

__global__ void pack_closed_soa_kernel(const double *__restrict__ aos, const int64_t *__restrict__ in_off,
                                       const int64_t *__restrict__ voff, int64_t L, int64_t total,
                                       const int *__restrict__ d_exp, double *__restrict__ X,
                                       double *__restrict__ Y, double *__restrict__ Z) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= total) return;
    // loop of closed vertex v: largest loop with voff[loop] <= v
    int64_t lo = 0, hi = L;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (voff[mid] <= v) lo = mid; else hi = mid;
    }
    const int64_t local = v - voff[lo];
    const int64_t n = in_off[lo + 1] - in_off[lo];
    const int64_t src = in_off[lo] + (local < n ? local : 0);   // closing vertex repeats vertex 0
    int e = *d_exp - 1023;                                         // unbiased exponent of max |coord|
    e = e < -1022 ? -1022 : (e > 1022 ? 1022 : e);
    const double scale = __hiloint2double((1023 - e) << 20, 0);   // 2^-e, exact
    X[v] = aos[3 * src + 0] * scale;
    Y[v] = aos[3 * src + 1] * scale;
    Z[v] = aos[3 * src + 2] * scale;
}

__global__ void max_exponent_kernel(const double *__restrict__ a, int64_t n, int *__restrict__ d_exp) {
    int best = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const int e = (__double2hiint(a[k]) >> 20) & 0x7ff;
        best = e > best ? e : best;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        const int o = __shfl_xor_sync(0xffffffffu, best, off);
        best = o > best ? o : best;
    }
    if ((threadIdx.x & 31) == 0 && best > 0) atomicMax(d_exp, best);
}

__global__ void segment_pairs_kernel(const double *__restrict__ q, int64_t n, double *__restrict__ out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double *a = q + 12 * k;   // l_j, l_j1, k_i, k_i1 (direct.py:137-146)
    out[k] = ref_pair_lambda(a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], a[9], a[10], a[11]);
}

__device__ __forceinline__ ItemRec make_item(const PairGeom &g, int64_t local) {
    ItemRec r;
    r.g = g;
    r.ir = (int32_t)(local / g.items_c);
    r.ic = (int32_t)(local % g.items_c);
    return r;
}

__global__ void item_pair_kernel(const int64_t *__restrict__ item_off, const PairGeom *__restrict__ pg, int64_t P,
                                 int64_t n_items, ItemRec *__restrict__ items) {
    const int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (it >= n_items) return;
    const int64_t p = find_pair(item_off, P, it);
    items[it] = make_item(pg[p], it - item_off[p]);
}

// Fused path: warp per pair writes its item range (item count not known on the host).
__global__ void item_pair_fill_kernel(const int64_t *__restrict__ item_off, const PairGeom *__restrict__ pg, int64_t P,
                                      const int64_t *__restrict__ dP, int64_t cap_items, ItemRec *__restrict__ items) {
    const int lane = threadIdx.x & 31;
    if (*dP < P) P = *dP;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; p < P; p += nwarps) {
        const int64_t b = item_off[p], e = item_off[p + 1] < cap_items ? item_off[p + 1] : cap_items;
        const PairGeom g = pg[p];
        for (int64_t it = b + lane; it < e; it += 32) items[it] = make_item(g, it - b);
    }
}

// Cost-balanced split of the item list over `shards` ranks: the cost
// of pair p is nrows x ncols segment pairs; boundary k sits where the running
// cost crosses floor(k * total / shards), inside pair p at item
// item_off[p] + ceil((t_k - C_p) * items_p / cost_p) (items of a pair are
// near-equal).  One block; bounds[0] = 0, bounds[shards] = the item count.
// Segment pairs of the first k items of pair tiling g (items in order: ir * items_c + ic;
// only the last item row / column of a pair is partial).
__device__ __forceinline__ int64_t items_prefix_cost(const PairGeom &g, int64_t k, bool seq) {
    const int64_t rows_per = seq ? 32 : (int64_t)kRowsPerLane << g.rb_log2;
    const int64_t span = seq ? g.ncols : (int64_t)(32 >> g.rb_log2) * g.cl;
    const int64_t ir = k / g.items_c, ic = k % g.items_c;
    const int64_t rows_done = ir * rows_per < g.nrows ? ir * rows_per : g.nrows;
    const int64_t rows_cur = g.nrows - rows_done < rows_per ? g.nrows - rows_done : rows_per;
    const int64_t cols_done = ic * span < g.ncols ? ic * span : g.ncols;
    return rows_done * g.ncols + rows_cur * cols_done;
}

__global__ void __launch_bounds__(1024) shard_bounds_kernel(const PairGeom *__restrict__ pg,
                                                            const int64_t *__restrict__ item_off, int64_t Pcap,
                                                            const int64_t *__restrict__ dP, int shards,
                                                            int64_t *__restrict__ bounds, bool seq) {
    __shared__ int64_t wsum[32];
    __shared__ int64_t s_total, s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int64_t P = dP && *dP < Pcap ? *dP : Pcap;
    int64_t part = 0;
    for (int64_t p = tid; p < P; p += blockDim.x) part += (int64_t)pg[p].nrows * pg[p].ncols;
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) wsum[warp] = part;
    __syncthreads();
    if (tid == 0) {
        int64_t t = 0;
        for (int w = 0; w < nw; ++w) t += wsum[w];
        s_total = t;
        s_carry = 0;
        const int64_t n = P > 0 ? (item_off ? item_off[P] : P) : 0;   // item_off null: pair ranges
        bounds[0] = 0;
        for (int k = 1; k <= shards; ++k) bounds[k] = n;
    }
    __syncthreads();
    const int64_t total = s_total;
    for (int64_t base = 0; base < P; base += blockDim.x) {
        const int64_t p = base + tid;
        const int64_t c = p < P ? (int64_t)pg[p].nrows * pg[p].ncols : 0;
        int64_t incl = c;   // inclusive block scan of the pair costs
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        __syncthreads();
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int64_t before = 0;
        for (int w = 0; w < warp; ++w) before += wsum[w];
        const int64_t excl = s_carry + before + incl - c;
        if (p < P && c > 0)
            for (int k = 1; k < shards; ++k) {
                const int64_t t = (int64_t)((__int128)total * k / shards);
                if (excl <= t && t < excl + c) {
                    // the first item of the pair that starts at or after the target cost
                    const int64_t items_p = item_off ? item_off[p + 1] - item_off[p] : 1;
                    int64_t lo = 0, hi = items_p;
                    if (item_off) {
                        const PairGeom g = pg[p];
                        while (lo < hi) {
                            const int64_t mid = (lo + hi) >> 1;
                            if (items_prefix_cost(g, mid, seq) >= t - excl) hi = mid; else lo = mid + 1;
                        }
                    } else {
                        lo = t > excl ? 1 : 0;
                    }
                    bounds[k] = (item_off ? item_off[p] : p) + lo;
                }
            }
        __syncthreads();
        if (tid == blockDim.x - 1) s_carry += before + incl;
        __syncthreads();
    }
}

}  // namespace

void launch_shard_bounds(const PairGeom *pg, const int64_t *item_off, int64_t Pcap, const int64_t *d_P, int shards,
                         int64_t *bounds, cudaStream_t s, bool seq) {
    shard_bounds_kernel<<<1, 1024, 0, s>>>(pg, item_off, Pcap, d_P, shards, bounds, seq);
    LC_CHECK_LAUNCH();
}

void launch_item_pairs_dev(const int64_t *item_off, const PairGeom *pg, int64_t P_cap, const int64_t *d_P,
                           int64_t cap_items, ItemRec *items, cudaStream_t s) {
    if (P_cap == 0) return;
    int64_t blocks = ceil_div(P_cap * 32, 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    item_pair_fill_kernel<<<(unsigned)blocks, 256, 0, s>>>(item_off, pg, P_cap, d_P, cap_items, items);
    LC_CHECK_LAUNCH();
}

void launch_item_pairs(const int64_t *item_off, const PairGeom *pg, int64_t P, int64_t n_items, ItemRec *items,
                       cudaStream_t s) {
    if (n_items == 0) return;
    item_pair_kernel<<<(unsigned)ceil_div(n_items, 256), 256, 0, s>>>(item_off, pg, P, n_items, items);
    LC_CHECK_LAUNCH();
}

void launch_segment_pairs(const double *quads, int64_t n, double *out, cudaStream_t s) {
    if (n == 0) return;
    segment_pairs_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, s>>>(quads, n, out);
    LC_CHECK_LAUNCH();
}

void launch_max_exponent(const double *aos, int64_t n, int *d_exp, cudaStream_t s) {
    if (n == 0) return;
    int64_t blocks = ceil_div(n, 256);
    if (blocks > 4 * 148) blocks = 4 * 148;
    max_exponent_kernel<<<(unsigned)blocks, 256, 0, s>>>(aos, n, d_exp);
    LC_CHECK_LAUNCH();
}

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        LC_CUDA(cudaGetDevice(&dev));
        LC_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    }
    return n;
}

size_t build_items_scan_bytes(int64_t P) { return exclusive_scan_i64_tmp_bytes(P + 1) + 16; }

int64_t build_items(const int32_t *d_pairs, int64_t P, const int64_t *d_voff, PairGeom *d_pg,
                    int64_t *d_item_off, void *d_scan_tmp, size_t scan_tmp_bytes, cudaStream_t s, bool read_back,
                    const int64_t *d_P, bool seq, int max_cl) {
    if (P == 0) {
        LC_CUDA(cudaMemsetAsync(d_item_off, 0, sizeof(int64_t), s));
        return 0;
    }
    // nitems written into item_off[0..P), item_off[P] = 0, then in-place exclusive scan.
    LC_CUDA(cudaMemsetAsync(d_item_off + P, 0, sizeof(int64_t), s));
    pair_geom_kernel<<<(unsigned)ceil_div(P, 256), 256, 0, s>>>(d_pairs, P, d_P, d_voff, d_pg, d_item_off, seq,
                                                                 max_cl);
    LC_CHECK_LAUNCH();
    exclusive_scan_i64(d_item_off, d_item_off, P + 1, d_scan_tmp, scan_tmp_bytes, s);
    if (!read_back) return -1;   // caller reads item_off[P] together with other results
    int64_t total = 0;
    LC_CUDA(cudaMemcpyAsync(&total, d_item_off + P, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
    return total;
}

void launch_gauss_items(int mode, const double *X, const double *Y, const double *Z, const ItemRec *items,
                        int64_t item_begin,
                        int64_t item_end, unsigned long long *counter, double *partials, cudaStream_t s,
                        const int64_t *d_end, int shard, int shards, const int *abort, bool counter_zeroed,
                        const int64_t *d_bounds) {
    if (item_end <= item_begin) return;
    if (!counter_zeroed) LC_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s));
    using Kern = void (*)(const double *, const double *, const double *, const ItemRec *, int64_t, int64_t,
                          unsigned long long *, double *, const int64_t *, int, int, const int *, const int64_t *);
    // default phase kernel: 3 resident CTAs/SM (168 regs); modes 16-20 are A/B variants
    // (1 CTA/SM with 232 regs; 4 CTAs; row vertices in shared memory; 2 CTAs/SM)
    static const Kern table[] = {gauss_items_kernel<GAUSS_PHASE, LC_MINB>, gauss_items_kernel<GAUSS_ATAN, 1>,
                                 gauss_items_kernel<GAUSS_REF, 1>,         gauss_items_kernel<GAUSS_ANGLESUM, 4>,
                                 gauss_items_kernel<GAUSS_PHASE, 1>,       gauss_items_kernel<GAUSS_PHASE, 4>,
                                 gauss_items_kernel<GAUSS_PHASE, 4, true>, gauss_items_kernel<GAUSS_PHASE, 3, true>,
                                 gauss_items_kernel<GAUSS_PHASE, 2>};
    if (!gauss_mode_valid(mode)) throw Error(LC_ERR_ARG, "unknown Gauss-sum mode");
    const int slot = mode < GAUSS_AB_FIRST ? mode : mode - GAUSS_AB_FIRST + 4;
    const Kern fn = table[slot];
    constexpr int kModes = (int)(sizeof table / sizeof table[0]);
    static int occ[kModes] = {};   // resident CTAs per SM, queried once per mode
    const int threads = 128;
    if (!occ[slot]) {
        LC_CUDA(cudaFuncSetAttribute((const void *)fn, cudaFuncAttributePreferredSharedMemoryCarveout, kGaussCarveout));
        int per = 0;
        LC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void *)fn, threads, 0));
        occ[slot] = per < 1 ? 1 : per;
    }
    const int per_sm = occ[slot];
    const int64_t warps_needed = item_end - item_begin;
    int64_t blocks = (int64_t)num_sms() * per_sm;
    const int64_t blocks_needed = ceil_div(warps_needed, threads / 32);
    if (blocks > blocks_needed) blocks = blocks_needed;
    fn<<<(unsigned)blocks, threads, 0, s>>>(X, Y, Z, items, item_begin, item_end, counter, partials, d_end, shard,
                                            shards, abort, d_bounds);
    LC_CHECK_LAUNCH();
}

void launch_gauss_pairs(int mode, const double *X, const double *Y, const double *Z, const PairGeom *pg,
                        const int64_t *d_P, int64_t pcap, unsigned long long *counter, const int *abort,
                        const int64_t *d_bounds, int shard, double *partials, double *raw, int64_t *lk, uint8_t *flags,
                        double *h_raw, int64_t *h_lk, uint8_t *h_flags, cudaStream_t s, const EarlyExitArgs &ee,
                        bool pdl) {
    if (pcap <= 0) return;
    using Kern = void (*)(const double *, const double *, const double *, const PairGeom *, const int64_t *, int64_t,
                          unsigned long long *, const int *, const int64_t *, int, double *, double *, int64_t *,
                          uint8_t *, double *, int64_t *, uint8_t *, const EarlyExitArgs);
    Kern fn;
    switch (mode) {
        case GAUSS_PHASE: fn = gauss_pairs_kernel<GAUSS_PHASE, LC_PAIRS_MINB>; break;
        case GAUSS_ATAN: fn = gauss_pairs_kernel<GAUSS_ATAN, 1>; break;
        case GAUSS_REF: fn = gauss_pairs_kernel<GAUSS_REF, 1>; break;
        default: throw Error(LC_ERR_ARG, "the pair-claiming Gauss kernel takes modes phase / atan / ref");
    }
    static int occ[3] = {};
    const int threads = kCtaThreads;
    if (!occ[mode]) {
        // keep a slice of the SM's unified L1 as shared memory: the pass-1 checks
        // (brute_any_lite, 4.6 KB of shared memory per block) then co-reside with the
        // persistent Gauss CTAs instead of waiting for them to exit
        LC_CUDA(cudaFuncSetAttribute((const void *)fn, cudaFuncAttributePreferredSharedMemoryCarveout, kGaussCarveout));
        int per = 0;
        LC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void *)fn, threads, 0));
        occ[mode] = per < 1 ? 1 : per;
    }
    int64_t blocks = (int64_t)num_sms() * occ[mode];
    const int64_t need = ceil_div(pcap, threads / 32);
    if (blocks > need) blocks = need;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(threads);
    cfg.stream = s;
    // pdl: a programmatic dependent of the kernel before it on the stream (the pass-1
    // check), launched once that kernel's CTAs are all resident
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    LC_CUDA(cudaLaunchKernelEx(&cfg, fn, X, Y, Z, pg, d_P, pcap, counter, abort, d_bounds, shard, partials, raw, lk,
                               flags, h_raw, h_lk, h_flags, ee));
    LC_CHECK_LAUNCH();
}

namespace {
__device__ __forceinline__ int64_t find_key(const uint64_t *__restrict__ keys, int64_t n, uint64_t k) {
    int64_t lo = 0, hi = n;   // first index with keys[idx] >= k
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < k) lo = mid + 1; else hi = mid;
    }
    return lo < n && keys[lo] == k ? lo : -1;
}

__device__ __forceinline__ uint64_t pair_key(const int32_t *__restrict__ pairs, int64_t p) {
    return ((uint64_t)(uint32_t)pairs[2 * p] << 32) | (uint32_t)pairs[2 * p + 1];
}

// Threads [0, pcap): candidate pairs; threads [pcap, pcap + n_ref): certificate entries.
__global__ void early_exit_order_kernel(const int32_t *__restrict__ pairs, const int64_t *__restrict__ dP,
                                        int64_t pcap, const uint64_t *__restrict__ ref_keys,
                                        const int64_t *__restrict__ ref_lk, int64_t n_ref,
                                        int64_t *__restrict__ posv, int64_t *__restrict__ want,
                                        unsigned long long *__restrict__ first_fail) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t P = *dP < pcap ? *dP : pcap;
    if (t < pcap) {
        if (t >= P) return;
        const int64_t r = find_key(ref_keys, n_ref, pair_key(pairs, t));
        posv[t] = r >= 0 ? r : n_ref + t;   // certificate pairs first, then the other candidates
        want[t] = r >= 0 ? ref_lk[r] : 0;
        return;
    }
    const int64_t r = t - pcap;
    if (r >= n_ref) return;
    // binary search of the certificate pair among the P sorted candidates
    const uint64_t k = ref_keys[r];
    int64_t lo = 0, hi = P;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (pair_key(pairs, mid) < k) lo = mid + 1; else hi = mid;
    }
    if (!(lo < P && pair_key(pairs, lo) == k) && ref_lk[r] != 0)
        atomicMin(first_fail, (unsigned long long)r);   // not a candidate: computed as 0 (certify.py:203-206)
}
}  // namespace

void launch_early_exit_order(const int32_t *pairs, const int64_t *d_P, int64_t pcap, const uint64_t *ref_keys,
                             const int64_t *ref_lk, int64_t n_ref, int64_t *posv, int64_t *want,
                             unsigned long long *first_fail, cudaStream_t s) {
    const int64_t n = pcap + n_ref;
    if (n <= 0) return;
    early_exit_order_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(pairs, d_P, pcap, ref_keys, ref_lk, n_ref, posv,
                                                                       want, first_fail);
    LC_CHECK_LAUNCH();
}

void launch_reduce_pairs(const double *partials, const int64_t *item_off, int64_t P, double *raw, int64_t *lk,
                         uint8_t *flags, cudaStream_t s, const int64_t *d_P) {
    if (P == 0) return;
    int64_t blocks = ceil_div(P * 32, 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    reduce_pairs_kernel<<<(unsigned)blocks, 256, 0, s>>>(partials, item_off, P, d_P, raw, lk, flags);
    LC_CHECK_LAUNCH();
}

void launch_pack_closed_soa(const double *aos, const int64_t *in_off, const int64_t *voff, int64_t L,
                            int64_t total_closed, const int *d_exp, double *X, double *Y, double *Z,
                            cudaStream_t s) {
    if (total_closed == 0) return;
    pack_closed_soa_kernel<<<(unsigned)ceil_div(total_closed, 256), 256, 0, s>>>(aos, in_off, voff, L, total_closed,
                                                                                  d_exp, X, Y, Z);
    LC_CHECK_LAUNCH();
}

}  // namespace lc
