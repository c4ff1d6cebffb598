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
// operands are bitwise the ones the reference formula would form.
// Item partials go through a warp butterfly (fixed order) into
// partials[item]; pairs are reduced from their contiguous item range in a
// fixed order, so raw sums are identical run to run and for any split of
// the item range across GPUs.
#include "gauss.cuh"

#include <cub/device/device_scan.cuh>

namespace lc {

namespace {

constexpr double kTwoPi = 6.283185307179586;          // 2.0 * math.pi (direct.py:16)
constexpr double kInvTwoPi = 0.15915494309189535;     // 1 / (2 pi), correctly rounded

__device__ __forceinline__ int sign_bit(double x) { return (int)((unsigned)__double2hiint(x) >> 31); }

// S <- S * (zx + i zy), counting full turns so that
//   arg_total = 2*pi*turns + atan2(S.y, S.x)   (atan2 semantics incl. signed zero)
// Classification by the sign bit of the imaginary part: "upper" = arg in
// [+0, pi], "lower" = arg in [-pi, -0].  Two factors in the same half whose
// product lands in the other half wrapped by one turn in that direction —
// the full-turn rule of _link_angle_sum (direct.py:120-123), which is exact
// given the computed product.
__device__ __forceinline__ void phase_mul(double &sx, double &sy, double zx, double zy, int &turns) {
    const double ux = sx * zx - sy * zy;
    const double uy = sx * zy + sy * zx;
    const int ss = sign_bit(sy), sz = sign_bit(zy), su = sign_bit(uy);
    turns += ((ss == sz) & (su != ss)) ? (1 - 2 * ss) : 0;
    sx = ux;
    sy = uy;
}

// Rescale S by an exact power of two so max(|Sx|,|Sy|) is in [1, 2).
__device__ __forceinline__ void phase_renorm(double &sx, double &sy) {
    const int ex = __double2hiint(sx) & 0x7ff00000;
    const int ey = __double2hiint(sy) & 0x7ff00000;
    const int e = ex > ey ? ex : ey;
    const double scale = __hiloint2double(0x7fe00000 - e, 0);
    sx *= scale;
    sy *= scale;
}

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

// Sum over rows [row0, row0+R) x columns [c0, c1) of one pair, in turns.
template <int MODE>
__device__ double lane_strip(const double *__restrict__ X, const double *__restrict__ Y,
                             const double *__restrict__ Z, int64_t row_off, int nrows,
                             int64_t col_off, int row0, int c0, int c1) {
    constexpr int R = kRowsPerLane;
    double kx[R + 1], ky[R + 1], kz[R + 1];
    bool rv[R];
#pragma unroll
    for (int m = 0; m <= R; ++m) {
        const int v = min(row0 + m, nrows);   // closing vertex sits at index nrows
        kx[m] = __ldg(X + row_off + v);
        ky[m] = __ldg(Y + row_off + v);
        kz[m] = __ldg(Z + row_off + v);
    }
#pragma unroll
    for (int m = 0; m < R; ++m) rv[m] = row0 + m < nrows;

    if (MODE == GAUSS_REF) {
        double acc = 0.0;
        double lx = __ldg(X + col_off + c0), ly = __ldg(Y + col_off + c0), lz = __ldg(Z + col_off + c0);
        for (int c = c0; c < c1; ++c) {
            const double nx = __ldg(X + col_off + c + 1), ny = __ldg(Y + col_off + c + 1),
                         nz = __ldg(Z + col_off + c + 1);
#pragma unroll
            for (int m = 0; m < R; ++m) {
                if (rv[m])
                    acc = __dadd_rn(acc, ref_pair_lambda(lx, ly, lz, nx, ny, nz, kx[m], ky[m], kz[m],
                                                         kx[m + 1], ky[m + 1], kz[m + 1]));
            }
            lx = nx;
            ly = ny;
            lz = nz;
        }
        return acc;
    }

    // Previous column: r(c, m) = l_c - k_m, its norm, and v[m] = r(c,m).r(c,m+1).
    double rx[R + 1], ry[R + 1], rz[R + 1], rn[R + 1], vv[R];
    {
        const double lx = __ldg(X + col_off + c0), ly = __ldg(Y + col_off + c0), lz = __ldg(Z + col_off + c0);
#pragma unroll
        for (int m = 0; m <= R; ++m) {
            rx[m] = lx - kx[m];
            ry[m] = ly - ky[m];
            rz[m] = lz - kz[m];
            rn[m] = sqrt(rx[m] * rx[m] + ry[m] * ry[m] + rz[m] * rz[m]);
        }
#pragma unroll
        for (int m = 0; m < R; ++m) vv[m] = rx[m] * rx[m + 1] + ry[m] * ry[m + 1] + rz[m] * rz[m + 1];
    }

    double sx = 1.0, sy = 0.0;   // PHASE accumulator
    double ang = 0.0;            // ATAN accumulator (radians)
    int turns = 0, halves = 0;

    double nlx = __ldg(X + col_off + c0 + 1), nly = __ldg(Y + col_off + c0 + 1), nlz = __ldg(Z + col_off + c0 + 1);
    for (int c = c0; c < c1; ++c) {
        const double lx = nlx, ly = nly, lz = nlz;
        if (c + 2 <= c1) {
            nlx = __ldg(X + col_off + c + 2);
            nly = __ldg(Y + col_off + c + 2);
            nlz = __ldg(Z + col_off + c + 2);
        }
        double qx[R + 1], qy[R + 1], qz[R + 1], qn[R + 1], hh[R + 1], ww[R];
#pragma unroll
        for (int m = 0; m <= R; ++m) {
            qx[m] = lx - kx[m];
            qy[m] = ly - ky[m];
            qz[m] = lz - kz[m];
            qn[m] = sqrt(qx[m] * qx[m] + qy[m] * qy[m] + qz[m] * qz[m]);
            hh[m] = rx[m] * qx[m] + ry[m] * qy[m] + rz[m] * qz[m];   // r(c,m) . r(c+1,m)
        }
#pragma unroll
        for (int m = 0; m < R; ++m) ww[m] = qx[m] * qx[m + 1] + qy[m] * qy[m + 1] + qz[m] * qz[m + 1];

#pragma unroll
        for (int m = 0; m < R; ++m) {
            // Corner vectors of pair (row m, column c): a = r(c,m), b = r(c,m+1),
            // c = r(c+1,m+1), d = r(c+1,m)  (direct.py:21-32).
            const double ax = rx[m], ay = ry[m], az = rz[m];
            const double bx = rx[m + 1], by = ry[m + 1], bz = rz[m + 1];
            const double cx = qx[m + 1], cy = qy[m + 1], cz = qz[m + 1];
            const double an = rn[m], bn = rn[m + 1], cn = qn[m + 1], dn = qn[m];
            const double ab = vv[m], bc = hh[m + 1], ad = hh[m], dc = ww[m];
            const double ca = cx * ax + cy * ay + cz * az;
            const double p = ax * (by * cz - bz * cy) + ay * (bz * cx - bx * cz) + az * (bx * cy - by * cx);
            const double d1 = an * bn * cn + ab * cn + bc * an + ca * bn;
            const double d2 = an * dn * cn + ad * cn + dc * an + ca * dn;
            if (!rv[m]) continue;
            if (p == 0.0) {
                // atan2(+-0, d) is +-pi for d < 0 or d == -0, else +-0: exact half turns.
                const int hsum = sign_bit(d1) + sign_bit(d2);
                halves += sign_bit(p) ? -hsum : hsum;
            } else if (MODE == GAUSS_PHASE) {
                phase_mul(sx, sy, d1, p, turns);
                phase_mul(sx, sy, d2, p, turns);
            } else {
                const double xp = d1 * d2 - p * p;
                const double yp = p * (d1 + d2);
                ang += atan2(yp, xp);
                const int sp = sign_bit(p);
                turns += (sign_bit(yp) != sp) ? (1 - 2 * sp) : 0;
            }
        }
        if (MODE == GAUSS_PHASE) phase_renorm(sx, sy);
#pragma unroll
        for (int m = 0; m <= R; ++m) {
            rx[m] = qx[m];
            ry[m] = qy[m];
            rz[m] = qz[m];
            rn[m] = qn[m];
        }
#pragma unroll
        for (int m = 0; m < R; ++m) vv[m] = ww[m];
    }
    const double frac = (MODE == GAUSS_PHASE) ? atan2(sy, sx) * kInvTwoPi : ang * kInvTwoPi;
    return (double)turns + 0.5 * (double)halves + frac;
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

template <int MODE>
__global__ void __launch_bounds__(128) gauss_items_kernel(
    const double *__restrict__ X, const double *__restrict__ Y, const double *__restrict__ Z,
    const PairGeom *__restrict__ pg, const int64_t *__restrict__ item_off, int64_t P,
    int64_t item_begin, int64_t item_end, unsigned long long *__restrict__ counter,
    double *__restrict__ partials) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned long long k = 0;
        if (lane == 0) k = atomicAdd(counter, 1ULL);
        k = __shfl_sync(0xffffffffu, k, 0);
        const int64_t it = item_begin + (int64_t)k;
        if (it >= item_end) break;
        const int64_t p = find_pair(item_off, P, it);
        const PairGeom g = pg[p];
        const int64_t local = it - __ldg(item_off + p);
        const int ir = (int)(local / g.items_c), ic = (int)(local % g.items_c);
        const int rbm = (1 << g.rb_log2) - 1;
        const int my_rb = lane & rbm, my_cs = lane >> g.rb_log2;
        const int row0 = ((ir << g.rb_log2) + my_rb) * kRowsPerLane;
        const int64_t c0l = ((int64_t)ic * (32 >> g.rb_log2) + my_cs) * g.cl;
        const int c0 = (int)(c0l < g.ncols ? c0l : g.ncols);
        const int c1 = min(c0 + g.cl, g.ncols);
        double val = 0.0;
        if (row0 < g.nrows && c0 < c1)
            val = lane_strip<MODE>(X, Y, Z, g.row_off, g.nrows, g.col_off, row0, c0, c1);
#pragma unroll
        for (int off = 16; off; off >>= 1) val += __shfl_xor_sync(0xffffffffu, val, off);
        if (lane == 0) partials[it] = val;
    }
}

__global__ void pair_geom_kernel(const int32_t *__restrict__ pairs, int64_t P,
                                 const int64_t *__restrict__ voff, PairGeom *__restrict__ pg,
                                 int64_t *__restrict__ nitems) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int i = pairs[2 * p], j = pairs[2 * p + 1];
    PairGeom g;
    g.col_off = voff[i];
    g.row_off = voff[j];
    g.ncols = (int)(voff[i + 1] - voff[i] - 1);
    g.nrows = (int)(voff[j + 1] - voff[j] - 1);
    const int nb = (g.nrows + kRowsPerLane - 1) / kRowsPerLane;
    int rbl = 0;
    while ((1 << rbl) < nb && rbl < 5) ++rbl;
    g.rb_log2 = rbl;
    const int cs = 32 >> rbl;
    const int cl = (g.ncols + cs - 1) / cs;
    g.cl = cl < kMaxColsPerLane ? (cl > 0 ? cl : 1) : kMaxColsPerLane;
    g.items_r = (g.nrows + (kRowsPerLane << rbl) - 1) / (kRowsPerLane << rbl);
    const int64_t span = (int64_t)cs * g.cl;
    g.items_c = (int)((g.ncols + span - 1) / span);
    if (g.nrows <= 0 || g.ncols <= 0) g.items_r = g.items_c = 0;
    pg[p] = g;
    nitems[p] = (int64_t)g.items_r * g.items_c;
}

__global__ void reduce_pairs_kernel(const double *__restrict__ partials, const int64_t *__restrict__ item_off,
                                    int64_t P, double *__restrict__ raw, int64_t *__restrict__ lk,
                                    uint8_t *__restrict__ flags) {
    const int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= P) return;
    const int64_t b = item_off[p], e = item_off[p + 1];
    double s = 0.0;
    for (int64_t k = b + lane; k < e; k += 32) s += partials[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) {
        raw[p] = s;
        uint8_t f = 0;
        int64_t r = 0;
        if (isnan(s)) {
            f = 1;
        } else {
            const double rr = rint(s);   // half-to-even, like Python round()
            if (fabs(s - rr) > 0.25) f |= 2;
            r = (int64_t)rr;
        }
        lk[p] = r;
        flags[p] = f;
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
    int e = *d_exp - 1023;                       // unbiased exponent of max |coord|
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

}  // namespace

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

size_t build_items_scan_bytes(int64_t P) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int64_t *)nullptr, (int64_t *)nullptr, (int)(P + 1));
    return bytes;
}

int64_t build_items(const int32_t *d_pairs, int64_t P, const int64_t *d_voff, PairGeom *d_pg,
                    int64_t *d_item_off, void *d_scan_tmp, size_t scan_tmp_bytes, cudaStream_t s) {
    if (P == 0) {
        LC_CUDA(cudaMemsetAsync(d_item_off, 0, sizeof(int64_t), s));
        return 0;
    }
    // nitems written into item_off[0..P), item_off[P] = 0, then in-place exclusive scan.
    LC_CUDA(cudaMemsetAsync(d_item_off + P, 0, sizeof(int64_t), s));
    pair_geom_kernel<<<(unsigned)ceil_div(P, 256), 256, 0, s>>>(d_pairs, P, d_voff, d_pg, d_item_off);
    LC_CHECK_LAUNCH();
    size_t bytes = scan_tmp_bytes;
    LC_CUB(cub::DeviceScan::ExclusiveSum(d_scan_tmp, bytes, d_item_off, d_item_off, (int)(P + 1), s));
    int64_t total = 0;
    LC_CUDA(cudaMemcpyAsync(&total, d_item_off + P, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
    return total;
}

void launch_gauss_items(int mode, const double *X, const double *Y, const double *Z, const PairGeom *pg,
                        const int64_t *item_off, int64_t P, int64_t item_begin, int64_t item_end,
                        unsigned long long *counter, double *partials, cudaStream_t s) {
    if (item_end <= item_begin) return;
    LC_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s));
    int per_sm = 0;
    const int threads = 128;
    const void *fn = mode == GAUSS_PHASE ? (const void *)gauss_items_kernel<GAUSS_PHASE>
                     : mode == GAUSS_ATAN ? (const void *)gauss_items_kernel<GAUSS_ATAN>
                                          : (const void *)gauss_items_kernel<GAUSS_REF>;
    LC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0));
    if (per_sm < 1) per_sm = 1;
    const int64_t warps_needed = item_end - item_begin;
    int64_t blocks = (int64_t)num_sms() * per_sm;
    const int64_t blocks_needed = ceil_div(warps_needed, threads / 32);
    if (blocks > blocks_needed) blocks = blocks_needed;
    switch (mode) {
        case GAUSS_PHASE:
            gauss_items_kernel<GAUSS_PHASE><<<(unsigned)blocks, threads, 0, s>>>(X, Y, Z, pg, item_off, P, item_begin, item_end, counter, partials);
            break;
        case GAUSS_ATAN:
            gauss_items_kernel<GAUSS_ATAN><<<(unsigned)blocks, threads, 0, s>>>(X, Y, Z, pg, item_off, P, item_begin, item_end, counter, partials);
            break;
        default:
            gauss_items_kernel<GAUSS_REF><<<(unsigned)blocks, threads, 0, s>>>(X, Y, Z, pg, item_off, P, item_begin, item_end, counter, partials);
            break;
    }
    LC_CHECK_LAUNCH();
}

void launch_reduce_pairs(const double *partials, const int64_t *item_off, int64_t P, double *raw, int64_t *lk,
                         uint8_t *flags, cudaStream_t s) {
    if (P == 0) return;
    reduce_pairs_kernel<<<(unsigned)ceil_div(P * 32, 256), 256, 0, s>>>(partials, item_off, P, raw, lk, flags);
    LC_CHECK_LAUNCH();
}

void launch_pack_closed_soa(const double *aos, const int64_t *in_off, const int64_t *voff, int64_t L,
                            int64_t total_closed, const int *d_exp, double *X, double *Y, double *Z,
                            cudaStream_t s) {
    if (total_closed == 0) return;
    pack_closed_soa_kernel<<<(unsigned)ceil_div(total_closed, 256), 256, 0, s>>>(aos, in_off, voff, L, total_closed, d_exp, X, Y, Z);
    LC_CHECK_LAUNCH();
}

}  // namespace lc
