// Barnes-Hut linking integral on the GPU: moment-tree forests and the
// dual-tree traversal (reference: linkcert/barneshut.py, linkcert/bvh.py).
//
// Compiled with -fmad=false (build.py): every expression below is evaluated
// in the operation order of the reference's numba code (fastmath off, no
// contraction), so node boxes, moments, far-field terms and the opening test
// are bitwise the reference's; only the leaf-pair atan2 (ulps) and the order
// of the final summation differ.
//
// Tree build (bvh._build, bvh.py:17-90, leaf_size 1).  The node ranges of a
// median-split tree depend only on the loop length m, so the node table
// (numbering, start/end, children, depth) is computed in closed form on the
// device (bh_table_kernel, the reference's DFS numbering).  The geometry only decides the permutation:
// level by level, every node's primitives are ordered by (center on the
// node's longest axis, input index).  On the device that is one radix sort of
// all primitives per level with the key (node start, rank of the primitive on
// the node's axis) — ranks per axis come from three global stable sorts, and
// a (center, index) rank order restricted to a node is exactly the
// reference's argsort-with-index-ties.  Node boxes are reduced with ordered
// 64-bit atomics (min / max are order-free, hence exact and deterministic).
//
// Moments (barneshut._compute_moments) bottom-up, one launch per depth over
// the depth-ordered node list, one warp per node (coalesced 384 B records).
//
// Traversal (barneshut._dual_eval): breadth-first over node pairs.  Each
// level's frontier is classified (far field / leaf pair / split); splits are
// expanded to the next frontier at scanned offsets, so the frontier stays in
// pair order and each level's contributions are reduced per pair with
// cub::DeviceReduce::ReduceByKey (fixed decomposition: deterministic).  The
// set of visited node pairs and far/leaf decisions equal the reference's
// depth-first traversal exactly (each decision depends only on the pair).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>

#include "bh.cuh"
#include "geom.cuh"

namespace lc {

namespace {

constexpr double kFourPi = 12.566370614359172;   // 4.0 * math.pi (barneshut.py:22)

__device__ __forceinline__ unsigned long long ord_key(double x) {
    if (x == 0.0) x = 0.0;   // -0.0 == 0.0 in the reference's comparisons
    const unsigned long long u = (unsigned long long)__double_as_longlong(x);
    return (u >> 63) ? ~u : (u | (1ull << 63));
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
    const unsigned long long u = (k >> 63) ? (k & ~(1ull << 63)) : ~k;
    return __longlong_as_double((long long)u);
}

// ------------------------------------------------------------------ build

__global__ void bh_prims_kernel(const double *__restrict__ v, const int64_t *__restrict__ loff,
                                const int64_t *__restrict__ noff, int64_t L, int64_t M, double *__restrict__ seg,
                                unsigned long long *__restrict__ ckey, int *__restrict__ iota, int *__restrict__ order,
                                int *__restrict__ nodeid) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= M) return;
    int64_t lo_t = 0, hi_t = L;   // tree t: loff[t] <= p < loff[t + 1]
    while (hi_t - lo_t > 1) {
        const int64_t mid = (lo_t + hi_t) >> 1;
        if (loff[mid] <= p) lo_t = mid; else hi_t = mid;
    }
    const int64_t nxt = (p + 1 == loff[lo_t + 1]) ? loff[lo_t] : p + 1;   // np.roll(verts, -1)
    double a[3], b[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a[k] = v[3 * p + k];
        b[k] = v[3 * nxt + k];
        seg[6 * p + k] = a[k];
        seg[6 * p + 3 + k] = b[k];
        const double lo = b[k] < a[k] ? b[k] : a[k], hi = b[k] > a[k] ? b[k] : a[k];
        ckey[k * M + p] = ord_key(0.5 * (lo + hi));   // centers = 0.5 * (lo + hi) (bvh.py:20)
    }
    iota[p] = (int)p;
    order[p] = (int)p;
    nodeid[p] = (int)noff[lo_t];
}

__global__ void bh_rank_kernel(const int *__restrict__ sorted_ids, int64_t M, int *__restrict__ rank) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < M) rank[sorted_ids ? sorted_ids[i] : i] = (int)i;   // no ids: iota
}

// Node boxes of depth d: union of the primitive boxes in the node's range.
// Positions of one node are contiguous: a warp-segmented min/max (idempotent)
// leaves each run's value at its first lane, which issues the atomics; a
// block whose positions all lie in one node reduces through shared memory.
__global__ void __launch_bounds__(256) bh_bbox_kernel(const int *__restrict__ nodeid, const int *__restrict__ order,
                                                      const int *__restrict__ depth, int d,
                                                      const double *__restrict__ seg, int64_t M,
                                                      unsigned long long *__restrict__ enc_lo,
                                                      unsigned long long *__restrict__ enc_hi) {
    __shared__ unsigned long long s_v[8][6];
    __shared__ int s_uniform;
    const int64_t base = blockIdx.x * (int64_t)blockDim.x;
    const int64_t p = base + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int node = -1;
    if (p < M) {
        node = nodeid[p];
        if (depth[node] != d) node = -1;
    }
    unsigned long long v[6];
    if (node >= 0) {
        const double *sg = seg + 6 * (int64_t)order[p];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double a = sg[k], b = sg[3 + k];
            v[k] = ord_key(b < a ? b : a);
            v[3 + k] = ord_key(b > a ? b : a);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            v[k] = ~0ull;
            v[3 + k] = 0ull;
        }
    }
    if (threadIdx.x == 0) {
        const int64_t last = (base + blockDim.x <= M ? base + blockDim.x : M) - 1;
        const int n0 = nodeid[base], n1 = nodeid[last];
        s_uniform = (n0 == n1 && depth[n0] == d && last - base + 1 == blockDim.x) ? n0 : -1;
    }
    __syncthreads();
    const int uni = s_uniform;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int on = __shfl_down_sync(0xffffffffu, node, off);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const unsigned long long o = __shfl_down_sync(0xffffffffu, v[k], off);
            if (lane + off < 32 && on == node) v[k] = k < 3 ? (o < v[k] ? o : v[k]) : (o > v[k] ? o : v[k]);
        }
    }
    if (uni >= 0) {
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < 6; ++k) s_v[warp][k] = v[k];
        __syncthreads();
        if (threadIdx.x < 6) {
            const int k = threadIdx.x;
            unsigned long long r = s_v[0][k];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
                const unsigned long long o = s_v[w][k];
                r = k < 3 ? (o < r ? o : r) : (o > r ? o : r);
            }
            if (k < 3) atomicMin(enc_lo + 3 * (int64_t)uni + k, r);
            else atomicMax(enc_hi + 3 * (int64_t)uni + k - 3, r);
        }
        return;
    }
    const int prev = __shfl_up_sync(0xffffffffu, node, 1);
    if (node >= 0 && (lane == 0 || prev != node)) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            atomicMin(enc_lo + 3 * (int64_t)node + k, v[k]);
            atomicMax(enc_hi + 3 * (int64_t)node + k, v[3 + k]);
        }
    }
}

// Sort keys of depth d: (node start, rank on the node's longest axis) for the
// primitives of internal depth-d nodes, (own position, 0) for everything else.
__global__ void bh_key_kernel(const int *__restrict__ nodeid, const int *__restrict__ order,
                              const int *__restrict__ depth, const int *__restrict__ left,
                              const int *__restrict__ start, int d, const unsigned long long *__restrict__ enc_lo,
                              const unsigned long long *__restrict__ enc_hi, const int *__restrict__ rank,
                              int64_t M, int rank_bits, unsigned long long *__restrict__ key) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= M) return;
    const int node = nodeid[p];
    if (depth[node] != d || left[node] < 0) {
        key[p] = (unsigned long long)p << rank_bits;
        return;
    }
    // longest axis of the node box, first axis on ties (bvh.py:56-62)
    int axis = 0;
    double best = ord_val(enc_hi[3 * (int64_t)node]) - ord_val(enc_lo[3 * (int64_t)node]);
#pragma unroll
    for (int k = 1; k < 3; ++k) {
        const double w = ord_val(enc_hi[3 * (int64_t)node + k]) - ord_val(enc_lo[3 * (int64_t)node + k]);
        if (w > best) {
            best = w;
            axis = k;
        }
    }
    key[p] = ((unsigned long long)start[node] << rank_bits) | (unsigned long long)rank[axis * M + order[p]];
}

__global__ void bh_descend_kernel(int *__restrict__ nodeid, const int *__restrict__ depth,
                                  const int *__restrict__ left, const int *__restrict__ right,
                                  const int *__restrict__ start, const int *__restrict__ end, int d, int64_t M) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= M) return;
    const int node = nodeid[p];
    if (depth[node] != d || left[node] < 0) return;
    const int mid = start[node] + (end[node] - start[node]) / 2;
    nodeid[p] = p < mid ? left[node] : right[node];
}

// Moments of the depth-d nodes, one warp per node (the depth-ordered node
// list gives the nodes of a level): the children's 384 B records are read
// and the node's record written as whole coalesced rows through shared
// memory; lane l computes moment components l and l + 32 (cm 0-2, cd 3-11,
// cq 12-38), each in the reference's expression order; lane 0 forms the norms
// in their sequential order (barneshut.py:93-112).
__global__ void __launch_bounds__(256) bh_moments_warp_kernel(
    const int *__restrict__ nodes, int64_t count, const int *__restrict__ left, const int *__restrict__ right,
    const int *__restrict__ start, const int *__restrict__ order, const double *__restrict__ seg,
    const unsigned long long *__restrict__ enc_lo, const unsigned long long *__restrict__ enc_hi,
    double *__restrict__ box, double *__restrict__ rec, int *__restrict__ leaf_prim) {
    __shared__ double sm[8][3][kBhRec];   // per warp: left child, right child, own record
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *sL = sm[w][0], *sR = sm[w][1], *sO = sm[w][2];
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t q = blockIdx.x * (int64_t)(blockDim.x >> 5) + w; q < count; q += warps) {
        const int v = nodes[q];
        double lo[3], hi[3], c[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            lo[k] = ord_val(enc_lo[3 * (int64_t)v + k]);
            hi[k] = ord_val(enc_hi[3 * (int64_t)v + k]);
            c[k] = 0.5 * (lo[k] + hi[k]);
        }
        if (lane < 6) box[6 * (int64_t)v + lane] = lane < 3 ? lo[lane] : hi[lane - 3];
        const int lv = left[v];
        if (lv >= 0) {
            const double *L = rec + kBhRec * (int64_t)lv, *R = rec + kBhRec * (int64_t)right[v];
            sL[lane] = L[lane];
            sR[lane] = R[lane];
            if (lane < kBhRec - 32) {
                sL[32 + lane] = L[32 + lane];
                sR[32 + lane] = R[32 + lane];
            }
        }
        __syncwarp();
        double dd[3], rl[3];
        if (lv < 0) {
            const int sp = order[start[v]];
            if (lane == 0) leaf_prim[v] = sp;
            const double *a = seg + 6 * (int64_t)sp, *b = a + 3;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const double mid = 0.5 * (a[i] + b[i]);
                dd[i] = b[i] - a[i];
                rl[i] = mid - c[i];
            }
        } else if (lane == 0) {
            leaf_prim[v] = -1;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int o = lane + 32 * h;
            if (o >= 39) break;
            double out;
            if (lv < 0) {
                if (o < 3) {
                    out = dd[o];
                } else if (o < 12) {
                    const int i = (o - 3) / 3, j = (o - 3) % 3;
                    out = dd[i] * rl[j];
                } else {
                    const int i = (o - 12) / 9, j = ((o - 12) / 3) % 3, k = (o - 12) % 3;
                    out = dd[i] * (dd[j] * dd[k] / 12.0 + rl[j] * rl[k]);
                }
            } else {
                out = 0.0;
#pragma unroll
                for (int ch = 0; ch < 2; ++ch) {
                    const double *C = ch ? sR : sL;
                    const double rc0 = C[BH_CENTER + 0] - c[0], rc1 = C[BH_CENTER + 1] - c[1],
                                 rc2 = C[BH_CENTER + 2] - c[2];
                    const double rc[3] = {rc0, rc1, rc2};
                    if (o < 3) {
                        out += C[BH_CM + o];
                    } else if (o < 12) {
                        const int i = (o - 3) / 3, j = (o - 3) % 3;
                        out += C[BH_CD + 3 * i + j] + C[BH_CM + i] * rc[j];
                    } else {
                        const int i = (o - 12) / 9, j = ((o - 12) / 3) % 3, k = (o - 12) % 3;
                        out += C[BH_CQ + 9 * i + 3 * j + k] + C[BH_CD + 3 * i + j] * rc[k] +
                               C[BH_CD + 3 * i + k] * rc[j] + C[BH_CM + i] * rc[j] * rc[k];
                    }
                }
            }
            sO[BH_CM + o] = out;
        }
        __syncwarp();
        if (lane == 0) {
            const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
            sO[BH_CENTER + 0] = c[0];
            sO[BH_CENTER + 1] = c[1];
            sO[BH_CENTER + 2] = c[2];
            sO[BH_RADIUS] = 0.5 * sqrt(dx * dx + dy * dy + dz * dz);
            sO[BH_NCM] = sqrt(sO[BH_CM] * sO[BH_CM] + sO[BH_CM + 1] * sO[BH_CM + 1] + sO[BH_CM + 2] * sO[BH_CM + 2]);
            double s2 = 0.0, s3 = 0.0;
            for (int i = 0; i < 9; ++i) s2 += sO[BH_CD + i] * sO[BH_CD + i];
            for (int i = 0; i < 27; ++i) s3 += sO[BH_CQ + i] * sO[BH_CQ + i];
            sO[BH_NCD] = sqrt(s2);
            sO[BH_NCQ] = sqrt(s3);
            sO[46] = 0.0;
            sO[47] = 0.0;
        }
        __syncwarp();
        double *Rv = rec + kBhRec * (int64_t)v;
        Rv[lane] = sO[lane];
        if (lane < kBhRec - 32) Rv[32 + lane] = sO[32 + lane];
        __syncwarp();
    }
}

// Depth-ordered node list: first node of each depth in the sorted key array.
__global__ void bh_level_starts_kernel(const int *__restrict__ sorted_depth, int64_t N, int *__restrict__ starts) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < N && (i == 0 || sorted_depth[i] != sorted_depth[i - 1])) starts[sorted_depth[i]] = (int)i;
}

// ------------------------------------------------------------------ far field

__device__ __forceinline__ void cross3(double ax, double ay, double az, double bx, double by, double bz, double &ox,
                                       double &oy, double &oz) {
    ox = ay * bz - az * by;
    oy = az * bx - ax * bz;
    oz = ax * by - ay * bx;
}

// barneshut._far_field (barneshut.py:120-172), same operation order.
__device__ double far_field(double rx, double ry, double rz, const double *__restrict__ A,
                            const double *__restrict__ B, bool quadrupole) {
    const double r[3] = {rx, ry, rz};
    const double r2 = rx * rx + ry * ry + rz * rz;
    const double rn = sqrt(r2);
    const double inv3 = 1.0 / (kFourPi * r2 * rn);
    const double inv5 = inv3 / r2;
    const double inv7 = inv5 / r2;
    const double *cm1 = A + BH_CM, *cd1 = A + BH_CD, *cq1 = A + BH_CQ;
    const double *cm2 = B + BH_CM, *cd2 = B + BH_CD, *cq2 = B + BH_CQ;
    double wx, wy, wz;
    cross3(cm1[0], cm1[1], cm1[2], cm2[0], cm2[1], cm2[2], wx, wy, wz);
    double total = -(wx * rx + wy * ry + wz * rz) * inv3;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        double u1x, u1y, u1z, u2x, u2y, u2z;
        cross3(cd1[b], cd1[3 + b], cd1[6 + b], cm2[0], cm2[1], cm2[2], u1x, u1y, u1z);
        cross3(cm1[0], cm1[1], cm1[2], cd2[b], cd2[3 + b], cd2[6 + b], u2x, u2y, u2z);
        const double vx = u2x - u1x, vy = u2y - u1y, vz = u2z - u1z;
        const double rb = r[b];
        const double dot_vr = vx * rx + vy * ry + vz * rz;
        const double hv = vx * (b == 0 ? 1.0 : 0.0) + vy * (b == 1 ? 1.0 : 0.0) + vz * (b == 2 ? 1.0 : 0.0);
        total -= (hv * r2 - 3.0 * dot_vr * rb) * inv5;
    }
    if (quadrupole) {
#pragma unroll 1
        for (int b = 0; b < 3; ++b) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double q1x, q1y, q1z, q2x, q2y, q2z, dxx, dxy, dxz;
                cross3(cq1[3 * b + c], cq1[9 + 3 * b + c], cq1[18 + 3 * b + c], cm2[0], cm2[1], cm2[2], q1x, q1y,
                       q1z);
                cross3(cm1[0], cm1[1], cm1[2], cq2[3 * b + c], cq2[9 + 3 * b + c], cq2[18 + 3 * b + c], q2x, q2y,
                       q2z);
                cross3(cd1[b], cd1[3 + b], cd1[6 + b], cd2[c], cd2[3 + c], cd2[6 + c], dxx, dxy, dxz);
                const double vx = q1x + q2x - 2.0 * dxx;
                const double vy = q1y + q2y - 2.0 * dxy;
                const double vz = q1z + q2z - 2.0 * dxz;
                const double rb = r[b], rc = r[c];
                const double dot_vr = vx * rx + vy * ry + vz * rz;
                const double vb = b == 0 ? vx : (b == 1 ? vy : vz);
                const double vc = c == 0 ? vx : (c == 1 ? vy : vz);
                double t = 0.0;
                if (b == c) t += -3.0 * dot_vr * inv5;
                t += -3.0 * vb * rc * inv5;
                t += -3.0 * vc * rb * inv5;
                t += 15.0 * dot_vr * rb * rc * inv7;
                total -= 0.5 * t;
            }
        }
    }
    return total;
}

__global__ void bh_far_field_kernel(const double *__restrict__ A, const double *__restrict__ B, int quad,
                                    double *__restrict__ out) {
    out[0] = far_field(B[0] - A[0], B[1] - A[1], B[2] - A[2], A, B, quad != 0);
}

// ------------------------------------------------------------------ traversal

struct View {
    const double *rec, *seg;
    const int *left, *right, *leaf_prim;
};

__global__ void bh_roots_kernel(const int32_t *__restrict__ pairs, int64_t P, const int64_t *__restrict__ noff_a,
                                const int64_t *__restrict__ noff_b, int4 *__restrict__ fr) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < P) fr[p] = make_int4((int)noff_a[pairs[2 * p]], (int)noff_b[pairs[2 * p + 1]], (int)p, 0);
}

// One frontier level: far field, leaf pair, or split (barneshut.py:196-240).
// The far field is evaluated here; a leaf pair is only flagged — the level's
// leaf pairs are evaluated together by bh_leaf_pairs_kernel (no divergence
// between the far-field and segment-pair arithmetic inside a warp).
// cnt packs the split count (low 32 bits) and the leaf flag (high 32 bits), so
// one exclusive scan gives both the next frontier's and the leaf list's offsets.
__global__ void __launch_bounds__(128) bh_visit_kernel(const int4 *__restrict__ fr, int64_t n, View A, View B,
                                                       const double *__restrict__ beta, int quad, double k_const,
                                                       double2 *__restrict__ val, int64_t *__restrict__ cnt,
                                                       int *__restrict__ key) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i == n) cnt[n] = 0;
    if (i >= n) return;
    const int4 e = fr[i];
    const double *Ra = A.rec + kBhRec * (int64_t)e.x, *Rb = B.rec + kBhRec * (int64_t)e.y;
    const double rx = Rb[0] - Ra[0], ry = Rb[1] - Ra[1], rz = Rb[2] - Ra[2];
    const double dist = sqrt(rx * rx + ry * ry + rz * rz);
    const double ra = Ra[BH_RADIUS], rb = Rb[BH_RADIUS];
    double lam = 0.0, est = 0.0;
    int64_t c = 0;
    if (dist > beta[e.z] * (ra + rb)) {
        lam = far_field(rx, ry, rz, Ra, Rb, quad != 0);
        const double inv5 = 1.0 / (dist * ((dist * dist) * (dist * dist)));   // numba dist**5
        est = k_const * inv5 *
              (ra * Rb[BH_NCM] * Ra[BH_NCQ] + rb * Ra[BH_NCM] * Rb[BH_NCQ] +
               3.0 * (Ra[BH_NCD] * Rb[BH_NCQ] + Ra[BH_NCQ] * Rb[BH_NCD]));
    } else if (A.left[e.x] < 0 && B.left[e.y] < 0) {
        c = int64_t(1) << 32;   // leaf pair: batched (bh_leaf_pairs_kernel)
    } else {
        c = 2;
    }
    val[i] = make_double2(lam, est);
    cnt[i] = c;
    key[i] = e.z;
}

__global__ void bh_expand_kernel(const int4 *__restrict__ fr, int64_t n, View A, View B,
                                 const int64_t *__restrict__ cnt, const int64_t *__restrict__ off,
                                 int4 *__restrict__ next, int *__restrict__ leaves) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n || cnt[i] == 0) return;
    if (cnt[i] >> 32) {   // leaf pair: its frontier index into the level's leaf list
        leaves[off[i] >> 32] = (int)i;
        return;
    }
    const int4 e = fr[i];
    const bool a_leaf = A.left[e.x] < 0, b_leaf = B.left[e.y] < 0;
    const bool descend_a = !a_leaf && (b_leaf || A.rec[kBhRec * (int64_t)e.x + BH_RADIUS] >
                                                     B.rec[kBhRec * (int64_t)e.y + BH_RADIUS]);
    const int64_t o = off[i] & 0xffffffffLL;
    if (descend_a) {
        next[o] = make_int4(A.left[e.x], e.y, e.z, 0);
        next[o + 1] = make_int4(A.right[e.x], e.y, e.z, 0);
    } else {
        next[o] = make_int4(e.x, B.left[e.y], e.z, 0);
        next[o + 1] = make_int4(e.x, B.right[e.y], e.z, 0);
    }
}

// The level's leaf pairs as one batch: thread per pair, the reference formula
// (direct._pair_lambda, direct.py:19-46) — the per-pair arithmetic of the Gauss
// kernel's reference mode (geom.cuh ref_pair_lambda), bitwise as before.
__global__ void __launch_bounds__(128) bh_leaf_pairs_kernel(const int4 *__restrict__ fr,
                                                            const int *__restrict__ leaves, int64_t n_leaf, View A,
                                                            View B, double2 *__restrict__ val) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n_leaf) return;
    const int i = leaves[k];
    const int4 e = fr[i];
    const double *sa = A.seg + 6 * (int64_t)A.leaf_prim[e.x], *sb = B.seg + 6 * (int64_t)B.leaf_prim[e.y];
    val[i] = make_double2(
        ref_pair_lambda(sa[0], sa[1], sa[2], sa[3], sa[4], sa[5], sb[0], sb[1], sb[2], sb[3], sb[4], sb[5]), 0.0);
}

__global__ void bh_accumulate_kernel(const int *__restrict__ uniq, const double2 *__restrict__ agg,
                                     const int *__restrict__ nruns, int64_t n, double2 *__restrict__ tot) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n || i >= *nruns) return;
    const double2 a = agg[i];
    double2 t = tot[uniq[i]];
    t.x += a.x;
    t.y += a.y;
    tot[uniq[i]] = t;
}

struct Add2 {
    __device__ __forceinline__ double2 operator()(const double2 &a, const double2 &b) const {
        return make_double2(a.x + b.x, a.y + b.y);
    }
};

// ------------------------------------------------------------------ node tables

// Node table of every tree in the reference numbering (bvh.py:31-80), one
// thread per position walking root -> leaf.  The reference pops a LIFO stack,
// so internal nodes are numbered in a right-first preorder: the k-th popped
// internal node allocates children 2k+1 (left) and 2k+2 (right).  With leaf
// size 1 a subtree of n primitives has n-1 internal nodes, hence
// k(right) = k + 1 and k(left) = k + size(right).  A node is written by the
// thread of its first position.
__global__ void bh_table_kernel(const int64_t *__restrict__ loff, const int64_t *__restrict__ noff, int64_t L,
                                int64_t M, int *__restrict__ left, int *__restrict__ right, int *__restrict__ start,
                                int *__restrict__ end, int *__restrict__ depth) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= M) return;
    int64_t lo_t = 0, hi_t = L;
    while (hi_t - lo_t > 1) {
        const int64_t mid = (lo_t + hi_t) >> 1;
        if (loff[mid] <= p) lo_t = mid; else hi_t = mid;
    }
    const int64_t po = loff[lo_t], no = noff[lo_t];
    const int64_t q = p - po;
    int64_t s = 0, e = loff[lo_t + 1] - po, id = 0, k = 0;
    for (int d = 0;; ++d) {
        const bool mine = q == s;
        if (mine) {
            start[no + id] = (int)(s + po);
            end[no + id] = (int)(e + po);
            depth[no + id] = d;
        }
        if (e - s <= 1) {
            if (mine) left[no + id] = right[no + id] = -1;
            break;
        }
        const int64_t mid = s + (e - s) / 2, lc = 2 * k + 1, rc = 2 * k + 2;
        if (mine) {
            left[no + id] = (int)(no + lc);
            right[no + id] = (int)(no + rc);
        }
        if (q < mid) {
            id = lc;
            k += e - mid;
            e = mid;
        } else {
            id = rc;
            k += 1;
            s = mid;
        }
    }
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)ceil_div(n > 0 ? n : 1, t); }

}  // namespace

namespace {
// LC_BH_STATS=1: per-phase wall times of bh_build on stderr (stream synced per phase)
struct PhaseClock {
    bool on = false;
    cudaStream_t s;
    std::chrono::steady_clock::time_point t0;
    explicit PhaseClock(cudaStream_t st) : s(st) {
        const char *e = getenv("LC_BH_STATS");
        on = e && e[0] == '1';
        t0 = std::chrono::steady_clock::now();
    }
    void mark(const char *what) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto t1 = std::chrono::steady_clock::now();
        fprintf(stderr, "bh_build %-10s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};
}  // namespace

void bh_build(BhForest &f, const double *verts, const int64_t *loop_off, int64_t L, cudaStream_t s) {
    PhaseClock clk(s);
    if (L < 1) throw Error(LC_ERR_ARG, "moment forest needs at least one loop");
    if (loop_off[0] != 0) throw Error(LC_ERR_ARG, "loop offsets must start at 0");
    f.L = L;
    f.loop_off.assign(loop_off, loop_off + L + 1);
    f.node_off.assign(L + 1, 0);
    int64_t M = 0, N = 0;
    for (int64_t t = 0; t < L; ++t) {
        const int64_t m = loop_off[t + 1] - loop_off[t];
        if (m < 1) throw Error(LC_ERR_ARG, "every loop needs at least one vertex");
        f.node_off[t] = N;
        N += 2 * m - 1;
        M += m;
    }
    f.node_off[L] = N;
    if (M >= (int64_t(1) << 30)) throw Error(LC_ERR_ARG, "moment forest too large (2^30 segments)");
    f.M = M;
    f.N = N;
    int64_t max_m = 1;
    for (int64_t t = 0; t < L; ++t) max_m = std::max(max_m, loop_off[t + 1] - loop_off[t]);
    int levels = 1;   // leaves of a median split of m sit at depth <= ceil(log2 m)
    while ((int64_t(1) << (levels - 1)) < max_m) ++levels;
    f.levels = levels;
    clk.mark("table");
    const size_t i4 = sizeof(int32_t);
    f.seg.reserve(sizeof(double) * 6 * M, s);
    f.left.reserve(i4 * N, s);
    f.right.reserve(i4 * N, s);
    f.start.reserve(i4 * N, s);
    f.end.reserve(i4 * N, s);
    f.depth.reserve(i4 * N, s);
    f.order.reserve(i4 * M, s);
    f.leaf_prim.reserve(i4 * N, s);
    f.box.reserve(sizeof(double) * 6 * N, s);
    f.rec.reserve(sizeof(double) * kBhRec * N, s);
    f.d_node_off.reserve(sizeof(int64_t) * (L + 1), s);
    // build scratch
    DevBuf d_verts, d_loff, ckey, ckey_out, iota, ids_out, rank, nodeid, order2, key, key2, enc_lo, enc_hi, tmp;
    d_verts.reserve(sizeof(double) * 3 * M, s);
    d_loff.reserve(sizeof(int64_t) * (L + 1), s);
    ckey.reserve(sizeof(unsigned long long) * 3 * M, s);
    ckey_out.reserve(sizeof(unsigned long long) * M, s);
    iota.reserve(i4 * M, s);
    ids_out.reserve(i4 * M, s);
    rank.reserve(i4 * 3 * M, s);
    nodeid.reserve(i4 * M, s);
    order2.reserve(i4 * M, s);
    key.reserve(sizeof(unsigned long long) * M, s);
    key2.reserve(sizeof(unsigned long long) * M, s);
    enc_lo.reserve(sizeof(unsigned long long) * 3 * N, s);
    enc_hi.reserve(sizeof(unsigned long long) * 3 * N, s);
    LC_CUDA(cudaMemcpyAsync(d_verts.ptr, verts, sizeof(double) * 3 * M, cudaMemcpyHostToDevice, s));
    LC_CUDA(cudaMemcpyAsync(d_loff.ptr, loop_off, sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice, s));
    LC_CUDA(cudaMemcpyAsync(f.d_node_off.ptr, f.node_off.data(), sizeof(int64_t) * (L + 1), cudaMemcpyHostToDevice, s));
    LC_CUDA(cudaMemsetAsync(enc_lo.ptr, 0xFF, sizeof(unsigned long long) * 3 * N, s));
    LC_CUDA(cudaMemsetAsync(enc_hi.ptr, 0x00, sizeof(unsigned long long) * 3 * N, s));
    clk.mark("alloc+h2d");

    bh_table_kernel<<<blocks_for(M, 256), 256, 0, s>>>(d_loff.as<int64_t>(), f.d_node_off.as<int64_t>(), L, M,
                                                       f.left.as<int>(), f.right.as<int>(), f.start.as<int>(),
                                                       f.end.as<int>(), f.depth.as<int>());
    LC_CHECK_LAUNCH();
    bh_prims_kernel<<<blocks_for(M, 256), 256, 0, s>>>(d_verts.as<double>(), d_loff.as<int64_t>(),
                                                       f.d_node_off.as<int64_t>(), L, M, f.seg.as<double>(),
                                                       ckey.as<unsigned long long>(), iota.as<int>(), f.order.as<int>(),
                                                       nodeid.as<int>());
    LC_CHECK_LAUNCH();
    // ranks per axis: stable radix sort of (center key, index)
    int rank_bits = 1;
    while ((int64_t(1) << rank_bits) < M) ++rank_bits;
    size_t b1 = 0, b2 = 0;
    LC_CUB(cub::DeviceRadixSort::SortPairs(nullptr, b1, (unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                           (int *)nullptr, (int *)nullptr, (int)M));
    LC_CUB(cub::DeviceRadixSort::SortPairs(nullptr, b2, (unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                           (int *)nullptr, (int *)nullptr, (int)M, 0, 2 * rank_bits));
    tmp.reserve(std::max(b1, b2), s);
    for (int k = 0; k < 3; ++k) {
        size_t b = tmp.bytes;
        LC_CUB(cub::DeviceRadixSort::SortPairs(tmp.ptr, b, ckey.as<unsigned long long>() + k * M,
                                               ckey_out.as<unsigned long long>(), iota.as<int>(), ids_out.as<int>(),
                                               (int)M, 0, 64, s));
        bh_rank_kernel<<<blocks_for(M, 256), 256, 0, s>>>(ids_out.as<int>(), M, rank.as<int>() + k * M);
        LC_CHECK_LAUNCH();
    }
    clk.mark("ranks");
    int *ord = f.order.as<int>(), *ord_alt = order2.as<int>();
    for (int d = 0; d < levels; ++d) {
        bh_bbox_kernel<<<blocks_for(M, 256), 256, 0, s>>>(nodeid.as<int>(), ord, f.depth.as<int>(), d,
                                                          f.seg.as<double>(), M, enc_lo.as<unsigned long long>(),
                                                          enc_hi.as<unsigned long long>());
        LC_CHECK_LAUNCH();
        if (d == levels - 1) continue;   // leaves only
        bh_key_kernel<<<blocks_for(M, 256), 256, 0, s>>>(nodeid.as<int>(), ord, f.depth.as<int>(), f.left.as<int>(),
                                                         f.start.as<int>(), d, enc_lo.as<unsigned long long>(),
                                                         enc_hi.as<unsigned long long>(), rank.as<int>(), M, rank_bits,
                                                         key.as<unsigned long long>());
        LC_CHECK_LAUNCH();
        size_t b = tmp.bytes;
        LC_CUB(cub::DeviceRadixSort::SortPairs(tmp.ptr, b, key.as<unsigned long long>(),
                                               key2.as<unsigned long long>(), ord, ord_alt, (int)M, 0, 2 * rank_bits,
                                               s));
        std::swap(ord, ord_alt);
        bh_descend_kernel<<<blocks_for(M, 256), 256, 0, s>>>(nodeid.as<int>(), f.depth.as<int>(), f.left.as<int>(),
                                                             f.right.as<int>(), f.start.as<int>(), f.end.as<int>(), d,
                                                             M);
        LC_CHECK_LAUNCH();
    }
    if (ord != f.order.as<int>())
        LC_CUDA(cudaMemcpyAsync(f.order.ptr, ord, i4 * M, cudaMemcpyDeviceToDevice, s));
    clk.mark("levels");
    // nodes grouped by depth (stable radix sort of (depth, id)), then bottom-up
    {
        DevBuf nid, nid_sorted, dsorted, starts, tmp2;
        nid.reserve(i4 * N, s);
        nid_sorted.reserve(i4 * N, s);
        dsorted.reserve(i4 * N, s);
        starts.reserve(i4 * (levels + 1), s);
        bh_rank_kernel<<<blocks_for(N, 256), 256, 0, s>>>(nullptr, N, nid.as<int>());   // iota
        LC_CHECK_LAUNCH();
        int dbits = 1;
        while ((1 << dbits) < levels) ++dbits;
        size_t bt = 0;
        LC_CUB(cub::DeviceRadixSort::SortPairs(nullptr, bt, (int *)nullptr, (int *)nullptr, (int *)nullptr,
                                               (int *)nullptr, (int)N, 0, dbits));
        tmp2.reserve(bt, s);
        bt = tmp2.bytes;
        LC_CUB(cub::DeviceRadixSort::SortPairs(tmp2.ptr, bt, f.depth.as<int>(), dsorted.as<int>(), nid.as<int>(),
                                               nid_sorted.as<int>(), (int)N, 0, dbits, s));
        bh_level_starts_kernel<<<blocks_for(N, 256), 256, 0, s>>>(dsorted.as<int>(), N, starts.as<int>());
        LC_CHECK_LAUNCH();
        std::vector<int> h_starts(levels + 1);
        LC_CUDA(cudaMemcpyAsync(h_starts.data(), starts.ptr, i4 * levels, cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaStreamSynchronize(s));
        h_starts[levels] = (int)N;
        for (int d = levels - 1; d >= 0; --d) {
            const int64_t cnt = h_starts[d + 1] - h_starts[d];
            const int64_t blocks = std::min<int64_t>(ceil_div(cnt, 8), 148 * 16);
            bh_moments_warp_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(
                nid_sorted.as<int>() + h_starts[d], cnt, f.left.as<int>(), f.right.as<int>(), f.start.as<int>(),
                f.order.as<int>(), f.seg.as<double>(), enc_lo.as<unsigned long long>(),
                enc_hi.as<unsigned long long>(), f.box.as<double>(), f.rec.as<double>(), f.leaf_prim.as<int>());
            LC_CHECK_LAUNCH();
        }
        for (DevBuf *b : {&nid, &nid_sorted, &dsorted, &starts, &tmp2}) b->release(s);
    }
    clk.mark("moments");
    for (DevBuf *b : {&d_verts, &d_loff, &ckey, &ckey_out, &iota, &ids_out, &rank, &nodeid, &order2, &key, &key2,
                      &enc_lo, &enc_hi, &tmp})
        b->release(s);
    LC_CUDA(cudaStreamSynchronize(s));
    clk.mark("release");
}

void bh_download(const BhForest &f, int64_t *node_off, int64_t *left, int64_t *right, int64_t *start, int64_t *end,
                 int64_t *prim_order, double *node_lo, double *node_hi, double *center, double *radius, double *cm,
                 double *cd, double *cq, double *ncm, double *ncd, double *ncq, cudaStream_t s) {
    const int64_t N = f.N, M = f.M;
    if (node_off) std::copy(f.node_off.begin(), f.node_off.end(), node_off);
    std::vector<int32_t> tmp;
    auto fetch32 = [&](const DevBuf &b, int64_t n) {
        tmp.resize(n);
        LC_CUDA(cudaMemcpyAsync(tmp.data(), b.ptr, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaStreamSynchronize(s));
    };
    // per-tree (reference) numbering: node ids and positions relative to the tree
    auto local_nodes = [&](const DevBuf &b, int64_t *out, bool node_ids) {
        if (!out) return;
        fetch32(b, N);
        for (int64_t t = 0; t < f.L; ++t) {
            const int64_t off = node_ids ? f.node_off[t] : f.loop_off[t];
            for (int64_t v = f.node_off[t]; v < f.node_off[t + 1]; ++v)
                out[v] = tmp[v] < 0 ? -1 : (int64_t)tmp[v] - off;
        }
    };
    local_nodes(f.left, left, true);
    local_nodes(f.right, right, true);
    local_nodes(f.start, start, false);
    local_nodes(f.end, end, false);
    if (prim_order) {
        fetch32(f.order, M);
        for (int64_t t = 0; t < f.L; ++t)
            for (int64_t p = f.loop_off[t]; p < f.loop_off[t + 1]; ++p) prim_order[p] = tmp[p] - f.loop_off[t];
    }
    if (node_lo || node_hi) {
        std::vector<double> bx(6 * N);
        LC_CUDA(cudaMemcpyAsync(bx.data(), f.box.ptr, sizeof(double) * 6 * N, cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaStreamSynchronize(s));
        for (int64_t v = 0; v < N; ++v)
            for (int k = 0; k < 3; ++k) {
                if (node_lo) node_lo[3 * v + k] = bx[6 * v + k];
                if (node_hi) node_hi[3 * v + k] = bx[6 * v + 3 + k];
            }
    }
    if (center || radius || cm || cd || cq || ncm || ncd || ncq) {
        std::vector<double> r((size_t)kBhRec * N);
        LC_CUDA(cudaMemcpyAsync(r.data(), f.rec.ptr, sizeof(double) * kBhRec * N, cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaStreamSynchronize(s));
        for (int64_t v = 0; v < N; ++v) {
            const double *R = r.data() + kBhRec * v;
            if (center) std::copy(R + BH_CENTER, R + BH_CENTER + 3, center + 3 * v);
            if (radius) radius[v] = R[BH_RADIUS];
            if (cm) std::copy(R + BH_CM, R + BH_CM + 3, cm + 3 * v);
            if (cd) std::copy(R + BH_CD, R + BH_CD + 9, cd + 9 * v);
            if (cq) std::copy(R + BH_CQ, R + BH_CQ + 27, cq + 27 * v);
            if (ncm) ncm[v] = R[BH_NCM];
            if (ncd) ncd[v] = R[BH_NCD];
            if (ncq) ncq[v] = R[BH_NCQ];
        }
    }
}

double bh_far_field(const BhForest &a, int64_t na, const BhForest &b, int64_t nb, bool quadrupole, BhScratch &sc,
                    cudaStream_t s) {
    if (na < 0 || na >= a.N || nb < 0 || nb >= b.N) throw Error(LC_ERR_ARG, "node index out of range");
    sc.tot.reserve(sizeof(double), s);
    sc.host.reserve(sizeof(double));
    bh_far_field_kernel<<<1, 1, 0, s>>>(a.rec.as<double>() + kBhRec * na, b.rec.as<double>() + kBhRec * nb,
                                        quadrupole ? 1 : 0, sc.tot.as<double>());
    LC_CHECK_LAUNCH();
    LC_CUDA(cudaMemcpyAsync(sc.host.ptr, sc.tot.ptr, sizeof(double), cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
    return *static_cast<double *>(sc.host.ptr);
}

void bh_eval(const BhForest &a, const BhForest &b, const int32_t *pairs, int64_t P, const double *beta, bool quadrupole,
             double k_const, double *lam, double *e_est, int64_t *visits, BhScratch &sc, cudaStream_t s) {
    if (visits) *visits = 0;
    if (P <= 0) return;
    for (int64_t p = 0; p < P; ++p)
        if (pairs[2 * p] < 0 || pairs[2 * p] >= a.L || pairs[2 * p + 1] < 0 || pairs[2 * p + 1] >= b.L)
            throw Error(LC_ERR_ARG, "tree index out of range");
    const View A{a.rec.as<double>(), a.seg.as<double>(), a.left.as<int>(), a.right.as<int>(), a.leaf_prim.as<int>()};
    const View B{b.rec.as<double>(), b.seg.as<double>(), b.left.as<int>(), b.right.as<int>(), b.leaf_prim.as<int>()};
    sc.pairs.reserve(sizeof(int32_t) * 2 * P, s);
    sc.beta.reserve(sizeof(double) * P, s);
    sc.tot.reserve(sizeof(double2) * P, s);
    sc.host.reserve(sizeof(double2) * P + 64);
    sc.fr[0].reserve(sizeof(int4) * P, s);
    LC_CUDA(cudaMemcpyAsync(sc.pairs.ptr, pairs, sizeof(int32_t) * 2 * P, cudaMemcpyHostToDevice, s));
    LC_CUDA(cudaMemcpyAsync(sc.beta.ptr, beta, sizeof(double) * P, cudaMemcpyHostToDevice, s));
    LC_CUDA(cudaMemsetAsync(sc.tot.ptr, 0, sizeof(double2) * P, s));
    bh_roots_kernel<<<blocks_for(P, 256), 256, 0, s>>>(sc.pairs.as<int32_t>(), P, a.d_node_off.as<int64_t>(),
                                                       b.d_node_off.as<int64_t>(), sc.fr[0].as<int4>());
    LC_CHECK_LAUNCH();
    int cur = 0;
    int64_t n = P, total = 0;
    int64_t *h_next = static_cast<int64_t *>(sc.host.ptr);
    while (n > 0) {
        if (n >= (int64_t(1) << 30)) throw Error(LC_ERR_ARG, "Barnes-Hut frontier exceeds 2^30 node pairs");
        total += n;
        sc.val.reserve(sizeof(double2) * n, s);
        sc.agg.reserve(sizeof(double2) * n, s);
        sc.cnt.reserve(sizeof(int64_t) * (n + 1), s);
        sc.off.reserve(sizeof(int64_t) * (n + 1), s);
        sc.key.reserve(sizeof(int) * n, s);
        sc.uniq.reserve(sizeof(int) * n, s);
        sc.nruns.reserve(sizeof(int), s);
        size_t bs = 0, br = 0;
        LC_CUB(cub::DeviceScan::ExclusiveSum(nullptr, bs, (int64_t *)nullptr, (int64_t *)nullptr, (int)(n + 1)));
        LC_CUB(cub::DeviceReduce::ReduceByKey(nullptr, br, (int *)nullptr, (int *)nullptr, (double2 *)nullptr,
                                              (double2 *)nullptr, (int *)nullptr, Add2(), (int)n));
        sc.tmp.reserve(std::max(bs, br), s);
        bh_visit_kernel<<<blocks_for(n + 1, 128), 128, 0, s>>>(sc.fr[cur].as<int4>(), n, A, B, sc.beta.as<double>(),
                                                               quadrupole ? 1 : 0, k_const, sc.val.as<double2>(),
                                                               sc.cnt.as<int64_t>(), sc.key.as<int>());
        LC_CHECK_LAUNCH();
        bs = sc.tmp.bytes;
        LC_CUB(cub::DeviceScan::ExclusiveSum(sc.tmp.ptr, bs, sc.cnt.as<int64_t>(), sc.off.as<int64_t>(), (int)(n + 1),
                                             s));
        LC_CUDA(cudaMemcpyAsync(h_next, sc.off.as<int64_t>() + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        LC_CUDA(cudaStreamSynchronize(s));
        const int64_t nn = *h_next & 0xffffffffLL, n_leaf = *h_next >> 32;
        sc.fr[cur ^ 1].reserve(sizeof(int4) * (nn > 0 ? nn : 1), s);
        sc.leaves.reserve(sizeof(int) * (n_leaf > 0 ? n_leaf : 1), s);
        bh_expand_kernel<<<blocks_for(n, 256), 256, 0, s>>>(sc.fr[cur].as<int4>(), n, A, B, sc.cnt.as<int64_t>(),
                                                            sc.off.as<int64_t>(), sc.fr[cur ^ 1].as<int4>(),
                                                            sc.leaves.as<int>());
        LC_CHECK_LAUNCH();
        if (n_leaf > 0) {
            bh_leaf_pairs_kernel<<<blocks_for(n_leaf, 128), 128, 0, s>>>(sc.fr[cur].as<int4>(), sc.leaves.as<int>(),
                                                                         n_leaf, A, B, sc.val.as<double2>());
            LC_CHECK_LAUNCH();
        }
        br = sc.tmp.bytes;
        LC_CUB(cub::DeviceReduce::ReduceByKey(sc.tmp.ptr, br, sc.key.as<int>(), sc.uniq.as<int>(), sc.val.as<double2>(),
                                              sc.agg.as<double2>(), sc.nruns.as<int>(), Add2(), (int)n, s));
        bh_accumulate_kernel<<<blocks_for(n, 256), 256, 0, s>>>(sc.uniq.as<int>(), sc.agg.as<double2>(),
                                                                sc.nruns.as<int>(), n, sc.tot.as<double2>());
        LC_CHECK_LAUNCH();
        cur ^= 1;
        n = nn;
    }
    LC_CUDA(cudaMemcpyAsync(sc.host.ptr, sc.tot.ptr, sizeof(double2) * P, cudaMemcpyDeviceToHost, s));
    LC_CUDA(cudaStreamSynchronize(s));
    const double2 *h = static_cast<const double2 *>(sc.host.ptr);
    for (int64_t p = 0; p < P; ++p) {
        if (lam) lam[p] = h[p].x;
        if (e_est) e_est[p] = h[p].y;
    }
    if (visits) *visits = total;
}

}  // namespace lc
