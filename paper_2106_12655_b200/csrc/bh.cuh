// Barnes-Hut evaluation of the Gauss linking integral on moment trees
// (reference: linkcert/barneshut.py, tree build linkcert/bvh.py:17-90).
//
// A forest holds the moment trees of L closed polylines (one tree per loop,
// leaf size 1, the reference's median split and node numbering).  Node
// records are 48 doubles (AoS, one 384 B record per node, read whole by the
// traversal): center[3] radius cm[3] cd[9] cq[27] ncm ncd ncq pad[2].
#pragma once
#include <vector>

#include "common.cuh"

namespace lc {

constexpr int kBhRec = 48;
enum { BH_CENTER = 0, BH_RADIUS = 3, BH_CM = 4, BH_CD = 7, BH_CQ = 16, BH_NCM = 43, BH_NCD = 44, BH_NCQ = 45 };

struct BhForest {
    int64_t L = 0, M = 0, N = 0;                // trees, segments (primitives), nodes
    int levels = 0;                             // max node depth + 1
    std::vector<int64_t> loop_off, node_off;    // host, L + 1 each
    DevBuf seg;                                 // M x 6 doubles: segment start a, end b
    DevBuf left, right, start, end, depth;      // int32 per node (global ids / positions)
    DevBuf order;                               // int32 per position: global primitive id
    DevBuf leaf_prim;                           // int32 per node: primitive of a leaf, -1 inside
    DevBuf box;                                 // N x 6 doubles: lo[3] hi[3]
    DevBuf rec;                                 // N x kBhRec doubles
    DevBuf d_node_off;                          // int64, L + 1 (roots of the traversal)
    void release(cudaStream_t s) {
        for (DevBuf *b : {&seg, &left, &right, &start, &end, &depth, &order, &leaf_prim, &box, &rec, &d_node_off})
            b->release(s);
    }
};

// Scratch of the dual-tree traversal (grow-only, reused across calls).
struct BhScratch {
    DevBuf fr[2], val, cnt, off, key, uniq, agg, nruns, tmp, tot, beta, pairs, leaves;
    PinnedBuf host;
};

// Build from host vertices (M x 3, loop t = rows [loop_off[t], loop_off[t+1]),
// closed implicitly: segment i runs from vertex i to the next one of its loop).
void bh_build(BhForest &f, const double *verts, const int64_t *loop_off, int64_t L, cudaStream_t s);

// Copy node data to the host in the reference's per-tree numbering (any pointer
// may be null): left/right (-1 for leaves), start/end, prim_order per tree.
void bh_download(const BhForest &f, int64_t *node_off, int64_t *left, int64_t *right, int64_t *start, int64_t *end,
                 int64_t *prim_order, double *node_lo, double *node_hi, double *center, double *radius, double *cm,
                 double *cd, double *cq, double *ncm, double *ncd, double *ncq, cudaStream_t s);

// barneshut._far_field for one node pair (global node ids).
double bh_far_field(const BhForest &a, int64_t na, const BhForest &b, int64_t nb, bool quadrupole, BhScratch &sc,
                    cudaStream_t s);

// barneshut._dual_eval for P tree pairs (tree ids into a and b), opening
// parameter beta[p] per pair; lam/e_est per pair; visits = node pairs visited.
void bh_eval(const BhForest &a, const BhForest &b, const int32_t *pairs, int64_t P, const double *beta, bool quadrupole,
             double k_const, double *lam, double *e_est, int64_t *visits, BhScratch &sc, cudaStream_t s);

}  // namespace lc
