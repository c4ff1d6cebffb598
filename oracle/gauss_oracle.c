/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the direct-summation Gauss
 * linking integral.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library; the product
 * path (paper_2106_12655_b200) never does.
 *
 * Plain-C restatement of the reference's numba kernels:
 *   oracle_pair_lambda      <- linkcert/direct.py:19-46  (_pair_lambda)
 *   oracle_link_atan        <- linkcert/direct.py:49-65  (_link_atan)
 *   oracle_link_anglesum    <- linkcert/direct.py:68-134 (_sgn, _link_angle_sum)
 *   oracle_evaluate_pairs   <- linkcert/certify.py:108-127 (_evaluate_pairs,
 *                              DS branch of kernels.compute_link :45-73)
 *
 * The reference compiles with numba fastmath=False: no FMA contraction, no
 * reassociation, llvm.sqrt (correctly rounded) and libm atan2.  Build this
 * file with -ffp-contract=off -fno-fast-math so the same IEEE operation
 * sequence is executed; tests/test_oracle_golden.py pins the result bitwise
 * against vectors produced by the reference itself (tests/golden/).
 *
 * Vertex arrays are the reference's "closed" layout (direct.py:164-166):
 * (n+1, 3) float64 C-order, vertex 0 repeated at the end.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

static const double TWO_PI = 6.283185307179586; /* 2.0 * math.pi */

double oracle_pair_lambda(double ljx, double ljy, double ljz,
                          double lj1x, double lj1y, double lj1z,
                          double kix, double kiy, double kiz,
                          double ki1x, double ki1y, double ki1z) {
    /* Four corner vectors of the segment-pair quadrilateral. */
    double ax = ljx - kix, ay = ljy - kiy, az = ljz - kiz;
    double bx = ljx - ki1x, by = ljy - ki1y, bz = ljz - ki1z;
    double cx = lj1x - ki1x, cy = lj1y - ki1y, cz = lj1z - ki1z;
    double dx = lj1x - kix, dy = lj1y - kiy, dz = lj1z - kiz;
    double an = sqrt(ax * ax + ay * ay + az * az);
    double bn = sqrt(bx * bx + by * by + bz * bz);
    double cn = sqrt(cx * cx + cy * cy + cz * cz);
    double dn = sqrt(dx * dx + dy * dy + dz * dz);
    double p = ax * (by * cz - bz * cy) + ay * (bz * cx - bx * cz) + az * (bx * cy - by * cx);
    double ab = ax * bx + ay * by + az * bz;
    double bc = bx * cx + by * cy + bz * cz;
    double ca = cx * ax + cy * ay + cz * az;
    double ad = ax * dx + ay * dy + az * dz;
    double dc = dx * cx + dy * cy + dz * cz;
    double d1 = an * bn * cn + ab * cn + bc * an + ca * bn;
    double d2 = an * dn * cn + ad * cn + dc * an + ca * dn;
    return (atan2(p, d1) + atan2(p, d2)) / TWO_PI;
}

/* l: inner loop (loop1), k: outer loop (loop2); both closed (n+1, 3). */
double oracle_link_atan(const double *l, int64_t nl, const double *k, int64_t nk) {
    double total = 0.0;
    for (int64_t i = 0; i < nk; ++i) {
        const double *ki = k + 3 * i;
        double row = 0.0;
        for (int64_t j = 0; j < nl; ++j) {
            const double *lj = l + 3 * j;
            row += oracle_pair_lambda(lj[0], lj[1], lj[2], lj[3], lj[4], lj[5],
                                      ki[0], ki[1], ki[2], ki[3], ki[4], ki[5]);
        }
        total += row;
    }
    return total;
}

static double sgn2(double x, double y) {
    return (y > 0.0 || (y == 0.0 && x < 0.0)) ? 1.0 : -1.0;
}

double oracle_link_anglesum(const double *l, int64_t nl, const double *k, int64_t nk) {
    double total = 0.0;
    for (int64_t i = 0; i < nk; ++i) {
        const double *ki = k + 3 * i;
        double xs = 1.0, ys = 0.0, s_prev = -1.0, lam = 0.0;
        for (int64_t j = 0; j < nl; ++j) {
            const double *lj = l + 3 * j;
            double ax = lj[0] - ki[0], ay = lj[1] - ki[1], az = lj[2] - ki[2];
            double bx = lj[0] - ki[3], by = lj[1] - ki[4], bz = lj[2] - ki[5];
            double cx = lj[3] - ki[3], cy = lj[4] - ki[4], cz = lj[5] - ki[5];
            double dx = lj[3] - ki[0], dy = lj[4] - ki[1], dz = lj[5] - ki[2];
            double an = sqrt(ax * ax + ay * ay + az * az);
            double bn = sqrt(bx * bx + by * by + bz * bz);
            double cn = sqrt(cx * cx + cy * cy + cz * cz);
            double dn = sqrt(dx * dx + dy * dy + dz * dz);
            double p = ax * (by * cz - bz * cy) + ay * (bz * cx - bx * cz) + az * (bx * cy - by * cx);
            double ab = ax * bx + ay * by + az * bz;
            double bc = bx * cx + by * cy + bz * cz;
            double ca = cx * ax + cy * ay + cz * az;
            double ad = ax * dx + ay * dy + az * dz;
            double dc = dx * cx + dy * cy + dz * cz;
            double d1 = an * bn * cn + ab * cn + bc * an + ca * bn;
            double d2 = an * dn * cn + ad * cn + dc * an + ca * dn;
            double xp = d1 * d2 - p * p;
            double yp = p * (d1 + d2);
            double s1 = sgn2(d1, p);
            if (s1 * sgn2(d2, p) > 0.0 && s1 * sgn2(xp, yp) < 0.0) lam += s1;
            double xpp = xs * xp - ys * yp;
            double ypp = xs * yp + ys * xp;
            if (sgn2(xp, yp) * s_prev > 0.0 && sgn2(xpp, ypp) * s_prev < 0.0) lam += s_prev;
            s_prev = sgn2(xpp, ypp);
            double norm = fmax(fabs(xpp), fabs(ypp));
            xs = xpp / norm;
            ys = ypp / norm;
        }
        lam += atan2(ys, xs) / TWO_PI;
        total += lam;
    }
    return total;
}

/* ---- batched pair evaluation (the _evaluate_pairs seam), pthreads ---- */

typedef struct {
    const double *verts;   /* all loops, closed AoS, concatenated */
    const int64_t *voff;   /* loop v occupies rows [voff[v], voff[v+1]) incl. closing vertex */
    const int32_t *pairs;  /* (P, 2): (i, j), i < j */
    int64_t P;
    int anglesum;
    double *raw;
    int64_t next;          /* shared cursor */
    pthread_mutex_t mu;
} pair_job;

static void *pair_worker(void *arg) {
    pair_job *job = (pair_job *)arg;
    for (;;) {
        pthread_mutex_lock(&job->mu);
        int64_t p = job->next++;
        pthread_mutex_unlock(&job->mu);
        if (p >= job->P) break;
        int32_t i = job->pairs[2 * p], j = job->pairs[2 * p + 1];
        /* compute_link(polylines[i], polylines[j]): loop1 = i -> l, loop2 = j -> k */
        const double *l = job->verts + 3 * job->voff[i];
        const double *k = job->verts + 3 * job->voff[j];
        int64_t nl = job->voff[i + 1] - job->voff[i] - 1;
        int64_t nk = job->voff[j + 1] - job->voff[j] - 1;
        job->raw[p] = job->anglesum ? oracle_link_anglesum(l, nl, k, nk)
                                    : oracle_link_atan(l, nl, k, nk);
    }
    return NULL;
}

int oracle_evaluate_pairs(const double *verts, const int64_t *voff, const int32_t *pairs,
                          int64_t P, int anglesum, int nthreads, double *raw) {
    pair_job job = {verts, voff, pairs, P, anglesum, raw, 0};
    pthread_mutex_init(&job.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, pair_worker, &job);
    pair_worker(&job);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&job.mu);
    return 0;
}

/* Rows [r0, r1) of one pair (for bounded CPU samples of huge pairs), split
 * across threads by rows; returns the partial sum in row order. */
typedef struct {
    const double *l, *k;
    int64_t nl, r0, r1;
    double *rows;
    int64_t next;
    pthread_mutex_t mu;
} row_job;

static void *row_worker(void *arg) {
    row_job *job = (row_job *)arg;
    for (;;) {
        pthread_mutex_lock(&job->mu);
        int64_t i = job->r0 + job->next++;
        pthread_mutex_unlock(&job->mu);
        if (i >= job->r1) break;
        const double *ki = job->k + 3 * i;
        double row = 0.0;
        for (int64_t j = 0; j < job->nl; ++j) {
            const double *lj = job->l + 3 * j;
            row += oracle_pair_lambda(lj[0], lj[1], lj[2], lj[3], lj[4], lj[5],
                                      ki[0], ki[1], ki[2], ki[3], ki[4], ki[5]);
        }
        job->rows[i - job->r0] = row;
    }
    return NULL;
}

double oracle_link_atan_rows(const double *l, int64_t nl, const double *k, int64_t r0,
                             int64_t r1, int nthreads) {
    if (r1 <= r0) return 0.0;
    row_job job = {l, k, nl, r0, r1, (double *)malloc(sizeof(double) * (size_t)(r1 - r0)), 0};
    pthread_mutex_init(&job.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, row_worker, &job);
    row_worker(&job);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    double total = 0.0;
    for (int64_t i = 0; i < r1 - r0; ++i) total += job.rows[i];
    free(job.rows);
    pthread_mutex_destroy(&job.mu);
    return total;
}
