/*
 * oracle.c -- the fp64 CPU ORACLE for the ICP hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1807_00399_b200/, libcil.so) never links, imports or calls it, and this file
 * shares no code, header, helper or constant generator with csrc/.
 *
 * What it computes (plain definition, fp64 throughout, inputs are fp32 promoted):
 *   - exact nearest neighbour(s) in 3-D L2, ties to the lowest target index
 *       PAPER.md:122 (KDTree k-NN), PAPER.md:195 ("nearest neighbor kd-tree queries");
 *       tie rule: SPEC.md:160 / DESIGN.md reading R1.
 *     Brute force (orc_knn with kd == NULL) and a plain median-split kd-tree (leaf 16,
 *     widest axis) that prunes only when (plane distance)^2 > worst,
 *     so it returns exactly what the brute force returns (pinned in tests/).
 *   - one ICP iteration: transform s = R p + t, 1-NN, reject d^2 > max_dist^2
 *     ("rejection distance threshold", inclusive per SPEC.md:386),
 *     per-pair residual/Jacobian and normal equations H = sum J^T J, g = sum J^T r
 *       point-to-point  [Besl & McKay]  r = s - t,        J = [-[s]x , I3]  (3x6)
 *       point-to-plane  [Low 2004]      r = (s - t).n,    J = [s x n ; n]   (1x6)
 *     ("optimizers for rigid ... registration under the point-to-point and
 *     point-to-plane metrics"; linearisation SPEC.md:411-413; R4, R6).
 *     Accumulated serially in source-index order.
 *   - solve H x = -g by Cholesky, degenerate iff count < 6, a pivot <= 0 or
 *     min pivot / max pivot < 1e-12 (R9); pose update
 *     R <- exp([alpha]x) R, t <- exp([alpha]x) t + tau (R5).
 *   - the ICP loop ("alternating between correspondence estimation and
 *     transformation parameter optimization", PAPER.md:195 fixed iteration count).
 *   - projective data association for organised clouds (
 *     SPEC.md:392-400): project s through the target intrinsics, round half away from
 *     zero, take that pixel's point if valid and within max_dist.
 *   - voxel-grid downsampling: bin key
 *     floor((p - origin) / bin) per axis, one fp64 mean per non-empty bin (normals: mean
 *     renormalised), bins in ascending lexicographic key order.
 *   - PCA normals over k-NN (used only to build config-3 inputs, as
 *     BASELINE.json configs[2] asks for "normals from oracle PCA over 10-NN").
 *
 * Threads: OpenMP over independent queries only (each query's result is written to
 * its own slot); every reduction is serial and in index order.
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (see Makefile).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_DEGENERATE 16
#define ORC_NO_CORRESPONDENCES 17
#define ORC_KMAX 32

/* ------------------------------------------------------------------ threads */
void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------ geometry */
/* s = R p + t, pose is 4x4 row-major (source -> target) */
static void transform_point(const double pose[16], const float* p, double s[3]) {
    double x = p[0], y = p[1], z = p[2];
    for (int a = 0; a < 3; ++a)
        s[a] = pose[4 * a + 0] * x + pose[4 * a + 1] * y + pose[4 * a + 2] * z + pose[4 * a + 3];
}

void orc_transform(const double pose[16], const float* p, int64_t m, double* s) {
    for (int64_t i = 0; i < m; ++i) transform_point(pose, p + 3 * i, s + 3 * i);
}

/* squared Euclidean distance, fixed evaluation order */
static double dist2(const double q[3], const float* t) {
    double dx = q[0] - (double)t[0];
    double dy = q[1] - (double)t[1];
    double dz = q[2] - (double)t[2];
    return dx * dx + dy * dy + dz * dz;
}

/* ------------------------------------------------------------------ k-best list */
/* sorted ascending by (d2, index) lexicographically; at most k entries, all d2 <= bound */
typedef struct {
    int k, cnt;
    double bound;
    double d2[ORC_KMAX];
    int64_t id[ORC_KMAX];
} kbest;

static void kb_init(kbest* b, int k, double bound) {
    b->k = k; b->cnt = 0; b->bound = bound;
}

/* the current pruning radius^2: a subtree whose lower bound exceeds it cannot contribute */
static double kb_worst(const kbest* b) {
    return b->cnt < b->k ? b->bound : b->d2[b->cnt - 1];
}

static int kb_less(double da, int64_t ia, double db, int64_t ib) {
    return da < db || (da == db && ia < ib);
}

static void kb_offer(kbest* b, double d2, int64_t id) {
    if (!(d2 <= b->bound)) return;
    if (b->cnt == b->k && !kb_less(d2, id, b->d2[b->cnt - 1], b->id[b->cnt - 1])) return;
    int pos = b->cnt < b->k ? b->cnt++ : b->cnt - 1;
    while (pos > 0 && kb_less(d2, id, b->d2[pos - 1], b->id[pos - 1])) {
        b->d2[pos] = b->d2[pos - 1];
        b->id[pos] = b->id[pos - 1];
        --pos;
    }
    b->d2[pos] = d2;
    b->id[pos] = id;
}

/* ------------------------------------------------------------------ kd-tree */
typedef struct {
    int32_t axis;      /* -1 for a leaf */
    double split;
    int64_t left, right;  /* child node ids */
    int64_t lo, hi;       /* leaf: range in perm[] */
} kdnode;

typedef struct {
    const float* pts;  /* caller-owned, must outlive the tree */
    int64_t n;
    int leaf;
    int64_t* perm;
    kdnode* nodes;
    int64_t nn, cap;
} kdtree;

static double coord(const kdtree* t, int64_t i, int a) { return (double)t->pts[3 * i + a]; }

/* total order used for the median: (coordinate, index) */
static int before(const kdtree* t, int64_t i, int64_t j, int a) {
    double ci = coord(t, i, a), cj = coord(t, j, a);
    return ci < cj || (ci == cj && i < j);
}

/* quickselect: place the element of rank k (within [lo,hi)) at perm[k] */
static void select_k(kdtree* t, int64_t lo, int64_t hi, int64_t k, int a) {
    int64_t* P = t->perm;
    while (hi - lo > 1) {
        /* median-of-three pivot, deterministic */
        int64_t mid = lo + (hi - lo) / 2;
        int64_t x = P[lo], y = P[mid], z = P[hi - 1], piv;
        if (before(t, x, y, a)) piv = before(t, y, z, a) ? y : (before(t, x, z, a) ? z : x);
        else piv = before(t, x, z, a) ? x : (before(t, y, z, a) ? z : y);
        /* three-way partition around piv: [< piv][== piv][> piv] (== only piv itself) */
        int64_t i = lo, j = lo, g = hi;
        while (j < g) {
            if (P[j] == piv) { ++j; }
            else if (before(t, P[j], piv, a)) { int64_t s = P[i]; P[i] = P[j]; P[j] = s; ++i; ++j; }
            else { --g; int64_t s = P[g]; P[g] = P[j]; P[j] = s; }
        }
        /* now [lo,i) < piv, [i,g) == piv (exactly one element), [g,hi) > piv */
        if (k < i) hi = i;
        else if (k >= g) lo = g;
        else return;
    }
}

static int64_t new_node(kdtree* t) {
    if (t->nn == t->cap) {
        t->cap = t->cap ? 2 * t->cap : 1024;
        t->nodes = (kdnode*)realloc(t->nodes, (size_t)t->cap * sizeof(kdnode));
    }
    return t->nn++;
}

static int64_t build_rec(kdtree* t, int64_t lo, int64_t hi) {
    int64_t id = new_node(t);
    if (hi - lo <= t->leaf) {
        kdnode* nd = &t->nodes[id];
        nd->axis = -1; nd->lo = lo; nd->hi = hi; nd->left = nd->right = -1; nd->split = 0;
        return id;
    }
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t q = lo; q < hi; ++q)
        for (int a = 0; a < 3; ++a) {
            double c = coord(t, t->perm[q], a);
            if (c < mn[a]) mn[a] = c;
            if (c > mx[a]) mx[a] = c;
        }
    int ax = 0;
    for (int a = 1; a < 3; ++a)
        if (mx[a] - mn[a] > mx[ax] - mn[ax]) ax = a;
    int64_t mid = lo + (hi - lo) / 2;
    select_k(t, lo, hi, mid, ax);
    double split = coord(t, t->perm[mid], ax);
    /* left = [lo,mid) has coordinates <= split, right = [mid,hi) has coordinates >= split */
    int64_t l = build_rec(t, lo, mid);
    int64_t r = build_rec(t, mid, hi);
    kdnode* nd = &t->nodes[id];
    nd->axis = ax; nd->split = split; nd->left = l; nd->right = r; nd->lo = lo; nd->hi = hi;
    return id;
}

void* orc_kd_build(const float* pts, int64_t n, int leaf) {
    kdtree* t = (kdtree*)calloc(1, sizeof(kdtree));
    t->pts = pts; t->n = n; t->leaf = leaf > 0 ? leaf : 16;
    t->perm = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) t->perm[i] = i;
    if (n > 0) build_rec(t, 0, n);
    return t;
}

void orc_kd_free(void* p) {
    kdtree* t = (kdtree*)p;
    if (!t) return;
    free(t->perm); free(t->nodes); free(t);
}

static void kd_search(const kdtree* t, int64_t id, const double q[3], kbest* b) {
    const kdnode* nd = &t->nodes[id];
    if (nd->axis < 0) {
        for (int64_t r = nd->lo; r < nd->hi; ++r) {
            int64_t j = t->perm[r];
            kb_offer(b, dist2(q, t->pts + 3 * j), j);
        }
        return;
    }
    double diff = q[nd->axis] - nd->split;
    int64_t near_ = diff < 0 ? nd->left : nd->right;
    int64_t far_ = diff < 0 ? nd->right : nd->left;
    kd_search(t, near_, q, b);
    /* every point on the far side is at least |diff| away along this axis;
       visit when diff^2 <= worst so that equal-distance (tied) points are kept */
    if (diff * diff <= kb_worst(b)) kd_search(t, far_, q, b);
}

/* one query: kd == NULL -> brute force over all n targets */
static void knn_one(const kdtree* kd, const float* pts, int64_t n, const double q[3], int k,
                    double bound2, kbest* b) {
    kb_init(b, k, bound2);
    if (kd) {
        if (kd->n > 0) kd_search(kd, 0, q, b);
    } else {
        for (int64_t j = 0; j < n; ++j) kb_offer(b, dist2(q, pts + 3 * j), j);
    }
}

/* k nearest targets of each fp64 query within bound2 (use INFINITY for unbounded).
   idx/d2 are [m*k]; missing entries are -1 / +inf. */
int orc_knn(const void* kd, const float* pts, int64_t n, const double* q, int64_t m, int k,
            double bound2, int64_t* idx, double* d2) {
    if (k < 1 || k > ORC_KMAX) return 1;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < m; ++i) {
        kbest b;
        knn_one((const kdtree*)kd, pts, n, q + 3 * i, k, bound2, &b);
        for (int r = 0; r < k; ++r) {
            idx[i * k + r] = r < b.cnt ? b.id[r] : -1;
            d2[i * k + r] = r < b.cnt ? b.d2[r] : INFINITY;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ normal equations */
#define MET_P2POINT 0
#define MET_P2PLANE 1
#define MET_COMBINED 2   /* w_point * point-to-point + w_plane * point-to-plane ("weighted combinations") */

static double g_w_point = 0.0, g_w_plane = 0.0;

/* weights of MET_COMBINED (reading R22) */
void orc_set_combined_weights(double w_point, double w_plane) {
    g_w_point = w_point;
    g_w_plane = w_plane;
}

/* add one accepted pair (s, t, n) to H, g, sse and the absolute-value scales */
static void add_pair(int metric, const double s[3], const float* tp, const float* np_,
                     double H[36], double g[6], double* sse, double Habs[36], double gabs[6]) {
    double t[3] = {tp[0], tp[1], tp[2]};
    if (metric == MET_COMBINED) {
        /* the weighted sum of the two single-metric contributions of this pair */
        double Hp[36] = {0}, gp[6] = {0}, sp = 0.0, Hl[36] = {0}, gl[6] = {0}, sl = 0.0;
        add_pair(MET_P2POINT, s, tp, np_, Hp, gp, &sp, NULL, NULL);
        add_pair(MET_P2PLANE, s, tp, np_, Hl, gl, &sl, NULL, NULL);
        for (int a = 0; a < 36; ++a) {
            const double v = g_w_point * Hp[a] + g_w_plane * Hl[a];
            H[a] += v;
            if (Habs) Habs[a] += fabs(v);
        }
        for (int a = 0; a < 6; ++a) {
            const double v = g_w_point * gp[a] + g_w_plane * gl[a];
            g[a] += v;
            if (gabs) gabs[a] += fabs(v);
        }
        *sse += g_w_point * sp + g_w_plane * sl;
        return;
    }
    if (metric == MET_P2PLANE) {
        double n[3] = {np_[0], np_[1], np_[2]};
        double d[3] = {s[0] - t[0], s[1] - t[1], s[2] - t[2]};
        double r = d[0] * n[0] + d[1] * n[1] + d[2] * n[2];
        double J[6] = {s[1] * n[2] - s[2] * n[1], s[2] * n[0] - s[0] * n[2], s[0] * n[1] - s[1] * n[0],
                       n[0], n[1], n[2]};
        for (int a = 0; a < 6; ++a) {
            for (int c = 0; c < 6; ++c) {
                H[6 * a + c] += J[a] * J[c];
                if (Habs) Habs[6 * a + c] += fabs(J[a] * J[c]);
            }
            g[a] += J[a] * r;
            if (gabs) gabs[a] += fabs(J[a] * r);
        }
        *sse += r * r;
    } else {
        double r[3] = {s[0] - t[0], s[1] - t[1], s[2] - t[2]};
        /* J = [ -[s]x , I3 ] written out as a 3x6 matrix */
        double J[3][6] = {{0.0, s[2], -s[1], 1.0, 0.0, 0.0},
                          {-s[2], 0.0, s[0], 0.0, 1.0, 0.0},
                          {s[1], -s[0], 0.0, 0.0, 0.0, 1.0}};
        for (int a = 0; a < 6; ++a) {
            for (int c = 0; c < 6; ++c) {
                double v = 0.0, va = 0.0;
                for (int k = 0; k < 3; ++k) { v += J[k][a] * J[k][c]; }
                H[6 * a + c] += v;
                if (Habs) { for (int k = 0; k < 3; ++k) va += J[k][a] * J[k][c]; Habs[6 * a + c] += fabs(va); }
            }
            double v = 0.0;
            for (int k = 0; k < 3; ++k) v += J[k][a] * r[k];
            g[a] += v;
            if (gabs) gabs[a] += fabs(v);
        }
        *sse += r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
    }
}

/* One correspondence + normal-equation pass (steps a1-a5).
   corr_idx / corr_d2 / corr_d2nd (nullable, length m): matched target (or -1),
   its squared distance, and the second-best squared distance (+inf if none <= max_dist^2). */
int orc_icp_system(const void* kd, const float* tgt, const float* nrm, int64_t n,
                   const float* src, int64_t m, const double pose[16], int metric, double max_dist,
                   double H[36], double g[6], double* sse, int64_t* count,
                   double* Habs, double* gabs,
                   int64_t* corr_idx, double* corr_d2, double* corr_d2nd) {
    if ((metric == MET_P2PLANE || metric == MET_COMBINED) && !nrm) return 3;
    double bound2 = max_dist * max_dist;
    int64_t* ci = (int64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
    double* s = (double*)malloc((size_t)(m > 0 ? m : 1) * 3 * sizeof(double));
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < m; ++i) {
        kbest b;
        transform_point(pose, src + 3 * i, s + 3 * i);
        knn_one((const kdtree*)kd, tgt, n, s + 3 * i, 2, bound2, &b);
        ci[i] = b.cnt > 0 ? b.id[0] : -1;
        if (corr_d2) corr_d2[i] = b.cnt > 0 ? b.d2[0] : INFINITY;
        if (corr_d2nd) corr_d2nd[i] = b.cnt > 1 ? b.d2[1] : INFINITY;
    }
    memset(H, 0, 36 * sizeof(double));
    memset(g, 0, 6 * sizeof(double));
    if (Habs) memset(Habs, 0, 36 * sizeof(double));
    if (gabs) memset(gabs, 0, 6 * sizeof(double));
    *sse = 0.0;
    int64_t cnt = 0;
    for (int64_t i = 0; i < m; ++i) {
        if (corr_idx) corr_idx[i] = ci[i];
        if (ci[i] < 0) continue;
        add_pair(metric, s + 3 * i, tgt + 3 * ci[i], nrm ? nrm + 3 * ci[i] : NULL, H, g, sse, Habs, gabs);
        ++cnt;
    }
    *count = cnt;
    free(ci); free(s);
    return 0;
}

/* The same accumulation from GIVEN correspondences (reading R17):
   corr[i] = target index or -1.  Used to reconcile near-tie flips. */
int orc_icp_system_from_corr(const float* tgt, const float* nrm, int64_t n, const float* src, int64_t m,
                             const double pose[16], int metric, const int32_t* corr,
                             double H[36], double g[6], double* sse, int64_t* count,
                             double* Habs, double* gabs) {
    if ((metric == MET_P2PLANE || metric == MET_COMBINED) && !nrm) return 3;
    memset(H, 0, 36 * sizeof(double));
    memset(g, 0, 6 * sizeof(double));
    if (Habs) memset(Habs, 0, 36 * sizeof(double));
    if (gabs) memset(gabs, 0, 6 * sizeof(double));
    *sse = 0.0;
    int64_t cnt = 0;
    for (int64_t i = 0; i < m; ++i) {
        if (corr[i] < 0) continue;
        if (corr[i] >= n) return 1;
        double s[3];
        transform_point(pose, src + 3 * i, s);
        add_pair(metric, s, tgt + 3 * (int64_t)corr[i], nrm ? nrm + 3 * (int64_t)corr[i] : NULL, H, g, sse, Habs, gabs);
        ++cnt;
    }
    *count = cnt;
    return 0;
}

/* ------------------------------------------------------------------ solve + update */
/* Rodrigues: R = I + (sin th / th) [a]x + ((1 - cos th) / th^2) [a]x^2 */
void orc_rodrigues(const double a[3], double R[9]) {
    double th2 = a[0] * a[0] + a[1] * a[1] + a[2] * a[2];
    double th = sqrt(th2);
    double A, B;
    if (th < 1e-4) { A = 1.0 - th2 / 6.0; B = 0.5 - th2 / 24.0; }
    else { A = sin(th) / th; B = (1.0 - cos(th)) / th2; }
    double K[9] = {0.0, -a[2], a[1], a[2], 0.0, -a[0], -a[1], a[0], 0.0};
    double K2[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double v = 0.0;
            for (int k = 0; k < 3; ++k) v += K[3 * i + k] * K[3 * k + j];
            K2[3 * i + j] = v;
        }
    for (int i = 0; i < 9; ++i) R[i] = A * K[i] + B * K2[i];
    R[0] += 1.0; R[4] += 1.0; R[8] += 1.0;
}

/* Solve H x = -g (Cholesky, fp64) and left-compose the increment onto pose_in.
   Returns ORC_OK, ORC_NO_CORRESPONDENCES (count == 0) or ORC_DEGENERATE; in the latter
   two cases pose_out = pose_in and x = 0. */
int orc_solve_update(const double H[36], const double g[6], int64_t count, const double pose_in[16],
                     double pose_out[16], double x[6], double* theta, double* tnorm) {
    double P[16];
    memcpy(P, pose_in, sizeof(P));
    for (int i = 0; i < 6; ++i) x[i] = 0.0;
    *theta = 0.0; *tnorm = 0.0;
    if (count == 0) { memcpy(pose_out, P, sizeof(P)); return ORC_NO_CORRESPONDENCES; }
    if (count < 6) { memcpy(pose_out, P, sizeof(P)); return ORC_DEGENERATE; }
    double L[36] = {0};
    double pmin = INFINITY, pmax = 0.0;
    for (int j = 0; j < 6; ++j) {
        double d = H[6 * j + j];
        for (int k = 0; k < j; ++k) d -= L[6 * j + k] * L[6 * j + k];
        if (!(d > 0.0)) { memcpy(pose_out, P, sizeof(P)); return ORC_DEGENERATE; }
        if (d < pmin) pmin = d;
        if (d > pmax) pmax = d;
        double ljj = sqrt(d);
        L[6 * j + j] = ljj;
        for (int i = j + 1; i < 6; ++i) {
            double v = H[6 * i + j];
            for (int k = 0; k < j; ++k) v -= L[6 * i + k] * L[6 * j + k];
            L[6 * i + j] = v / ljj;
        }
    }
    if (pmin < 1e-12 * pmax) { memcpy(pose_out, P, sizeof(P)); return ORC_DEGENERATE; }
    double y[6];
    for (int i = 0; i < 6; ++i) {     /* L y = -g */
        double v = -g[i];
        for (int k = 0; k < i; ++k) v -= L[6 * i + k] * y[k];
        y[i] = v / L[6 * i + i];
    }
    for (int i = 5; i >= 0; --i) {    /* L^T x = y */
        double v = y[i];
        for (int k = i + 1; k < 6; ++k) v -= L[6 * k + i] * x[k];
        x[i] = v / L[6 * i + i];
    }
    double dR[9];
    orc_rodrigues(x, dR);
    double Rn[9], tn[3];
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) {
            double v = 0.0;
            for (int k = 0; k < 3; ++k) v += dR[3 * i + k] * P[4 * k + j];
            Rn[3 * i + j] = v;
        }
        double v = 0.0;
        for (int k = 0; k < 3; ++k) v += dR[3 * i + k] * P[4 * k + 3];
        tn[i] = v + x[3 + i];
    }
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) P[4 * i + j] = Rn[3 * i + j];
        P[4 * i + 3] = tn[i];
    }
    P[12] = 0.0; P[13] = 0.0; P[14] = 0.0; P[15] = 1.0;
    memcpy(pose_out, P, sizeof(P));
    *theta = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
    *tnorm = sqrt(x[3] * x[3] + x[4] * x[4] + x[5] * x[5]);
    return ORC_OK;
}

/* ------------------------------------------------------------------ projective association */
/* The second correspondence engine of the paper: projective data association for organised
   3-D clouds ("different correspondence search engines (e.g., kd-tree based or
   projective)", "one for correspondences by projective data association for the
   3D case"; SPEC.md:392-400 correspondences_projective; pixel rounding SPEC.md:117; DESIGN.md
   readings R23-R26).
   The target is organised: tgt[3 * (v * w + u)] is the point of pixel (u, v) in the target
   camera frame; a pixel is invalid when its z <= 0 or a coordinate is not finite.
   intr = {fx, fy, cx, cy}.  For source point p: s = R p + t; if s_z > 0 then
   u = round(fx * s_x / s_z + cx), v = round(fy * s_y / s_z + cy) with C round() (half away
   from zero); the pair (i, v * w + u) exists iff 0 <= u < w, 0 <= v < h, the pixel is valid
   and |s - t|^2 <= max_dist^2 (inclusive, as R2).
   Returns the pixel index or -1; *d2 = |s - t|^2 of an accepted pair, else +inf; uv (nullable)
   = the unrounded (u, v), NaN when s_z <= 0 (tests use it for the rounding band R24). */
static int64_t proj_one(const float* tgt, int64_t w, int64_t h, const double intr[4], const double s[3],
                        double bound2, double* d2, double* uv) {
    *d2 = INFINITY;
    if (uv) { uv[0] = NAN; uv[1] = NAN; }
    if (!(s[2] > 0.0)) return -1;
    double uf = intr[0] * s[0] / s[2] + intr[2];
    double vf = intr[1] * s[1] / s[2] + intr[3];
    if (uv) { uv[0] = uf; uv[1] = vf; }
    double ur = round(uf), vr = round(vf);
    if (!(ur >= 0.0 && ur < (double)w && vr >= 0.0 && vr < (double)h)) return -1;
    int64_t k = (int64_t)vr * w + (int64_t)ur;
    const float* t = tgt + 3 * k;
    if (!(t[2] > 0.0f) || !isfinite(t[0]) || !isfinite(t[1]) || !isfinite(t[2])) return -1;
    double e = dist2(s, t);
    if (!(e <= bound2)) return -1;
    *d2 = e;
    return k;
}

/* One projective correspondence + normal-equation pass (a1, projective a2, a3-a5), the
   accumulation serial in source-index order exactly as orc_icp_system. */
int orc_proj_system(const float* tgt, const float* nrm, int64_t w, int64_t h, const double intr[4],
                    const float* src, int64_t m, const double pose[16], int metric, double max_dist,
                    double H[36], double g[6], double* sse, int64_t* count, double* Habs, double* gabs,
                    int64_t* corr_idx, double* corr_d2, double* uv) {
    if ((metric == MET_P2PLANE || metric == MET_COMBINED) && !nrm) return 3;
    if (w < 1 || h < 1) return 1;
    double bound2 = max_dist * max_dist;
    memset(H, 0, 36 * sizeof(double));
    memset(g, 0, 6 * sizeof(double));
    if (Habs) memset(Habs, 0, 36 * sizeof(double));
    if (gabs) memset(gabs, 0, 6 * sizeof(double));
    *sse = 0.0;
    int64_t cnt = 0;
    for (int64_t i = 0; i < m; ++i) {
        double s[3], d2;
        transform_point(pose, src + 3 * i, s);
        int64_t k = proj_one(tgt, w, h, intr, s, bound2, &d2, uv ? uv + 2 * i : NULL);
        if (corr_idx) corr_idx[i] = k;
        if (corr_d2) corr_d2[i] = d2;
        if (k < 0) continue;
        add_pair(metric, s, tgt + 3 * k, nrm ? nrm + 3 * k : NULL, H, g, sse, Habs, gabs);
        ++cnt;
    }
    *count = cnt;
    return 0;
}

/* ------------------------------------------------------------------ ICP loop */
/* iter_log (nullable) [max_iters*2] = {n_corr, rmse}; H_log [max_iters*36], g_log [max_iters*6]
   (nullable) record each executed iteration's system; pose_log [max_iters*16] the pose
   after each executed iteration. */
/* engine 0: exact NN (kd or brute force); engine 1: projective (w, h, intr) */
static int icp_loop(int engine, const void* kd, const float* tgt, const float* nrm, int64_t n,
                    int64_t w, int64_t h, const double* intr,
                    const float* src, int64_t m, const double pose_init[16], int metric, int max_iters,
                    double max_dist, double rot_tol, double trans_tol,
                    double pose_out[16], double* rmse, int64_t* n_corr, int32_t* iterations,
                    int32_t* converged, int32_t* status,
                    double* iter_log, double* H_log, double* g_log, double* pose_log) {
    double P[16];
    memcpy(P, pose_init, sizeof(P));
    *rmse = 0.0; *n_corr = 0; *iterations = 0; *converged = 0; *status = ORC_OK;
    for (int it = 0; it < max_iters; ++it) {
        double H[36], g[6], sse, x[6], th, tn;
        int64_t cnt;
        int rc = engine == 0
                     ? orc_icp_system(kd, tgt, nrm, n, src, m, P, metric, max_dist, H, g, &sse, &cnt,
                                      NULL, NULL, NULL, NULL, NULL)
                     : orc_proj_system(tgt, nrm, w, h, intr, src, m, P, metric, max_dist, H, g, &sse, &cnt,
                                       NULL, NULL, NULL, NULL, NULL);
        if (rc) return rc;
        *iterations = it + 1;
        double r = cnt > 0 ? sqrt(sse / (double)cnt) : 0.0;
        if (iter_log) { iter_log[2 * it] = (double)cnt; iter_log[2 * it + 1] = r; }
        if (H_log) memcpy(H_log + 36 * it, H, sizeof(H));
        if (g_log) memcpy(g_log + 6 * it, g, sizeof(g));
        *n_corr = cnt;
        *rmse = r;
        int st = orc_solve_update(H, g, cnt, P, P, x, &th, &tn);
        if (pose_log) memcpy(pose_log + 16 * it, P, sizeof(P));
        if (st != ORC_OK) { *status = st; *converged = 0; break; }
        if (th < rot_tol && tn < trans_tol) { *converged = 1; break; }
    }
    memcpy(pose_out, P, sizeof(P));
    return 0;
}

int orc_icp_run(const void* kd, const float* tgt, const float* nrm, int64_t n,
                const float* src, int64_t m, const double pose_init[16], int metric, int max_iters,
                double max_dist, double rot_tol, double trans_tol,
                double pose_out[16], double* rmse, int64_t* n_corr, int32_t* iterations,
                int32_t* converged, int32_t* status,
                double* iter_log, double* H_log, double* g_log, double* pose_log) {
    return icp_loop(0, kd, tgt, nrm, n, 0, 0, NULL, src, m, pose_init, metric, max_iters, max_dist, rot_tol,
                    trans_tol, pose_out, rmse, n_corr, iterations, converged, status, iter_log, H_log, g_log, pose_log);
}

/* the ICP loop with projective correspondences (the same solve/update and stop rules) */
int orc_proj_run(const float* tgt, const float* nrm, int64_t w, int64_t h, const double intr[4],
                 const float* src, int64_t m, const double pose_init[16], int metric, int max_iters,
                 double max_dist, double rot_tol, double trans_tol,
                 double pose_out[16], double* rmse, int64_t* n_corr, int32_t* iterations,
                 int32_t* converged, int32_t* status,
                 double* iter_log, double* H_log, double* g_log, double* pose_log) {
    if (w < 1 || h < 1) return 1;
    return icp_loop(1, NULL, tgt, nrm, w * h, w, h, intr, src, m, pose_init, metric, max_iters, max_dist, rot_tol,
                    trans_tol, pose_out, rmse, n_corr, iterations, converged, status, iter_log, H_log, g_log, pose_log);
}

/* ------------------------------------------------------------------ PCA normals */
/* cyclic Jacobi eigen-decomposition of a symmetric 3x3 matrix; V columns = eigenvectors */
static void jacobi3(double A[9], double w[3], double V[9]) {
    for (int i = 0; i < 9; ++i) V[i] = (i % 4 == 0) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 50; ++sweep) {
        double off = fabs(A[1]) + fabs(A[2]) + fabs(A[5]);
        if (off == 0.0) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                double apq = A[3 * p + q];
                if (apq == 0.0) continue;
                double app = A[3 * p + p], aqq = A[3 * q + q];
                double tau = (aqq - app) / (2.0 * apq);
                double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                for (int k = 0; k < 3; ++k) {   /* A <- A J */
                    double akp = A[3 * k + p], akq = A[3 * k + q];
                    A[3 * k + p] = c * akp - s * akq;
                    A[3 * k + q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) {   /* A <- J^T A */
                    double apk = A[3 * p + k], aqk = A[3 * q + k];
                    A[3 * p + k] = c * apk - s * aqk;
                    A[3 * q + k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 3; ++k) {   /* V <- V J */
                    double vkp = V[3 * k + p], vkq = V[3 * k + q];
                    V[3 * k + p] = c * vkp - s * vkq;
                    V[3 * k + q] = s * vkp + c * vkq;
                }
            }
    }
    w[0] = A[0]; w[1] = A[4]; w[2] = A[8];
}

/* normal of each point = eigenvector of the smallest eigenvalue of the 1/k covariance of its
   k nearest neighbours (self included), flipped to face `view`. */
int orc_pca_normals(const void* kd, const float* pts, int64_t n, int k, const double view[3],
                    float* nrm_out, float* curvature_out) {
    if (k < 1 || k > ORC_KMAX) return 1;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
        double q[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
        kbest b;
        knn_one((const kdtree*)kd, pts, n, q, k, INFINITY, &b);
        double mu[3] = {0, 0, 0};
        for (int r = 0; r < b.cnt; ++r)
            for (int a = 0; a < 3; ++a) mu[a] += pts[3 * b.id[r] + a];
        for (int a = 0; a < 3; ++a) mu[a] /= (double)b.cnt;
        double C[9] = {0};
        for (int r = 0; r < b.cnt; ++r) {
            double d[3];
            for (int a = 0; a < 3; ++a) d[a] = pts[3 * b.id[r] + a] - mu[a];
            for (int a = 0; a < 3; ++a)
                for (int c = 0; c < 3; ++c) C[3 * a + c] += d[a] * d[c];
        }
        for (int a = 0; a < 9; ++a) C[a] /= (double)b.cnt;
        double w[3], V[9];
        jacobi3(C, w, V);
        int sm = 0;
        for (int a = 1; a < 3; ++a) if (w[a] < w[sm]) sm = a;
        double nv[3] = {V[0 * 3 + sm], V[1 * 3 + sm], V[2 * 3 + sm]};
        double nn = sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
        for (int a = 0; a < 3; ++a) nv[a] /= nn;
        double dv = (view[0] - q[0]) * nv[0] + (view[1] - q[1]) * nv[1] + (view[2] - q[2]) * nv[2];
        if (dv < 0) for (int a = 0; a < 3; ++a) nv[a] = -nv[a];
        for (int a = 0; a < 3; ++a) nrm_out[3 * i + a] = (float)nv[a];
        if (curvature_out) {
            double tr = w[0] + w[1] + w[2];
            curvature_out[i] = (float)(tr > 0 ? w[sm] / tr : 0.0);
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ voxel-grid downsampling */
/* "general dimension grid-based point cloud downsampling",
   "downsampled using a voxel grid of bin size equal to 1cm"; SPEC.md:242-256
   (grid_downsample) and DESIGN.md readings R27-R29:
     key_a(p) = floor((p_a - origin_a) / bin)     (fp64: promote, subtract, divide, floor)
     output: one point per non-empty bin = the fp64 mean of its points (summed in increasing
     input index, divided by the count, cast to fp32); normals (nullable): the fp64 mean of the
     bin's normals, divided by its norm sqrt(x*x + y*y + z*z), or 0 if that norm < 1e-12;
     bins in ascending lexicographic (key_x, key_y, key_z) order.
   Returns the number of bins, or -1 when a key is not finite / outside int32. */
typedef struct { int64_t kx, ky, kz, idx; } vox_item;

static int vox_cmp(const void* a, const void* b) {
    const vox_item* x = (const vox_item*)a;
    const vox_item* y = (const vox_item*)b;
    if (x->kx != y->kx) return x->kx < y->kx ? -1 : 1;
    if (x->ky != y->ky) return x->ky < y->ky ? -1 : 1;
    if (x->kz != y->kz) return x->kz < y->kz ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

int64_t orc_voxel_downsample(const float* pts, const float* nrm, int64_t n, double bin, const double origin[3],
                             float* out_pts, float* out_nrm, int64_t* out_keys /* nullable [3*bins] */) {
    if (n <= 0) return 0;
    vox_item* it = (vox_item*)malloc((size_t)n * sizeof(vox_item));
    for (int64_t i = 0; i < n; ++i) {
        double k[3];
        for (int a = 0; a < 3; ++a) {
            k[a] = floor(((double)pts[3 * i + a] - origin[a]) / bin);
            if (!(k[a] >= -2147483648.0 && k[a] <= 2147483647.0)) { free(it); return -1; }
        }
        it[i].kx = (int64_t)k[0]; it[i].ky = (int64_t)k[1]; it[i].kz = (int64_t)k[2]; it[i].idx = i;
    }
    qsort(it, (size_t)n, sizeof(vox_item), vox_cmp);
    int64_t nb = 0;
    for (int64_t s = 0; s < n;) {
        int64_t e = s;
        while (e < n && it[e].kx == it[s].kx && it[e].ky == it[s].ky && it[e].kz == it[s].kz) ++e;
        double c[3] = {0.0, 0.0, 0.0}, m[3] = {0.0, 0.0, 0.0};
        for (int64_t r = s; r < e; ++r)         /* increasing input index (the sort's tie order) */
            for (int a = 0; a < 3; ++a) {
                c[a] += (double)pts[3 * it[r].idx + a];
                if (nrm) m[a] += (double)nrm[3 * it[r].idx + a];
            }
        const double cnt = (double)(e - s);
        for (int a = 0; a < 3; ++a) out_pts[3 * nb + a] = (float)(c[a] / cnt);
        if (nrm) {
            for (int a = 0; a < 3; ++a) m[a] = m[a] / cnt;
            const double len = sqrt(m[0] * m[0] + m[1] * m[1] + m[2] * m[2]);
            for (int a = 0; a < 3; ++a) out_nrm[3 * nb + a] = len < 1e-12 ? 0.0f : (float)(m[a] / len);
        }
        if (out_keys) { out_keys[3 * nb] = it[s].kx; out_keys[3 * nb + 1] = it[s].ky; out_keys[3 * nb + 2] = it[s].kz; }
        ++nb;
        s = e;
    }
    free(it);
    return nb;
}
