// icp.cu -- the fused ICP iteration and the device-resident
// loop.  BASELINE.json north_star subsystems (4) "the fused transform+reject+J^TJ/J^Tr kernel,
// with per-warp shuffle reductions and per-block fp32 partials reduced in fp64" and (5) "the
// on-device 6x6 Cholesky solve and pose update, so an iteration loop launches with no host
// round-trip".
//
// One iteration of cil_icp_run = three launches:
//   K_sel (certified warm start): for every source point, its previous
//         exact match j1 found at anchor pose T_a with 2nd-best gap G = d2 - d1 stays exact
//         at the current pose T if G > 2 |(R - R_a) p + (t - t_a)| (with rounding margins);
//         every other point is appended to the search list.
//   K_nn  (correspondence kernel, north_star subsystem (3)): persistent warp-packet search
//         engine (search.cuh) over the list -- a1 s = R p_i + t (fp64 -> double-float), a2
//         exact 1-NN and exact 2nd-best d2 bounded by rho = 1.1 max_corr_dist, hint leaf =
//         the previous match; writes nn[i] (original target index or -1) and the gap word
//         (gap rounded toward zero, low 8 bits = anchor slot).
//   K_acc (fused transform+reject+J^TJ/J^Tr kernel, subsystem (4)), static grid-stride:
//     a1  s = R p_i + t again (fp64 -> double-float), d2 to t_nn[i] (same arithmetic as K_nn)
//     a3  accept iff d2 <= fl32(max_corr_dist^2)
//     a4  residual + Jacobian of the metric for accepted pairs (PAPER.md:140 [Besl], [Low])
//     a5  fp32 per-thread sums (29 point-to-plane / 17 point-to-point values)
//   warp: transposed butterfly reduce (31 SHFL for 32 values; lane k ends with sum k)
//   block: per-warp fp64 sums -> per-CTA fp64 partial in the workspace
//   last CTA (ticket): ordered fp64 sum of the partials -> a6 Cholesky solve -> a7 pose update,
//   status, log, anchor-pose table for the next K_sel.  Results are bitwise reproducible run
//   to run (fixed grid, fixed orders, no floating-point atomics; the search result of a
//   query does not depend on which warp searches it).
// cil_icp_iterate = K_nn over all points (no hints, bound max_corr_dist) + K_acc.
#include "internal.cuh"
#include "search.cuh"
#include "grid.cuh"

#include <algorithm>
#include <cmath>

namespace cil {
namespace {

constexpr int kIcpThreads = 256;
#ifndef CIL_SKIN_CUT
#define CIL_SKIN_CUT 8.0f
#endif
// a point whose kappa x last-step displacement exceeds kSkinCut x gap_max searches with the
// minimal skin (it would not keep a certificate anyway)
constexpr float kSkinCut = CIL_SKIN_CUT;
#ifndef CIL_KD_WARP_SOLVE
#define CIL_KD_WARP_SOLVE true   // the last-CTA solve of the kd path by one warp (solve6_warp)
#endif
#ifndef CIL_RHO
#define CIL_RHO 1.1           // certificate search bound rho = CIL_RHO x max_corr_dist
#endif
#ifndef CIL_STALE
#define CIL_STALE 0.01        // a warm hint beyond sqrt(CIL_STALE) x max_corr_dist also tries the cold hint
#endif
constexpr int kIcpWarps = kIcpThreads / 32;

struct IterArgs {
    TargetView T;
    const float* src;
    int m;
    float bound2;            // fl32(max_corr_dist^2): acceptance (a3)
    float w_pp, w_pl;        // CIL_COMBINED weights (fl32 of w_point, w_plane)
    float search2;           // search bound: bound2, or fl32(rho^2) with certificates
    float gap_none;          // certificate of "no target within rho": rho - max_corr_dist (rounded down)
    float gap_min, gap_max, kappa;   // per-point certificate skin clamp(kappa * last step, gap_min, gap_max)
    float stale2;            // (max_corr_dist / 10)^2: a warm hint beyond it is stale
    const double* pose_in;
    double* pose_out;
    double* partials;        // [kSlots][kMaxCtas] slot-major: per-CTA fp64 partial sums
    IcpState* st;
    cil_icp_system* sys;     // iterate only, nullable
    int32_t* corr_idx;       // iterate only, nullable (indexed by the caller's source order)
    float* corr_d2;          // iterate only, nullable
    const uint32_t* perm;    // sorted slot -> caller's source index (the kernels run in Morton order)
    float* srcs;             // [m*3] the source in Morton order (workspace)
    int* nn;                 // [m] match per query (original target index or -1)
    uint32_t* gw;            // [m] leaf-certificate word (run): bits(G1) & ~255 | anchor slot
    float* gs;               // [m] list-certificate margin G_S (run)
    float* gd1;              // [m] d1 at the search anchor, rounded up (run)
    uint32_t* gp;            // [m] point certificate: bits(G_pt) & ~255 | slot of the iteration it was measured
    int* vlist;              // [m][kListLeaves] candidate leaves of the last search (run), -1 padded
    uint32_t* pmask;         // [ceil(m/32)] per 32-query packet: lanes that need a full search (run)
    int* plist;              // [ceil(m/32)] packets with a non-empty mask (any order; count st->plist_n)
    double* apose;           // [kAnchorSlots][12] pose of each anchor slot (run)
    float* adelta;           // [kAnchorSlots][16] (R - R_a | t - t_a | max|dR| | max|dt|) for the current pose
    double* iter_log;        // run only, nullable
    // projective data association (cil_proj_*): organised target, intrinsics (R23-R25)
    const float* ptgt;       // [pw * ph * 3] row-major pixels, caller's buffer
    const float* pnrm;       // [pw * ph * 3] or nullptr
    int pw, ph;
    double pfx, pfy, pcx, pcy;
    unsigned long long* stamps;   // diagnostics (cil_debug_timestamps), normally nullptr
    double* sums_out;        // shard mode (cil_icp_shard_accumulate): the rank-local reduced sums [kSlots]
    int run;
    int cert;                // run: certified warm start on
    int point_cert;          // run: the point-level certificate on (diagnostics switch)
    double rot_tol, trans_tol;
};

// Programmatic dependent launch: the per-iteration kernels are launched with the
// programmatic-stream-serialization attribute (launch_pdl); each calls pdl_trigger() first
// (its dependent may be scheduled once every CTA of it has started) and pdl_wait() before it
// reads anything an earlier kernel wrote (the wait returns when the previous grid has
// completed and flushed), so the launch latency of kernel k+1 overlaps the tail of kernel k.

// diagnostics: %globaltimer stamp k of the running iteration (first = earliest CTA)
__device__ __forceinline__ void stamp(const IterArgs& a, int k, bool first) {
    if (!a.stamps || threadIdx.x != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const int it = a.run ? *(volatile int*)&a.st->iters : 0;
    if (first) atomicMin(a.stamps + 8 * it + k, t);
    else a.stamps[8 * it + k] = t;
}

__device__ __forceinline__ float warp_transpose_reduce(float (&v)[kSlots]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int j = 0; j < off; ++j) {
            float send = upper ? v[j] : v[j + off];
            float keep = upper ? v[j + off] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return v[0];
}

// ---------------------------------------------------------------- a6 + a7 (one thread)
// The tail below runs once per iteration on one thread of one CTA (from a cold instruction
// cache; measured with cil_debug_timestamps: ~5 us of the iteration).
__device__ __noinline__ void rodrigues_sc(double th, double th2, double* A, double* Bc) {
    double sn, cs;
    sincos(th, &sn, &cs);
    *A = sn / th;
    *Bc = (1.0 - cs) / th2;
}

__device__ __noinline__ void rodrigues(const double a[3], double R[9]) {
    const double th2 = a[0] * a[0] + a[1] * a[1] + a[2] * a[2];
    double A, Bc;
    if (th2 < 1e-4) {
        // theta < 1e-2: sin(t)/t and (1 - cos t)/t^2 by their Taylor series through t^10
        // (the first omitted term is < 1e-24 relative)
        const double u = th2;
        A = 1.0 - u * (1.0 / 6.0) * (1.0 - u * (1.0 / 20.0) * (1.0 - u * (1.0 / 42.0) * (1.0 - u * (1.0 / 72.0) *
                                                                                      (1.0 - u * (1.0 / 110.0)))));
        Bc = 0.5 * (1.0 - u * (1.0 / 12.0) * (1.0 - u * (1.0 / 30.0) * (1.0 - u * (1.0 / 56.0) *
                                                                        (1.0 - u * (1.0 / 90.0) * (1.0 - u * (1.0 / 132.0))))));
    } else {
        rodrigues_sc(sqrt(th2), th2, &A, &Bc);
    }
    // R = I + A [a]x + Bc [a]x^2,  [a]x^2 = a a^T - th2 I
    R[0] = 1.0 + Bc * (a[0] * a[0] - th2);
    R[4] = 1.0 + Bc * (a[1] * a[1] - th2);
    R[8] = 1.0 + Bc * (a[2] * a[2] - th2);
    R[1] = -A * a[2] + Bc * a[0] * a[1];
    R[3] = A * a[2] + Bc * a[0] * a[1];
    R[2] = A * a[1] + Bc * a[0] * a[2];
    R[6] = -A * a[1] + Bc * a[0] * a[2];
    R[5] = -A * a[0] + Bc * a[1] * a[2];
    R[7] = A * a[0] + Bc * a[1] * a[2];
}

// Build (H, g, sse, count) from the reduced sums of the metric.
template <int METRIC>
__device__ __noinline__ void assemble(const double* S, double H[36], double g[6], double& sse, double& cnt) {
    if (METRIC != CIL_POINT_TO_POINT) {          // point-to-plane and combined: 21 + 6 + sse + count
        int k = 0;
        for (int a = 0; a < 6; ++a)
            for (int b = a; b < 6; ++b, ++k) { H[6 * a + b] = S[k]; H[6 * b + a] = S[k]; }
        for (int a = 0; a < 6; ++a) g[a] = S[21 + a];
        sse = S[27];
        cnt = S[28];
    } else {
        cnt = S[0];
        const double Sx = S[1], Sy = S[2], Sz = S[3];
        const double xx = S[4], yy = S[5], zz = S[6], xy = S[7], xz = S[8], yz = S[9];
        // H_rr = sum(|s|^2 I - s s^T), formed from the diagonal sums (no cancellation)
        H[0] = yy + zz; H[1] = -xy;     H[2] = -xz;
        H[6] = -xy;     H[7] = xx + zz; H[8] = -yz;
        H[12] = -xz;    H[13] = -yz;    H[14] = xx + yy;
        // H_rt = [sum s]x, H_tr = H_rt^T, H_tt = count I
        const double Hrt[9] = {0.0, -Sz, Sy, Sz, 0.0, -Sx, -Sy, Sx, 0.0};
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                H[6 * a + 3 + b] = Hrt[3 * a + b];
                H[6 * (3 + b) + a] = Hrt[3 * a + b];
                H[6 * (3 + a) + 3 + b] = a == b ? cnt : 0.0;
            }
        g[0] = S[13]; g[1] = S[14]; g[2] = S[15];   // sum s x r
        g[3] = S[10]; g[4] = S[11]; g[5] = S[12];   // sum r
        sse = S[16];
    }
}

// Cholesky solve of H x = -g with the degeneracy rule of DESIGN.md R9; returns status.
__device__ __noinline__ int solve6(const double H[36], const double g[6], double cnt, double x[6]) {
    for (int i = 0; i < 6; ++i) x[i] = 0.0;
    if (cnt == 0.0) return CIL_NO_CORRESPONDENCES;
    if (cnt < 6.0) return CIL_ERR_DEGENERATE;
    double L[36];
    double pmin = INFINITY, pmax = 0.0;
    for (int j = 0; j < 6; ++j) {
        double d = H[6 * j + j];
        for (int k = 0; k < j; ++k) d -= L[6 * j + k] * L[6 * j + k];
        if (!(d > 0.0)) return CIL_ERR_DEGENERATE;
        pmin = fmin(pmin, d);
        pmax = fmax(pmax, d);
        const double ljj = sqrt(d);
        L[6 * j + j] = ljj;
        const double inv = 1.0 / ljj;
        for (int i = j + 1; i < 6; ++i) {
            double v = H[6 * i + j];
            for (int k = 0; k < j; ++k) v -= L[6 * i + k] * L[6 * j + k];
            L[6 * i + j] = v * inv;
        }
    }
    if (pmin < 1e-12 * pmax) return CIL_ERR_DEGENERATE;
    double y[6];
    for (int i = 0; i < 6; ++i) {
        double v = -g[i];
        for (int k = 0; k < i; ++k) v -= L[6 * i + k] * y[k];
        y[i] = v / L[6 * i + i];
    }
    for (int i = 5; i >= 0; --i) {
        double v = y[i];
        for (int k = i + 1; k < 6; ++k) v -= L[6 * k + i] * x[k];
        x[i] = v / L[6 * i + i];
    }
    return CIL_OK;
}

// a6 + a7 as a pure function of the reduced sums S and the pose P: the solve x, the new pose
// Pn (= P unless the status is CIL_OK), the system (H, g), sse and the pair count
template <int METRIC>
__device__ __forceinline__ int solve_pose(const double* S, const double* P, double H[36], double g[6], double x[6],
                                          double Pn[16], double& sse, double& cnt) {
    assemble<METRIC>(S, H, g, sse, cnt);
    const int status = solve6(H, g, cnt, x);
    for (int i = 0; i < 16; ++i) Pn[i] = P[i];
    if (status == CIL_OK) {
        double dR[9];
        rodrigues(x, dR);
        for (int i = 0; i < 3; ++i) {
            for (int j = 0; j < 3; ++j)
                Pn[4 * i + j] = dR[3 * i] * P[j] + dR[3 * i + 1] * P[4 + j] + dR[3 * i + 2] * P[8 + j];
            Pn[4 * i + 3] = dR[3 * i] * P[3] + dR[3 * i + 1] * P[7] + dR[3 * i + 2] * P[11] + x[3 + i];
        }
        Pn[12] = 0.0; Pn[13] = 0.0; Pn[14] = 0.0; Pn[15] = 1.0;
    }
    return status;
}

// The same solve by one whole warp, register-resident (the persistent projective loop, where
// it runs every iteration on every SM from a warm instruction cache): lane i < 6 holds row i
// of H and of the factor L; column j takes lane j's pivot and L's row j by shuffles, lanes
// i > j form L[i][j] in parallel; reciprocal pivots from rsqrt (1 ulp); every lane then runs
// both triangular solves on a shuffled copy of L.  H and g in shared memory; returns the status
// (uniform over the warp) and x (every lane).
__device__ __forceinline__ int solve6_warp(const double* Hs, const double* gs, double cnt, double (&x)[6]) {
    const int lane = threadIdx.x & 31;
    const int r = lane < 6 ? lane : 0;
#pragma unroll
    for (int i = 0; i < 6; ++i) x[i] = 0.0;
    if (cnt == 0.0) return CIL_NO_CORRESPONDENCES;
    if (cnt < 6.0) return CIL_ERR_DEGENERATE;
    double h[6], l[6], rinv[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) { h[k] = Hs[6 * r + k]; l[k] = 0.0; }
    double pmin = INFINITY, pmax = 0.0;
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        double lj[6];
#pragma unroll
        for (int k = 0; k < j; ++k) lj[k] = __shfl_sync(0xffffffffu, l[k], j);
        double v = h[j];
#pragma unroll
        for (int k = 0; k < j; ++k) v -= l[k] * lj[k];
        const double d = __shfl_sync(0xffffffffu, v, j);
        if (!(d > 0.0)) return CIL_ERR_DEGENERATE;
        pmin = fmin(pmin, d);
        pmax = fmax(pmax, d);
        const double iv = rsqrt(d);
        rinv[j] = iv;
        l[j] = lane == j ? d * iv : (lane > j ? v * iv : 0.0);
    }
    if (pmin < 1e-12 * pmax) return CIL_ERR_DEGENERATE;
    double L[6][6];
#pragma unroll
    for (int i = 1; i < 6; ++i)
#pragma unroll
        for (int k = 0; k < i; ++k) L[i][k] = __shfl_sync(0xffffffffu, l[k], i);
    double y[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        double v = -gs[i];
#pragma unroll
        for (int k = 0; k < i; ++k) v -= L[i][k] * y[k];
        y[i] = v * rinv[i];
    }
#pragma unroll
    for (int i = 5; i >= 0; --i) {
        double v = y[i];
#pragma unroll
        for (int k = i + 1; k < 6; ++k) v -= L[k][i] * x[k];
        x[i] = v * rinv[i];
    }
    return CIL_OK;
}

// a6 + a7 by one warp (all 32 lanes; every lane ends with the same x and Pn): lane 0 assembles
// H and g into shared memory, solve6_warp, then every lane composes the pose (identical
// arithmetic on every lane).  Hs / gsh / scal: shared scratch (36 / 6 / 2 doubles).
template <int METRIC>
__device__ __forceinline__ int solve_pose_warp(const double* S, const double* P, double* Hs, double* gsh, double* scal,
                                               double (&x)[6], double (&Pn)[16]) {
    if ((threadIdx.x & 31) == 0) assemble<METRIC>(S, Hs, gsh, scal[0], scal[1]);
    __syncwarp();
    const int status = solve6_warp(Hs, gsh, scal[1], x);
#pragma unroll
    for (int i = 0; i < 16; ++i) Pn[i] = P[i];
    if (status == CIL_OK) {
        double dR[9];
        rodrigues(x, dR);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
#pragma unroll
            for (int j = 0; j < 3; ++j)
                Pn[4 * i + j] = dR[3 * i] * P[j] + dR[3 * i + 1] * P[4 + j] + dR[3 * i + 2] * P[8 + j];
            Pn[4 * i + 3] = dR[3 * i] * P[3] + dR[3 * i + 1] * P[7] + dR[3 * i + 2] * P[11] + x[3 + i];
        }
        Pn[12] = 0.0; Pn[13] = 0.0; Pn[14] = 0.0; Pn[15] = 1.0;
    }
    return status;
}

// What a6 + a7 write, by value: passing the whole kernel-parameter IterArgs by reference into a
// noinline function made every thread of the accumulation kernels copy it (~430 B) to local
// memory at kernel entry (32 MB of local stores per C4 iteration).
struct FinArgs {
    IcpState* st;
    double* iter_log;
    double* pose_out;
    cil_icp_system* sys;
    unsigned long long* stamps;
    double rot_tol, trans_tol;
    int run;
};

__device__ __forceinline__ FinArgs fin_args(const IterArgs& a) {
    FinArgs f;
    f.st = a.st; f.iter_log = a.iter_log; f.pose_out = a.pose_out; f.sys = a.sys; f.stamps = a.stamps;
    f.rot_tol = a.rot_tol; f.trans_tol = a.trans_tol; f.run = a.run;
    return f;
}

// finalize with the warp solve (warp 0 of the last CTA; the projective engine)
template <int METRIC>
__device__ __noinline__ void finalize_warp(const FinArgs a, const double* S, const double* P) {
    __shared__ double Hs[36], gsh[6], scal[2];
    double x[6], Pn[16];
    const int status = solve_pose_warp<METRIC>(S, P, Hs, gsh, scal, x, Pn);
    if ((threadIdx.x & 31) != 0) return;
    const double sse = scal[0], cnt = scal[1];
    const double rmse = cnt > 0.0 ? sqrt(sse / cnt) : 0.0;
    if (a.run) {
        IcpState* st = a.st;
        const int it = st->iters;
        if (a.iter_log) { a.iter_log[2 * it] = cnt; a.iter_log[2 * it + 1] = rmse; }
        st->iters = it + 1;
        st->n_corr = (long long)cnt;
        st->rmse = rmse;
        if (status != CIL_OK) {
            st->status = status;
            st->converged = 0;
            st->done = 1;
        } else {
            for (int i = 0; i < 16; ++i) st->pose[i] = Pn[i];
            const double th = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
            const double tn = sqrt(x[3] * x[3] + x[4] * x[4] + x[5] * x[5]);
            if (th < a.rot_tol && tn < a.trans_tol) { st->converged = 1; st->done = 1; }
        }
    } else {
        for (int i = 0; i < 16; ++i) a.pose_out[i] = Pn[i];
        if (a.sys) {
            for (int i = 0; i < 36; ++i) a.sys->H[i] = Hs[i];
            for (int i = 0; i < 6; ++i) { a.sys->g[i] = gsh[i]; a.sys->x[i] = x[i]; }
            a.sys->sse = sse;
            a.sys->n_corr = (long long)cnt;
            a.sys->status = status;
            a.sys->pad = 0;
        }
    }
}

template <int METRIC>
__device__ __noinline__ void finalize(const FinArgs a, const double* S, const double* P) {
    double H[36], g[6], x[6], Pn[16], sse, cnt;
    const int status = solve_pose<METRIC>(S, P, H, g, x, Pn, sse, cnt);
    if (a.stamps) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.stamps[8 * (a.run ? a.st->iters : 0) + 6] = t;
    }
    const double rmse = cnt > 0.0 ? sqrt(sse / cnt) : 0.0;
    if (a.run) {
        IcpState* st = a.st;
        const int it = st->iters;
        if (a.iter_log) { a.iter_log[2 * it] = cnt; a.iter_log[2 * it + 1] = rmse; }
        st->iters = it + 1;
        st->n_corr = (long long)cnt;
        st->rmse = rmse;
        if (status != CIL_OK) {
            st->status = status;
            st->converged = 0;
            st->done = 1;
        } else {
            for (int i = 0; i < 16; ++i) st->pose[i] = Pn[i];
            const double th = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
            const double tn = sqrt(x[3] * x[3] + x[4] * x[4] + x[5] * x[5]);
            if (th < a.rot_tol && tn < a.trans_tol) { st->converged = 1; st->done = 1; }
        }
    } else {
        for (int i = 0; i < 16; ++i) a.pose_out[i] = Pn[i];
        if (a.sys) {
            for (int i = 0; i < 36; ++i) a.sys->H[i] = H[i];
            for (int i = 0; i < 6; ++i) { a.sys->g[i] = g[i]; a.sys->x[i] = x[i]; }
            a.sys->sse = sse;
            a.sys->n_corr = (long long)cnt;
            a.sys->status = status;
            a.sys->pad = 0;
        }
    }
}

// ---------------------------------------------------------------- K_sel (certified warm start)
// Displacement bound of source point p between its anchor pose T_a and the current pose T:
// v = (R - R_a) p + (t - t_a) in fp32 from the per-slot table; the bound adds the rounding
// of the table entries and of the 3-term dot products (|err_k| <= 2^-21 (max|dR| |p|_1 +
// max|dt|)), and an absolute 2^-30 (|p|_1 + 1) for the double-float representation of s.
__device__ __forceinline__ float displacement_bound(const float* __restrict__ D, float px, float py, float pz) {
    const float4 d0 = __ldg(reinterpret_cast<const float4*>(D));
    const float4 d1 = __ldg(reinterpret_cast<const float4*>(D) + 1);
    const float4 d2 = __ldg(reinterpret_cast<const float4*>(D) + 2);
    const float4 d3 = __ldg(reinterpret_cast<const float4*>(D) + 3);
    // D = [dR00 dR01 dR02 dR10 | dR11 dR12 dR20 dR21 | dR22 dt0 dt1 dt2 | M T 0 0]
    const float vx = fmaf(d0.x, px, fmaf(d0.y, py, fmaf(d0.z, pz, d2.y)));
    const float vy = fmaf(d0.w, px, fmaf(d1.x, py, fmaf(d1.y, pz, d2.z)));
    const float vz = fmaf(d1.z, px, fmaf(d1.w, py, fmaf(d2.x, pz, d2.w)));
    const float p1 = fabsf(px) + fabsf(py) + fabsf(pz);
    const float nv = sqrtf(fmaf(vx, vx, fmaf(vy, vy, vz * vz)));
    return fmaf(nv, 1.0f + 0x1p-20f, fmaf(0x1p-19f, fmaf(d3.x, p1, d3.y), 0x1p-30f * (p1 + 1.0f)));
}

// K_sel writes, per packet of 32 consecutive source points, the mask of the points that need
// a full search; K_nn then runs its packets in source order with only those lanes active, so
// an uncertified remainder stays spatially coherent (a compacted list would scatter it).
#ifndef CIL_SEL_THREADS
#define CIL_SEL_THREADS 128     // (6 CTAs per SM; 256: C4 run +2.7 %, 64: +2.4 %, 384: +4 %)
#endif
constexpr int kSelThreads = CIL_SEL_THREADS;
#ifndef CIL_SEL_PREFETCH
#define CIL_SEL_PREFETCH 1     // a queued record's candidate list prefetched at classification (C4 run -0.4 %)
#endif
#ifndef CIL_SEL_ROUNDS
#define CIL_SEL_ROUNDS 4
#endif
constexpr int kSelRounds = CIL_SEL_ROUNDS;
constexpr int kSelTile = kSelThreads * kSelRounds;     // 1024 queries per CTA
#ifndef CIL_SEL_PERSIST
#define CIL_SEL_PERSIST 1
#endif

// Certificates of query i at the current pose, one query per lane, the
// whole warp together: returns true if the lane's query needs a full search; otherwise its
// exact nearest neighbour is known after this call (nn[i]):
//   point certificate G_pt > 2 D_p: the match j1 itself is unchanged (no evaluation at all);
//     G_pt is re-measured whenever the leaf / list is evaluated (anchor = that iteration);
//   leaf certificate  G1 > 2 D : the NN is in the search anchor's leaf L1 (one leaf evaluated);
//   list certificate  G_S > 2 D: the NN is in the stored candidate-leaf list (a Verlet list
//                                with skin g: every other target was beyond r_S = d1 + G_S);
//   nothing within rho, G1 = rho - max_corr_dist > D: still nothing within max_corr_dist.
// Evaluations are flattened over the warp into rounds of 32 independent (query, leaf) items
// (shared-memory atomicMin on u64 keys), so a warp keeps 32 leaf loads in flight.
struct SelWarp {
    float q[6][32];                          // -s_hi, -s_lo per lane
    unsigned long long best[32];
    unsigned sec[32];                        // point-level 2nd best (float bits)
    int items[32 * kListLeaves];
    uint32_t rec[32 * kSelRounds];           // queued evaluations: index | leaf-certificate flag
    float outer[32 * kSelRounds];            // their outer bounds
    int npc;                                 // point-certified queries (diagnostics)
    int nleaf, nlist, nitems;                // evaluations by kind (diagnostics)
};

// leaf item for K_sel: best key and the point-level second best (the loser of every merge and
// the within-leaf second minimum)
template <int B>
__device__ __forceinline__ void sel_leaf_item(const TargetView& T, const NegQuery& q, int leaf,
                                              unsigned long long* bestS, unsigned* secS) {
    float d2[B];
    leaf_d2<B>(T, q, leaf, d2);
    float m1 = d2[0], m2 = INFINITY;
#pragma unroll
    for (int c = 1; c < B; ++c) { m2 = fminf(m2, fmaxf(m1, d2[c])); m1 = fminf(m1, d2[c]); }
    float push = m1;
    if (m1 <= key_d2(*(volatile unsigned long long*)bestS)) {
        const unsigned long long k = make_key(m1, leaf_argmin<B>(T, leaf, d2, m1));
        const unsigned long long old = atomicMin(bestS, k);
        push = old == k ? INFINITY : key_d2(old > k ? old : k);
    }
    const unsigned v = __float_as_uint(fminf(push, m2));
    if (v < *(volatile unsigned*)secS) atomicMin(secS, v);
}

// Phase 1 (per round of 32 points, one per lane): classify.  Points that need their leaf / list
// evaluated are queued as records (index | leaf-certificate flag, outer bound) in the warp's
// buffer, so that phase 2 evaluates them packed 32 per step instead of idling the lanes of
// every round in which one point needs an evaluation.
struct SelIn {                               // per-point state, loaded up front for every round
    uint32_t w, wp;
    int j;
    float gs, gd1, px, py, pz;
};

__device__ __forceinline__ SelIn sel_load(const IterArgs& a, int i) {
    SelIn v;
    if (i < a.m) {
        v.w = a.gw[i]; v.wp = a.gp[i]; v.j = a.nn[i]; v.gs = a.gs[i]; v.gd1 = a.gd1[i];
        v.px = a.src[3 * (size_t)i]; v.py = a.src[3 * (size_t)i + 1]; v.pz = a.src[3 * (size_t)i + 2];
    } else {
        v.w = 0; v.wp = 0; v.j = -1; v.gs = 0.0f; v.gd1 = 0.0f; v.px = v.py = v.pz = 0.0f;
    }
    return v;
}

template <int B>
__device__ __forceinline__ bool classify(const IterArgs& a, int i, const SelIn& in, uint32_t kslot, SelWarp& S,
                                         int& nrec) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    bool need = false, eval = false;
    uint32_t rec = 0;
    float outer = 0.0f;                      // lower bound of |s' - t| for every t outside the evaluated leaves
    if (i < a.m) {
        const uint32_t w = in.w, wp = in.wp;
        const float px = in.px, py = in.py, pz = in.pz;
        // slot == kslot: never anchored (iteration 0) or an anchor pose being recycled (k >= 256)
        if ((w & 255u) == kslot) {
            need = true;
        } else {
            const float D = displacement_bound(a.adelta + 16 * (w & 255u), px, py, pz);
            const float G1 = __uint_as_float(w & ~255u);
            const int j = in.j;
            if (j < 0) {
                need = !(G1 > D);
            } else {
                const bool leaf_ok = G1 > 2.0f * D;
                const float GS = leaf_ok ? 0.0f : in.gs;
                const float Gp = __uint_as_float(wp & ~255u);
                if (!leaf_ok && !(GS > 2.0f * D)) {
                    need = true;
                } else if (a.point_cert && (wp & 255u) != kslot && Gp > 0.0f &&
                           Gp > 2.0f * displacement_bound(a.adelta + 16 * (wp & 255u), px, py, pz)) {
                    // point certificate (only where the leaf / list certificate holds too, so it
                    // never postpones a search): nn[i] stays, nothing to evaluate
                    atomicAdd(&S.npc, 1);
                } else {
                    eval = true;
                    rec = (uint32_t)i | (leaf_ok ? 0x80000000u : 0u);
#if CIL_SEL_PREFETCH
                    // its candidate-leaf list is read by the evaluation step: start the fetch now
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(a.vlist + (size_t)kListLeaves * i));
#endif
                    // targets outside the evaluated leaves were >= d_out (resp. r_S) from the anchor
                    outer = (leaf_ok ? G1 : GS) + in.gd1 - D;
                }
            }
        }
    }
    const unsigned mk = __ballot_sync(FULL, eval);
    if (eval) {
        const int pos = nrec + __popc(mk & ((1u << lane) - 1u));
        S.rec[pos] = rec;
        S.outer[pos] = outer;
    }
    nrec += __popc(mk);
    return need;
}

// Phase 2: the queued records, 32 per step: L1 (entry 0) of every record -- usually the winner
// -- then the rest of the lists, flattened into rounds of 32 (query, leaf) items, each evaluated
// only if the leaf box can still beat the query's current best (else its bound joins the 2nd
// best); writes nn[i] and the re-measured point certificate.
template <int B>
__device__ __forceinline__ void evaluate_records(const IterArgs& a, const Pose34& P, uint32_t kslot, SelWarp& S,
                                                 int nrec) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    for (int c0 = 0; c0 < nrec; c0 += 32) {
        const bool on = c0 + lane < nrec;
        int i = 0, nit = 0;
        float outer = 0.0f;
        constexpr int NQ = kListLeaves / 4;
        int4 lv[NQ];
#pragma unroll
        for (int c = 0; c < NQ; ++c) lv[c] = make_int4(-1, -1, -1, -1);
        if (on) {
            const uint32_t rec = S.rec[c0 + lane];
            outer = S.outer[c0 + lane];
            i = (int)(rec & 0x7fffffffu);
            const bool leaf_ok = (rec >> 31) != 0;
            const int4* vl = reinterpret_cast<const int4*>(a.vlist + (size_t)kListLeaves * i);
            lv[0] = vl[0];
            if (!leaf_ok)
#pragma unroll
                for (int c = 1; c < NQ; ++c) lv[c] = vl[c];
            nit = 0;
#pragma unroll
            for (int c = 0; c < NQ; ++c) nit += (lv[c].x >= 0) + (lv[c].y >= 0) + (lv[c].z >= 0) + (lv[c].w >= 0);
            if (leaf_ok) nit = 1;
            const DF3 s = transform_df(P, a.src[3 * (size_t)i], a.src[3 * (size_t)i + 1], a.src[3 * (size_t)i + 2]);
            S.q[0][lane] = -s.hx; S.q[1][lane] = -s.hy; S.q[2][lane] = -s.hz;
            S.q[3][lane] = -s.lx; S.q[4][lane] = -s.ly; S.q[5][lane] = -s.lz;
            S.best[lane] = bound_key(INFINITY);
            S.sec[lane] = __float_as_uint(INFINITY);
            NegQuery nq0;
            nq0.hx = make_float2(-s.hx, -s.hx); nq0.hy = make_float2(-s.hy, -s.hy); nq0.hz = make_float2(-s.hz, -s.hz);
            nq0.lx = make_float2(-s.lx, -s.lx); nq0.ly = make_float2(-s.ly, -s.ly); nq0.lz = make_float2(-s.lz, -s.lz);
            sel_leaf_item<B>(a.T, nq0, lv[0].x, &S.best[lane], &S.sec[lane]);
        }
        const int rest = nit > 1 ? nit - 1 : 0;
        {
            const unsigned lf = __ballot_sync(FULL, on && nit == 1 && (S.rec[c0 + lane] >> 31) != 0);
            const unsigned ls = __ballot_sync(FULL, on) & ~lf;
            if (lane == 0) { S.nleaf += __popc(lf); S.nlist += __popc(ls); }
        }
        int incl = rest;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += v;
        }
        const int total = __shfl_sync(FULL, incl, 31);
        if (lane == 0) S.nitems += total;
        if (total > 0) {
            const int excl = incl - rest;
            int Ls[kListLeaves];
#pragma unroll
            for (int c = 0; c < NQ; ++c) {
                Ls[4 * c] = lv[c].x; Ls[4 * c + 1] = lv[c].y; Ls[4 * c + 2] = lv[c].z; Ls[4 * c + 3] = lv[c].w;
            }
#pragma unroll
            for (int c = 1; c < kListLeaves; ++c)
                if (c <= rest) S.items[excl + c - 1] = (Ls[c] << 5) | lane;
            __syncwarp();
            for (int r0 = 0; r0 < total; r0 += 32) {
                const int k = r0 + lane;
                if (k < total) {
                    const int it = S.items[k];
                    const int q = it & 31;
                    NegQuery qq;
                    qq.hx = make_float2(S.q[0][q], S.q[0][q]);
                    qq.hy = make_float2(S.q[1][q], S.q[1][q]);
                    qq.hz = make_float2(S.q[2][q], S.q[2][q]);
                    qq.lx = make_float2(S.q[3][q], S.q[3][q]);
                    qq.ly = make_float2(S.q[4][q], S.q[4][q]);
                    qq.lz = make_float2(S.q[5][q], S.q[5][q]);
                    const float lb = leaf_lb2(a.T, qq, it >> 5);
                    if (lb <= key_d2(*(volatile unsigned long long*)&S.best[q])) sel_leaf_item<B>(a.T, qq, it >> 5, &S.best[q], &S.sec[q]);
                    else atomicMin(&S.sec[q], __float_as_uint(lb));
                }
            }
        }
        __syncwarp();
        if (on) {
            const unsigned long long b = S.best[lane];
            const int jn = (int)key_idx(b);
            if (jn != a.nn[i]) a.nn[i] = jn;
            // point certificate measured here: every other target is at >= min(2nd best, outer)
            const float o2 = fminf(sqrtf(__uint_as_float(S.sec[lane])), outer);
            const float Gp = fmaxf(o2 * (1.0f - 4e-6f) - sqrtf(key_d2(b)) * (1.0f + 4e-6f), 0.0f);
            a.gp[i] = (__float_as_uint(Gp) & ~255u) | kslot;
        }
        __syncwarp();
    }
}

#if CIL_SEL_PERSIST
#ifndef CIL_SEL_MINB
#define CIL_SEL_MINB (768 / kSelThreads)
#endif
#define CIL_SEL_BOUNDS __launch_bounds__(kSelThreads, CIL_SEL_MINB)
#else
#define CIL_SEL_BOUNDS __launch_bounds__(kSelThreads)
#endif
template <int B>
__global__ void CIL_SEL_BOUNDS
icp_select_kernel(const IterArgs a) {
    __shared__ SelWarp s_w[kSelThreads / 32];
    __shared__ double s_pose[12];
    __shared__ int s_cnt, s_np, s_base;
#if !CIL_SEL_PERSIST
    __shared__ int s_tile;
#endif
    __shared__ int s_pk[kSelTile / 32];
    pdl_trigger();
    pdl_wait();
    if (*(volatile int*)&a.st->done) return;
    stamp(a, 0, true);
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t kslot = (uint32_t)(*(volatile int*)&a.st->iters) & (kAnchorSlots - 1);
    if (threadIdx.x < 12) s_pose[threadIdx.x] = a.st->pose[threadIdx.x];
    __syncthreads();
    Pose34 P;
#pragma unroll
    for (int e = 0; e < 12; ++e) P.r[e] = s_pose[e];
#if CIL_SEL_PERSIST
    // persistent: tiles of 1024 points claimed from a counter (no wave quantisation)
    __shared__ int s_tile;
    const int ntiles = (a.m + kSelTile - 1) / kSelTile;
    for (;;) {
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(&a.st->sel_work, 1u);
#else
    {
    if (threadIdx.x == 0) s_tile = blockIdx.x;
#endif
    if (threadIdx.x == 0) { s_cnt = 0; s_np = 0; }
    if ((threadIdx.x & 31) == 0) {
        SelWarp& S0 = s_w[threadIdx.x >> 5];
        S0.npc = 0; S0.nleaf = 0; S0.nlist = 0; S0.nitems = 0;
    }
    __syncthreads();
    const int tile = s_tile;
#if CIL_SEL_PERSIST
    if (tile >= ntiles) break;
#endif
    const int wbase = tile * kSelTile + warp * (32 * kSelRounds);
    int cnt = 0, nrec = 0;
    SelIn in[kSelRounds];                    // every round's loads in flight together
#pragma unroll
    for (int r = 0; r < kSelRounds; ++r) in[r] = sel_load(a, wbase + 32 * r + lane);
#pragma unroll
    for (int r = 0; r < kSelRounds; ++r) {
        const int i0 = wbase + 32 * r;
        if (i0 >= a.m) break;
        const unsigned mk = __ballot_sync(FULL, classify<B>(a, i0 + lane, in[r], kslot, s_w[warp], nrec));
        if (lane == 0) {
            a.pmask[i0 >> 5] = mk;
            if (mk) s_pk[atomicAdd(&s_np, 1)] = i0 >> 5;
        }
        cnt += __popc(mk);
    }
    __syncwarp();
    evaluate_records<B>(a, P, kslot, s_w[warp], nrec);
    if (lane == 0 && cnt) atomicAdd(&s_cnt, cnt);
    __syncthreads();
    // packets that need a search go to the list (one global atomic per CTA; any order: a
    // packet is a self-contained, spatially coherent unit)
    if (threadIdx.x == 0) {
        s_base = s_np ? atomicAdd(&a.st->plist_n, s_np) : 0;
        if (s_cnt) atomicAdd(&a.st->list_n, s_cnt);                    // diagnostics: searched points
        int npc = 0, nlf = 0, nls = 0, nit = 0;
        for (int w = 0; w < kSelThreads / 32; ++w) {
            npc += s_w[w].npc; nlf += s_w[w].nleaf; nls += s_w[w].nlist; nit += s_w[w].nitems;
        }
        if (npc) atomicAdd(reinterpret_cast<unsigned long long*>(&a.st->pcert_n), (unsigned long long)npc);
        if (nlf) atomicAdd(reinterpret_cast<unsigned long long*>(&a.st->rec_leaf), (unsigned long long)nlf);
        if (nls) atomicAdd(reinterpret_cast<unsigned long long*>(&a.st->rec_list), (unsigned long long)nls);
        if (nit) atomicAdd(reinterpret_cast<unsigned long long*>(&a.st->rec_items), (unsigned long long)nit);
    }
    __syncthreads();
    if (threadIdx.x < s_np) a.plist[s_base + threadIdx.x] = s_pk[threadIdx.x];
    __syncthreads();
    }
}

// ---------------------------------------------------------------- K_nn
constexpr int kNNThreads = 32 * kEngineWarps;

template <int B, bool CERT>
struct IcpQueries {
    const float* src;
    const float4* opts;
    Pose34 P;
    float search2;
    float gap_none;
    float gap_min, gap_max;  // CERT: the skin g of a point = clamp(kappa x its last-step displacement)
    float kappa;
    const float* prev_delta; // anchor-table entry of the previous iteration (pose_k - pose_{k-1}) or nullptr
    mutable float skin;      // out of load(): this query's skin
    float stale2;            // a warm hint farther than this (d^2) is complemented by the cold hint
    int* nn;
    uint32_t* gw;
    float* gs;
    float* gd1;
    uint32_t* gp;
    int* vlist;
    const uint32_t* pmask;
    const int* plist;        // CERT: packets with a non-empty mask, count at *plist_n
    const int* plist_n;
    int warm;
    uint32_t slot;
    int32_t* corr_idx;
    float* corr_d2;
    const uint32_t* perm;
    __device__ __forceinline__ int packets(int m) const { return plist ? *(volatile const int*)plist_n : (m + 31) / 32; }
    __device__ __forceinline__ int tag() const { return (int)slot; }
    __device__ __forceinline__ int packet_base(int c) const { return 32 * (plist ? plist[c] : c); }
    __device__ __forceinline__ bool load(int i, DF3& s, unsigned long long& init, int& hint) const {
        if (pmask && !((pmask[i >> 5] >> (i & 31)) & 1u)) return false;    // certified in K_sel
        const float px = src[3 * (size_t)i], py = src[3 * (size_t)i + 1], pz = src[3 * (size_t)i + 2];
        s = transform_df(P, px, py, pz);
        init = bound_key(search2);
        if (CERT) {
            // per-point skin: a multiple of the point's own displacement in the last iteration
            // (the certificate then tends to hold for the next several, geometrically shrinking steps)
            // (a point moving faster than 4 gap_max / kappa per iteration would not keep a
            // certificate anyway: it searches with the minimal skin, the cheapest search)
            float sk = gap_min;
            if (prev_delta) {
                const float want = kappa * displacement_bound(prev_delta, px, py, pz);
                sk = want <= kSkinCut * gap_max ? fminf(fmaxf(want, gap_min), gap_max) : gap_min;
            }
            skin = sk;
        }
        const int j = warm ? nn[i] : -1;
        hint = j >= 0 ? __float_as_int(__ldg(&opts[j].w)) / B : -1;
        return true;
    }
    __device__ __forceinline__ void store(int i, unsigned long long best, float) const {
        const bool found = best != bound_key(search2);
        nn[i] = found ? (int)key_idx(best) : -1;
        const size_t o = perm[i];                      // outputs in the caller's source order
        if (corr_idx) corr_idx[o] = found ? (int32_t)key_idx(best) : -1;
        if (corr_d2) corr_d2[o] = found ? key_d2(best) : INFINITY;
    }
    // CERT: the certificates of the new anchor (this iteration's pose).  G1 = d_out - d1 (leaf
    // form), G_S = r_S - d1 (candidate-leaf list); 4e-6 relative slack covers the fp32 d^2
    // error; G1 is rounded toward zero by clearing the low 8 bits (they hold the anchor slot).
    __device__ __forceinline__ void store(int i, unsigned long long best, float lb_out2, const int* lst, int cnt,
                                          float rS2) const {
        const bool found = best != bound_key(search2);
        nn[i] = found ? (int)key_idx(best) : -1;
        float G1 = gap_none, GS = 0.0f;
        if (found) {
            const float d1 = sqrtf(key_d2(best)) * (1.0f + 4e-6f);
            G1 = fmaxf(sqrtf(lb_out2) * (1.0f - 4e-6f) - d1, 0.0f);
            GS = cnt > 0 ? fmaxf(sqrtf(rS2) * (1.0f - 4e-6f) - d1, 0.0f) : 0.0f;
        }
        gw[i] = (__float_as_uint(G1) & ~255u) | slot;
        gs[i] = GS;
        gd1[i] = found ? sqrtf(key_d2(best)) * (1.0f + 4e-6f) : 0.0f;
        gp[i] = slot;                        // no point certificate yet (G_pt = 0)
        // entry 0 = L1, the anchor match's leaf (the leaf certificate refers to it even after a
        // list-certified iteration moved the match to another leaf), then the rest of the list
        const int L1 = found ? __float_as_int(__ldg(&opts[key_idx(best)].w)) / B : -1;
        int e[kListLeaves];
        e[0] = L1;
        int n = 1;
        bool has_L1 = false;
#pragma unroll
        for (int c = 0; c < kListLeaves; ++c) {
            const int v = c < cnt ? lst[c] : -1;
            has_L1 |= v == L1;
            if (v >= 0 && v != L1 && n < kListLeaves) e[n++] = v;
        }
#pragma unroll
        for (int c = 1; c < kListLeaves; ++c) if (c >= n) e[c] = -1;
        // no list, or L1 missing from a full list (an entry would be lost): no list certificate
        if (cnt == 0 || (!has_L1 && cnt == kListLeaves)) GS = 0.0f;
        int4* dst = reinterpret_cast<int4*>(vlist + (size_t)kListLeaves * i);
#pragma unroll
        for (int c = 0; c < kListLeaves / 4; ++c) dst[c] = make_int4(e[4 * c], e[4 * c + 1], e[4 * c + 2], e[4 * c + 3]);
    }
};

template <int B, bool CERT>
#ifndef CIL_NN_MINB
#define CIL_NN_MINB 4
#endif
__global__ void __launch_bounds__(kNNThreads, CIL_NN_MINB)
icp_nn_kernel(const IterArgs a) {
    pdl_trigger();
    pdl_wait();
    if (a.run && *(volatile int*)&a.st->done) return;
    stamp(a, 1, true);
    IcpQueries<B, CERT> qs;
    qs.src = a.src;
    qs.opts = a.T.opts;
#pragma unroll
    for (int k = 0; k < 12; ++k) qs.P.r[k] = __ldg(a.pose_in + k);
    qs.search2 = a.search2;
    qs.gap_none = a.gap_none;
    qs.gap_min = a.gap_min;
    qs.gap_max = a.gap_max;
    qs.kappa = a.kappa;
    {
        const int k = a.run ? *(volatile int*)&a.st->iters : 0;
        qs.prev_delta = (a.cert && k > 0) ? a.adelta + 16 * ((k - 1) & (kAnchorSlots - 1)) : nullptr;
    }
    qs.skin = 0.0f;
    qs.stale2 = a.stale2;
    qs.nn = a.nn;
    qs.gw = a.gw;
    qs.gs = a.gs;
    qs.gd1 = a.gd1;
    qs.gp = a.gp;
    qs.vlist = a.vlist;
    qs.pmask = a.cert ? a.pmask : nullptr;
    qs.plist = a.cert ? a.plist : nullptr;
    qs.plist_n = &a.st->plist_n;
    qs.warm = a.run;
    qs.slot = (uint32_t)(*(volatile int*)&a.st->iters) & (kAnchorSlots - 1);
    qs.corr_idx = a.corr_idx;
    qs.corr_d2 = a.corr_d2;
    qs.perm = a.perm;
    nn_packet_engine<B, CERT>(a.T, qs, a.m, &a.st->work);
}

// K_nn on the grid index (CIL_INDEX_GRID, stateless cil_icp_iterate only): one source point
// per thread, a1 transform (double-float) + exact grid search bounded by max_corr_dist
template <int B>
__global__ void __launch_bounds__(kNNThreads)
icp_grid_nn_kernel(const IterArgs a) {
    pdl_trigger();
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.m) return;
    Pose34 P;
#pragma unroll
    for (int k = 0; k < 12; ++k) P.r[k] = __ldg(a.pose_in + k);
    const DF3 s = transform_df(P, a.src[3 * (size_t)i], a.src[3 * (size_t)i + 1], a.src[3 * (size_t)i + 2]);
    const unsigned long long none = bound_key(a.search2);
    const unsigned long long best = grid_search<B, true>(a.T, s, none);
    const bool found = best != none;
    a.nn[i] = found ? (int)key_idx(best) : -1;
    const size_t o = a.perm[i];
    if (a.corr_idx) a.corr_idx[o] = found ? (int32_t)key_idx(best) : -1;
    if (a.corr_d2) a.corr_d2[o] = found ? key_d2(best) : INFINITY;
}

// a1 + a3 + a4 + a5 for the pair (p, t): transform, inclusive rejection (R2), residual,
// Jacobian, fp32 per-thread sums (29 point-to-plane / 17 point-to-point values)
// (accumulate_s: the same for an already transformed s; returns whether the pair was accepted
// and its d^2 in *d2)
template <int METRIC>
__device__ __forceinline__ bool accumulate_s(float (&acc)[kSlots], const DF3& s, float4 t, float4 n, float bound2,
                                             float wpp, float wpl, float* d2) {
    const float dx = dfdiff(s.hx, s.lx, t.x);
    const float dy = dfdiff(s.hy, s.ly, t.y);
    const float dz = dfdiff(s.hz, s.lz, t.z);
    *d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    if (!(*d2 <= bound2)) return false;
    if (METRIC == CIL_COMBINED) {
        // w_pl J_pl J_pl^T + w_pp J_pp^T J_pp per pair, J_pp = [-[s]x, I3] (R22): the
        // point-to-point blocks are |s|^2 I - s s^T, [s]x, I written out per pair (no
        // cross-pair cancellation), in the 21 + 6 + sse + count layout of point-to-plane
        const float sx = s.hx, sy = s.hy, sz = s.hz;
        const float r = fmaf(dx, n.x, fmaf(dy, n.y, dz * n.z));
        const float J[6] = {fmaf(sy, n.z, -sz * n.y), fmaf(sz, n.x, -sx * n.z), fmaf(sx, n.y, -sy * n.x),
                            n.x, n.y, n.z};
        // H_pp upper triangle, row-major over (0..5) x (p..5)
        const float Hp[21] = {fmaf(sy, sy, sz * sz), -sx * sy, -sx * sz, 0.0f, -sz, sy,
                              fmaf(sx, sx, sz * sz), -sy * sz, sz, 0.0f, -sx,
                              fmaf(sx, sx, sy * sy), -sy, sx, 0.0f,
                              1.0f, 0.0f, 0.0f,
                              1.0f, 0.0f,
                              1.0f};
        // g_pp = [s x r_pp; r_pp], r_pp = s - t
        const float gp[6] = {fmaf(sy, dz, -sz * dy), fmaf(sz, dx, -sx * dz), fmaf(sx, dy, -sy * dx), dx, dy, dz};
        int k = 0;
#pragma unroll
        for (int p = 0; p < 6; ++p)
#pragma unroll
            for (int q = p; q < 6; ++q, ++k) acc[k] = fmaf(wpl * J[p], J[q], fmaf(wpp, Hp[k], acc[k]));
#pragma unroll
        for (int p = 0; p < 6; ++p) acc[21 + p] = fmaf(wpl * J[p], r, fmaf(wpp, gp[p], acc[21 + p]));
        acc[27] = fmaf(wpl * r, r, fmaf(wpp, fmaf(dx, dx, fmaf(dy, dy, dz * dz)), acc[27]));
        acc[28] += 1.0f;
    } else if (METRIC == CIL_POINT_TO_PLANE) {
        const float r = fmaf(dx, n.x, fmaf(dy, n.y, dz * n.z));
        const float J[6] = {fmaf(s.hy, n.z, -s.hz * n.y), fmaf(s.hz, n.x, -s.hx * n.z),
                            fmaf(s.hx, n.y, -s.hy * n.x), n.x, n.y, n.z};
        int k = 0;
#pragma unroll
        for (int p = 0; p < 6; ++p)
#pragma unroll
            for (int q = p; q < 6; ++q, ++k) acc[k] = fmaf(J[p], J[q], acc[k]);
#pragma unroll
        for (int p = 0; p < 6; ++p) acc[21 + p] = fmaf(J[p], r, acc[21 + p]);
        acc[27] = fmaf(r, r, acc[27]);
        acc[28] += 1.0f;
    } else {
        const float sx = s.hx, sy = s.hy, sz = s.hz;
        acc[0] += 1.0f;
        acc[1] += sx; acc[2] += sy; acc[3] += sz;
        acc[4] = fmaf(sx, sx, acc[4]); acc[5] = fmaf(sy, sy, acc[5]); acc[6] = fmaf(sz, sz, acc[6]);
        acc[7] = fmaf(sx, sy, acc[7]); acc[8] = fmaf(sx, sz, acc[8]); acc[9] = fmaf(sy, sz, acc[9]);
        acc[10] += dx; acc[11] += dy; acc[12] += dz;
        acc[13] += fmaf(sy, dz, -sz * dy);
        acc[14] += fmaf(sz, dx, -sx * dz);
        acc[15] += fmaf(sx, dy, -sy * dx);
        acc[16] = fmaf(dx, dx, fmaf(dy, dy, fmaf(dz, dz, acc[16])));
    }
    return true;
}

template <int METRIC>
__device__ __forceinline__ void accumulate_pair(float (&acc)[kSlots], const Pose34& P, float px, float py, float pz,
                                                float4 t, float4 n, float bound2, float wpp, float wpl) {
    float d2;
    (void)accumulate_s<METRIC>(acc, transform_df(P, px, py, pz), t, n, bound2, wpp, wpl, &d2);
}

// Per-CTA partial of the 32 fp32 per-thread sums: warp transpose-reduce (fp32) -> per-warp fp64
// -> fixed-order sum over the warps -> partials[slot * kMaxCtas + blockIdx.x] (slot-major)
template <int NW = kIcpWarps>
__device__ __forceinline__ void cta_partial(float (&acc)[kSlots], double (*wsum)[kSlots], double* partials) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float mine = warp_transpose_reduce(acc);
    wsum[warp][lane] = (double)mine;
    __syncthreads();
    if (threadIdx.x < kSlots) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) v += wsum[w][threadIdx.x];
        partials[(size_t)threadIdx.x * kMaxCtas + blockIdx.x] = v;
        __threadfence();
    }
}

// Fixed-order fp64 sum of G slot-major per-CTA partials into Ssum (all threads of the CTA):
// warp w sums slots w, w+8, w+16, w+24: lane l takes CTAs l, l+32, ... (coalesced rows,
// sixteen loads in flight), then a fixed xor-butterfly; lane 0's value is the sum (the order is
// a fixed function of G: bitwise reproducible, and identical in every CTA that runs it).
__device__ __forceinline__ void sum_partials(const double* partials, int G, double* Ssum) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp >= 8) return;                        // (CTAs of more than 8 warps: the first 8 sum)
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int b0 = 0; b0 < G; b0 += 4 * 32) {
        double xv[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int b = b0 + 32 * u + lane;
                xv[q][u] = b < G ? __ldcg(partials + (size_t)(warp + 8 * q) * kMaxCtas + b) : 0.0;
            }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int u = 0; u < 4; ++u) v[q] += xv[q][u];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], off);
        if (lane == 0) Ssum[warp + 8 * q] = v[q];
    }
}

template <int METRIC, bool WARP = false>
__device__ __forceinline__ void solve_tail(const IterArgs& a, const double* Ssum, const double* Psh);

// ---------------------------------------------------------------- a5 reduction + a6 + a7
// Epilogue of the accumulation kernels: warp transpose-reduce (fp32) -> per-warp fp64 ->
// per-CTA partial; the last CTA (ticket) sums the partials in fixed order, solves, updates
// the pose and (certified run) writes the anchor table of the next iteration.
template <int METRIC, bool WARP = false, int NW = kIcpWarps>
__device__ __forceinline__ void reduce_finalize(const IterArgs& a, float (&acc)[kSlots], const double* Psh) {
    __shared__ double wsum[NW][kSlots];
    __shared__ double Ssum[kSlots];
    __shared__ int last;
    // ---- reductions (a5): warp transpose-reduce (fp32) -> per-warp fp64 -> per-CTA partial
    cta_partial<NW>(acc, wsum, a.partials);
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&a.st->ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    stamp(a, 3, false);

    // ---- last CTA: fixed-order fp64 reduction of the per-CTA partials, solve, update.
    // Warp w sums slots w, w+8, w+16, w+24: lane l takes CTAs l, l+32, ... (coalesced rows of
    // the slot-major partials, sixteen loads in flight), then a fixed xor-butterfly; lane 0's
    // value is the sum (the order is a fixed function of the grid size: bitwise reproducible).
    __threadfence();
    sum_partials(a.partials, (int)gridDim.x, Ssum);
    __syncthreads();
    if (a.sums_out) {                                       // shard mode: the caller all-reduces
        if (threadIdx.x < kSlots) a.sums_out[threadIdx.x] = Ssum[threadIdx.x];
        if (threadIdx.x == 0) {
            a.st->ticket = 0;
            a.st->work = 0;
            a.st->sel_work = 0;
            a.st->searched += a.run ? a.st->list_n : 0;
            a.st->list_n = 0;
            a.st->plist_n = 0;
        }
        return;
    }
    solve_tail<METRIC, WARP>(a, Ssum, Psh);
}

// a6 + a7 and the next iteration's anchor table, from the reduced sums Ssum (shared) and the
// pose the iteration ran at (Psh); all threads of the CTA.
template <int METRIC, bool WARP>
__device__ __forceinline__ void solve_tail(const IterArgs& a, const double* Ssum, const double* Psh) {
    const int it = a.run ? a.st->iters : 0;                 // index of this iteration
    if (a.cert && threadIdx.x < 12) a.apose[12 * (it & (kAnchorSlots - 1)) + threadIdx.x] = Psh[threadIdx.x];
    __syncthreads();
    const int it_stamp = a.run ? a.st->iters : 0;
    if (a.stamps && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.stamps[8 * it_stamp + 5] = t;
    }
    if (WARP) {
        if (threadIdx.x < 32) finalize_warp<METRIC>(fin_args(a), Ssum, Psh);
    } else if (threadIdx.x == 0) {
        finalize<METRIC>(fin_args(a), Ssum, Psh);
    }
    if (threadIdx.x == 0) {
        if (a.stamps) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.stamps[8 * it_stamp + 4] = t;
        }
        a.st->ticket = 0;
        a.st->work = 0;      // K_nn's counter, for the next iteration
        a.st->sel_work = 0;  // K_sel's tile counter
        a.st->searched += a.run ? a.st->list_n : 0;
        a.st->list_n = 0;
        a.st->plist_n = 0;
    }
    __syncthreads();
    // anchor table for the next iteration's K_sel: delta of every live slot to the new pose
    if (a.cert && !a.st->done) {
        const int a_slot = threadIdx.x;
        if (a_slot < kAnchorSlots && a_slot <= it) {
            const double* Pa = a.apose + 12 * a_slot;
            const volatile double* Pn = a.st->pose;
            float* D = a.adelta + 16 * a_slot;
            double M = 0.0, Tm = 0.0;
            const int rot[9] = {0, 1, 2, 4, 5, 6, 8, 9, 10};
            for (int e = 0; e < 9; ++e) {
                const double d = Pn[rot[e]] - Pa[rot[e]];
                D[e] = (float)d;
                M = fmax(M, fabs(d));
            }
            for (int e = 0; e < 3; ++e) {
                const double d = Pn[4 * e + 3] - Pa[4 * e + 3];
                D[9 + e] = (float)d;
                Tm = fmax(Tm, fabs(d));
            }
            D[12] = __double2float_ru(M);
            D[13] = __double2float_ru(Tm);
            D[14] = 0.0f;
            D[15] = 0.0f;
        }
    }
}

// ---------------------------------------------------------------- K_acc (+ a6, a7)
#ifndef CIL_ACC_PREFETCH
#define CIL_ACC_PREFETCH 2     // next trip's matches / source (1), and its gathers (2) prefetched
#endif
#ifndef CIL_ACC_MINB
#define CIL_ACC_MINB 2
#endif
template <int METRIC>
__global__ void __launch_bounds__(kIcpThreads, CIL_ACC_MINB)
icp_acc_kernel(const IterArgs a) {
    __shared__ double Psh[16];
    pdl_trigger();
    pdl_wait();
    if (a.run && *(volatile int*)&a.st->done) return;
    stamp(a, 2, true);

    if (threadIdx.x < 16) Psh[threadIdx.x] = a.pose_in[threadIdx.x];
    __syncthreads();
    Pose34 P;
#pragma unroll
    for (int k = 0; k < 12; ++k) P.r[k] = Psh[k];

    float acc[kSlots];
#pragma unroll
    for (int k = 0; k < kSlots; ++k) acc[k] = 0.0f;

    const TargetView& T = a.T;
    // four queries per trip with every load issued before the arithmetic (the gathers depend on
    // nn[]; four independent chains in flight per thread); summation order = grid-stride order
    constexpr int U = 4;
    const int stride = gridDim.x * blockDim.x;
#if CIL_ACC_PREFETCH >= 2
    int jn[U];                                   // the matches of the next trip (one trip ahead)
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int iu = blockIdx.x * blockDim.x + threadIdx.x + u * stride;
        jn[u] = iu < a.m ? a.nn[iu] : -1;
    }
#endif
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.m; i += U * stride) {
        int jj[U];
        float4 tt[U], nn4[U];
        float px[U], py[U], pz[U];
#if CIL_ACC_PREFETCH >= 2
#pragma unroll
        for (int u = 0; u < U; ++u) {
            jj[u] = jn[u];
            const int iu = i + (U + u) * stride;
            jn[u] = iu < a.m ? a.nn[iu] : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int iu = i + (2 * U + u) * stride;
            if (iu < a.m) asm volatile("prefetch.global.L1 [%0];" ::"l"(a.nn + iu));
        }
#else
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int iu = i + u * stride;
            jj[u] = iu < a.m ? a.nn[iu] : -1;
        }
#endif
#if CIL_ACC_PREFETCH
        // the next trip's matches and source points: their fetch overlaps this trip's gathers
        // (prefetch, no registers held)
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int iu = i + (U + u) * stride;
            if (iu < a.m) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a.nn + iu));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a.src + 3 * (size_t)iu));
            }
        }
#endif
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int iu = i + u * stride;
            tt[u] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            nn4[u] = tt[u];
            px[u] = py[u] = pz[u] = 0.0f;
            if (jj[u] >= 0) {
                tt[u] = __ldg(T.opts + jj[u]);
                if (METRIC != CIL_POINT_TO_POINT) nn4[u] = __ldg(T.onrm + jj[u]);
                px[u] = a.src[3 * (size_t)iu]; py[u] = a.src[3 * (size_t)iu + 1]; pz[u] = a.src[3 * (size_t)iu + 2];
            }
        }
#if CIL_ACC_PREFETCH >= 2
#pragma unroll
        for (int u = 0; u < U; ++u)                                    // the next trip's gathers
            if (jn[u] >= 0) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(T.opts + jn[u]));
                if (METRIC != CIL_POINT_TO_POINT) asm volatile("prefetch.global.L1 [%0];" ::"l"(T.onrm + jn[u]));
            }
#endif
#pragma unroll
        for (int u = 0; u < U; ++u)                                    // a3: nn < 0 = nothing within the bound
            if (jj[u] >= 0) accumulate_pair<METRIC>(acc, P, px[u], py[u], pz[u], tt[u], nn4[u], a.bound2, a.w_pp, a.w_pl);
    }

    reduce_finalize<METRIC, CIL_KD_WARP_SOLVE>(a, acc, Psh);
}

// ---------------------------------------------------------------- K_proj
// Projective data association (R23-R25): the pixel the
// transformed source point projects to in the organised target IS its correspondence, so
// a2 is O(1) per point and the whole iteration is one streaming kernel:
//   a1  s = R p + t (fp64), a2' (u, v) = round(((f s) / s_z) + c) in fp64, half away from zero
//   (CUDA round()), bounds, pixel validity (z > 0, finite), a3-a5 as K_acc on the
//   double-float s, then the shared epilogue (fixed-order reduction, solve, pose update).
// Source order = the caller's (an organised source projects coherently: neighbouring lanes
// gather neighbouring pixels).
__device__ __forceinline__ int project_pixel(const IterArgs& a, double x, double y, double z) {
    if (!(z > 0.0)) return -1;
    const double uf = __dadd_rn(__ddiv_rn(__dmul_rn(a.pfx, x), z), a.pcx);
    const double vf = __dadd_rn(__ddiv_rn(__dmul_rn(a.pfy, y), z), a.pcy);
    const double ur = round(uf), vr = round(vf);
    if (!(ur >= 0.0 && ur < (double)a.pw && vr >= 0.0 && vr < (double)a.ph)) return -1;
    return (int)vr * a.pw + (int)ur;
}

// the streaming body of the projective iteration: a1, a2', a3-a5 for this thread's points
// (grid-stride, four per trip); corr outputs when requested (iterate)
template <int METRIC>
__device__ __forceinline__ void proj_accumulate(const IterArgs& a, const Pose34& P, float (&acc)[kSlots]) {
    constexpr int U = 4;     // four points per trip, every load issued before the arithmetic
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.m; i += U * stride) {
        float px[U], py[U], pz[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int iu = i + u * stride;
            px[u] = py[u] = pz[u] = 0.0f;
            if (iu < a.m) {
                px[u] = __ldg(a.src + 3 * (size_t)iu);
                py[u] = __ldg(a.src + 3 * (size_t)iu + 1);
                pz[u] = __ldg(a.src + 3 * (size_t)iu + 2);
            }
        }
        double sx[U], sy[U], sz[U];
        int kk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            sx[u] = fma(P.r[0], (double)px[u], fma(P.r[1], (double)py[u], fma(P.r[2], (double)pz[u], P.r[3])));
            sy[u] = fma(P.r[4], (double)px[u], fma(P.r[5], (double)py[u], fma(P.r[6], (double)pz[u], P.r[7])));
            sz[u] = fma(P.r[8], (double)px[u], fma(P.r[9], (double)py[u], fma(P.r[10], (double)pz[u], P.r[11])));
            kk[u] = i + u * stride < a.m ? project_pixel(a, sx[u], sy[u], sz[u]) : -1;
        }
        float4 tt[U], nn4[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            tt[u] = make_float4(0.0f, 0.0f, -1.0f, 0.0f);
            nn4[u] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            if (kk[u] >= 0) {
                const float* t = a.ptgt + 3 * (size_t)kk[u];
                tt[u] = make_float4(__ldg(t), __ldg(t + 1), __ldg(t + 2), 0.0f);
                if (METRIC != CIL_POINT_TO_POINT) {
                    const float* n = a.pnrm + 3 * (size_t)kk[u];
                    nn4[u] = make_float4(__ldg(n), __ldg(n + 1), __ldg(n + 2), 0.0f);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int iu = i + u * stride;
            const float4 t = tt[u];
            const bool valid = kk[u] >= 0 && t.z > 0.0f && isfinite(t.x) && isfinite(t.y) && isfinite(t.z);
            float d2 = INFINITY;
            bool ok = false;
            if (valid) ok = accumulate_s<METRIC>(acc, split_df(sx[u], sy[u], sz[u]), t, nn4[u], a.bound2, a.w_pp,
                                                 a.w_pl, &d2);
            if (iu < a.m) {
                if (a.corr_idx) a.corr_idx[iu] = ok ? kk[u] : -1;
                if (a.corr_d2) a.corr_d2[iu] = ok ? d2 : INFINITY;
            }
        }
    }
}

template <int METRIC>
__global__ void __launch_bounds__(kIcpThreads, 2)
icp_proj_kernel(const IterArgs a) {
    __shared__ double Psh[16];
    pdl_trigger();
    pdl_wait();
    if (a.run && *(volatile int*)&a.st->done) return;
    stamp(a, 2, true);
    if (threadIdx.x < 16) Psh[threadIdx.x] = a.pose_in[threadIdx.x];
    __syncthreads();
    Pose34 P;
#pragma unroll
    for (int k = 0; k < 12; ++k) P.r[k] = Psh[k];
    float acc[kSlots];
#pragma unroll
    for (int k = 0; k < kSlots; ++k) acc[k] = 0.0f;

    proj_accumulate<METRIC>(a, P, acc);
    reduce_finalize<METRIC, true>(a, acc, Psh);
}

// Grid-wide barrier of a cooperatively launched grid (every CTA co-resident): arrival counter +
// generation word in the workspace state.
__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            atomicExch(count, 0u);
            __threadfence();
            atomicAdd(const_cast<unsigned*>(gen), 1u);
        } else {
            while (*gen == g) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

// The whole projective loop in one persistent launch (cil_proj_run): per iteration every CTA
// streams its points, writes its partial (double-buffered by iteration parity), meets the
// others at one grid barrier, then EVERY CTA sums all partials in the same fixed order and
// solves redundantly -- identical inputs, identical code, so every CTA holds the bitwise same
// new pose (and the loop equals the chain of cil_proj_iterate launches bit for bit: same grid,
// same point assignment, same reduction order).  CTA 0 writes the run state.  No launch gap,
// no last-CTA hand-off; the solve runs from a warm instruction cache on every SM.
template <int METRIC>
__global__ void __launch_bounds__(kIcpThreads, 2)
icp_proj_run_kernel(const IterArgs a, int iters) {
    __shared__ double Psh[16];
    __shared__ double wsum[kIcpWarps][kSlots];
    __shared__ double Ssum[kSlots];
    __shared__ double Hs[36], gsh[6], scal[2];
    __shared__ int s_stop;
    if (threadIdx.x < 16) Psh[threadIdx.x] = a.st->pose[threadIdx.x];
    __syncthreads();
    auto tick = [&](int it, int k) {
        if (a.stamps && blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.stamps[8 * it + k] = t;
        }
    };
    for (int it = 0; it < iters; ++it) {
        tick(it, 0);
        Pose34 P;
#pragma unroll
        for (int k = 0; k < 12; ++k) P.r[k] = Psh[k];
        float acc[kSlots];
#pragma unroll
        for (int k = 0; k < kSlots; ++k) acc[k] = 0.0f;
        proj_accumulate<METRIC>(a, P, acc);
        double* part = a.partials + (size_t)(it & 1) * kSlots * kMaxCtas;
        cta_partial(acc, wsum, part);
        tick(it, 1);
        grid_barrier(&a.st->bar_count, &a.st->bar_gen);
        tick(it, 2);
        sum_partials(part, (int)gridDim.x, Ssum);
        __syncthreads();
        tick(it, 3);
        if (threadIdx.x < 32) {
            double x[6], Pn[16];
            const int status = solve_pose_warp<METRIC>(Ssum, Psh, Hs, gsh, scal, x, Pn);
            __syncwarp();
            if (threadIdx.x == 0) {
                const double sse = scal[0], cnt = scal[1];
                bool stop = status != CIL_OK;
                bool conv = false;
                if (!stop) {
                    const double th = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
                    const double tn = sqrt(x[3] * x[3] + x[4] * x[4] + x[5] * x[5]);
                    conv = th < a.rot_tol && tn < a.trans_tol;
                    stop = conv;
                }
                if (blockIdx.x == 0) {
                    IcpState* st = a.st;
                    const double rmse = cnt > 0.0 ? sqrt(sse / cnt) : 0.0;
                    if (a.iter_log) { a.iter_log[2 * it] = cnt; a.iter_log[2 * it + 1] = rmse; }
                    st->iters = it + 1;
                    st->n_corr = (long long)cnt;
                    st->rmse = rmse;
                    if (status != CIL_OK) {
                        st->status = status;
                        st->converged = 0;
                        st->done = 1;
                    } else {
                        for (int i = 0; i < 16; ++i) st->pose[i] = Pn[i];
                        if (conv) { st->converged = 1; st->done = 1; }
                    }
                }
                if (status == CIL_OK)
                    for (int i = 0; i < 16; ++i) Psh[i] = Pn[i];
                s_stop = stop;
            }
        }
        __syncthreads();
        tick(it, 4);
        if (s_stop) break;
    }
}

// ---------------------------------------------------------------- small problems (brute force)
// A target of at most kSmallMaxN points fits in shared memory, and for m * n <= kSmallMaxPairs
// the exact 1-NN by brute force (every target, u64 key minimum: R1 ties) costs a few
// microseconds spread over the whole GPU, while a tree search of a few thousand queries is
// bound by the latency of one warp's traversal (C1: ~25 us per iteration).  Each query is
// taken by a group of G lanes (G = a power of two chosen so that m * G fills the grid); lane k
// of the group scans targets k, k + G, ...; the group reduces its keys by shuffles and the
// group leader accumulates the pair (a3-a5), so the iteration is ONE launch (iterate) or the
// whole loop is one cooperative persistent launch (run: grid barrier, every CTA sums the
// partials in the same fixed order and solves redundantly, as the projective loop does; the
// same grid, assignment and reduction as the iterate kernel, so run == chained iterates bit for
// bit).  The source is used in the caller's order (no Morton sort needed).
constexpr int kSmallMaxN = 8192;                   // 96 KB of SoA targets in shared memory
constexpr long long kSmallMaxPairs = 1ll << 26;
constexpr int kSmallThreads = 512;                 // one CTA of 16 warps per SM

// padded length of the staged SoA rows: a multiple of 4 candidates per lane step x 32 lanes
__host__ __device__ __forceinline__ int small_npad(int n) { return (n + 127) & ~127; }

// the target in ORIGINAL order as SoA rows x[np], y[np], z[np] (position = original index);
// padding is NaN (its d^2 compares false: never a candidate, even for an unbounded search)
__device__ __forceinline__ void small_stage(const IterArgs& a, float* sT) {
    const int n = a.T.n, np = small_npad(n);
    for (int k = threadIdx.x; k < np; k += blockDim.x) {
        float4 p = k < n ? __ldg(a.T.opts + k) : make_float4(NAN, NAN, NAN, 0.0f);
        sT[k] = p.x;
        sT[np + k] = p.y;
        sT[2 * np + k] = p.z;
    }
    __syncthreads();
}

// nn + a3-a5 of this CTA's queries into acc (group leaders only); corr outputs when requested.
// Lane k of a query's group of G lanes evaluates the candidate quads k, k + G, ... with packed
// FP32 (two candidates per FADD2/FFMA2; -dx = (t + (-s_hi)) + (-s_lo), the same d^2 bits as
// cand_d2) and keeps the u64 key minimum; the group then reduces its keys by shuffles.
template <int METRIC>
__device__ __forceinline__ void small_pass(const IterArgs& a, const float* sT, const Pose34& P, int glog,
                                          float (&acc)[kSlots]) {
    const int n = a.T.n, np = small_npad(n), nq = np >> 2;
    const int G = 1 << glog;
    const int sub = threadIdx.x & (G - 1);
    const int qpb = kSmallThreads >> glog;
    const unsigned FULL = 0xffffffffu;
    const unsigned long long none = bound_key(a.bound2);
    const float4* X = reinterpret_cast<const float4*>(sT);
    const float4* Y = reinterpret_cast<const float4*>(sT + np);
    const float4* Z = reinterpret_cast<const float4*>(sT + 2 * np);
    // every lane of a warp runs the same number of rounds (the shuffles need the whole group)
    const int rounds = (a.m + qpb * (int)gridDim.x - 1) / (qpb * (int)gridDim.x);
    for (int rd = 0; rd < rounds; ++rd) {
        const int q = (rd * (int)gridDim.x + (int)blockIdx.x) * qpb + ((int)threadIdx.x >> glog);
        const bool on = q < a.m;
        DF3 s;
        unsigned long long best = none;
        if (on) {
            s = transform_df(P, a.src[3 * (size_t)q], a.src[3 * (size_t)q + 1], a.src[3 * (size_t)q + 2]);
            const NegQuery nq2 = neg_query(s);
            float bd = key_d2(best);
#pragma unroll 2
            for (int k = sub; k < nq; k += G) {
                const float4 x = X[k], y = Y[k], z = Z[k];
                const float2 d01 = pair_d2(nq2, make_float2(x.x, x.y), make_float2(y.x, y.y), make_float2(z.x, z.y));
                const float2 d23 = pair_d2(nq2, make_float2(x.z, x.w), make_float2(y.z, y.w), make_float2(z.z, z.w));
                if (fminf(fminf(d01.x, d01.y), fminf(d23.x, d23.y)) <= bd) {   // rare after the first few
                    const float dd[4] = {d01.x, d01.y, d23.x, d23.y};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const unsigned long long kk = make_key(dd[c], (uint32_t)(4 * k + c));
                        if (dd[c] <= bd && kk < best) { best = kk; bd = dd[c]; }
                    }
                }
            }
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            if (o >= G) break;
            const unsigned long long ot = __shfl_xor_sync(FULL, best, o);
            best = ot < best ? ot : best;
        }
        if (on && sub == 0) {
            const bool found = best != none;
            const int j = found ? (int)key_idx(best) : -1;
            if (a.corr_idx) a.corr_idx[q] = j;
            if (a.corr_d2) a.corr_d2[q] = found ? key_d2(best) : INFINITY;
            if (found) {
                const float4 t = make_float4(sT[j], sT[np + j], sT[2 * np + j], 0.0f);
                const float4 nrm = METRIC != CIL_POINT_TO_POINT ? __ldg(a.T.onrm + j) : make_float4(0.f, 0.f, 0.f, 0.f);
                float d2;
                (void)accumulate_s<METRIC>(acc, s, t, nrm, a.bound2, a.w_pp, a.w_pl, &d2);
            }
        }
    }
}

template <int METRIC>
__global__ void __launch_bounds__(kSmallThreads, 1)
icp_small_kernel(const IterArgs a, int glog) {
    extern __shared__ float sT[];
    __shared__ double Psh[16];
    pdl_trigger();
    pdl_wait();
    if (a.run && *(volatile int*)&a.st->done) return;
    if (threadIdx.x < 16) Psh[threadIdx.x] = a.pose_in[threadIdx.x];
    small_stage(a, sT);
    Pose34 P;
#pragma unroll
    for (int k = 0; k < 12; ++k) P.r[k] = Psh[k];
    float acc[kSlots];
#pragma unroll
    for (int k = 0; k < kSlots; ++k) acc[k] = 0.0f;
    small_pass<METRIC>(a, sT, P, glog, acc);
    reduce_finalize<METRIC, true, kSmallThreads / 32>(a, acc, Psh);
}

template <int METRIC>
__global__ void __launch_bounds__(kSmallThreads, 1)
icp_small_run_kernel(const IterArgs a, int glog, int iters) {
    extern __shared__ float sT[];
    __shared__ double Psh[16];
    __shared__ double wsum[kSmallThreads / 32][kSlots];
    __shared__ double Ssum[kSlots];
    __shared__ double Hs[36], gsh[6], scal[2];
    __shared__ int s_stop;
    if (threadIdx.x < 16) Psh[threadIdx.x] = a.st->pose[threadIdx.x];
    small_stage(a, sT);
    const int G = (int)gridDim.x;
    for (int it = 0; it < iters; ++it) {
        Pose34 P;
#pragma unroll
        for (int k = 0; k < 12; ++k) P.r[k] = Psh[k];
        float acc[kSlots];
#pragma unroll
        for (int k = 0; k < kSlots; ++k) acc[k] = 0.0f;
        small_pass<METRIC>(a, sT, P, glog, acc);
        double* part = a.partials + (size_t)(it & 1) * G;      // double-buffered columns
        cta_partial<kSmallThreads / 32>(acc, wsum, part);
        grid_barrier(&a.st->bar_count, &a.st->bar_gen);
        sum_partials(part, G, Ssum);
        __syncthreads();
        if (threadIdx.x < 32) {
            double x[6], Pn[16];
            const int status = solve_pose_warp<METRIC>(Ssum, Psh, Hs, gsh, scal, x, Pn);
            __syncwarp();
            if (threadIdx.x == 0) {
                const double sse = scal[0], cnt = scal[1];
                bool stop = status != CIL_OK;
                bool conv = false;
                if (!stop) {
                    const double th = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
                    const double tn = sqrt(x[3] * x[3] + x[4] * x[4] + x[5] * x[5]);
                    conv = th < a.rot_tol && tn < a.trans_tol;
                    stop = conv;
                }
                if (blockIdx.x == 0) {
                    IcpState* st = a.st;
                    const double rmse = cnt > 0.0 ? sqrt(sse / cnt) : 0.0;
                    if (a.iter_log) { a.iter_log[2 * it] = cnt; a.iter_log[2 * it + 1] = rmse; }
                    st->iters = it + 1;
                    st->n_corr = (long long)cnt;
                    st->rmse = rmse;
                    st->searched += a.m;
                    if (status != CIL_OK) {
                        st->status = status;
                        st->converged = 0;
                        st->done = 1;
                    } else {
                        for (int i = 0; i < 16; ++i) st->pose[i] = Pn[i];
                        if (conv) { st->converged = 1; st->done = 1; }
                    }
                }
                if (status == CIL_OK)
                    for (int i = 0; i < 16; ++i) Psh[i] = Pn[i];
                s_stop = stop;
            }
        }
        __syncthreads();
        if (s_stop) break;
    }
}

// ---------------------------------------------------------------- run bookkeeping kernels
__global__ void run_init_kernel(IcpState* st, const double* pose_init, int* nn, uint32_t* gw, uint32_t* gp, int m,
                                double* iter_log, int log_len) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    if (tid == 0) {
        for (int i = 0; i < 16; ++i) st->pose[i] = pose_init[i];
        st->rmse = 0.0; st->n_corr = 0; st->iters = 0; st->converged = 0; st->status = CIL_OK;
        st->done = 0; st->ticket = 0; st->work = 0; st->list_n = 0; st->searched = 0; st->plist_n = 0;
        st->sel_work = 0;
        st->pcert_n = 0; st->rec_leaf = 0; st->rec_list = 0; st->rec_items = 0;
        st->bar_count = 0; st->bar_gen = 0;
    }
    for (int i = tid; i < m; i += gridDim.x * blockDim.x) { nn[i] = -1; gw[i] = 0u; gp[i] = 0u; }
    if (iter_log)
        for (int i = tid; i < log_len; i += gridDim.x * blockDim.x) iter_log[i] = 0.0;
}

__global__ void run_final_kernel(const IcpState* st, cil_icp_result* res) {
    if (threadIdx.x != 0) return;
    for (int i = 0; i < 16; ++i) res->pose[i] = st->pose[i];
    res->rmse = st->rmse;
    res->n_corr = st->n_corr;
    res->iterations = st->iters;
    res->converged = st->converged;
    res->status = st->status;
    res->pad = 0;
}

// shard mode: a6 + a7 from the all-reduced sums, on every rank
template <int METRIC>
__global__ void __launch_bounds__(kIcpThreads)
icp_shard_finish_kernel(const IterArgs a, const double* __restrict__ sums) {
    __shared__ double Psh[16];
    __shared__ double Ssum[kSlots];
    pdl_trigger();
    pdl_wait();
    if (*(volatile int*)&a.st->done) return;
    if (threadIdx.x < 16) Psh[threadIdx.x] = a.st->pose[threadIdx.x];
    if (threadIdx.x < kSlots) Ssum[threadIdx.x] = sums[threadIdx.x];
    __syncthreads();
    solve_tail<METRIC, CIL_KD_WARP_SOLVE>(a, Ssum, Psh);
}

__global__ void reset_ticket_kernel(IcpState* st) { st->ticket = 0; st->work = 0; st->list_n = 0; st->sel_work = 0; }

// preferred shared-memory carveouts in percent (-1: the driver's default)
#ifndef CIL_CARVE_SEL
#define CIL_CARVE_SEL 40
#endif
#ifndef CIL_CARVE_NN
#define CIL_CARVE_NN -1
#endif
#ifndef CIL_CARVE_ACC
#define CIL_CARVE_ACC 0
#endif
template <class K>
void set_carve(K kernel, int pct) {
    if (pct >= 0) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

template <class K>
int occupancy_of(K kernel, int threads) {
    int occ = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, 0) != cudaSuccess) occ = 1;
    return std::max(occ, 1);
}

inline int persistent_grid(int occ, int threads, int m, int cap_ctas) {
    const int64_t want = ((int64_t)m + threads - 1) / threads;
    const int64_t cap = std::min<int64_t>((int64_t)sm_count() * occ, cap_ctas);
    return (int)std::max<int64_t>(1, std::min(want, cap));
}

template <int B, bool CERT>
cudaError_t launch_nn_b(const IterArgs& a, cudaStream_t s) {
    // (the carveout is set before the occupancy is queried)
    static const int occ = (set_carve(icp_nn_kernel<B, CERT>, CIL_CARVE_NN), occupancy_of(icp_nn_kernel<B, CERT>, kNNThreads));
    const int g = persistent_grid(occ, kNNThreads, a.m, 1 << 20);
    prof_begin(kProfNN, s);
    IterArgs ad = a;
    ad.T.trace = debug_trace();
    ad.T.dbg_mode = (int)(debug_flags() >> 1) & 3;
    cudaError_t e = launch_pdl(icp_nn_kernel<B, CERT>, g, kNNThreads, s, ad);
    prof_end(s);
    return e;
}

template <int B>
cudaError_t launch_grid_nn_b(const IterArgs& a, cudaStream_t s) {
    prof_begin(kProfNN, s);
    cudaError_t e = launch_pdl(icp_grid_nn_kernel<B>, std::max(1, (a.m + kNNThreads - 1) / kNNThreads), kNNThreads, s, a);
    prof_end(s);
    return e;
}

template <bool CERT>
cudaError_t launch_nn_t(const IterArgs& a, cudaStream_t s) {
    if (!CERT && !a.run && a.T.gpts) {             // stateless iterate on the grid index
        switch (a.T.leaf_size) {
            case 4: return launch_grid_nn_b<4>(a, s);
            case 8: return launch_grid_nn_b<8>(a, s);
            case 16: return launch_grid_nn_b<16>(a, s);
            default: return launch_grid_nn_b<32>(a, s);
        }
    }
    switch (a.T.leaf_size) {
        case 4: return launch_nn_b<4, CERT>(a, s);
        case 8: return launch_nn_b<8, CERT>(a, s);
        case 16: return launch_nn_b<16, CERT>(a, s);
        default: return launch_nn_b<32, CERT>(a, s);
    }
}

template <int METRIC>
cudaError_t launch_acc_m(const IterArgs& a, cudaStream_t s) {
    static const int occ = (set_carve(icp_acc_kernel<METRIC>, CIL_CARVE_ACC), occupancy_of(icp_acc_kernel<METRIC>, kIcpThreads));
    const int g = persistent_grid(occ, kIcpThreads, a.m, kMaxCtas);
    prof_begin(kProfAcc, s);
    cudaError_t e = launch_pdl(icp_acc_kernel<METRIC>, g, kIcpThreads, s, a);
    prof_end(s);
    return e;
}

// one ICP iteration = [K_sel] + K_nn + K_acc
cudaError_t launch_iter(const IterArgs& a0, int metric, cudaStream_t s) {
    IterArgs a = a0;
    a.stamps = debug_stamps();
    cudaError_t e0 = cudaSuccess;
    int n = 2;
    if (a.cert) {
        const int g = std::max(1, (a.m + kSelTile - 1) / kSelTile);
        // persistent grid: the resident CTAs per SM of the instance launched.  The certificate
        // kernel's evaluations re-read leaves through L1, the accumulation's gathers too: both run
        // with the smallest shared-memory carveout that keeps their occupancy (measured: C4 run
        // 14.52 -> 14.34 ms)
        auto persist = [&](int occ) { return CIL_SEL_PERSIST ? std::min(g, occ * sm_count()) : g; };
        auto occ_of = [](auto kernel) { set_carve(kernel, CIL_CARVE_SEL); return occupancy_of(kernel, kSelThreads); };
        static const int occ4 = occ_of(icp_select_kernel<4>), occ8 = occ_of(icp_select_kernel<8>),
                         occ16 = occ_of(icp_select_kernel<16>), occ32 = occ_of(icp_select_kernel<32>);
        prof_begin(kProfSel, s);
        switch (a.T.leaf_size) {
            case 4: e0 = launch_pdl(icp_select_kernel<4>, persist(occ4), kSelThreads, s, a); break;
            case 8: e0 = launch_pdl(icp_select_kernel<8>, persist(occ8), kSelThreads, s, a); break;
            case 16: e0 = launch_pdl(icp_select_kernel<16>, persist(occ16), kSelThreads, s, a); break;
            default: e0 = launch_pdl(icp_select_kernel<32>, persist(occ32), kSelThreads, s, a); break;
        }
        prof_end(s);
        if (e0 != cudaSuccess) return e0;
        ++n;
    }
    count_launches(n);
    cudaError_t e = a.cert ? launch_nn_t<true>(a, s) : launch_nn_t<false>(a, s);
    if (e != cudaSuccess) return e;
    switch (metric) {
        case CIL_POINT_TO_PLANE: return launch_acc_m<CIL_POINT_TO_PLANE>(a, s);
        case CIL_COMBINED: return launch_acc_m<CIL_COMBINED>(a, s);
        default: return launch_acc_m<CIL_POINT_TO_POINT>(a, s);
    }
}

template <int METRIC>
cudaError_t launch_proj_m(const IterArgs& a, cudaStream_t s) {
    static const int occ = occupancy_of(icp_proj_kernel<METRIC>, kIcpThreads);
    const int g = persistent_grid(occ, kIcpThreads, (a.m + 3) / 4, kMaxCtas);
    prof_begin(kProfAcc, s);
    cudaError_t e = launch_pdl(icp_proj_kernel<METRIC>, g, kIcpThreads, s, a);
    prof_end(s);
    count_launches(1);
    return e;
}

template <int METRIC>
cudaError_t launch_proj_run_m(const IterArgs& a, int iters, cudaStream_t s) {
    static const int occ = occupancy_of(icp_proj_kernel<METRIC>, kIcpThreads);
    static const int occ_run = occupancy_of(icp_proj_run_kernel<METRIC>, kIcpThreads);
    const int g = persistent_grid(occ, kIcpThreads, (a.m + 3) / 4, kMaxCtas);    // the iterate grid
    if (g > occ_run * sm_count()) return cudaErrorCooperativeLaunchTooLarge;
    IterArgs ad = a;
    ad.stamps = debug_stamps();
    int it = iters;
    void* args[] = {(void*)&ad, (void*)&it};
    prof_begin(kProfAcc, s);
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)icp_proj_run_kernel<METRIC>, dim3(g), dim3(kIcpThreads),
                                                args, 0, s);
    prof_end(s);
    count_launches(1);
    return e;
}

cudaError_t launch_proj_run(const IterArgs& a, int metric, int iters, cudaStream_t s) {
    switch (metric) {
        case CIL_POINT_TO_PLANE: return launch_proj_run_m<CIL_POINT_TO_PLANE>(a, iters, s);
        case CIL_COMBINED: return launch_proj_run_m<CIL_COMBINED>(a, iters, s);
        default: return launch_proj_run_m<CIL_POINT_TO_POINT>(a, iters, s);
    }
}

cudaError_t launch_proj(const IterArgs& a0, int metric, cudaStream_t s) {
    IterArgs a = a0;
    a.stamps = debug_stamps();
    switch (metric) {
        case CIL_POINT_TO_PLANE: return launch_proj_m<CIL_POINT_TO_PLANE>(a, s);
        case CIL_COMBINED: return launch_proj_m<CIL_COMBINED>(a, s);
        default: return launch_proj_m<CIL_POINT_TO_POINT>(a, s);
    }
}

// ---------------------------------------------------------------- small-problem launches
bool small_path(const cil_target* t, int64_t m) {
    return !(debug_flags() & 64u) && m > 0 && t->v.n <= kSmallMaxN && (long long)m * t->v.n <= kSmallMaxPairs;
}

// lanes per query: the largest power of two <= 32 with m * G <= the grid's threads
int small_glog(int64_t m) {
    const int64_t threads = (int64_t)sm_count() * kSmallThreads;
    int g = 0;
    while (g < 5 && m * (int64_t)(2 << g) <= threads) ++g;
    return g;
}

template <class K>
cudaError_t small_attr(K kernel) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * small_npad(kSmallMaxN) * (int)sizeof(float));
}

template <int METRIC>
cudaError_t launch_small_m(const IterArgs& a0, bool run, int iters, cudaStream_t s) {
    static const cudaError_t e_attr = [] {
        cudaError_t e1 = small_attr(icp_small_kernel<METRIC>);
        cudaError_t e2 = small_attr(icp_small_run_kernel<METRIC>);
        return e1 != cudaSuccess ? e1 : e2;
    }();
    if (e_attr != cudaSuccess) return e_attr;
    IterArgs a = a0;
    a.stamps = nullptr;
    const int glog = small_glog(a.m);
    const int grid = sm_count();                  // one CTA per SM (the staged target fills shared memory)
    const size_t smem = 3 * (size_t)small_npad(a.T.n) * sizeof(float);
    prof_begin(kProfAcc, s);
    cudaError_t e = cudaSuccess;
    if (run) {
        int it = iters, gl = glog;
        void* args[] = {(void*)&a, (void*)&gl, (void*)&it};
        e = cudaLaunchCooperativeKernel((const void*)icp_small_run_kernel<METRIC>, dim3(grid), dim3(kSmallThreads), args,
                                        smem, s);
        count_launches(1);
        if (e != cudaSuccess) {
            // not co-schedulable: one launch per iteration (same grid and arithmetic)
            (void)cudaGetLastError();
            e = cudaSuccess;
            for (int k = 0; k < iters && e == cudaSuccess; ++k) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3((unsigned)grid);
                cfg.blockDim = dim3((unsigned)kSmallThreads);
                cfg.dynamicSmemBytes = smem;
                cfg.stream = s;
                e = cudaLaunchKernelEx(&cfg, icp_small_kernel<METRIC>, a, glog);
                count_launches(1);
            }
        }
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3((unsigned)kSmallThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, icp_small_kernel<METRIC>, a, glog);
        count_launches(1);
    }
    prof_end(s);
    return e;
}

cudaError_t launch_small(const IterArgs& a, int metric, bool run, int iters, cudaStream_t s) {
    switch (metric) {
        case CIL_POINT_TO_PLANE: return launch_small_m<CIL_POINT_TO_PLANE>(a, run, iters, s);
        case CIL_COMBINED: return launch_small_m<CIL_COMBINED>(a, run, iters, s);
        default: return launch_small_m<CIL_POINT_TO_POINT>(a, run, iters, s);
    }
}

struct WsLayout {
    size_t state, partials, apose, adelta, nn, gw, pmask, plist, gs, gd1, gp, vlist, perm, srcs, total;
};

WsLayout ws_layout(int64_t m) {
    const size_t mm = (size_t)std::max<int64_t>(m, 1);
    WsLayout L;
    L.state = 0;
    L.partials = 256;
    L.apose = L.partials + align_up((size_t)kMaxCtas * kSlots * sizeof(double), 256);
    L.adelta = L.apose + align_up((size_t)kAnchorSlots * 12 * sizeof(double), 256);
    L.nn = L.adelta + align_up((size_t)kAnchorSlots * 16 * sizeof(float), 256);
    L.gw = L.nn + align_up(mm * sizeof(int), 256);
    L.pmask = L.gw + align_up(mm * sizeof(uint32_t), 256);
    L.plist = L.pmask + align_up((mm + 31) / 32 * sizeof(uint32_t), 256);
    L.gs = L.plist + align_up((mm + 31) / 32 * sizeof(int), 256);
    L.gd1 = L.gs + align_up(mm * sizeof(float), 256);
    L.gp = L.gd1 + align_up(mm * sizeof(float), 256);
    L.vlist = L.gp + align_up(mm * sizeof(uint32_t), 256);
    L.perm = L.vlist + align_up(mm * kListLeaves * sizeof(int), 256);
    L.srcs = L.perm + align_up(mm * sizeof(uint32_t), 256);
    L.total = L.srcs + align_up(mm * 3 * sizeof(float), 256);
    return L;
}

void bind_ws(IterArgs& a, void* ws, int64_t m) {
    const WsLayout L = ws_layout(m);
    char* w = (char*)ws;
    a.st = (IcpState*)(w + L.state);
    a.partials = (double*)(w + L.partials);
    a.apose = (double*)(w + L.apose);
    a.adelta = (float*)(w + L.adelta);
    a.nn = (int*)(w + L.nn);
    a.gw = (uint32_t*)(w + L.gw);
    a.pmask = (uint32_t*)(w + L.pmask);
    a.plist = (int*)(w + L.plist);
    a.gs = (float*)(w + L.gs);
    a.gd1 = (float*)(w + L.gd1);
    a.gp = (uint32_t*)(w + L.gp);
    a.perm = (const uint32_t*)(w + L.perm);
    a.srcs = (float*)(w + L.srcs);
    a.vlist = (int*)(w + L.vlist);
}

__global__ void identity_perm_kernel(uint32_t* perm, int m) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) perm[k] = (uint32_t)k;
}

// The kernels visit the source in Morton order of its own frame (once per call; rigid motion
// keeps the order spatially coherent), so a 32-query packet is a compact neighbourhood even
// when the caller's order is not (C5's patch-major random samples).  a.src -> the sorted copy.
cudaError_t sort_source(IterArgs& a, const float* src, cudaStream_t s) {
    if (a.m == 0) { a.src = src; return cudaSuccess; }
    if (debug_flags() & 16u) { a.src = src; identity_perm_kernel<<<std::max(1, std::min((a.m + 255) / 256, 4096)), 256, 0, s>>>(const_cast<uint32_t*>(a.perm), a.m); return cudaGetLastError(); }
    int nl = 0;
    cudaError_t e = morton_order_points(src, a.m, const_cast<uint32_t*>(a.perm), a.srcs, s, &nl);
    count_launches(nl);
    a.src = a.srcs;
    return e;
}

cil_status check_params(const char* fn, const cil_icp_params* p) {
    if (!p) { set_error("%s: NULL params", fn); return CIL_ERR_INVALID_ARG; }
    if (p->metric != CIL_POINT_TO_POINT && p->metric != CIL_POINT_TO_PLANE && p->metric != CIL_COMBINED) {
        set_error("%s: metric %d not supported", fn, p->metric);
        return CIL_ERR_INVALID_ARG;
    }
    if (p->metric == CIL_COMBINED) {
        if (!(p->w_point >= 0.0) || !(p->w_plane >= 0.0) || !(p->w_point + p->w_plane > 0.0) ||
            !std::isfinite(p->w_point) || !std::isfinite(p->w_plane)) {
            set_error("%s: combined metric needs finite weights >= 0, not both 0", fn);
            return CIL_ERR_INVALID_ARG;
        }
    } else if (p->w_point != 0.0 || p->w_plane != 0.0) {
        set_error("%s: w_point/w_plane are only used by CIL_COMBINED (must be 0)", fn);
        return CIL_ERR_INVALID_ARG;
    }
    if (!(p->max_corr_dist > 0.0)) { set_error("%s: max_corr_dist must be > 0", fn); return CIL_ERR_INVALID_ARG; }
    if (!(p->rot_tol >= 0.0) || !(p->trans_tol >= 0.0)) { set_error("%s: tolerances must be >= 0", fn); return CIL_ERR_INVALID_ARG; }
    return CIL_OK;
}

cil_status check_common(const char* fn, const cil_target* t, const float* src, int64_t m, const cil_icp_params* p,
                        void* ws, size_t ws_bytes) {
    // parameters first (host-only, no target needed), then the target and buffers
    cil_status rc = check_params(fn, p);
    if (rc != CIL_OK) return rc;
    if (!t) { set_error("%s: NULL target", fn); return CIL_ERR_INVALID_ARG; }
    if (m < 0 || m > INT32_MAX) { set_error("%s: m=%lld out of range", fn, (long long)m); return CIL_ERR_INVALID_ARG; }
    if (m > 0 && !src) { set_error("%s: src is NULL", fn); return CIL_ERR_INVALID_ARG; }
    if ((p->metric == CIL_POINT_TO_PLANE || p->metric == CIL_COMBINED) && !t->has_normals) {
        set_error("%s: point-to-plane / combined need a target built with normals", fn);
        return CIL_ERR_NO_NORMALS;
    }
    if (!ws || ((uintptr_t)ws & 255u)) { set_error("%s: workspace NULL or not 256-B aligned", fn); return CIL_ERR_WORKSPACE; }
    if (ws_bytes < ws_layout(m).total) {
        set_error("%s: workspace %zu B < required %zu B", fn, ws_bytes, ws_layout(m).total);
        return CIL_ERR_WORKSPACE;
    }
    return CIL_OK;
}

size_t proj_ws_bytes() { return 256 + align_up(2 * (size_t)kMaxCtas * kSlots * sizeof(double), 256); }

cil_status check_proj(const char* fn, const float* tgt, const float* nrm, const cil_intrinsics* K, const float* src,
                      int64_t m, const cil_icp_params* p, void* ws, size_t ws_bytes) {
    cil_status rc = check_params(fn, p);
    if (rc != CIL_OK) return rc;
    if (!K) { set_error("%s: NULL intrinsics", fn); return CIL_ERR_INVALID_ARG; }
    if (K->width < 1 || K->height < 1 || (int64_t)K->width * K->height > INT32_MAX) {
        set_error("%s: image %d x %d out of range", fn, K->width, K->height);
        return CIL_ERR_INVALID_ARG;
    }
    if (!(K->fx > 0.0) || !(K->fy > 0.0) || !std::isfinite(K->fx) || !std::isfinite(K->fy) || !std::isfinite(K->cx) ||
        !std::isfinite(K->cy)) {
        set_error("%s: intrinsics need finite fx, fy > 0 and finite cx, cy", fn);
        return CIL_ERR_INVALID_ARG;
    }
    if (!tgt) { set_error("%s: NULL target", fn); return CIL_ERR_INVALID_ARG; }
    if (m < 0 || m > INT32_MAX) { set_error("%s: m=%lld out of range", fn, (long long)m); return CIL_ERR_INVALID_ARG; }
    if (m > 0 && !src) { set_error("%s: src is NULL", fn); return CIL_ERR_INVALID_ARG; }
    if ((p->metric == CIL_POINT_TO_PLANE || p->metric == CIL_COMBINED) && !nrm) {
        set_error("%s: point-to-plane / combined need target normals", fn);
        return CIL_ERR_NO_NORMALS;
    }
    if (!ws || ((uintptr_t)ws & 255u)) { set_error("%s: workspace NULL or not 256-B aligned", fn); return CIL_ERR_WORKSPACE; }
    if (ws_bytes < proj_ws_bytes()) {
        set_error("%s: workspace %zu B < required %zu B", fn, ws_bytes, proj_ws_bytes());
        return CIL_ERR_WORKSPACE;
    }
    return CIL_OK;
}

void bind_proj(IterArgs& a, const float* tgt, const float* nrm, const cil_intrinsics* K, const float* src, int64_t m,
               const cil_icp_params* p, void* ws) {
    a.st = (IcpState*)ws;
    a.partials = (double*)((char*)ws + 256);
    a.ptgt = tgt;
    a.pnrm = nrm;
    a.pw = K->width;
    a.ph = K->height;
    a.pfx = K->fx; a.pfy = K->fy; a.pcx = K->cx; a.pcy = K->cy;
    a.src = src;
    a.m = (int)m;
    a.w_pp = (float)p->w_point;
    a.w_pl = (float)p->w_plane;
    a.rot_tol = p->rot_tol;
    a.trans_tol = p->trans_tol;
}

float bound2_of(double max_dist) {
    return std::isinf(max_dist) ? INFINITY : (float)(max_dist * max_dist);
}

}  // namespace
}  // namespace cil

using namespace cil;

CIL_API size_t cil_icp_workspace_bytes(int64_t m, const cil_icp_params* params) {
    (void)params;
    if (m < 0 || m > INT32_MAX) return 0;
    return ws_layout(m).total;
}

CIL_API cil_status cil_icp_iterate(const cil_target* t, const float* src, int64_t m, const double* pose_in,
                                   const cil_icp_params* params, void* ws, size_t ws_bytes, double* pose_out,
                                   cil_icp_system* sys, int32_t* corr_idx, float* corr_sqdist, cil_stream_t stream) {
    cil_status rc = check_common("cil_icp_iterate", t, src, m, params, ws, ws_bytes);
    if (rc != CIL_OK) return rc;
    if (!pose_in || !pose_out) { set_error("cil_icp_iterate: pose_in/pose_out NULL"); return CIL_ERR_INVALID_ARG; }
    IterArgs a{};
    bind_ws(a, ws, m);
    a.T = t->v;
    a.src = src;
    a.m = (int)m;
    a.bound2 = bound2_of(params->max_corr_dist);
    a.search2 = a.bound2;
    a.w_pp = (float)params->w_point;
    a.w_pl = (float)params->w_plane;
    a.pose_in = pose_in;
    a.pose_out = pose_out;
    a.sys = sys;
    a.corr_idx = corr_idx;
    a.corr_d2 = corr_sqdist;
    a.run = 0;
    a.cert = 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (small_path(t, m)) {                       // brute force in one launch (caller's source order)
        reset_ticket_kernel<<<1, 1, 0, s>>>(a.st);
        count_launches(1);
        cudaError_t e = launch_small(a, params->metric, false, 1, s);
        if (e != cudaSuccess) return cuda_fail(e, "icp_small_kernel launch");
        return CIL_OK;
    }
    cudaError_t e = sort_source(a, src, s);
    if (e != cudaSuccess) return cuda_fail(e, "source Morton order");
    reset_ticket_kernel<<<1, 1, 0, s>>>(a.st);
    count_launches(1);
    e = launch_iter(a, params->metric, s);
    if (e != cudaSuccess) return cuda_fail(e, "icp_iter_kernel launch");
    return CIL_OK;
}

namespace cil {
namespace {
// IterArgs of the device-resident loop (cil_icp_run and the shard API)
void run_args(IterArgs& a, const cil_target* t, const float* src, int64_t m, const cil_icp_params* params, void* ws,
              double* iter_log) {
    a = IterArgs{};
    bind_ws(a, ws, m);
    a.T = t->v;
    a.src = src;
    a.m = (int)m;
    a.bound2 = bound2_of(params->max_corr_dist);
    a.w_pp = (float)params->w_point;
    a.w_pl = (float)params->w_plane;
    a.cert = (debug_flags() & 1u) ? 0 : 1;
    a.point_cert = (debug_flags() & 8u) ? 0 : 1;
    // certificates search to rho = 1.1 max_corr_dist so that a point with
    // nothing within rho stays provably rejected while it moves less than rho - max_corr_dist
    const double rho = std::isinf(params->max_corr_dist) ? INFINITY : CIL_RHO * params->max_corr_dist;
    a.search2 = a.cert ? bound2_of(rho) : a.bound2;
    {
        const double gn = (rho - params->max_corr_dist) * (1.0 - 1e-6);
        float g = std::isfinite(gn) ? (float)gn : 0.0f;
        if ((double)g > gn) g = std::nextafter(g, 0.0f);
        a.gap_none = g;
    }
    // leaf-certificate margin g: the search threshold of K_nn is (sqrt(best) + g)^2
    {
        double gmin = 0.0, gmax = 0.0, kap = 0.0;
        cert_skin_params(&gmin, &gmax, &kap);
        const double md = std::isinf(params->max_corr_dist) ? 0.0 : params->max_corr_dist;
        a.gap_min = (float)(gmin * md);
        a.gap_max = (float)(gmax * md);
        a.kappa = (float)kap;
    }
    a.stale2 = std::isinf(params->max_corr_dist) ? INFINITY : (float)(CIL_STALE * params->max_corr_dist * params->max_corr_dist);
    a.pose_in = a.st->pose;
    a.pose_out = a.st->pose;
    a.iter_log = iter_log;
    a.run = 1;
    a.rot_tol = params->rot_tol;
    a.trans_tol = params->trans_tol;
}

// sorted source + state initialisation of a run
cil_status run_begin(IterArgs& a, const float* src, int64_t m, const double* pose_init, int max_iters, cudaStream_t s,
                     bool ordered = false) {
    if (ordered) {
        // icp_order_source already filled the workspace's permutation / ordered copy (host.cu)
        a.src = (m == 0 || (debug_flags() & 16u)) ? src : a.srcs;
    } else {
        cudaError_t e0 = sort_source(a, src, s);
        if (e0 != cudaSuccess) return cuda_fail(e0, "source Morton order");
    }
    const int init_blocks = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)m + 255) / 256, (int64_t)sm_count() * 4));
    run_init_kernel<<<init_blocks, 256, 0, s>>>(a.st, pose_init, a.nn, a.gw, a.gp, (int)m, a.iter_log, 2 * max_iters);
    count_launches(1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "run_init_kernel launch");
    return CIL_OK;
}
}  // namespace
}  // namespace cil

namespace cil {
// host.cu: the source-order step of cil_icp_run on its own stream (it only depends on the source,
// so the host-buffer call runs it next to the target's copy and build), then the run with
// `ordered` set.  Same kernels, same workspace contents as cil_icp_run.
bool icp_small_path_nm(int64_t n, int64_t m) {
    return !(debug_flags() & 64u) && m > 0 && n <= kSmallMaxN && (long long)m * n <= kSmallMaxPairs;
}
cudaError_t icp_order_source(void* ws, const float* src, int64_t m, cudaStream_t s) {
    IterArgs a{};
    bind_ws(a, ws, m);
    a.m = (int)m;
    return sort_source(a, src, s);
}
}  // namespace cil

static cil_status icp_run_impl(const cil_target* t, const float* src, int64_t m, const double* pose_init,
                               const cil_icp_params* params, void* ws, size_t ws_bytes, cil_icp_result* res,
                               double* iter_log, cil_stream_t stream, bool ordered);

CIL_API cil_status cil_icp_run(const cil_target* t, const float* src, int64_t m, const double* pose_init,
                               const cil_icp_params* params, void* ws, size_t ws_bytes, cil_icp_result* res,
                               double* iter_log, cil_stream_t stream) {
    return icp_run_impl(t, src, m, pose_init, params, ws, ws_bytes, res, iter_log, stream, false);
}

namespace cil {
cil_status icp_run_ordered(const cil_target* t, const float* src, int64_t m, const double* pose_init,
                           const cil_icp_params* params, void* ws, size_t ws_bytes, cil_icp_result* res,
                           cil_stream_t stream) {
    return icp_run_impl(t, src, m, pose_init, params, ws, ws_bytes, res, nullptr, stream, true);
}
}  // namespace cil

static cil_status icp_run_impl(const cil_target* t, const float* src, int64_t m, const double* pose_init,
                               const cil_icp_params* params, void* ws, size_t ws_bytes, cil_icp_result* res,
                               double* iter_log, cil_stream_t stream, bool ordered) {
    cil_status rc = check_common("cil_icp_run", t, src, m, params, ws, ws_bytes);
    if (rc != CIL_OK) return rc;
    if (!pose_init || !res) { set_error("cil_icp_run: pose_init/res NULL"); return CIL_ERR_INVALID_ARG; }
    if (params->max_iters < 1) { set_error("cil_icp_run: max_iters must be >= 1"); return CIL_ERR_INVALID_ARG; }
    IterArgs a;
    run_args(a, t, src, m, params, ws, iter_log);
    cudaStream_t s = (cudaStream_t)stream;
    if (small_path(t, m)) {
        // the whole loop in one cooperative launch, brute-force correspondences (no certificates)
        a.cert = 0;
        a.src = src;
        run_init_kernel<<<1, 256, 0, s>>>(a.st, pose_init, nullptr, nullptr, nullptr, 0, iter_log, 2 * params->max_iters);
        count_launches(1);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = launch_small(a, params->metric, true, params->max_iters, s);
        if (e != cudaSuccess) return cuda_fail(e, "icp_small_run_kernel launch");
        run_final_kernel<<<1, 32, 0, s>>>(a.st, res);
        count_launches(1);
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "run_final_kernel launch");
        return CIL_OK;
    }
    rc = run_begin(a, src, m, pose_init, params->max_iters, s, ordered);
    if (rc != CIL_OK) return rc;
    for (int it = 0; it < params->max_iters; ++it) {
        cudaError_t e = launch_iter(a, params->metric, s);
        if (e != cudaSuccess) return cuda_fail(e, "icp_iter_kernel launch");
    }
    run_final_kernel<<<1, 32, 0, s>>>(a.st, res);
    count_launches(1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "run_final_kernel launch");
    return CIL_OK;
}

// ---------------------------------------------------------------- one problem across ranks
// The source is partitioned across ranks; every rank keeps its own workspace (warm-start state
// of its shard) and the same target.  Per iteration: cil_icp_shard_accumulate (K_sel + K_nn +
// K_acc on the shard, rank-local fp64 sums) -> the caller's all-reduce of the 32 sums ->
// cil_icp_shard_finish (solve + update + anchor table, redundantly and identically on every
// rank).  iter_log of cil_icp_shard_begin receives the global {n_corr, rmse} per iteration.
CIL_API cil_status cil_icp_shard_begin(const cil_target* t, const float* src, int64_t m, const double* pose_init,
                                       const cil_icp_params* params, void* ws, size_t ws_bytes, double* iter_log,
                                       cil_stream_t stream) {
    cil_status rc = check_common("cil_icp_shard_begin", t, src, m, params, ws, ws_bytes);
    if (rc != CIL_OK) return rc;
    if (!pose_init) { set_error("cil_icp_shard_begin: pose_init NULL"); return CIL_ERR_INVALID_ARG; }
    if (params->max_iters < 1) { set_error("cil_icp_shard_begin: max_iters must be >= 1"); return CIL_ERR_INVALID_ARG; }
    IterArgs a;
    run_args(a, t, src, m, params, ws, iter_log);
    return run_begin(a, src, m, pose_init, params->max_iters, (cudaStream_t)stream);
}

CIL_API cil_status cil_icp_shard_accumulate(const cil_target* t, const float* src, int64_t m,
                                            const cil_icp_params* params, void* ws, size_t ws_bytes, double* sums,
                                            cil_stream_t stream) {
    cil_status rc = check_common("cil_icp_shard_accumulate", t, src, m, params, ws, ws_bytes);
    if (rc != CIL_OK) return rc;
    if (!sums) { set_error("cil_icp_shard_accumulate: sums NULL"); return CIL_ERR_INVALID_ARG; }
    IterArgs a;
    run_args(a, t, src, m, params, ws, nullptr);
    a.src = (debug_flags() & 16u) ? src : a.srcs;            // the order cil_icp_shard_begin chose
    a.sums_out = sums;
    cudaError_t e = launch_iter(a, params->metric, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "icp shard iteration launch");
    return CIL_OK;
}

CIL_API cil_status cil_icp_shard_finish(const cil_target* t, int64_t m, const cil_icp_params* params, void* ws,
                                        size_t ws_bytes, const double* sums, double* iter_log, cil_stream_t stream) {
    cil_status rc = check_params("cil_icp_shard_finish", params);
    if (rc != CIL_OK) return rc;
    if (!t) { set_error("cil_icp_shard_finish: NULL target"); return CIL_ERR_INVALID_ARG; }
    if (m < 0 || m > INT32_MAX) { set_error("cil_icp_shard_finish: m out of range"); return CIL_ERR_INVALID_ARG; }
    if (!ws || ((uintptr_t)ws & 255u) || ws_bytes < ws_layout(m).total) {
        set_error("cil_icp_shard_finish: workspace NULL, unaligned or too small");
        return CIL_ERR_WORKSPACE;
    }
    if (!sums) { set_error("cil_icp_shard_finish: sums NULL"); return CIL_ERR_INVALID_ARG; }
    IterArgs a;
    run_args(a, t, nullptr, m, params, ws, iter_log);
    a.stamps = debug_stamps();
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e;
    switch (params->metric) {
        case CIL_POINT_TO_PLANE: e = launch_pdl(icp_shard_finish_kernel<CIL_POINT_TO_PLANE>, 1, kIcpThreads, s, a, sums); break;
        case CIL_COMBINED: e = launch_pdl(icp_shard_finish_kernel<CIL_COMBINED>, 1, kIcpThreads, s, a, sums); break;
        default: e = launch_pdl(icp_shard_finish_kernel<CIL_POINT_TO_POINT>, 1, kIcpThreads, s, a, sums); break;
    }
    count_launches(1);
    if (e != cudaSuccess) return cuda_fail(e, "icp_shard_finish_kernel launch");
    return CIL_OK;
}

CIL_API cil_status cil_icp_shard_result(void* ws, cil_icp_result* res, cil_stream_t stream) {
    if (!ws || ((uintptr_t)ws & 255u) || !res) { set_error("cil_icp_shard_result: NULL / unaligned argument"); return CIL_ERR_INVALID_ARG; }
    run_final_kernel<<<1, 32, 0, (cudaStream_t)stream>>>((const IcpState*)ws, res);
    count_launches(1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "run_final_kernel launch");
    return CIL_OK;
}

// ---------------------------------------------------------------- projective engine (NEXT-2)
CIL_API size_t cil_proj_workspace_bytes(int64_t m, const cil_icp_params* params) {
    (void)params;
    if (m < 0 || m > INT32_MAX) return 0;
    return proj_ws_bytes();
}

CIL_API cil_status cil_proj_iterate(const float* tgt, const float* tgt_normals, const cil_intrinsics* K, const float* src,
                                    int64_t m, const double* pose_in, const cil_icp_params* params, void* ws,
                                    size_t ws_bytes, double* pose_out, cil_icp_system* sys, int32_t* corr_idx,
                                    float* corr_sqdist, cil_stream_t stream) {
    cil_status rc = check_proj("cil_proj_iterate", tgt, tgt_normals, K, src, m, params, ws, ws_bytes);
    if (rc != CIL_OK) return rc;
    if (!pose_in || !pose_out) { set_error("cil_proj_iterate: pose_in/pose_out NULL"); return CIL_ERR_INVALID_ARG; }
    IterArgs a{};
    bind_proj(a, tgt, tgt_normals, K, src, m, params, ws);
    a.bound2 = bound2_of(params->max_corr_dist);
    a.pose_in = pose_in;
    a.pose_out = pose_out;
    a.sys = sys;
    a.corr_idx = corr_idx;
    a.corr_d2 = corr_sqdist;
    cudaStream_t s = (cudaStream_t)stream;
    reset_ticket_kernel<<<1, 1, 0, s>>>(a.st);
    count_launches(1);
    cudaError_t e = launch_proj(a, params->metric, s);
    if (e != cudaSuccess) return cuda_fail(e, "icp_proj_kernel launch");
    return CIL_OK;
}

CIL_API cil_status cil_proj_run(const float* tgt, const float* tgt_normals, const cil_intrinsics* K, const float* src,
                                int64_t m, const double* pose_init, const cil_icp_params* params, void* ws,
                                size_t ws_bytes, cil_icp_result* res, double* iter_log, cil_stream_t stream) {
    cil_status rc = check_proj("cil_proj_run", tgt, tgt_normals, K, src, m, params, ws, ws_bytes);
    if (rc != CIL_OK) return rc;
    if (!pose_init || !res) { set_error("cil_proj_run: pose_init/res NULL"); return CIL_ERR_INVALID_ARG; }
    if (params->max_iters < 1) { set_error("cil_proj_run: max_iters must be >= 1"); return CIL_ERR_INVALID_ARG; }
    IterArgs a{};
    bind_proj(a, tgt, tgt_normals, K, src, m, params, ws);
    a.bound2 = bound2_of(params->max_corr_dist);
    a.pose_in = a.st->pose;
    a.pose_out = a.st->pose;
    a.iter_log = iter_log;
    a.run = 1;
    cudaStream_t s = (cudaStream_t)stream;
    run_init_kernel<<<1, 256, 0, s>>>(a.st, pose_init, nullptr, nullptr, nullptr, 0, iter_log, 2 * params->max_iters);
    count_launches(1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "run_init_kernel launch");
    // one persistent cooperative launch for the whole loop; per-iteration launches if the device
    // cannot co-schedule the grid (same results: same grid, same arithmetic)
    e = launch_proj_run(a, params->metric, params->max_iters, s);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        for (int it = 0; it < params->max_iters; ++it) {
            e = launch_proj(a, params->metric, s);
            if (e != cudaSuccess) return cuda_fail(e, "icp_proj_kernel launch");
        }
    }
    run_final_kernel<<<1, 32, 0, s>>>(a.st, res);
    count_launches(1);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "run_final_kernel launch");
    return CIL_OK;
}
