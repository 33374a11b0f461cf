// normals.cu -- cil_estimate_normals: PCA surface normals of the target over its k nearest
// neighbours ("normal estimation", PAPER.md:172-176 the
// benchmark's 10-NN normals oriented towards the viewpoint; BASELINE.json configs[2] "normals
// from oracle PCA over 10-NN").
//
// One query per lane, queries taken in Morton order (the warp's lanes are spatial neighbours,
// so their traversals share nodes in L1/L2):
//   1. exact k-NN of the target point itself (self included): a sorted top-16 list of u64
//      keys (bits(d2) << 32 | original index, so equal distances order by the lowest index);
//      seeded from the point's own leaf and its two neighbours in Morton order, then an
//      independent nearest-child-first DFS of the BVH that enters a box iff its lower bound
//      is <= the k-th key's d2 (the lower bound uses the candidate arithmetic, so the search
//      is exact under the kernel's own fp32 distances);
//   2. mean and 1/k covariance of the k neighbours in fp64;
//   3. smallest eigenpair of the symmetric 3x3 covariance: eigenvalues by the trigonometric
//      closed form, eigenvector as the largest cross product of two rows of (C - lambda I);
//   4. orientation: n . (view - p) >= 0; curvature = lambda_min / trace.
#include "internal.cuh"
#include "search.cuh"

#include <algorithm>
#include <cmath>

namespace cil {
namespace {

constexpr int kKmax = 16;
constexpr int kNormThreads = 128;

template <int K>
__device__ __forceinline__ void topk_insert(unsigned long long (&top)[K], unsigned long long x) {
    // top[] ascending; x < top[K-1] (checked by the caller): shift the larger keys up by one
    bool done = false;
#pragma unroll
    for (int c = K - 1; c >= 1; --c) {
        const bool shift = !done && top[c - 1] > x;
        const bool put = !done && !shift;
        top[c] = shift ? top[c - 1] : (put ? x : top[c]);
        done = done || put;
    }
    if (!done) top[0] = x;
}

template <int K>
__device__ __forceinline__ unsigned long long kth(const unsigned long long (&top)[K], int k) {
    unsigned long long v = top[0];
#pragma unroll
    for (int c = 1; c < K; ++c) v = (c == k - 1) ? top[c] : v;
    return v;
}

template <int B>
__device__ __forceinline__ void offer_leaf(const TargetView& T, const NegQuery& nq, int leaf,
                                           unsigned long long (&top)[kKmax], int k) {
    float d2[B];
    leaf_d2<B>(T, nq, leaf, d2);
    const int* ids = reinterpret_cast<const int*>(T.leafsoa + (size_t)leaf * B + 3 * (B / 4));
    // candidates that can enter the top k (d2 at most the k-th distance; padding d2 = +inf never
    // does) as a bit mask, then ONE insertion site for them, lowest slot first (the order of the
    // per-candidate test it replaces); a candidate's d2 is recomputed from the leaf with the same
    // operations as leaf_d2, so no array is indexed at run time
    unsigned long long thr = kth(top, k);
    unsigned mask = 0;
#pragma unroll
    for (int c = 0; c < B; ++c) mask |= (d2[c] <= key_d2(thr) ? 1u : 0u) << c;
    const float* row = reinterpret_cast<const float*>(T.leafsoa + (size_t)leaf * B);
#pragma unroll 1
    while (mask) {
        const int c = __ffs(mask) - 1;
        mask &= mask - 1;
        const float2 x = make_float2(__ldg(row + c), 0.0f), y = make_float2(__ldg(row + B + c), 0.0f),
                     z = make_float2(__ldg(row + 2 * B + c), 0.0f);
        const float dc = pair_d2(nq, x, y, z).x;
        const unsigned long long key = make_key(dc, (uint32_t)__ldg(ids + c));
        if (key < thr) {
            topk_insert(top, key);
            thr = kth(top, k);
        }
    }
}

// smallest eigenpair of a symmetric 3x3 (fp64): returns lambda_min, the unit eigenvector in v,
// and the trace in tr
__device__ double min_eigen3(const double C[6], double v[3], double& tr) {
    // C = [c00 c01 c02; . c11 c12; . . c22] as {c00, c01, c02, c11, c12, c22}
    const double a = C[0], b = C[1], c = C[2], d = C[3], e = C[4], f = C[5];
    tr = a + d + f;
    const double q = tr / 3.0;
    const double p1 = b * b + c * c + e * e;
    const double p2 = (a - q) * (a - q) + (d - q) * (d - q) + (f - q) * (f - q) + 2.0 * p1;
    double lmin;
    if (p2 <= 0.0) {
        lmin = q;                                        // C = q I: every direction is an eigenvector
    } else {
        const double p = sqrt(p2 / 6.0);
        const double ip = 1.0 / p;
        const double B00 = (a - q) * ip, B11 = (d - q) * ip, B22 = (f - q) * ip;
        const double B01 = b * ip, B02 = c * ip, B12 = e * ip;
        double r = 0.5 * (B00 * (B11 * B22 - B12 * B12) - B01 * (B01 * B22 - B12 * B02) + B02 * (B01 * B12 - B11 * B02));
        r = fmin(fmax(r, -1.0), 1.0);
        const double phi = acos(r) / 3.0;
        lmin = q + 2.0 * p * cos(phi + 2.0943951023931954923);   // + 2 pi / 3
    }
    // eigenvector: the largest cross product of two rows of (C - lmin I)
    const double r0[3] = {a - lmin, b, c}, r1[3] = {b, d - lmin, e}, r2[3] = {c, e, f - lmin};
    const double x01[3] = {r0[1] * r1[2] - r0[2] * r1[1], r0[2] * r1[0] - r0[0] * r1[2], r0[0] * r1[1] - r0[1] * r1[0]};
    const double x02[3] = {r0[1] * r2[2] - r0[2] * r2[1], r0[2] * r2[0] - r0[0] * r2[2], r0[0] * r2[1] - r0[1] * r2[0]};
    const double x12[3] = {r1[1] * r2[2] - r1[2] * r2[1], r1[2] * r2[0] - r1[0] * r2[2], r1[0] * r2[1] - r1[1] * r2[0]};
    const double n01 = x01[0] * x01[0] + x01[1] * x01[1] + x01[2] * x01[2];
    const double n02 = x02[0] * x02[0] + x02[1] * x02[1] + x02[2] * x02[2];
    const double n12 = x12[0] * x12[0] + x12[1] * x12[1] + x12[2] * x12[2];
    const double* x = x01;
    double nn = n01;
    if (n02 > nn) { x = x02; nn = n02; }
    if (n12 > nn) { x = x12; nn = n12; }
    if (nn > 0.0) {
        const double s = 1.0 / sqrt(nn);
        v[0] = x[0] * s; v[1] = x[1] * s; v[2] = x[2] * s;
    } else {
        // (C - lmin I) of rank <= 1: lmin is a double eigenvalue; any unit vector orthogonal
        // to a non-zero row is an eigenvector of it
        const double* rr = r0;
        double m = r0[0] * r0[0] + r0[1] * r0[1] + r0[2] * r0[2];
        const double m1 = r1[0] * r1[0] + r1[1] * r1[1] + r1[2] * r1[2];
        const double m2 = r2[0] * r2[0] + r2[1] * r2[1] + r2[2] * r2[2];
        if (m1 > m) { rr = r1; m = m1; }
        if (m2 > m) { rr = r2; m = m2; }
        if (m == 0.0) { v[0] = 0.0; v[1] = 0.0; v[2] = 1.0; }
        else {
            // orthogonal to rr: cross with the axis least aligned with it
            const double ax = fabs(rr[0]), ay = fabs(rr[1]), az = fabs(rr[2]);
            const double e3[3] = {ax <= ay && ax <= az ? 1.0 : 0.0, ay < ax && ay <= az ? 1.0 : 0.0,
                                  az < ax && az < ay ? 1.0 : 0.0};
            double w[3] = {rr[1] * e3[2] - rr[2] * e3[1], rr[2] * e3[0] - rr[0] * e3[2], rr[0] * e3[1] - rr[1] * e3[0]};
            const double s = 1.0 / sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
            v[0] = w[0] * s; v[1] = w[1] * s; v[2] = w[2] * s;
        }
    }
    return lmin;
}

template <int B>
__global__ void __launch_bounds__(kNormThreads)
knn_normals_kernel(TargetView T, int k, double vx, double vy, double vz, float* __restrict__ normals,
                   float* __restrict__ curvature) {
    const int sp = blockIdx.x * blockDim.x + threadIdx.x;        // sorted position of the query
    if (sp >= T.n) return;
    const int leaf0 = sp / B;
    const float* blk = reinterpret_cast<const float*>(T.leafsoa + (size_t)leaf0 * B);
    const float qx = __ldg(blk + sp % B), qy = __ldg(blk + B + sp % B), qz = __ldg(blk + 2 * B + sp % B);
    const uint32_t qid = (uint32_t)__ldg(reinterpret_cast<const int*>(blk) + 3 * B + sp % B);
    DF3 s;
    s.hx = qx; s.hy = qy; s.hz = qz; s.lx = s.ly = s.lz = 0.0f;
    const NegQuery nq = neg_query(s);
    unsigned long long top[kKmax];
#pragma unroll
    for (int c = 0; c < kKmax; ++c) top[c] = bound_key(INFINITY);
    // 1. seed: own leaf and its Morton neighbours, then the exact DFS
    const int nl = (T.n + B - 1) / B;
    offer_leaf<B>(T, nq, leaf0, top, k);
    if (leaf0 > 0) offer_leaf<B>(T, nq, leaf0 - 1, top, k);
    if (leaf0 + 1 < nl) offer_leaf<B>(T, nq, leaf0 + 1, top, k);
    int sv[kDfsStack];
    float slb[kDfsStack];
    int stp = 0, v = 1;
    const int l_pad = T.l_pad;
    while (true) {
        const float thr = key_d2(kth(top, k));
        while (v < l_pad) {
            const int c = 2 * v;
            const float4* bx = T.box + 2 * (size_t)c;
            const float lb0 = box_lb2(s, __ldg(bx), __ldg(bx + 1));
            const float lb1 = box_lb2(s, __ldg(bx + 2), __ldg(bx + 3));
            const bool g0 = lb0 <= thr, g1 = lb1 <= thr;
            if (g0 && g1) {
                const bool r1 = lb1 < lb0;
                sv[stp] = r1 ? c : c + 1;
                slb[stp] = r1 ? lb0 : lb1;
                ++stp;
                v = r1 ? c + 1 : c;
            } else if (g0) {
                v = c;
            } else if (g1) {
                v = c + 1;
            } else {
                v = 0;
                break;
            }
        }
        if (v >= l_pad) {
            const int leaf = v - l_pad;
            if (leaf != leaf0 && leaf != leaf0 - 1 && leaf != leaf0 + 1) offer_leaf<B>(T, nq, leaf, top, k);
        }
        v = 0;
        while (stp > 0) {
            --stp;
            if (slb[stp] <= key_d2(kth(top, k))) { v = sv[stp]; break; }
        }
        if (v == 0) break;
    }
    // 2. mean and 1/k covariance (fp64) of the k neighbours actually found (a non-finite query
    //    or target coordinate leaves slots at the "nothing" key: fewer than 3 -> zero normal)
    int kk = 0;
#pragma unroll
    for (int c = 0; c < kKmax; ++c)
        kk += (c < min(k, T.n) && key_idx(top[c]) != 0xffffffffu && (uint32_t)(top[c] >> 32) <= 0x7f800000u) ? 1 : 0;
    if (kk < 3) {
        normals[3 * (size_t)qid] = 0.0f;
        normals[3 * (size_t)qid + 1] = 0.0f;
        normals[3 * (size_t)qid + 2] = 0.0f;
        if (curvature) curvature[qid] = 0.0f;
        return;
    }
    double mu[3] = {0.0, 0.0, 0.0};
    float4 P[kKmax];
#pragma unroll
    for (int c = 0; c < kKmax; ++c) {
        P[c] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (c < kk) {
            P[c] = __ldg(T.opts + key_idx(top[c]));
            mu[0] += P[c].x; mu[1] += P[c].y; mu[2] += P[c].z;
        }
    }
    const double ik = 1.0 / (double)kk;
    mu[0] *= ik; mu[1] *= ik; mu[2] *= ik;
    double C[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < kKmax; ++c) {
        if (c < kk) {
            const double dx = P[c].x - mu[0], dy = P[c].y - mu[1], dz = P[c].z - mu[2];
            C[0] += dx * dx; C[1] += dx * dy; C[2] += dx * dz;
            C[3] += dy * dy; C[4] += dy * dz; C[5] += dz * dz;
        }
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) C[c] *= ik;
    // 3. smallest eigenpair, 4. orientation towards the viewpoint
    double nv[3], tr;
    const double lmin = min_eigen3(C, nv, tr);
    const double dv = (vx - qx) * nv[0] + (vy - qy) * nv[1] + (vz - qz) * nv[2];
    const double sg = dv < 0.0 ? -1.0 : 1.0;
    normals[3 * (size_t)qid] = (float)(sg * nv[0]);
    normals[3 * (size_t)qid + 1] = (float)(sg * nv[1]);
    normals[3 * (size_t)qid + 2] = (float)(sg * nv[2]);
    if (curvature) curvature[qid] = (float)(tr > 0.0 ? fmax(lmin, 0.0) / tr : 0.0);
}

}  // namespace
}  // namespace cil

using namespace cil;

CIL_API cil_status cil_estimate_normals(const cil_target* t, int32_t k, const double* view, float* normals,
                                        float* curvature, cil_stream_t stream) {
    if (!t) { set_error("cil_estimate_normals: target is NULL"); return CIL_ERR_INVALID_ARG; }
    if (!normals) { set_error("cil_estimate_normals: normals is NULL"); return CIL_ERR_INVALID_ARG; }
    if (k < 3 || k > kKmax) { set_error("cil_estimate_normals: k=%d not in [3, %d]", k, kKmax); return CIL_ERR_INVALID_ARG; }
    const double vx = view ? view[0] : 0.0, vy = view ? view[1] : 0.0, vz = view ? view[2] : 0.0;
    if (!std::isfinite(vx) || !std::isfinite(vy) || !std::isfinite(vz)) {
        set_error("cil_estimate_normals: viewpoint must be finite");
        return CIL_ERR_INVALID_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int g = (int)((t->v.n + kNormThreads - 1) / kNormThreads);
    switch (t->v.leaf_size) {
        case 4: knn_normals_kernel<4><<<g, kNormThreads, 0, s>>>(t->v, k, vx, vy, vz, normals, curvature); break;
        case 8: knn_normals_kernel<8><<<g, kNormThreads, 0, s>>>(t->v, k, vx, vy, vz, normals, curvature); break;
        case 16: knn_normals_kernel<16><<<g, kNormThreads, 0, s>>>(t->v, k, vx, vy, vz, normals, curvature); break;
        default: knn_normals_kernel<32><<<g, kNormThreads, 0, s>>>(t->v, k, vx, vy, vz, normals, curvature); break;
    }
    count_launches(1);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? CIL_OK : cuda_fail(e, "knn_normals_kernel launch");
}
