// lnl.cu -- leaf neighbour lists over the BVH leaves (part of the spatial index, north_star
// subsystem (2); consumed by the exact-NN search, search.cuh "per-query list search").
//
// For every leaf h (a run of B Morton-consecutive target points with its AABB box(h)) the build
// stores up to K other leaves M sorted by their box-to-box distance dist(h, M), and a cut D_h
// such that EVERY leaf that is not in the list (other than h) has real box distance >= D_h.
// A query s whose hint leaf is h can then be resolved by scanning h's list alone: every point x
// of the ball B(s, r) lies within r + dist(s, box(h)) of box(h), so when r + dist(s, box(h)) <
// D_h the leaves that can hold a target inside the ball are all in the list, and, the list being
// sorted by distance, the scan stops at the first entry with dist(h, M) > r + dist(s, box(h)).
// This is the exact-NN search ("KDTree ... exact k-NN"; the per-iteration
// correspondence search of PAPER.md:140) with the candidate leaves found by a per-leaf table
// instead of a per-query traversal.
//
// Exactness of the table: every distance here is computed with round-down arithmetic
// (__fsub_rd / __fmaf_rd / __fsqrt_rd), so a computed distance never exceeds the real one;
// a node's computed distance is <= that of every leaf below it (its box contains theirs and
// the rounded operations are monotone), so a subtree pruned at computed distance > R holds
// only leaves at real distance > R.
//
// Build (one warp per leaf): a radius R from the leaf's 32 Morton neighbours, a breadth-first
// range query from the root collecting every leaf with computed distance <= R (frontier and
// candidates in shared memory; R halves on overflow and doubles while fewer than K + 1 leaves
// were found), a bitonic sort of the candidates by (distance, leaf), then the first K entries
// and the cut (the (K+1)-th distance, or R when all candidates fit).
#include "internal.cuh"

namespace cil {
namespace {

constexpr int kLnlWarps = 4;            // warps per CTA of the build (one leaf per warp)
constexpr int kLnlCap = 512;            // frontier / candidate capacity per warp (power of two)
constexpr int kLnlTries = 8;

__device__ __forceinline__ float box_dist_rd(float4 alo, float4 ahi, float4 blo, float4 bhi) {
    const float gx = fmaxf(fmaxf(__fsub_rd(blo.x, ahi.x), __fsub_rd(alo.x, bhi.x)), 0.0f);
    const float gy = fmaxf(fmaxf(__fsub_rd(blo.y, ahi.y), __fsub_rd(alo.y, bhi.y)), 0.0f);
    const float gz = fmaxf(fmaxf(__fsub_rd(blo.z, ahi.z), __fsub_rd(alo.z, bhi.z)), 0.0f);
    return __fsqrt_rd(__fmaf_rd(gx, gx, __fmaf_rd(gy, gy, __fmul_rd(gz, gz))));
}

// ascending bitonic sort of 32 floats held one per lane
__device__ __forceinline__ float warp_sort32(float v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const float o = __shfl_xor_sync(0xffffffffu, v, j);
            const bool up = (lane & k) == 0;
            const bool lower = (lane & j) == 0;
            v = (lower == up) ? fminf(v, o) : fmaxf(v, o);
        }
    }
    return v;
}

__global__ void __launch_bounds__(32 * kLnlWarps)
lnl_build_kernel(const float4* __restrict__ box, int l_pad, int n_leaves, int K, int2* __restrict__ lnl,
                 float* __restrict__ cut) {
    __shared__ int sF[kLnlWarps][2][kLnlCap];
    __shared__ unsigned long long sC[kLnlWarps][kLnlCap];
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int h = blockIdx.x * kLnlWarps + wid;
    if (h >= n_leaves) return;
    const float4 alo = __ldg(box + 2 * (size_t)(l_pad + h)), ahi = __ldg(box + 2 * (size_t)(l_pad + h) + 1);
    unsigned long long* C = sC[wid];
    // initial radius: the 16th smallest distance to the 16 Morton neighbours on either side
    float R;
    {
        const int o = lane < 16 ? h - 16 + lane : h + lane - 15;
        float d = INFINITY;
        if (o >= 0 && o < n_leaves)
            d = box_dist_rd(alo, ahi, __ldg(box + 2 * (size_t)(l_pad + o)), __ldg(box + 2 * (size_t)(l_pad + o) + 1));
        d = warp_sort32(d);
        R = __shfl_sync(FULL, d, 15);
        if (!(R < INFINITY)) R = __shfl_sync(FULL, d, 0);
    }
    // range query: every leaf != h with computed distance <= R; returns the count (> kLnlCap:
    // overflow, the buffer content is then incomplete)
    auto query = [&](float Rq) -> int {
        int* F = sF[wid][0];
        int* G = sF[wid][1];
        if (lane == 0) F[0] = 1;
        int nF = 1, nC = 0;
        __syncwarp();
        while (nF > 0) {
            const int nK = 2 * nF;
            int nN = 0;
            for (int b0 = 0; b0 < nK; b0 += 32) {
                const int j = b0 + lane;
                int c = 0;
                float d = INFINITY;
                if (j < nK) {
                    c = 2 * F[j >> 1] + (j & 1);
                    d = box_dist_rd(alo, ahi, __ldg(box + 2 * (size_t)c), __ldg(box + 2 * (size_t)c + 1));
                }
                const bool leaf = c >= l_pad;
                const bool keep = j < nK && d <= Rq && !(leaf && c - l_pad == h);
                const unsigned mk = __ballot_sync(FULL, keep);
                if (leaf) {     // uniform: every node of a level has the same depth
                    const int pos = nC + __popc(mk & lt);
                    if (keep && pos < kLnlCap)
                        C[pos] = ((unsigned long long)__float_as_uint(d) << 32) | (unsigned)(c - l_pad);
                    nC += __popc(mk);
                } else {
                    const int pos = nN + __popc(mk & lt);
                    if (keep && pos < kLnlCap) G[pos] = c;
                    nN += __popc(mk);
                }
            }
            __syncwarp();
            if (nN > kLnlCap) return kLnlCap + 1;
            int* t = F; F = G; G = t;
            nF = nN;
        }
        return nC;
    };
    float Rgood = -1.0f;
    int cgood = 0;
    float Rlast = -1.0f;
    for (int tr = 0; tr < kLnlTries && R < INFINITY; ++tr) {
        const int c = query(R);
        Rlast = R;
        if (c <= kLnlCap) {
            Rgood = R;
            cgood = c;
            if (c > K || R == 0.0f) break;
            R = R * 2.0f;
        } else {
            if (Rgood >= 0.0f) break;
            R = R * 0.5f;
        }
    }
    if (Rgood < 0.0f) {            // never fitted (pathological duplicates): an empty list, cut 0
        cgood = 0;
        Rgood = 0.0f;
    } else if (Rlast != Rgood) {
        cgood = query(Rgood);
    }
    // bitonic sort of the cgood keys (padded to a power of two with ~0)
    int np = 1;
    while (np < cgood) np <<= 1;
    for (int j = cgood + lane; j < np; j += 32) C[j] = ~0ull;
    __syncwarp();
    for (int k = 2; k <= np; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < np; i += 32) {
                const int p = i ^ j;
                if (p > i) {
                    const unsigned long long a = C[i], b = C[p];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) { C[i] = b; C[p] = a; }
                }
            }
            __syncwarp();
        }
    }
    int2* dst = lnl + (size_t)h * K;
    for (int e = lane; e < K; e += 32) {
        int2 v = make_int2(-1, __float_as_int(INFINITY));
        if (e < cgood) v = make_int2((int)(unsigned)(C[e] & 0xffffffffu), (int)(unsigned)(C[e] >> 32));
        dst[e] = v;
    }
    if (lane == 0) cut[h] = cgood > K ? __uint_as_float((unsigned)(C[K] >> 32)) : Rgood;
}

}  // namespace

size_t lnl_bytes(int64_t n_leaves, int K) {
    return align_up((size_t)n_leaves * K * sizeof(int2), 256) + align_up((size_t)n_leaves * sizeof(float), 256);
}

// Build the lists of every leaf into mem (lnl_bytes(n_leaves, K) bytes) after the tree passes.
cudaError_t lnl_build(const float4* box, int l_pad, int64_t n_leaves, int K, void* mem, cudaStream_t s,
                      TargetView* v) {
    int2* lnl = (int2*)mem;
    float* cut = (float*)((char*)mem + align_up((size_t)n_leaves * K * sizeof(int2), 256));
    const int grid = (int)((n_leaves + kLnlWarps - 1) / kLnlWarps);
    lnl_build_kernel<<<grid, 32 * kLnlWarps, 0, s>>>(box, l_pad, (int)n_leaves, K, lnl, cut);
    v->lnl = lnl;
    v->lnl_cut = cut;
    v->lnl_k = K;
    return cudaGetLastError();
}

}  // namespace cil
