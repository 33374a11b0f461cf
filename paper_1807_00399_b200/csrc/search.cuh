// search.cuh -- device side of the exact 1-NN search.
//
// Index: target points sorted by 48-bit Morton key, grouped into leaves of B consecutive
// points, with an implicit complete binary tree of AABBs over the leaves (node v has
// children 2v, 2v+1; leaves are nodes l_pad .. 2 l_pad - 1).
//
// Search ("hint leaf, then ascend"): evaluate a hint leaf (the warm-start match of the
// previous ICP iteration, or the leaf holding the first target of the query's coarse Morton
// cell), then walk up the ancestors of that leaf.  At each ancestor u:
//   * STOP if the ball B(s, sqrt(best)) provably holds no target outside u's subtree:
//     every target in the ball has a Morton key in [code(ball_lo), code(ball_hi)] (the key is
//     monotone in each quantised coordinate; one quantum of margin absorbs rounding), and
//     u's subtree is exactly the sorted key range [key[a], key[b-1]]; so if
//     key[a-1] < code(ball_lo) and code(ball_hi) < key[b] nothing outside can be in the ball;
//   * otherwise test u's sibling box and search it (nearest-child-first DFS) if its lower
//     bound does not exceed the best distance.
// The subtrees of the siblings of all ancestors partition the tree, so the search is exact.
//
// Precision contract:
//  * the transformed query s = R p + t is computed in fp64 and carried as a double-float
//    pair (hi = fl32(s), lo = fl32(s - hi)), never materialised in fp32 alone;
//  * per candidate the difference is (s_hi - t) + s_lo in fp32 -- accurate to ~1 ulp of
//    |s - t| rather than of |s| -- and d^2 = fma(dx,dx, fma(dy,dy, dz*dz)) in fp32;
//  * the minimum is taken over the u64 key (bits(d^2) << 32) | original_index, which orders
//    by d^2 (non-negative IEEE floats order like their bit patterns) and breaks exact ties
//    by the lowest original index (R1);
//  * a box is pruned iff its lower bound lb^2 > best d^2, where lb is computed with the
//    SAME rounded operations as the candidate differences, so by monotonicity of IEEE
//    rounding lb^2 <= d^2 of every point inside the box: pruning never drops a point that
//    could win (or tie) under the kernel's own arithmetic -- the search is exact.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "internal.cuh"

namespace cil {

struct DF3 {
    float hx, hy, hz;   // fl32(s)
    float lx, ly, lz;   // fl32(s - fl32(s))
};

__device__ __forceinline__ DF3 split_df(double x, double y, double z) {
    DF3 s;
    s.hx = __double2float_rn(x);
    s.hy = __double2float_rn(y);
    s.hz = __double2float_rn(z);
    s.lx = __double2float_rn(x - (double)s.hx);
    s.ly = __double2float_rn(y - (double)s.hy);
    s.lz = __double2float_rn(z - (double)s.hz);
    return s;
}

// s = R p + t with the 3x4 top of a row-major fp64 pose held in registers.
struct Pose34 {
    double r[12];
};

__device__ __forceinline__ DF3 transform_df(const Pose34& P, float px, float py, float pz) {
    double x = fma(P.r[0], (double)px, fma(P.r[1], (double)py, fma(P.r[2], (double)pz, P.r[3])));
    double y = fma(P.r[4], (double)px, fma(P.r[5], (double)py, fma(P.r[6], (double)pz, P.r[7])));
    double z = fma(P.r[8], (double)px, fma(P.r[9], (double)py, fma(P.r[10], (double)pz, P.r[11])));
    return split_df(x, y, z);
}

// ---------------------------------------------------------------- Morton quantisation
// (used identically by the index build and by the search's containment test)
__device__ __forceinline__ unsigned long long spread3(unsigned long long x) {
    x &= 0xffffull;                                  // 16 bits -> every third bit of 48
    x = (x | (x << 16)) & 0x0000ff0000ffull;
    x = (x | (x << 8)) & 0x00f00f00f00full;
    x = (x | (x << 4)) & 0x0c30c30c30c3ull;
    x = (x | (x << 2)) & 0x249249249249ull;
    return x;
}

__device__ __forceinline__ unsigned quantize1(float x, float mn, float sc) {
    return (unsigned)fminf(fmaxf((x - mn) * sc, 0.0f), (float)((1 << kMortonBits) - 1));
}

__device__ __forceinline__ unsigned long long morton3(unsigned qx, unsigned qy, unsigned qz) {
    return (spread3(qx) << 2) | (spread3(qy) << 1) | spread3(qz);
}

__device__ __forceinline__ unsigned long long morton_of(float4 Q, float x, float y, float z) {
    return morton3(quantize1(x, Q.x, Q.w), quantize1(y, Q.y, Q.w), quantize1(z, Q.z, Q.w));
}

// ---------------------------------------------------------------- keys and distances
__device__ __forceinline__ unsigned long long make_key(float d2, uint32_t idx) {
    return ((unsigned long long)__float_as_uint(d2) << 32) | (unsigned long long)idx;
}
__device__ __forceinline__ float key_d2(unsigned long long k) { return __uint_as_float((uint32_t)(k >> 32)); }
__device__ __forceinline__ uint32_t key_idx(unsigned long long k) { return (uint32_t)(k & 0xffffffffull); }

// The "nothing found" key for a search bounded by d^2 <= bound2 (inclusive): any real
// candidate with d^2 <= bound2 has an index < 0xffffffff and therefore a smaller key.
__device__ __forceinline__ unsigned long long bound_key(float bound2) { return make_key(bound2, 0xffffffffu); }

// Precise difference s - t for one coordinate.
__device__ __forceinline__ float dfdiff(float sh, float sl, float t) { return (sh - t) + sl; }

__device__ __forceinline__ float cand_d2(const DF3& s, float4 t) {
    float dx = dfdiff(s.hx, s.lx, t.x);
    float dy = dfdiff(s.hy, s.ly, t.y);
    float dz = dfdiff(s.hz, s.lz, t.z);
    return fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}

// Lower bound of cand_d2 over every point inside [lo, hi] (see header comment).
__device__ __forceinline__ float box_lb2(const DF3& s, float4 lo, float4 hi) {
    float gx = fmaxf(fmaxf((lo.x - s.hx) - s.lx, (s.hx - hi.x) + s.lx), 0.0f);
    float gy = fmaxf(fmaxf((lo.y - s.hy) - s.ly, (s.hy - hi.y) + s.ly), 0.0f);
    float gz = fmaxf(fmaxf((lo.z - s.hz) - s.lz, (s.hz - hi.z) + s.lz), 0.0f);
    return fmaf(gx, gx, fmaf(gy, gy, gz * gz));
}

__device__ __forceinline__ float node_lb2(const TargetView& T, const DF3& s, int v) {
    const float4* bx = T.box + 2 * (size_t)v;
    return box_lb2(s, __ldg(bx), __ldg(bx + 1));
}

// Evaluate candidate at sorted position j; keep the best key and its sorted position.
__device__ __forceinline__ void offer(const DF3& s, float4 t, int j, unsigned long long& best, int& bpos) {
    unsigned long long k = make_key(cand_d2(s, t), (uint32_t)__float_as_int(t.w));
    if (k < best) { best = k; bpos = j; }
}

// ---------------------------------------------------------------- leaf evaluation
// A leaf is a block of B consecutive sorted targets stored as rows x[B], y[B], z[B], idx[B]
// (leafsoa).  Two candidates per instruction with the sm_100 packed FP32 ops (FADD2, FFMA2,
// FMUL2): -dx = (t + (-s_hi)) + (-s_lo) is exactly the negation of (s_hi - t) + s_lo (IEEE
// rounding is sign-symmetric), so d^2 is bit-identical to cand_d2().
struct NegQuery {
    float2 hx, hy, hz, lx, ly, lz;   // broadcast -s_hi, -s_lo
};

__device__ __forceinline__ NegQuery neg_query(const DF3& s) {
    NegQuery q;
    q.hx = make_float2(-s.hx, -s.hx); q.hy = make_float2(-s.hy, -s.hy); q.hz = make_float2(-s.hz, -s.hz);
    q.lx = make_float2(-s.lx, -s.lx); q.ly = make_float2(-s.ly, -s.ly); q.lz = make_float2(-s.lz, -s.lz);
    return q;
}

__device__ __forceinline__ float2 pair_d2(const NegQuery& q, float2 x, float2 y, float2 z) {
    const float2 dx = __fadd2_rn(__fadd2_rn(x, q.hx), q.lx);
    const float2 dy = __fadd2_rn(__fadd2_rn(y, q.hy), q.ly);
    const float2 dz = __fadd2_rn(__fadd2_rn(z, q.hz), q.lz);
    return __ffma2_rn(dx, dx, __ffma2_rn(dy, dy, __fmul2_rn(dz, dz)));
}

template <int B>
__device__ __forceinline__ void eval_leaf(const TargetView& T, const NegQuery& q, int leaf,
                                          unsigned long long& best, int& bpos) {
    constexpr int R = B / 4;                                   // float4 per row
    const float4* blk = T.leafsoa + (size_t)leaf * (4 * R);
    float d2[B];
#pragma unroll
    for (int c = 0; c < R; ++c) {
        const float4 X = __ldg(blk + c), Y = __ldg(blk + R + c), Z = __ldg(blk + 2 * R + c);
        const float2 a = pair_d2(q, make_float2(X.x, X.y), make_float2(Y.x, Y.y), make_float2(Z.x, Z.y));
        const float2 b = pair_d2(q, make_float2(X.z, X.w), make_float2(Y.z, Y.w), make_float2(Z.z, Z.w));
        d2[4 * c + 0] = a.x; d2[4 * c + 1] = a.y; d2[4 * c + 2] = b.x; d2[4 * c + 3] = b.y;
    }
    float mn = d2[0];
#pragma unroll
    for (int c = 1; c < B; ++c) mn = fminf(mn, d2[c]);
    if (mn <= key_d2(best)) {                                   // an improvement or a tie is possible
        // lowest original index among the candidates at the minimum (R1), then one key compare
        const int* ids = reinterpret_cast<const int*>(blk + 3 * R);
        uint32_t imin = 0xffffffffu;
        int cmin = 0;
#pragma unroll
        for (int c = 0; c < B; ++c) {
            const uint32_t id = (uint32_t)__ldg(ids + c);
            const bool take = d2[c] == mn && id < imin;
            imin = take ? id : imin;
            cmin = take ? c : cmin;
        }
        const unsigned long long k = make_key(mn, imin);
        if (k < best) { best = k; bpos = leaf * B + cmin; }
    }
}

// Morton codes bounding every target that may lie in the ball B(s, sqrt(r2)).
__device__ __forceinline__ void ball_codes(const float4 Q, const DF3& s, float r2,
                                           unsigned long long& clo, unsigned long long& chi) {
    const unsigned qmax = (1u << kMortonBits) - 1u;
    if (!(r2 < INFINITY)) { clo = 0ull; chi = ~0ull; return; }
    const float r = sqrtf(r2) * 1.000001f + 1e-30f;
    unsigned lx = quantize1((s.hx - r) + s.lx, Q.x, Q.w), hx = quantize1((s.hx + r) + s.lx, Q.x, Q.w);
    unsigned ly = quantize1((s.hy - r) + s.ly, Q.y, Q.w), hy = quantize1((s.hy + r) + s.ly, Q.y, Q.w);
    unsigned lz = quantize1((s.hz - r) + s.lz, Q.z, Q.w), hz = quantize1((s.hz + r) + s.lz, Q.z, Q.w);
    // one quantum of margin against rounding in the quantisation of the ball corners
    lx = lx > 0 ? lx - 1 : 0; ly = ly > 0 ? ly - 1 : 0; lz = lz > 0 ? lz - 1 : 0;
    hx = hx < qmax ? hx + 1 : qmax; hy = hy < qmax ? hy + 1 : qmax; hz = hz < qmax ? hz + 1 : qmax;
    clo = morton3(lx, ly, lz);
    chi = morton3(hx, hy, hz);
}

// Cold-start hint: the leaf holding the target whose Morton key follows the query's own key
// (coarse-cell table, then a binary search inside the query's coarse cell).
__device__ __forceinline__ int coarse_hint_leaf(const TargetView& T, const DF3& s) {
    const float4 Q = __ldg(T.quant);
    const unsigned long long code = morton_of(Q, s.hx, s.hy, s.hz);
    const unsigned c = (unsigned)(code >> (3 * kMortonBits - T.coarse_bits));
    int lo = (int)__ldg(T.cell_first + c), hi = (int)__ldg(T.cell_first + c + 1);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(T.keys + mid) < code) lo = mid + 1; else hi = mid;
    }
    return min(lo, T.n - 1) / T.leaf_size;
}

// ---------------------------------------------------------------- per-lane search state
struct NoStats {
    __device__ __forceinline__ void node() {}
    __device__ __forceinline__ void leaf() {}
    __device__ __forceinline__ void level() {}
};
struct CountStats {
    int nodes = 0, leaves = 0, levels = 0;
    __device__ __forceinline__ void node() { ++nodes; }
    __device__ __forceinline__ void leaf() { ++leaves; }
    __device__ __forceinline__ void level() { ++levels; }
};

constexpr int kMaxDepth = 32;

struct LaneSearch {
    DF3 s;
    unsigned long long best;
    int bpos;
    int sp;            // DFS stack depth
    int k;             // ascent level (0 = the hint leaf itself)
    int u;             // current ancestor node
    float r2;          // radius^2 the ball codes were computed for
    unsigned long long clo, chi;
};

// DFS stack of one lane (local memory, kept apart from the register-resident LaneSearch)
struct LaneStack {
    int v[kMaxDepth];
    float lb[kMaxDepth];
};

__device__ __forceinline__ void lane_start(LaneSearch& L, const TargetView& T, const DF3& s,
                                           unsigned long long init, int hint_leaf) {
    L.s = s;
    L.best = init;
    L.bpos = -1;
    L.sp = 0;
    L.k = 0;
    L.u = T.l_pad + hint_leaf;
    L.r2 = -1.0f;
}

// Advance this lane's search to the next leaf that must be evaluated; returns the leaf or -1
// when the search is complete (see the header comment for the ascent / containment rule).
template <class Stats>
__device__ __forceinline__ int next_leaf(LaneSearch& L, LaneStack& K, const TargetView& T, Stats* st) {
    while (true) {
        if (L.sp > 0) {
            --L.sp;
            int v = K.v[L.sp];
            if (K.lb[L.sp] > key_d2(L.best)) continue;
            while (v < T.l_pad) {
                if (st) st->node();
                const int c = 2 * v;
                const float4* bx = T.box + 2 * (size_t)c;
                const float4 lo0 = __ldg(bx + 0), hi0 = __ldg(bx + 1), lo1 = __ldg(bx + 2), hi1 = __ldg(bx + 3);
                const float lb0 = box_lb2(L.s, lo0, hi0);
                const float lb1 = box_lb2(L.s, lo1, hi1);
                const float bd = key_d2(L.best);
                const bool g0 = lb0 <= bd, g1 = lb1 <= bd;
                if (g0 && g1) {
                    const bool right_first = lb1 < lb0;
                    K.v[L.sp] = right_first ? c : c + 1;
                    K.lb[L.sp] = right_first ? lb0 : lb1;
                    ++L.sp;
                    v = right_first ? c + 1 : c;
                } else if (g0) {
                    v = c;
                } else if (g1) {
                    v = c + 1;
                } else {
                    v = -1;
                    break;
                }
            }
            if (v >= 0) return v - T.l_pad;
            continue;
        }
        if (L.k >= T.levels) return -1;
        if (st) st->level();
        const float bd = key_d2(L.best);
        if (bd != L.r2) { ball_codes(__ldg(T.quant), L.s, bd, L.clo, L.chi); L.r2 = bd; }
        const int a = min(((L.u << L.k) - T.l_pad) * T.leaf_size, T.n);
        const int b = min((((L.u + 1) << L.k) - T.l_pad) * T.leaf_size, T.n);
        const bool lo_in = a == 0 || __ldg(T.keys + a - 1) < L.clo;
        const bool hi_in = b >= T.n || L.chi < __ldg(T.keys + b);
        if (lo_in && hi_in) { L.k = T.levels; return -1; }
        const int sib = L.u ^ 1;
        const float lb = node_lb2(T, L.s, sib);
        ++L.k;
        L.u >>= 1;
        if (lb <= bd) {
            K.v[0] = sib;
            K.lb[0] = lb;
            L.sp = 1;
        }
    }
}

// ---------------------------------------------------------------- warp-packet engine
// A warp takes 32 consecutive queries (one per lane; consecutive = spatially coherent for
// Morton- or scan-ordered inputs).
//   A. every lane evaluates its own hint leaf (warm-start match or cold hint): a per-lane
//      bound r_i = sqrt(best_i).
//   B. lanes whose r_i is far above the packet mean are "outliers"; the others define the
//      packet box P = AABB of their balls B(s_i, r_i) (conservatively inflated).
//   C. breadth-first frontier walk of the BVH: children of the frontier are tested against P,
//      one box per lane, and compacted with ballots; the last frontier is the list of leaves
//      whose box meets P -- a superset of the leaves meeting any normal lane's ball.
//   D. every lane tests every candidate leaf's box against its own ball and appends the
//      leaves it needs to a private work list (shared memory); the lists are then evaluated in
//      rounds, each lane gathering its own leaf (packed FP32), so the number of evaluation
//      rounds is the longest list, not the size of the packet's union.
//   E. outlier lanes (and whole packets whose frontier overflowed) finish with the exact
//      ballot DFS: a node is entered iff its lower bound is <= some active lane's best.
// Every lane therefore examines every leaf that can hold a target inside its ball: each
// lane's result is its exact nearest neighbour.
// Q supplies
//   __device__ bool load(int i, DF3& s, unsigned long long& init, int& hint_leaf)
//   __device__ void store(int i, unsigned long long best, int bpos, const DF3& s)
constexpr int kFrontierCap = 256;
constexpr int kListCap = 8;         // per-lane work-list entries before an evaluation batch
constexpr int kEngineWarps = 8;     // warps per block of the engine kernels (blockDim 256)

template <int B>
__device__ __forceinline__ void ballot_dfs(const TargetView& T, const DF3& s, const NegQuery& nq, bool on,
                                           unsigned long long& best, int& bpos) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int l_pad = T.l_pad;
    // lanes that are not searching use a negative radius: no lower bound can pass it
    const float neg = -1.0f;
    int stk = 0, sp = 0, v = 1;
    while (true) {
        const float bd = on ? key_d2(best) : neg;
        if (v >= l_pad) {
            eval_leaf<B>(T, nq, v - l_pad, best, bpos);
        } else {
            const int c = 2 * v;
            const float4* bx = T.box + 2 * (size_t)c;
            const float4 lo0 = __ldg(bx + 0), hi0 = __ldg(bx + 1), lo1 = __ldg(bx + 2), hi1 = __ldg(bx + 3);
            const float lb0 = box_lb2(s, lo0, hi0), lb1 = box_lb2(s, lo1, hi1);
            const unsigned m0 = __ballot_sync(FULL, lb0 <= bd);
            const unsigned m1 = __ballot_sync(FULL, lb1 <= bd);
            if (m0 && m1) {
                const unsigned pref1 = __ballot_sync(FULL, lb1 < lb0);
                const bool right_first = __popc(pref1 & (m0 | m1)) * 2 > __popc(m0 | m1);
                if (lane == sp) stk = right_first ? c : c + 1;
                ++sp;
                v = right_first ? c + 1 : c;
                continue;
            }
            if (m0) { v = c; continue; }
            if (m1) { v = c + 1; continue; }
        }
        bool found = false;
        while (sp > 0) {
            --sp;
            const int cand = __shfl_sync(FULL, stk, sp);
            const float lb = node_lb2(T, s, cand);
            if (__any_sync(FULL, lb <= (on ? key_d2(best) : neg))) { v = cand; found = true; break; }
        }
        if (!found) break;
    }
}

__device__ __forceinline__ bool box_meets(float4 lo, float4 hi, float4 plo, float4 phi) {
    return lo.x <= phi.x && lo.y <= phi.y && lo.z <= phi.z && hi.x >= plo.x && hi.y >= plo.y && hi.z >= plo.z;
}

template <int B, class Q, class Stats = NoStats>
__device__ __forceinline__ void nn_packet_engine(const TargetView& T, Q& qs, int m, unsigned int* counter,
                                                 Stats* st = nullptr) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int l_pad = T.l_pad;
    __shared__ int frontier[kEngineWarps][2][kFrontierCap];
    __shared__ int worklist[kEngineWarps][1][kListCap * 32];
    int* F = frontier[threadIdx.x >> 5][0];
    int* G = frontier[threadIdx.x >> 5][1];
    while (true) {
        int base = 0;
        if (lane == 0) base = (int)atomicAdd(counter, 32u);
        base = __shfl_sync(FULL, base, 0);
        if (base >= m) break;
        const int qi = base + lane;
        DF3 s;
        unsigned long long best = 0ull;
        int bpos = -1;
        int hint = -1;
        bool active = false;
        if (qi < m) {
            active = qs.load(qi, s, best, hint);
            if (active && hint < 0) hint = coarse_hint_leaf(T, s);
        }
        if (!active) { s.hx = s.hy = s.hz = 0.0f; s.lx = s.ly = s.lz = 0.0f; }
        const NegQuery nq = neg_query(s);
        // ---- A
        if (active) {
            if (st) st->leaf();
            eval_leaf<B>(T, nq, hint, best, bpos);
        }
        // ---- B: outliers and the packet box
        const float r = active ? sqrtf(key_d2(best)) : 0.0f;
        float rsum = r;
        int na = active ? 1 : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            rsum += __shfl_xor_sync(FULL, rsum, o);
            na += __shfl_xor_sync(FULL, na, o);
        }
        const float rcap = 3.0f * rsum / (float)max(na, 1);
        const bool normal = active && r <= rcap && r < INFINITY;
        const bool outlier = active && !normal;
        // inflate for the double-float offset and for rounding of s_hi -/+ r
        const float rx = r * 1.000001f + fabsf(s.lx) + 1e-6f * fabsf(s.hx) + 1e-30f;
        const float ry = r * 1.000001f + fabsf(s.ly) + 1e-6f * fabsf(s.hy) + 1e-30f;
        const float rz = r * 1.000001f + fabsf(s.lz) + 1e-6f * fabsf(s.hz) + 1e-30f;
        float4 plo = make_float4(normal ? s.hx - rx : INFINITY, normal ? s.hy - ry : INFINITY,
                                 normal ? s.hz - rz : INFINITY, 0.0f);
        float4 phi = make_float4(normal ? s.hx + rx : -INFINITY, normal ? s.hy + ry : -INFINITY,
                                 normal ? s.hz + rz : -INFINITY, 0.0f);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            plo.x = fminf(plo.x, __shfl_xor_sync(FULL, plo.x, o));
            plo.y = fminf(plo.y, __shfl_xor_sync(FULL, plo.y, o));
            plo.z = fminf(plo.z, __shfl_xor_sync(FULL, plo.z, o));
            phi.x = fmaxf(phi.x, __shfl_xor_sync(FULL, phi.x, o));
            phi.y = fmaxf(phi.y, __shfl_xor_sync(FULL, phi.y, o));
            phi.z = fmaxf(phi.z, __shfl_xor_sync(FULL, phi.z, o));
        }
        bool overflow = false;
        if (__any_sync(FULL, normal)) {
            // ---- C: frontier walk from the root against the packet box
            if (lane == 0) F[0] = 1;
            __syncwarp();
            int nF = 1;
            for (int lev = 0; lev < T.levels && nF > 0; ++lev) {
                const int nC = 2 * nF;
                int nN = 0;
                for (int b0 = 0; b0 < nC; b0 += 32) {
                    const int j = b0 + lane;
                    int c = 0;
                    bool hit = false;
                    if (j < nC) {
                        c = 2 * F[j >> 1] + (j & 1);
                        const float4* bx = T.box + 2 * (size_t)c;
                        hit = box_meets(__ldg(bx), __ldg(bx + 1), plo, phi);
                    }
                    const unsigned mk = __ballot_sync(FULL, hit);
                    const int pos = nN + __popc(mk & lt);
                    if (hit && pos < kFrontierCap) G[pos] = c;
                    nN += __popc(mk);
                }
                __syncwarp();
                if (st && lane == 0) st->node();
                if (nN > kFrontierCap) { overflow = true; break; }
                int* tmp = F; F = G; G = tmp;
                nF = nN;
            }
            // ---- D: candidate leaves -> per-lane work lists -> gather-evaluation rounds
            if (!overflow) {
                int* wl = worklist[threadIdx.x >> 5][0];   // [kListCap][32], lane-major
                int cnt = 0;
                for (int k = 0; k < nF; ++k) {
                    const int v = F[k];
                    const float lb = node_lb2(T, s, v);
                    const bool need = normal && lb <= key_d2(best);
                    if (need) { wl[cnt * 32 + lane] = v - l_pad; ++cnt; }
                    if (__any_sync(FULL, cnt == kListCap) || k == nF - 1) {
                        int rounds = cnt;
#pragma unroll
                        for (int o = 16; o; o >>= 1) rounds = max(rounds, __shfl_xor_sync(FULL, rounds, o));
                        for (int q = 0; q < rounds; ++q) {
                            if (q < cnt) {
                                if (st) st->leaf();
                                eval_leaf<B>(T, nq, wl[q * 32 + lane], best, bpos);
                            }
                        }
                        cnt = 0;
                    }
                }
            }
            __syncwarp();
        }
        // ---- E: exact ballot DFS for outliers (or everyone after an overflow)
        const bool dfs_on = outlier || (overflow && normal);
        if (__any_sync(FULL, dfs_on)) ballot_dfs<B>(T, s, nq, dfs_on, best, bpos);
        if (active) qs.store(qi, best, bpos, s);
    }
}

}  // namespace cil
