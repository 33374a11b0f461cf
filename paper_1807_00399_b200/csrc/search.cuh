// search.cuh -- device side of the exact 1-NN search.
//
// Index (target.cu): target points sorted by 48-bit Morton key, grouped into leaves of B
// consecutive points (SoA blocks x[B], y[B], z[B], idx[B]), per-leaf boxes in an interleaved
// layout for the packed lower-bound test, and an implicit complete binary tree of AABBs over
// the leaves (node v has children 2v, 2v+1; leaves are nodes l_pad .. 2 l_pad - 1).
// The search itself is the warp-packet engine at the end of this file.
//
// Precision contract:
//  * the transformed query s = R p + t is computed in fp64 and carried as a double-float
//    pair (hi = fl32(s), lo = fl32(s - hi)), never materialised in fp32 alone;
//  * per candidate the difference is (s_hi - t) + s_lo in fp32 -- accurate to ~1 ulp of
//    |s - t| rather than of |s| -- and d^2 = fma(dx,dx, fma(dy,dy, dz*dz)) in fp32;
//  * the minimum is taken over the u64 key (bits(d^2) << 32) | original_index, which orders
//    by d^2 (non-negative IEEE floats order like their bit patterns) and breaks exact ties
//    by the lowest original index (R1);
//  * a box is pruned iff its lower bound lb^2 > the search threshold, where lb is computed
//    with the SAME rounded operations as the candidate differences, so by monotonicity of
//    IEEE rounding lb^2 <= d^2 of every point inside the box: pruning never drops a point
//    that could win (or tie) under the kernel's own arithmetic -- the search is exact.
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
// Two candidates per instruction with the sm_100 packed FP32 ops (FADD2, FFMA2, FMUL2):
// -dx = (t + (-s_hi)) + (-s_lo) is exactly the negation of (s_hi - t) + s_lo (IEEE rounding
// is sign-symmetric), so d^2 is bit-identical to cand_d2().
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

// d2[c] for the B candidates of a leaf (padding slots are +inf -> d2 = +inf)
template <int B>
__device__ __forceinline__ void leaf_d2(const TargetView& T, const NegQuery& q, int leaf, float (&d2)[B]) {
    constexpr int R = B / 4;
    const float4* blk = T.leafsoa + (size_t)leaf * (4 * R);
#pragma unroll
    for (int c = 0; c < R; ++c) {
        const float4 X = __ldg(blk + c), Y = __ldg(blk + R + c), Z = __ldg(blk + 2 * R + c);
        const float2 a = pair_d2(q, make_float2(X.x, X.y), make_float2(Y.x, Y.y), make_float2(Z.x, Z.y));
        const float2 b = pair_d2(q, make_float2(X.z, X.w), make_float2(Y.z, Y.w), make_float2(Z.z, Z.w));
        d2[4 * c + 0] = a.x; d2[4 * c + 1] = a.y; d2[4 * c + 2] = b.x; d2[4 * c + 3] = b.y;
    }
}

template <int B>
__device__ __forceinline__ float leaf_min(const float (&d2)[B]) {
    float m = d2[0];
#pragma unroll
    for (int c = 1; c < B; ++c) m = fminf(m, d2[c]);
    return m;
}

// lowest original index among the leaf's candidates at d2 == m1 (R1 tie rule)
template <int B>
__device__ __forceinline__ uint32_t leaf_argmin(const TargetView& T, int leaf, const float (&d2)[B], float m1) {
    const int* ids = reinterpret_cast<const int*>(T.leafsoa + (size_t)leaf * B + 3 * (B / 4));
    uint32_t imin = 0xffffffffu;
#pragma unroll
    for (int c = 0; c < B; ++c) {
        const uint32_t id = (uint32_t)__ldg(ids + c);
        imin = (d2[c] == m1 && id < imin) ? id : imin;
    }
    return imin;
}

// best <- min(best, key of the leaf's nearest candidate); CERT: sec <- the smallest leaf
// minimum of any OTHER leaf (the value that loses against the running best is pushed:
// sec <- min(sec, max(best_d2, m1)))
template <int B, bool CERT>
__device__ __forceinline__ void eval_leaf_seq(const TargetView& T, const NegQuery& q, int leaf,
                                              unsigned long long& best, float& sec) {
    float d2[B];
    leaf_d2<B>(T, q, leaf, d2);
    const float m1 = leaf_min<B>(d2);
    if (m1 <= key_d2(best)) {
        const unsigned long long k = make_key(m1, leaf_argmin<B>(T, leaf, d2, m1));
        // (k == best: the same point was already offered, e.g. by a neighbour lane -- not a loser)
        if (CERT && k != best) sec = fminf(sec, fmaxf(key_d2(best), m1));
        if (k < best) best = k;
    } else if (CERT) {
        sec = fminf(sec, m1);
    }
}

// work-item evaluation (any lane, for a query slot in shared memory): atomicMin on the
// query's best key; with CERT the key that loses is pushed into the leaf-level 2nd best
// (linearisable: every leaf minimum that is not the final one is pushed once it loses), and
// a leaf whose minimum is within the query's current threshold joins the query's candidate-
// leaf list (capacity kListLeaves; the minimum of a leaf that does not fit is kept in drop).
#ifndef CIL_RCAP
#define CIL_RCAP 8.0f         // outlier cap: a lane whose radius exceeds CIL_RCAP x the packet mean
#endif
#ifndef CIL_LIST_LEAVES
#define CIL_LIST_LEAVES 12
#endif
constexpr int kListLeaves = CIL_LIST_LEAVES;   // multiple of 4
struct CertSlots {
    unsigned* sec;       // leaf-level 2nd best (float bits)
    int* list;           // [kListLeaves] candidate leaves
    int* cnt;
    unsigned* drop;      // smallest leaf minimum that did not fit in the list (float bits)
    const float* thr;    // the query's current threshold
};

template <int B, bool CERT>
__device__ __forceinline__ void eval_leaf_item(const TargetView& T, const NegQuery& q, int leaf,
                                               unsigned long long* bestS, const CertSlots& cs) {
    float d2[B];
    leaf_d2<B>(T, q, leaf, d2);
    const float m1 = leaf_min<B>(d2);
    float push = m1;
    if (m1 <= key_d2(*(volatile unsigned long long*)bestS)) {
        const unsigned long long k = make_key(m1, leaf_argmin<B>(T, leaf, d2, m1));
        const unsigned long long old = atomicMin(bestS, k);
        push = old == k ? INFINITY : key_d2(old > k ? old : k);   // same point offered before: no loser
    }
    if (CERT) {
        if (__float_as_uint(push) < *(volatile unsigned*)cs.sec) atomicMin(cs.sec, __float_as_uint(push));
        if (m1 <= *(volatile const float*)cs.thr) {
            const int pos = atomicAdd(cs.cnt, 1);
            if (pos < kListLeaves) cs.list[pos] = leaf;
            else atomicMin(cs.drop, __float_as_uint(m1));
        }
    }
}

// Lower bound of cand_d2 over the leaf box, bit-identical to box_lb2 (the (lo, hi) pair of
// an axis goes through one FADD2: x.x = (lo - s_hi) - s_lo, -x.y = (s_hi - hi) + s_lo).
// lbox[2 leaf] = (lo.x, hi.x, lo.y, hi.y), lbox[2 leaf + 1] = (lo.z, hi.z, 0, 0).
__device__ __forceinline__ float leaf_lb2(const TargetView& T, const NegQuery& q, int leaf) {
    const float4 A = __ldg(T.lbox + 2 * (size_t)leaf), Z = __ldg(T.lbox + 2 * (size_t)leaf + 1);
    const float2 x = __fadd2_rn(__fadd2_rn(make_float2(A.x, A.y), q.hx), q.lx);
    const float2 y = __fadd2_rn(__fadd2_rn(make_float2(A.z, A.w), q.hy), q.ly);
    const float2 z = __fadd2_rn(__fadd2_rn(make_float2(Z.x, Z.y), q.hz), q.lz);
    const float gx = fmaxf(fmaxf(x.x, -x.y), 0.0f);
    const float gy = fmaxf(fmaxf(y.x, -y.y), 0.0f);
    const float gz = fmaxf(fmaxf(z.x, -z.y), 0.0f);
    return fmaf(gx, gx, fmaf(gy, gy, gz * gz));
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

// ---------------------------------------------------------------- warp-packet engine
// A warp takes 32 consecutive queries (one per lane; consecutive = spatially coherent for
// Morton- or scan-ordered inputs).
//   A. every lane evaluates its own hint leaf (warm-start match or cold Morton hint): a per-
//      lane search threshold thr_i = best d2 (with the certificate margin, see CERT below).
//   B. lanes whose radius is far above the packet mean are "outliers"; the others define the
//      packet box P = AABB of their balls B(s_i, sqrt(thr_i)) (conservatively inflated).
//   C. every target inside P has a Morton key in [code(P.lo), code(P.hi)] (the key is
//      monotone in each quantised coordinate and is computed by the same function), i.e. a
//      contiguous sorted range, bracketed by the coarse-cell table: the candidate leaves are
//      the leaves of that range whose box meets P -- tested directly (32 leaves per step)
//      when the range is short, else by a breadth-first walk (one child box per lane, ballot
//      compaction) from the lowest common ancestor of the range.
//   D. every lane tests every candidate leaf against its own ball (lb^2 <= thr); the needed
//      (leaf, query) pairs are appended, grouped by leaf, to a work list in shared memory.
//   E. the work list is evaluated 32 items per round (any lane takes any item, so the number
//      of rounds is sum/32, not the longest per-lane list; lanes of a round mostly share the
//      leaf and its loads); results merge through shared-memory atomicMin on the u64 keys.
//   F. outlier lanes (and whole packets whose frontier overflowed) finish with the exact
//      ballot DFS: a node is entered iff its lower bound is <= some active lane's threshold.
// Every lane therefore examines every leaf that can hold a target inside its ball: each
// lane's result is its exact nearest neighbour.
//
// CERT (cil_icp_run, SURVEY.md 8(a) a2 certified warm start, leaf form): the threshold is
// inflated to (sqrt(best) + g)^2 and every lane also keeps sec = the smallest leaf minimum
// of the evaluated leaves other than the winner's leaf L1.  Every target outside L1 is in an
// evaluated leaf (d2 >= sec) or in a leaf pruned against the threshold (d2 > thr), so
// d_out^2 >= min(sec, thr) and the nearest neighbour stays in L1 while the query moves less
// than (d_out - d1) / 2.
//
// Q supplies
//   __device__ int packets(int m), packet_base(int c)   (work unit c = queries base .. base+31)
//   __device__ bool load(int i, DF3& s, unsigned long long& init, int& hint_leaf)
//   __device__ void store(int i, unsigned long long best, float lb_out2)   (lb_out2 = 0: no certificate)
//   CERT: store(int i, best, lb_out2, const int* list, int cnt, float rS2) with the candidate-
//   leaf list (cnt leaves; every target outside them is at d2 >= rS2; cnt = 0: no list)
//   float skin  (CERT only: the threshold margin g of the query just loaded)
#ifndef CIL_FRONTIER_CAP
#define CIL_FRONTIER_CAP 256
#endif
#ifndef CIL_DIRECT_LEAVES
#define CIL_DIRECT_LEAVES 512
#endif
constexpr int kFrontierCap = CIL_FRONTIER_CAP;
#ifndef CIL_ITEM_CAP
#define CIL_ITEM_CAP 256
#endif
constexpr int kItemCap = CIL_ITEM_CAP;
#ifndef CIL_DGROUP
#define CIL_DGROUP 2
#endif
#ifndef CIL_TRACE_D
#define CIL_TRACE_D CIL_TRACE // (per-query item counts in that trace)
#endif
constexpr int kDGroup = CIL_DGROUP;      // frontier leaves tested per step of phase D
constexpr int kDirectLeaves = CIL_DIRECT_LEAVES;
#ifndef CIL_ENGINE_WARPS
#define CIL_ENGINE_WARPS 8
#endif
constexpr int kEngineWarps = CIL_ENGINE_WARPS;     // warps per block of the engine kernels (blockDim 32 x this)

// Independent per-lane exact DFS (nearest-child first, a subtree is entered iff its lower
// bound is <= the lane's current threshold), for outlier lanes, overflowed packets and
// sparse packets, whose lanes would otherwise drag each other through the union of their
// traversals.  The hint leaf (already evaluated in phase A) is skipped.  CERT: the leaf-level
// 2nd best and the candidate-leaf list are kept exactly as in the packet phases.
constexpr int kDfsStack = 32;

template <int B, bool CERT>
__device__ __forceinline__ void lane_dfs(const TargetView& T, const DF3& s, const NegQuery& nq, int skip,
                                         int skip2, float g, float cap2, unsigned long long& best, float& sec,
                                         int* lst, int* cnt, unsigned* drop) {
    int sv[kDfsStack];
    float slb[kDfsStack];
    int sp = 0;
    int v = 1;
    const int l_pad = T.l_pad;
    auto thr_of = [&]() {
        const float d = key_d2(best);
        if (g == 0.0f) return d;
        const float r = sqrtf(d) + g;
        return fmaxf(fminf(r * r, cap2), d);
    };
    while (true) {
        const float thr = thr_of();
        while (v < l_pad) {
            const int c = 2 * v;
            const float4* bx = T.box + 2 * (size_t)c;
            const float lb0 = box_lb2(s, __ldg(bx), __ldg(bx + 1));
            const float lb1 = box_lb2(s, __ldg(bx + 2), __ldg(bx + 3));
            const bool g0 = lb0 <= thr, g1 = lb1 <= thr;
            if (g0 && g1) {
                const bool r1 = lb1 < lb0;
                sv[sp] = r1 ? c : c + 1;
                slb[sp] = r1 ? lb0 : lb1;
                ++sp;
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
        if (v >= l_pad && v - l_pad != skip && v - l_pad != skip2) {
            const int leaf = v - l_pad;
            float d2[B];
            leaf_d2<B>(T, nq, leaf, d2);
            const float m1 = leaf_min<B>(d2);
            if (CERT) {
                sec = fminf(sec, fmaxf(key_d2(best), m1));
                if (m1 <= thr) {
                    if (*cnt < kListLeaves) lst[*cnt] = leaf;
                    else *drop = min(*drop, __float_as_uint(m1));
                    ++*cnt;
                }
            }
            if (m1 <= key_d2(best)) {
                const unsigned long long k = make_key(m1, leaf_argmin<B>(T, leaf, d2, m1));
                if (k < best) best = k;
            }
        }
        v = 0;
        while (sp > 0) {
            --sp;
            if (slb[sp] <= thr_of()) { v = sv[sp]; break; }
        }
        if (v == 0) break;
    }
}

// Ballot DFS for the outlier lanes of a coherent packet and for packets whose frontier
// overflowed: one traversal for the warp, a node is entered iff its lower bound is <= the
// threshold of some searching lane (lanes that are not searching use a negative threshold).
// Leaves are evaluated by the whole (converged) warp; only searching lanes keep the result.
template <int B, bool CERT>
__device__ __forceinline__ void ballot_dfs(const TargetView& T, const DF3& s, const NegQuery& nq, bool on,
                                           int skip, int skip2, float g, float cap2, unsigned long long& best, float& sec,
                                           int* lst, int* cnt, unsigned* drop) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int l_pad = T.l_pad;
    auto thr_of = [&]() {
        const float d = key_d2(best);
        if (!on) return -1.0f;
        if (g == 0.0f) return d;
        const float r = sqrtf(d) + g;
        return fmaxf(fminf(r * r, cap2), d);
    };
    int stk = 0, sp = 0, v = 1;
    while (true) {
        const float bd = thr_of();
        if (v >= l_pad) {
            const int leaf = v - l_pad;
            float d2[B];
            leaf_d2<B>(T, nq, leaf, d2);
            const float m1 = leaf_min<B>(d2);
            const uint32_t id = leaf_argmin<B>(T, leaf, d2, m1);
            if (on && leaf != skip && leaf != skip2) {
                if (CERT) {
                    sec = fminf(sec, fmaxf(key_d2(best), m1));
                    if (m1 <= bd) {
                        if (*cnt < kListLeaves) lst[*cnt] = leaf;
                        else *drop = min(*drop, __float_as_uint(m1));
                        ++*cnt;
                    }
                }
                const unsigned long long k = make_key(m1, id);
                if (k < best) best = k;
            }
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
            if (__any_sync(FULL, lb <= thr_of())) { v = cand; found = true; break; }
        }
        if (!found) break;
    }
}

__device__ __forceinline__ bool box_meets(float4 lo, float4 hi, float4 plo, float4 phi) {
    return lo.x <= phi.x && lo.y <= phi.y && lo.z <= phi.z && hi.x >= plo.x && hi.y >= plo.y && hi.z >= plo.z;
}

// first sorted index with key >= code (upper = false) or key > code (upper = true)
__device__ __forceinline__ int key_bound(const TargetView& T, unsigned long long code, bool upper) {
    const unsigned c = (unsigned)(code >> (3 * kMortonBits - T.coarse_bits));
    int lo = (int)__ldg(T.cell_first + c), hi = (int)__ldg(T.cell_first + c + 1);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const unsigned long long k = __ldg(T.keys + mid);
        if (upper ? k <= code : k < code) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Warp-cooperative bounds of the sorted key range [first key >= clo, first key > chi): each
// half-warp runs a 16-ary search (16 pivots split the bracket into 17 segments per step) inside
// the coarse cell of its code, so a bracket of n keys takes ~log17(n) dependent loads.
__device__ __forceinline__ void key_range_warp(const TargetView& T, unsigned long long clo, unsigned long long chi,
                                               int& i0, int& i1) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, h = lane >> 4, l = lane & 15;
    const bool upper = h != 0;
    const unsigned long long code = upper ? chi : clo;
    const unsigned c = (unsigned)(code >> (3 * kMortonBits - T.coarse_bits));
    int lo = (int)__ldg(T.cell_first + c), hi = (int)__ldg(T.cell_first + c + 1);   // answer in [lo, hi]
    while (true) {
        const int n = hi - lo;
        if (!__any_sync(FULL, n > 0)) break;
        int idx;
        if (n <= 16) idx = lo + l;
        else idx = lo + (int)(((long long)(l + 1) * n) / 17);
        bool pred = false;
        if (n > 0 && idx < hi) {
            const unsigned long long k = __ldg(T.keys + idx);
            pred = upper ? k <= code : k < code;
        }
        const unsigned t = __popc((__ballot_sync(FULL, pred) >> (16 * h)) & 0xffffu);
        if (n > 0) {
            if (n <= 16) {
                lo = hi = lo + (int)t;
            } else {
                const int a = t == 0 ? lo : lo + (int)(((long long)t * n) / 17) + 1;
                const int b = t == 16 ? hi : lo + (int)(((long long)(t + 1) * n) / 17);
                lo = a;
                hi = b;
            }
        }
    }
    i0 = __shfl_sync(FULL, lo, 0);
    i1 = __shfl_sync(FULL, lo, 16);
}

template <int B, bool CERT, class Q>
__device__ __forceinline__ void nn_packet_engine(const TargetView& T, Q& qs, int m, unsigned int* counter) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int l_pad = T.l_pad;
    __shared__ int sF[kEngineWarps][2][kFrontierCap];
    __shared__ int sItem[kEngineWarps][kItemCap];
    __shared__ float sQ[kEngineWarps][6][32];                 // -s_hi, -s_lo per lane
    __shared__ unsigned long long sBest[kEngineWarps][32];
    __shared__ unsigned sSec[kEngineWarps][32];
    __shared__ int sList[CERT ? kEngineWarps : 1][32][kListLeaves];
    __shared__ int sCnt[CERT ? kEngineWarps : 1][32];
    __shared__ unsigned sDrop[CERT ? kEngineWarps : 1][32];
    __shared__ float sThr[CERT ? kEngineWarps : 1][32];
    int* items = sItem[wid];
    const float stale2 = qs.stale2;                         // warm-hint distance^2 that counts as stale
    const int npk = qs.packets(m);
    while (true) {
        int c = 0;
        // (read before claiming: warps of an almost empty work list leave without an atomic)
        if (lane == 0) c = *(volatile unsigned*)counter >= (unsigned)npk ? npk : (int)atomicAdd(counter, 1u);
        c = __shfl_sync(FULL, c, 0);
        if (c >= npk) break;
        const int base = qs.packet_base(c);
        const int qi = base + lane;
        const bool tracing = CIL_TRACE && T.trace != nullptr;
        unsigned ck0 = tracing ? (unsigned)clock() : 0u, ckA = 0, ckB = 0, ckC = 0, ckD = 0;
        DF3 s;
        unsigned long long best = 0ull;
        int hint = -1;
        bool active = false;
        bool warm = false;
        float g = 0.0f;                                       // CERT: this lane's threshold margin
        if (qi < m) {
            active = qs.load(qi, s, best, hint);
            if constexpr (CERT) g = qs.skin;
            warm = hint >= 0;
            if (active && hint < 0) hint = coarse_hint_leaf(T, s);
        }
        if (!__any_sync(FULL, active)) continue;                 // nothing to search in this packet
        if (!active) { s.hx = s.hy = s.hz = 0.0f; s.lx = s.ly = s.lz = 0.0f; best = 0ull; hint = -1; }
        const float cap2 = key_d2(best);                      // the search bound (rho^2 / max^2 / inf)
        auto thr_of = [&](unsigned long long b) {
            const float d = key_d2(b);
            if (!CERT) return d;
            const float rr = sqrtf(d) + g;
            return fmaxf(fminf(rr * rr, cap2), d);
        };
        // ---- A
        float sec = INFINITY;                                 // CERT: leaf-level 2nd best
        int hint2 = -1;                                       // second hint leaf (cold), or -1
        if (active) {
            eval_leaf_seq<B, CERT>(T, neg_query(s), hint, best, sec);
            // a warm hint that went stale (large early ICP steps): also try the leaf that
            // follows the query's own Morton key, and keep the better of the two
            if (warm && key_d2(best) > stale2) {
                hint2 = coarse_hint_leaf(T, s);
                if (hint2 != hint) eval_leaf_seq<B, CERT>(T, neg_query(s), hint2, best, sec);
                else hint2 = -1;
            }
        }
        // A2: the packet's queries are spatial neighbours: try the matches of the lanes +-1, +-2
        // (an upper bound only -- their leaves are still evaluated in D/E if inside the ball)
        {
            const bool has = active && best != bound_key(cap2);
            float4 tb = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            if (has) tb = __ldg(&T.opts[key_idx(best)]);
            const uint32_t ib = has ? key_idx(best) : 0xffffffffu;
#pragma unroll
            for (int o = 1; o <= 2; ++o) {
#pragma unroll
                for (int dir = 0; dir < 2; ++dir) {
                    const float x = dir ? __shfl_down_sync(FULL, tb.x, o) : __shfl_up_sync(FULL, tb.x, o);
                    const float y = dir ? __shfl_down_sync(FULL, tb.y, o) : __shfl_up_sync(FULL, tb.y, o);
                    const float z = dir ? __shfl_down_sync(FULL, tb.z, o) : __shfl_up_sync(FULL, tb.z, o);
                    const uint32_t id = dir ? __shfl_down_sync(FULL, ib, o) : __shfl_up_sync(FULL, ib, o);
                    const bool in = dir ? lane + o < 32 : lane >= o;
                    if (active && in && id != 0xffffffffu) {
                        const unsigned long long k = make_key(cand_d2(s, make_float4(x, y, z, 0.0f)), id);
                        if (k < best) {
                            // CERT: the replaced best loses (the hint leaf's minimum, or a point of
                            // a leaf that D/E evaluates anyway -- an upper bound is conservative)
                            if (CERT && best != bound_key(cap2)) sec = fminf(sec, key_d2(best));
                            best = k;
                        }
                    }
                }
            }
        }
        float thr = active ? thr_of(best) : 0.0f;
        if (CERT) {
            // the hint leaf opens the candidate list (its minimum is the current best)
            // (a second hint leaf joins the list through its own slot)
            sList[wid][lane][0] = hint;
            sList[wid][lane][1] = hint2;
            sCnt[wid][lane] = (active && best != bound_key(cap2)) ? (hint2 >= 0 ? 2 : 1) : 0;
            sDrop[wid][lane] = __float_as_uint(INFINITY);
            sThr[wid][lane] = thr;
        }
        if (tracing) ckA = (unsigned)clock();
        // ---- B: outliers and the packet box
        const float r = active ? sqrtf(thr) : 0.0f;
        float rsum = r;
        int na = active ? 1 : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            rsum += __shfl_xor_sync(FULL, rsum, o);
            na += __shfl_xor_sync(FULL, na, o);
        }
        const float rcap = CIL_RCAP * rsum / (float)max(na, 1);
        bool normal = active && r <= rcap && r < INFINITY;
        const int dbg_mode = CIL_TRACE ? T.dbg_mode : 0;       // (diagnostic engine modes: trace builds)
        if (dbg_mode == 1) normal = false;
        if (dbg_mode == 2) normal = active && r < INFINITY;
        // an outlier (radius above the cap) joins the packet with its ball capped at rcap: if its
        // nearest neighbour lies within the cap the packet phases find it exactly, otherwise it
        // finishes with the ballot DFS
        const bool outlier = active && !normal;
        const bool capped = outlier && r < INFINITY && dbg_mode == 0;
        const float rcap2 = rcap * rcap;
        if (CERT && capped) sThr[wid][lane] = fminf(thr, rcap2);     // list appends stop at the cap
        const bool inP = normal || capped;
        const float rP = normal ? r : rcap;
        // inflate for the double-float offset and for rounding of s_hi -/+ r
        const float rx = rP * 1.000001f + fabsf(s.lx) + 1e-6f * fabsf(s.hx) + 1e-30f;
        const float ry = rP * 1.000001f + fabsf(s.ly) + 1e-6f * fabsf(s.hy) + 1e-30f;
        const float rz = rP * 1.000001f + fabsf(s.lz) + 1e-6f * fabsf(s.hz) + 1e-30f;
        float4 plo = make_float4(inP ? s.hx - rx : INFINITY, inP ? s.hy - ry : INFINITY,
                                 inP ? s.hz - rz : INFINITY, 0.0f);
        float4 phi = make_float4(inP ? s.hx + rx : -INFINITY, inP ? s.hy + ry : -INFINITY,
                                 inP ? s.hz + rz : -INFINITY, 0.0f);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            plo.x = fminf(plo.x, __shfl_xor_sync(FULL, plo.x, o));
            plo.y = fminf(plo.y, __shfl_xor_sync(FULL, plo.y, o));
            plo.z = fminf(plo.z, __shfl_xor_sync(FULL, plo.z, o));
            phi.x = fmaxf(phi.x, __shfl_xor_sync(FULL, phi.x, o));
            phi.y = fmaxf(phi.y, __shfl_xor_sync(FULL, phi.y, o));
            phi.z = fmaxf(phi.z, __shfl_xor_sync(FULL, phi.z, o));
        }
        // sparse packet (the balls fill a small part of P: e.g. an uncertified remainder
        // spread along the scan): every lane searches on its own
        float vb = inP ? 8.0f * rx * ry * rz : 0.0f;
#pragma unroll
        for (int o = 16; o; o >>= 1) vb += __shfl_xor_sync(FULL, vb, o);
        const bool sparse = (phi.x - plo.x) * (phi.y - plo.y) * (phi.z - plo.z) > 32.0f * vb;
        if (tracing) ckB = (unsigned)clock();
        bool overflow = false;
        int dbg_i0 = -1, dbg_i1 = -1, dbg_nF = -1, dbg_items = 0;
        if (!sparse && __any_sync(FULL, inP)) {
            int* F = sF[wid][0];
            int* G = sF[wid][1];
            // ---- C: Morton range of P -> leaf range -> candidate leaves (node ids)
            // (exact bounds by a warp-cooperative 16-ary search: lanes 0-15 find the first key
            // >= code(P.lo), lanes 16-31 the first key > code(P.hi), inside the coarse cells)
            int i0, i1;
            {
                const float4 Qz = __ldg(T.quant);
                const unsigned long long clo = morton_of(Qz, plo.x, plo.y, plo.z);
                const unsigned long long chi = morton_of(Qz, phi.x, phi.y, phi.z);
                key_range_warp(T, clo, chi, i0, i1);
            }
            int nF = 0;
            dbg_i0 = i0; dbg_i1 = i1;
            if (i1 > i0) {
                const int la = i0 / B, lb = (i1 - 1) / B;
                if (lb - la < kDirectLeaves) {
                    // 4 x 32 leaves per step, all box loads in flight together
                    for (int b0 = la; b0 <= lb; b0 += 128) {
                        bool hit[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int f = b0 + 32 * u + lane;
                            hit[u] = false;
                            if (f <= lb) {
                                const float4* bx = T.box + 2 * (size_t)(l_pad + f);
                                hit[u] = box_meets(__ldg(bx), __ldg(bx + 1), plo, phi);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const unsigned mk = __ballot_sync(FULL, hit[u]);
                            const int pos = nF + __popc(mk & lt);
                            if (hit[u] && pos < kFrontierCap) F[pos] = b0 + 32 * u + lane;
                            nF += __popc(mk);
                        }
                    }
                    if (nF > kFrontierCap) overflow = true;
                } else {
                    int a = l_pad + la;
                    const int k = 32 - __clz(a ^ (l_pad + lb));
                    a >>= k;
                    if (lane == 0) F[0] = a;
                    nF = 1;
                    __syncwarp();
                    for (int lev = 0; lev < k && nF > 0; ++lev) {
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
                            if (hit && pos < kFrontierCap) G[pos] = (lev == k - 1) ? c - l_pad : c;
                            nN += __popc(mk);
                        }
                        __syncwarp();
                        if (nN > kFrontierCap) { overflow = true; break; }
                        int* tmp = F; F = G; G = tmp;
                        nF = nN;
                    }
                    if (k == 0 && lane == 0) F[0] = a - l_pad;      // the range is one leaf
                }
            }
            __syncwarp();
            dbg_nF = nF;
            if (tracing) ckC = (unsigned)clock();
            // ---- D + E: per-lane need tests -> leaf-grouped work items -> shared rounds
            if (!overflow && nF > 0) {
                sQ[wid][0][lane] = -s.hx; sQ[wid][1][lane] = -s.hy; sQ[wid][2][lane] = -s.hz;
                sQ[wid][3][lane] = -s.lx; sQ[wid][4][lane] = -s.ly; sQ[wid][5][lane] = -s.lz;
                sBest[wid][lane] = best;
                if (CERT) sSec[wid][lane] = __float_as_uint(sec);
                __syncwarp();
                int nI = 0;
                // evaluate the collected items (32 per round) and refresh the lane thresholds
                auto flush = [&]() {
                    __syncwarp();
                    for (int r0 = 0; r0 < nI; r0 += 32) {
                        const int jj = r0 + lane;
                        if (jj < nI) {
                            const int it = items[jj];
                            const int q = it & 31;
                            NegQuery qq;
                            qq.hx = make_float2(sQ[wid][0][q], sQ[wid][0][q]);
                            qq.hy = make_float2(sQ[wid][1][q], sQ[wid][1][q]);
                            qq.hz = make_float2(sQ[wid][2][q], sQ[wid][2][q]);
                            qq.lx = make_float2(sQ[wid][3][q], sQ[wid][3][q]);
                            qq.ly = make_float2(sQ[wid][4][q], sQ[wid][4][q]);
                            qq.lz = make_float2(sQ[wid][5][q], sQ[wid][5][q]);
                            CertSlots cs;
                            if (CERT) {
                                cs.sec = &sSec[wid][q]; cs.list = sList[wid][q]; cs.cnt = &sCnt[wid][q];
                                cs.drop = &sDrop[wid][q]; cs.thr = &sThr[wid][q];
                            }
                            eval_leaf_item<B, CERT>(T, qq, it >> 5, &sBest[wid][q], cs);
                        }
                    }
                    __syncwarp();
                    nI = 0;
                    best = sBest[wid][lane];
                    if (CERT) sec = __uint_as_float(sSec[wid][lane]);
                    if (active) thr = thr_of(best);
                    if (CERT) sThr[wid][lane] = capped ? fminf(thr, rcap2) : thr;
                };
                // kDGroup candidate leaves per step: their box loads are in flight together
                for (int k = 0; k < nF; k += kDGroup) {
                    int f[kDGroup];
                    float lb[kDGroup];
#pragma unroll
                    for (int u = 0; u < kDGroup; ++u) f[u] = k + u < nF ? F[k + u] : -1;
#pragma unroll
                    for (int u = 0; u < kDGroup; ++u) lb[u] = f[u] >= 0 ? leaf_lb2(T, neg_query(s), f[u]) : INFINITY;
                    const float lim = capped ? fminf(thr, rcap2) : thr;
#pragma unroll
                    for (int u = 0; u < kDGroup; ++u) {
                        const bool need = inP && f[u] >= 0 && f[u] != hint && f[u] != hint2 && lb[u] <= lim;
                        const unsigned mk = __ballot_sync(FULL, need);
                        if (need) items[nI + __popc(mk & lt)] = (f[u] << 5) | lane;
                        nI += __popc(mk);
#if CIL_TRACE_D
                        if (tracing) dbg_items += need ? 1 : 0;
#endif
                    }
                    if (nI > kItemCap - 32 * kDGroup || (k + kDGroup >= nF && nI > 0)) flush();
                }
            }
        }
        if (tracing) { ckD = (unsigned)clock(); if (!ckC) ckC = ckD; }
        int* trace = CIL_TRACE ? T.trace : nullptr;
        if (trace && qi < m) {
            int* rec = trace + 16 * (size_t)qi;
            rec[0] = normal | (outlier << 1) | (overflow << 2) | (sparse << 3);
            rec[1] = __float_as_int(r);
            rec[2] = dbg_i0; rec[3] = dbg_i1; rec[4] = dbg_nF;
            rec[5] = __float_as_int(key_d2(best));
            rec[6] = dbg_items;
            rec[8] = (int)(ckA - ck0); rec[9] = (int)(ckB - ckA); rec[10] = (int)(ckC - ckB); rec[11] = (int)(ckD - ckC);
            rec[13] = qs.tag();
            rec[14] = __popc(__ballot_sync(__activemask(), active));
        }
        // ---- F: exact ballot DFS for outliers (or everyone after an overflow)
        // a capped lane whose match lies within its cap is done (every leaf reaching into the
        // cap ball was examined); its certificate bookkeeping stops at the cap
        const bool cap_done = capped && !sparse && !overflow && key_d2(best) <= rcap2;
        // sparse packet: independent per-lane DFS; outliers / overflow: ballot DFS
        const bool lane_on = sparse && inP;
        const bool ballot_on = (outlier && !cap_done && !(sparse && capped)) || (overflow && inP);
        {
            unsigned drop = 0u;
            int cnt = 0;
            int* lst = nullptr;
            if constexpr (CERT) { drop = sDrop[wid][lane]; cnt = sCnt[wid][lane]; lst = sList[wid][lane]; }
            if (lane_on) lane_dfs<B, CERT>(T, s, neg_query(s), hint, hint2, g, cap2, best, sec, lst, &cnt, &drop);
            if (__any_sync(FULL, ballot_on))
                ballot_dfs<B, CERT>(T, s, neg_query(s), ballot_on, hint, hint2, g, cap2, best, sec, lst, &cnt, &drop);
            if constexpr (CERT) { sDrop[wid][lane] = drop; sCnt[wid][lane] = cnt; }
            if (active && (lane_on || ballot_on)) thr = thr_of(best);
        }
        if (trace && qi < m) {
            trace[16 * (size_t)qi + 7] = __float_as_int(key_d2(best));
            trace[16 * (size_t)qi + 12] = (int)((unsigned)clock() - ckD);
        }
        if (active) {
            // targets outside the evaluated leaves are beyond the final threshold
            const bool cert_ok = CERT;
            const float thr_done = cap_done ? fminf(thr, rcap2) : thr;   // what was examined
            const float lb_out2 = cert_ok ? fminf(sec, thr_done) : 0.0f;
            if constexpr (CERT) {
                // candidate-leaf list: every target outside it is beyond min(thr, drop)
                const int cnt = cert_ok ? min(sCnt[wid][lane], kListLeaves) : 0;
                const float rS2 = fminf(thr_done, __uint_as_float(sDrop[wid][lane]));
                qs.store(qi, best, lb_out2, sList[wid][lane], cnt, rS2);
            } else {
                qs.store(qi, best, lb_out2);
            }
        }
        __syncwarp();
    }
}

}  // namespace cil
