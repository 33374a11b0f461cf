// search.cuh -- device side of the exact 1-NN search.
//
// Precision contract:
//  * the transformed query s = R p + t is computed in fp64 and carried as a double-float
//    pair (hi = fl32(s), lo = fl32(s - hi)), never materialised in fp32 alone;
//  * per candidate the difference is (s_hi - t) + s_lo in fp32 -- exact-ish to ~1 ulp of
//    |s - t| rather than of |s| -- and d^2 = fma(dx,dx, fma(dy,dy, dz*dz)) in fp32;
//  * the minimum is taken over the u64 key (bits(d^2) << 32) | original_index, which orders
//    by d^2 (non-negative IEEE floats order like their bit patterns) and breaks exact ties
//    by the lowest original index (R1);
//  * a BVH node is pruned iff its lower bound lb^2 > best d^2, where lb is computed with the
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

// Evaluate candidate at sorted position j; keep the best key and its sorted position.
__device__ __forceinline__ void offer(const DF3& s, float4 t, int j, unsigned long long& best, int& bpos) {
    unsigned long long k = make_key(cand_d2(s, t), (uint32_t)__float_as_int(t.w));
    if (k < best) { best = k; bpos = j; }
}

constexpr int kMaxDepth = 32;

// Exact nearest neighbour of s over the implicit BVH: nearest-child-first depth-first
// traversal with a short stack; `best`/`bpos` carry in an initial bound (bound_key or a
// warm-start candidate) and carry out the result.
template <int B>
__device__ __forceinline__ void bvh_nearest(const TargetView& T, const DF3& s,
                                            unsigned long long& best, int& bpos) {
    int stk_v[kMaxDepth];
    float stk_lb[kMaxDepth];
    int sp = 0;
    int v = 1;
    const int l_pad = T.l_pad;
    while (true) {
        if (v >= l_pad) {
            const int beg = (v - l_pad) * B;
            const int cnt = min(B, T.n - beg);
            float4 t[B];
#pragma unroll
            for (int q = 0; q < B; ++q)
                if (q < cnt) t[q] = __ldg(T.pts + beg + q);
#pragma unroll
            for (int q = 0; q < B; ++q)
                if (q < cnt) offer(s, t[q], beg + q, best, bpos);
        } else {
            const int c = 2 * v;
            const float4* bx = T.box + 2 * c;
            float4 lo0 = __ldg(bx + 0), hi0 = __ldg(bx + 1), lo1 = __ldg(bx + 2), hi1 = __ldg(bx + 3);
            float lb0 = box_lb2(s, lo0, hi0);
            float lb1 = box_lb2(s, lo1, hi1);
            const float bd = key_d2(best);
            const bool g0 = lb0 <= bd, g1 = lb1 <= bd;
            if (g0 && g1) {
                const bool right_first = lb1 < lb0;
                stk_v[sp] = right_first ? c : c + 1;
                stk_lb[sp] = right_first ? lb0 : lb1;
                ++sp;
                v = right_first ? c + 1 : c;
                continue;
            }
            if (g0) { v = c; continue; }
            if (g1) { v = c + 1; continue; }
        }
        const float bd = key_d2(best);
        while (sp > 0 && stk_lb[sp - 1] > bd) --sp;
        if (sp == 0) break;
        --sp;
        v = stk_v[sp];
    }
}

}  // namespace cil
