// grid.cuh -- device side of the exact 1-NN search over the uniform grid (SURVEY.md 8(a) row
// a2; BASELINE.json north_star (2) "a uniform grid ... built by a device radix sort plus a
// cell-offset scan ... chosen by measurement"; index_kind CIL_INDEX_GRID, built by grid.cu).
//
// One query per thread.  The search visits shells of cells around the query's own cell:
// shell r = the cells at Chebyshev distance r, the first step being the whole 3 x 3 x 3 block
// (shells 0 and 1) as nine contiguous x-row ranges of the x-major cell order.  A row (a cell
// of a larger shell) is evaluated unless its lower bound exceeds the best d^2 so far (ties are
// never pruned); after shell r every target outside the
// searched block lies beyond its faces, so the search stops as soon as best < (gap to the
// nearest face not on the grid boundary)^2, or when the block covers the grid.  Queries still
// unresolved after kGridShells shells finish with the exact per-lane BVH DFS (the BVH is
// always built), starting from the best found so far.
//
// Exactness under the kernel's own arithmetic (the same argument as search.cuh):
//  * every point of cell c lies in [lo + c h - eps, lo + (c + 1) h + eps] (GridDesc::eps
//    bounds the rounding of the build's cell assignment); cells on the grid boundary extend
//    to infinity (the assignment clamps);
//  * a gap to such a slab is computed as max((a - s_hi) - s_lo, (s_hi - b) + s_lo, 0), the
//    candidate difference as (s_hi - t) + s_lo: by monotonicity of IEEE rounding (and its
//    sign symmetry) |dx| >= gap for every point of the slab, so the fma chain of the lower
//    bound never exceeds the candidate's d^2, and fl(gap^2) never exceeds it either;
//  * the minimum is taken over the u64 key (bits(d^2) << 32) | original index (R1 ties).
#pragma once

#include "search.cuh"

namespace cil {

constexpr int kGridShells = 2;      // shells searched on the grid before the BVH fallback
#ifndef CIL_GRID_W
#define CIL_GRID_W 4                // candidate loads in flight per step of a row scan
#endif

__device__ __forceinline__ float grid_face_lo(int c, float lo, float h, float eps) {
    return c <= 0 ? -INFINITY : fmaf((float)c, h, lo) - eps;
}
__device__ __forceinline__ float grid_face_hi(int c, int n, float lo, float h, float eps) {
    return c >= n - 1 ? INFINITY : fmaf((float)(c + 1), h, lo) + eps;
}
// gap of the double-float coordinate (sh, sl) to the slab [a, b] (see the header comment)
__device__ __forceinline__ float grid_gap(float sh, float sl, float a, float b) {
    return fmaxf(fmaxf((a - sh) - sl, (sh - b) + sl), 0.0f);
}
__device__ __forceinline__ int grid_cell1(float x, float lo, float inv_h, int n) {
    const float f = floorf((x - lo) * inv_h);
    // (NaN and out-of-range coordinates clamp to the boundary cells)
    return f >= (float)(n - 1) ? n - 1 : (f >= 0.0f ? (int)f : 0);
}

// Exact nearest neighbour of s among the targets with d^2 <= key_d2(best) (inclusive), as the
// u64 key; best enters as bound_key(bound2) (or a better key already known).  DF = false when
// s_lo is zero (untransformed queries): the same values with one FADD less per coordinate.
template <int B, bool DF>
__device__ __forceinline__ unsigned long long grid_search(const TargetView& T, const DF3& s, unsigned long long best) {
    const GridDesc* G = T.gdesc;
    const float4 lh = __ldg(&G->lo_h);
    const float4 ie = __ldg(&G->inv_eps);
    const int4 dm = __ldg(&G->dims);
    const float h = lh.w, inv_h = ie.x, eps = ie.y;
    const int nx = dm.x, ny = dm.y, nz = dm.z;
    const int cx = grid_cell1(s.hx, lh.x, inv_h, nx);
    const int cy = grid_cell1(s.hy, lh.y, inv_h, ny);
    const int cz = grid_cell1(s.hz, lh.z, inv_h, nz);
    const float slx = DF ? s.lx : 0.0f, sly = DF ? s.ly : 0.0f, slz = DF ? s.lz : 0.0f;
    bool done = false;
    // candidates of the sorted range [a, b) (cells in x-major order: consecutive x cells of a
    // row are one contiguous range)
    // (four loads in flight per step; slots past b read a +inf point: key (inf, ~0), never better)
    auto scan = [&](uint32_t a, uint32_t b) {
        constexpr int W = CIL_GRID_W;
        for (uint32_t j = a; j < b; j += W) {
            float4 t[W];
#pragma unroll
            for (int u = 0; u < W; ++u)
                t[u] = j + u < b ? __ldg(T.gpts + j + u) : make_float4(INFINITY, INFINITY, INFINITY, __uint_as_float(~0u));
#pragma unroll
            for (int u = 0; u < W; ++u) {
                const float dx = DF ? (s.hx - t[u].x) + s.lx : s.hx - t[u].x;
                const float dy = DF ? (s.hy - t[u].y) + s.ly : s.hy - t[u].y;
                const float dz = DF ? (s.hz - t[u].z) + s.lz : s.hz - t[u].z;
                const unsigned long long k = make_key(fmaf(dx, dx, fmaf(dy, dy, dz * dz)), __float_as_uint(t[u].w));
                best = k < best ? k : best;
            }
        }
    };
    for (int r = 1; r <= kGridShells && !done; ++r) {
        const int z0 = max(cz - r, 0), z1 = min(cz + r, nz - 1);
        const int y0 = max(cy - r, 0), y1 = min(cy + r, ny - 1);
        for (int z = z0; z <= z1; ++z) {
            const float gz = grid_gap(s.hz, slz, grid_face_lo(z, lh.z, h, eps), grid_face_hi(z, nz, lh.z, h, eps));
            const bool zedge = z == cz - r || z == cz + r;
            for (int y = y0; y <= y1; ++y) {
                const float gy = grid_gap(s.hy, sly, grid_face_lo(y, lh.y, h, eps), grid_face_hi(y, ny, lh.y, h, eps));
                const float lrow = fmaf(gy, gy, gz * gz);
                if (lrow > key_d2(best)) continue;
                const uint32_t* rowp = T.gstart + ((size_t)z * ny + y) * nx;
                const bool full = zedge || y == cy - r || y == cy + r;   // a face row of the shell
                if (r == 1 || full) {
                    // shell 1 = the whole 3 x 3 x 3 block (shell 0 included), a face row of a
                    // larger shell is new in full: one contiguous range per row; the query's
                    // x lies inside the row's x extent for r = 1 (its lower bound is lrow)
                    const int xa = max(cx - r, 0), xb = min(cx + r, nx - 1);
                    scan(__ldg(rowp + xa), __ldg(rowp + xb + 1));
                } else {
                    // an inner row of shell r >= 2: only its two end cells are new
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int x = e ? cx + r : cx - r;
                        if (x < 0 || x >= nx) continue;
                        const float gx = grid_gap(s.hx, slx, grid_face_lo(x, lh.x, h, eps), grid_face_hi(x, nx, lh.x, h, eps));
                        if (fmaf(gx, gx, lrow) > key_d2(best)) continue;
                        scan(__ldg(rowp + x), __ldg(rowp + x + 1));
                    }
                }
            }
        }
        // every target outside the searched block is beyond one of its inner faces
        float D2 = INFINITY;
        if (cx - r > 0) { const float g = fmaxf((s.hx - grid_face_hi(cx - r - 1, nx, lh.x, h, eps)) + slx, 0.0f); D2 = fminf(D2, g * g); }
        if (cx + r < nx - 1) { const float g = fmaxf((grid_face_lo(cx + r + 1, lh.x, h, eps) - s.hx) - slx, 0.0f); D2 = fminf(D2, g * g); }
        if (cy - r > 0) { const float g = fmaxf((s.hy - grid_face_hi(cy - r - 1, ny, lh.y, h, eps)) + sly, 0.0f); D2 = fminf(D2, g * g); }
        if (cy + r < ny - 1) { const float g = fmaxf((grid_face_lo(cy + r + 1, lh.y, h, eps) - s.hy) - sly, 0.0f); D2 = fminf(D2, g * g); }
        if (cz - r > 0) { const float g = fmaxf((s.hz - grid_face_hi(cz - r - 1, nz, lh.z, h, eps)) + slz, 0.0f); D2 = fminf(D2, g * g); }
        if (cz + r < nz - 1) { const float g = fmaxf((grid_face_lo(cz + r + 1, lh.z, h, eps) - s.hz) - slz, 0.0f); D2 = fminf(D2, g * g); }
        const bool all = cx - r <= 0 && cx + r >= nx - 1 && cy - r <= 0 && cy + r >= ny - 1 && cz - r <= 0 && cz + r >= nz - 1;
        done = all || key_d2(best) < D2;
    }
    if (!done) {
        // far from every target (relative to the cell size): the exact BVH DFS from the best so far
        const NegQuery nq = neg_query(s);
        float sec = INFINITY;
        lane_dfs<B, false>(T, s, nq, -1, -1, 0.0f, key_d2(best), best, sec, nullptr, nullptr, nullptr);
    }
    return best;
}

}  // namespace cil
