// target.cu -- cil_target_build: the GPU spatial index over the target cloud
// (BASELINE.json north_star subsystem (2): "a GPU spatial index over
// the target, such as ... Morton-sorted cells built by a device radix sort plus a
// cell-offset scan ... chosen by measurement").
//
// Pipeline (all hand-written kernels, one stream, no host synchronisation):
//   K1a bbox partials -> K1b bbox final -> K1c 48-bit Morton key per point
//   K2  stable LSD radix sort of (key, index) (6 passes x 8 bits: histogram, 3-phase scan,
//       stable warp-ranked scatter)
//   K4  gather: sorted float4 (x, y, z, orig index) points (build temp) and the original-order
//       float4 points (x, y, z, sorted position) and normals the ICP kernels gather from
//   K5  leaf AABBs (leaf_size consecutive sorted points) and SoA leaf blocks, then internal
//       AABBs of an implicit complete binary tree (node v has children 2v, 2v+1), 8 levels per
//       shared-memory pass; K6 coarse-cell table (first sorted index of every coarse cell).
#include "internal.cuh"
#include "search.cuh"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>

namespace cil {
namespace {

constexpr int kThreads = 256;

// ------------------------------------------------------------------ bbox
__global__ void bbox_partial_kernel(const float* __restrict__ p, int n, float* __restrict__ part) {
    pdl_entry();
    float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            float c = p[3 * (size_t)i + a];
            mn[a] = fminf(mn[a], c);
            mx[a] = fmaxf(mx[a], c);
        }
    }
    __shared__ float s[6][kThreads / 32];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o; o >>= 1) {
            mn[a] = fminf(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = fmaxf(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) { s[a][w] = mn[a]; s[3 + a][w] = mx[a]; }
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        float v = s[threadIdx.x][0];
        for (int k = 1; k < kThreads / 32; ++k)
            v = threadIdx.x < 3 ? fminf(v, s[threadIdx.x][k]) : fmaxf(v, s[threadIdx.x][k]);
        part[6 * blockIdx.x + threadIdx.x] = v;
    }
}

// quant = (min.x, min.y, min.z, cells per unit); one block of kThreads
__global__ void bbox_final_kernel(const float* __restrict__ part, int nblk, float4* __restrict__ quant) {
    pdl_entry();
    float mn[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    for (int b = threadIdx.x; b < nblk; b += blockDim.x)
        for (int a = 0; a < 3; ++a) {
            mn[a] = fminf(mn[a], part[6 * b + a]);
            mx[a] = fmaxf(mx[a], part[6 * b + 3 + a]);
        }
    __shared__ float sm[6][kThreads / 32];
#pragma unroll
    for (int a = 0; a < 3; ++a)
        for (int o = 16; o; o >>= 1) {
            mn[a] = fminf(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = fmaxf(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0)
        for (int a = 0; a < 3; ++a) { sm[a][w] = mn[a]; sm[3 + a][w] = mx[a]; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < kThreads / 32; ++k)
            for (int a = 0; a < 3; ++a) { sm[a][0] = fminf(sm[a][0], sm[a][k]); sm[3 + a][0] = fmaxf(sm[3 + a][0], sm[3 + a][k]); }
        const float ext = fmaxf(fmaxf(sm[3][0] - sm[0][0], sm[4][0] - sm[1][0]), sm[5][0] - sm[2][0]);
        const float cells = (float)((1 << kMortonBits) - 1);
        *quant = make_float4(sm[0][0], sm[1][0], sm[2][0], ext > 0.0f ? cells / ext : 0.0f);
        quant[1] = make_float4(sm[3][0], sm[4][0], sm[5][0], 0.0f);      // the maximum (grid.cu)
    }
}

__global__ void morton_kernel(const float* __restrict__ p, int n, const float4* __restrict__ quant,
                              unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals) {
    pdl_entry();
    const float4 Q = *quant;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        keys[i] = morton_of(Q, p[3 * (size_t)i], p[3 * (size_t)i + 1], p[3 * (size_t)i + 2]);
        vals[i] = (uint32_t)i;
    }
}

// ------------------------------------------------------------------ radix sort (stable LSD)
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kSortWarps = kThreads / 32;
#ifndef CIL_SORT_IPW
#define CIL_SORT_IPW 128
#endif
constexpr int kItemsPerWarp = CIL_SORT_IPW;                       // 4 rounds of 32 (tile 1024: C4 build 0.459 -> 0.424 ms; 2048: 0.422, 4096: 0.459, 8192: 0.486)
// Small inputs are launch- and latency-bound (a 65,536-key pass at 4096 keys per block is 16
// blocks of sequential rounds): their tile shrinks (down to one round per warp) until the pass
// has up to kSmallBlocks blocks, which also keeps the digit x tile table within the one-block scan.
#ifndef CIL_SMALL_TILES
#define CIL_SMALL_TILES 1
#endif
#ifndef CIL_SMALL_BLOCKS
#define CIL_SMALL_BLOCKS 64
#endif
constexpr int kSmallBlocks = CIL_SMALL_BLOCKS;       // 64 x 256 digits = the one-block scan's 16,384
// items per warp of a sort over n keys (32 .. 512, a power of two)
inline int sort_ipw(int n) {
    int ipw = kItemsPerWarp;
#if CIL_SMALL_TILES
    while (ipw > 32 && ((int64_t)n + (kSortWarps * ipw / 2) - 1) / (kSortWarps * ipw / 2) <= kSmallBlocks) ipw >>= 1;
#endif
    return ipw;
}
inline int sort_blocks(int n) { const int tile = kSortWarps * sort_ipw(n); return std::max(1, (n + tile - 1) / tile); }
// programmatic dependent launch for the build / ordering pipelines of inputs up to this size
// (dozens of short kernels: launch gaps dominate; at 2M points it measured slower)
#ifndef CIL_PDL_MAX_N
#define CIL_PDL_MAX_N (1 << 15)
#endif
inline bool pipeline_pdl(int64_t n) { return n <= (int64_t)CIL_PDL_MAX_N; }

__device__ __forceinline__ int digit_of(unsigned long long k, int shift) { return (int)((k >> shift) & (kRadix - 1)); }

// hist[d * nblk + b] = number of keys with digit d in tile b
__global__ void radix_hist_kernel(const unsigned long long* __restrict__ keys, int n, int shift,
                                  uint32_t* __restrict__ hist, int nblk, int ipw) {
    pdl_entry();
    __shared__ uint32_t h[kRadix];
    for (int d = threadIdx.x; d < kRadix; d += blockDim.x) h[d] = 0;
    __syncthreads();
    const int tile = kSortWarps * ipw;
    const int base = blockIdx.x * tile;
    for (int i = threadIdx.x; i < tile; i += blockDim.x) {
        int g = base + i;
        if (g < n) atomicAdd(&h[digit_of(keys[g], shift)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += blockDim.x) hist[(size_t)d * nblk + blockIdx.x] = h[d];
}

// stable scatter: within a tile, warp w owns keys [w*ipw, (w+1)*ipw) processed in rounds of 32
__global__ void radix_scatter_kernel(const unsigned long long* __restrict__ kin, const uint32_t* __restrict__ vin,
                                     unsigned long long* __restrict__ kout, uint32_t* __restrict__ vout,
                                     int n, int shift, const uint32_t* __restrict__ offs, int nblk, int ipw) {
    pdl_entry();
    __shared__ uint32_t cnt[kSortWarps][kRadix];   // per-warp digit counts, then offsets
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    for (int d = l; d < kRadix; d += 32) cnt[w][d] = 0;
    __syncwarp();
    const int wbase = blockIdx.x * kSortWarps * ipw + w * ipw;
    const unsigned lt_mask = (1u << l) - 1u;
    // pass 1: per-warp digit histogram
    for (int r = 0; r < ipw; r += 32) {
        int g = wbase + r + l;
        bool ok = g < n;
        int d = ok ? digit_of(kin[g], shift) : -1;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        if (ok && (peers & lt_mask) == 0) cnt[w][d] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // offsets: global base of (digit, tile) + counts of lower warps in this tile
    for (int d = threadIdx.x; d < kRadix; d += blockDim.x) {
        uint32_t run = offs[(size_t)d * nblk + blockIdx.x];
        for (int k = 0; k < kSortWarps; ++k) {
            uint32_t c = cnt[k][d];
            cnt[k][d] = run;
            run += c;
        }
    }
    __syncthreads();
    // pass 2: scatter in position order
    for (int r = 0; r < ipw; r += 32) {
        int g = wbase + r + l;
        bool ok = g < n;
        unsigned long long k = ok ? kin[g] : 0ull;
        int d = ok ? digit_of(k, shift) : -1;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        if (ok) {
            uint32_t dst = cnt[w][d] + __popc(peers & lt_mask);
            kout[dst] = k;
            vout[dst] = vin[g];
        }
        __syncwarp();
        if (ok && (peers & lt_mask) == 0) cnt[w][d] += __popc(peers);
        __syncwarp();
    }
}

// ------------------------------------------------------------------ gather + tree
// sorted points (build temp: x, y, z, orig index) and the ORIGINAL-order copies the ICP
// kernels gather from: opts[o] = (x, y, z, sorted position), onrm[o] = (nx, ny, nz, 0)
__global__ void gather_kernel(const float* __restrict__ p, const float* __restrict__ nrm, int n,
                              const uint32_t* __restrict__ perm, float4* __restrict__ spts,
                              float4* __restrict__ opts, float4* __restrict__ onrm) {
    pdl_entry();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t o = perm[i];
        const float x = p[3 * (size_t)o], y = p[3 * (size_t)o + 1], z = p[3 * (size_t)o + 2];
        spts[i] = make_float4(x, y, z, __int_as_float((int)o));
        opts[o] = make_float4(x, y, z, __int_as_float(i));
        if (onrm) onrm[o] = make_float4(nrm[3 * (size_t)o], nrm[3 * (size_t)o + 1], nrm[3 * (size_t)o + 2], 0.0f);
    }
}

__global__ void leaf_box_kernel(const float4* __restrict__ pts, int n, int B, int l_pad, float4* __restrict__ box,
                                int n_leaves, float4* __restrict__ lbox) {
    pdl_entry();
    for (int leaf = blockIdx.x * blockDim.x + threadIdx.x; leaf < l_pad; leaf += gridDim.x * blockDim.x) {
        float4 lo = make_float4(INFINITY, INFINITY, INFINITY, 0.0f);
        float4 hi = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.0f);
        const int beg = leaf * B, end = min(beg + B, n);
        for (int j = beg; j < end; ++j) {
            float4 t = pts[j];
            lo.x = fminf(lo.x, t.x); lo.y = fminf(lo.y, t.y); lo.z = fminf(lo.z, t.z);
            hi.x = fmaxf(hi.x, t.x); hi.y = fmaxf(hi.y, t.y); hi.z = fmaxf(hi.z, t.z);
        }
        const size_t v = (size_t)l_pad + leaf;
        box[2 * v] = lo;
        box[2 * v + 1] = hi;
        if (leaf < n_leaves) {
            lbox[2 * (size_t)leaf] = make_float4(lo.x, hi.x, lo.y, hi.y);
            lbox[2 * (size_t)leaf + 1] = make_float4(lo.z, hi.z, 0.0f, 0.0f);
        }
    }
}

// SoA leaf blocks: leaf L holds rows x[B], y[B], z[B], idx[B]; padding slots get +inf / ~0
__global__ void leaf_soa_kernel(const float4* __restrict__ pts, int n, int B, int64_t n_leaves, float* __restrict__ soa) {
    pdl_entry();
    const int64_t total = n_leaves * B;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t leaf = g / B;
        const int q = (int)(g % B);
        float4 t = g < n ? pts[g] : make_float4(INFINITY, INFINITY, INFINITY, __int_as_float(-1));
        float* blk = soa + leaf * 4 * B;
        blk[q] = t.x;
        blk[B + q] = t.y;
        blk[2 * B + q] = t.z;
        blk[3 * B + q] = t.w;
    }
}

// cell_first[c] = first sorted index whose key >> shift >= c, for c in [0, ncell] (binary search)
__global__ void cell_first_kernel(const unsigned long long* __restrict__ keys, int n, int shift, uint32_t ncell,
                                  uint32_t* __restrict__ cell_first) {
    pdl_entry();
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= (int64_t)ncell;
         c += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = (unsigned long long)c << shift;
        int lo = 0, hi = n;                    // first index with keys[i] >= key
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (keys[mid] < key) lo = mid + 1; else hi = mid;
        }
        cell_first[c] = (uint32_t)lo;
    }
}

// Internal node boxes, 8 levels per pass: block b reduces nodes [first + 256 b, first + 256 (b+1))
// of the current bottom level up `lv` levels, through shared memory.
constexpr int kPassNodes = 256;
__global__ void tree_pass_kernel(float4* __restrict__ box, int first, int lv) {
    pdl_entry();
    __shared__ float4 slo[kPassNodes], shi[kPassNodes];
    const int t = threadIdx.x;
    const int width = min(kPassNodes, first);          // nodes per block at the bottom level
    const int v0 = first + blockIdx.x * width;
    if (t < width) { slo[t] = box[2 * (size_t)(v0 + t)]; shi[t] = box[2 * (size_t)(v0 + t) + 1]; }
    __syncthreads();
    int cnt = width;
    for (int j = 1; j <= lv; ++j) {
        cnt >>= 1;
        float4 lo, hi;
        if (t < cnt) {
            const float4 l0 = slo[2 * t], l1 = slo[2 * t + 1], h0 = shi[2 * t], h1 = shi[2 * t + 1];
            lo = make_float4(fminf(l0.x, l1.x), fminf(l0.y, l1.y), fminf(l0.z, l1.z), 0.0f);
            hi = make_float4(fmaxf(h0.x, h1.x), fmaxf(h0.y, h1.y), fmaxf(h0.z, h1.z), 0.0f);
        }
        __syncthreads();
        if (t < cnt) {
            slo[t] = lo; shi[t] = hi;
            const size_t v = (size_t)(v0 >> j) + t;
            box[2 * v] = lo;
            box[2 * v + 1] = hi;
        }
        __syncthreads();
    }
}

inline int grid_for(int64_t work, int threads = kThreads) {
    int64_t b = (work + threads - 1) / threads;
    int cap = sm_count() * 8;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, cap));
}

// src_sorted[k] = src[perm[k]] (packed xyz)
__global__ void gather_xyz_kernel(const float* __restrict__ p, const uint32_t* __restrict__ perm, int n,
                                  float* __restrict__ out) {
    pdl_entry();
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const size_t o = perm[k];
        out[3 * (size_t)k] = p[3 * o];
        out[3 * (size_t)k + 1] = p[3 * o + 1];
        out[3 * (size_t)k + 2] = p[3 * o + 2];
    }
}

// Mean log path length of the 32-point packets of two orders of the same set (a: the caller's
// order, b: Morton order): per-block partials, the last block (ticket) adds them in a fixed
// order and keeps the caller's order (writes perm = identity, sorted = the caller's points)
// unless the Morton order is clearly more coherent.  Deterministic run to run.  (Measured:
// scan-ordered LiDAR and depth frames search faster in their scan order even though Morton
// packets have slightly shorter paths; random-order samples gain up to 10x from the sort.)
#ifndef CIL_EXT_BLOCKS
#define CIL_EXT_BLOCKS 592     // (4 per SM; 256 measured 0.2 % slower on the C4 run, 1184 equal)
#endif
constexpr int kExtBlocks = CIL_EXT_BLOCKS;
// path length of a 32-point packet, sum |p_{i+1} - p_i| (rotation invariant): ~ the arc length
// for a scan line, much more for a packet that zigzags between scan lines or jumps around
__device__ __forceinline__ float packet_diag(const float* p, int base, int n) {
    const int lane = threadIdx.x & 31;
    const int i = base + lane;
    const bool ok = i < n;
    const float x = ok ? p[3 * (size_t)i] : 0.0f, y = ok ? p[3 * (size_t)i + 1] : 0.0f, z = ok ? p[3 * (size_t)i + 2] : 0.0f;
    const float xn = __shfl_down_sync(0xffffffffu, x, 1), yn = __shfl_down_sync(0xffffffffu, y, 1),
                zn = __shfl_down_sync(0xffffffffu, z, 1);
    float d = (lane < 31 && i + 1 < n) ? sqrtf((xn - x) * (xn - x) + (yn - y) * (yn - y) + (zn - z) * (zn - z)) : 0.0f;
#pragma unroll
    for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    return d;
}

__global__ void __launch_bounds__(kThreads)
order_choice_kernel(const float* __restrict__ a, const float* __restrict__ b, int n, double* __restrict__ part,
                    unsigned* __restrict__ ticket, int* __restrict__ keep_caller) {
    pdl_entry();
    __shared__ double sa[kThreads / 32], sb[kThreads / 32];
    __shared__ int last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int npk = (n + 31) / 32;
    double ea = 0.0, eb = 0.0;
    for (int pk = blockIdx.x * (kThreads / 32) + warp; pk < npk; pk += gridDim.x * (kThreads / 32)) {
        ea += (double)__logf(packet_diag(a, 32 * pk, n) + 1e-30f);     // (fp32 log: a heuristic, deterministic)
        eb += (double)__logf(packet_diag(b, 32 * pk, n) + 1e-30f);
    }
    if (lane == 0) { sa[warp] = ea; sb[warp] = eb; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double ta = 0.0, tb = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) { ta += sa[w]; tb += sb[w]; }
        part[2 * blockIdx.x] = ta;
        part[2 * blockIdx.x + 1] = tb;
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x >= 32) return;
    __threadfence();
    // the last block's first warp adds the partials in a fixed order (lane-strided, then a
    // butterfly: every lane ends with the same bits)
    double ta = 0.0, tb = 0.0;
    for (int k = lane; k < (int)gridDim.x; k += 32) { ta += __ldcg(part + 2 * k); tb += __ldcg(part + 2 * k + 1); }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ta += __shfl_xor_sync(0xffffffffu, ta, o);
        tb += __shfl_xor_sync(0xffffffffu, tb, o);
    }
    if (lane != 0) return;
    // keep the caller's order unless its packets are clearly less coherent: geometric-mean path
    // length more than 4x the Morton order's (random-order samples: C5 patch-major, C1)
    const double npk_d = (double)((n + 31) / 32);
    *keep_caller = (ta / npk_d) <= (tb / npk_d) + 1.3862943611198906 ? 1 : 0;     // log(4)
    *ticket = 0u;
}

__global__ void apply_order_kernel(const float* __restrict__ p, int n, const int* __restrict__ keep_caller,
                                   uint32_t* __restrict__ perm, float* __restrict__ sorted) {
    pdl_entry();
    if (!*keep_caller) return;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        perm[k] = (uint32_t)k;
        sorted[3 * (size_t)k] = p[3 * (size_t)k];
        sorted[3 * (size_t)k + 1] = p[3 * (size_t)k + 1];
        sorted[3 * (size_t)k + 2] = p[3 * (size_t)k + 2];
    }
}

}  // namespace

// Stable LSD radix sort of (key, value) pairs by key bits [0, bits) in passes of 8 bits,
// ping-ponging between (k0, v0) and (k1, v1); *in_alt = true when the result ends in (k1, v1).
// scratch: radix_sort_scratch_bytes(n) bytes of device memory.
size_t radix_sort_scratch_bytes(int n) {
    const int nblk = sort_blocks(n);
    return align_up((size_t)kRadix * nblk * 4, 256) + scan_temp_bytes((int64_t)kRadix * nblk);
}

cudaError_t radix_sort_pairs(unsigned long long* k0, uint32_t* v0, unsigned long long* k1, uint32_t* v1, int n,
                             int bits, void* scratch, cudaStream_t s, int* nlaunch, bool* in_alt, bool pdl) {
    const int nblk = sort_blocks(n), ipw = sort_ipw(n);
    uint32_t* hist = (uint32_t*)scratch;
    void* scan_tmp = (char*)scratch + align_up((size_t)kRadix * nblk * 4, 256);
    int nl = 0;
    bool alt = false;
    for (int shift = 0; shift < bits; shift += kRadixBits) {
        launch_k(pdl, radix_hist_kernel, nblk, kThreads, s, (const unsigned long long*)k0, n, shift, hist, nblk, ipw);
        nl += 2 + scan_exclusive_u32(hist, (int64_t)kRadix * nblk, scan_tmp, s, pdl);
        launch_k(pdl, radix_scatter_kernel, nblk, kThreads, s, (const unsigned long long*)k0, (const uint32_t*)v0, k1, v1, n, shift,
                 (const uint32_t*)hist, nblk, ipw);
        std::swap(k0, k1);
        std::swap(v0, v1);
        alt = !alt;
    }
    if (nlaunch) *nlaunch += nl;
    if (in_alt) *in_alt = alt;
    return cudaGetLastError();
}

// Spatially coherent order of a point set (SURVEY.md 7 "source Morton-sorted once per run in its
// own frame"): the top 32 bits of the 48-bit Morton key in the set's own bounding box, stable
// LSD radix sort (4 passes of 8 bits) -> perm (sorted position -> original index) and the
// points in that order (packed xyz); then the caller's own order is kept instead if its 32-point
// packets are at least as compact (decided on the device, no host synchronisation).  Scratch
// from the library pool, stream-ordered.
cudaError_t morton_order_points(const float* pts, int n, uint32_t* perm, float* sorted, cudaStream_t s, int* nlaunch) {
    const int nblk_sort = sort_blocks(n), ipw = sort_ipw(n);
    const bool pdl = pipeline_pdl(n);
    const int nblk_bbox = grid_for(n);
    const size_t s_keys = align_up((size_t)n * 8, 256), s_vals = align_up((size_t)n * 4, 256);
    const size_t s_hist = align_up((size_t)kRadix * nblk_sort * 4, 256);
    const size_t s_bb = align_up((size_t)(6 * nblk_bbox) * 4, 256);
    const size_t s_scan = scan_temp_bytes((int64_t)kRadix * nblk_sort);
    void* tmp = nullptr;
    const size_t s_choice = align_up((size_t)(2 * kExtBlocks) * 8, 256) + 256;
    cudaError_t e = pool_alloc(&tmp, 2 * s_keys + s_vals + s_hist + s_bb + s_scan + 256 + s_choice, s);
    if (e != cudaSuccess) return e;
    char* tb = (char*)tmp;
    unsigned long long* k0 = (unsigned long long*)tb;
    unsigned long long* k1 = (unsigned long long*)(tb + s_keys);
    uint32_t* v1 = (uint32_t*)(tb + 2 * s_keys);
    uint32_t* hist = (uint32_t*)(tb + 2 * s_keys + s_vals);
    float* bbp = (float*)(tb + 2 * s_keys + s_vals + s_hist);
    void* scan_tmp = (void*)(tb + 2 * s_keys + s_vals + s_hist + s_bb);
    float4* quant = (float4*)(tb + 2 * s_keys + s_vals + s_hist + s_bb + s_scan);
    double* cpart = (double*)(tb + 2 * s_keys + s_vals + s_hist + s_bb + s_scan + 256);
    unsigned* cticket = (unsigned*)(tb + 2 * s_keys + s_vals + s_hist + s_bb + s_scan + 256 + align_up((size_t)(2 * kExtBlocks) * 8, 256));
    int* keep = (int*)(cticket + 1);
    uint32_t* v0 = perm;                       // the values ping-pong between perm and v1
    int nl = 0;
    launch_k(pdl, bbox_partial_kernel, nblk_bbox, kThreads, s, pts, n, bbp);
    launch_k(pdl, bbox_final_kernel, 1, kThreads, s, (const float*)bbp, nblk_bbox, quant);
    launch_k(pdl, morton_kernel, grid_for(n), kThreads, s, pts, n, (const float4*)quant, k0, v0);
    nl += 3;
    for (int shift = 3 * kMortonBits - 32; shift < 3 * kMortonBits; shift += kRadixBits) {
        launch_k(pdl, radix_hist_kernel, nblk_sort, kThreads, s, (const unsigned long long*)k0, n, shift, hist, nblk_sort, ipw);
        nl += 2 + scan_exclusive_u32(hist, (int64_t)kRadix * nblk_sort, scan_tmp, s, pdl);
        launch_k(pdl, radix_scatter_kernel, nblk_sort, kThreads, s, (const unsigned long long*)k0, (const uint32_t*)v0, k1, v1, n,
                 shift, (const uint32_t*)hist, nblk_sort, ipw);
        std::swap(k0, k1);
        std::swap(v0, v1);
    }
    // 4 passes: the sorted values are back in perm
    launch_k(pdl, gather_xyz_kernel, grid_for(n), kThreads, s, pts, (const uint32_t*)perm, n, sorted);
    // keep the caller's order when it is at least as coherent (scan-ordered LiDAR / depth frames)
    if (!(debug_flags() & 32u)) {                 // diagnostics bit 5: always the Morton order
        cudaMemsetAsync(cticket, 0, 8, s);
        launch_k(pdl, order_choice_kernel, kExtBlocks, kThreads, s, pts, (const float*)sorted, n, cpart, cticket, keep);
        launch_k(pdl, apply_order_kernel, grid_for(n), kThreads, s, pts, n, (const int*)keep, perm, sorted);
        nl += 3;
    }
    e = cudaGetLastError();
    pool_free(tmp, s);
    if (nlaunch) *nlaunch = nl;
    return e;
}

}  // namespace cil

using namespace cil;

CIL_API cil_status cil_target_build(const float* pts, const float* normals, int64_t n,
                                    const cil_index_params* params, cil_stream_t stream, cil_target** out) {
    if (!out) { set_error("cil_target_build: out is NULL"); return CIL_ERR_INVALID_ARG; }
    *out = nullptr;
    if (n == 0) { set_error("cil_target_build: empty target (n == 0)"); return CIL_ERR_EMPTY_TARGET; }
    if (n < 0 || n > INT32_MAX) { set_error("cil_target_build: n=%lld out of range", (long long)n); return CIL_ERR_INVALID_ARG; }
    if (!pts) { set_error("cil_target_build: pts is NULL"); return CIL_ERR_INVALID_ARG; }
    int B = 16;                 // default leaf size (measured over C1-C5)
    int kind = CIL_INDEX_BVH;
    float grid_points = 1.0f;   // targets per grid cell (1 beats 2 on C2 since the row-range search)
    if (params) {
        if (params->leaf_size) B = params->leaf_size;
        kind = params->index_kind;
        if (params->grid_points != 0.0f) grid_points = params->grid_points;
        for (int k = 0; k < 5; ++k)
            if (params->reserved[k]) { set_error("cil_target_build: reserved index params must be 0"); return CIL_ERR_INVALID_ARG; }
    }
    if (kind != CIL_INDEX_BVH && kind != CIL_INDEX_GRID) {
        set_error("cil_target_build: index_kind %d not supported", kind);
        return CIL_ERR_INVALID_ARG;
    }
    if (!(grid_points > 0.0f) || !std::isfinite(grid_points)) {
        set_error("cil_target_build: grid_points must be finite and > 0");
        return CIL_ERR_INVALID_ARG;
    }
    if (B != 4 && B != 8 && B != 16 && B != 32) {
        set_error("cil_target_build: leaf_size %d not in {4, 8, 16, 32}", B);
        return CIL_ERR_INVALID_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int N = (int)n;
    const int64_t n_leaves = (N + B - 1) / B;
    int64_t l_pad = 1;
    while (l_pad < n_leaves) l_pad <<= 1;

    int levels = 0;
    while ((1ll << levels) < l_pad) ++levels;
    // coarse Morton cells: about one cell per point, a multiple of 3 bits, at most 21
    int coarse_bits = 3;
    while (coarse_bits < 21 && (1ll << coarse_bits) < n) coarse_bits += 3;
    const int64_t ncell = 1ll << coarse_bits;

    // one allocation: opts (16N), onrm (16N), box (2 * 2*l_pad * 16), keys (8N), cell table, quant,
    // SoA leaves (16N), interleaved leaf boxes (32 per leaf)
    const size_t b_pts = align_up((size_t)N * 16, 256);
    const size_t b_nrm = normals ? align_up((size_t)N * 16, 256) : 0;
    const size_t b_box = align_up((size_t)4 * l_pad * 16, 256);
    const size_t b_keys = align_up((size_t)N * 8, 256);
    const size_t b_cell = align_up((size_t)(ncell + 1) * 4, 256);
    const size_t b_quant = 256;
    const size_t b_soa = align_up((size_t)n_leaves * B * 16, 256);
    const size_t b_lbox = align_up((size_t)n_leaves * 32, 256);
    const size_t bytes = b_pts + b_nrm + b_box + b_keys + b_cell + b_quant + b_soa + b_lbox;
    int dev = 0;
    CIL_CUDA_TRY(cudaGetDevice(&dev), "cudaGetDevice");
    void* mem = nullptr;
    CIL_CUDA_TRY(pool_alloc(&mem, bytes, s), "pool_alloc(target)");
    char* base = (char*)mem;
    float4* d_pts = (float4*)base;
    float4* d_nrm = normals ? (float4*)(base + b_pts) : nullptr;
    float4* d_box = (float4*)(base + b_pts + b_nrm);
    unsigned long long* d_keys = (unsigned long long*)(base + b_pts + b_nrm + b_box);
    uint32_t* d_cell = (uint32_t*)(base + b_pts + b_nrm + b_box + b_keys);
    float4* d_quant = (float4*)(base + b_pts + b_nrm + b_box + b_keys + b_cell);
    float* d_soa = (float*)(base + b_pts + b_nrm + b_box + b_keys + b_cell + b_quant);
    float4* d_lbox = (float4*)(base + b_pts + b_nrm + b_box + b_keys + b_cell + b_quant + b_soa);

    // scratch: keys x2 (8N), vals x2 (4N), hist (256 * nblk), bbox partials
    const int nblk_sort = sort_blocks(N), ipw = sort_ipw(N);
    const bool pdl = pipeline_pdl(N);
    const int nblk_bbox = grid_for(N);
    const size_t s_keys = align_up((size_t)N * 8, 256), s_vals = align_up((size_t)N * 4, 256);
    const size_t s_hist = align_up((size_t)kRadix * nblk_sort * 4, 256);
    const size_t s_bb = align_up((size_t)(6 * nblk_bbox) * 4, 256);
    const size_t s_scan = scan_temp_bytes((int64_t)kRadix * nblk_sort);
    const size_t s_spts = align_up((size_t)N * 16, 256);
    const size_t scratch = 2 * s_keys + 2 * s_vals + s_hist + s_bb + s_scan + s_spts;
    void* tmp = nullptr;
    cudaError_t e = pool_alloc(&tmp, scratch, s);
    if (e != cudaSuccess) { pool_free(mem, s); return cuda_fail(e, "pool_alloc(scratch)"); }
    char* tb = (char*)tmp;
    unsigned long long* k0 = (unsigned long long*)tb;
    unsigned long long* k1 = (unsigned long long*)(tb + s_keys);
    uint32_t* v0 = (uint32_t*)(tb + 2 * s_keys);
    uint32_t* v1 = (uint32_t*)(tb + 2 * s_keys + s_vals);
    uint32_t* hist = (uint32_t*)(tb + 2 * s_keys + 2 * s_vals);
    float* bbp = (float*)(tb + 2 * s_keys + 2 * s_vals + s_hist);
    void* scan_tmp = (void*)(tb + 2 * s_keys + 2 * s_vals + s_hist + s_bb);
    float4* spts = (float4*)(tb + 2 * s_keys + 2 * s_vals + s_hist + s_bb + s_scan);
    int nlaunch = 0;

    prof_begin(kProfBuild, s);
    launch_k(pdl, bbox_partial_kernel, nblk_bbox, kThreads, s, pts, N, bbp);
    launch_k(pdl, bbox_final_kernel, 1, kThreads, s, (const float*)bbp, nblk_bbox, d_quant);
    launch_k(pdl, morton_kernel, grid_for(N), kThreads, s, pts, N, (const float4*)d_quant, k0, v0);
    for (int shift = 0; shift < 3 * kMortonBits; shift += kRadixBits) {
        launch_k(pdl, radix_hist_kernel, nblk_sort, kThreads, s, (const unsigned long long*)k0, N, shift, hist, nblk_sort, ipw);
        nlaunch += scan_exclusive_u32(hist, (int64_t)kRadix * nblk_sort, scan_tmp, s, pdl);
        launch_k(pdl, radix_scatter_kernel, nblk_sort, kThreads, s, (const unsigned long long*)k0, (const uint32_t*)v0, k1, v1, N,
                 shift, (const uint32_t*)hist, nblk_sort, ipw);
        std::swap(k0, k1);
        std::swap(v0, v1);
    }
    launch_k(pdl, gather_kernel, grid_for(N), kThreads, s, pts, normals, N, v0, spts, d_pts, d_nrm);
    cudaMemcpyAsync(d_keys, k0, (size_t)N * 8, cudaMemcpyDeviceToDevice, s);
    launch_k(pdl, cell_first_kernel, grid_for(ncell + 1), kThreads, s, k0, N, 3 * kMortonBits - coarse_bits, (uint32_t)ncell, d_cell);
    launch_k(pdl, leaf_box_kernel, grid_for(l_pad), kThreads, s, spts, N, B, (int)l_pad, d_box, (int)n_leaves, d_lbox);
    launch_k(pdl, leaf_soa_kernel, grid_for(n_leaves * B), kThreads, s, spts, N, B, n_leaves, d_soa);
    int tree_passes = 0;
    for (int first = (int)l_pad, rem = levels; rem > 0; ++tree_passes) {
        const int lv = std::min(rem, 8);
        const int width = std::min(kPassNodes, first);
        launch_k(pdl, tree_pass_kernel, first / width, kPassNodes, s, d_box, first, lv);
        first >>= lv;
        rem -= lv;
    }
    TargetView gv{};
    void* gmem = nullptr;
    size_t gbytes = 0;
    if (kind == CIL_INDEX_GRID && e == cudaSuccess) {
        int ng = 0;
        e = grid_build(pts, N, d_quant, d_quant + 1, grid_points, s, &gmem, &gbytes, &gv, &ng);
        nlaunch += ng;
    }
    count_launches(3 + 2 * ((3 * kMortonBits + kRadixBits - 1) / kRadixBits) + nlaunch + 4 + tree_passes);
    prof_end(s);
    if (e == cudaSuccess) e = cudaGetLastError();
    pool_free(tmp, s);
    if (e != cudaSuccess) {
        pool_free(mem, s);
        if (gmem) pool_free(gmem, s);
        return cuda_fail(e, "cil_target_build launch");
    }

    cil_target* t = new cil_target;
    t->v.gpts = gv.gpts;
    t->v.gstart = gv.gstart;
    t->v.gdesc = gv.gdesc;
    t->gmem = gmem;
    t->index_kind = kind;
    t->v.opts = d_pts;
    t->v.onrm = d_nrm;
    t->v.box = d_box;
    t->v.n = N;
    t->v.l_pad = (int)l_pad;
    t->v.leaf_size = B;
    t->v.keys = d_keys;
    t->v.leafsoa = (const float4*)d_soa;
    t->v.lbox = d_lbox;
    t->v.cell_first = d_cell;
    t->v.quant = d_quant;
    t->v.levels = levels;
    t->v.coarse_bits = coarse_bits;
    t->v.trace = nullptr;
    t->v.dbg_mode = 0;
    t->n_leaves = n_leaves;
    t->has_normals = normals ? 1 : 0;
    t->device = dev;
    t->mem = mem;
    t->bytes = bytes + gbytes;
    *out = t;
    return CIL_OK;
}

CIL_API cil_status cil_target_free(cil_target* t, cil_stream_t stream) {
    if (!t) return CIL_OK;
    cudaError_t e = pool_free(t->mem, (cudaStream_t)stream);
    if (t->gmem) {
        const cudaError_t e2 = pool_free(t->gmem, (cudaStream_t)stream);
        if (e == cudaSuccess) e = e2;
    }
    delete t;
    if (e != cudaSuccess) return cuda_fail(e, "pool_free(target)");
    return CIL_OK;
}

CIL_API cil_status cil_target_get_info(const cil_target* t, cil_target_info* info) {
    if (!t || !info) { set_error("cil_target_get_info: NULL argument"); return CIL_ERR_INVALID_ARG; }
    info->n = t->v.n;
    info->n_leaves = t->n_leaves;
    info->n_nodes = 2 * (int64_t)t->v.l_pad;
    info->leaf_size = t->v.leaf_size;
    info->has_normals = t->has_normals;
    info->device_bytes = (int64_t)t->bytes;
    info->index_kind = t->index_kind;
    info->pad = 0;
    return CIL_OK;
}
