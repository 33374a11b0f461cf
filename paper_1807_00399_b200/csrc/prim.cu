// prim.cu -- device-wide primitives used by the index build and the query sort:
// exclusive scan of uint32 (3 phases: tile sums, scan of tile sums, tile scans with carry).
#include "internal.cuh"

#include <algorithm>

namespace cil {
namespace {

constexpr int kScanThreads = 256;
#ifndef CIL_SCAN_ITEMS
#define CIL_SCAN_ITEMS 4      // (tiles of 1,024 counters: C4 build 0.426 -> 0.410 ms; 16: 0.426, 8: 0.414, 2: 0.400 but 2^24 build +2.6 %)
#endif
constexpr int kScanItems = CIL_SCAN_ITEMS;                          // per thread
constexpr int kScanTile = kScanThreads * kScanItems;    // 1024 per block
#ifndef CIL_SCAN_FUSED_PREFIX
#define CIL_SCAN_FUSED_PREFIX 1
#endif
constexpr int kFusedPrefixTiles = 2048;                 // up to this many tiles every block sums its predecessors itself

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
    __shared__ uint32_t warp_tot[kScanThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t t = lane < kScanThreads / 32 ? warp_tot[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < kScanThreads / 32) warp_tot[lane] = t;
    }
    __syncthreads();
    const uint32_t wbase = w > 0 ? warp_tot[w - 1] : 0u;
    if (total) *total = warp_tot[kScanThreads / 32 - 1];
    __syncthreads();
    return wbase + x - v;
}

__global__ void tile_sum_kernel(const uint32_t* __restrict__ a, int64_t len, uint32_t* __restrict__ tsum) {
    pdl_entry();
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;
        if (i < len) s += a[i];
    }
    uint32_t tot;
    block_exclusive_scan(s, &tot);
    if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
}

// exclusive scan of tsum[0..nt) in place, by one block (chunks of 256 with carry)
__global__ void tile_prefix_kernel(uint32_t* __restrict__ tsum, int nt) {
    pdl_entry();
    uint32_t carry = 0;
    for (int b = 0; b < nt; b += kScanThreads) {
        const int i = b + threadIdx.x;
        const uint32_t v = i < nt ? tsum[i] : 0u;
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan(v, &tot);
        if (i < nt) tsum[i] = carry + ex;
        carry += tot;
    }
}

// raw = true: tsum holds the tiles' sums (no tile_prefix_kernel ran): the block adds up the sums
// of the tiles before it (a few hundred values: cheaper than a third launch)
__global__ void tile_scan_kernel(uint32_t* __restrict__ a, int64_t len, const uint32_t* __restrict__ tsum, bool raw) {
    pdl_entry();
    // each thread owns kScanItems consecutive elements of the tile
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = base + k < len ? a[base + k] : 0u;
        s += v[k];
    }
    uint32_t tile_base;
    if (raw) {
        uint32_t p = 0;
        for (int b = threadIdx.x; b < (int)blockIdx.x; b += kScanThreads) p += tsum[b];
        uint32_t tot;
        block_exclusive_scan(p, &tot);
        tile_base = tot;
    } else {
        tile_base = tsum[blockIdx.x];
    }
    uint32_t run = tile_base + block_exclusive_scan(s, nullptr);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < len) a[base + k] = run;
        run += v[k];
    }
}

// Short arrays (the digit x tile tables of small sorts): the whole exclusive scan by one block of
// 1024 threads, each owning a run of consecutive uint4 quads -- one launch instead of three.
constexpr int kSmallScanThreads = 1024;
constexpr int kSmallScanQuads = 8;                                         // per thread at most (loads issued together)
constexpr int64_t kSmallScanMax = (int64_t)kSmallScanThreads * kSmallScanQuads * 4;   // 32,768

template <int kSmallScanQuads>
__global__ void __launch_bounds__(kSmallScanThreads)
scan_small_kernel(uint32_t* a, int nquads) {
    pdl_entry();
    __shared__ uint32_t warp_tot[kSmallScanThreads / 32];
    const int q0 = threadIdx.x * kSmallScanQuads;
    uint4* a4 = reinterpret_cast<uint4*>(a);
    uint4 v[kSmallScanQuads];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kSmallScanQuads; ++k) v[k] = q0 + k < nquads ? a4[q0 + k] : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int k = 0; k < kSmallScanQuads; ++k) s += v[k].x + v[k].y + v[k].z + v[k].w;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t t = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        warp_tot[lane] = t;
    }
    __syncthreads();
    uint32_t run = (w > 0 ? warp_tot[w - 1] : 0u) + x - s;
#pragma unroll
    for (int k = 0; k < kSmallScanQuads; ++k) {
        uint4 o;
        o.x = run; run += v[k].x;
        o.y = run; run += v[k].y;
        o.z = run; run += v[k].z;
        o.w = run; run += v[k].w;
        if (q0 + k < nquads) a4[q0 + k] = o;
    }
}

}  // namespace

size_t scan_temp_bytes(int64_t len) {
    return align_up((size_t)((len + kScanTile - 1) / kScanTile) * 4, 256);
}

int scan_exclusive_u32(uint32_t* a, int64_t len, void* temp, cudaStream_t s, bool pdl) {
    if (len <= kSmallScanMax && len % 4 == 0 && (reinterpret_cast<uintptr_t>(a) & 15) == 0) {
        if (len <= kSmallScanMax / 2) launch_k(pdl, scan_small_kernel<kSmallScanQuads / 2>, 1, kSmallScanThreads, s, a, (int)(len / 4));
        else launch_k(pdl, scan_small_kernel<kSmallScanQuads>, 1, kSmallScanThreads, s, a, (int)(len / 4));
        return 1;
    }
    const int nt = (int)((len + kScanTile - 1) / kScanTile);
    uint32_t* tsum = (uint32_t*)temp;
    launch_k(pdl, tile_sum_kernel, nt, kScanThreads, s, (const uint32_t*)a, len, tsum);
    const bool raw = CIL_SCAN_FUSED_PREFIX && nt <= kFusedPrefixTiles;
    if (!raw) launch_k(pdl, tile_prefix_kernel, 1, kScanThreads, s, tsum, nt);
    launch_k(pdl, tile_scan_kernel, nt, kScanThreads, s, a, len, (const uint32_t*)tsum, raw);
    return raw ? 2 : 3;
}

}  // namespace cil
