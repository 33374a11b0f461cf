// voxel.cu -- cil_voxel_downsample: voxel-grid downsampling on the GPU (
// PAPER.md:125 "general dimension grid-based point cloud downsampling", "downsampled
// using a voxel grid of bin size equal to 1cm"; readings R27-R29).
//
// Pipeline (one stream, no host synchronisation; the bin count stays on the device):
//   V1 key per point: k_a = floor((p_a - o_a) / bin) in fp64 (bit-exact with the definition),
//      block min/max per axis -> device atomics; non-finite / out-of-int32 keys raise a flag
//   V2 pack (k - k_min) into 21 bits per axis (lexicographic x, y, z) + the input index
//   V3 stable LSD radix sort of (key, index), 8 passes of 8 bits (target.cu)
//   V4 bin heads (key change) -> exclusive scan -> bin start offsets, *n_out
//   V5 one thread per bin: fp64 sums in increasing input index (the sort is stable), mean,
//      cast to fp32; normals: fp64 mean / its norm (no FMA), 0 below 1e-12
#include "internal.cuh"

#include <algorithm>
#include <climits>
#include <cmath>

namespace cil {
namespace {

constexpr int kVThreads = 256;
constexpr int kAxisBits = 21;

inline int vgrid(int64_t work) {
    const int64_t b = (work + kVThreads - 1) / kVThreads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)sm_count() * 8));
}

__global__ void voxel_init_kernel(int* mm, int* bad) {
    if (threadIdx.x < 3) { mm[threadIdx.x] = INT_MAX; mm[3 + threadIdx.x] = INT_MIN; }
    if (threadIdx.x == 0) *bad = 0;
}

__global__ void __launch_bounds__(kVThreads)
voxel_key_kernel(const float* __restrict__ p, int n, double bin, double ox, double oy, double oz,
                 int* __restrict__ k3, int* __restrict__ mm, int* __restrict__ bad) {
    int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
    int flag = 0;
    const double o[3] = {ox, oy, oz};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double k = floor(__ddiv_rn(__dsub_rn((double)__ldg(p + 3 * (size_t)i + a), o[a]), bin));
            int ki = 0;
            if (k >= -2147483648.0 && k <= 2147483647.0) ki = (int)k;
            else flag = 1;                                   // also NaN
            k3[3 * (size_t)i + a] = ki;
            mn[a] = min(mn[a], ki);
            mx[a] = max(mx[a], ki);
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], off));
            mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], off));
        }
    flag = __any_sync(0xffffffffu, flag);
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (mn[a] != INT_MAX) atomicMin(mm + a, mn[a]);
            if (mx[a] != INT_MIN) atomicMax(mm + 3 + a, mx[a]);
        }
        if (flag) atomicOr(bad, 1);
    }
}

__global__ void voxel_pack_kernel(const int* __restrict__ k3, int n, const int* __restrict__ mm, int* __restrict__ bad,
                                  unsigned long long* __restrict__ key, uint32_t* __restrict__ idx) {
    const long long span = (long long)kAxisBits;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int a = 0; a < 3; ++a)
            if ((long long)mm[3 + a] - (long long)mm[a] >= (1ll << span)) atomicOr(bad, 2);
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long x = (unsigned long long)((long long)k3[3 * (size_t)i] - mm[0]) & ((1ull << span) - 1);
        const unsigned long long y = (unsigned long long)((long long)k3[3 * (size_t)i + 1] - mm[1]) & ((1ull << span) - 1);
        const unsigned long long z = (unsigned long long)((long long)k3[3 * (size_t)i + 2] - mm[2]) & ((1ull << span) - 1);
        key[i] = (x << (2 * span)) | (y << span) | z;
        idx[i] = (uint32_t)i;
    }
}

// head[i] = 1 where a new bin starts in sorted order
__global__ void voxel_head_kernel(const unsigned long long* __restrict__ key, int n, uint32_t* __restrict__ head) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        head[i] = (i == 0 || key[i] != key[i - 1]) ? 1u : 0u;
}

// after the exclusive scan of head: start[bin] = first sorted position, start[nb] = n, *n_out
__global__ void voxel_start_kernel(const unsigned long long* __restrict__ key, const uint32_t* __restrict__ scan, int n,
                                   uint32_t* __restrict__ start, const int* __restrict__ bad,
                                   long long* __restrict__ n_out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const bool is_head = i == 0 || key[i] != key[i - 1];
        if (is_head) start[scan[i]] = (uint32_t)i;
        if (i == n - 1) {
            const uint32_t nb = scan[i] + (is_head ? 1u : 0u);   // exclusive scan: heads before i
            start[nb] = (uint32_t)n;
            *n_out = *bad ? -1ll : (long long)nb;
        }
    }
}

__global__ void __launch_bounds__(kVThreads)
voxel_mean_kernel(const float* __restrict__ p, const float* __restrict__ nrm, const uint32_t* __restrict__ perm,
                  const uint32_t* __restrict__ start, const long long* __restrict__ n_out, float* __restrict__ out,
                  float* __restrict__ out_n) {
    const long long nb = *n_out;
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb; b += (long long)gridDim.x * blockDim.x) {
        const uint32_t s = start[b], e = start[b + 1];
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, m0 = 0.0, m1 = 0.0, m2 = 0.0;
        for (uint32_t r = s; r < e; ++r) {
            const size_t o = 3 * (size_t)perm[r];
            c0 = __dadd_rn(c0, (double)__ldg(p + o));
            c1 = __dadd_rn(c1, (double)__ldg(p + o + 1));
            c2 = __dadd_rn(c2, (double)__ldg(p + o + 2));
            if (nrm) {
                m0 = __dadd_rn(m0, (double)__ldg(nrm + o));
                m1 = __dadd_rn(m1, (double)__ldg(nrm + o + 1));
                m2 = __dadd_rn(m2, (double)__ldg(nrm + o + 2));
            }
        }
        const double cnt = (double)(e - s);
        out[3 * b] = (float)__ddiv_rn(c0, cnt);
        out[3 * b + 1] = (float)__ddiv_rn(c1, cnt);
        out[3 * b + 2] = (float)__ddiv_rn(c2, cnt);
        if (nrm) {
            m0 = __ddiv_rn(m0, cnt);
            m1 = __ddiv_rn(m1, cnt);
            m2 = __ddiv_rn(m2, cnt);
            const double len = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(m0, m0), __dmul_rn(m1, m1)), __dmul_rn(m2, m2)));
            const bool z = len < 1e-12;
            out_n[3 * b] = z ? 0.0f : (float)__ddiv_rn(m0, len);
            out_n[3 * b + 1] = z ? 0.0f : (float)__ddiv_rn(m1, len);
            out_n[3 * b + 2] = z ? 0.0f : (float)__ddiv_rn(m2, len);
        }
    }
}

}  // namespace
}  // namespace cil

using namespace cil;

CIL_API cil_status cil_voxel_downsample(const float* pts, const float* normals, int64_t n, double bin_size,
                                        const double* origin, float* out_pts, float* out_normals, int64_t* n_out,
                                        cil_stream_t stream) {
    if (n < 0 || n > INT32_MAX) { set_error("cil_voxel_downsample: n=%lld out of range", (long long)n); return CIL_ERR_INVALID_ARG; }
    if (!(bin_size > 0.0) || !std::isfinite(bin_size)) {
        set_error("cil_voxel_downsample: bin_size must be finite and > 0");
        return CIL_ERR_INVALID_ARG;
    }
    const double o[3] = {origin ? origin[0] : 0.0, origin ? origin[1] : 0.0, origin ? origin[2] : 0.0};
    if (!std::isfinite(o[0]) || !std::isfinite(o[1]) || !std::isfinite(o[2])) {
        set_error("cil_voxel_downsample: origin must be finite");
        return CIL_ERR_INVALID_ARG;
    }
    if (!n_out) { set_error("cil_voxel_downsample: n_out is NULL"); return CIL_ERR_INVALID_ARG; }
    if (n > 0 && (!pts || !out_pts)) { set_error("cil_voxel_downsample: pts/out_pts NULL"); return CIL_ERR_INVALID_ARG; }
    if (out_normals && !normals) {
        set_error("cil_voxel_downsample: out_normals needs input normals");
        return CIL_ERR_NO_NORMALS;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) {
        CIL_CUDA_TRY(cudaMemsetAsync(n_out, 0, sizeof(int64_t), s), "cil_voxel_downsample");
        return CIL_OK;
    }
    const int m = (int)n;
    const size_t s_k3 = align_up((size_t)m * 12, 256), s_key = align_up((size_t)m * 8, 256);
    const size_t s_u32 = align_up((size_t)m * 4, 256), s_start = align_up(((size_t)m + 1) * 4, 256);
    const size_t s_sort = radix_sort_scratch_bytes(m), s_scan = scan_temp_bytes(m);
    const size_t total = s_k3 + 2 * s_key + 3 * s_u32 + s_start + s_sort + s_scan + 256;
    void* tmp = nullptr;
    CIL_CUDA_TRY(pool_alloc(&tmp, total, s), "cil_voxel_downsample: scratch");
    char* t = (char*)tmp;
    int* k3 = (int*)t;                                         t += s_k3;
    unsigned long long* ka = (unsigned long long*)t;           t += s_key;
    unsigned long long* kb = (unsigned long long*)t;           t += s_key;
    uint32_t* va = (uint32_t*)t;                               t += s_u32;
    uint32_t* vb = (uint32_t*)t;                               t += s_u32;
    uint32_t* head = (uint32_t*)t;                             t += s_u32;
    uint32_t* start = (uint32_t*)t;                            t += s_start;
    void* sort_tmp = (void*)t;                                 t += s_sort;
    void* scan_tmp = (void*)t;                                 t += s_scan;
    int* mm = (int*)t;                                         // 6 ints + bad flag
    int* bad = mm + 6;
    int nl = 0;
    voxel_init_kernel<<<1, 32, 0, s>>>(mm, bad);
    voxel_key_kernel<<<vgrid(m), kVThreads, 0, s>>>(pts, m, bin_size, o[0], o[1], o[2], k3, mm, bad);
    voxel_pack_kernel<<<vgrid(m), kVThreads, 0, s>>>(k3, m, mm, bad, ka, va);
    nl += 3;
    bool alt = false;
    cudaError_t e = radix_sort_pairs(ka, va, kb, vb, m, 3 * kAxisBits, sort_tmp, s, &nl, &alt);
    if (e != cudaSuccess) { pool_free(tmp, s); return cuda_fail(e, "cil_voxel_downsample: sort"); }
    const unsigned long long* ks = alt ? kb : ka;
    const uint32_t* perm = alt ? vb : va;
    voxel_head_kernel<<<vgrid(m), kVThreads, 0, s>>>(ks, m, head);
    nl += 1 + scan_exclusive_u32(head, m, scan_tmp, s);
    voxel_start_kernel<<<vgrid(m), kVThreads, 0, s>>>(ks, head, m, start, bad, reinterpret_cast<long long*>(n_out));
    voxel_mean_kernel<<<vgrid(m), kVThreads, 0, s>>>(pts, out_normals ? normals : nullptr, perm, start,
                                                      reinterpret_cast<const long long*>(n_out), out_pts, out_normals);
    nl += 2;
    count_launches(nl);
    e = cudaGetLastError();
    pool_free(tmp, s);
    if (e != cudaSuccess) return cuda_fail(e, "cil_voxel_downsample launch");
    return CIL_OK;
}
