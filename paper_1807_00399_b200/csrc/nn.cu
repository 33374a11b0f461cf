// nn.cu -- cil_nn_query: exact 1-NN of independent queries (SURVEY.md 8(a) row a2,
// BASELINE.json configs[1]; "k-NN ... queries").
#include "internal.cuh"
#include "search.cuh"
#include "grid.cuh"

#include <algorithm>
#include <cmath>

namespace cil {
namespace {

constexpr int kNNThreads = 32 * kEngineWarps;
#ifndef CIL_NNQ_MINB
#define CIL_NNQ_MINB 4
#endif

// Queries are processed in the order of perm (a counting sort by the target's coarse Morton
// cell) so that the 32 queries of a warp packet are spatial neighbours; results are written
// back in the caller's order.
struct NNQueries {
    const float* q;
    const uint32_t* perm;
    float bound2;
    float stale2;            // unused (no warm hints)
    int32_t* idx;
    float* sqd;
    __device__ __forceinline__ int packets(int m) const { return (m + 31) / 32; }
    __device__ __forceinline__ int packet_base(int c) const { return 32 * c; }
    __device__ __forceinline__ int tag() const { return 0; }
    __device__ __forceinline__ bool load(int k, DF3& s, unsigned long long& init, int& hint) const {
        const size_t i = perm[k];
        s.hx = q[3 * i]; s.hy = q[3 * i + 1]; s.hz = q[3 * i + 2];
        s.lx = s.ly = s.lz = 0.0f;
        init = bound_key(bound2);
        hint = -1;
        return true;
    }
    __device__ __forceinline__ void store(int k, unsigned long long best, float) const {
        const size_t i = perm[k];
        const bool found = best != bound_key(bound2);
        if (idx) idx[i] = found ? (int32_t)key_idx(best) : -1;
        if (sqd) sqd[i] = found ? key_d2(best) : INFINITY;
    }
};

// counting sort of the queries by coarse cell: count, (scan), scatter
__global__ void qcell_count_kernel(TargetView T, const float* __restrict__ q, int m, int qbits,
                                   uint32_t* __restrict__ qcell, uint32_t* __restrict__ cnt) {
    const float4 Q = __ldg(T.quant);
    const int shift = 3 * kMortonBits - qbits;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const uint32_t c = (uint32_t)(morton_of(Q, q[3 * (size_t)i], q[3 * (size_t)i + 1], q[3 * (size_t)i + 2]) >> shift);
        qcell[i] = c;
        atomicAdd(cnt + c, 1u);
    }
}

__global__ void qcell_scatter_kernel(const uint32_t* __restrict__ qcell, int m, uint32_t* __restrict__ cursor,
                                     uint32_t* __restrict__ perm) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        perm[atomicAdd(cursor + qcell[i], 1u)] = (uint32_t)i;
}

template <int B>
__global__ void __launch_bounds__(kNNThreads, CIL_NNQ_MINB)
nn_query_kernel(TargetView T, NNQueries qs, int m, unsigned int* counter) {
    nn_packet_engine<B, false>(T, qs, m, counter);
}

// the grid index (CIL_INDEX_GRID): one query per thread, in the same Morton-cell order
template <int B>
__global__ void __launch_bounds__(kNNThreads)
grid_query_kernel(TargetView T, NNQueries qs, int m) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    DF3 s;
    unsigned long long best;
    int hint;
    qs.load(k, s, best, hint);
    qs.store(k, grid_search<B, false>(T, s, best), 0.0f);
}

template <int B>
cudaError_t launch_nn(const TargetView& T, const NNQueries& qs, int m, unsigned int* counter, cudaStream_t s) {
    static int occ = -1;   // per-process cache; all supported devices are sm_100a
    if (occ < 0) {
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, nn_query_kernel<B>, kNNThreads, 0);
        if (e != cudaSuccess) return e;
        occ = std::max(occ, 1);
    }
    const int64_t want = ((int64_t)m + kNNThreads - 1) / kNNThreads;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * occ));
    TargetView Tv = T;
    Tv.trace = debug_trace();
    Tv.dbg_mode = (int)(debug_flags() >> 1) & 3;
    if (T.gpts) {
        grid_query_kernel<B><<<(int)(((int64_t)m + kNNThreads - 1) / kNNThreads), kNNThreads, 0, s>>>(Tv, qs, m);
        count_launches(1);
        return cudaGetLastError();
    }
    nn_query_kernel<B><<<blocks, kNNThreads, 0, s>>>(Tv, qs, m, counter);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace
}  // namespace cil

using namespace cil;

CIL_API cil_status cil_nn_query(const cil_target* t, const float* queries, int64_t m, float max_dist,
                                int32_t* idx, float* sqdist, cil_stream_t stream) {
    if (!t) { set_error("cil_nn_query: target is NULL"); return CIL_ERR_INVALID_ARG; }
    if (m < 0 || m > INT32_MAX) { set_error("cil_nn_query: m=%lld out of range", (long long)m); return CIL_ERR_INVALID_ARG; }
    if (std::isnan(max_dist) || max_dist < 0.0f) { set_error("cil_nn_query: max_dist must be >= 0 or INFINITY"); return CIL_ERR_INVALID_ARG; }
    if (m == 0) return CIL_OK;
    if (!queries) { set_error("cil_nn_query: queries is NULL"); return CIL_ERR_INVALID_ARG; }
    if (!idx && !sqdist) return CIL_OK;
    cudaStream_t s = (cudaStream_t)stream;
    // stream-ordered scratch: work counter | cell counts | qcell | perm | scan temp
    // query order: counting sort by coarse Morton cell (the grid search only needs packets of
    // neighbours: at most 2^18 cells, a cheaper scan)
    const int qbits = t->v.gpts ? std::min(t->v.coarse_bits, 18) : t->v.coarse_bits;
    const int64_t ncell = 1ll << qbits;
    const size_t b_cnt = align_up((size_t)(ncell + 1) * 4, 256);
    const size_t b_q = align_up((size_t)m * 4, 256);
    const size_t b_scan = scan_temp_bytes(ncell + 1);
    void* scratch = nullptr;
    CIL_CUDA_TRY(pool_alloc(&scratch, 256 + b_cnt + 2 * b_q + b_scan, s), "pool_alloc(nn scratch)");
    char* sb = (char*)scratch;
    unsigned int* counter = (unsigned int*)sb;
    uint32_t* cnt = (uint32_t*)(sb + 256);
    uint32_t* qcell = (uint32_t*)(sb + 256 + b_cnt);
    uint32_t* perm = (uint32_t*)(sb + 256 + b_cnt + b_q);
    void* scan_tmp = (void*)(sb + 256 + b_cnt + 2 * b_q);
    prof_begin(kProfQuery, s);
    cudaError_t e = cudaMemsetAsync(sb, 0, 256 + b_cnt, s);
    NNQueries qs{queries, perm, std::isinf(max_dist) ? INFINITY : (float)((double)max_dist * (double)max_dist),
                 INFINITY, idx, sqdist};
    if (e == cudaSuccess) {
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, (int64_t)sm_count() * 8));
        qcell_count_kernel<<<g, 256, 0, s>>>(t->v, queries, (int)m, qbits, qcell, cnt);
        const int nscan = scan_exclusive_u32(cnt, ncell + 1, scan_tmp, s);
        qcell_scatter_kernel<<<g, 256, 0, s>>>(qcell, (int)m, cnt, perm);
        count_launches(2 + nscan);
        switch (t->v.leaf_size) {
            case 4: e = launch_nn<4>(t->v, qs, (int)m, counter, s); break;
            case 8: e = launch_nn<8>(t->v, qs, (int)m, counter, s); break;
            case 16: e = launch_nn<16>(t->v, qs, (int)m, counter, s); break;
            default: e = launch_nn<32>(t->v, qs, (int)m, counter, s); break;
        }
    }
    prof_end(s);
    pool_free(scratch, s);
    if (e != cudaSuccess) return cuda_fail(e, "nn_query_kernel launch");
    return CIL_OK;
}
