// nn.cu -- cil_nn_query: exact 1-NN of independent queries (SURVEY.md 8(a) row a2,
// BASELINE.json configs[1]; "k-NN ... queries").
#include "internal.cuh"
#include "search.cuh"

#include <algorithm>
#include <cmath>

namespace cil {
namespace {

constexpr int kNNThreads = 256;

template <int B>
__global__ void __launch_bounds__(kNNThreads)
nn_query_kernel(TargetView T, const float* __restrict__ q, int m, float bound2,
                int32_t* __restrict__ idx, float* __restrict__ sqd) {
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        DF3 s;
        s.hx = q[3 * (size_t)i]; s.hy = q[3 * (size_t)i + 1]; s.hz = q[3 * (size_t)i + 2];
        s.lx = s.ly = s.lz = 0.0f;
        const unsigned long long none = bound_key(bound2);
        unsigned long long best = none;
        int bpos = -1;
        bvh_nearest<B>(T, s, best, bpos);
        const bool found = best != none;
        if (idx) idx[i] = found ? (int32_t)key_idx(best) : -1;
        if (sqd) sqd[i] = found ? key_d2(best) : INFINITY;
    }
}

template <int B>
cudaError_t launch_nn(const TargetView& T, const float* q, int m, float bound2, int32_t* idx, float* sqd,
                      cudaStream_t s) {
    static int occ = -1;   // per-process cache; all supported devices are sm_100a
    if (occ < 0) {
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, nn_query_kernel<B>, kNNThreads, 0);
        if (e != cudaSuccess) return e;
    }
    int blocks = (int)std::min<int64_t>(((int64_t)m + kNNThreads - 1) / kNNThreads, (int64_t)sm_count() * std::max(occ, 1));
    nn_query_kernel<B><<<std::max(blocks, 1), kNNThreads, 0, s>>>(T, q, m, bound2, idx, sqd);
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
    const float bound2 = std::isinf(max_dist) ? INFINITY : (float)((double)max_dist * (double)max_dist);
    cudaError_t e;
    cudaStream_t s = (cudaStream_t)stream;
    switch (t->v.leaf_size) {
        case 4: e = launch_nn<4>(t->v, queries, (int)m, bound2, idx, sqdist, s); break;
        case 8: e = launch_nn<8>(t->v, queries, (int)m, bound2, idx, sqdist, s); break;
        case 16: e = launch_nn<16>(t->v, queries, (int)m, bound2, idx, sqdist, s); break;
        default: e = launch_nn<32>(t->v, queries, (int)m, bound2, idx, sqdist, s); break;
    }
    if (e != cudaSuccess) return cuda_fail(e, "nn_query_kernel launch");
    return CIL_OK;
}
