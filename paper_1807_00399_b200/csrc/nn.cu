// nn.cu -- cil_nn_query: exact 1-NN of independent queries (SURVEY.md 8(a) row a2,
// BASELINE.json configs[1]; "k-NN ... queries").
#include "internal.cuh"
#include "search.cuh"

#include <algorithm>
#include <cmath>

namespace cil {
namespace {

constexpr int kNNThreads = 256;

struct NNQueries {
    const float* q;
    float bound2;
    int32_t* idx;
    float* sqd;
    __device__ __forceinline__ bool load(int i, DF3& s, unsigned long long& init, int& hint) const {
        s.hx = q[3 * (size_t)i]; s.hy = q[3 * (size_t)i + 1]; s.hz = q[3 * (size_t)i + 2];
        s.lx = s.ly = s.lz = 0.0f;
        init = bound_key(bound2);
        hint = -1;
        return true;
    }
    __device__ __forceinline__ void store(int i, unsigned long long best, int, const DF3&) const {
        const bool found = best != bound_key(bound2);
        if (idx) idx[i] = found ? (int32_t)key_idx(best) : -1;
        if (sqd) sqd[i] = found ? key_d2(best) : INFINITY;
    }
};

template <int B>
__global__ void __launch_bounds__(kNNThreads)
nn_query_kernel(TargetView T, NNQueries qs, int m, unsigned int* counter) {
    nn_packet_engine<B>(T, qs, m, counter);
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
    nn_query_kernel<B><<<blocks, kNNThreads, 0, s>>>(T, qs, m, counter);
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
    NNQueries qs{queries, std::isinf(max_dist) ? INFINITY : (float)((double)max_dist * (double)max_dist),
                 idx, sqdist};
    cudaStream_t s = (cudaStream_t)stream;
    unsigned int* counter = nullptr;   // dynamic work counter (stream-ordered scratch)
    CIL_CUDA_TRY(cudaMallocAsync((void**)&counter, sizeof(unsigned int), s), "cudaMallocAsync(counter)");
    cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned int), s);
    if (e == cudaSuccess) {
        switch (t->v.leaf_size) {
            case 4: e = launch_nn<4>(t->v, qs, (int)m, counter, s); break;
            case 8: e = launch_nn<8>(t->v, qs, (int)m, counter, s); break;
            case 16: e = launch_nn<16>(t->v, qs, (int)m, counter, s); break;
            default: e = launch_nn<32>(t->v, qs, (int)m, counter, s); break;
        }
    }
    cudaFreeAsync(counter, s);
    if (e != cudaSuccess) return cuda_fail(e, "nn_query_kernel launch");
    return CIL_OK;
}
