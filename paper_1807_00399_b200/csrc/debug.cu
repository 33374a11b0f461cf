// debug.cu -- diagnostics only (not on the hot path): per-query traversal statistics of
// the exact NN search engine, for tuning the index (DFS nodes, leaves, ascent levels).
#include "internal.cuh"
#include "search.cuh"

namespace cil {
namespace {
template <int B>
struct StatQueries {
    const float* q;
    Pose34 P;
    float bound2;
    const int* hint_pos;     // nullable: warm hints (sorted target positions)
    __device__ bool load(int i, DF3& s, unsigned long long& init, int& hint) const {
        s = transform_df(P, q[3 * (size_t)i], q[3 * (size_t)i + 1], q[3 * (size_t)i + 2]);
        init = bound_key(bound2);
        const int jp = hint_pos ? hint_pos[i] : -1;
        hint = jp >= 0 ? jp / B : -1;
        return true;
    }
    __device__ void store(int, unsigned long long, int, const DF3&) const {}
};

struct PerLaneStats {
    int* nodes;
    int* leaves;
    int* levels;
};

template <int B>
__global__ void nn_stats_kernel(TargetView T, StatQueries<B> qs, int m, int* nodes, int* leaves, int* levels,
                                unsigned int* counter) {
    // one query per thread, no engine: sequential per-lane search with counters
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        DF3 s;
        unsigned long long init;
        int hint;
        qs.load(i, s, init, hint);
        if (hint < 0) hint = coarse_hint_leaf(T, s);
        LaneSearch L;
        LaneStack K;
        lane_start(L, T, s, init, hint);
        const NegQuery nq = neg_query(s);
        CountStats st;
        int leaf = hint;
        while (leaf >= 0) {
            st.leaf();
            eval_leaf<B>(T, nq, leaf, L.best, L.bpos);
            leaf = next_leaf(L, K, T, &st);
        }
        nodes[i] = st.nodes;
        leaves[i] = st.leaves;
        levels[i] = st.levels;
    }
    (void)counter;
}
}  // namespace
}  // namespace cil

using namespace cil;

// Diagnostics: DFS nodes / leaves / ascent levels visited by the exact NN search of each
// transformed query (hint_pos: optional warm-start positions, NULL = cold coarse hints).
CIL_API cil_status cil_debug_nn_stats(const cil_target* t, const float* q, int64_t m, const double* pose,
                                      float max_dist, const int32_t* hint_pos, int32_t* nodes, int32_t* leaves,
                                      int32_t* levels, cil_stream_t stream) {
    if (!t || !q || !pose || !nodes || !leaves || !levels || m <= 0 || m > INT32_MAX) return CIL_ERR_INVALID_ARG;
    const float b2 = isinf(max_dist) ? INFINITY : (float)((double)max_dist * max_dist);
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = (int)((m + 255) / 256);
    double P[16];
    if (cudaMemcpy(P, pose, sizeof(P), cudaMemcpyDeviceToHost) != cudaSuccess) return CIL_ERR_CUDA;
#define CIL_STATS_CASE(BB)                                                                     \
    case BB: {                                                                                 \
        StatQueries<BB> qs;                                                                    \
        qs.q = q; qs.bound2 = b2; qs.hint_pos = hint_pos;                                      \
        for (int k = 0; k < 12; ++k) qs.P.r[k] = P[k];                                         \
        nn_stats_kernel<BB><<<blocks, 256, 0, s>>>(t->v, qs, (int)m, nodes, leaves, levels, nullptr); \
        break;                                                                                 \
    }
    switch (t->v.leaf_size) {
        CIL_STATS_CASE(4)
        CIL_STATS_CASE(8)
        CIL_STATS_CASE(16)
        CIL_STATS_CASE(32)
    }
#undef CIL_STATS_CASE
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? CIL_OK : cuda_fail(e, "nn_stats_kernel");
}
