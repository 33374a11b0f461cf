// host.cu -- cil_icp_align_host: one frame pair end to end from HOST buffers (cil.h): H2D copies
// (the source and its ordering step on a second stream, overlapping the target's copy and index
// build), cil_target_build, cil_icp_run, the result copied back.  Only plumbing around the device-pointer calls: no arithmetic here.
#include "internal.cuh"

#include <algorithm>

namespace cil {
namespace {

// per host thread and device: the second stream and its events (created once, kept)
struct SideStream {
    int dev = -1;
    cudaStream_t s = nullptr;
    cudaEvent_t ready = nullptr, copied = nullptr;
};

cudaError_t side_stream(SideStream** out) {
    thread_local SideStream side[8];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    SideStream& S = side[dev & 7];
    if (S.dev != dev) {
        if (S.s) { cudaStreamDestroy(S.s); cudaEventDestroy(S.ready); cudaEventDestroy(S.copied); S = SideStream{}; }
        if ((e = cudaStreamCreateWithFlags(&S.s, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&S.ready, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&S.copied, cudaEventDisableTiming)) != cudaSuccess) return e;
        S.dev = dev;
    }
    *out = &S;
    return cudaSuccess;
}

}  // namespace
}  // namespace cil

using namespace cil;

CIL_API cil_status cil_icp_align_host(const float* target, const float* normals, int64_t n, const float* source,
                                      int64_t m, const double* pose_init, const cil_icp_params* params,
                                      const cil_index_params* index, cil_icp_result* result, cil_stream_t stream) {
    if (!result) { set_error("cil_icp_align_host: result is NULL"); return CIL_ERR_INVALID_ARG; }
    if (!params) { set_error("cil_icp_align_host: params is NULL"); return CIL_ERR_INVALID_ARG; }
    if (n == 0) { set_error("cil_icp_align_host: empty target (n == 0)"); return CIL_ERR_EMPTY_TARGET; }
    if (n < 0 || n > INT32_MAX || m < 0 || m > INT32_MAX) {
        set_error("cil_icp_align_host: n=%lld / m=%lld out of range", (long long)n, (long long)m);
        return CIL_ERR_INVALID_ARG;
    }
    if (!target || (m > 0 && !source)) { set_error("cil_icp_align_host: target/source is NULL"); return CIL_ERR_INVALID_ARG; }
    const size_t ws_bytes = cil_icp_workspace_bytes(m, params);
    if (ws_bytes == 0) { set_error("cil_icp_align_host: bad ICP parameters"); return CIL_ERR_INVALID_ARG; }
    cudaStream_t s = (cudaStream_t)stream;
    SideStream* side = nullptr;
    CIL_CUDA_TRY(side_stream(&side), "cil_icp_align_host: side stream");

    // one stream-ordered block: target | normals | source | pose | result | workspace
    const size_t b_t = align_up((size_t)n * 12, 256), b_n = normals ? b_t : 0;
    const size_t b_s = align_up((size_t)std::max<int64_t>(m, 1) * 12, 256);
    const size_t b_pose = 256, b_res = align_up(sizeof(cil_icp_result), 256);
    void* mem = nullptr;
    {
        cudaError_t e = pool_alloc(&mem, b_t + b_n + b_s + b_pose + b_res + align_up(ws_bytes, 256), s);
        if (e != cudaSuccess) { (void)cudaGetLastError(); set_error("cil_icp_align_host: device allocation failed"); return CIL_ERR_OOM; }
    }
    char* base = (char*)mem;
    float* d_t = (float*)base;
    float* d_n = normals ? (float*)(base + b_t) : nullptr;
    float* d_s = (float*)(base + b_t + b_n);
    double* d_pose = (double*)(base + b_t + b_n + b_s);
    cil_icp_result* d_res = (cil_icp_result*)(base + b_t + b_n + b_s + b_pose);
    void* d_ws = (void*)(base + b_t + b_n + b_s + b_pose + b_res);
    static const double kIdentity[16] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};

    cil_target* t = nullptr;
    cil_status rc = CIL_OK;
    cudaError_t e = cudaSuccess;
    auto fail = [&](const char* what) {
        if (rc == CIL_OK && e != cudaSuccess) rc = cuda_fail(e, what);
        // the second stream may still be copying from the caller's buffers into the block:
        // drain it before the block is released and before the caller gets its buffers back
        cudaStreamSynchronize(side->s);
        if (t) cil_target_free(t, stream);
        pool_free(mem, s);
        cudaStreamSynchronize(s);
        return rc;
    };
    // the block exists once `stream` reaches this point: the second stream starts after it
    if ((e = cudaEventRecord(side->ready, s)) != cudaSuccess) return fail("cudaEventRecord");
    if ((e = cudaStreamWaitEvent(side->s, side->ready, 0)) != cudaSuccess) return fail("cudaStreamWaitEvent");
    if (m > 0 && (e = cudaMemcpyAsync(d_s, source, (size_t)m * 12, cudaMemcpyHostToDevice, side->s)) != cudaSuccess)
        return fail("H2D source");
    if ((e = cudaMemcpyAsync(d_pose, pose_init ? pose_init : kIdentity, 128, cudaMemcpyHostToDevice, side->s)) != cudaSuccess)
        return fail("H2D pose");
    // the run's source-order step depends only on the source: on the second stream too, under the
    // target's copy and build (the small-problem path does not order its source)
    const bool ordered = m > 0 && !icp_small_path_nm(n, m);
    if (ordered && (e = icp_order_source(d_ws, d_s, m, side->s)) != cudaSuccess) return fail("source order");
    if ((e = cudaEventRecord(side->copied, side->s)) != cudaSuccess) return fail("cudaEventRecord");
    // target (+ normals) on the launching stream: the build needs them first
    if ((e = cudaMemcpyAsync(d_t, target, (size_t)n * 12, cudaMemcpyHostToDevice, s)) != cudaSuccess) return fail("H2D target");
    if (d_n && (e = cudaMemcpyAsync(d_n, normals, (size_t)n * 12, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return fail("H2D normals");
    if ((rc = cil_target_build(d_t, d_n, n, index, stream, &t)) != CIL_OK) return fail("");
    if ((e = cudaStreamWaitEvent(s, side->copied, 0)) != cudaSuccess) return fail("cudaStreamWaitEvent");
    rc = ordered ? icp_run_ordered(t, d_s, m, d_pose, params, d_ws, ws_bytes, d_res, stream)
                 : cil_icp_run(t, d_s, m, d_pose, params, d_ws, ws_bytes, d_res, nullptr, stream);
    if (rc != CIL_OK) return fail("");
    cil_icp_result tmp;
    if ((e = cudaMemcpyAsync(&tmp, d_res, sizeof(tmp), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return fail("D2H result");
    cil_target_free(t, stream);
    t = nullptr;
    pool_free(mem, s);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "cil_icp_align_host: synchronize");
    *result = tmp;
    return CIL_OK;
}
