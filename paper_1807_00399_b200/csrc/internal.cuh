// internal.cuh -- host-side internals shared by the libcil.so translation units.
// (Product code.  Shares nothing with oracle/.)
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <string>

#include "cil.h"

#define CIL_API extern "C" __attribute__((visibility("default")))

// Largest grid the reduction workspace is sized for (148 SMs x 8 resident CTAs).
constexpr int kMaxCtas = 1184;
// Doubles per per-CTA partial (the 29 point-to-plane / 17 point-to-point sums, padded).
constexpr int kSlots = 32;
// Morton bits per axis (48-bit keys -> 6 radix passes of 8 bits).
constexpr int kMortonBits = 16;

// The target, as the kernels see it (device pointers + sizes).  Passed by value.
struct TargetView {
    const float4* pts;    // [n] sorted by Morton key: x, y, z, __int_as_float(original index)
    const float4* nrm;    // [n] normals in the same order (w unused) or nullptr
    const float4* box;    // [2 * 2 * l_pad]: node v (1-based heap) -> box[2v] = lo, box[2v+1] = hi
    int n;
    int l_pad;            // power of two >= number of leaves; leaves are nodes l_pad .. 2*l_pad-1
    int leaf_size;
};

struct cil_target {
    TargetView v;
    int64_t n_leaves;
    int has_normals;
    int device;
    void* mem;            // single stream-ordered allocation holding pts / nrm / box
    size_t bytes;
};

// Device-resident ICP state at the head of the workspace.
struct alignas(256) IcpState {
    double pose[16];
    double rmse;
    long long n_corr;
    int iters;
    int converged;
    int status;
    int done;
    unsigned int ticket;
    int pad_[3];
};

namespace cil {

void set_error(const char* fmt, ...);
inline cil_status cuda_fail(cudaError_t e, const char* what) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? CIL_ERR_OOM : CIL_ERR_CUDA;
}
int sm_count();            // of the current device (cached per device)
void count_launches(int k);   // diagnostics counter behind cil_launch_count()

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace cil

#define CIL_CUDA_TRY(expr, what)                              \
    do {                                                      \
        cudaError_t e__ = (expr);                             \
        if (e__ != cudaSuccess) return cil::cuda_fail(e__, what); \
    } while (0)
