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
    const float4* leafsoa;  // [n_leaves * B]: per leaf rows x[B], y[B], z[B], idx[B] (padding: +inf, idx ~0)
    const unsigned long long* keys;  // [n] sorted 48-bit Morton keys of pts
    const uint32_t* cell_first;      // [2^coarse_bits + 1]: first sorted index with key >> (48-coarse_bits) >= c
    const float4* quant;  // [1]: (min.x, min.y, min.z, cells per unit) of the Morton quantisation
    int n;
    int l_pad;            // power of two >= number of leaves; leaves are nodes l_pad .. 2*l_pad-1
    int levels;           // log2(l_pad)
    int leaf_size;
    int coarse_bits;      // multiple of 3, <= 21
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
    unsigned int work;    // dynamic work counter of the correspondence kernel
    int pad_[2];
};

namespace cil {

void set_error(const char* fmt, ...);
inline cil_status cuda_fail(cudaError_t e, const char* what) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? CIL_ERR_OOM : CIL_ERR_CUDA;
}
int sm_count();            // of the current device (cached per device)
// stream-ordered allocation from the library's own pool (release threshold: never trim, so
// repeated builds/queries after a synchronize do not re-map memory)
cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t s);
cudaError_t pool_free(void* p, cudaStream_t s);
void count_launches(int k);   // diagnostics counter behind cil_launch_count()

// diagnostics: per-launch event timing (cil_profile_*)
enum ProfClass { kProfBuild = 0, kProfNN = 1, kProfAcc = 2, kProfQuery = 3 };
bool prof_on();
void prof_begin(int cls, cudaStream_t s);   // records the start event of a timed region
void prof_end(cudaStream_t s);              // records the end event

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// prim.cu: in-place exclusive scan of uint32 (returns the number of kernels launched)
size_t scan_temp_bytes(int64_t len);
int scan_exclusive_u32(uint32_t* a, int64_t len, void* temp, cudaStream_t s);

}  // namespace cil

#define CIL_CUDA_TRY(expr, what)                              \
    do {                                                      \
        cudaError_t e__ = (expr);                             \
        if (e__ != cudaSuccess) return cil::cuda_fail(e__, what); \
    } while (0)
