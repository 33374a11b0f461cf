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

// The diagnostic engine trace (cil_debug_engine_trace) exists only in a build with -DCIL_TRACE=1
// (tools/variants.sh): its bookkeeping costs the search kernels registers (spills) and time.
#ifndef CIL_TRACE
#define CIL_TRACE 0
#endif

// Largest grid the reduction workspace is sized for (148 SMs x 8 resident CTAs).
constexpr int kMaxCtas = 1184;
// Doubles per per-CTA partial (the 29 point-to-plane / 17 point-to-point sums, padded).
constexpr int kSlots = 32;
// Morton bits per axis (48-bit keys -> 6 radix passes of 8 bits).
constexpr int kMortonBits = 16;

// Uniform grid over the target (index_kind CIL_INDEX_GRID; grid.cu): cell size and dimensions
// are chosen on the device from the bounding box, so the kernels read them from this
// descriptor.  Cell (cx, cy, cz) has the x-major linear id (cz * ny + cy) * nx + cx; a point p
// is in cell clamp(floor((p - lo) * inv_h), 0, n - 1) per axis.  eps bounds the rounding of
// that assignment: every point of cell c lies in [lo + c h - eps, lo + (c + 1) h + eps].
struct GridDesc {
    float4 lo_h;          // lo.x, lo.y, lo.z, h
    float4 inv_eps;       // inv_h, eps, 0, 0
    int4 dims;            // nx, ny, nz, nx * ny * nz
};

// The target, as the kernels see it (device pointers + sizes).  Passed by value.
struct TargetView {
    const float4* opts;   // [n] ORIGINAL order: x, y, z, __int_as_float(sorted position)
    const float4* onrm;   // [n] ORIGINAL order normals (w unused) or nullptr
    const float4* box;    // [2 * 2 * l_pad]: node v (1-based heap) -> box[2v] = lo, box[2v+1] = hi
    const float4* leafsoa;  // [n_leaves * B]: per leaf rows x[B], y[B], z[B], idx[B] (padding: +inf, idx ~0)
    const float4* lbox;   // [2 * n_leaves]: leaf boxes interleaved (lo.x, hi.x, lo.y, hi.y), (lo.z, hi.z, 0, 0)
    const unsigned long long* keys;  // [n] sorted 48-bit Morton keys of pts
    const uint32_t* cell_first;      // [2^coarse_bits + 1]: first sorted index with key >> (48-coarse_bits) >= c
    const float4* quant;  // [1]: (min.x, min.y, min.z, cells per unit) of the Morton quantisation
    int n;
    int l_pad;            // power of two >= number of leaves; leaves are nodes l_pad .. 2*l_pad-1
    int levels;           // log2(l_pad)
    int leaf_size;
    int coarse_bits;      // multiple of 3, <= 21
    const float4* gpts;   // grid: [n] points sorted by cell (x, y, z, original index bits), or nullptr
    const uint32_t* gstart;  // grid: [cells + 1] first sorted position of every cell
    const GridDesc* gdesc;   // grid: descriptor (device)
    int* trace;           // diagnostics only (cil_debug_engine_trace), normally nullptr
    int dbg_mode;         // diagnostics only (cil_debug_set_flags bits 1-2), normally 0
};

struct cil_target {
    TargetView v;
    int64_t n_leaves;
    int has_normals;
    int index_kind;       // CIL_INDEX_BVH or CIL_INDEX_GRID (BVH + grid)
    int device;
    void* mem;            // single stream-ordered allocation holding pts / nrm / box
    void* gmem;           // the grid's allocation (CIL_INDEX_GRID) or nullptr
    size_t bytes;
};

// Device-resident ICP state at the head of the workspace (offsets are read by tools/).
struct alignas(256) IcpState {
    double pose[16];      // 0
    double rmse;          // 128
    long long n_corr;     // 136
    int iters;            // 144: iterations executed so far (= index of the running one)
    int converged;        // 148
    int status;           // 152
    int done;             // 156
    unsigned int ticket;  // 160: last-CTA ticket of the accumulation kernel
    unsigned int work;    // 164: dynamic work counter of the search kernel
    int list_n;           // 168: uncertified queries of the running iteration (diagnostics)
    int plist_n;          // 172: packets in the search list of the running iteration
    long long searched;   // 176: sum over executed iterations of list_n (diagnostics)
    long long pcert_n;    // 184: sum over iterations of point-certified points (diagnostics)
    long long rec_leaf;   // 192: K_sel evaluations of the anchor leaf only (leaf certificate)
    long long rec_list;   // 200: K_sel evaluations of a candidate-leaf list (list certificate)
    long long rec_items;  // 208: leaves of those lists beyond the first
    unsigned int bar_count;  // 216: grid barrier of the persistent projective loop
    unsigned int bar_gen;    // 220
    unsigned int sel_work;   // 224: tile counter of the persistent certificate kernel
};

// Certified warm start: anchor-pose ring of cil_icp_run.
constexpr int kAnchorSlots = 256;   // anchor id = iteration & 255 (low 8 bits of the gap word)

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
unsigned debug_flags();       // cil_debug_set_flags (bit 0: no certified warm start)
int* debug_trace();           // cil_debug_engine_trace buffer (nullptr = off)
void cert_skin_params(double* gmin, double* gmax, double* kappa);   // cil_debug_set_cert_skin
void set_debug_trace(int* p);
unsigned long long* debug_stamps();            // cil_debug_timestamps buffer (nullptr = off)
void set_debug_stamps(unsigned long long* p);

// diagnostics: per-launch event timing (cil_profile_*)
enum ProfClass { kProfBuild = 0, kProfNN = 1, kProfAcc = 2, kProfQuery = 3, kProfSel = 4 };
bool prof_on();
void prof_begin(int cls, cudaStream_t s);   // records the start event of a timed region
void prof_end(cudaStream_t s);              // records the end event

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Programmatic dependent launch: kernels of a dependent chain are launched with the
// programmatic-stream-serialization attribute (launch_pdl); each calls pdl_trigger() first (its
// dependent may be scheduled once every CTA of it has started) and pdl_wait() before it reads
// anything an earlier kernel wrote (the wait returns when the previous grid has completed and
// flushed), so the launch latency of kernel k+1 overlaps the tail of kernel k.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_entry() { pdl_trigger(); pdl_wait(); }

template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// the same launch with or without the attribute (pdl = false: an ordinary stream-ordered launch;
// the kernels' griddepcontrol instructions are then no-ops)
template <class... KArgs, class... Args>
cudaError_t launch_k(bool pdl, void (*kernel)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// target.cu: Morton order of a point set (perm: sorted position -> original index, sorted: the
// points in that order, packed xyz); n >= 1
cudaError_t morton_order_points(const float* pts, int n, uint32_t* perm, float* sorted, cudaStream_t s, int* nlaunch);

// target.cu: stable LSD radix sort of (u64 key, u32 value) pairs by key bits [0, bits)
size_t radix_sort_scratch_bytes(int n);
cudaError_t radix_sort_pairs(unsigned long long* k0, uint32_t* v0, unsigned long long* k1, uint32_t* v1, int n,
                             int bits, void* scratch, cudaStream_t s, int* nlaunch, bool* in_alt, bool pdl = false);

// grid.cu: the uniform grid of a target (after its BVH build; quant = bbox min, qmax = bbox max
// written by the build); allocates from the pool into *mem (owned by the target afterwards)
cudaError_t grid_build(const float* pts, int n, const float4* quant, const float4* qmax, float pts_per_cell,
                       cudaStream_t s, void** mem, size_t* bytes, TargetView* v, int* nlaunch);

// icp.cu (for host.cu): whether (n, m) takes the small-problem path (no source ordering), the
// source-order step of cil_icp_run alone on stream s, and the run with that step already done
bool icp_small_path_nm(int64_t n, int64_t m);
cudaError_t icp_order_source(void* ws, const float* src, int64_t m, cudaStream_t s);
cil_status icp_run_ordered(const cil_target* t, const float* src, int64_t m, const double* pose_init,
                           const cil_icp_params* params, void* ws, size_t ws_bytes, cil_icp_result* res,
                           cil_stream_t stream);

// prim.cu: in-place exclusive scan of uint32 (returns the number of kernels launched)
size_t scan_temp_bytes(int64_t len);
// (len <= 32,768, a multiple of 4: one launch of one block; pdl: programmatic dependent launches)
int scan_exclusive_u32(uint32_t* a, int64_t len, void* temp, cudaStream_t s, bool pdl = false);

}  // namespace cil

#define CIL_CUDA_TRY(expr, what)                              \
    do {                                                      \
        cudaError_t e__ = (expr);                             \
        if (e__ != cudaSuccess) return cil::cuda_fail(e__, what); \
    } while (0)
