// grid.cu -- the uniform-grid index of a target (index_kind CIL_INDEX_GRID; BASELINE.json
// north_star (2) "a uniform grid ... built by a device radix sort plus a cell-offset scan ...
// chosen by measurement"; SURVEY.md 7 kernels K1-K4).  Built after the BVH, on the same
// stream, with no host synchronisation:
//   G1 setup (one thread): cell size h from the bounding box so that the box holds about
//      grid_points targets per cell on average, at most 2n cells (host-known allocation);
//   G2 cell id per point + cell counts (atomics);  G3 exclusive scan of the counts (prim.cu)
//   -> the cell-offset table gstart;  G4 scatter of (x, y, z, original index) into cell order.
// The order inside a cell is not deterministic (atomic cursors); nothing depends on it: the
// search keeps the minimum u64 key (d^2 bits, original index), an order-free reduction.
#include "internal.cuh"

#include <algorithm>
#include <cfloat>
#include <cmath>

namespace cil {
namespace {

constexpr int kThreads = 256;

inline int blocks_for(int64_t work) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((work + kThreads - 1) / kThreads, (int64_t)sm_count() * 8));
}

__global__ void grid_setup_kernel(const float4* __restrict__ quant, const float4* __restrict__ qmax, int n,
                                  int64_t cap, float pts_per_cell, GridDesc* __restrict__ G) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const float4 mn = *quant, mx = *qmax;
    const double ext[3] = {(double)mx.x - mn.x, (double)mx.y - mn.y, (double)mx.z - mn.z};
    const double emax = fmax(fmax(ext[0], ext[1]), ext[2]);
    double h = 1.0;
    int dim[3] = {1, 1, 1};
    if (emax > 0.0) {
        // volume with degenerate (flat) axes thickened to 1e-3 of the largest extent
        const double floor_e = emax * 1e-3;
        const double vol = fmax(ext[0], floor_e) * fmax(ext[1], floor_e) * fmax(ext[2], floor_e);
        h = cbrt(vol * (double)pts_per_cell / (double)n);
        for (int it = 0; it < 200; ++it) {
            int64_t tot = 1;
            for (int a = 0; a < 3; ++a) {
                const double c = ceil(ext[a] / h);
                dim[a] = (int)fmin(fmax(c, 1.0), 2147483647.0);
                tot *= dim[a];
                if (tot > cap) break;
            }
            if (tot <= cap) break;
            h *= 1.05;
        }
    }
    const float hf = (float)h;
    const double amax = fmax(fmax(fmax(fabs((double)mn.x), fabs((double)mx.x)), fmax(fabs((double)mn.y), fabs((double)mx.y))),
                             fmax(fabs((double)mn.z), fabs((double)mx.z)));
    // rounding of the cell assignment floor((p - lo) * inv_h) and of the face fma (grid.cuh)
    const float eps = (float)((2.0 * emax + amax + (double)hf) * 0x1p-20) + FLT_MIN;
    G->lo_h = make_float4(mn.x, mn.y, mn.z, hf);
    G->inv_eps = make_float4(1.0f / hf, eps, 0.0f, 0.0f);
    G->dims = make_int4(dim[0], dim[1], dim[2], dim[0] * dim[1] * dim[2]);
}

__device__ __forceinline__ uint32_t cell_of(const GridDesc& G, float x, float y, float z) {
    const float inv_h = G.inv_eps.x;
    auto c1 = [&](float v, float lo, int n) {
        const float f = floorf((v - lo) * inv_h);
        return f >= (float)(n - 1) ? n - 1 : (f >= 0.0f ? (int)f : 0);
    };
    const int cx = c1(x, G.lo_h.x, G.dims.x), cy = c1(y, G.lo_h.y, G.dims.y), cz = c1(z, G.lo_h.z, G.dims.z);
    return (uint32_t)(((int64_t)cz * G.dims.y + cy) * G.dims.x + cx);
}

__global__ void grid_count_kernel(const float* __restrict__ p, int n, const GridDesc* __restrict__ Gp,
                                  uint32_t* __restrict__ cid, uint32_t* __restrict__ cnt) {
    const GridDesc G = *Gp;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t c = cell_of(G, p[3 * (size_t)i], p[3 * (size_t)i + 1], p[3 * (size_t)i + 2]);
        cid[i] = c;
        atomicAdd(cnt + c, 1u);
    }
}

__global__ void grid_scatter_kernel(const float* __restrict__ p, int n, const uint32_t* __restrict__ cid,
                                    uint32_t* __restrict__ cursor, float4* __restrict__ gpts) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t pos = atomicAdd(cursor + cid[i], 1u);
        gpts[pos] = make_float4(p[3 * (size_t)i], p[3 * (size_t)i + 1], p[3 * (size_t)i + 2], __uint_as_float((uint32_t)i));
    }
}

}  // namespace

cudaError_t grid_build(const float* pts, int n, const float4* quant, const float4* qmax, float pts_per_cell,
                       cudaStream_t s, void** mem, size_t* bytes, TargetView* v, int* nlaunch) {
    const int64_t cap = std::max<int64_t>(64, 2 * (int64_t)n);
    const size_t b_pts = align_up((size_t)n * 16, 256);
    const size_t b_start = align_up((size_t)(cap + 1) * 4, 256);
    const size_t b_desc = 256;
    *bytes = b_pts + b_start + b_desc;
    void* m = nullptr;
    cudaError_t e = pool_alloc(&m, *bytes, s);
    if (e != cudaSuccess) return e;
    char* base = (char*)m;
    float4* gpts = (float4*)base;
    uint32_t* gstart = (uint32_t*)(base + b_pts);
    GridDesc* G = (GridDesc*)(base + b_pts + b_start);
    // scratch: cell id per point, the scatter cursors, scan temp
    const size_t s_cid = align_up((size_t)n * 4, 256);
    const size_t s_scan = scan_temp_bytes(cap + 1);
    void* tmp = nullptr;
    e = pool_alloc(&tmp, s_cid + b_start + s_scan, s);
    if (e != cudaSuccess) { pool_free(m, s); return e; }
    uint32_t* cid = (uint32_t*)tmp;
    uint32_t* cursor = (uint32_t*)((char*)tmp + s_cid);
    void* scan_tmp = (void*)((char*)tmp + s_cid + b_start);
    int nl = 0;
    grid_setup_kernel<<<1, 32, 0, s>>>(quant, qmax, n, cap, pts_per_cell, G);
    cudaMemsetAsync(gstart, 0, (size_t)(cap + 1) * 4, s);
    grid_count_kernel<<<blocks_for(n), kThreads, 0, s>>>(pts, n, G, cid, gstart);
    nl += 2 + scan_exclusive_u32(gstart, cap + 1, scan_tmp, s);
    cudaMemcpyAsync(cursor, gstart, (size_t)(cap + 1) * 4, cudaMemcpyDeviceToDevice, s);
    grid_scatter_kernel<<<blocks_for(n), kThreads, 0, s>>>(pts, n, cid, cursor, gpts);
    ++nl;
    e = cudaGetLastError();
    pool_free(tmp, s);
    if (e != cudaSuccess) { pool_free(m, s); return e; }
    v->gpts = gpts;
    v->gstart = gstart;
    v->gdesc = G;
    *mem = m;
    if (nlaunch) *nlaunch = nl;
    return cudaSuccess;
}

}  // namespace cil
