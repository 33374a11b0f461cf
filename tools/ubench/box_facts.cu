// box_facts.cu -- SURVEY.md 7 step 0 "box facts" measured on the GPU box (one JSON object on
// stdout, committed as profiles/box.json): issue throughput of FFMA / FFMA2 / FADD2 (the packed
// FP32 ops the leaf evaluation is written with), the SM clock under that load, dependent-load
// latency by footprint (L1 / L2 / HBM pointer chase), and read bandwidth by footprint (the L2
// knee).  Standalone diagnostic, not part of libcil.so.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o box_facts tools/ubench/box_facts.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int kIters = 65536;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// 8 independent chains per thread, one op per chain per step
__global__ void ffma_kernel(float* out, float a, float b, unsigned long long* clk) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
    const unsigned long long c0 = clock64(), g0 = gtimer();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
    }
    const unsigned long long c1 = clock64(), g1 = gtimer();
    float s = 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.0f) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = g1 - g0; }
}

__global__ void ffma2_kernel(float* out, float a, float b, unsigned long long* clk) {
    float2 x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x * 1e-3f + k, threadIdx.x * 2e-3f + k);
    const float2 A = make_float2(a, a), Bv = make_float2(b, b);
    const unsigned long long c0 = clock64(), g0 = gtimer();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __ffma2_rn(x[k], A, Bv);
    }
    const unsigned long long c1 = clock64(), g1 = gtimer();
    float s = 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
    if (s == 12345.0f) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = g1 - g0; }
}

__global__ void fadd2_kernel(float* out, float b, unsigned long long* clk) {
    float2 x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x * 1e-3f + k, threadIdx.x * 2e-3f + k);
    const float2 Bv = make_float2(b, -b);
    const unsigned long long c0 = clock64(), g0 = gtimer();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __fadd2_rn(x[k], Bv);
    }
    const unsigned long long c1 = clock64(), g1 = gtimer();
    float s = 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
    if (s == 12345.0f) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = g1 - g0; }
}

// pointer chase: one thread, dependent loads
__global__ void chase_kernel(const uint32_t* next, int warm, int steps, uint32_t* sink, unsigned long long* clk) {
    uint32_t p = 0;
    for (int i = 0; i < warm; ++i) p = next[p];          // (small footprints: one full cycle first)
    const unsigned long long c0 = clock64();
    for (int i = 0; i < steps; ++i) p = next[p];
    const unsigned long long c1 = clock64();
    *sink = p;
    *clk = c1 - c0;
}

__global__ void read_kernel(const float4* __restrict__ a, size_t n, int reps, float* out) {
    float4 s = make_float4(0, 0, 0, 0);
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            const float4 v = __ldcg(a + i);
            s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
        }
    if (s.x + s.y + s.z + s.w == 12345.0f) out[0] = s.x;
}

int main() {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int l2 = 0;
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    float* out;
    unsigned long long* clk;
    CK(cudaMalloc(&out, 16));
    CK(cudaMalloc(&clk, 16));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    printf("{\n \"sms\": %d,\n \"l2_bytes_attribute\": %d,\n", sms, l2);

    // ---- issue throughput: blocks of 256 threads, 8 per SM (64 warps/SM)
    const int blocks = sms * 8, threads = 256;
    auto run_alu = [&](const char* name, auto launch, double lanes_per_inst) -> int {
        launch(); CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        unsigned long long c[2] = {0, 0};
        CK(cudaMemcpy(c, clk, 16, cudaMemcpyDeviceToHost));
        const double warp_inst = (double)blocks * (threads / 32) * kIters * 8.0;
        const double per_s = warp_inst / (ms * 1e-3);
        // SM clock of one SM during its loop: clock64 cycles over %globaltimer nanoseconds
        const double mhz = (double)c[0] / (double)c[1] * 1e3;
        const double per_clk_sm = per_s / sms / (mhz * 1e6);
        printf(" \"%s\": {\"warp_inst_per_s\": %.4g, \"warp_inst_per_clk_per_sm\": %.3f, \"fp32_lane_ops_per_clk_per_sm\": %.1f, \"sm_mhz_from_clock64\": %.0f, \"ms\": %.4f},\n",
               name, per_s, per_clk_sm, per_clk_sm * 32 * lanes_per_inst, mhz, ms);
        return 0;
    };
    if (run_alu("ffma", [&] { ffma_kernel<<<blocks, threads>>>(out, 0.999f, 1e-3f, clk); }, 1.0)) return 1;
    if (run_alu("ffma2", [&] { ffma2_kernel<<<blocks, threads>>>(out, 0.999f, 1e-3f, clk); }, 2.0)) return 1;
    if (run_alu("fadd2", [&] { fadd2_kernel<<<blocks, threads>>>(out, 1e-3f, clk); }, 2.0)) return 1;

    // ---- dependent-load latency by footprint (random cyclic permutation, 128-byte stride)
    printf(" \"chase_latency_cycles\": {");
    const size_t foots[] = {16 << 10, 96 << 10, 4 << 20, 32 << 20, 96 << 20, 512 << 20};
    bool first = true;
    for (size_t fb : foots) {
        const size_t n = fb / 4, stride = 32, nodes = n / stride;
        std::vector<uint32_t> order(nodes);
        for (size_t i = 0; i < nodes; ++i) order[i] = (uint32_t)i;
        uint64_t st = 1807;
        for (size_t i = nodes - 1; i > 0; --i) {
            st = st * 6364136223846793005ull + 1442695040888963407ull;
            std::swap(order[i], order[(st >> 33) % (i + 1)]);
        }
        std::vector<uint32_t> h(n, 0);
        for (size_t i = 0; i < nodes; ++i) h[order[i] * stride] = order[(i + 1) % nodes] * (uint32_t)stride;
        uint32_t* d;
        CK(cudaMalloc(&d, n * 4));
        CK(cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice));
        // small footprints: the whole cycle twice (warm); large ones: one cold pass over fewer
        // nodes than the cycle holds (every load a new line)
        const bool small = nodes <= 100000;
        const int steps = small ? (int)std::min<size_t>(2 * nodes, 20000) : 20000;
        chase_kernel<<<1, 1>>>(d, small ? (int)nodes : 0, steps, (uint32_t*)out, clk);
        unsigned long long c = 0;
        CK(cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost));
        printf("%s\"%zu_KiB\": %.0f", first ? "" : ", ", fb >> 10, (double)c / steps);
        first = false;
        CK(cudaFree(d));
    }
    printf("},\n");

    // ---- read bandwidth by footprint (ld.global.cg, the footprint re-read 8x per launch)
    printf(" \"read_gbs_by_footprint\": {");
    first = true;
    const size_t rfoots[] = {16ull << 20, 48ull << 20, 80ull << 20, 112ull << 20, 128ull << 20, 160ull << 20, 256ull << 20, 1024ull << 20};
    for (size_t fb : rfoots) {
        float4* a;
        CK(cudaMalloc(&a, fb));
        CK(cudaMemset(a, 0, fb));
        const size_t n = fb / 16;
        const int reps = fb >= (512ull << 20) ? 2 : 8;
        read_kernel<<<sms * 8, 256>>>(a, n, 1, out);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        read_kernel<<<sms * 8, 256>>>(a, n, reps, out);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("%s\"%zu_MiB\": %.0f", first ? "" : ", ", fb >> 20, (double)fb * reps / (ms * 1e-3) / 1e9);
        first = false;
        CK(cudaFree(a));
    }
    printf("}\n}\n");
    return 0;
}
