// Microbenchmark (diagnostics only): latency of fp64 primitives and of 6x6 solve variants on
// one warp, timed with clock64 inside the kernel.  nvcc -arch=sm_100a -O3 solve_lat.cu
#include <cstdio>
#include <cmath>

__device__ double sink;
#define TICKD(t, v) asm volatile("mov.u64 %0, %%clock64;" : "=l"(t), "+d"(v))
#define TICKF(t, v) asm volatile("mov.u64 %0, %%clock64;" : "=l"(t), "+f"(v))

__global__ void lat(double a, double b, long long* out) {
    long long t0, t1, t2, t3, t4, t5, t6, t7, u;
    double x = a;
    TICKD(t0, x);
    for (int i = 0; i < 64; ++i) x = fma(x, b, a);
    TICKD(t1, x);
    double y = a + (double)(t1 & 1);
    TICKD(u, y); t1 = u;
    for (int i = 0; i < 16; ++i) y = sqrt(y + 1.0);
    TICKD(t2, y);
    double z = a + (double)(t2 & 1);
    TICKD(u, z); t2 = u;
    for (int i = 0; i < 16; ++i) z = 1.0 / (z + 1.0);
    TICKD(t3, z);
    double w = a + (double)(t3 & 1);
    TICKD(u, w); t3 = u;
    for (int i = 0; i < 16; ++i) w = rsqrt(w + 1.0);
    TICKD(t4, w);
    double s = a + (double)(t4 & 1), c;
    TICKD(u, s); t4 = u;
    for (int i = 0; i < 4; ++i) { sincos(s, &s, &c); s += c; }
    TICKD(t5, s);
    float f = (float)a + (float)(t5 & 1);
    TICKF(u, f); t5 = u;
    for (int i = 0; i < 64; ++i) f = fmaf(f, (float)b, (float)a);
    TICKF(t6, f);
    double q = a + (double)(t6 & 1);
    TICKD(u, q); t6 = u;
    for (int i = 0; i < 16; ++i) q = __shfl_sync(0xffffffffu, q, (threadIdx.x + 1) & 31) + 1.0;
    TICKD(t7, q);
    t1 = t1; (void)u;
    if (threadIdx.x == 0) {
        out[0] = (t1 - t0) / 64; out[1] = (t2 - t1) / 16;  /* t1->t2 includes a re-tick */ out[2] = (t3 - t2) / 16; out[3] = (t4 - t3) / 16;
        out[4] = (t5 - t4) / 4; out[5] = (t6 - t5) / 64; out[6] = (t7 - t6) / 16;
    }
    sink = x + y + z + w + s + f + q;
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    long long h[8];
    for (int threads : {1, 32}) {
        lat<<<1, threads>>>(0.5, 0.999, d);
        lat<<<1, threads>>>(0.5, 0.999, d);
        cudaMemcpy(h, d, 56, cudaMemcpyDeviceToHost);
        printf("threads %d: cycles per dep. op: dfma %lld  dsqrt %lld  ddiv %lld  drsqrt %lld  dsincos %lld  ffma %lld  shfl.f64 %lld\n",
               threads, h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
    }
    return 0;
}
