// api.cu -- status strings, thread-local error detail, device facts.
#include "internal.cuh"

#include <atomic>
#include <cstring>

namespace cil {

namespace {
thread_local char g_err[512] = "";
int g_sm[64] = {0};
std::atomic<unsigned long long> g_launches{0};
}  // namespace

void count_launches(int k) { g_launches.fetch_add((unsigned long long)k, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int sm_count() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (g_sm[dev] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        g_sm[dev] = v;
    }
    return g_sm[dev];
}

}  // namespace cil

CIL_API const char* cil_status_string(cil_status s) {
    switch (s) {
        case CIL_OK: return "CIL_OK";
        case CIL_ERR_INVALID_ARG: return "CIL_ERR_INVALID_ARG";
        case CIL_ERR_EMPTY_TARGET: return "CIL_ERR_EMPTY_TARGET";
        case CIL_ERR_NO_NORMALS: return "CIL_ERR_NO_NORMALS";
        case CIL_ERR_CUDA: return "CIL_ERR_CUDA";
        case CIL_ERR_OOM: return "CIL_ERR_OOM";
        case CIL_ERR_WORKSPACE: return "CIL_ERR_WORKSPACE";
        case CIL_ERR_DEGENERATE: return "CIL_ERR_DEGENERATE";
        case CIL_NO_CORRESPONDENCES: return "CIL_NO_CORRESPONDENCES";
    }
    return "CIL_UNKNOWN_STATUS";
}

CIL_API const char* cil_last_error(void) { return cil::g_err; }

CIL_API uint64_t cil_launch_count(void) { return (uint64_t)cil::g_launches.load(); }

CIL_API const char* cil_version(void) { return "cil-b200 0.1 (sm_100a)"; }
