// api.cu -- status strings, thread-local error detail, device facts.
#include "internal.cuh"

#include <atomic>
#include <cstring>
#include <vector>

namespace cil {

namespace {
thread_local char g_err[512] = "";
int g_sm[64] = {0};
std::atomic<unsigned long long> g_launches{0};
}  // namespace

void count_launches(int k) { g_launches.fetch_add((unsigned long long)k, std::memory_order_relaxed); }

namespace {
unsigned g_debug_flags = 0;
}
unsigned debug_flags() { return g_debug_flags; }
namespace {
int* g_trace = nullptr;
}
int* debug_trace() { return g_trace; }
namespace {
double g_skin_min = 0.001, g_skin_max = 0.005, g_skin_kappa = 16.0;
}
void cert_skin_params(double* gmin, double* gmax, double* kappa) {
    *gmin = g_skin_min;
    *gmax = g_skin_max;
    *kappa = g_skin_kappa;
}
void set_debug_trace(int* p) { g_trace = p; }
namespace {
unsigned long long* g_stamps = nullptr;
}
unsigned long long* debug_stamps() { return g_stamps; }
void set_debug_stamps(unsigned long long* p) { g_stamps = p; }

namespace {
struct ProfRec { int cls; cudaEvent_t a, b; };
bool g_prof = false;
std::vector<cudaEvent_t> g_pool;
std::vector<ProfRec> g_recs;
cudaEvent_t take_event() {
    if (!g_pool.empty()) { cudaEvent_t e = g_pool.back(); g_pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

namespace {
cudaMemPool_t g_pool_dev[64] = {};
}  // namespace

cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, s);
    if (!g_pool_dev[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool;
        e = cudaMemPoolCreate(&pool, &props);
        if (e != cudaSuccess) return e;
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        g_pool_dev[dev] = pool;
    }
    return cudaMallocFromPoolAsync(p, bytes, g_pool_dev[dev], s);
}

cudaError_t pool_free(void* p, cudaStream_t s) { return cudaFreeAsync(p, s); }

bool prof_on() { return g_prof; }

void prof_begin(int cls, cudaStream_t s) {
    if (!g_prof) return;
    ProfRec r{cls, take_event(), take_event()};
    cudaEventRecord(r.a, s);
    g_recs.push_back(r);
}

void prof_end(cudaStream_t s) {
    if (!g_prof || g_recs.empty()) return;
    cudaEventRecord(g_recs.back().b, s);
}

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

CIL_API cil_status cil_profile_enable(int on) {
    cil::g_prof = on != 0;
    return CIL_OK;
}

CIL_API cil_status cil_profile_read(cil_profile_stats* out) {
    if (!out) return CIL_ERR_INVALID_ARG;
    std::memset(out, 0, sizeof(*out));
    for (auto& r : cil::g_recs) {
        float ms = 0.0f;
        cudaEventSynchronize(r.b);
        if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) ms = 0.0f;
        switch (r.cls) {
            case cil::kProfBuild: out->build_ms += ms; ++out->n_build; break;
            case cil::kProfNN: out->nn_ms += ms; ++out->n_nn; break;
            case cil::kProfAcc: out->acc_ms += ms; ++out->n_acc; break;
            case cil::kProfSel: out->sel_ms += ms; ++out->n_sel; break;
            default: out->query_ms += ms; ++out->n_query; break;
        }
        cil::g_pool.push_back(r.a);
        cil::g_pool.push_back(r.b);
    }
    cil::g_recs.clear();
    return CIL_OK;
}

CIL_API cil_status cil_debug_set_cert_skin(double min_frac, double max_frac, double kappa) {
    if (!(min_frac >= 0.0) || !(max_frac >= min_frac) || max_frac > 1.0 || !(kappa >= 0.0)) return CIL_ERR_INVALID_ARG;
    cil::g_skin_min = min_frac;
    cil::g_skin_max = max_frac;
    cil::g_skin_kappa = kappa;
    return CIL_OK;
}

CIL_API cil_status cil_debug_set_flags(uint32_t flags) {
    cil::g_debug_flags = flags;
    return CIL_OK;
}

CIL_API uint64_t cil_launch_count(void) { return (uint64_t)cil::g_launches.load(); }

CIL_API const char* cil_version(void) { return "cil-b200 0.2 (sm_100a)"; }
