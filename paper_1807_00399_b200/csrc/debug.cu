// debug.cu -- diagnostics only (not on the hot path).
#include "internal.cuh"

using namespace cil;

// Diagnostics: every engine launch after this call writes 16 ints per processed query slot
// into buf (device, >= 16 * slots ints; see include/cil.h); buf == NULL switches tracing off.
CIL_API cil_status cil_debug_engine_trace(int32_t* buf) {
    if (buf && !CIL_TRACE) {
        cil::set_error("cil_debug_engine_trace: library built without the trace (rebuild with -DCIL_TRACE=1)");
        return CIL_ERR_INVALID_ARG;
    }
    cil::set_debug_trace(buf);
    return CIL_OK;
}

// Diagnostics: per-iteration %globaltimer stamps of the ICP kernels (see include/cil.h).
CIL_API cil_status cil_debug_timestamps(uint64_t* buf) {
    cil::set_debug_stamps(reinterpret_cast<unsigned long long*>(buf));
    return CIL_OK;
}
