// Version and error strings of the semimat_b200 C ABI (include/semimat_b200.h).
#include <cuda_runtime.h>

#include "common.cuh"

#include <atomic>

namespace smx {
static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace smx

extern "C" {

int smx_version(void) { return 100; }

unsigned long long smx_launch_count(void) { return smx::g_launches.load(); }

const char* smx_error_string(int code) {
    switch (code) {
        case SMX_OK: return "ok";
        case SMX_E_ARG: return "invalid argument (size, kind or flag)";
        case SMX_E_ALIGN: return "pointer or leading dimension not 16-byte aligned";
        case SMX_E_WORKSPACE: return "workspace missing or too small";
        case SMX_E_DRIVER: return "CUDA driver entry point unavailable";
        default: return code > 0 ? cudaGetErrorString((cudaError_t)code) : "unknown error";
    }
}

}  // extern "C"
