// Version and error strings of the semimat_b200 C ABI (include/semimat_b200.h).
#include <cuda_runtime.h>

#include "common.cuh"

#include <atomic>

namespace smx {
static std::atomic<unsigned long long> g_launches{0};
static std::atomic<int> g_bounded{1};
static std::atomic<int> g_lookahead{1};
int lookahead_enabled() { return g_lookahead.load(std::memory_order_relaxed); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int bounded_fastpath_enabled() { return g_bounded.load(std::memory_order_relaxed); }

int scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
    static bool pool_configured[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return SMX_E_ARG;
    if (!pool_configured[dev]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            unsigned long long threshold = ~0ULL;   // keep freed blocks cached
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
        }
        pool_configured[dev] = true;
    }
    cudaError_t e = cudaMallocAsync(p, bytes, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return (int)e;
    }
    return SMX_OK;
}

int scratch_free(void* p, cudaStream_t s) {
    cudaError_t e = cudaFreeAsync(p, s);
    return e == cudaSuccess ? SMX_OK : (int)e;
}

int side_stream(SideStream** out) {
    static SideStream per_dev[64];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    if (dev < 0 || dev >= 64) return SMX_E_ARG;
    SideStream& f = per_dev[dev];
    if (!f.side) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if ((e = cudaStreamCreateWithPriority(&f.side, cudaStreamNonBlocking, hi)) != cudaSuccess) return (int)e;
        if ((e = cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming)) != cudaSuccess) return (int)e;
        if ((e = cudaEventCreateWithFlags(&f.join, cudaEventDisableTiming)) != cudaSuccess) return (int)e;
    }
    *out = &f;
    return SMX_OK;
}
}  // namespace smx

extern "C" {

int smx_version(void) { return 100; }

unsigned long long smx_launch_count(void) { return smx::g_launches.load(); }

int smx_set_bounded_fastpath(int enable) {
    return smx::g_bounded.exchange(enable ? 1 : 0);
}

int smx_set_fw_lookahead(int enable) {
    return smx::g_lookahead.exchange(enable ? 1 : 0);
}

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
