// Shared helpers for the semimat_b200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <utility>

#include "semimat_b200.h"   // include/ (on the -I path of _build.py)

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "semimat_b200 targets sm_100a only"
#endif

namespace smx {
// Counts every kernel this library launches (smx_launch_count), so bench.py
// reports launches it observed rather than a formula.
void count_launch();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `func` on the current
// device, done once per (device, function, size) and thread-safe: a process
// that drives several GPUs, or calls from several threads, never launches a
// kernel whose > 48 KB opt-in was set on another device only.
int set_max_smem(const void* func, size_t bytes);
// smx_fw_trace_arm measurement hook (fw.cu): CUDA events around a dominant-
// kernel launch on `s` with its cell-update count; no-ops unless armed.
void trace_begin(cudaStream_t s, long long cells);
void trace_end(cudaStream_t s);

// Per-device highest-priority side stream with fork/join events, used by the
// look-ahead closure schedules (created once, reused; see abi.cu).
struct SideStream {
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr, aux = nullptr;
    // a second side stream at the same priority (the FW look-ahead runs the
    // off-diagonal part of 3a on it beside the pivot) and its done event
    cudaStream_t side2 = nullptr;
    cudaEvent_t aux2 = nullptr;
    int priority = 0;   // the side stream's (highest) priority
};
int side_stream(SideStream** out);
// smx_set_fw_lookahead switch, shared by the lane FW and Boolean Warshall.
int lookahead_enabled();

// Multi-launch schedules (closures, the one-call Boolean product) are
// recorded once into a CUDA graph per distinct call -- same entry point,
// pointers, sizes and switches -- and replayed afterwards, so the host issues
// one graph launch instead of 5-8 launches and event waits per round.
// run_graphed captures body() on a private stream and launches the graph on
// `user`; when graphs are off (smx_set_graphs), the caller's stream is itself
// being captured, or `eager` is set, body(user) runs directly.
// Launch priority for kernels of the look-ahead side stream.  A stream's
// priority is not recorded into a captured graph, so the side-stream kernels
// carry it per launch (cudaLaunchAttributePriority), which graph kernel nodes
// keep.  0 = plain launch.  Set with PriorityScope around side-stream work.
int& launch_priority();
struct PriorityScope {
    int old;
    explicit PriorityScope(int p) : old(launch_priority()) { launch_priority() = p; }
    ~PriorityScope() { launch_priority() = old; }
};
// Programmatic dependent launch for the next launch_kernel call on this
// thread (consumed by it): the kernel may start while the preceding kernel in
// the stream finishes, and must execute griddepcontrol.wait (pdl_wait())
// before touching anything that kernel writes.  Only for a kernel that
// directly follows another kernel in the same stream.
bool& launch_pdl_next();
struct PdlNext {   // scoped: a path that launches nothing leaves no stale flag
    PdlNext() { launch_pdl_next() = true; }
    ~PdlNext() { launch_pdl_next() = false; }
};
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                 Args&&... args) {
    const int prio = launch_priority();
    const bool pdl = launch_pdl_next();
    launch_pdl_next() = false;
    if (prio == 0 && !pdl) {
        kern<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (prio != 0) {
        attr[na].id = cudaLaunchAttributePriority;
        attr[na].val.priority = prio;
        ++na;
    }
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

struct GraphKey {
    int fn = 0;
    unsigned long long v[14] = {};
};
int run_graphed(const GraphKey& key, cudaStream_t user, bool eager,
                const std::function<int(cudaStream_t)>& body);
}

// Placed directly after each kernel launch.
#define SMX_RETURN_LAUNCH()                          \
    do {                                             \
        smx::count_launch();                         \
        cudaError_t _e = cudaGetLastError();         \
        return _e == cudaSuccess ? SMX_OK : (int)_e; \
    } while (0)

#define SMX_LAUNCHED_OR_RETURN()                     \
    do {                                             \
        smx::count_launch();                         \
        cudaError_t _e = cudaGetLastError();         \
        if (_e != cudaSuccess) return (int)_e;       \
    } while (0)

#define SMX_TRY(expr)                 \
    do {                              \
        int _rc = (expr);             \
        if (_rc != SMX_OK) return _rc; \
    } while (0)

namespace smx {

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool ld_ok(long long ld, int elem_bytes) { return ((ld * elem_bytes) & 15) == 0; }
inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// SM count of the current device (queried once per device).
inline int sm_count() {
    static int cached[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = n > 0 ? n : 148;
    }
    return cached[dev];
}

// Saturation limit S = 2^w - 1 per element type.
template <typename T> struct Limit;
template <> struct Limit<uint8_t>  { static constexpr uint32_t value = 0xFFu; };
template <> struct Limit<uint16_t> { static constexpr uint32_t value = 0xFFFFu; };
template <> struct Limit<uint32_t> { static constexpr uint32_t value = 0xFFFFFFFFu; };

}  // namespace smx
