// Version and error strings of the semimat_b200 C ABI (include/semimat_b200.h).
#include <cuda_runtime.h>

#include "common.cuh"

#include <atomic>
#include <cstring>
#include <mutex>
#include <vector>

namespace smx {
static std::atomic<unsigned long long> g_launches{0};
static std::atomic<int> g_bounded{1};
static std::atomic<int> g_lookahead{1};
static std::atomic<int> g_graphs{1};
int lookahead_enabled() { return g_lookahead.load(std::memory_order_relaxed); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int set_max_smem(const void* func, size_t bytes) {
    struct Entry { int dev; const void* fn; size_t bytes; };
    static std::mutex mu;
    static std::vector<Entry> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    std::lock_guard<std::mutex> lock(mu);
    for (const Entry& x : done)
        if (x.dev == dev && x.fn == func && x.bytes >= bytes) return SMX_OK;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return (int)e;
    done.push_back({dev, func, bytes});
    return SMX_OK;
}
int bounded_fastpath_enabled() { return g_bounded.load(std::memory_order_relaxed); }
static std::atomic<int> g_packed_tpc{1};
int packed_tiles_per_cta() { return g_packed_tpc.load(std::memory_order_relaxed); }
static std::atomic<int> g_packed_backoff{0};
int packed_producer_backoff() { return g_packed_backoff.load(std::memory_order_relaxed); }

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

int& launch_priority() {
    thread_local int prio = 0;
    return prio;
}

bool& launch_pdl_next() {
    thread_local bool pdl = false;
    return pdl;
}

int side_stream(SideStream** out) {
    static SideStream per_dev[64];
    static std::mutex mu;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    if (dev < 0 || dev >= 64) return SMX_E_ARG;
    SideStream& f = per_dev[dev];
    std::lock_guard<std::mutex> lock(mu);
    if (!f.side) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if ((e = cudaStreamCreateWithPriority(&f.side, cudaStreamNonBlocking, hi)) != cudaSuccess) return (int)e;
        f.priority = hi;
        if ((e = cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming)) != cudaSuccess) return (int)e;
        if ((e = cudaEventCreateWithFlags(&f.join, cudaEventDisableTiming)) != cudaSuccess) return (int)e;
        if ((e = cudaEventCreateWithFlags(&f.aux, cudaEventDisableTiming)) != cudaSuccess) return (int)e;
        if ((e = cudaStreamCreateWithPriority(&f.side2, cudaStreamNonBlocking, hi)) != cudaSuccess) return (int)e;
        if ((e = cudaEventCreateWithFlags(&f.aux2, cudaEventDisableTiming)) != cudaSuccess) return (int)e;
    }
    *out = &f;
    return SMX_OK;
}
namespace {
struct GraphEntry {
    GraphKey key;
    int dev;
    cudaGraphExec_t exec;
    unsigned long long launches;   // kernels recorded in the graph
    unsigned long long stamp;      // LRU
};
constexpr size_t kMaxGraphs = 16;
constexpr size_t kMaxSeen = 64;
std::vector<std::pair<GraphKey, int>> g_seen;   // keys called once, not yet recorded
std::mutex g_graph_mu;
std::vector<GraphEntry> g_graph_cache;
unsigned long long g_graph_clock = 0;
cudaStream_t g_capture_stream[64] = {};

bool same_key(const GraphKey& a, const GraphKey& b) {
    return a.fn == b.fn && std::memcmp(a.v, b.v, sizeof(a.v)) == 0;
}
}  // namespace

int run_graphed(const GraphKey& key, cudaStream_t user, bool eager,
                const std::function<int(cudaStream_t)>& body) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (eager || !g_graphs.load(std::memory_order_relaxed) ||
        cudaStreamIsCapturing(user, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return body(user);
    }
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    if (dev < 0 || dev >= 64) return body(user);
    std::unique_lock<std::mutex> lock(g_graph_mu);
    for (auto& g : g_graph_cache) {
        if (g.dev == dev && same_key(g.key, key)) {
            g.stamp = ++g_graph_clock;
            if ((e = cudaGraphLaunch(g.exec, user)) != cudaSuccess) return (int)e;
            g_launches.fetch_add(g.launches, std::memory_order_relaxed);
            return SMX_OK;
        }
    }
    // Record a graph only for a call seen before: a one-off call launches
    // eagerly instead of paying the capture and instantiation (18 ms for the
    // n = 2048 closure, whose work is 1.7 ms).
    bool seen = false;
    for (size_t i = 0; i < g_seen.size(); ++i) {
        if (g_seen[i].second == dev && same_key(g_seen[i].first, key)) {
            seen = true;
            g_seen.erase(g_seen.begin() + i);
            break;
        }
    }
    if (!seen) {
        if (g_seen.size() >= kMaxSeen) g_seen.erase(g_seen.begin());
        g_seen.emplace_back(key, dev);
        lock.unlock();
        return body(user);
    }
    cudaStream_t& cap = g_capture_stream[dev];
    if (!cap && (e = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking)) != cudaSuccess) return (int)e;
    if ((e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) return (int)e;
    const unsigned long long before = g_launches.load();
    const int rc = body(cap);
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(cap, &graph);
    if (rc != SMX_OK || e != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        return rc != SMX_OK ? rc : (int)e;
    }
    GraphEntry ent{key, dev, nullptr, g_launches.load() - before, ++g_graph_clock};
    // kernel nodes keep their launch priority (the look-ahead side chain)
    e = cudaGraphInstantiate(&ent.exec, graph, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return (int)e;
    if ((e = cudaGraphLaunch(ent.exec, user)) != cudaSuccess) {
        cudaGraphExecDestroy(ent.exec);
        return (int)e;
    }
    if (g_graph_cache.size() >= kMaxGraphs) {
        size_t lru = 0;
        for (size_t i = 1; i < g_graph_cache.size(); ++i)
            if (g_graph_cache[i].stamp < g_graph_cache[lru].stamp) lru = i;
        // the evicted graph may still be executing: destroy is deferred by the driver
        cudaGraphExecDestroy(g_graph_cache[lru].exec);
        g_graph_cache.erase(g_graph_cache.begin() + lru);
    }
    g_graph_cache.push_back(ent);
    return SMX_OK;
}

}  // namespace smx

extern "C" {

int smx_set_graphs(int enable) {
    return smx::g_graphs.exchange(enable ? 1 : 0);
}

int smx_version(void) { return 100; }

unsigned long long smx_launch_count(void) { return smx::g_launches.load(); }

int smx_set_packed_tiles_per_cta(int tpc) {
    if (tpc != 1 && tpc != 2) return SMX_E_ARG;
    return smx::g_packed_tpc.exchange(tpc);
}
int smx_set_packed_producer_backoff(int ns) {
    // (a negative setting is valid, so the return value is always the previous
    // setting, never an error code: out-of-range values are clamped)
    ns = ns < -100000 ? -100000 : (ns > 100000 ? 100000 : ns);
    return smx::g_packed_backoff.exchange(ns);
}
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
        case SMX_E_COMM: return "collective (broadcast callback or NCCL) failed or unavailable";
        default: return code > 0 ? cudaGetErrorString((cudaError_t)code) : "unknown error";
    }
}

}  // extern "C"
