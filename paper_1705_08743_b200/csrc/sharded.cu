// Row-panel-sharded Floyd-Warshall across GPUs, as one C-ABI call per rank
// (SURVEY.md 8(b) `smx_fw_sharded_u16(Tpanel, n, row0, rows, ld, kind,
// ncclComm, stream)`; 8(e) the schedule).
//
// Rank p owns rows [p*per, (p+1)*per) (per = ceil(n/P) rounded up to whole
// pivot blocks), so every pivot block K has one owner.  Per block:
//   owner : close the pivot tile T[K,K] and update its row panel T[K,:]
//           (smx_fw_pivot + smx_semiring_gemm_skip, in place);
//   all   : broadcast the row panel (block x ld lanes) from the owner;
//           T[own,:] (+)= T[own,K] (x) T[K,:] over the own rows (the owner
//           skips its pivot rows) -- phases 2b and 3 in one product.
// Pipelined like the single-GPU look-ahead (fw.cu): on the high-priority
// side stream the owner of block r+1 applies round r to rows K_{r+1} (3a),
// closes pivot r+1, updates its row panel and broadcasts it into the second
// receive buffer, while the main stream applies round r to every other own
// row (3b).  The broadcast is enqueued on the side stream itself, so NCCL's
// kernel inherits its priority and the panel lands ahead of the next round.
// The first two rounds' updates take the certified 1-instruction encoding
// (their operands are the mostly unreachable input graph).
//
// The exchange is a callback (smx_bcast_fn), so one orchestration serves
// NCCL (smx_nccl_broadcast on an ncclComm_t, e.g. the one torch's
// ProcessGroupNCCL created) and any other transport (the tests drive it
// over gloo).  NCCL is resolved at run time with dlopen: the process's
// already-loaded libnccl (torch's) is used, so the communicator and the
// broadcast come from the same library.
//
// Exactness: every closure order over the semiring is bit-identical
// (SURVEY.md 0.1 fact 2), so the gathered panels equal the single-GPU
// closure; tests/test_bench_multirank.py checks it against the oracle digest.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include "common.cuh"

namespace smx {
namespace {

struct NcclApi {
    using BcastFn = int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t);
    using IntQueryFn = int (*)(void*, int*);
    using AsyncErrFn = int (*)(void*, int*);   // ncclCommGetAsyncError(comm, ncclResult_t*)
    BcastFn bcast = nullptr;
    IntQueryFn count = nullptr, user_rank = nullptr;
    AsyncErrFn async_error = nullptr;          // optional
    bool ok = false;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        // prefer the copy already mapped into the process (torch's), so the
        // communicator and the calls share one library instance
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.bcast = reinterpret_cast<NcclApi::BcastFn>(dlsym(h, "ncclBroadcast"));
        a.count = reinterpret_cast<NcclApi::IntQueryFn>(dlsym(h, "ncclCommCount"));
        a.user_rank = reinterpret_cast<NcclApi::IntQueryFn>(dlsym(h, "ncclCommUserRank"));
        a.async_error = reinterpret_cast<NcclApi::AsyncErrFn>(dlsym(h, "ncclCommGetAsyncError"));
        a.ok = a.bcast && a.count && a.user_rank;
        return a;
    }();
    return api;
}

constexpr int kNcclUint8 = 1;   // ncclDataType_t ncclUint8

inline long long rows_per_rank(int n, int world, int block) {
    const long long per = (n + (long long)world - 1) / world;
    return (per + block - 1) / block * block;
}

inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

inline size_t sharded_ws_bytes(int rows, long long ld, int eb, int block) {
    return al256((size_t)(rows > 0 ? rows : 1) * block * eb) + 2 * al256((size_t)block * ld * eb);
}

template <typename T>
int fw_sharded_run(T* Tl, int n, int row0, int rows, long long ld, int kind, int rank, int world, int B,
                   smx_bcast_fn bcast, void* ctx, void* ws, size_t ws_bytes, cudaStream_t s) {
    constexpr int eb = sizeof(T);
    if (n < 0 || rows < 0 || ld < n || world < 1 || rank < 0 || rank >= world) return SMX_E_ARG;
    if (kind != SMX_ANTI && kind != SMX_DIST) return SMX_E_ARG;
    if (B <= 0 || B % 128 || B > smx_fw_block(eb)) return SMX_E_ARG;
    const long long per = rows_per_rank(n, world, B);
    const long long r0 = per * rank < n ? per * rank : n;
    const long long r1 = per * (rank + 1) < n ? per * (rank + 1) : n;
    if (row0 != r0 || rows != r1 - r0) return SMX_E_ARG;            // not this rank's panel
    if (world > 1 && bcast == nullptr) return SMX_E_ARG;
    if (n == 0) return SMX_OK;
    if (!aligned16(Tl) || !ld_ok(ld, eb)) return SMX_E_ALIGN;
    if (ws == nullptr || ws_bytes < sharded_ws_bytes(rows, ld, eb, B)) return SMX_E_WORKSPACE;
    T* cp = reinterpret_cast<T*>(ws);                                  // own rows x B column panel
    T* recv[2];
    recv[0] = reinterpret_cast<T*>(reinterpret_cast<char*>(ws) + al256((size_t)(rows > 0 ? rows : 1) * B * eb));
    recv[1] = reinterpret_cast<T*>(reinterpret_cast<char*>(recv[0]) + al256((size_t)B * ld * eb));
    SideStream* fs = nullptr;
    SMX_TRY(side_stream(&fs));
    const int R = (n + B - 1) / B;
    auto blk = [&](int r) { return n - r * B < B ? n - r * B : B; };
    auto owner = [&](int r) { return (int)((long long)r * B / per); };
    auto panel = [&](int r) -> T* {
        return owner(r) == rank ? Tl + ((long long)r * B - row0) * ld : recv[r & 1];
    };
    auto owner_work = [&](int r, cudaStream_t st) -> int {
        if (owner(r) != rank) return SMX_OK;
        const long long lk = (long long)r * B - row0;
        T* rowK = Tl + lk * ld;
        SMX_TRY(smx_fw_pivot(rowK + (long long)r * B, blk(r), (int)ld, eb, kind, st));
        return smx_semiring_gemm_skip(rowK + (long long)r * B, rowK, rowK, blk(r), n, blk(r), (int)ld, (int)ld,
                                      (int)ld, eb, kind, 0, 0, st);
    };
    auto broadcast = [&](int r, cudaStream_t st) -> int {
        if (world == 1) return SMX_OK;
        return bcast(panel(r), (size_t)blk(r) * ld * eb, owner(r), ctx, st);
    };
    auto update = [&](int r, const T* A, T* C, int m, int skip0, int skipn, cudaStream_t st) -> int {
        if (m <= 0) return SMX_OK;
        auto fn = r < 2 ? smx_semiring_gemm_skip_certified : smx_semiring_gemm_skip;
        return fn(A, panel(r), C, m, n, blk(r), B, (int)ld, (int)ld, eb, kind, skip0, skipn, st);
    };
    cudaError_t e;
    SMX_TRY(owner_work(0, s));
    SMX_TRY(broadcast(0, s));
    for (int r = 0; r < R; ++r) {
        const int k0 = r * B, bb = blk(r);
        if (rows > 0) {
            e = cudaMemcpy2DAsync(cp, (size_t)B * eb, Tl + k0, (size_t)ld * eb, (size_t)bb * eb, rows,
                                  cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return (int)e;
        }
        const bool own_r = owner(r) == rank;
        int skip_lo = own_r ? k0 - row0 : 0, skip_n = own_r ? bb : 0;
        if (r + 1 < R) {
            const int k1 = k0 + B, bb1 = blk(r + 1);
            const bool own_n = owner(r + 1) == rank;
            const int lk1 = k1 - row0;
            if (own_n) {
                if (own_r) skip_n += bb1;          // K_r and K_{r+1} are adjacent rows
                else { skip_lo = lk1; skip_n = bb1; }
            }
            if ((e = cudaEventRecord(fs->fork, s)) != cudaSuccess) return (int)e;
            if ((e = cudaStreamWaitEvent(fs->side, fs->fork, 0)) != cudaSuccess) return (int)e;
            {
                PriorityScope ps(fs->priority);
                if (own_n) SMX_TRY(update(r, cp + (long long)lk1 * B, Tl + (long long)lk1 * ld, bb1, 0, 0, fs->side));
                SMX_TRY(owner_work(r + 1, fs->side));
                SMX_TRY(broadcast(r + 1, fs->side));
            }
            if ((e = cudaEventRecord(fs->join, fs->side)) != cudaSuccess) return (int)e;
            trace_begin(s, (long long)(rows - skip_n) * n * bb);
            SMX_TRY(update(r, cp, Tl, rows, skip_lo, skip_n, s));        // 3b
            trace_end(s);
            if ((e = cudaStreamWaitEvent(s, fs->join, 0)) != cudaSuccess) return (int)e;
        } else {
            trace_begin(s, (long long)(rows - skip_n) * n * bb);
            SMX_TRY(update(r, cp, Tl, rows, skip_lo, skip_n, s));
            trace_end(s);
        }
    }
    return SMX_OK;
}

}  // namespace
}  // namespace smx

using namespace smx;

extern "C" {

int smx_nccl_broadcast(void* buf, size_t bytes, int root, void* comm, void* stream) {
    const NcclApi& api = nccl();
    if (!api.ok) return SMX_E_COMM;
    // a communicator that already failed asynchronously (a peer died, a
    // network error) would hang the next collective: fail fast instead
    if (api.async_error) {
        int st = 0;
        if (api.async_error(comm, &st) != 0 || st != 0) return SMX_E_COMM;
    }
    const int rc = api.bcast(buf, buf, bytes, kNcclUint8, root, comm, as_stream(stream));
    return rc == 0 ? SMX_OK : SMX_E_COMM;
}

int smx_nccl_async_error(void* comm) {
    const NcclApi& api = nccl();
    if (!api.ok) return SMX_E_COMM;
    if (!api.async_error) return SMX_OK;
    int st = 0;
    const int rc = api.async_error(comm, &st);
    return (rc == 0 && st == 0) ? SMX_OK : SMX_E_COMM;
}

int smx_fw_sharded_block(int n, int world, int elem_bytes) {
    if (n < 0 || world < 1) return SMX_E_ARG;
    const int mx = smx_fw_block(elem_bytes);
    if (mx <= 0) return SMX_E_ARG;
    const int b = (elem_bytes == 2 && n / world >= 4096) ? 512 : 256;
    return b < mx ? b : mx;
}

size_t smx_fw_sharded_workspace_bytes(int rows, int ld, int elem_bytes, int block) {
    if (rows < 0 || ld <= 0 || block <= 0) return 0;
    return sharded_ws_bytes(rows, ld, elem_bytes, block);
}

int smx_fw_sharded(void* T, int n, int row0, int rows, int ld, int elem_bytes, int kind, int rank, int world,
                   int block, smx_bcast_fn bcast, void* ctx, void* ws, size_t ws_bytes, void* stream) {
    cudaStream_t s = as_stream(stream);
    switch (elem_bytes) {
        case 1: return fw_sharded_run<uint8_t>((uint8_t*)T, n, row0, rows, ld, kind, rank, world, block, bcast, ctx,
                                               ws, ws_bytes, s);
        case 2: return fw_sharded_run<uint16_t>((uint16_t*)T, n, row0, rows, ld, kind, rank, world, block, bcast,
                                                ctx, ws, ws_bytes, s);
        case 4: return fw_sharded_run<uint32_t>((uint32_t*)T, n, row0, rows, ld, kind, rank, world, block, bcast,
                                                ctx, ws, ws_bytes, s);
        default: return SMX_E_ARG;
    }
}

int smx_fw_sharded_u16(uint16_t* Tpanel, int n, int row0, int rows, int ld, int kind, void* nccl_comm, void* ws,
                       size_t ws_bytes, void* stream) {
    const NcclApi& api = nccl();
    if (!api.ok || nccl_comm == nullptr) return SMX_E_COMM;
    int world = 0, rank = 0;
    if (api.count(nccl_comm, &world) != 0 || api.user_rank(nccl_comm, &rank) != 0) return SMX_E_COMM;
    const int block = smx_fw_sharded_block(n, world, 2);
    return fw_sharded_run<uint16_t>(Tpanel, n, row0, rows, ld, kind, rank, world, block,
                                    [](void* buf, size_t bytes, int root, void* ctx, void* st) {
                                        return smx_nccl_broadcast(buf, bytes, root, ctx, st);
                                    },
                                    nccl_comm, ws, ws_bytes, as_stream(stream));
}

}  // extern "C"
