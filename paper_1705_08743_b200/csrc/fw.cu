// Blocked three-phase Floyd-Warshall over the saturated semirings, plus the
// C-ABI entry points of the lane semiring products.
//
// Replaces _close_vector / _minplus_close_vector
// (pkg/src/semimat/antidist.py:390-398, :440-448).  The reference sweeps k
// one vertex at a time over the whole matrix; here k advances in blocks of
// B = 128 / 256 / 512 vertices (fw_block_for_n; SURVEY.md 0.1 fact 2
// verifies the blocked order is bit-identical: x -> min(x, S) is a semiring
// homomorphism from (min,+) on [0, inf] onto the clipped lanes, so every
// correct closure order agrees):
//
//   round r, pivot block K = [k0, k0 + bb):
//   1. pivot   : close the bb x bb tile T[K,K] in place (the 128 register
//                kernel, or a 2 x 2 blocked recursion on it above 128).
//   2. row     : T[K,:] (+)= T[K,K]* (x) T[K,:], in place (see
//                fw_pivot_and_row_panel for why no snapshot is needed).
//   3. rest    : T[i,:] (+)= T[i,K] (x) T[K,:] for every i outside K, with
//                T[i,K] read from a snapshot of the column panel (the packed
//                A tiles on the u8/u16 path, CP otherwise).  The j in K part
//                of this product is exactly the column-panel update
//                T[i,K] (x) (I (+) T[K,K]*), so phases 2b and 3 fuse into one
//                semiring GEMM over the full row width.
// Phase 3 is the packed kernel of semiring_packed.cuh (u8/u16) or the
// register-staged one of semiring_gemm.cuh (u32, smx_set_fw_packed(0)); the
// look-ahead schedules overlap round r's phase 3 with round r+1's steps 1-2
// on a high-priority side stream.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "host_stage.cuh"
#include "semiring_packed.cuh"

namespace smx {

// Largest pivot block: 512 vertices for u16 (the packed phase 3 runs K = 512
// per CTA), 256 for u8 and u32.  Tiles above 128 close by 2 x 2 recursion
// (the 1024-thread register pivot holds at most 128 x 128).
template <typename T> struct FwBlock { static constexpr int value = sizeof(T) == 2 ? 512 : 256; };
inline int fw_block_for(int eb) { return eb == 2 ? 512 : 256; }
// Block used for an n-vertex closure.  A larger block halves the rounds and
// doubles phase 3's K per CTA, amortising each CTA's ramp and C fold; it
// costs a longer pivot chain, which must hide behind one round's phase 3.
// Measured (u16): 256 over 128 +6% at n = 8192, +9% at 16384, +10% at 32768;
// 512 over 256 at n >= 16384: see DESIGN.md 4.2.  Below 8192 vertices the
// pivot chain no longer hides behind phase 3 and 128 wins.
static std::atomic<int> g_fw_block_override{0};   // smx_set_fw_block: 0 = automatic
template <typename T> inline int fw_block_for_n(int n) {
    const int mx = FwBlock<T>::value;
    const int ov = g_fw_block_override.load(std::memory_order_relaxed);
    if (ov != 0) return ov < mx ? ov : mx;
    if (sizeof(T) == 2 && n >= 16384) return 512;
    return n >= 8192 ? 256 : 128;
}

// ---- phase 1: pivot tile closure ------------------------------------------
// 1024 threads, 1024/B per tile row; each owns B*B/1024 cells of its row in
// registers.  Step k reads pivot column value T[r,k] and pivot row T[k,:]
// from double-buffered smem (one barrier per step); the owners of row k+1
// and column k+1 publish them for the next step.  During step k row k and
// column k do not change (T[k,k] >= 0 in distance form), so no hazard.
template <typename T, int BLK>
__global__ void __launch_bounds__(1024, 1)
fw_pivot_kernel(T* P, int b, long long ld, int anti) {
    using L = Lane<T>;
    constexpr int CPW = L::kCellsPerWord;
    constexpr int WPR = BLK / CPW;        // words per tile row
    constexpr int TPR = 1024 / BLK;       // threads per tile row
    constexpr int WPT = WPR / TPR;        // words per thread
    constexpr int CPT = WPT * CPW;        // cells per thread
    __shared__ __align__(16) uint32_t prow[2][WPR];
    __shared__ uint32_t pcol[2][BLK];

    const int tid = threadIdx.x;
    const int r = tid / TPR, g = tid % TPR;
    const int c0 = g * CPT;

    auto to_dist = [&](uint32_t v) { return anti ? (L::kS - v) : v; };
    uint32_t w[WPT];
#pragma unroll
    for (int i = 0; i < WPT; ++i) {
        uint32_t word = 0;
#pragma unroll
        for (int l = 0; l < CPW; ++l) {
            const int col = c0 + i * CPW + l;
            const uint32_t v = (r < b && col < b) ? to_dist((uint32_t)P[(long long)r * ld + col]) : L::kS;
            word |= (CPW == 2) ? (v << (16 * l)) : v;
        }
        w[i] = word;
    }
    auto cell_of = [&](int local) {
        uint32_t v = 0;
#pragma unroll
        for (int i = 0; i < WPT; ++i)
#pragma unroll
            for (int l = 0; l < CPW; ++l)
                if (i * CPW + l == local) v = (CPW == 2) ? ((w[i] >> (16 * l)) & 0xFFFFu) : w[i];
        return v;
    };
    if (r == 0) {
#pragma unroll
        for (int i = 0; i < WPT; ++i) prow[0][g * WPT + i] = w[i];
    }
    if (g == 0) pcol[0][r] = cell_of(0);
    __syncthreads();

    // k = g0 * CPT + j with j unrolled, so the cell that becomes the next
    // pivot column (local index (j + 1) % CPT of group g0 or g0 + 1) is a
    // compile-time register, not a dynamic select.
    for (int g0 = 0; g0 < TPR; ++g0) {
        if (g0 * CPT >= b) break;
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const int k = g0 * CPT + j;
            if (k >= b) break;
            const int cur = k & 1;
            const uint32_t e = pcol[cur][r];
            const uint32_t a = L::splat(e), sa = L::splat(L::kS - e);
#pragma unroll
            for (int i = 0; i < WPT; i += 4) {   // 4 words at a time: bounded registers
                const uint4 v = *reinterpret_cast<const uint4*>(&prow[cur][g * WPT + i]);
                w[i] = L::step(w[i], v.x, a, sa);
                w[i + 1] = L::step(w[i + 1], v.y, a, sa);
                w[i + 2] = L::step(w[i + 2], v.z, a, sa);
                w[i + 3] = L::step(w[i + 3], v.w, a, sa);
            }
            const int kn = k + 1;
            if (kn < b) {
                if (r == kn) {
#pragma unroll
                    for (int i = 0; i < WPT; ++i) prow[cur ^ 1][g * WPT + i] = w[i];
                }
                const int jn = (j + 1) % CPT, gn = (j + 1 == CPT) ? g0 + 1 : g0;
                if (g == gn) {
                    const uint32_t word = w[jn / CPW];
                    pcol[cur ^ 1][r] = (CPW == 2) ? ((word >> (16 * (jn % CPW))) & 0xFFFFu) : word;
                }
            }
            __syncthreads();
        }
    }
    if (r < b) {
#pragma unroll
        for (int i = 0; i < WPT; ++i) {
#pragma unroll
            for (int l = 0; l < CPW; ++l) {
                const int col = c0 + i * CPW + l;
                if (col < b) {
                    const uint32_t v = (CPW == 2) ? ((w[i] >> (16 * l)) & 0xFFFFu) : w[i];
                    P[(long long)r * ld + col] = (T)(anti ? (L::kS - v) : v);
                }
            }
        }
    }
}

// Blocked pivot closure (u8/u16 tiles up to 128 vertices): Floyd-Warshall
// inside one CTA in 32-vertex sub-blocks, on a 32 KB shared-memory tile in
// distance form.  Per sub-block K:
//   P1  D = T[K,K] closed by one warp, vertex at a time, rows in registers
//       and row k broadcast by shuffles (no CTA barrier inside);
//   P2  T[K,:] (+)= D* (x) T[K,:]      (the row panel, in place);
//   P3  T[i,:] (+)= T[i,K] (x) T[K,:]  for i outside K (the j in K part is the
//       column panel: T[K,K] = D* by then).
// 3 barriers per sub-block instead of one per vertex (fw_pivot_kernel: 128
// barriers, 58 us), and 512 threads with few registers and 32 KB of shared
// memory, so it fits on an SM in place of one retired phase-3 CTA instead of
// waiting for a whole SM to drain.  Every in-place read of a value another
// thread may already have lowered reads the weight of a real walk of the
// same kind (the fw_pivot_and_row_panel argument), so any interleaving gives
// the same bits.
// Sub-block sweep of fw_pivot_blocked_kernel.  BD: every lane of the tile
// is < 2^15 (voted once after the load), so a + b <= 65534 < S and the
// clamp is a no-op: the 1-instruction update L::step_bounded replaces the
// general 2-instruction form.  Values only decrease during the closure, so
// the bound holds to the end.  After the first few rounds of a closure the
// pivot tiles are almost always bounded.
template <typename T, bool BD>
__device__ __forceinline__ void pivot_blocked_sweep(uint32_t* tile, uint32_t* As, int b) {
    using L = Lane<T>;
    constexpr int WPR = 64;
    constexpr int APITCH = 34;
    const int tid = threadIdx.x;
    auto cell = [&](int r, int c) {         // one cell of the tile
        const uint32_t w = tile[r * WPR + (c >> 1)];
        return (c & 1) ? (w >> 16) : (w & 0xFFFFu);
    };
    auto upd = [](uint32_t c, uint32_t bw, uint32_t a, uint32_t sa) {
        if constexpr (BD) return L::step_bounded(c, bw, a);
        else return L::step(c, bw, a, sa);
    };
    const int nsb = (b + 31) / 32;
    const int g = tid >> 4, q = tid & 15;   // 32 row slots x 16 word slots
    for (int kb = 0; kb < nsb; ++kb) {
        const int K0 = kb * 32, KW0 = kb * 16;
        // P1: warp 0 closes D with the vertex-at-a-time sweep, lane j holding
        // D's row j (16 words) in registers; row k reaches the other lanes by
        // shuffles, so the 32 steps need no CTA barrier (row k does not change
        // during step k: T[k][k] >= 0 in distance form)
        if (tid < 32) {
            uint32_t w[16];
            const uint4* src = reinterpret_cast<const uint4*>(&tile[(K0 + tid) * WPR + KW0]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint4 v = src[i];
                w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
            }
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const uint32_t e = (w[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu;
                const uint32_t a = L::splat(e), sa = L::splat(L::kS - e);
#pragma unroll
                for (int i = 0; i < 16; ++i) w[i] = upd(w[i], __shfl_sync(0xFFFFFFFFu, w[i], k), a, sa);
            }
            uint4* dst = reinterpret_cast<uint4*>(&tile[(K0 + tid) * WPR + KW0]);
#pragma unroll
            for (int i = 0; i < 4; ++i) dst[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        }
        __syncthreads();
        // P2: row K0 + g, words 4q .. 4q + 3
        {
            uint4* rw = reinterpret_cast<uint4*>(&tile[(K0 + g) * WPR + 4 * q]);
            uint4 acc = *rw;
#pragma unroll 4
            for (int k = 0; k < 32; ++k) {
                const uint32_t e = cell(K0 + g, K0 + k);
                const uint32_t a = L::splat(e), sa = L::splat(L::kS - e);
                const uint4 bw = *reinterpret_cast<const uint4*>(&tile[(K0 + k) * WPR + 4 * q]);
                acc.x = upd(acc.x, bw.x, a, sa);
                acc.y = upd(acc.y, bw.y, a, sa);
                acc.z = upd(acc.z, bw.z, a, sa);
                acc.w = upd(acc.w, bw.w, a, sa);
            }
            *rw = acc;
        }
        // P3's A operand: splat(T[i][K0 + k]) for the 96 rows outside K (not
        // written by P2), one LDS.64 per row and k pair in the P3 loop
#pragma unroll
        for (int i = 0; i < 96 * 32 / 512; ++i) {
            const int x = tid + i * 512, slot = x >> 5, k = x & 31;
            const int row = slot < K0 ? slot : slot + 32;
            As[slot * APITCH + k] = L::splat(cell(row, K0 + k));
        }
        __syncthreads();
        // P3: rows outside K, three per thread (96 rows), words 4q .. 4q + 3
        {
            int rows[3];
            uint4 acc[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const int idx = 3 * g + i;
                rows[i] = idx < K0 ? idx : idx + 32;
                acc[i] = *reinterpret_cast<const uint4*>(&tile[rows[i] * WPR + 4 * q]);
            }
            const bool live = rows[0] < b;   // rows[] ascend: all padding beyond
#pragma unroll 2
            for (int kk = 0; kk < 16 && live; ++kk) {
                const uint4 b0 = *reinterpret_cast<const uint4*>(&tile[(K0 + 2 * kk) * WPR + 4 * q]);
                const uint4 b1 = *reinterpret_cast<const uint4*>(&tile[(K0 + 2 * kk + 1) * WPR + 4 * q]);
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const uint2 av = *reinterpret_cast<const uint2*>(&As[(3 * g + i) * APITCH + 2 * kk]);
                    const uint32_t a0 = av.x, s0 = L::kIdentityWord - av.x;   // splat(S - e)
                    const uint32_t a1 = av.y, s1 = L::kIdentityWord - av.y;
                    acc[i].x = upd(upd(acc[i].x, b0.x, a0, s0), b1.x, a1, s1);
                    acc[i].y = upd(upd(acc[i].y, b0.y, a0, s0), b1.y, a1, s1);
                    acc[i].z = upd(upd(acc[i].z, b0.z, a0, s0), b1.z, a1, s1);
                    acc[i].w = upd(upd(acc[i].w, b0.w, a0, s0), b1.w, a1, s1);
                }
            }
            if (live) {
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    *reinterpret_cast<uint4*>(&tile[rows[i] * WPR + 4 * q]) = acc[i];
            }
        }
        __syncthreads();
    }
}

template <typename T>
__global__ void __launch_bounds__(512, 3)
fw_pivot_blocked_kernel(T* P, int b, long long ld, int anti, int allow_bounded) {
    using L = Lane<T>;
    static_assert(L::kCellsPerWord == 2, "u8 / u16 lanes");
    constexpr int WPR = 64;                 // words per tile row (128 cells)
    constexpr int APITCH = 34;              // splat rows: 32 k + 2 (no bank conflicts between row slots)
    __shared__ __align__(16) uint32_t tile[128 * WPR];
    __shared__ __align__(16) uint32_t As[96 * APITCH];   // P3's A operand, splat, per row slot
    const int tid = threadIdx.x;
    auto to_dist = [&](uint32_t v) { return anti ? (L::kS - v) : v; };
    // 8 global loads of a thread in flight at a time, then their tile stores
    uint32_t high = 0;                      // OR of the stored words: the bounded vote
    for (int i0 = 0; i0 < 128 * WPR / 512; i0 += 4) {
        uint32_t v[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int w = tid + (i0 + i) * 512, r = w / WPR, c = (w % WPR) * 2;
            v[2 * i] = (r < b && c < b) ? (uint32_t)P[(long long)r * ld + c] : 0u;
            v[2 * i + 1] = (r < b && c + 1 < b) ? (uint32_t)P[(long long)r * ld + c + 1] : 0u;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int w = tid + (i0 + i) * 512, r = w / WPR, c = (w % WPR) * 2;
            const uint32_t v0 = (r < b && c < b) ? to_dist(v[2 * i]) : L::kS;
            const uint32_t v1 = (r < b && c + 1 < b) ? to_dist(v[2 * i + 1]) : L::kS;
            tile[w] = v0 | (v1 << 16);
            high |= tile[w];
        }
    }
    // (padding is S, so a padded tile takes the general form)
    const bool bd = __syncthreads_and((high & L::kHalfMask) == 0u) && allow_bounded && L::kHalfMask != 0u;
    if (bd) pivot_blocked_sweep<T, true>(tile, As, b);
    else pivot_blocked_sweep<T, false>(tile, As, b);
    for (int w = tid; w < 128 * WPR; w += 512) {
        const int r = w / WPR, c = (w % WPR) * 2;
        if (r >= b || c >= b) continue;
        const uint32_t v = tile[w];
        P[(long long)r * ld + c] = (T)(anti ? (L::kS - (v & 0xFFFFu)) : (v & 0xFFFFu));
        if (c + 1 < b) P[(long long)r * ld + c + 1] = (T)(anti ? (L::kS - (v >> 16)) : (v >> 16));
    }
}

// smx_set_fw_pivot_blocked: u8/u16 pivot tiles <= 128 on the blocked kernel
// (default) or on the one-barrier-per-vertex register kernel.
static std::atomic<int> g_pivot_blocked{1};

// Lightweight pivot closure for the look-ahead side stream: the tile lives in
// shared memory (B x B/2 words) and 256 threads with few registers sweep it,
// so the kernel fits on an SM *beside* two phase-3 CTAs (which hold most of
// the register file) and starts as soon as it is launched instead of waiting
// for a whole SM to drain.  Per step k every cell is updated in place from
// row k and column k of the same buffer: neither changes during step k
// (T[k][k] >= 0 in distance form), and a thread that rewrites the word
// holding column k only changes the other lane of that word.
template <typename T, int BLK>
__global__ void __launch_bounds__(256)
fw_pivot_lite_kernel(T* P, int b, long long ld, int anti) {
    using L = Lane<T>;
    constexpr int CPW = L::kCellsPerWord;
    constexpr int WPR = BLK / CPW;               // words per tile row
    constexpr int WORDS = BLK * WPR;
    extern __shared__ __align__(16) uint32_t tile[];   // [BLK][WPR], distance form
    const int tid = threadIdx.x;
    auto to_dist = [&](uint32_t v) { return anti ? (L::kS - v) : v; };
    for (int w = tid; w < WORDS; w += 256) {
        const int r = w / WPR, c0 = (w % WPR) * CPW;
        uint32_t word = 0;
#pragma unroll
        for (int l = 0; l < CPW; ++l) {
            const int col = c0 + l;
            const uint32_t v = (r < b && col < b) ? to_dist((uint32_t)P[(long long)r * ld + col]) : L::kS;
            word |= (CPW == 2) ? (v << (16 * l)) : v;
        }
        tile[w] = word;
    }
    __syncthreads();
    for (int k = 0; k < b; ++k) {
        const uint32_t* prow = tile + k * WPR;
        const int kw = k / CPW, ksh = (k % CPW) * 16;
        for (int w4 = tid * 4; w4 < WORDS; w4 += 256 * 4) {
            const int r = w4 / WPR, c = w4 % WPR;
            uint32_t e = tile[r * WPR + kw];
            if (CPW == 2) e = (e >> ksh) & 0xFFFFu;
            const uint32_t a = L::splat(e), sa = L::splat(L::kS - e);
            uint4 v = *reinterpret_cast<const uint4*>(tile + w4);
            const uint4 pv = *reinterpret_cast<const uint4*>(prow + c);
            v.x = L::step(v.x, pv.x, a, sa);
            v.y = L::step(v.y, pv.y, a, sa);
            v.z = L::step(v.z, pv.z, a, sa);
            v.w = L::step(v.w, pv.w, a, sa);
            *reinterpret_cast<uint4*>(tile + w4) = v;
        }
        __syncthreads();
    }
    for (int w = tid; w < WORDS; w += 256) {
        const int r = w / WPR, c0 = (w % WPR) * CPW;
        if (r >= b) continue;
#pragma unroll
        for (int l = 0; l < CPW; ++l) {
            const int col = c0 + l;
            if (col < b) {
                const uint32_t v = (CPW == 2) ? ((tile[w] >> (16 * l)) & 0xFFFFu) : tile[w];
                P[(long long)r * ld + col] = (T)(anti ? (L::kS - v) : v);
            }
        }
    }
}

template <typename T, int BLK>
int launch_pivot_lite(T* P, int b, long long ld, int kind, cudaStream_t s) {
    constexpr size_t smem = (size_t)BLK * (BLK / Lane<T>::kCellsPerWord) * 4;
    auto kern = fw_pivot_lite_kernel<T, BLK>;
    SMX_TRY(set_max_smem((const void*)kern, smem));
    smx::count_launch();
    const cudaError_t e = launch_kernel(kern, dim3(1), dim3(256), smem, s, P, b, ld, kind == SMX_ANTI);
    return e == cudaSuccess ? SMX_OK : (int)e;
}

template <typename T>
int fw_pivot_lite(T* P, int b, long long ld, int kind, cudaStream_t s) {
    if (b < 1 || b > FwBlock<T>::value || ld < b || (kind != SMX_ANTI && kind != SMX_DIST)) return SMX_E_ARG;
    if (b <= 128) return launch_pivot_lite<T, 128>(P, b, ld, kind, s);
    if (b > 256) return SMX_E_ARG;   // the shared-memory tile holds at most 256 x 256
    return launch_pivot_lite<T, (FwBlock<T>::value < 256 ? FwBlock<T>::value : 256)>(P, b, ld, kind, s);
}

// Tile copy dst[0:rows, 0:cols] = src[0:rows, 0:cols] (16-byte vectors; a
// ragged last column chunk element-wise): the column-panel snapshot
// CP[i, 0:bb] = T[i, k0:k0+bb] and the pivot/row-panel snapshots.  A kernel
// rather than cudaMemcpy2DAsync: in a captured graph a D2D memcpy node goes
// to a copy engine with several microseconds of latency on the pivot chain.
template <typename T>
__global__ void copy_panel_kernel(const T* __restrict__ src, long long ld, T* __restrict__ dst,
                                  long long ldd, int rows, int cols) {
    constexpr int E = 16 / sizeof(T);
    const int cpr = (cols + E - 1) / E;
    const long long total = (long long)rows * cpr;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i / cpr), c = (int)(i % cpr) * E;
        const T* s = src + r * ld + c;
        T* d = dst + r * ldd + c;
        if (c + E <= cols) *reinterpret_cast<uint4*>(d) = __ldg(reinterpret_cast<const uint4*>(s));
        else
            for (int j = 0; c + j < cols; ++j) d[j] = s[j];
    }
}

template <typename T>
int copy_panel(const T* src, long long ld, T* dst, long long ldd, int rows, int cols, cudaStream_t s) {
    const long long work = (long long)rows * ((cols * (long long)sizeof(T) + 15) / 16);
    long long blocks = (work + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    count_launch();
    const cudaError_t e = launch_kernel(copy_panel_kernel<T>, dim3((unsigned)(blocks < 1 ? 1 : blocks)), dim3(256),
                                        0, s, src, ld, dst, ldd, rows, cols);
    return e == cudaSuccess ? SMX_OK : (int)e;
}

// Pivot tiles above 128 vertices: blocked FW with two blocks, h = 128 for
// b <= 256 and h = 256 above (the same three phases as fw_run, one level
// down):
//   P11* ; P12 (+)= P11 (x) P12 ; P21 (+)= P21 (x) P11 ; P22 (+)= P21 (x) P12 ;
//   P22* ; P21 (+)= P22 (x) P21 ; P12 (+)= P12 (x) P22 ; P11 (+)= P12 (x) P21.
// The closures recurse down to the 128 kernels, the products are Lite tiles.
// The four panel products run in place, with no operand snapshot: one
// operand is a closed tile X*, and a value another CTA has already lowered
// is the weight of a real walk of the same kind, so it can only tighten
// towards the exact result (the fw_pivot_and_row_panel argument).  256:
// 146 us with the blocked leaves and the snapshots (185 us with the register
// leaves), against 500 us for the single-CTA shared-memory pivot
// (fw_pivot_lite), which moved 3 x 512 B of shared memory per row per step
// and was bandwidth-bound.  (`scratch` is no longer read; the signature
// keeps it.)
template <typename T>
int fw_pivot(T* P, int b, long long ld, int kind, cudaStream_t s, T* scratch);

// smx_set_fw_pivot_pairs: the recursion's two independent panel products per
// half in one launch (semiring_gemm_lite_pair).
static std::atomic<int> g_pivot_pairs{1};

template <typename T>
int fw_pivot_2x2(T* P, int b, long long ld, int kind, T* scratch, cudaStream_t s) {
    const int h = b <= 256 ? 128 : 256;
    const int m = b - h;
    T* P12 = P + h;
    T* P21 = P + (long long)h * ld;
    T* P22 = P21 + h;
#ifdef SMX_TRACE_PIVOT_PARTS   // development builds: each step of the recursion (cells -10 .. -17)
#define SMX_PP(i, expr) do { trace_begin(s, -10 - (i)); SMX_TRY(expr); trace_end(s); } while (0)
#else
#define SMX_PP(i, expr) SMX_TRY(expr)
#endif
    SMX_PP(0, (fw_pivot<T>(P, h, ld, kind, s, scratch)));
    if (g_pivot_pairs.load(std::memory_order_relaxed)) {
        // the two independent panel products of each half in one launch
        SMX_PP(1, (semiring_gemm_lite_pair<T>(P, P12, P12, h, m, h,          // P12 (+)= P11* (x) P12
                                              P21, P, P21, m, h, h, ld, kind, s)));   // P21 (+)= P21 (x) P11*
    } else {
        SMX_PP(1, (semiring_gemm_lite<T>(P, P12, P12, h, m, h, ld, ld, ld, kind, s)));     // P12 (+)= P11* (x) P12
        SMX_PP(2, (semiring_gemm_lite<T>(P21, P, P21, m, h, h, ld, ld, ld, kind, s)));     // P21 (+)= P21 (x) P11*
    }
    SMX_PP(3, (semiring_gemm_lite<T>(P21, P12, P22, m, m, h, ld, ld, ld, kind, s)));
    SMX_PP(4, (fw_pivot<T>(P22, m, ld, kind, s, scratch)));
    if (g_pivot_pairs.load(std::memory_order_relaxed)) {
        SMX_PP(5, (semiring_gemm_lite_pair<T>(P22, P21, P21, m, h, m,        // P21 (+)= P22* (x) P21
                                              P12, P22, P12, h, m, m, ld, kind, s)));  // P12 (+)= P12 (x) P22*
    } else {
        SMX_PP(5, (semiring_gemm_lite<T>(P22, P21, P21, m, h, m, ld, ld, ld, kind, s)));   // P21 (+)= P22* (x) P21
        SMX_PP(6, (semiring_gemm_lite<T>(P12, P22, P12, h, m, m, ld, ld, ld, kind, s)));   // P12 (+)= P12 (x) P22*
    }
    SMX_PP(7, (semiring_gemm_lite<T>(P12, P21, P, h, h, m, ld, ld, ld, kind, s)));
#undef SMX_PP
    return SMX_OK;
}

int scratch_alloc(void** p, size_t bytes, cudaStream_t s);
int scratch_free(void* p, cudaStream_t s);

// scratch: 2 x h x h elements for b > 128, h as in fw_pivot_2x2 (nullptr:
// stream-ordered scratch)
template <typename T>
int fw_pivot(T* P, int b, long long ld, int kind, cudaStream_t s, T* scratch) {
    if (b < 1 || b > FwBlock<T>::value || ld < b || (kind != SMX_ANTI && kind != SMX_DIST)) return SMX_E_ARG;
    // The register-resident kernel unrolls CPT steps (16 cells/thread at 128);
    // at 256 that unroll (64 steps x 32 words) no longer fits the instruction
    // caches (measured 688 us per pivot), so 256 recurses on 128 blocks.
    if (b > 128) {
        if (!aligned16(P) || !ld_ok(ld, sizeof(T))) return SMX_E_ALIGN;
        if (scratch) return fw_pivot_2x2<T>(P, b, ld, kind, scratch, s);
        void* sc = nullptr;
        const size_t h = b <= 256 ? 128 : 256;
        SMX_TRY(scratch_alloc(&sc, 2 * h * h * sizeof(T), s));
        const int rc = fw_pivot_2x2<T>(P, b, ld, kind, reinterpret_cast<T*>(sc), s);
        scratch_free(sc, s);
        return rc;
    }
    count_launch();
    if constexpr (sizeof(T) <= 2) {
        if (g_pivot_blocked.load(std::memory_order_relaxed)) {
            const cudaError_t e = launch_kernel(fw_pivot_blocked_kernel<T>, dim3(1), dim3(512), 0, s, P, b, ld,
                                                kind == SMX_ANTI, bounded_fastpath_enabled());
            return e == cudaSuccess ? SMX_OK : (int)e;
        }
    }
    const cudaError_t e = launch_kernel(fw_pivot_kernel<T, 128>, dim3(1), dim3(1024), 0, s, P, b, ld,
                                        kind == SMX_ANTI);
    return e == cudaSuccess ? SMX_OK : (int)e;
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// RP: the row-panel region: the serial schedule's row-panel snapshot (B x
// ld), or the look-ahead's packed row-panel operands (semiring_gemm_packed of
// B x n x B, g_fw_packed_panel) -- whichever is larger.
inline size_t fw_rp_bytes(int n, long long ld, int eb) {
    const size_t B = fw_block_for(eb);
    const size_t snap = align256(B * ld * eb);
    const size_t packed = align256(packed_ws_bytes_eb((int)B, n, (int)B, eb));
    return snap > packed ? snap : packed;
}

inline size_t fw_b2_bytes(int n, int eb) { return align256(packed_b_ws_bytes_eb(n, fw_block_for(eb), eb)); }

inline size_t fw_ws_bytes(int n, long long ld, int eb) {
    // RP: the row-panel region (fw_rp_bytes); CP: column panel snapshot
    // (n x B); the packed phase-3 operand tiles (semiring_packed.cuh); a
    // second block of packed B tiles (the look-ahead's row panels alternate
    // between the two, fw_rounds_packed); a 256-byte slot for the per-round
    // operand certificate
    const size_t B = fw_block_for(eb);
    const size_t base = fw_rp_bytes(n, ld, eb) + align256((size_t)n * B * eb);
    return base + align256(packed_ws_bytes_eb(n, n, (int)B, eb)) + fw_b2_bytes(n, eb) + 256;
}
// The certificate slot: the last 256 bytes of fw_ws_bytes.
inline int* fw_cert_slot(void* ws, int n, long long ld, int eb) {
    return reinterpret_cast<int*>(reinterpret_cast<char*>(ws) + fw_ws_bytes(n, ld, eb) - 256);
}
// The second packed-B block: just before the certificate slot.
inline void* fw_b2_slot(void* ws, int n, long long ld, int eb) {
    return reinterpret_cast<char*>(ws) + fw_ws_bytes(n, ld, eb) - 256 - fw_b2_bytes(n, eb);
}

// smx_set_fw_packed: phase 3 on the warp-specialised packed-tile kernel
static std::atomic<int> g_fw_packed{1};

// Phase 3 (3b) product: C rows outside [skip0, skip0 + skipn) (+)= CP (x) rowK.
template <typename T>
int fw_phase3(const T* CP, long long ldcp, const T* rowK, T* Tm, int n, long long ld, int bb, int kind,
              int skip0, int skipn, void* pws, size_t pws_bytes, cudaStream_t s) {
    if (g_fw_packed && pws != nullptr)
        return semiring_gemm_packed<T>(CP, rowK, Tm, n, n, bb, ldcp, ld, ld, kind, 1, skip0, skipn, pws,
                                       pws_bytes, s);
    return semiring_gemm<T>(CP, rowK, Tm, n, n, bb, ldcp, ld, ld, kind, 1, skip0, skipn, s);
}



// Optional CUDA-event trace of the phase-3 launches (the dominant kernel), so
// bench.py can time that kernel live inside the timed region on the stream
// it runs on.  Armed by smx_fw_trace_arm, filled by the next smx_fw_* call.
struct FwTrace {
    static constexpr int kCap = 2048;
    cudaEvent_t ev[2 * kCap] = {};
    long long cells[kCap] = {};
    int count = 0, cap = 0;
    bool armed = false;
};
static FwTrace g_trace;

void trace_begin(cudaStream_t s, long long cells) {
    if (!g_trace.armed || g_trace.count >= g_trace.cap) return;
    g_trace.cells[g_trace.count] = cells;
    cudaEventRecord(g_trace.ev[2 * g_trace.count], s);
}
void trace_end(cudaStream_t s) {
    if (!g_trace.armed || g_trace.count >= g_trace.cap) return;
    cudaEventRecord(g_trace.ev[2 * g_trace.count + 1], s);
    ++g_trace.count;
}

// Pivot tile + pivot row panel of block [k0, k0+bb): T[K,:] (+)= T[K,K]* (x) T[K,:].
// smx_set_fw_packed_panel: the look-ahead's row panel on the packed kernel
// (its A = the closed pivot tile and B = the panel itself packed first, into
// the RP region, then C = the panel updated in place from the snapshot).
// 0 = never, 1 = automatic (n >= 8192), 2 = always.  Measured
// (tools/perf_switch.py, profiles/r03c_packed_panel_ab.jsonl): n = 8192
// 17.26 -> 16.93-17.11 ms (the 6% of the cells the side chain computes run
// at the packed kernel's rate); n = 2048 / 4096 +10% / +4.5% (two more
// launches on a chain that binds there); n = 16384 unchanged.
static std::atomic<int> g_fw_packed_panel{1};
inline bool packed_panel_for(int n) {
    const int m = g_fw_packed_panel.load(std::memory_order_relaxed);
    return m == 2 || (m == 1 && n >= 8192);
}

template <typename T>
int fw_pivot_and_row_panel(T* Tm, int n, long long ld, int kind, T* RP, int k0, int bb, cudaStream_t s,
                           bool lite = false, bool packed_panel = false) {
    T* rowK = Tm + (long long)k0 * ld;
    // (the lite pivot's shared-memory tile holds 256 x 256 u16 or 128 x 128 u32)
    if (lite && bb <= (sizeof(T) == 4 ? 128 : 256)) SMX_TRY(fw_pivot_lite<T>(rowK + k0, bb, ld, kind, s));
    else SMX_TRY(fw_pivot<T>(rowK + k0, bb, ld, kind, s, RP));   // RP: the pivot's scratch
    // Row panel in place, no snapshot: T[K,:] (+)= P* (x) T[K,:] with
    // P* = T[K,K] closed.  A CTA may read (through the read-only path) rows K
    // that another CTA has already updated; every such value lies between the
    // old value and the final one, and P* (x) final = P* (x) old because
    // P* (x) P* = P* (closure, weights >= 0) -- so the result is the same for
    // any interleaving.  The P* tile itself is rewritten with its own value.
    if (lite) return semiring_gemm_lite<T>(rowK + k0, rowK, rowK, bb, n, bb, ld, ld, ld, kind, s);
    if (packed_panel && RP != nullptr && packed_panel_for(n))
        return semiring_gemm_packed<T>(rowK + k0, rowK, rowK, bb, n, bb, ld, ld, ld, kind, 1, 0, 0, RP,
                                       packed_ws_bytes_t<T>(bb, n, bb), s);
    return semiring_gemm<T>(rowK + k0, rowK, rowK, bb, n, bb, ld, ld, ld, kind, 1, 0, 0, s);
}

// smx_set_fw_split_3a: the look-ahead's 3a in two parts (diagonal tile
// first, the pivot right behind it, the rest of the rows on a second side
// stream): 0 = never, 1 = automatic (currently never: see fw_rounds_packed),
// 2 = always.
static std::atomic<int> g_fw_split_3a{1};

// Side-stream kernel footprint.  Measured: the co-residable Lite row-panel
// tiles gain nothing over the regular ones (the side chain already hides
// behind phase 3) and lose ~1-2%, so the regular tiles are the default.
static std::atomic<int> g_side_lite{0};

// Look-ahead schedule.  The main stream s runs the phase-3 GEMMs; the side
// stream computes pivot block r+1 (pivot tile + row panel) as soon as its
// rows have received round r's update, concurrently with the bulk of round
// r's phase 3:
//   s   : 3a(r): rows K_{r+1}      -> fork ->  3b(r): rows outside K_r, K_{r+1}
//         -> CP(r+1) snapshot -> wait(join) -> 3a(r+1) ...
//   side: wait(fork) -> pivot(r+1), row panel(r+1) -> join
// 3b(r) only reads CP(r) and T[K_r,:] and writes rows outside K_r u K_{r+1},
// the side stream only touches rows K_{r+1} and RP, so the two never touch
// the same bytes.  Rows K_{r+1} of CP(r+1) are copied while the side stream
// may still write them, but phase 3 of round r+1 skips exactly those rows.
template <typename T>
int fw_run_lookahead(T* Tm, int n, long long ld, int kind, T* RP, T* CP, void* pws, size_t pws_bytes,
                     cudaStream_t s) {
    SideStream* fs = nullptr;
    SMX_TRY(side_stream(&fs));
    const int BLK = fw_block_for_n<T>(n);
    const long long ldcp = BLK;
    const int R = (n + BLK - 1) / BLK;
    SMX_TRY(fw_pivot_and_row_panel<T>(Tm, n, ld, kind, RP, 0, n < BLK ? n : BLK, s));
    SMX_TRY(copy_panel<T>(Tm, ld, CP, ldcp, n, n < BLK ? n : BLK, s));
    cudaError_t e;
    for (int r = 0; r < R; ++r) {
        const int k0 = r * BLK, bb = n - k0 < BLK ? n - k0 : BLK;
        T* rowK = Tm + (long long)k0 * ld;
        if (r + 1 < R) {
            const int k1 = k0 + BLK, bb1 = n - k1 < BLK ? n - k1 : BLK;
            // 3a: the next pivot block's rows first
            SMX_TRY(semiring_gemm<T>(CP + k1 * ldcp, rowK, Tm + (long long)k1 * ld, bb1, n, bb, ldcp, ld, ld,
                                     kind, 1, 0, 0, s));
            if ((e = cudaEventRecord(fs->fork, s)) != cudaSuccess) return (int)e;
            if ((e = cudaStreamWaitEvent(fs->side, fs->fork, 0)) != cudaSuccess) return (int)e;
            {
                PriorityScope ps(fs->priority);
                SMX_TRY(fw_pivot_and_row_panel<T>(Tm, n, ld, kind, RP, k1, bb1, fs->side, g_side_lite != 0));
            }
            if ((e = cudaEventRecord(fs->join, fs->side)) != cudaSuccess) return (int)e;
            // 3b: everything else (skips K_r and K_{r+1}, adjacent tiles)
            trace_begin(s, (long long)(n - bb - bb1) * n * bb);
            SMX_TRY(fw_phase3<T>(CP, ldcp, rowK, Tm, n, ld, bb, kind, k0, bb + bb1, pws, pws_bytes, s));
            trace_end(s);
            SMX_TRY(copy_panel<T>(Tm + k1, ld, CP, ldcp, n, bb1, s));
            if ((e = cudaStreamWaitEvent(s, fs->join, 0)) != cudaSuccess) return (int)e;
        } else {
            trace_begin(s, (long long)(n - bb) * n * bb);
            SMX_TRY(fw_phase3<T>(CP, ldcp, rowK, Tm, n, ld, bb, kind, k0, bb, pws, pws_bytes, s));
            trace_end(s);
        }
    }
    return SMX_OK;
}

// u8/u16 look-ahead on packed operand tiles.  Round r:
//   main: pack B(r) from T[K_r,:] -> fork -> 3b: packed rows outside K_r,
//         K_{r+1} -> wait(3a done) -> pack A(r+1) from T[:, K_{r+1}] -> wait(join)
//   side: wait(fork) -> 3a: packed rows K_{r+1} -> record(3a done) ->
//         pivot(r+1) -> row panel(r+1) -> record(join)
// 3a sits on the side chain, so the main stream never runs the one-wave 3a
// product on a mostly idle GPU: the side chain (3a, pivot, row panel) hides
// behind 3b.  3a writes rows K_{r+1}, which 3b skips; both only read the
// packed tiles, and pack A(r+1) (which rewrites them) waits for 3a.
// The packed A tiles are the column-panel snapshot (no separate CP copy).
// pack A(r+1) reads rows K_{r+1} while the side stream may still rewrite
// them, but only tiles of rows K_{r+2} (3a) and of rows outside K_{r+1} u
// K_{r+2} (3b) are read in round r+1, as with the CP copy of fw_run_lookahead.
//
// Rounds [ra, rb) over the row window [lo, hi) (the whole closure: rows
// [0, n), rounds [0, R)).  Every pivot block of those rounds lies inside the
// window; lo is a multiple of the 128-row tile, hi one too or n.  Rows
// outside the window are neither read as A nor written (the host-streamed
// closure below runs rounds on the rows that have arrived so far).
// The first kFwCertRounds rounds of a call run certified when their operands
// allow it: the column panel and the row panel hold only unreachable (S) or
// lanes < 2^14 -- true of the input graph (weights <= 1000) -- so every tile
// takes the 1-instruction shifted encoding of the public products
// (Lane<uint16_t>::to_shifted).  Without it round 0 runs the general
// 2-instruction form on every tile (the input is 98% unreachable, so no tile
// passes the per-tile bounded test): measured 16.5 against 33.9 Tcell/s at
// n = 32768.  Later rounds are bounded anyway.  A certified round packs its
// A tiles after the previous round's join (its row panel must be final).
constexpr int kFwCertRounds = 2;

template <typename T>
int fw_rounds_packed(T* Tm, int n, long long ld, int kind, T* RP, void* pws, size_t pws_bytes, int lo, int hi,
                     int ra, int rb, cudaStream_t s, int* cert = nullptr, void* b2 = nullptr) {
    using G = PackedCfg<T>;
    SideStream* fs = nullptr;
    SMX_TRY(side_stream(&fs));
    const int BLK = fw_block_for_n<T>(n);
    auto blk = [&](int r) { return n - r * BLK < BLK ? n - r * BLK : BLK; };
    const int t0 = lo / G::BM, tiles = ceil_div(hi, G::BM) - t0;
    if (ra >= rb) return SMX_OK;
    const bool can_cert = cert != nullptr && !Lane<T>::kOneInstr && bounded_fastpath_enabled();
    auto certified = [&](int r) { return can_cert && r - ra < kFwCertRounds; };
    // Double-buffered row panels (b2 != nullptr): round r's packed B lives in
    // the workspace's own B block (r - ra even) or in b2 (odd), so the side
    // chain of round r packs round r+1's row panel right after computing it,
    // beside round r's phase 3, instead of the main stream packing it between
    // the two phase-3 launches.  Round r+1's buffer was last read by round
    // r-1's 3a (earlier on the side stream) and 3b (before this round's fork
    // on the main stream).  A certified round packs its B on the main stream
    // after its certificate, as before.
    auto bbuf = [&](int r) -> void* { return (b2 != nullptr && ((r - ra) & 1)) ? b2 : nullptr; };
    // The workspace's own B block sits behind the packed A tiles, whose size
    // depends on the round's K: a ragged last block (blk(r) < BLK) puts its B
    // tiles inside the region round r-1's A tiles still occupy, so the side
    // chain may not pack them there beside round r-1's phase 3 (it corrupted
    // A tiles phase 3 had yet to read: wrong closures, timing dependent, for
    // n with an odd number of rounds and a last block of fewer k-tiles, e.g.
    // n = 7000 or 8000 at BLK = 128, 8300 at 256).  That round packs its B
    // on the main stream after the join, as a single-buffered round does.
    auto side_packs_b = [&](int r) {
        return b2 != nullptr && r > ra && !certified(r) && (bbuf(r) != nullptr || blk(r) == BLK);
    };
    SMX_TRY(fw_pivot_and_row_panel<T>(Tm, n, ld, kind, RP, ra * BLK, blk(ra), s, false, true));
    if (!certified(ra))
        SMX_TRY(packed_pack_a_rows<T>(Tm + ra * BLK, n, n, blk(ra), ld, kind, pws, pws_bytes, t0, tiles, s));
    cudaError_t e;
    for (int r = ra; r < rb; ++r) {
        const int k0 = r * BLK, bb = blk(r);
        T* rowK = Tm + (long long)k0 * ld;
        const int* cr = nullptr;
        if constexpr (!Lane<T>::kOneInstr) {
            if (certified(r)) {
                SMX_TRY(run_cert<T>(Tm + (long long)lo * ld + k0, hi - lo, bb, ld, rowK, bb, n, ld,
                                    kind == SMX_ANTI, cert, s));
                cr = cert;
                SMX_TRY(packed_pack_a_rows<T>(Tm + k0, n, n, bb, ld, kind, pws, pws_bytes, t0, tiles, s, cr));
            }
        }
        if (!side_packs_b(r))
            SMX_TRY(packed_pack<T>(nullptr, rowK, n, n, bb, ld, ld, kind, pws, pws_bytes, s, cr, bbuf(r)));
        void* wb = bbuf(r);
        if (r + 1 < rb) {
            const int k1 = k0 + BLK, bb1 = blk(r + 1);
            if ((e = cudaEventRecord(fs->fork, s)) != cudaSuccess) return (int)e;
            if ((e = cudaStreamWaitEvent(fs->side, fs->fork, 0)) != cudaSuccess) return (int)e;
            // 3a split (g_fw_split_3a): the pivot only needs the diagonal
            // tile T[K1, K1] updated by round r, so that part goes first on
            // the side stream and the pivot follows it at once, while the
            // rest of rows K1 (every other column) is updated on the second
            // side stream; the row panel waits for both.  The two parts
            // write disjoint columns of rows K1, and the pivot touches only
            // T[K1, K1].
            // Automatic = off: measured (tools/perf_switch.py smx_set_fw_split_3a 0 2) a gain only
            // at n = 4096 (2.88 -> 2.69-2.79 ms) and small losses at 1024,
            // 2048, 6144 and 8192 (17.50 -> 17.65 ms): the extra launches and
            // the second stream's 3a CTAs beside the pivot cost about what
            // the shorter chain saves.
            const int sm3 = g_fw_split_3a.load(std::memory_order_relaxed);
            const bool split = n > bb1 && sm3 == 2;
            if (split && (e = cudaStreamWaitEvent(fs->side2, fs->fork, 0)) != cudaSuccess) return (int)e;
            {
                PriorityScope ps(fs->priority);
#if defined(SMX_TRACE_SIDE) && !defined(SMX_TRACE_SIDE_PARTS)   // development builds: side-chain spans (cells = -1)
                trace_begin(fs->side, -1);
#endif
#ifdef SMX_TRACE_SIDE_PARTS   // 3a, pivot, row panel as separate entries (cells -2, -3, -4)
                trace_begin(fs->side, -2);
#endif
                // 3a: the next pivot block's rows
                if (split) {
                    const int c0 = k1 / G::BN, cn = ceil_div(k1 + bb1, G::BN) - c0;
                    SMX_TRY(packed_run<T>(Tm, n, n, bb, ld, kind, 1, k1 / G::BM, ceil_div(bb1, G::BM), 0, 0, pws,
                                          pws_bytes, fs->side, cr, c0, cn, wb));
                    SMX_TRY(packed_run<T>(Tm, n, n, bb, ld, kind, 1, k1 / G::BM, ceil_div(bb1, G::BM), 0, 0, pws,
                                          pws_bytes, fs->side2, cr, 0, c0, wb));
                    SMX_TRY(packed_run<T>(Tm, n, n, bb, ld, kind, 1, k1 / G::BM, ceil_div(bb1, G::BM), 0, 0, pws,
                                          pws_bytes, fs->side2, cr, c0 + cn, -1, wb));
                    if ((e = cudaEventRecord(fs->aux2, fs->side2)) != cudaSuccess) return (int)e;
                } else {
                    SMX_TRY(packed_run<T>(Tm, n, n, bb, ld, kind, 1, k1 / G::BM, ceil_div(bb1, G::BM), 0, 0, pws,
                                          pws_bytes, fs->side, cr, 0, -1, wb));
                }
#ifdef SMX_TRACE_SIDE_PARTS
                trace_end(fs->side);
                trace_begin(fs->side, -3);
                SMX_TRY(fw_pivot<T>(Tm + (long long)k1 * ld + k1, bb1, ld, kind, fs->side, RP));
                trace_end(fs->side);
                trace_begin(fs->side, -4);
                SMX_TRY(semiring_gemm<T>(Tm + (long long)k1 * ld + k1, Tm + (long long)k1 * ld, Tm + (long long)k1 * ld,
                                         bb1, n, bb1, ld, ld, ld, kind, 1, 0, 0, fs->side));
                trace_end(fs->side);
#endif
                if ((e = cudaEventRecord(fs->aux, fs->side)) != cudaSuccess) return (int)e;
#ifndef SMX_TRACE_SIDE_PARTS
                if (split) {
                    SMX_TRY(fw_pivot<T>(Tm + (long long)k1 * ld + k1, bb1, ld, kind, fs->side, RP));
                    if ((e = cudaStreamWaitEvent(fs->side, fs->aux2, 0)) != cudaSuccess) return (int)e;
                    T* rowK1 = Tm + (long long)k1 * ld;
                    if (packed_panel_for(n))
                        SMX_TRY(semiring_gemm_packed<T>(rowK1 + k1, rowK1, rowK1, bb1, n, bb1, ld, ld, ld, kind, 1,
                                                        0, 0, RP, packed_ws_bytes_t<T>(bb1, n, bb1), fs->side));
                    else
                        SMX_TRY(semiring_gemm<T>(rowK1 + k1, rowK1, rowK1, bb1, n, bb1, ld, ld, ld, kind, 1, 0, 0,
                                                 fs->side));
                } else {
                    SMX_TRY(fw_pivot_and_row_panel<T>(Tm, n, ld, kind, RP, k1, bb1, fs->side, g_side_lite != 0,
                                                      true));
                }
#endif
                // round r+1's row panel, packed as soon as it is final
                if (side_packs_b(r + 1))
                    SMX_TRY(packed_pack<T>(nullptr, Tm + (long long)k1 * ld, n, n, bb1, ld, ld, kind, pws, pws_bytes,
                                           fs->side, nullptr, bbuf(r + 1)));
#if defined(SMX_TRACE_SIDE) && !defined(SMX_TRACE_SIDE_PARTS)
                trace_end(fs->side);
#endif
            }
            if ((e = cudaEventRecord(fs->join, fs->side)) != cudaSuccess) return (int)e;
            // 3b: everything else in the window (skips K_r and K_{r+1}, adjacent tiles)
            trace_begin(s, (long long)(hi - lo - bb - bb1) * n * bb);
            SMX_TRY(packed_run<T>(Tm, n, n, bb, ld, kind, 1, t0, tiles, k0, bb + bb1, pws, pws_bytes, s, cr, 0, -1,
                                  wb));
            trace_end(s);
            if ((e = cudaStreamWaitEvent(s, fs->aux, 0)) != cudaSuccess) return (int)e;
            // (pack A(r+1) overwrites the packed A tiles both 3a parts read)
            if (split && (e = cudaStreamWaitEvent(s, fs->aux2, 0)) != cudaSuccess) return (int)e;
            if (!certified(r + 1))   // (a certified round packs its own A after the join)
                SMX_TRY(packed_pack_a_rows<T>(Tm + k1, n, n, bb1, ld, kind, pws, pws_bytes, t0, tiles, s));
            if ((e = cudaStreamWaitEvent(s, fs->join, 0)) != cudaSuccess) return (int)e;
        } else {
            trace_begin(s, (long long)(hi - lo - bb) * n * bb);
            SMX_TRY(packed_run<T>(Tm, n, n, bb, ld, kind, 1, t0, tiles, k0, bb, pws, pws_bytes, s, cr, 0, -1, wb));
            trace_end(s);
        }
    }
    return SMX_OK;
}

// smx_set_fw_panel_buffers: 2 = double-buffered packed row panels (the side
// chain packs the next one), 1 = one buffer packed on the main stream.
static std::atomic<int> g_fw_panel_buffers{2};

template <typename T>
int fw_run_lookahead_packed(T* Tm, int n, long long ld, int kind, T* RP, void* pws, size_t pws_bytes,
                            cudaStream_t s, int* cert = nullptr, void* b2 = nullptr) {
    const int BLK = fw_block_for_n<T>(n);
    return fw_rounds_packed<T>(Tm, n, ld, kind, RP, pws, pws_bytes, 0, n, 0, (n + BLK - 1) / BLK, s, cert, b2);
}

template <typename T>
int fw_run_serial(T* Tm, int n, long long ld, int kind, T* RP, T* CP, void* pws, size_t pws_bytes, int BLK,
                  cudaStream_t s);

template <typename T>
int fw_run(T* Tm, int n, long long ld, int kind, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (n < 0 || ld < n || (kind != SMX_ANTI && kind != SMX_DIST)) return SMX_E_ARG;
    if (n == 0) return SMX_OK;
    if (!aligned16(Tm) || !ld_ok(ld, sizeof(T))) return SMX_E_ALIGN;
    const int BLK = fw_block_for_n<T>(n);
    if (n <= FwBlock<T>::value) return fw_pivot<T>(Tm, n, ld, kind, s, nullptr);
    if (ws == nullptr || ws_bytes < fw_ws_bytes(n, ld, sizeof(T))) return SMX_E_WORKSPACE;
    T* RP = reinterpret_cast<T*>(ws);
    T* CP = reinterpret_cast<T*>(reinterpret_cast<char*>(ws) + fw_rp_bytes(n, ld, sizeof(T)));
    const size_t pws_off = fw_rp_bytes(n, ld, sizeof(T)) +
                           align256((size_t)n * FwBlock<T>::value * sizeof(T));
    void* pws = reinterpret_cast<char*>(ws) + pws_off;
    const size_t pws_bytes = ws_bytes - pws_off;
    GraphKey key;
    key.fn = 100 + (int)sizeof(T);
    const unsigned long long kv[] = {(uintptr_t)Tm, (unsigned long long)n, (unsigned long long)ld,
                                     (unsigned long long)kind, (uintptr_t)ws, ws_bytes,
                                     (unsigned long long)lookahead_enabled(), (unsigned long long)g_side_lite.load(),
                                     (unsigned long long)g_fw_block_override.load(), (unsigned long long)g_fw_packed.load(),
                                     (unsigned long long)bounded_fastpath_enabled(),
                                     (unsigned long long)g_pivot_blocked.load() |
                                         ((unsigned long long)g_fw_split_3a.load() << 1) |
                                         ((unsigned long long)g_pivot_pairs.load() << 3) |
                                         ((unsigned long long)g_fw_packed_panel.load() << 4) |
                                         ((unsigned long long)g_fw_panel_buffers.load() << 6) |
                                         ((unsigned long long)(unsigned)packed_producer_backoff() << 8)};
    for (size_t i = 0; i < sizeof(kv) / sizeof(kv[0]); ++i) key.v[i] = kv[i];
    // the phase-3 trace records host-side state per launch: trace runs stay eager
    return run_graphed(key, s, g_trace.armed, [&](cudaStream_t st) -> int {
        if (lookahead_enabled() && g_fw_packed)
            return fw_run_lookahead_packed<T>(Tm, n, ld, kind, RP, pws, pws_bytes, st,
                                              fw_cert_slot(ws, n, ld, sizeof(T)),
                                              g_fw_panel_buffers.load() == 2 ? fw_b2_slot(ws, n, ld, sizeof(T))
                                                                             : nullptr);
        if (lookahead_enabled()) return fw_run_lookahead<T>(Tm, n, ld, kind, RP, CP, pws, pws_bytes, st);
        return fw_run_serial<T>(Tm, n, ld, kind, RP, CP, pws, pws_bytes, BLK, st);
    });
}

template <typename T>
int fw_run_serial(T* Tm, int n, long long ld, int kind, T* RP, T* CP, void* pws, size_t pws_bytes, int BLK,
                  cudaStream_t s) {
    const long long ldcp = BLK;
    for (int k0 = 0; k0 < n; k0 += BLK) {
        const int bb = n - k0 < BLK ? n - k0 : BLK;
        T* rowK = Tm + (long long)k0 * ld;
        SMX_TRY(fw_pivot<T>(rowK + k0, bb, ld, kind, s, RP));   // RP is free until the snapshot
        cudaError_t e = cudaMemcpyAsync(RP, rowK, (size_t)bb * ld * sizeof(T),
                                        cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return (int)e;
        SMX_TRY(semiring_gemm<T>(RP + k0, RP, rowK, bb, n, bb, ld, ld, ld, kind, 1, 0, 0, s));
        e = cudaMemcpy2DAsync(CP, ldcp * sizeof(T), Tm + k0, ld * sizeof(T), bb * sizeof(T), n,
                              cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return (int)e;
        trace_begin(s, (long long)(n - bb) * n * bb);
        SMX_TRY(fw_phase3<T>(CP, ldcp, rowK, Tm, n, ld, bb, kind, k0, bb, pws, pws_bytes, s));
        trace_end(s);
    }
    return SMX_OK;
}

// ---- closure of a host matrix (smx_fw_host_*) -------------------------------
// Host in -> device -> closure -> host out in one call, with the PCIe copies
// hidden behind the closure instead of before and after it.  Two exact
// identities let rows enter and leave the computation at different times
// (d_X(i, x): shortest walk i -> x with >= 1 edge and intermediates in X;
// rows are in distance form, saturation commutes with both: SURVEY 0.1 fact 2):
//
//  * ingest (first vertex of [0, s) on the walk): rows that arrive after the
//    rows [0, s) were closed over intermediates [0, s) catch up with ONE
//    product of K = s,
//        T[G, :] (+)= T[G, 0:s] (x) T[0:s, :],
//    then join the ordinary rounds.  A walk i -> x through [0, s) leaves i by
//    a single edge (i, l), l the first vertex of [0, s) on it, and continues
//    as a walk l -> x over [0, s): that is T[i, l] (x) d_[0,s)(l, x).
//  * egress (first vertex of L on the walk): once the last rows L are
//    closed (their own rounds, on rows L only), every other row finishes with
//    ONE product of K = |L|,
//        T[i, :] (+)= T[i, L] (x) T[L, :],
//    T[i, L] closed over [0, n) \ L: the walk i -> l (l the first vertex of L)
//    avoids L, the rest l -> x is anything.  So rows [0, n) \ L finish chunk
//    by chunk, and each chunk's D2H starts as soon as its product is done.
// Any in-place update that a later K-block of the same product reads is the
// weight of a real walk of the same kind, so it can only tighten towards the
// exact value (the argument of fw_pivot_and_row_panel).  Every (row, pivot)
// pair is still applied exactly once: no extra work.
//
// Rows arrive in groups [0, B), [B, 2B), [2B, 4B), ... [8B, 16B), [16B, 64B),
// ..., the last one running to n; the main stream waits for each group's H2D event only when
// it needs that group, so the copy engine and the SMs run concurrently.  The
// products run one pivot block of K per launch, like phase 3: with K = 512
// the packed operands of a launch (~60 MB) stay in L2, while K = 2048 spills
// and ran the catch-up products 12% slower (n = 32768: 1080 vs 1040 ms).
namespace {
struct CopyStreams {
    cudaStream_t in = nullptr, out = nullptr;
    std::vector<cudaEvent_t> ev;
    std::mutex mu;   // one streamed call at a time per device (shared events)
};
int copy_streams(CopyStreams** out) {
    static CopyStreams per_dev[64];
    static std::mutex mu;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    if (dev < 0 || dev >= 64) return SMX_E_ARG;
    CopyStreams& c = per_dev[dev];
    std::lock_guard<std::mutex> lock(mu);
    if (!c.in) {
        if ((e = cudaStreamCreateWithFlags(&c.in, cudaStreamNonBlocking)) != cudaSuccess) return (int)e;
        if ((e = cudaStreamCreateWithFlags(&c.out, cudaStreamNonBlocking)) != cudaSuccess) return (int)e;
    }
    *out = &c;
    return SMX_OK;
}
int copy_events(CopyStreams* c, size_t count) {
    while (c->ev.size() < count) {
        cudaEvent_t ev;
        cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return (int)e;
        c->ev.push_back(ev);
    }
    return SMX_OK;
}
}  // namespace

// The last four pivot blocks L are closed alone at the end (egress); their
// four row blocks stay packed as B while the other rows finish.
constexpr int kFwHostTailBlocks = 4;
// smx_set_fw_host_stream: 0 = never stream (copy in, close, copy out),
// 1 = automatic, 2 = stream whenever the closure has >= 8 pivot blocks (tests).
// Automatic streams from n = 16384: below that the copies are a few ms and
// the small early windows' rounds, bound by the pivot chain, cost more than
// the overlap saves (n = 8192: 23.7 ms streamed vs 23.0 ms serial; 16384:
// 141 vs 152 ms; 32768: 1040 vs 1105 ms, tools/perf_host_fw.py).
static std::atomic<int> g_fw_host_stream{1};

inline size_t fw_host_slot_bytes(int n, int eb) {
    return align256(packed_ws_bytes_eb(n, n, fw_block_for(eb), eb));
}
inline size_t fw_host_ws_bytes(int n, long long ld, int eb) {
    return fw_ws_bytes(n, ld, eb) + kFwHostTailBlocks * fw_host_slot_bytes(n, eb);
}

// Egress chunk boundaries over rows [0, sL): from the end, 1, 1, 2, 4, 8, 16,
// 16, ... blocks, so each chunk's D2H (0.85 ms per 1024 rows at n = 32768)
// hides behind the next chunk's product (2 ms per 1024 rows) and only the
// last block of rows is copied after the final product.
inline std::vector<int> fw_host_egress_cuts(int sL, int BLK) {
    std::vector<int> sizes;
    int left = sL / BLK, next = 1, ones = 0;
    while (left > 0) {
        const int take = next < left ? next : left;
        sizes.push_back(take);
        left -= take;
        if (next == 1 && ones++ == 0) continue;   // two single blocks at the end
        if (next < 16) next *= 2;
    }
    std::vector<int> cuts{0};
    for (auto it = sizes.rbegin(); it != sizes.rend(); ++it) cuts.push_back(cuts.back() + *it * BLK);
    return cuts;
}

template <typename T>
int fw_host_run(const T* hin, T* hout, T* Tm, int n, long long ld, int kind, void* ws, size_t ws_bytes,
                cudaStream_t s) {
    using G = PackedCfg<T>;
    if (n < 0 || ld < n || (kind != SMX_ANTI && kind != SMX_DIST)) return SMX_E_ARG;
    if (n == 0) return SMX_OK;
    if (hin == nullptr || hout == nullptr || Tm == nullptr) return SMX_E_ARG;
    if (!aligned16(Tm) || !ld_ok(ld, sizeof(T))) return SMX_E_ALIGN;
    const size_t row_bytes = (size_t)ld * sizeof(T);
    const int BLK = fw_block_for_n<T>(n);
    const int R = (n + BLK - 1) / BLK;
    cudaError_t e;
    const int mode = g_fw_host_stream.load(std::memory_order_relaxed);
    const bool streamed = lookahead_enabled() && g_fw_packed && R >= 2 * kFwHostTailBlocks &&
                          (mode == 2 || (mode == 1 && n >= 16384));
    if (!streamed) {   // small: copy in, close, copy out, in stream order
        if ((e = cudaMemcpyAsync(Tm, hin, (size_t)n * row_bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return (int)e;
        SMX_TRY(fw_run<T>(Tm, n, ld, kind, ws, ws_bytes, s));
        e = cudaMemcpyAsync(hout, Tm, (size_t)n * row_bytes, cudaMemcpyDeviceToHost, s);
        return e == cudaSuccess ? SMX_OK : (int)e;
    }
    if (ws == nullptr || ws_bytes < fw_host_ws_bytes(n, ld, sizeof(T))) return SMX_E_WORKSPACE;
    T* RP = reinterpret_cast<T*>(ws);
    const size_t pws_off = fw_rp_bytes(n, ld, sizeof(T)) +
                           align256((size_t)n * FwBlock<T>::value * sizeof(T));
    void* pws = reinterpret_cast<char*>(ws) + pws_off;
    const size_t slot = fw_host_slot_bytes(n, sizeof(T));
    int* cert = fw_cert_slot(ws, n, ld, sizeof(T));
    void* b2 = g_fw_panel_buffers.load() == 2 ? fw_b2_slot(ws, n, ld, sizeof(T)) : nullptr;
    auto egress_slot = [&](int j) { return reinterpret_cast<char*>(ws) + fw_ws_bytes(n, ld, sizeof(T)) + j * slot; };

    const int sL = (R - kFwHostTailBlocks) * BLK;   // L = rows [sL, n)
    std::vector<int> ends;                          // ingest groups; the last one runs to n
    // Doubling while a group's work (~n r^2 cells) is shorter than the next
    // group's copy, x4 after that: the SMs never wait on the copy engine
    // after the first block (n = 32768: 512, 1024, 2048, 4096, 8192, n).
    for (long long x = BLK; x < sL; x *= (x < 16LL * BLK ? 2 : 4)) ends.push_back((int)x);
    ends.push_back(n);
    const std::vector<int> cuts = fw_host_egress_cuts(sL, BLK);
    const int chunks = (int)cuts.size() - 1;

    CopyStreams* cs = nullptr;
    SMX_TRY(copy_streams(&cs));
    std::lock_guard<std::mutex> lock(cs->mu);
    // events: fork, join, one per group, one per D2H piece (L + chunks)
    SMX_TRY(copy_events(cs, 2 + ends.size() + 1 + chunks));
    cudaEvent_t ev_fork = cs->ev[0], ev_join = cs->ev[1];
    cudaEvent_t* ev_in = cs->ev.data() + 2;
    cudaEvent_t* ev_out = ev_in + ends.size();
    if ((e = cudaEventRecord(ev_fork, s)) != cudaSuccess) return (int)e;
    if ((e = cudaStreamWaitEvent(cs->in, ev_fork, 0)) != cudaSuccess) return (int)e;
    if ((e = cudaStreamWaitEvent(cs->out, ev_fork, 0)) != cudaSuccess) return (int)e;
    // Page-locked input: every group's H2D is queued now.  Pageable input
    // (an ordinary numpy array, the reference's own call): staged through
    // page-locked slots by a coordinator thread (host_stage.cuh), which
    // records each group's event; the loop below waits on the host for that
    // record before making the main stream wait on the event.
    HostStager stager;
    const bool staged = is_pageable(hin);
    if (staged) {
        SMX_TRY(stager.start(hin, Tm, row_bytes, ends, ev_in, cs->in));
    } else {
        for (size_t g = 0, r0 = 0; g < ends.size(); r0 = ends[g], ++g) {
            if ((e = cudaMemcpyAsync(Tm + r0 * ld, hin + r0 * ld, (ends[g] - r0) * row_bytes,
                                     cudaMemcpyHostToDevice, cs->in)) != cudaSuccess)
                return (int)e;
            if ((e = cudaEventRecord(ev_in[g], cs->in)) != cudaSuccess) return (int)e;
        }
    }
    // Page-locked output: each finished piece is one D2H on the copy-out
    // stream.  Pageable output (an ordinary numpy array, e.g. the in-place
    // closure of the caller's own array): staged back through the
    // page-locked ring by a coordinator thread (HostEgress), so the copy out
    // still overlaps the rest of the closure; the call then returns once
    // every row is in host_out.
    HostEgress egress;
    const bool egress_staged = is_pageable(hout);
    if (egress_staged) SMX_TRY(egress.start(Tm, hout, cs->out));
    auto d2h = [&](int r0, int r1, cudaEvent_t ev) -> int {
        cudaError_t e2;
        if ((e2 = cudaEventRecord(ev, s)) != cudaSuccess) return (int)e2;
        if (egress_staged) {
            egress.push((size_t)r0 * row_bytes, (size_t)r1 * row_bytes, ev);
            return SMX_OK;
        }
        if ((e2 = cudaStreamWaitEvent(cs->out, ev, 0)) != cudaSuccess) return (int)e2;
        e2 = cudaMemcpyAsync(hout + (size_t)r0 * ld, Tm + (size_t)r0 * ld, (size_t)(r1 - r0) * row_bytes,
                             cudaMemcpyDeviceToHost, cs->out);
        return e2 == cudaSuccess ? SMX_OK : (int)e2;
    };

    for (size_t g = 0, r0 = 0; g < ends.size(); r0 = ends[g], ++g) {
        const int r1 = ends[g];
        const int t0 = (int)r0 / G::BM, tiles = ceil_div(r1, G::BM) - t0;
        if (staged) SMX_TRY(stager.wait_recorded((int)g));
        if ((e = cudaStreamWaitEvent(s, ev_in[g], 0)) != cudaSuccess) return (int)e;
        // ingest: T[G, :] (+)= T[G, 0:r0] (x) T[0:r0, :], one pivot block of K per launch.
        // The first block's A tiles are the raw arrived rows (mostly
        // unreachable): certified like fw_rounds_packed's first rounds; later
        // blocks read rows the first product has already filled in.
        for (int k0 = 0; k0 < (int)r0; k0 += BLK) {
            const int* cr = nullptr;
            if constexpr (!Lane<T>::kOneInstr) {
                if (k0 == 0 && bounded_fastpath_enabled()) {
                    SMX_TRY(run_cert<T>(Tm + r0 * ld, r1 - (int)r0, BLK, ld, Tm, BLK, n, ld, kind == SMX_ANTI,
                                        cert, s));
                    cr = cert;
                }
            }
            SMX_TRY(packed_pack<T>(nullptr, Tm + (long long)k0 * ld, n, n, BLK, ld, ld, kind, pws, slot, s, cr));
            SMX_TRY(packed_pack_a_rows<T>(Tm + k0, n, n, BLK, ld, kind, pws, slot, t0, tiles, s, cr));
            SMX_TRY(packed_run<T>(Tm, n, n, BLK, ld, kind, 1, t0, tiles, 0, 0, pws, slot, s, cr));
        }
        // the group's rounds over every row that has arrived (the last group:
        // all rows, up to the blocks of L)
        const int rb = (r1 < n ? r1 : sL) / BLK;
        SMX_TRY(fw_rounds_packed<T>(Tm, n, ld, kind, RP, pws, slot, 0, r1, (int)r0 / BLK, rb, s, cert, b2));
    }
    // L: its rounds on rows L alone; then L is final
    SMX_TRY(fw_rounds_packed<T>(Tm, n, ld, kind, RP, pws, slot, sL, n, sL / BLK, R, s, cert, b2));
    SMX_TRY(d2h(sL, n, ev_out[0]));
    // egress: rows [0, sL) (+)= T[rows, L] (x) T[L, :]; L's blocks packed once as B
    for (int j = 0; j < kFwHostTailBlocks; ++j) {
        const int k0 = sL + j * BLK, bb = n - k0 < BLK ? n - k0 : BLK;
        SMX_TRY(packed_pack<T>(nullptr, Tm + (long long)k0 * ld, n, n, bb, ld, ld, kind, egress_slot(j), slot, s));
    }
    for (int c = 0; c < chunks; ++c) {
        const int t0 = cuts[c] / G::BM, tiles = ceil_div(cuts[c + 1], G::BM) - t0;
        for (int j = 0; j < kFwHostTailBlocks; ++j) {
            const int k0 = sL + j * BLK, bb = n - k0 < BLK ? n - k0 : BLK;
            SMX_TRY(packed_pack_a_rows<T>(Tm + k0, n, n, bb, ld, kind, egress_slot(j), slot, t0, tiles, s));
            SMX_TRY(packed_run<T>(Tm, n, n, bb, ld, kind, 1, t0, tiles, 0, 0, egress_slot(j), slot, s));
        }
        SMX_TRY(d2h(cuts[c], cuts[c + 1], ev_out[1 + c]));
    }
    if (egress_staged) SMX_TRY(egress.finish());   // (every row is in host_out)
    if ((e = cudaEventRecord(ev_join, cs->out)) != cudaSuccess) return (int)e;
    e = cudaStreamWaitEvent(s, ev_join, 0);
    if (staged) SMX_TRY(stager.finish());
    return e == cudaSuccess ? SMX_OK : (int)e;
}

// Bulk row-panel updates of the sharded closure take the packed kernel, its
// operand tiles in stream-ordered scratch.
// certify: the sharded closure's first rounds (fw_rounds_packed's certified
// rounds): check A and B for the shifted 1-instruction encoding first.
template <typename T>
static int gemm_skip(const T* A, const T* B, T* C, int M, int N, int K, int lda, int ldb, int ldc, int kind,
                     int skip_row0, int skip_rows, cudaStream_t s, bool certify = false) {
    // the packed path (and its certificate pass, which reads 16-byte
    // vectors at X + r*ld) needs 16-byte aligned bases AND row strides;
    // anything else takes the register-staged GEMM below
    if (g_fw_packed && (long long)M * N >= (1LL << 24) && K > 0 && aligned16(A) && aligned16(B) &&
        aligned16(C) && ld_ok(lda, sizeof(T)) && ld_ok(ldb, sizeof(T)) && ld_ok(ldc, sizeof(T)) &&
        lda >= K && ldb >= N && ldc >= N) {
        const size_t bytes = packed_ws_bytes_t<T>(M, N, K);
        void* ws = nullptr;
        if (scratch_alloc(&ws, bytes + 256, s) == SMX_OK) {
            int* cert = reinterpret_cast<int*>(reinterpret_cast<char*>(ws) + bytes);
            const int* cr = nullptr;
            int rc = SMX_OK;
            if constexpr (!Lane<T>::kOneInstr) {
                if (certify && bounded_fastpath_enabled()) {
                    rc = run_cert<T>(A, M, K, lda, B, K, N, ldb, kind == SMX_ANTI, cert, s);
                    cr = cert;
                }
            }
            if (rc == SMX_OK) rc = packed_pack<T>(A, B, M, N, K, lda, ldb, kind, ws, bytes, s, cr);
            if (rc == SMX_OK)
                rc = packed_run<T>(C, M, N, K, ldc, kind, 1, 0, -1, skip_row0, skip_rows, ws, bytes, s, cr);
            scratch_free(ws, s);
            return rc;
        }
    }
    return semiring_gemm<T>(A, B, C, M, N, K, lda, ldb, ldc, kind, 1, skip_row0, skip_rows, s);
}

}  // namespace smx

using namespace smx;

extern "C" {

int smx_semiring_gemm_u8(const uint8_t* A, const uint8_t* B, uint8_t* C, int M, int N, int K,
                         int lda, int ldb, int ldc, int kind, int accumulate, void* stream) {
    if (g_fw_packed && (long long)M * N >= (1LL << 22) && K >= 256)
        return semiring_gemm_packed_public<uint8_t>(A, B, C, M, N, K, lda, ldb, ldc, kind, accumulate,
                                                    as_stream(stream));
    return semiring_gemm<uint8_t>(A, B, C, M, N, K, lda, ldb, ldc, kind, accumulate, 0, 0,
                                  as_stream(stream));
}
int smx_semiring_gemm_u16(const uint16_t* A, const uint16_t* B, uint16_t* C, int M, int N, int K,
                          int lda, int ldb, int ldc, int kind, int accumulate, void* stream) {
    if (g_fw_packed && (long long)M * N >= (1LL << 22) && K >= 256)
        return semiring_gemm_packed_public_u16(A, B, C, M, N, K, lda, ldb, ldc, kind, accumulate,
                                               as_stream(stream));
    return semiring_gemm<uint16_t>(A, B, C, M, N, K, lda, ldb, ldc, kind, accumulate, 0, 0,
                                   as_stream(stream), /*certify=*/true);
}
int smx_semiring_gemm_u32(const uint32_t* A, const uint32_t* B, uint32_t* C, int M, int N, int K,
                          int lda, int ldb, int ldc, int kind, int accumulate, void* stream) {
    if (g_fw_packed && (long long)M * N >= (1LL << 22) && K >= 256)
        return semiring_gemm_packed_public<uint32_t>(A, B, C, M, N, K, lda, ldb, ldc, kind, accumulate,
                                                     as_stream(stream));
    return semiring_gemm<uint32_t>(A, B, C, M, N, K, lda, ldb, ldc, kind, accumulate, 0, 0,
                                   as_stream(stream), /*certify=*/true);
}

static int gemm_skip_entry(const void* A, const void* B, void* C, int M, int N, int K, int lda, int ldb, int ldc,
                           int elem_bytes, int kind, int skip_row0, int skip_rows, void* stream, bool certify) {
    cudaStream_t s = as_stream(stream);
    switch (elem_bytes) {
        case 1: return gemm_skip<uint8_t>((const uint8_t*)A, (const uint8_t*)B, (uint8_t*)C, M, N, K, lda, ldb,
                                          ldc, kind, skip_row0, skip_rows, s);
        case 2: return gemm_skip<uint16_t>((const uint16_t*)A, (const uint16_t*)B, (uint16_t*)C, M, N, K, lda, ldb,
                                           ldc, kind, skip_row0, skip_rows, s, certify);
        case 4: return gemm_skip<uint32_t>((const uint32_t*)A, (const uint32_t*)B, (uint32_t*)C, M, N, K, lda,
                                           ldb, ldc, kind, skip_row0, skip_rows, s, certify);
        default: return SMX_E_ARG;
    }
}

int smx_semiring_gemm_skip_certified(const void* A, const void* B, void* C, int M, int N, int K, int lda,
                                     int ldb, int ldc, int elem_bytes, int kind, int skip_row0,
                                     int skip_rows, void* stream) {
    return gemm_skip_entry(A, B, C, M, N, K, lda, ldb, ldc, elem_bytes, kind, skip_row0, skip_rows, stream, true);
}

int smx_semiring_gemm_skip(const void* A, const void* B, void* C, int M, int N, int K, int lda,
                           int ldb, int ldc, int elem_bytes, int kind, int skip_row0,
                           int skip_rows, void* stream) {
    return gemm_skip_entry(A, B, C, M, N, K, lda, ldb, ldc, elem_bytes, kind, skip_row0, skip_rows, stream, false);
}

int smx_fw_block_for(int n, int elem_bytes) {
    switch (elem_bytes) {
        case 1: return fw_block_for_n<uint8_t>(n);
        case 2: return fw_block_for_n<uint16_t>(n);
        case 4: return fw_block_for_n<uint32_t>(n);
        default: return SMX_E_ARG;
    }
}

int smx_set_fw_packed(int enable) {
    return g_fw_packed.exchange(enable ? 1 : 0);
}

int smx_set_fw_block(int block) {
    if (block != 0 && block != 128 && block != 256 && block != 512) return SMX_E_ARG;
    return g_fw_block_override.exchange(block);
}

int smx_set_fw_pivot_blocked(int enable) {
    return g_pivot_blocked.exchange(enable ? 1 : 0);
}

int smx_set_fw_panel_buffers(int count) {
    if (count != 1 && count != 2) return SMX_E_ARG;
    return g_fw_panel_buffers.exchange(count);
}
int smx_set_fw_packed_panel(int mode) {
    if (mode < 0 || mode > 2) return SMX_E_ARG;
    return g_fw_packed_panel.exchange(mode);
}
int smx_set_fw_pivot_pairs(int enable) {
    return g_pivot_pairs.exchange(enable != 0);
}
int smx_set_fw_split_3a(int mode) {
    if (mode < 0 || mode > 2) return SMX_E_ARG;
    return g_fw_split_3a.exchange(mode);
}
int smx_set_fw_side_lite(int enable) {
    return g_side_lite.exchange(enable ? 1 : 0);
}

int smx_fw_trace_arm(int max_launches) {
    if (max_launches < 0) return SMX_E_ARG;
    if (max_launches > FwTrace::kCap) max_launches = FwTrace::kCap;
    for (int i = 0; i < 2 * max_launches; ++i) {
        if (!g_trace.ev[i]) {
            cudaError_t e = cudaEventCreate(&g_trace.ev[i]);
            if (e != cudaSuccess) return (int)e;
        }
    }
    g_trace.cap = max_launches;
    g_trace.count = 0;
    g_trace.armed = max_launches > 0;
    return SMX_OK;
}

// Begin / end of every traced launch relative to the first begin (ms), for
// the gaps between phase-3 launches; call before smx_fw_trace_read (which
// disarms the trace).
int smx_fw_trace_offsets(float* begin_ms, float* end_ms, int cap) {
    const int n = g_trace.count < cap ? g_trace.count : cap;
    for (int i = 0; i < n; ++i) {
        cudaError_t e = cudaEventSynchronize(g_trace.ev[2 * i + 1]);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&begin_ms[i], g_trace.ev[0], g_trace.ev[2 * i]);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&end_ms[i], g_trace.ev[0], g_trace.ev[2 * i + 1]);
        if (e != cudaSuccess) return -(int)e;
    }
    return n;
}
int smx_fw_trace_read(float* ms, long long* cells, int cap) {
    g_trace.armed = false;
    const int n = g_trace.count < cap ? g_trace.count : cap;
    for (int i = 0; i < n; ++i) {
        cudaError_t e = cudaEventSynchronize(g_trace.ev[2 * i + 1]);
        if (e != cudaSuccess) return -(int)e;
        e = cudaEventElapsedTime(&ms[i], g_trace.ev[2 * i], g_trace.ev[2 * i + 1]);
        if (e != cudaSuccess) return -(int)e;
        cells[i] = g_trace.cells[i];
    }
    return n;
}

int smx_fw_block(int elem_bytes) {
    return (elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4) ? fw_block_for(elem_bytes) : 0;
}

int smx_fw_pivot(void* P, int b, int ld, int elem_bytes, int kind, void* stream) {
    cudaStream_t s = as_stream(stream);
    switch (elem_bytes) {
        case 1: return fw_pivot<uint8_t>((uint8_t*)P, b, ld, kind, s, nullptr);
        case 2: return fw_pivot<uint16_t>((uint16_t*)P, b, ld, kind, s, nullptr);
        case 4: return fw_pivot<uint32_t>((uint32_t*)P, b, ld, kind, s, nullptr);
        default: return SMX_E_ARG;
    }
}

size_t smx_fw_workspace_bytes(int n, int ld, int elem_bytes) {
    if (n <= 0 || ld < n) return 0;
    return fw_ws_bytes(n, ld, elem_bytes);
}

int smx_fw_u8(uint8_t* T, int n, int ld, int kind, void* ws, size_t ws_bytes, void* stream) {
    return fw_run<uint8_t>(T, n, ld, kind, ws, ws_bytes, as_stream(stream));
}
int smx_fw_u16(uint16_t* T, int n, int ld, int kind, void* ws, size_t ws_bytes, void* stream) {
    return fw_run<uint16_t>(T, n, ld, kind, ws, ws_bytes, as_stream(stream));
}
int smx_fw_u32(uint32_t* T, int n, int ld, int kind, void* ws, size_t ws_bytes, void* stream) {
    return fw_run<uint32_t>(T, n, ld, kind, ws, ws_bytes, as_stream(stream));
}

size_t smx_fw_host_workspace_bytes(int n, int ld, int elem_bytes) {
    if (n <= 0 || ld < n) return 0;
    return fw_host_ws_bytes(n, ld, elem_bytes);
}
int smx_set_fw_host_stream(int mode) {
    if (mode < 0 || mode > 2) return SMX_E_ARG;
    return g_fw_host_stream.exchange(mode);
}
int smx_fw_host_u8(const uint8_t* host_in, uint8_t* host_out, uint8_t* T, int n, int ld, int kind, void* ws,
                   size_t ws_bytes, void* stream) {
    return fw_host_run<uint8_t>(host_in, host_out, T, n, ld, kind, ws, ws_bytes, as_stream(stream));
}
int smx_fw_host_u16(const uint16_t* host_in, uint16_t* host_out, uint16_t* T, int n, int ld, int kind, void* ws,
                    size_t ws_bytes, void* stream) {
    return fw_host_run<uint16_t>(host_in, host_out, T, n, ld, kind, ws, ws_bytes, as_stream(stream));
}
int smx_fw_host_u32(const uint32_t* host_in, uint32_t* host_out, uint32_t* T, int n, int ld, int kind, void* ws,
                    size_t ws_bytes, void* stream) {
    return fw_host_run<uint32_t>(host_in, host_out, T, n, ld, kind, ws, ws_bytes, as_stream(stream));
}

}  // extern "C"
