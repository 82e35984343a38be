// Blocked three-phase Floyd-Warshall over the saturated semirings, plus the
// C-ABI entry points of the lane semiring products.
//
// Replaces _close_vector / _minplus_close_vector
// (pkg/src/semimat/antidist.py:390-398, :440-448).  The reference sweeps k
// one vertex at a time over the whole matrix; here k advances in blocks of
// B = 128 vertices (SURVEY.md 0.1 fact 2 verifies the blocked order is
// bit-identical: x -> min(x, S) is a semiring homomorphism from (min,+) on
// [0, inf] onto the clipped lanes, so every correct closure order agrees):
//
//   round r, pivot block K = [k0, k0 + bb):
//   1. pivot   : close the bb x bb tile T[K,K] in place (one CTA, tile in
//                registers, pivot row/column broadcast through smem).
//   2. row     : T[K,:] (+)= T[K,K]* (x) T[K,:]   (snapshot RP of the panel)
//   3. rest    : T[i,:] (+)= T[i,K] (x) T[K,:] for every i outside K, with
//                T[i,K] read from a snapshot CP of the column panel.  The
//                j in K part of this product is exactly the column-panel
//                update T[i,K] (x) (I (+) T[K,K]*), so phases 2b and 3 fuse
//                into one semiring GEMM over the full row width.
// Phases 2 and 3 are the semiring GEMM of semiring_gemm.cuh.
#include <cuda_runtime.h>

#include "semiring_gemm.cuh"

namespace smx {

constexpr int kFwBlock = 128;

// ---- phase 1: pivot tile closure ------------------------------------------
// 1024 threads, 8 per tile row; each owns 128/8 cells of its row in
// registers.  Step k reads pivot column value T[r,k] and pivot row T[k,:]
// from double-buffered smem (one barrier per step); the owners of row k+1
// and column k+1 publish them for the next step.  During step k row k and
// column k do not change (T[k,k] >= 0 in distance form), so no hazard.
template <typename T>
__global__ void __launch_bounds__(1024, 1)
fw_pivot_kernel(T* P, int b, long long ld, int anti) {
    using L = Lane<T>;
    constexpr int CPW = L::kCellsPerWord;
    constexpr int WPR = kFwBlock / CPW;   // words per tile row
    constexpr int TPR = 8;                // threads per tile row
    constexpr int WPT = WPR / TPR;        // words per thread
    constexpr int CPT = WPT * CPW;        // cells per thread
    __shared__ __align__(16) uint32_t prow[2][WPR];
    __shared__ uint32_t pcol[2][kFwBlock];

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

    for (int k = 0; k < b; ++k) {
        const int cur = k & 1;
        const uint32_t e = pcol[cur][r];
        const uint32_t a = L::splat(e), sa = L::splat(L::kS - e);
        uint32_t rk[WPT];
#pragma unroll
        for (int i = 0; i < WPT; i += 4) {
            const uint4 v = *reinterpret_cast<const uint4*>(&prow[cur][g * WPT + i]);
            rk[i] = v.x; rk[i + 1] = v.y; rk[i + 2] = v.z; rk[i + 3] = v.w;
        }
#pragma unroll
        for (int i = 0; i < WPT; ++i) w[i] = L::step(w[i], rk[i], a, sa);
        const int kn = k + 1;
        if (kn < b) {
            if (r == kn) {
#pragma unroll
                for (int i = 0; i < WPT; ++i) prow[cur ^ 1][g * WPT + i] = w[i];
            }
            if (g == kn / CPT) pcol[cur ^ 1][r] = cell_of(kn - c0);
        }
        __syncthreads();
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

template <typename T>
int fw_pivot(T* P, int b, long long ld, int kind, cudaStream_t s) {
    if (b < 1 || b > kFwBlock || ld < b || (kind != SMX_ANTI && kind != SMX_DIST)) return SMX_E_ARG;
    fw_pivot_kernel<T><<<1, 1024, 0, s>>>(P, b, ld, kind == SMX_ANTI);
    SMX_RETURN_LAUNCH();
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline size_t fw_ws_bytes(int n, long long ld, int eb) {
    // RP: pivot row panel snapshot (B x ld); CP: column panel snapshot (n x B)
    return align256((size_t)kFwBlock * ld * eb) + align256((size_t)n * kFwBlock * eb);
}

template <typename T>
int fw_run(T* Tm, int n, long long ld, int kind, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (n < 0 || ld < n || (kind != SMX_ANTI && kind != SMX_DIST)) return SMX_E_ARG;
    if (n == 0) return SMX_OK;
    if (!aligned16(Tm) || !ld_ok(ld, sizeof(T))) return SMX_E_ALIGN;
    if (n <= kFwBlock) return fw_pivot<T>(Tm, n, ld, kind, s);
    if (ws == nullptr || ws_bytes < fw_ws_bytes(n, ld, sizeof(T))) return SMX_E_WORKSPACE;
    T* RP = reinterpret_cast<T*>(ws);
    T* CP = reinterpret_cast<T*>(reinterpret_cast<char*>(ws) + align256((size_t)kFwBlock * ld * sizeof(T)));
    const long long ldcp = kFwBlock;
    for (int k0 = 0; k0 < n; k0 += kFwBlock) {
        const int bb = n - k0 < kFwBlock ? n - k0 : kFwBlock;
        T* rowK = Tm + (long long)k0 * ld;
        SMX_TRY(fw_pivot<T>(rowK + k0, bb, ld, kind, s));
        cudaError_t e = cudaMemcpyAsync(RP, rowK, (size_t)bb * ld * sizeof(T),
                                        cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return (int)e;
        SMX_TRY(semiring_gemm<T>(RP + k0, RP, rowK, bb, n, bb, ld, ld, ld, kind, 1, 0, 0, s));
        e = cudaMemcpy2DAsync(CP, ldcp * sizeof(T), Tm + k0, ld * sizeof(T), bb * sizeof(T), n,
                              cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return (int)e;
        SMX_TRY(semiring_gemm<T>(CP, rowK, Tm, n, n, bb, ldcp, ld, ld, kind, 1, k0, bb, s));
    }
    return SMX_OK;
}

}  // namespace smx

using namespace smx;

extern "C" {

int smx_semiring_gemm_u8(const uint8_t* A, const uint8_t* B, uint8_t* C, int M, int N, int K,
                         int lda, int ldb, int ldc, int kind, int accumulate, void* stream) {
    return semiring_gemm<uint8_t>(A, B, C, M, N, K, lda, ldb, ldc, kind, accumulate, 0, 0,
                                  as_stream(stream));
}
int smx_semiring_gemm_u16(const uint16_t* A, const uint16_t* B, uint16_t* C, int M, int N, int K,
                          int lda, int ldb, int ldc, int kind, int accumulate, void* stream) {
    return semiring_gemm<uint16_t>(A, B, C, M, N, K, lda, ldb, ldc, kind, accumulate, 0, 0,
                                   as_stream(stream));
}
int smx_semiring_gemm_u32(const uint32_t* A, const uint32_t* B, uint32_t* C, int M, int N, int K,
                          int lda, int ldb, int ldc, int kind, int accumulate, void* stream) {
    return semiring_gemm<uint32_t>(A, B, C, M, N, K, lda, ldb, ldc, kind, accumulate, 0, 0,
                                   as_stream(stream));
}

int smx_semiring_gemm_skip(const void* A, const void* B, void* C, int M, int N, int K, int lda,
                           int ldb, int ldc, int elem_bytes, int kind, int skip_row0,
                           int skip_rows, void* stream) {
    cudaStream_t s = as_stream(stream);
    switch (elem_bytes) {
        case 1: return semiring_gemm<uint8_t>((const uint8_t*)A, (const uint8_t*)B, (uint8_t*)C, M, N,
                                              K, lda, ldb, ldc, kind, 1, skip_row0, skip_rows, s);
        case 2: return semiring_gemm<uint16_t>((const uint16_t*)A, (const uint16_t*)B, (uint16_t*)C, M,
                                               N, K, lda, ldb, ldc, kind, 1, skip_row0, skip_rows, s);
        case 4: return semiring_gemm<uint32_t>((const uint32_t*)A, (const uint32_t*)B, (uint32_t*)C, M,
                                               N, K, lda, ldb, ldc, kind, 1, skip_row0, skip_rows, s);
        default: return SMX_E_ARG;
    }
}

int smx_fw_block(int elem_bytes) { return (elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4) ? kFwBlock : 0; }

int smx_fw_pivot(void* P, int b, int ld, int elem_bytes, int kind, void* stream) {
    cudaStream_t s = as_stream(stream);
    switch (elem_bytes) {
        case 1: return fw_pivot<uint8_t>((uint8_t*)P, b, ld, kind, s);
        case 2: return fw_pivot<uint16_t>((uint16_t*)P, b, ld, kind, s);
        case 4: return fw_pivot<uint32_t>((uint32_t*)P, b, ld, kind, s);
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

}  // extern "C"
