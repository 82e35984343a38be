// Boolean products and Warshall closure on bit-packed rows, plus the
// byte <-> bit layout helpers.
//
// Storage is the reference's own: bit j of row i at u64 block j>>6, bit j&63,
// LSB first (pkg/src/semimat/boolmat.py:3-5), which read as little-endian u32
// words is word j>>5, bit j&31.  The product replaces BoolMatrix.__mul__
// (boolmat.py:151-172, "row k of B is OR-ed into every row whose (i,k) bit is
// set"), the closure replaces transitive_closure (:174-189) with the same
// blocked three-phase schedule as fw.cu (B = 256 vertices per round).
//
// Inner loop: for each k the CTA's A bit (i,k) is tested once per row
// (LOP3 -> predicate) and row k of B is OR-ed in 32 cells per instruction --
// the paper's matBool.h inner loop with 32-bit words, 32 lanes
// per warp.
#include <cuda_runtime.h>

#include "common.cuh"

namespace smx {

struct BitsArgs {
    const uint32_t* A;
    const uint32_t* B;
    uint32_t* C;
    int M, Nw, K;
    long long lda, ldb, ldc;   // in words
    int accumulate;
    int skip_tile0, skip_tiles;
};

constexpr int kBitsBM = 128, kBitsBNW = 64, kBitsTM = 4, kBitsTNW = 8;
constexpr int kBitsThreads = (kBitsBM / kBitsTM) * (kBitsBNW / kBitsTNW);  // 256

__global__ void __launch_bounds__(kBitsThreads, 2) bool_bits_gemm_kernel(const BitsArgs p) {
    constexpr int BM = kBitsBM, BNW = kBitsBNW, TM = kBitsTM, TNW = kBitsTNW, HW = TNW / 2;
    constexpr int TCOLS = BNW / TNW;
    __shared__ uint32_t As[2][BM];            // one A word (32 k) per row
    __shared__ __align__(16) uint32_t Bs[2][32][BNW];

    const int tid = threadIdx.x;
    int mt = blockIdx.y;
    if (mt >= p.skip_tile0) mt += p.skip_tiles;
    const int row0 = mt * BM, w0 = blockIdx.x * BNW;
    const int tc = tid % TCOLS, tr = tid / TCOLS;

    uint32_t acc[TM][TNW];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int grow = row0 + tr * TM + i;
#pragma unroll
        for (int j = 0; j < TNW; ++j) {
            const int gw = w0 + (j / HW) * (BNW / 2) + tc * HW + (j % HW);
            acc[i][j] = (p.accumulate && grow < p.M && gw < p.Nw) ? p.C[(long long)grow * p.ldc + gw] : 0u;
        }
    }

    // staging: A: BM words (first BM threads); B: 32 x BNW words = 512 uint4
    uint32_t a_st = 0;
    uint4 b_st[2];
    auto gload = [&](int kw) {  // kw: k-word index
        const int k0 = kw * 32;
        if (tid < BM) {
            const int grow = row0 + tid;
            uint32_t v = 0;
            if (grow < p.M) {
                v = p.A[(long long)grow * p.lda + kw];
                const int valid = p.K - k0;
                if (valid < 32) v &= (1u << valid) - 1u;
            }
            a_st = v;
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int c = tid + q * kBitsThreads;     // 0..511
            const int kr = c / (BNW / 4), wc = (c % (BNW / 4)) * 4;
            const int gk = k0 + kr, gw = w0 + wc;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (gk < p.K) {
                const uint32_t* src = p.B + (long long)gk * p.ldb + gw;
                if (gw + 4 <= p.Nw) v = *reinterpret_cast<const uint4*>(src);
                else {
                    if (gw + 0 < p.Nw) v.x = src[0];
                    if (gw + 1 < p.Nw) v.y = src[1];
                    if (gw + 2 < p.Nw) v.z = src[2];
                }
            }
            b_st[q] = v;
        }
    };
    auto sstore = [&](int buf) {
        if (tid < BM) As[buf][tid] = a_st;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int c = tid + q * kBitsThreads;
            const int kr = c / (BNW / 4), wc = (c % (BNW / 4)) * 4;
            *reinterpret_cast<uint4*>(&Bs[buf][kr][wc]) = b_st[q];
        }
    };

    const int nkw = (p.K + 31) / 32;
    if (nkw > 0) { gload(0); sstore(0); __syncthreads(); }
    for (int kw = 0; kw < nkw; ++kw) {
        const int buf = kw & 1;
        if (kw + 1 < nkw) gload(kw + 1);
        uint32_t aw[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i) aw[i] = As[buf][tr * TM + i];
#pragma unroll
        for (int kk = 0; kk < 32; ++kk) {
            uint32_t b[TNW];
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                const uint4 v = *reinterpret_cast<const uint4*>(&Bs[buf][kk][g * (BNW / 2) + tc * HW]);
                b[g * 4 + 0] = v.x; b[g * 4 + 1] = v.y; b[g * 4 + 2] = v.z; b[g * 4 + 3] = v.w;
            }
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                if (aw[i] & (1u << kk)) {
#pragma unroll
                    for (int j = 0; j < TNW; ++j) acc[i][j] |= b[j];
                }
            }
        }
        if (kw + 1 < nkw) sstore(buf ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int grow = row0 + tr * TM + i;
        if (grow >= p.M) continue;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const int gw = w0 + g * (BNW / 2) + tc * HW;
            uint32_t* dst = p.C + (long long)grow * p.ldc + gw;
            if (gw + 4 <= p.Nw) {
                *reinterpret_cast<uint4*>(dst) = make_uint4(acc[i][g * 4], acc[i][g * 4 + 1],
                                                            acc[i][g * 4 + 2], acc[i][g * 4 + 3]);
            } else {
                for (int j = 0; j < 4; ++j)
                    if (gw + j < p.Nw) dst[j] = acc[i][g * 4 + j];
            }
        }
    }
}

int bool_bits_gemm(const uint32_t* A, const uint32_t* B, uint32_t* C, int M, int Nw, int K,
                   long long lda, long long ldb, long long ldc, int accumulate, int skip_row0,
                   int skip_rows, cudaStream_t s) {
    if (M < 0 || Nw < 0 || K < 0) return SMX_E_ARG;
    if (M == 0 || Nw == 0) return SMX_OK;
    if (!aligned16(A) || !aligned16(B) || !aligned16(C)) return SMX_E_ALIGN;
    if ((ldb & 3) || (ldc & 3)) return SMX_E_ALIGN;
    if (lda * 32 < K || ldb < Nw || ldc < Nw) return SMX_E_ARG;
    BitsArgs a{A, B, C, M, Nw, K, lda, ldb, ldc, accumulate != 0, 0, 0};
    if (skip_rows > 0) {
        if (skip_row0 % kBitsBM) return SMX_E_ARG;
        a.skip_tile0 = skip_row0 / kBitsBM;
        a.skip_tiles = ceil_div(skip_rows, kBitsBM);
        const int total = ceil_div(M, kBitsBM);
        if (a.skip_tile0 + a.skip_tiles > total) a.skip_tiles = total - a.skip_tile0;
    }
    const int mtiles = ceil_div(M, kBitsBM) - a.skip_tiles;
    if (mtiles <= 0) return SMX_OK;
    dim3 grid(ceil_div(Nw, kBitsBNW), mtiles);
    bool_bits_gemm_kernel<<<grid, kBitsThreads, 0, s>>>(a);
    SMX_RETURN_LAUNCH();
}

// ---- Warshall pivot tile on bits ------------------------------------------
// b <= 256: one thread per tile row, the row (8 words) in registers.  Step k:
// row k (as it stood after step k-1) comes from double-buffered smem; a row
// whose bit k is set ORs it in (boolmat.py:184-188).
constexpr int kWarshallBlock = 256;

__global__ void __launch_bounds__(kWarshallBlock, 1)
bool_pivot_kernel(uint32_t* P, int b, long long ld_w) {
    constexpr int W = kWarshallBlock / 32;
    __shared__ __align__(16) uint32_t prow[2][W];
    const int r = threadIdx.x;
    const int nw = (b + 31) / 32;
    uint32_t w[W];
#pragma unroll
    for (int i = 0; i < W; ++i) {
        uint32_t v = 0;
        if (r < b && i < nw) {
            v = P[(long long)r * ld_w + i];
            const int valid = b - i * 32;
            if (valid < 32) v &= (1u << valid) - 1u;
        }
        w[i] = v;
    }
    if (r == 0) {
#pragma unroll
        for (int i = 0; i < W; ++i) prow[0][i] = w[i];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < W; ++q) {
        if (q * 32 >= b) break;
        for (int kk = 0; kk < 32; ++kk) {
            const int k = q * 32 + kk;
            if (k >= b) break;
            const int cur = k & 1;
            if ((w[q] >> kk) & 1u) {
                const uint4 v0 = *reinterpret_cast<const uint4*>(&prow[cur][0]);
                const uint4 v1 = *reinterpret_cast<const uint4*>(&prow[cur][4]);
                w[0] |= v0.x; w[1] |= v0.y; w[2] |= v0.z; w[3] |= v0.w;
                w[4] |= v1.x; w[5] |= v1.y; w[6] |= v1.z; w[7] |= v1.w;
            }
            if (r == k + 1) {
#pragma unroll
                for (int i = 0; i < W; ++i) prow[cur ^ 1][i] = w[i];
            }
            __syncthreads();
        }
    }
    if (r < b) {
        for (int i = 0; i < nw; ++i) {
            const int valid = b - i * 32;
            uint32_t* dst = P + (long long)r * ld_w + i;
            if (valid >= 32) *dst = w[i];
            else {
                const uint32_t m = (1u << valid) - 1u;
                *dst = (*dst & ~m) | (w[i] & m);
            }
        }
    }
}

// Warshall pivot tiles are aligned to kWarshallBlock = 256 bits = 8 words.
inline size_t bits_ws_bytes(int n, long long ld_w) {
    const size_t rp = ((size_t)kWarshallBlock * ld_w * 4 + 255) & ~size_t(255);
    const size_t cp = (size_t)n * (kWarshallBlock / 32) * 4;
    return rp + ((cp + 255) & ~size_t(255));
}

int bool_warshall_bits(uint32_t* T, int n, long long ld_w, void* ws, size_t ws_bytes,
                       cudaStream_t s) {
    if (n < 0 || ld_w * 32 < n) return SMX_E_ARG;
    if (n == 0) return SMX_OK;
    if (!aligned16(T) || (ld_w & 3)) return SMX_E_ALIGN;
    const int nw = (n + 31) / 32;
    if (n <= kWarshallBlock) {
        bool_pivot_kernel<<<1, kWarshallBlock, 0, s>>>(T, n, ld_w);
        SMX_RETURN_LAUNCH();
    }
    if (ws == nullptr || ws_bytes < bits_ws_bytes(n, ld_w)) return SMX_E_WORKSPACE;
    uint32_t* RP = reinterpret_cast<uint32_t*>(ws);
    uint32_t* CP = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(ws) +
                                               (((size_t)kWarshallBlock * ld_w * 4 + 255) & ~size_t(255)));
    constexpr long long ldcp = kWarshallBlock / 32;
    for (int k0 = 0; k0 < n; k0 += kWarshallBlock) {
        const int bb = n - k0 < kWarshallBlock ? n - k0 : kWarshallBlock;
        const int kw0 = k0 / 32, bw = (bb + 31) / 32;
        uint32_t* rowK = T + (long long)k0 * ld_w;
        bool_pivot_kernel<<<1, kWarshallBlock, 0, s>>>(rowK + kw0, bb, ld_w);
        SMX_LAUNCHED_OR_RETURN();
        cudaError_t e = cudaMemcpyAsync(RP, rowK, (size_t)bb * ld_w * 4, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return (int)e;
        SMX_TRY(bool_bits_gemm(RP + kw0, RP, rowK, bb, nw, bb, ld_w, ld_w, ld_w, 1, 0, 0, s));
        e = cudaMemcpy2DAsync(CP, ldcp * 4, T + kw0, ld_w * 4, (size_t)bw * 4, n,
                              cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return (int)e;
        SMX_TRY(bool_bits_gemm(CP, rowK, T, n, nw, bb, ldcp, ld_w, ld_w, 1, k0, bb, s));
    }
    return SMX_OK;
}

// ---- layout helpers ---------------------------------------------------------
// pack: one warp per 32-column group of a row; lane l tests byte (r, 32g + l)
// and a ballot forms the LSB-first word (bit l = column 32g + l).
__global__ void pack_bits_kernel(const uint8_t* __restrict__ bytes, uint32_t* __restrict__ words,
                                 int rows, int cols, long long ld, long long ld_w, int nw_out) {
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long total = (long long)rows * nw_out;
    if (warp >= total) return;
    const int r = (int)(warp / nw_out), wi = (int)(warp % nw_out);
    const int c = wi * 32 + lane;
    const bool bit = c < cols && bytes[(long long)r * ld + c] != 0;
    const uint32_t word = __ballot_sync(0xFFFFFFFFu, bit);
    if (lane == 0) words[(long long)r * ld_w + wi] = word;
}

// unpack: one thread per (row, word) writes 32 bytes; 4 bits -> 4 bytes with
// the multiply-spread (x * 0x204081) & 0x01010101.
__global__ void unpack_bits_kernel(const uint32_t* __restrict__ words, uint8_t* __restrict__ bytes,
                                   int rows, int cols, long long ld_w, long long ld) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int nw = (cols + 31) / 32;
    if (t >= (long long)rows * nw) return;
    const int r = (int)(t / nw), wi = (int)(t % nw);
    const uint32_t w = words[(long long)r * ld_w + wi];
    uint32_t o[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = (((w >> (4 * q)) & 0xFu) * 0x00204081u) & 0x01010101u;
    uint8_t* dst = bytes + (long long)r * ld + wi * 32;
    const int valid = cols - wi * 32;
    if (valid >= 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        reinterpret_cast<uint4*>(dst)[0] = make_uint4(o[0], o[1], o[2], o[3]);
        reinterpret_cast<uint4*>(dst)[1] = make_uint4(o[4], o[5], o[6], o[7]);
    } else {
        const uint8_t* ob = reinterpret_cast<const uint8_t*>(o);
        for (int c = 0; c < 32 && c < valid; ++c) dst[c] = ob[c];
    }
}

__global__ void transpose_u8_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                    int rows, int cols, long long ld_in, long long ld_out) {
    __shared__ uint8_t tile[64][65];
    const int bx = blockIdx.x * 64, by = blockIdx.y * 64;
    for (int i = threadIdx.y; i < 64; i += blockDim.y) {
        const int r = by + i, c = bx + threadIdx.x;
        tile[i][threadIdx.x] = (r < rows && c < cols) ? in[(long long)r * ld_in + c] : 0;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 64; i += blockDim.y) {
        const int r = bx + i, c = by + threadIdx.x;   // out row = in col
        if (r < cols && c < rows) out[(long long)r * ld_out + c] = tile[threadIdx.x][i];
    }
}

int transpose_bytes(const uint8_t* in, uint8_t* out, int rows, int cols, long long ld_in, long long ld_out,
                    cudaStream_t s) {
    if (rows < 0 || cols < 0 || ld_in < cols || ld_out < rows) return SMX_E_ARG;
    if (rows == 0 || cols == 0) return SMX_OK;
    dim3 grid(ceil_div(cols, 64), ceil_div(rows, 64));
    transpose_u8_kernel<<<grid, dim3(64, 8), 0, s>>>(in, out, rows, cols, ld_in, ld_out);
    SMX_RETURN_LAUNCH();
}

}  // namespace smx

using namespace smx;

extern "C" {

int smx_bool_gemm_bits(const uint32_t* A, const uint32_t* B, uint32_t* C, int M, int Nwords, int K,
                       int lda_w, int ldb_w, int ldc_w, int accumulate, void* stream) {
    return bool_bits_gemm(A, B, C, M, Nwords, K, lda_w, ldb_w, ldc_w, accumulate, 0, 0,
                          as_stream(stream));
}

size_t smx_bool_warshall_workspace_bytes(int n, int ld_w) {
    if (n <= 0 || (long long)ld_w * 32 < n) return 0;
    return bits_ws_bytes(n, ld_w);
}

int smx_bool_warshall_bits(uint32_t* T, int n, int ld_w, void* ws, size_t ws_bytes, void* stream) {
    if (ws_bytes < bits_ws_bytes(n, ld_w)) return SMX_E_WORKSPACE;
    return bool_warshall_bits(T, n, ld_w, ws, ws_bytes, as_stream(stream));
}

int smx_pack_bits(const uint8_t* bytes, uint32_t* words, int rows, int cols, int ld, int ld_w,
                  void* stream) {
    if (rows < 0 || cols < 0 || ld < cols || (long long)ld_w * 32 < cols) return SMX_E_ARG;
    if (rows == 0) return SMX_OK;
    // write every word of the row stride so pad bits are zero
    const int nw_out = ld_w;
    const long long warps = (long long)rows * nw_out;
    const int threads = 256;
    const long long blocks = (warps * 32 + threads - 1) / threads;
    pack_bits_kernel<<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(bytes, words, rows, cols, ld,
                                                                        ld_w, nw_out);
    SMX_RETURN_LAUNCH();
}

int smx_unpack_bits(const uint32_t* words, uint8_t* bytes, int rows, int cols, int ld_w, int ld,
                    void* stream) {
    if (rows < 0 || cols < 0 || ld < cols || (long long)ld_w * 32 < cols) return SMX_E_ARG;
    if (rows == 0 || cols == 0) return SMX_OK;
    const long long t = (long long)rows * ((cols + 31) / 32);
    unpack_bits_kernel<<<(unsigned)((t + 255) / 256), 256, 0, as_stream(stream)>>>(words, bytes, rows,
                                                                                 cols, ld_w, ld);
    SMX_RETURN_LAUNCH();
}

int smx_transpose_u8(const uint8_t* in, uint8_t* out, int rows, int cols, int ld_in, int ld_out,
                     void* stream) {
    return transpose_bytes(in, out, rows, cols, ld_in, ld_out, as_stream(stream));
}

}  // extern "C"
