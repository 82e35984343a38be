// Lane kernels, the Boolean bridge and batched small-matrix products/closures.
//
// 1. The paper's 128-bit block primitives, re-expressed by
//    the reference as list-in/list-out functions (pkg/src/semimat/
//    kernels.py:129-189): clonenot, subsat, addsat, maxlanes, minlanes,
//    absdiff.  Here they run over a flat device array of lanes, 16 bytes (one
//    block) per thread step, on the same packed u16x2 instructions as the
//    semiring GEMM (semiring.cuh): u8 lanes are widened into u16x2 words
//    (PRMT), because sm_100 has no native byte-SIMD min/max/add.
//      subsat  max(a, b) - b           kernels.py:147-152 (np_subsat :195-196)
//      addsat  min(a, S - b) + b       kernels.py:155-161 (np_addsat :199-200)
//      max/min lanewise                kernels.py:164-177
//      absdiff (a -sat b) | (b -sat a) kernels.py:180-189 (np_absdiff :203-204)
//      clonenot S - a (bitwise NOT)    kernels.py:129-144
//
// 2. The Boolean bridge (antidist.py:213-224): AntidistMatrix.from_boolmat
//    (1 -> S = distance zero, 0 -> 0 = unreachable, padding 0) and
//    to_boolmat (any lane > 0 -> 1, padding bits 0), directly between the
//    packed bit rows and the lane rows in HBM.
//
// 3. Batched closures and products of many small matrices (one launch for a
//    whole batch): the reference's acceptance suite runs 262,144 3x3 Boolean
//    products and thousands of <= 64-vertex closures
//    (pkg/tests/test_acceptance.py:28-116); one launch per matrix would be
//    launch-bound by three orders of magnitude.
//      Boolean product : one thread per (matrix, row, output word):
//                        C[i] = OR over set bits k of A[i] of B[k]
//                        (boolmat.py:151-172, row-outer order, exact).
//      Boolean closure : n <= 32: one warp per matrix, row i in lane i, row k
//                        broadcast by shuffle; n <= 512: one CTA per matrix,
//                        rows in shared memory (boolmat.py:174-189).
//      Lane FW         : one CTA per matrix (n <= 128), the whole matrix in
//                        shared memory as 32-bit distance-form cells, the
//                        reference's k-sweep with one barrier per k
//                        (antidist.py:390-398, :440-448).  Row and column k
//                        do not change during step k,
//                        so the sweep runs in place.
#include <cuda_runtime.h>

#include "common.cuh"

namespace smx {

enum { LOP_SUBSAT = 0, LOP_ADDSAT = 1, LOP_MAX = 2, LOP_MIN = 3, LOP_ABSDIFF = 4, LOP_CLONENOT = 5 };

// u16x2 words (also the widened form of u8 lanes); S = all-ones lane of the
// width (0x00FF for widened u8, 0xFFFF for u16)
__device__ __forceinline__ uint32_t op_u16x2(uint32_t a, uint32_t b, int op, uint32_t S2) {
    switch (op) {
        case LOP_SUBSAT: return __vsub2(__vmaxu2(a, b), b);               // no wrap: max(a,b) >= b
        case LOP_ADDSAT: return __vadd2(__vminu2(a, S2 - b), b);          // no wrap: <= S
        case LOP_MAX: return __vmaxu2(a, b);
        case LOP_MIN: return __vminu2(a, b);
        case LOP_ABSDIFF: return __vsub2(__vmaxu2(a, b), b) | __vsub2(__vmaxu2(b, a), a);
        default: return S2 - a;                                            // lanes <= S: no borrow
    }
}

__device__ __forceinline__ uint32_t op_u32(uint32_t a, uint32_t b, int op) {
    switch (op) {
        case LOP_SUBSAT: return max(a, b) - b;
        case LOP_ADDSAT: return min(a, 0xFFFFFFFFu - b) + b;
        case LOP_MAX: return max(a, b);
        case LOP_MIN: return min(a, b);
        case LOP_ABSDIFF: return (max(a, b) - b) | (max(b, a) - a);
        default: return ~a;
    }
}

template <int EB>
__global__ void lane_op_kernel(const uint4* __restrict__ A, const uint4* __restrict__ B, uint4* __restrict__ C,
                               long long nblocks, int op) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nblocks;
         i += (long long)gridDim.x * blockDim.x) {
        const uint4 a = A[i];
        const uint4 b = op == LOP_CLONENOT ? a : B[i];
        const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
        uint32_t cv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (EB == 1) {
                // widen 4 bytes into two u16x2 words, operate, narrow
                const uint32_t a0 = __byte_perm(av[q], 0u, 0x4140), a1 = __byte_perm(av[q], 0u, 0x4342);
                const uint32_t b0 = __byte_perm(bv[q], 0u, 0x4140), b1 = __byte_perm(bv[q], 0u, 0x4342);
                const uint32_t c0 = op_u16x2(a0, b0, op, 0x00FF00FFu), c1 = op_u16x2(a1, b1, op, 0x00FF00FFu);
                cv[q] = __byte_perm(c0, c1, 0x6420);
            } else if (EB == 2) {
                cv[q] = op_u16x2(av[q], bv[q], op, 0xFFFFFFFFu);
            } else {
                cv[q] = op_u32(av[q], bv[q], op);
            }
        }
        C[i] = make_uint4(cv[0], cv[1], cv[2], cv[3]);
    }
}

inline unsigned grid_1d(long long n, int threads = 256) {
    long long g = (n + threads - 1) / threads;
    const long long cap = (long long)sm_count() * 16;
    if (g > cap) g = cap;
    return (unsigned)(g < 1 ? 1 : g);
}

// ---- Boolean bridge ------------------------------------------------------------

// from_boolmat: lane (r, c) = S if bit c of row r is set (c < cols), else 0;
// padding lanes [cols, ld) = 0 (the anti-distance (+)-identity).  One
// 16-byte chunk of E = 16 / sizeof(T) lanes per thread-iteration: its E bits
// sit in one word (E divides 32), spread to lanes of all-ones / zero.  Rows
// are walked incrementally (no per-chunk division).  HBM-bound.
template <typename T>
__device__ __forceinline__ uint4 spread_bits(uint32_t bits) {
    constexpr int E = 16 / sizeof(T);
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if constexpr (sizeof(T) == 1) {   // 4 bits -> 4 bytes of 0x00 / 0xFF
            const uint32_t nib = (bits >> (4 * q)) & 0xFu;
            w[q] = ((nib * 0x00204081u) & 0x01010101u) * 0xFFu;
        } else if constexpr (sizeof(T) == 2) {   // 2 bits -> 2 halves
            const uint32_t two = (bits >> (2 * q)) & 3u;
            w[q] = ((two & 1u) ? 0xFFFFu : 0u) | ((two & 2u) ? 0xFFFF0000u : 0u);
        } else {
            w[q] = ((bits >> q) & 1u) ? 0xFFFFFFFFu : 0u;
        }
    }
    (void)E;
    return make_uint4(w[0], w[1], w[2], w[3]);
}

template <typename T>
__global__ void __launch_bounds__(256) lanes_from_bits_kernel(const uint32_t* __restrict__ words, long long ld_w,
                                                              uint4* __restrict__ out, int rows, int cols, int cpr) {
    constexpr int E = 16 / sizeof(T);
    const long long total = (long long)rows * cpr;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    long long r = i / cpr;
    int c = (int)(i - r * cpr);
    const long long dr = stride / cpr;
    const int dc = (int)(stride - dr * cpr);
    for (; i < total; i += stride) {
        const int col0 = c * E;
        uint32_t bits = 0;
        if (col0 < cols) {
            bits = (__ldg(words + r * ld_w + (col0 >> 5)) >> (col0 & 31)) & ((1u << E) - 1u);   // (E <= 16)
            const int valid = cols - col0;
            if (valid < E) bits &= (1u << valid) - 1u;
        }
        out[i] = spread_bits<T>(bits);
        c += dc;
        r += dr;
        if (c >= cpr) { c -= cpr; ++r; }
    }
}

// to_boolmat: bit c of row r = (lane (r, c) > 0) for c < cols; every other
// bit of the row's ld_w words is 0.  One output word (32 lanes: 32 / 64 / 128
// bytes of 16-byte loads) per thread-iteration.  HBM-bound.
template <typename T>
__device__ __forceinline__ uint32_t nonzero_bits16(uint4 v) {   // one 16-byte chunk -> 16 / sizeof(T) bits
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t out = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if constexpr (sizeof(T) == 1) {
            const uint32_t nz = __vcmpne4(w[q], 0u);   // 0xFF per nonzero byte
            out |= ((nz & 0x01u) | ((nz >> 7) & 0x02u) | ((nz >> 14) & 0x04u) | ((nz >> 21) & 0x08u)) << (4 * q);
        } else if constexpr (sizeof(T) == 2) {
            const uint32_t nz = __vcmpne2(w[q], 0u);
            out |= ((nz & 0x1u) | ((nz >> 15) & 0x2u)) << (2 * q);
        } else {
            out |= (w[q] != 0u ? 1u : 0u) << q;
        }
    }
    return out;
}

template <typename T>
__global__ void __launch_bounds__(256) lanes_to_bits_kernel(const T* __restrict__ in, long long ld,
                                                            uint32_t* __restrict__ words, long long ld_w, int rows,
                                                            int cols) {
    constexpr int E = 16 / sizeof(T), CH = 32 / E;   // chunks per output word
    const long long total = (long long)rows * ld_w;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    long long r = i / ld_w;
    int w = (int)(i - r * ld_w);
    const long long dr = stride / ld_w;
    const int dw = (int)(stride - dr * ld_w);
    for (; i < total; i += stride) {
        const int col0 = w * 32;
        uint32_t word = 0;
        if (col0 < cols) {
            const uint4* src = reinterpret_cast<const uint4*>(in + r * ld + col0);
            const int nch = min(CH, (cols - col0 + E - 1) / E);   // (ld is whole chunks: reads stay in the row)
#pragma unroll
            for (int q = 0; q < CH; ++q)
                if (q < nch) word |= nonzero_bits16<T>(__ldg(src + q)) << (q * E);
            const int valid = cols - col0;
            if (valid < 32) word &= (1u << valid) - 1u;
        }
        words[i] = word;
        w += dw;
        r += dr;
        if (w >= ld_w) { w -= (int)ld_w; ++r; }
    }
}

// ---- batched Boolean products and closures -------------------------------------

__global__ void bool_mul_batched_kernel(const uint32_t* __restrict__ A, const uint32_t* __restrict__ B,
                                        uint32_t* __restrict__ C, int batch, int M, int K, int nw_out,
                                        int ld_a, int ld_b, int ld_c, long long sa, long long sb, long long sc) {
    const long long total = (long long)batch * M * ld_c;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(t % ld_c);
        const long long ri = t / ld_c;
        const int i = (int)(ri % M);
        const long long m = ri / M;
        uint32_t acc = 0;
        if (w < nw_out) {
            const uint32_t* arow = A + m * sa + (long long)i * ld_a;
            const uint32_t* bm = B + m * sb + w;
            for (int kw = 0; kw * 32 < K; ++kw) {
                uint32_t bits = arow[kw];
                if (K - kw * 32 < 32) bits &= (1u << (K - kw * 32)) - 1u;
                while (bits) {
                    const int k = kw * 32 + __ffs(bits) - 1;
                    bits &= bits - 1;
                    acc |= bm[(long long)k * ld_b];
                }
            }
        }
        C[m * sc + (long long)i * ld_c + w] = acc;   // padding words come out 0
    }
}

// n <= 32: warp per matrix; row i of matrix m held by lane i
__global__ void bool_close_batched_warp_kernel(uint32_t* __restrict__ T, int batch, int n, int ld_w,
                                               long long st) {
    const int lane = threadIdx.x & 31;
    const long long m = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (m >= batch) return;
    uint32_t* base = T + m * st;
    uint32_t row = lane < n ? base[(long long)lane * ld_w] : 0u;
    for (int k = 0; k < n; ++k) {
        const uint32_t rk = __shfl_sync(0xFFFFFFFFu, row, k);
        if ((row >> k) & 1u) row |= rk;
    }
    if (lane < n) base[(long long)lane * ld_w] = row;
}

// n <= 512: CTA per matrix, rows in shared memory (n x W words, W = ld_w)
__global__ void bool_close_batched_cta_kernel(uint32_t* __restrict__ T, int batch, int n, int ld_w,
                                              long long st) {
    extern __shared__ uint32_t srow[];
    uint32_t* base = T + (long long)blockIdx.x * st;
    const int W = (n + 31) / 32;
    for (int x = threadIdx.x; x < n * W; x += blockDim.x) srow[x] = base[(long long)(x / W) * ld_w + x % W];
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        // every (row i != k, word) pair with bit k of row i set ORs in row k
        // (row k itself is unchanged at step k: OR with itself)
        for (int x = threadIdx.x; x < n * W; x += blockDim.x) {
            const int i = x / W, w = x - i * W;
            if (i != k && ((srow[i * W + (k >> 5)] >> (k & 31)) & 1u)) srow[x] |= srow[k * W + w];
        }
        __syncthreads();
    }
    for (int x = threadIdx.x; x < n * W; x += blockDim.x) base[(long long)(x / W) * ld_w + x % W] = srow[x];
}

// ---- batched lane Floyd-Warshall ------------------------------------------------
//
// Cells are held in distance form (anti: S - a, i.e. bitwise NOT), one 32-bit
// word each; the update d[i][j] = min(d[i][j], min(d[i][k] + d[k][j], S)) is
// t = min(d[k][j], S - d[i][k]) + d[i][k] (no wrap: the np_addsat rewrite).
template <typename T>
__global__ void fw_batched_kernel(T* __restrict__ Tm, int batch, int n, long long ld, long long st, int anti) {
    extern __shared__ uint32_t d[];
    constexpr uint32_t S = Limit<T>::value;
    T* base = Tm + (long long)blockIdx.x * st;
    const int cells = n * n;
    for (int x = threadIdx.x; x < cells; x += blockDim.x) {
        const uint32_t v = base[(long long)(x / n) * ld + x % n];
        d[x] = anti ? S - v : v;
    }
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        for (int x = threadIdx.x; x < cells; x += blockDim.x) {
            const int i = x / n, j = x - i * n;
            const uint32_t e = d[i * n + k];
            const uint32_t t = min(d[k * n + j], S - e) + e;
            if (t < d[x]) d[x] = t;
        }
        __syncthreads();
    }
    for (int x = threadIdx.x; x < cells; x += blockDim.x) {
        const uint32_t v = d[x];
        base[(long long)(x / n) * ld + x % n] = (T)(anti ? S - v : v);
    }
}

}  // namespace smx

using namespace smx;

extern "C" {

int smx_lane_op(const void* A, const void* B, void* C, long long nlanes, int elem_bytes, int op,
                void* stream) {
    if (nlanes < 0 || op < LOP_SUBSAT || op > LOP_CLONENOT) return SMX_E_ARG;
    if (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4) return SMX_E_ARG;
    if ((nlanes * elem_bytes) % 16) return SMX_E_ARG;    // whole 128-bit blocks
    if (nlanes == 0) return SMX_OK;
    if (!aligned16(A) || !aligned16(C) || (op != LOP_CLONENOT && !aligned16(B))) return SMX_E_ALIGN;
    const long long nb = nlanes * elem_bytes / 16;
    cudaStream_t s = as_stream(stream);
    const uint4* a = static_cast<const uint4*>(A);
    const uint4* b = static_cast<const uint4*>(op == LOP_CLONENOT ? A : B);
    uint4* c = static_cast<uint4*>(C);
    switch (elem_bytes) {
        case 1: lane_op_kernel<1><<<grid_1d(nb), 256, 0, s>>>(a, b, c, nb, op); break;
        case 2: lane_op_kernel<2><<<grid_1d(nb), 256, 0, s>>>(a, b, c, nb, op); break;
        default: lane_op_kernel<4><<<grid_1d(nb), 256, 0, s>>>(a, b, c, nb, op); break;
    }
    SMX_RETURN_LAUNCH();
}

int smx_lanes_from_bits(const uint32_t* words, int ld_w, void* out, int rows, int cols, int ld, int elem_bytes,
                        void* stream) {
    if (rows < 0 || cols < 0 || ld < cols || (long long)ld_w * 32 < cols) return SMX_E_ARG;
    if (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4) return SMX_E_ARG;
    if (rows == 0 || ld == 0) return SMX_OK;
    if (((long long)ld * elem_bytes) % 16 != 0) return SMX_E_ARG;   // whole 128-bit lane blocks
    if (!aligned16(out)) return SMX_E_ALIGN;
    const int cpr = (int)((long long)ld * elem_bytes / 16);
    const long long total = (long long)rows * cpr;
    cudaStream_t s = as_stream(stream);
    uint4* o = static_cast<uint4*>(out);
    switch (elem_bytes) {
        case 1: lanes_from_bits_kernel<uint8_t><<<grid_1d(total), 256, 0, s>>>(words, ld_w, o, rows, cols, cpr); break;
        case 2: lanes_from_bits_kernel<uint16_t><<<grid_1d(total), 256, 0, s>>>(words, ld_w, o, rows, cols, cpr); break;
        default: lanes_from_bits_kernel<uint32_t><<<grid_1d(total), 256, 0, s>>>(words, ld_w, o, rows, cols, cpr); break;
    }
    SMX_RETURN_LAUNCH();
}

int smx_lanes_to_bits(const void* in, int ld, uint32_t* words, int ld_w, int rows, int cols, int elem_bytes,
                      void* stream) {
    if (rows < 0 || cols < 0 || ld < cols || (long long)ld_w * 32 < cols) return SMX_E_ARG;
    if (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4) return SMX_E_ARG;
    if (rows == 0 || ld_w == 0) return SMX_OK;
    if (((long long)ld * elem_bytes) % 16 != 0) return SMX_E_ARG;   // whole 128-bit lane blocks
    if (!aligned16(in)) return SMX_E_ALIGN;
    const long long total = (long long)rows * ld_w;
    cudaStream_t s = as_stream(stream);
    switch (elem_bytes) {
        case 1: lanes_to_bits_kernel<uint8_t><<<grid_1d(total), 256, 0, s>>>((const uint8_t*)in, ld, words, ld_w, rows, cols); break;
        case 2: lanes_to_bits_kernel<uint16_t><<<grid_1d(total), 256, 0, s>>>((const uint16_t*)in, ld, words, ld_w, rows, cols); break;
        default: lanes_to_bits_kernel<uint32_t><<<grid_1d(total), 256, 0, s>>>((const uint32_t*)in, ld, words, ld_w, rows, cols); break;
    }
    SMX_RETURN_LAUNCH();
}

int smx_bool_mul_batched(const uint32_t* A, const uint32_t* B, uint32_t* C, int batch, int M, int N, int K,
                         int lda_w, int ldb_w, int ldc_w, long long stride_a, long long stride_b,
                         long long stride_c, void* stream) {
    if (batch < 0 || M < 0 || N < 0 || K < 0) return SMX_E_ARG;
    if ((long long)lda_w * 32 < K || (long long)ldb_w * 32 < N || (long long)ldc_w * 32 < N) return SMX_E_ARG;
    if (batch == 0 || M == 0 || ldc_w == 0) return SMX_OK;
    const long long total = (long long)batch * M * ldc_w;
    bool_mul_batched_kernel<<<grid_1d(total), 256, 0, as_stream(stream)>>>(
        A, B, C, batch, M, K, (N + 31) / 32, lda_w, ldb_w, ldc_w, stride_a, stride_b, stride_c);
    SMX_RETURN_LAUNCH();
}

int smx_bool_warshall_batched(uint32_t* T, int batch, int n, int ld_w, long long stride, void* stream) {
    if (batch < 0 || n < 0 || n > 512 || (long long)ld_w * 32 < n) return SMX_E_ARG;
    if (batch == 0 || n == 0) return SMX_OK;
    cudaStream_t s = as_stream(stream);
    if (n <= 32) {
        const long long threads = (long long)batch * 32;
        bool_close_batched_warp_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(T, batch, n, ld_w, stride);
    } else {
        const size_t smem = (size_t)n * ((n + 31) / 32) * 4;
        bool_close_batched_cta_kernel<<<batch, 256, smem, s>>>(T, batch, n, ld_w, stride);
    }
    SMX_RETURN_LAUNCH();
}

// n <= 128 vertices per matrix, `batch` matrices of n x ld lanes, `stride`
// lanes apart; padding columns [n, ld) are left as they are (the (+)-identity).
int smx_fw_batched(void* T, int batch, int n, int ld, long long stride, int elem_bytes, int kind, void* stream) {
    if (batch < 0 || n < 0 || n > 128 || ld < n || stride < (long long)n * ld) return SMX_E_ARG;
    if (kind != SMX_ANTI && kind != SMX_DIST) return SMX_E_ARG;
    if (batch == 0 || n == 0) return SMX_OK;
    const size_t smem = (size_t)n * n * 4;
    const int anti = kind == SMX_ANTI;
    cudaStream_t s = as_stream(stream);
    // <= 64 KB of shared memory: opt in above the 48 KB default
    switch (elem_bytes) {
        case 1:
            SMX_TRY(set_max_smem((const void*)fw_batched_kernel<uint8_t>, smem));
            fw_batched_kernel<uint8_t><<<batch, 256, smem, s>>>((uint8_t*)T, batch, n, ld, stride, anti);
            break;
        case 2:
            SMX_TRY(set_max_smem((const void*)fw_batched_kernel<uint16_t>, smem));
            fw_batched_kernel<uint16_t><<<batch, 256, smem, s>>>((uint16_t*)T, batch, n, ld, stride, anti);
            break;
        case 4:
            SMX_TRY(set_max_smem((const void*)fw_batched_kernel<uint32_t>, smem));
            fw_batched_kernel<uint32_t><<<batch, 256, smem, s>>>((uint32_t*)T, batch, n, ld, stride, anti);
            break;
        default: return SMX_E_ARG;
    }
    SMX_RETURN_LAUNCH();
}

}  // extern "C"
