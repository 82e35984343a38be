// Entrywise matrix algebra on device, so whole
// workflows stay in HBM between products and closures.
//
// Lane matrices (pkg/src/semimat/antidist.py:128-156): & = lanewise min,
// | = lanewise max, ^ = |a - b| (kernels.py:180-189), ~ = S - a (switches the
// anti-distance / distance view).  Every op restores the padding columns to
// the result class's (+)-identity (antidist.py:111-113): 0 for anti-distance,
// S for distance.
// Boolean matrices (boolmat.py:120-137): |, &, ^ on words, ~ with the tail
// bits past `cols` cleared.
// HBM-bound: one pass, 16-byte vector accesses where rows allow.
#include <cuda_runtime.h>

#include "common.cuh"

namespace smx {

enum { OP_MIN = 0, OP_MAX = 1, OP_ABSDIFF = 2, OP_COMPLEMENT = 3 };

// One 32-bit word of packed lanes (u8x4, u16x2 or u32).  Complement at full
// width is S - a = ~a for every lane width.
template <int EB>
__device__ __forceinline__ uint32_t word_op(uint32_t a, uint32_t b, int op) {
    switch (op) {
        case OP_MIN: return EB == 1 ? __vminu4(a, b) : EB == 2 ? __vminu2(a, b) : min(a, b);
        case OP_MAX: return EB == 1 ? __vmaxu4(a, b) : EB == 2 ? __vmaxu2(a, b) : max(a, b);
        case OP_ABSDIFF: return EB == 1 ? __vabsdiffu4(a, b) : EB == 2 ? __vabsdiffu2(a, b) : (a > b ? a - b : b - a);
        default: return ~a;
    }
}

// Lane entrywise pass over rows x ld lanes (ld * EB a multiple of 16: the
// padded 128-bit lane blocks, antidist.py:38-55), one 16-byte chunk per
// thread-iteration.  The (+)-identity `pad` fills lanes [cols, ld) of every
// row: only the last lane blocks of a row hold padding, so chunks that start
// at or past `first_pad_chunk` of their row take the masked path.  Rows are
// walked with the chunk index split as (row, chunk) incrementally, with no
// per-chunk division.
template <int EB>
__global__ void __launch_bounds__(256) lane_entrywise_kernel(const uint4* __restrict__ A, const uint4* __restrict__ B,
                                                             uint4* __restrict__ C, int rows, int cols, int cpr,
                                                             int op, uint32_t pad) {
    constexpr int E = 16 / EB;   // lanes per chunk
    const int first_pad = cols / E;                  // first chunk of a row with padding
    const long long total = (long long)rows * cpr;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    int c = (int)(i % cpr);                          // (one division per thread)
    const int dc = (int)(stride % cpr);
    for (; i < total; i += stride) {
        const uint4 a = __ldg(A + i);
        const uint4 b = op == OP_COMPLEMENT ? a : __ldg(B + i);
        uint4 v = make_uint4(word_op<EB>(a.x, b.x, op), word_op<EB>(a.y, b.y, op), word_op<EB>(a.z, b.z, op),
                             word_op<EB>(a.w, b.w, op));
        if (c >= first_pad) {   // lanes [cols - c*E, E) of this chunk are padding
            uint32_t* w = reinterpret_cast<uint32_t*>(&v);
            const int valid = cols - c * E;          // lanes of data in this chunk (may be <= 0)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
#pragma unroll
                for (int l = 0; l < 4 / EB; ++l) {
                    const int lane = q * (4 / EB) + l;
                    if (lane >= valid) {
                        const int sh = 8 * EB * l;
                        const uint32_t m = EB == 4 ? 0xFFFFFFFFu : (((1u << (8 * EB)) - 1u) << sh);
                        w[q] = (w[q] & ~m) | (pad & m);
                    }
                }
            }
        }
        C[i] = v;
        c += dc;
        while (c >= cpr) c -= cpr;
    }
}

enum { BOP_OR = 0, BOP_AND = 1, BOP_XOR = 2, BOP_NOT = 3 };

// Boolean words, 16 bytes per thread-iteration when the row stride allows
// (ld_w % 4 == 0), with the tail bits past `cols` cleared in the row's last
// data word and the words past it zeroed.
__device__ __forceinline__ uint32_t bits_word(uint32_t a, uint32_t b, int op) {
    switch (op) {
        case BOP_OR: return a | b;
        case BOP_AND: return a & b;
        case BOP_XOR: return a ^ b;
        default: return ~a;
    }
}
__device__ __forceinline__ uint32_t bits_mask(uint32_t v, int w, int cols) {
    const int lo = w * 32;
    if (lo >= cols) return 0u;
    if (cols - lo < 32) return v & ((1u << (cols - lo)) - 1u);
    return v;
}

__global__ void __launch_bounds__(256) bits_entrywise_vec_kernel(const uint4* __restrict__ A,
                                                                 const uint4* __restrict__ B, uint4* __restrict__ C,
                                                                 int rows, int cols, int cpr, int op) {
    const long long total = (long long)rows * cpr;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    int c = (int)(i % cpr);
    const int dc = (int)(stride % cpr);
    const int first_tail = cols / 128;               // first chunk (4 words) holding bits past `cols`
    for (; i < total; i += stride) {
        const uint4 a = __ldg(A + i);
        const uint4 b = op == BOP_NOT ? a : __ldg(B + i);
        uint4 v = make_uint4(bits_word(a.x, b.x, op), bits_word(a.y, b.y, op), bits_word(a.z, b.z, op),
                             bits_word(a.w, b.w, op));
        if (c >= first_tail) {
            v.x = bits_mask(v.x, 4 * c, cols);
            v.y = bits_mask(v.y, 4 * c + 1, cols);
            v.z = bits_mask(v.z, 4 * c + 2, cols);
            v.w = bits_mask(v.w, 4 * c + 3, cols);
        }
        C[i] = v;
        c += dc;
        while (c >= cpr) c -= cpr;
    }
}

__global__ void bits_entrywise_kernel(const uint32_t* A, const uint32_t* B,
                                      uint32_t* C, int rows, int cols, long long ld_w,
                                      int op) {
    const long long total = (long long)rows * ld_w;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(i % ld_w);
        C[i] = bits_mask(bits_word(A[i], op == BOP_NOT ? 0u : B[i], op), w, cols);
    }
}

inline unsigned grid_for(long long n) {
    long long g = (n + 255) / 256;
    if (g > 148LL * 16) g = 148LL * 16;
    return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace smx

using namespace smx;

extern "C" int smx_lane_entrywise(const void* A, const void* B, void* C, int rows, int cols, int ld,
                                  int elem_bytes, int op, int pad_is_limit, void* stream) {
    if (rows < 0 || cols < 0 || ld < cols || op < 0 || op > 3) return SMX_E_ARG;
    if (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4) return SMX_E_ARG;
    if (rows == 0 || ld == 0) return SMX_OK;
    // rows are whole 128-bit lane blocks (the reference's padded layout)
    if (((long long)ld * elem_bytes) % 16 != 0) return SMX_E_ARG;
    if (!aligned16(A) || !aligned16(C) || (op != OP_COMPLEMENT && !aligned16(B))) return SMX_E_ALIGN;
    const int cpr = (int)((long long)ld * elem_bytes / 16);
    const unsigned g = grid_for((long long)rows * cpr);
    cudaStream_t s = as_stream(stream);
    const uint32_t pad = pad_is_limit ? 0xFFFFFFFFu : 0u;   // S in every lane, or 0
    auto a = static_cast<const uint4*>(A);
    auto b = static_cast<const uint4*>(op == OP_COMPLEMENT ? A : B);
    auto c = static_cast<uint4*>(C);
    switch (elem_bytes) {
        case 1: lane_entrywise_kernel<1><<<g, 256, 0, s>>>(a, b, c, rows, cols, cpr, op, pad); break;
        case 2: lane_entrywise_kernel<2><<<g, 256, 0, s>>>(a, b, c, rows, cols, cpr, op, pad); break;
        default: lane_entrywise_kernel<4><<<g, 256, 0, s>>>(a, b, c, rows, cols, cpr, op, pad); break;
    }
    SMX_RETURN_LAUNCH();
}

extern "C" int smx_bits_entrywise(const uint32_t* A, const uint32_t* B, uint32_t* C, int rows, int cols,
                                  int ld_w, int op, void* stream) {
    if (rows < 0 || cols < 0 || (long long)ld_w * 32 < cols || op < 0 || op > 3) return SMX_E_ARG;
    if (rows == 0 || ld_w == 0) return SMX_OK;
    cudaStream_t s = as_stream(stream);
    if (ld_w % 4 == 0 && aligned16(A) && aligned16(C) && (op == BOP_NOT || aligned16(B))) {
        const int cpr = ld_w / 4;
        bits_entrywise_vec_kernel<<<grid_for((long long)rows * cpr), 256, 0, s>>>(
            reinterpret_cast<const uint4*>(A), reinterpret_cast<const uint4*>(op == BOP_NOT ? A : B),
            reinterpret_cast<uint4*>(C), rows, cols, cpr, op);
        SMX_RETURN_LAUNCH();
    }
    bits_entrywise_kernel<<<grid_for((long long)rows * ld_w), 256, 0, s>>>(A, B, C, rows, cols, ld_w, op);
    SMX_RETURN_LAUNCH();
}
