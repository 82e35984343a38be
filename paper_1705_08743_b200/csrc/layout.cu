// Byte <-> bit layout helpers for Boolean matrices (the reference's LSB-first
// 64-bit block rows, pkg/src/semimat/boolmat.py:3-5, read as u32 words) and a
// byte transpose for the tensor-core B^T operand.
#include <cuda_runtime.h>

#include "common.cuh"

namespace smx {

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

// ---- E2M1 nibble operands (kind::mxf4 products, bool_tc.cu) ------------------
// Bit i of a word -> nibble i (byte i / 2, low nibble first) holding 0 or
// 0b0010 (E2M1 1.0).  A and B^T use the same order along K, so the product
// pairs the same elements whatever order the MMA reads the two nibbles of a
// byte in.
__device__ __forceinline__ uint32_t nib8(uint32_t x) {
    x = (x | (x << 12)) & 0x000F000Fu;
    x = (x | (x << 6)) & 0x03030303u;
    x = (x | (x << 3)) & 0x11111111u;
    return x << 1;
}

// 32 bits (valid of them) -> 16 bytes at dst
__device__ __forceinline__ void store_nibbles(uint8_t* dst, uint32_t w, int valid) {
    if (valid < 32) w &= (1u << (valid > 0 ? valid : 0)) - 1u;
    const uint4 o = make_uint4(nib8(w & 0xFFu), nib8((w >> 8) & 0xFFu), nib8((w >> 16) & 0xFFu), nib8(w >> 24));
    if (valid >= 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        *reinterpret_cast<uint4*>(dst) = o;
    } else {
        const uint8_t* ob = reinterpret_cast<const uint8_t*>(&o);
        for (int c = 0; c < 16 && 2 * c < valid; ++c) dst[c] = ob[c];
    }
}

// A: bit rows -> nibble rows (row r at r * ld bytes); B: bit rows (K x N) ->
// the transposed K-major nibble operand (N rows of ceil(K / 2) bytes), by
// the ballot transpose of unpack_bits_t_kernel.  Blocks [0, a_blocks) take
// A (when present), the rest B; blockIdx.y is the item of a batch (A words
// and bytes a_in / a_out apart, B likewise).
__global__ void unpack_nib_ab_kernel(const uint32_t* __restrict__ a_words, uint8_t* __restrict__ a_nib, int a_rows,
                                     int a_cols, long long a_ldw, long long a_ld, int a_blocks,
                                     long long a_in, long long a_out,
                                     const uint32_t* __restrict__ b_words, uint8_t* __restrict__ bt, int b_rows,
                                     int b_cols, long long b_ldw, long long b_ldt, long long b_in, long long b_out) {
    if ((int)blockIdx.x < a_blocks) {
        a_words += (long long)blockIdx.y * a_in;
        a_nib += (long long)blockIdx.y * a_out;
        const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
        const int nw = (a_cols + 31) / 32;
        if (t >= (long long)a_rows * nw) return;
        const int r = (int)(t / nw), wi = (int)(t % nw);
        store_nibbles(a_nib + (long long)r * a_ld + wi * 16, a_words[(long long)r * a_ldw + wi], a_cols - wi * 32);
        return;
    }
    b_words += (long long)blockIdx.y * b_in;
    bt += (long long)blockIdx.y * b_out;
    const long long warp = ((long long)(blockIdx.x - a_blocks) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int kt = (b_rows + 31) / 32, jt = (b_cols + 31) / 32;
    if (warp >= (long long)kt * jt) return;
    const int k0 = (int)(warp % kt) * 32, wj = (int)(warp / kt);
    const int k = k0 + lane;
    const uint32_t w = k < b_rows ? b_words[(long long)k * b_ldw + wj] : 0u;
    uint32_t mine = 0;
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, (w >> jj) & 1u);
        if (lane == jj) mine = m;
    }
    const int j = wj * 32 + lane;
    if (j >= b_cols) return;
    store_nibbles(bt + (long long)j * b_ldt + k0 / 2, mine, b_rows - k0);
}

// Bits -> transposed bytes in one pass (the K-major B^T operand of the
// tensor-core product straight from the reference's bit rows): a warp takes a
// 32 (k) x 32 (j) bit tile; lane l holds row k0+l's word, 32 ballots turn the
// tile around, lane l then owns output row j0+l and writes its 32 bytes.
// (blockIdx.y: the item of a batch: its words at + y * in_stride, its output
// at + y * out_stride)
__global__ void unpack_bits_t_kernel(const uint32_t* __restrict__ words, uint8_t* __restrict__ out,
                                     int rows, int cols, long long ld_w, long long ld_out,
                                     long long in_stride = 0, long long out_stride = 0) {
    words += (long long)blockIdx.y * in_stride;
    out += (long long)blockIdx.y * out_stride;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int kt = (rows + 31) / 32, jt = (cols + 31) / 32;
    if (warp >= (long long)kt * jt) return;
    const int k0 = (int)(warp % kt) * 32, wj = (int)(warp / kt);
    const int k = k0 + lane;
    const uint32_t w = k < rows ? words[(long long)k * ld_w + wj] : 0u;
    uint32_t mine = 0;
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, (w >> jj) & 1u);
        if (lane == jj) mine = m;
    }
    const int j = wj * 32 + lane;
    if (j >= cols) return;
    uint32_t o[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = (((mine >> (4 * q)) & 0xFu) * 0x00204081u) & 0x01010101u;
    uint8_t* dst = out + (long long)j * ld_out + k0;
    const int valid = rows - k0;
    if (valid >= 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        reinterpret_cast<uint4*>(dst)[0] = make_uint4(o[0], o[1], o[2], o[3]);
        reinterpret_cast<uint4*>(dst)[1] = make_uint4(o[4], o[5], o[6], o[7]);
    } else {
        const uint8_t* ob = reinterpret_cast<const uint8_t*>(o);
        for (int c = 0; c < 32 && c < valid; ++c) dst[c] = ob[c];
    }
}

// Both operands of the one-call tensor-core product in one launch: blocks
// [0, a_blocks) unpack A's bit rows (unpack_bits_kernel), the rest turn B's
// bit rows into the transposed K-major byte operand (unpack_bits_t_kernel).
__global__ void unpack_ab_kernel(const uint32_t* __restrict__ a_words, uint8_t* __restrict__ a_bytes, int a_rows,
                                 int a_cols, long long a_ldw, long long a_ld, int a_blocks,
                                 const uint32_t* __restrict__ b_words, uint8_t* __restrict__ bt, int b_rows,
                                 int b_cols, long long b_ldw, long long b_ldt) {
    if ((int)blockIdx.x < a_blocks) {
        const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
        const int nw = (a_cols + 31) / 32;
        if (t >= (long long)a_rows * nw) return;
        const int r = (int)(t / nw), wi = (int)(t % nw);
        const uint32_t w = a_words[(long long)r * a_ldw + wi];
        uint32_t o[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = (((w >> (4 * q)) & 0xFu) * 0x00204081u) & 0x01010101u;
        uint8_t* dst = a_bytes + (long long)r * a_ld + wi * 32;
        const int valid = a_cols - wi * 32;
        if (valid >= 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
            reinterpret_cast<uint4*>(dst)[0] = make_uint4(o[0], o[1], o[2], o[3]);
            reinterpret_cast<uint4*>(dst)[1] = make_uint4(o[4], o[5], o[6], o[7]);
        } else {
            const uint8_t* ob = reinterpret_cast<const uint8_t*>(o);
            for (int c = 0; c < 32 && c < valid; ++c) dst[c] = ob[c];
        }
        return;
    }
    const long long warp = ((long long)(blockIdx.x - a_blocks) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int kt = (b_rows + 31) / 32, jt = (b_cols + 31) / 32;
    if (warp >= (long long)kt * jt) return;
    const int k0 = (int)(warp % kt) * 32, wj = (int)(warp / kt);
    const int k = k0 + lane;
    const uint32_t w = k < b_rows ? b_words[(long long)k * b_ldw + wj] : 0u;
    uint32_t mine = 0;
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, (w >> jj) & 1u);
        if (lane == jj) mine = m;
    }
    const int j = wj * 32 + lane;
    if (j >= b_cols) return;
    uint32_t o[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = (((mine >> (4 * q)) & 0xFu) * 0x00204081u) & 0x01010101u;
    uint8_t* dst = bt + (long long)j * b_ldt + k0;
    const int valid = b_rows - k0;
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

int unpack_bits(const uint32_t* words, uint8_t* bytes, int rows, int cols, long long ld_w, long long ld,
                cudaStream_t s) {
    if (rows < 0 || cols < 0 || ld < cols || ld_w * 32 < cols) return SMX_E_ARG;
    if (rows == 0 || cols == 0) return SMX_OK;
    const long long t = (long long)rows * ((cols + 31) / 32);
    unpack_bits_kernel<<<(unsigned)((t + 255) / 256), 256, 0, s>>>(words, bytes, rows, cols, ld_w, ld);
    SMX_RETURN_LAUNCH();
}

// A (a_rows x a_cols bits) -> bytes, and B (b_rows x b_cols bits) -> B^T
// bytes (b_cols x b_rows), in one launch.
int unpack_ab(const uint32_t* a_words, uint8_t* a_bytes, int a_rows, int a_cols, long long a_ldw, long long a_ld,
              const uint32_t* b_words, uint8_t* bt, int b_rows, int b_cols, long long b_ldw, long long b_ldt,
              cudaStream_t s) {
    if (a_rows < 0 || a_cols < 0 || a_ld < a_cols || a_ldw * 32 < a_cols) return SMX_E_ARG;
    if (b_rows < 0 || b_cols < 0 || b_ldt < b_rows || b_ldw * 32 < b_cols) return SMX_E_ARG;
    const long long ta = (long long)a_rows * ((a_cols + 31) / 32);
    const long long a_blocks = (ta + 255) / 256;
    const long long warps = (long long)((b_rows + 31) / 32) * ((b_cols + 31) / 32);
    const long long b_blocks = (warps * 32 + 255) / 256;
    if (a_blocks + b_blocks == 0) return SMX_OK;
    unpack_ab_kernel<<<(unsigned)(a_blocks + b_blocks), 256, 0, s>>>(a_words, a_bytes, a_rows, a_cols, a_ldw, a_ld,
                                                                   (int)a_blocks, b_words, bt, b_rows, b_cols,
                                                                   b_ldw, b_ldt);
    SMX_RETURN_LAUNCH();
}

// `batch` matrices of rows x cols bits (words `in_stride` apart) -> their
// transposed bytes (`out_stride` apart), one launch.
int unpack_bits_transposed_batched(const uint32_t* words, uint8_t* out, int batch, int rows, int cols, long long ld_w,
                                   long long ld_out, long long in_stride, long long out_stride, cudaStream_t s) {
    if (batch < 0 || rows < 0 || cols < 0 || ld_out < rows || ld_w * 32 < cols) return SMX_E_ARG;
    if (batch == 0 || rows == 0 || cols == 0) return SMX_OK;
    const long long warps = (long long)((rows + 31) / 32) * ((cols + 31) / 32);
    unpack_bits_t_kernel<<<dim3((unsigned)((warps * 32 + 255) / 256), (unsigned)batch), 256, 0, s>>>(
        words, out, rows, cols, ld_w, ld_out, in_stride, out_stride);
    SMX_RETURN_LAUNCH();
}

// Nibble operands of `batch` products in one launch: A (a_rows x a_cols bits
// per item; a_words == nullptr skips A) and B (b_rows x b_cols bits per
// item) -> A nibbles (a_ld bytes per row) and B^T nibbles (b_ldt bytes per
// row); items a_in / a_out (B: b_in / b_out) words / bytes apart.
int unpack_nib_ab(const uint32_t* a_words, uint8_t* a_nib, int a_rows, int a_cols, long long a_ldw, long long a_ld,
                  const uint32_t* b_words, uint8_t* bt, int b_rows, int b_cols, long long b_ldw, long long b_ldt,
                  int batch, long long a_in, long long a_out, long long b_in, long long b_out, cudaStream_t s) {
    if (batch < 1) return batch == 0 ? SMX_OK : SMX_E_ARG;
    if (a_words && (a_rows < 0 || a_cols < 0 || 2 * a_ld < a_cols || a_ldw * 32 < a_cols)) return SMX_E_ARG;
    if (b_rows < 0 || b_cols < 0 || 2 * b_ldt < b_rows || b_ldw * 32 < b_cols) return SMX_E_ARG;
    const long long ta = a_words ? (long long)a_rows * ((a_cols + 31) / 32) : 0;
    const long long a_blocks = (ta + 255) / 256;
    const long long warps = (long long)((b_rows + 31) / 32) * ((b_cols + 31) / 32);
    const long long b_blocks = (warps * 32 + 255) / 256;
    if (a_blocks + b_blocks == 0) return SMX_OK;
    unpack_nib_ab_kernel<<<dim3((unsigned)(a_blocks + b_blocks), (unsigned)batch), 256, 0, s>>>(
        a_words, a_nib, a_rows, a_cols, a_ldw, a_ld, (int)a_blocks, a_in, a_out, b_words, bt, b_rows, b_cols, b_ldw,
        b_ldt, b_in, b_out);
    SMX_RETURN_LAUNCH();
}

int unpack_bits_transposed(const uint32_t* words, uint8_t* out, int rows, int cols, long long ld_w,
                           long long ld_out, cudaStream_t s) {
    if (rows < 0 || cols < 0 || ld_out < rows || ld_w * 32 < cols) return SMX_E_ARG;
    if (rows == 0 || cols == 0) return SMX_OK;
    const long long warps = (long long)((rows + 31) / 32) * ((cols + 31) / 32);
    unpack_bits_t_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(words, out, rows, cols, ld_w,
                                                                             ld_out);
    SMX_RETURN_LAUNCH();
}

}  // namespace smx

using namespace smx;

extern "C" {

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
    return unpack_bits(words, bytes, rows, cols, ld_w, ld, as_stream(stream));
}

int smx_unpack_bits_transposed(const uint32_t* words, uint8_t* bytes_t, int rows, int cols, int ld_w,
                               int ld_out, void* stream) {
    return unpack_bits_transposed(words, bytes_t, rows, cols, ld_w, ld_out, as_stream(stream));
}

int smx_unpack_nibbles(const uint32_t* a_words, uint8_t* a_nib, int a_rows, int a_cols, int a_ldw, int a_ld,
                       const uint32_t* b_words, uint8_t* bt_nib, int b_rows, int b_cols, int b_ldw, int b_ldt,
                       void* stream) {
    return unpack_nib_ab(a_words, a_nib, a_rows, a_cols, a_ldw, a_ld, b_words, bt_nib, b_rows, b_cols, b_ldw, b_ldt,
                         1, 0, 0, 0, 0, as_stream(stream));
}

int smx_transpose_u8(const uint8_t* in, uint8_t* out, int rows, int cols, int ld_in, int ld_out,
                     void* stream) {
    return transpose_bytes(in, out, rows, cols, ld_in, ld_out, as_stream(stream));
}

}  // extern "C"
