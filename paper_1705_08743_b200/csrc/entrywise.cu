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

template <typename T>
__device__ __forceinline__ T lane_op(T a, T b, int op, T S) {
    switch (op) {
        case OP_MIN: return a < b ? a : b;
        case OP_MAX: return a > b ? a : b;
        case OP_ABSDIFF: return a > b ? T(a - b) : T(b - a);
        default: return T(S - a);
    }
}

template <typename T>
__global__ void lane_entrywise_kernel(const T* A, const T* B,
                                      T* C, int rows, int cols, long long ld, int op,
                                      T pad) {
    const long long total = (long long)rows * ld;
    const T S = T(Limit<T>::value);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % ld);
        C[i] = c < cols ? lane_op<T>(A[i], op == OP_COMPLEMENT ? T(0) : B[i], op, S) : pad;
    }
}

enum { BOP_OR = 0, BOP_AND = 1, BOP_XOR = 2, BOP_NOT = 3 };

__global__ void bits_entrywise_kernel(const uint32_t* A, const uint32_t* B,
                                      uint32_t* C, int rows, int cols, long long ld_w,
                                      int op) {
    const long long total = (long long)rows * ld_w;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(i % ld_w);
        const uint32_t a = A[i];
        uint32_t v;
        switch (op) {
            case BOP_OR: v = a | B[i]; break;
            case BOP_AND: v = a & B[i]; break;
            case BOP_XOR: v = a ^ B[i]; break;
            default: v = ~a; break;
        }
        const int lo = w * 32;
        if (lo >= cols) v = 0;
        else if (cols - lo < 32) v &= (1u << (cols - lo)) - 1u;
        C[i] = v;
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
    if (rows == 0 || ld == 0) return SMX_OK;
    const unsigned g = grid_for((long long)rows * ld);
    cudaStream_t s = as_stream(stream);
    switch (elem_bytes) {
        case 1:
            lane_entrywise_kernel<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)A, (const uint8_t*)B,
                                                             (uint8_t*)C, rows, cols, ld, op,
                                                             pad_is_limit ? 0xFFu : 0u);
            break;
        case 2:
            lane_entrywise_kernel<uint16_t><<<g, 256, 0, s>>>((const uint16_t*)A, (const uint16_t*)B,
                                                              (uint16_t*)C, rows, cols, ld, op,
                                                              pad_is_limit ? 0xFFFFu : 0u);
            break;
        case 4:
            lane_entrywise_kernel<uint32_t><<<g, 256, 0, s>>>((const uint32_t*)A, (const uint32_t*)B,
                                                              (uint32_t*)C, rows, cols, ld, op,
                                                              pad_is_limit ? 0xFFFFFFFFu : 0u);
            break;
        default: return SMX_E_ARG;
    }
    SMX_RETURN_LAUNCH();
}

extern "C" int smx_bits_entrywise(const uint32_t* A, const uint32_t* B, uint32_t* C, int rows, int cols,
                                  int ld_w, int op, void* stream) {
    if (rows < 0 || cols < 0 || (long long)ld_w * 32 < cols || op < 0 || op > 3) return SMX_E_ARG;
    if (rows == 0 || ld_w == 0) return SMX_OK;
    bits_entrywise_kernel<<<grid_for((long long)rows * ld_w), 256, 0, as_stream(stream)>>>(
        A, B, C, rows, cols, ld_w, op);
    SMX_RETURN_LAUNCH();
}
