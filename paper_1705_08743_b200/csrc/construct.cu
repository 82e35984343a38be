// Matrix construction on device.
//
// AntidistMatrix.from_edges / DistMatrix.from_edges
// (pkg/src/semimat/antidist.py:191-211, :294-309) build an adjacency matrix in
// a Python loop: parallel edges keep the shortest distance, i.e. the largest
// anti-distance value S - w or the smallest distance w.  Here every edge is
// one thread that folds its value into the matrix with an atomic max / min on
// the aligned 32-bit word that holds its lane (compare-and-swap on the lane
// for u8/u16), so the result is independent of edge order -- exactly the
// reference's "keep the best parallel edge" rule.  The matrix is first filled
// with the class's (+)-identity (0 anti-distance, S distance) including the
// padding lanes.  Edge validation (vertex and weight ranges) happens in the
// Python layer with the reference's messages before anything is launched.
#include <cuda_runtime.h>

#include "common.cuh"

namespace smx {

template <typename T>
__global__ void fill_kernel(T* t, long long count, T value) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        t[i] = value;
}
// The same fill as 16-byte stores (the padded lane rows are whole 16-byte
// blocks, so the matrix is too); HBM-bound.
__global__ void fill16_kernel(uint4* t, long long chunks, uint32_t word) {
    const uint4 v = make_uint4(word, word, word, word);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < chunks;
         i += (long long)gridDim.x * blockDim.x)
        t[i] = v;
}

template <typename T>
__device__ __forceinline__ void fold_lane(T* cell, uint32_t value, bool take_max) {
    if constexpr (sizeof(T) == 4) {
        if (take_max) atomicMax(reinterpret_cast<unsigned int*>(cell), value);
        else atomicMin(reinterpret_cast<unsigned int*>(cell), value);
    } else {
        const uintptr_t addr = reinterpret_cast<uintptr_t>(cell);
        unsigned int* word = reinterpret_cast<unsigned int*>(addr & ~uintptr_t(3));
        const int shift = (int)(addr & 3) * 8;
        const uint32_t mask = (sizeof(T) == 1 ? 0xFFu : 0xFFFFu) << shift;
        unsigned int old = *word, assumed;
        do {
            assumed = old;
            const uint32_t cur = (assumed & mask) >> shift;
            const uint32_t nv = take_max ? (value > cur ? value : cur) : (value < cur ? value : cur);
            if (nv == cur) break;
            old = atomicCAS(word, assumed, (assumed & ~mask) | (nv << shift));
        } while (old != assumed);
    }
}

template <typename T>
__global__ void scatter_edges_kernel(const long long* __restrict__ edges, long long m, T* t, long long ld,
                                     bool anti) {
    const uint32_t S = Limit<T>::value;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (long long)gridDim.x * blockDim.x) {
        const long long u = edges[3 * e], v = edges[3 * e + 1];
        const uint32_t w = (uint32_t)edges[3 * e + 2];
        fold_lane<T>(t + u * ld + v, anti ? S - w : w, anti);
    }
}

// First invalid edge in edge order (the reference validates in order and
// reports the first offender, antidist.py:201-208): a vertex outside [0, n)
// or a weight outside [0, limit].  *first = the smallest offending index, or
// left at its initial value (the caller sets it to m).
__global__ void first_invalid_edge_kernel(const long long* __restrict__ edges, long long m, long long n,
                                          long long limit, unsigned long long* first) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (long long)gridDim.x * blockDim.x) {
        const long long u = edges[3 * e], v = edges[3 * e + 1], w = edges[3 * e + 2];
        if (u < 0 || u >= n || v < 0 || v >= n || w < 0 || w > limit)
            atomicMin(first, (unsigned long long)e);
    }
}

template <typename T>
int from_edges(const long long* edges, long long m, T* t, int n, long long ld, bool anti, cudaStream_t s) {
    const long long count = (long long)n * ld;
    const T fill = anti ? T(0) : T(Limit<T>::value);
    if (aligned16(t) && (count * (long long)sizeof(T)) % 16 == 0) {
        const long long chunks = count * (long long)sizeof(T) / 16;
        long long blocks = (chunks + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        const uint32_t word = anti ? 0u : 0xFFFFFFFFu;   // S in every lane, or 0
        fill16_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(reinterpret_cast<uint4*>(t), chunks, word);
    } else {
        long long blocks = (count + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        fill_kernel<T><<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(t, count, fill);
    }
    SMX_LAUNCHED_OR_RETURN();
    if (m == 0) return SMX_OK;
    long long eb = (m + 255) / 256;
    if (eb > 148 * 16) eb = 148 * 16;
    scatter_edges_kernel<T><<<(unsigned)eb, 256, 0, s>>>(edges, m, t, ld, anti);
    SMX_RETURN_LAUNCH();
}

}  // namespace smx

using namespace smx;

extern "C" int smx_from_edges(const long long* edges, long long m, void* T, int n, int ld, int elem_bytes,
                              int kind, void* stream) {
    if (n < 0 || ld < n || m < 0 || (kind != SMX_ANTI && kind != SMX_DIST)) return SMX_E_ARG;
    if (n == 0) return SMX_OK;
    const bool anti = kind == SMX_ANTI;
    cudaStream_t s = as_stream(stream);
    switch (elem_bytes) {
        case 1: return from_edges<uint8_t>(edges, m, (uint8_t*)T, n, ld, anti, s);
        case 2: return from_edges<uint16_t>(edges, m, (uint16_t*)T, n, ld, anti, s);
        case 4: return from_edges<uint32_t>(edges, m, (uint32_t*)T, n, ld, anti, s);
        default: return SMX_E_ARG;
    }
}

extern "C" int smx_edges_first_invalid(const long long* edges, long long m, int n, long long limit,
                                       unsigned long long* first, void* stream) {
    if (m < 0 || n < 0 || first == nullptr) return SMX_E_ARG;
    cudaStream_t s = as_stream(stream);
    const unsigned long long init = (unsigned long long)m;
    cudaError_t e = cudaMemcpyAsync(first, &init, sizeof(init), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return (int)e;
    if (m == 0) return SMX_OK;
    long long blocks = (m + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    first_invalid_edge_kernel<<<(unsigned)blocks, 256, 0, s>>>(edges, m, n, limit, first);
    SMX_RETURN_LAUNCH();
}
