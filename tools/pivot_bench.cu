// Development harness: Boolean 256x256 Warshall pivot variants (not part of the library).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pivot_bench tools/pivot_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

constexpr int B = 256, W = 8;

// V1: the library's current kernel (per-step shuffle chain, then fold).
__global__ void __launch_bounds__(B, 1) v1(const uint32_t* src, uint32_t* P, int ld_w) {
    __shared__ __align__(16) uint32_t panel[32][W];
    const int r = threadIdx.x, warp = r >> 5, lane = r & 31;
    uint32_t w[W];
#pragma unroll
    for (int i = 0; i < W; ++i) w[i] = src[r * ld_w + i];
#pragma unroll
    for (int q = 0; q < W; ++q) {
        const uint32_t orig = w[q];
        if (warp == q) {
            for (int kk = 0; kk < 32; ++kk) {
                uint32_t pv[W];
#pragma unroll
                for (int i = 0; i < W; ++i) pv[i] = __shfl_sync(0xFFFFFFFFu, w[i], kk);
                if ((w[q] >> kk) & 1u) {
#pragma unroll
                    for (int i = 0; i < W; ++i) w[i] |= pv[i];
                }
            }
            *reinterpret_cast<uint4*>(&panel[lane][0]) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4*>(&panel[lane][4]) = make_uint4(w[4], w[5], w[6], w[7]);
        }
        __syncthreads();
        if (warp != q) {
            for (int kk = 0; kk < 32; ++kk) {
                if ((orig >> kk) & 1u) {
                    const uint4 v0 = *reinterpret_cast<const uint4*>(&panel[kk][0]);
                    const uint4 v1 = *reinterpret_cast<const uint4*>(&panel[kk][4]);
                    w[0] |= v0.x; w[1] |= v0.y; w[2] |= v0.z; w[3] |= v0.w;
                    w[4] |= v1.x; w[5] |= v1.y; w[6] |= v1.z; w[7] |= v1.w;
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < W; ++i) P[r * ld_w + i] = w[i];
}

// Fold helper: w |= OR over set bits k of mask of panel row k (8 words).
__device__ __forceinline__ void fold(uint32_t (&w)[W], uint32_t mask, const uint32_t (*pan)[W]) {
    while (mask) {
        const int k = __ffs(mask) - 1;
        mask &= mask - 1;
        const uint4 v0 = *reinterpret_cast<const uint4*>(&pan[k][0]);
        const uint4 v1 = *reinterpret_cast<const uint4*>(&pan[k][4]);
        w[0] |= v0.x; w[1] |= v0.y; w[2] |= v0.z; w[3] |= v0.w;
        w[4] |= v1.x; w[5] |= v1.y; w[6] |= v1.z; w[7] |= v1.w;
    }
}
__device__ __forceinline__ void fold_all(uint32_t (&w)[W], uint32_t mask, const uint32_t (*pan)[W]) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        const uint32_t m = 0u - ((mask >> k) & 1u);
        const uint4 v0 = *reinterpret_cast<const uint4*>(&pan[k][0]);
        const uint4 v1 = *reinterpret_cast<const uint4*>(&pan[k][4]);
        w[0] |= v0.x & m; w[1] |= v0.y & m; w[2] |= v0.z & m; w[3] |= v0.w & m;
        w[4] |= v1.x & m; w[5] |= v1.y & m; w[6] |= v1.z & m; w[7] |= v1.w & m;
    }
}

// 32x32 transitive closure of one word per lane by 5 squarings.
__device__ __forceinline__ uint32_t close32(uint32_t d) {
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
            const uint32_t v0 = __shfl_sync(0xFFFFFFFFu, d, k);
            const uint32_t v1 = __shfl_sync(0xFFFFFFFFu, d, k + 1);
            const uint32_t v2 = __shfl_sync(0xFFFFFFFFu, d, k + 2);
            const uint32_t v3 = __shfl_sync(0xFFFFFFFFu, d, k + 3);
            a0 |= v0 & (0u - ((d >> k) & 1u));
            a1 |= v1 & (0u - ((d >> (k + 1)) & 1u));
            a2 |= v2 & (0u - ((d >> (k + 2)) & 1u));
            a3 |= v3 & (0u - ((d >> (k + 3)) & 1u));
        }
        const uint32_t nd = d | a0 | a1 | a2 | a3;
        if (__all_sync(0xFFFFFFFFu, nd == d)) break;
        d = nd;
    }
    return d;
}

// V3: diagonal closure by squaring, owner rows by one fold over the original rows, others by one fold.
// SPARSE selects the ffs-driven fold (skips zero bits) instead of the predicated full fold.
template <bool SPARSE>
__global__ void __launch_bounds__(B, 1) v3(const uint32_t* src, uint32_t* P, int ld_w) {
    __shared__ __align__(16) uint32_t orig_rows[32][W];
    __shared__ __align__(16) uint32_t panel[2][32][W];
    const int r = threadIdx.x, warp = r >> 5, lane = r & 31;
    uint32_t w[W];
#pragma unroll
    for (int i = 0; i < W; ++i) w[i] = src[r * ld_w + i];
#pragma unroll
    for (int q = 0; q < W; ++q) {
        if (warp == q) {
            *reinterpret_cast<uint4*>(&orig_rows[lane][0]) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4*>(&orig_rows[lane][4]) = make_uint4(w[4], w[5], w[6], w[7]);
            const uint32_t dplus = close32(w[q]);
            __syncwarp();
            if (SPARSE) fold(w, dplus, orig_rows); else fold_all(w, dplus, orig_rows);
            *reinterpret_cast<uint4*>(&panel[q & 1][lane][0]) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4*>(&panel[q & 1][lane][4]) = make_uint4(w[4], w[5], w[6], w[7]);
            __syncwarp();
        }
        __syncthreads();
        if (warp != q) {
            if (SPARSE) fold(w, w[q], panel[q & 1]); else fold_all(w, w[q], panel[q & 1]);
        }
    }
#pragma unroll
    for (int i = 0; i < W; ++i) P[r * ld_w + i] = w[i];
}

// V5: one table-driven fold per sub-round (method of four Russians over nibbles).
// Sub-round q: D+ = closure of the 32x32 diagonal block. Every row j then gains
// OR_{k in m_j u m_j.D+} orig_row_k, where m_j is its original K_q word (rows of K_q use D+).
__global__ void __launch_bounds__(B, 1) v5(const uint32_t* src, uint32_t* P, int ld_w) {
    __shared__ __align__(16) uint32_t orig[32][W];
    __shared__ __align__(16) uint32_t tab[8][16][W];
    __shared__ uint32_t dtab[8][16];
    __shared__ uint32_t dp[32];
    const int r = threadIdx.x, warp = r >> 5, lane = r & 31;
    uint32_t w[W];
#pragma unroll
    for (int i = 0; i < W; ++i) w[i] = src[r * ld_w + i];
#pragma unroll
    for (int q = 0; q < W; ++q) {
        if (warp == q) {
            *reinterpret_cast<uint4*>(&orig[lane][0]) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4*>(&orig[lane][4]) = make_uint4(w[4], w[5], w[6], w[7]);
            dp[lane] = close32(w[q]);
        }
        __syncthreads();
        {
            // Thread r builds half of table entry (g, e): words [4h, 4h+4).
            const int g = r >> 5, e = (r >> 1) & 15, h = r & 1;
            uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if ((e >> b) & 1) {
                    const uint4 v = *reinterpret_cast<const uint4*>(&orig[4 * g + b][4 * h]);
                    acc.x |= v.x; acc.y |= v.y; acc.z |= v.z; acc.w |= v.w;
                }
            *reinterpret_cast<uint4*>(&tab[g][e][4 * h]) = acc;
            if (r < 128) {
                const int g2 = r >> 4, e2 = r & 15;
                uint32_t d = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if ((e2 >> b) & 1) d |= dp[4 * g2 + b];
                dtab[g2][e2] = d;
            }
        }
        __syncthreads();
        uint32_t m = w[q];
        if (warp == q) {
            m = dp[lane];
        } else if (m) {
            uint32_t ext = m;
#pragma unroll
            for (int g = 0; g < 8; ++g) ext |= dtab[g][(m >> (4 * g)) & 15];
            m = ext;
        }
        if (__any_sync(0xFFFFFFFFu, m != 0)) {
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                const int e = (m >> (4 * g)) & 15;
                const uint4 v0 = *reinterpret_cast<const uint4*>(&tab[g][e][0]);
                const uint4 v1 = *reinterpret_cast<const uint4*>(&tab[g][e][4]);
                w[0] |= v0.x; w[1] |= v0.y; w[2] |= v0.z; w[3] |= v0.w;
                w[4] |= v1.x; w[5] |= v1.y; w[6] |= v1.z; w[7] |= v1.w;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < W; ++i) P[r * ld_w + i] = w[i];
}

__global__ void __launch_bounds__(B, 1) v0(const uint32_t* src, uint32_t* P, int ld_w) {
    const int r = threadIdx.x;
#pragma unroll
    for (int i = 0; i < W; ++i) P[r * ld_w + i] = src[r * ld_w + i];
}

__device__ __forceinline__ uint32_t close32_v6(uint32_t d) { return close32(d); }

// V6: V5 with 512 threads: thread t owns words [4h, 4h+4) of row t % 256,
// h = t / 256, so warp q (q < 4) or q + 4 (q >= 4)... holds the diagonal word
// of K_q for its 32 rows and runs the 32x32 closure directly.
__global__ void __launch_bounds__(2 * B, 1) v6(const uint32_t* src, uint32_t* P, int ld_w) {
    __shared__ __align__(16) uint32_t orig[32][W];
    __shared__ __align__(16) uint32_t tab[8][16][W];
    __shared__ uint32_t dtab[8][16];
    __shared__ uint32_t dp[32];
    __shared__ uint32_t mrow[B];   // each row's K_q word (original) for the other half
    const int t = threadIdx.x, r = t & (B - 1), h = t >> 8, warp = t >> 5, lane = t & 31;
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = src[r * ld_w + 4 * h + i];
#pragma unroll
    for (int q = 0; q < W; ++q) {
        const int hq = q >> 2, iq = q & 3;   // the half and slot holding word q
        const int wq = (hq << 3) + q;        // hmm: warp index of rows K_q in half hq: (hq*256 + 32q)/32
        (void)wq;
        const bool own = h == hq;            // this thread holds word q of its row
        if (own) mrow[r] = w[iq];
        // rows K_q: write their original 4 words into orig
        if ((r >> 5) == q) {
            *reinterpret_cast<uint4*>(&orig[r & 31][4 * h]) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        if (own && (r >> 5) == q) dp[r & 31] = 0;   // placeholder, closure below
        __syncthreads();
        if (warp == hq * 8 + q) {   // lanes = rows K_q, half hq: word q in slot iq
            dp[lane] = close32_v6(w[iq]);
        }
        __syncthreads();
        {
            const int g = t >> 6, e = (t >> 2) & 15, part = t & 3;   // 512 threads: (g,e) x 4 parts of 2 words
            uint2 acc = make_uint2(0, 0);
#pragma unroll
            for (int bit = 0; bit < 4; ++bit)
                if ((e >> bit) & 1) {
                    const uint2 v = *reinterpret_cast<const uint2*>(&orig[4 * g + bit][2 * part]);
                    acc.x |= v.x; acc.y |= v.y;
                }
            *reinterpret_cast<uint2*>(&tab[g][e][2 * part]) = acc;
            if (t < 128) {
                const int g2 = t >> 4, e2 = t & 15;
                uint32_t d = 0;
#pragma unroll
                for (int bit = 0; bit < 4; ++bit)
                    if ((e2 >> bit) & 1) d |= dp[4 * g2 + bit];
                dtab[g2][e2] = d;
            }
        }
        __syncthreads();
        uint32_t m = mrow[r];
        if ((r >> 5) == q) {
            m = dp[r & 31];
        } else if (m) {
            uint32_t ext = m;
#pragma unroll
            for (int g = 0; g < W; ++g) ext |= dtab[g][(m >> (4 * g)) & 15];
            m = ext;
        }
        if (__any_sync(0xFFFFFFFFu, m != 0)) {
#pragma unroll
            for (int g = 0; g < W; ++g) {
                const int e = (m >> (4 * g)) & 15;
                const uint4 v = *reinterpret_cast<const uint4*>(&tab[g][e][4 * h]);
                w[0] |= v.x; w[1] |= v.y; w[2] |= v.z; w[3] |= v.w;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) P[r * ld_w + 4 * h + i] = w[i];
}

static void cpu_ref(std::vector<uint32_t>& m, int ld_w) {
    for (int k = 0; k < B; ++k)
        for (int i = 0; i < B; ++i)
            if ((m[i * ld_w + k / 32] >> (k % 32)) & 1u)
                for (int x = 0; x < W; ++x) m[i * ld_w + x] |= m[k * ld_w + x];
}

template <typename F>
static float timeit(F f, int iters) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 10; ++i) f();
    cudaEventRecord(a);
    for (int i = 0; i < iters; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms * 1000.f / iters;
}

int main() {
    const int ld_w = 8;
    const double dens[] = {2.0 / 4096, 1.0 / 256, 4.0 / 256, 0.1};
    for (double d : dens) {
        std::vector<uint32_t> h(B * ld_w, 0);
        srand(7);
        for (int i = 0; i < B; ++i)
            for (int j = 0; j < B; ++j)
                if (rand() < d * RAND_MAX) h[i * ld_w + j / 32] |= 1u << (j % 32);
        std::vector<uint32_t> ref = h;
        cpu_ref(ref, ld_w);
        uint32_t *src, *dst;
        cudaMalloc(&src, h.size() * 4); cudaMalloc(&dst, h.size() * 4);
        cudaMemcpy(src, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
        auto check = [&](const char* name, float us) {
            std::vector<uint32_t> o(h.size());
            cudaMemcpy(o.data(), dst, o.size() * 4, cudaMemcpyDeviceToHost);
            printf("density %.5f %-10s %7.2f us  %s\n", d, name, us, o == ref ? "ok" : "MISMATCH");
        };
        timeit([&] { v0<<<1, B>>>(src, dst, ld_w); }, 200);
        printf("copy floor %.2f us\n", timeit([&] { v0<<<1, B>>>(src, dst, ld_w); }, 200));
        check("v1", timeit([&] { v1<<<1, B>>>(src, dst, ld_w); }, 200));
        check("v3sparse", timeit([&] { v3<true><<<1, B>>>(src, dst, ld_w); }, 200));
        check("v3full", timeit([&] { v3<false><<<1, B>>>(src, dst, ld_w); }, 200));
        check("v5", timeit([&] { v5<<<1, B>>>(src, dst, ld_w); }, 200));
        check("v6", timeit([&] { v6<<<1, 2 * B>>>(src, dst, ld_w); }, 200));
        cudaFree(src); cudaFree(dst);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
