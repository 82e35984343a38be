// Boolean Warshall pivot tile: shared by the bit-packed closure (bool_bits.cu)
// and the byte/tensor-core closure (bool_tc.cu).
#pragma once
#include "common.cuh"

namespace smx {

// ---- Warshall pivot tile on bits ------------------------------------------
// b <= 256 rows of 8 words, one thread per row, closed in 8 sub-rounds of 32
// pivots K_q (boolmat.py:174-189 restricted to the tile).  Within a
// sub-round, sequential Warshall over K_q is equivalent to one fold:
//   D+   = transitive closure of the 32x32 diagonal block (5 warp squarings);
//   row_j |= OR_{k in m_j u m_j.D+} orig_row_k,   m_j = row j's K_q word
//   (rows of K_q themselves use m = D+).
// The fold reads nibble tables (method of four Russians): tab[g][e] is the OR
// of the original rows {4g+b : bit b of e}, dtab[g][e] the same over D+.  A
// row then needs 8 table entries instead of up to 32 pivot rows, which cuts
// the shared-memory traffic that bound the per-pivot version 4x.
constexpr int kWarshallBlock = 256;

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

// Close the b x b (b <= 256) bit tile held one row per thread in w[8]
// (row r = threadIdx.x; bits beyond b already cleared), in place.
struct PivotSmem {
    uint32_t orig[32][8];
    uint32_t tab[8][16][8];
    uint32_t dtab[8][16];
    uint32_t dp[32];
};

__device__ __forceinline__ void close_tile_bits(uint32_t (&w)[8], int b, PivotSmem& sm) {
    constexpr int W = kWarshallBlock / 32;
    const int r = threadIdx.x, warp = r >> 5, lane = r & 31;
#pragma unroll
    for (int q = 0; q < W; ++q) {
        if (q * 32 >= b) break;
        if (warp == q) {
            *reinterpret_cast<uint4*>(&sm.orig[lane][0]) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4*>(&sm.orig[lane][4]) = make_uint4(w[4], w[5], w[6], w[7]);
            sm.dp[lane] = close32(w[q]);
        }
        __syncthreads();
        {
            const int g = r >> 5, e = (r >> 1) & 15, h = r & 1;
            uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int bit = 0; bit < 4; ++bit)
                if ((e >> bit) & 1) {
                    const uint4 v = *reinterpret_cast<const uint4*>(&sm.orig[4 * g + bit][4 * h]);
                    acc.x |= v.x; acc.y |= v.y; acc.z |= v.z; acc.w |= v.w;
                }
            *reinterpret_cast<uint4*>(&sm.tab[g][e][4 * h]) = acc;
            if (r < 128) {
                const int g2 = r >> 4, e2 = r & 15;
                uint32_t d = 0;
#pragma unroll
                for (int bit = 0; bit < 4; ++bit)
                    if ((e2 >> bit) & 1) d |= sm.dp[4 * g2 + bit];
                sm.dtab[g2][e2] = d;
            }
        }
        __syncthreads();
        uint32_t m = w[q];
        if (warp == q) {
            m = sm.dp[lane];
        } else if (m) {
            uint32_t ext = m;
#pragma unroll
            for (int g = 0; g < W; ++g) ext |= sm.dtab[g][(m >> (4 * g)) & 15];
            m = ext;
        }
        if (__any_sync(0xFFFFFFFFu, m != 0)) {
#pragma unroll
            for (int g = 0; g < W; ++g) {
                const int e = (m >> (4 * g)) & 15;
                const uint4 v0 = *reinterpret_cast<const uint4*>(&sm.tab[g][e][0]);
                const uint4 v1 = *reinterpret_cast<const uint4*>(&sm.tab[g][e][4]);
                w[0] |= v0.x; w[1] |= v0.y; w[2] |= v0.z; w[3] |= v0.w;
                w[4] |= v1.x; w[5] |= v1.y; w[6] |= v1.z; w[7] |= v1.w;
            }
        }
        __syncthreads();
    }
}

}  // namespace smx
