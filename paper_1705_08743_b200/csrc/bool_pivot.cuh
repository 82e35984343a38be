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
// the shared-memory traffic that bound the per-pivot version 4x.  Two
// barriers per sub-round: the next sub-round's pivot warp publishes its rows
// and closes its diagonal block during the other warps' fold.
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

// Close the b x b bit tile (b <= 32 W) held one row per thread in w[W]
// (row r = threadIdx.x, 32 W threads; bits beyond b already cleared), in
// place.  W = 8 (256-vertex tiles) or 16 (512).
template <int W>
struct PivotSmemT {
    uint32_t orig[32][W];
    uint32_t tab[8][16][W];
    uint32_t dtab[8][16];
    uint32_t dp[2][32];   // D+ of the current / next sub-round
};
using PivotSmem = PivotSmemT<8>;

// w[q] for a runtime q without dynamic register indexing (which would put w
// in local memory).
template <int W>
__device__ __forceinline__ uint32_t word_at(const uint32_t (&w)[W], int q) {
    uint32_t v = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) v = (i == q) ? w[i] : v;
    return v;
}

// Warp q publishes its rows (the sub-round's original pivot rows) and closes
// its 32 x 32 diagonal block.
template <int W>
__device__ __forceinline__ void publish_pivot_rows(const uint32_t (&w)[W], int q, PivotSmemT<W>& sm) {
    constexpr int PARTS = W / 4;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int p = 0; p < PARTS; ++p)
        *reinterpret_cast<uint4*>(&sm.orig[lane][4 * p]) = make_uint4(w[4 * p], w[4 * p + 1], w[4 * p + 2], w[4 * p + 3]);
    sm.dp[q & 1][lane] = close32(word_at<W>(w, q));
}

template <int W>
__device__ __forceinline__ void close_tile_bits(uint32_t (&w)[W], int b, PivotSmemT<W>& sm) {
    static_assert(W % 4 == 0, "rows are moved as uint4");
    constexpr int PARTS = W / 4;   // uint4 parts per table entry
    const int r = threadIdx.x, warp = r >> 5, lane = r & 31;
    const int nq = (b + 31) / 32;
    if (warp == 0) publish_pivot_rows<W>(w, 0, sm);
    __syncthreads();
    // not unrolled: the unrolled sub-rounds were ~19k instructions and the
    // kernel stalled on instruction fetch (ncu: "no instruction" the top stall)
#pragma unroll 1
    for (int q = 0; q < nq; ++q) {
        {
            // 128 table entries x PARTS uint4 parts = 32 W threads
            const int entry = r / PARTS, part = r % PARTS;
            const int g = entry >> 4, e = entry & 15;
            uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int bit = 0; bit < 4; ++bit)
                if ((e >> bit) & 1) {
                    const uint4 v = *reinterpret_cast<const uint4*>(&sm.orig[4 * g + bit][4 * part]);
                    acc.x |= v.x; acc.y |= v.y; acc.z |= v.z; acc.w |= v.w;
                }
            *reinterpret_cast<uint4*>(&sm.tab[g][e][4 * part]) = acc;
            if (r < 128) {
                const int g2 = r >> 4, e2 = r & 15;
                uint32_t d = 0;
#pragma unroll
                for (int bit = 0; bit < 4; ++bit)
                    if ((e2 >> bit) & 1) d |= sm.dp[q & 1][4 * g2 + bit];
                sm.dtab[g2][e2] = d;
            }
        }
        __syncthreads();
        uint32_t m = word_at<W>(w, q);
        if (warp == q) {
            m = sm.dp[q & 1][lane];
        } else if (m) {
            uint32_t ext = m;
#pragma unroll
            for (int g = 0; g < 8; ++g) ext |= sm.dtab[g][(m >> (4 * g)) & 15];
            m = ext;
        }
        if (__any_sync(0xFFFFFFFFu, m != 0)) {
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                const int e = (m >> (4 * g)) & 15;
#pragma unroll
                for (int p = 0; p < PARTS; ++p) {
                    const uint4 v = *reinterpret_cast<const uint4*>(&sm.tab[g][e][4 * p]);
                    w[4 * p] |= v.x; w[4 * p + 1] |= v.y; w[4 * p + 2] |= v.z; w[4 * p + 3] |= v.w;
                }
            }
        }
        // the next sub-round's pivot warp publishes right after its own fold,
        // while the other warps are still folding: the fold reads only tab /
        // dtab / dp[q & 1], and orig is read only before the barrier above
        if (warp == q + 1 && q + 1 < nq) publish_pivot_rows<W>(w, q + 1, sm);
        __syncthreads();
    }
}

}  // namespace smx
