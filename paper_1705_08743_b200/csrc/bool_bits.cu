// Boolean products and Warshall closure on bit-packed rows.
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

#include <atomic>

#include "common.cuh"
#include "bool_pivot.cuh"

namespace smx {

struct BitsArgs {
    const uint32_t* A;
    const uint32_t* B;
    uint32_t* C;
    int M, Nw, K;
    long long lda, ldb, ldc;   // in words
    int accumulate;
    int skip_tile0, skip_tiles;
    int kw_per;   // k-words per CTA (split-K when < ceil(K/32))
};

template <int BM_, int BNW_, int TM_, int TNW_, int MINB_>
struct BitsCfg {
    static constexpr int BM = BM_, BNW = BNW_, TM = TM_, TNW = TNW_, MINB = MINB_;
    static constexpr int HW = TNW / 2, TCOLS = BNW / TNW;
    static constexpr int THREADS = (BM / TM) * TCOLS;
    static constexpr int B_CHUNKS = 32 * BNW / 4;                  // uint4 per k-word stage
    static constexpr int B_PT = (B_CHUNKS + THREADS - 1) / THREADS;
    static_assert(HW == 4, "half-groups are one uint4");
};
using BitsLarge = BitsCfg<128, 64, 4, 8, 2>;   // 256 threads, 128 x 2048 bits
using BitsSmall = BitsCfg<64, 32, 2, 8, 2>;    // 128 threads, 64 x 1024 bits

template <typename Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) bool_bits_gemm_kernel(const BitsArgs p) {
    constexpr int BM = Cfg::BM, BNW = Cfg::BNW, TM = Cfg::TM, TNW = Cfg::TNW, HW = Cfg::HW;
    constexpr int TCOLS = Cfg::TCOLS, THREADS = Cfg::THREADS;
    __shared__ uint32_t As[2][BM];            // one A word (32 k) per row
    __shared__ __align__(16) uint32_t Bs[2][32][BNW];

    pdl_wait();   // PDL launches: the preceding kernel's output is read below
    const int tid = threadIdx.x;
    int mt = blockIdx.y;
    if (mt >= p.skip_tile0) mt += p.skip_tiles;
    const int row0 = mt * BM, w0 = blockIdx.x * BNW;
    const int tc = tid % TCOLS, tr = tid / TCOLS;

    // split-K: this CTA covers k-words [kw_lo, kw_hi); partial rows are OR-ed
    // into C with atomicOr (OR is idempotent: the merge is exact)
    const int nkw_all = (p.K + 31) / 32;
    const int kw_lo = blockIdx.z * p.kw_per;
    const int kw_hi = min(nkw_all, kw_lo + p.kw_per);
    const bool split = p.kw_per < nkw_all;

    uint32_t acc[TM][TNW];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int grow = row0 + tr * TM + i;
#pragma unroll
        for (int j = 0; j < TNW; ++j) {
            const int gw = w0 + (j / HW) * (BNW / 2) + tc * HW + (j % HW);
            acc[i][j] = (!split && p.accumulate && grow < p.M && gw < p.Nw)
                            ? p.C[(long long)grow * p.ldc + gw] : 0u;
        }
    }

    constexpr int A_PT = (BM + THREADS - 1) / THREADS;
    uint32_t a_st[A_PT];
    uint4 b_st[Cfg::B_PT];
    auto gload = [&](int kw) {  // kw: k-word index
        const int k0 = kw * 32;
#pragma unroll
        for (int q = 0; q < A_PT; ++q) {
            const int r = tid + q * THREADS, grow = row0 + r;
            uint32_t v = 0;
            if (r < BM && grow < p.M) {
                v = p.A[(long long)grow * p.lda + kw];
                const int valid = p.K - k0;
                if (valid < 32) v &= (1u << valid) - 1u;
            }
            a_st[q] = v;
        }
#pragma unroll
        for (int q = 0; q < Cfg::B_PT; ++q) {
            const int c = tid + q * THREADS;
            const int kr = c / (BNW / 4), wc = (c % (BNW / 4)) * 4;
            const int gk = k0 + kr, gw = w0 + wc;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (c < Cfg::B_CHUNKS && gk < p.K) {
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
#pragma unroll
        for (int q = 0; q < A_PT; ++q) {
            const int r = tid + q * THREADS;
            if (r < BM) As[buf][r] = a_st[q];
        }
#pragma unroll
        for (int q = 0; q < Cfg::B_PT; ++q) {
            const int c = tid + q * THREADS;
            if (c < Cfg::B_CHUNKS) {
                const int kr = c / (BNW / 4), wc = (c % (BNW / 4)) * 4;
                *reinterpret_cast<uint4*>(&Bs[buf][kr][wc]) = b_st[q];
            }
        }
    };

    if (kw_lo < kw_hi) { gload(kw_lo); sstore(0); __syncthreads(); }
    for (int kw = kw_lo; kw < kw_hi; ++kw) {
        const int buf = (kw - kw_lo) & 1;
        const int nkw = kw_hi;
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
            if (split) {
                for (int j = 0; j < 4; ++j)
                    if (gw + j < p.Nw && acc[i][g * 4 + j]) atomicOr(dst + j, acc[i][g * 4 + j]);
            } else if (gw + 4 <= p.Nw) {
                *reinterpret_cast<uint4*>(dst) = make_uint4(acc[i][g * 4], acc[i][g * 4 + 1],
                                                            acc[i][g * 4 + 2], acc[i][g * 4 + 3]);
            } else {
                for (int j = 0; j < 4; ++j)
                    if (gw + j < p.Nw) dst[j] = acc[i][g * 4 + j];
            }
        }
    }
}

// Method of four Russians (the paper's "sum of column-by-row outer products"
// taken four k at a time): per k-word stage the CTA builds, for each nibble
// g of the 32 k, the 16 ORs of subsets of B rows 4g..4g+3 (Tb[g][e]), and a
// row then ORs in one table entry per nibble -- 8 lookups for 32 k instead
// of a predicate test per k.  ALU work per 32 k per 8-word group: 8 x (1
// extract + 8 OR) against 32 x (1 test + 8 predicated OR).  Entries are
// stored with their 16-byte chunks rotated by e (chunk c at c ^ (e & 7)):
// threads reading different entries at the same columns then hit different
// banks.  Table build: each of 8 x BNW/4 work items loads 4 B rows x 4 words
// and writes the 16 entries of its columns.
template <typename Cfg>
struct M4rSmem {
    static constexpr int CH = Cfg::BNW / 4;                    // 16-byte chunks per entry
    static constexpr int ITEMS = 8 * CH;                       // (nibble, chunk) build items
    static constexpr int IT_PT = (ITEMS + Cfg::THREADS - 1) / Cfg::THREADS;
    static constexpr size_t TAB_WORDS = 8 * 16 * Cfg::BNW;
    static constexpr size_t BYTES = 2 * (TAB_WORDS * 4 + Cfg::BM * 4);
};

__device__ __forceinline__ int m4r_chunk(int c, int e, int nch) { return c ^ (e & (nch - 1) & 7); }

// Operand loads of the four-Russians tile.  CG = true reads through L2 only
// (ld.global.cg): the persistent Warshall kernel reads rows that other CTAs
// of the same launch have just OR-ed into, which a stale L1 line would miss.
template <bool CG>
__device__ __forceinline__ uint32_t m4r_ld(const uint32_t* p) {
    if constexpr (CG) return __ldcg(p);
    else return *p;
}
template <bool CG>
__device__ __forceinline__ uint4 m4r_ld4(const uint32_t* p) {
    if constexpr (CG) return __ldcg(reinterpret_cast<const uint4*>(p));
    else return *reinterpret_cast<const uint4*>(p);
}

// One output tile (row tile mt, word tile nt) over k-words [kw_lo, kw_hi):
// C |= A (x) B.  split: partial rows are OR-ed into C with atomics (other
// tiles cover the rest of K); otherwise the tile's C rows are read first
// (accumulate) and stored whole.
template <typename Cfg, bool CG>
__device__ __forceinline__ void m4r_tile(const BitsArgs& p, int mt, int nt, int kw_lo, int kw_hi, bool split,
                                         uint32_t* m4r_smem) {
    constexpr int BM = Cfg::BM, BNW = Cfg::BNW, TM = Cfg::TM, TNW = Cfg::TNW, HW = Cfg::HW;
    constexpr int TCOLS = Cfg::TCOLS, THREADS = Cfg::THREADS;
    using SM = M4rSmem<Cfg>;
    constexpr int CH = SM::CH;
    uint32_t* Tb = m4r_smem;                                  // [2][8][16][BNW]
    uint32_t* As = m4r_smem + 2 * SM::TAB_WORDS;              // [2][BM]

    const int tid = threadIdx.x;
    const int row0 = mt * BM, w0 = nt * BNW;
    const int tc = tid % TCOLS, tr = tid / TCOLS;

    uint32_t acc[TM][TNW];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int grow = row0 + tr * TM + i;
#pragma unroll
        for (int j = 0; j < TNW; ++j) {
            const int gw = w0 + (j / HW) * (BNW / 2) + tc * HW + (j % HW);
            acc[i][j] = (!split && p.accumulate && grow < p.M && gw < p.Nw)
                            ? m4r_ld<CG>(p.C + (long long)grow * p.ldc + gw) : 0u;
        }
    }

    constexpr int A_PT = (BM + THREADS - 1) / THREADS;
    uint32_t a_st[A_PT];
    uint4 b_st[SM::IT_PT][4];
    auto gload = [&](int kw) {
        const int k0 = kw * 32;
#pragma unroll
        for (int q = 0; q < A_PT; ++q) {
            const int r = tid + q * THREADS, grow = row0 + r;
            uint32_t v = 0;
            if (r < BM && grow < p.M) {
                v = m4r_ld<CG>(p.A + (long long)grow * p.lda + kw);
                const int valid = p.K - k0;
                if (valid < 32) v &= (1u << valid) - 1u;
            }
            a_st[q] = v;
        }
#pragma unroll
        for (int q = 0; q < SM::IT_PT; ++q) {
            const int it = tid + q * THREADS;
            const int g = it / CH, c = it % CH, gw = w0 + c * 4;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int gk = k0 + 4 * g + b;
                uint4 v = make_uint4(0, 0, 0, 0);
                if (it < SM::ITEMS && gk < p.K) {
                    const uint32_t* src = p.B + (long long)gk * p.ldb + gw;
                    if (gw + 4 <= p.Nw) v = m4r_ld4<CG>(src);
                    else {
                        if (gw + 0 < p.Nw) v.x = m4r_ld<CG>(src);
                        if (gw + 1 < p.Nw) v.y = m4r_ld<CG>(src + 1);
                        if (gw + 2 < p.Nw) v.z = m4r_ld<CG>(src + 2);
                    }
                }
                b_st[q][b] = v;
            }
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int q = 0; q < A_PT; ++q) {
            const int r = tid + q * THREADS;
            if (r < BM) As[buf * BM + r] = a_st[q];
        }
        uint32_t* tab = Tb + buf * SM::TAB_WORDS;
#pragma unroll
        for (int q = 0; q < SM::IT_PT; ++q) {
            const int it = tid + q * THREADS;
            if (it >= SM::ITEMS) break;
            const int g = it / CH, c = it % CH;
            // entries 0..7 from rows 0..2, then 8..15 = those | row 3 (8 live uint4)
            uint4 t[8];
            t[0] = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int e = 1; e < 8; ++e) {
                const int hb = e >= 4 ? 2 : (e >= 2 ? 1 : 0);   // highest set bit
                const uint4 lo = t[e ^ (1 << hb)], r = b_st[q][hb];
                t[e] = make_uint4(lo.x | r.x, lo.y | r.y, lo.z | r.z, lo.w | r.w);
            }
#pragma unroll
            for (int e = 0; e < 8; ++e)
                *reinterpret_cast<uint4*>(tab + (g * 16 + e) * BNW + m4r_chunk(c, e, CH) * 4) = t[e];
            const uint4 r3 = b_st[q][3];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint4 v = make_uint4(t[e].x | r3.x, t[e].y | r3.y, t[e].z | r3.z, t[e].w | r3.w);
                *reinterpret_cast<uint4*>(tab + (g * 16 + e + 8) * BNW + m4r_chunk(c, e + 8, CH) * 4) = v;
            }
        }
    };

    if (kw_lo < kw_hi) { gload(kw_lo); sstore(0); __syncthreads(); }
    for (int kw = kw_lo; kw < kw_hi; ++kw) {
        const int buf = (kw - kw_lo) & 1;
        if (kw + 1 < kw_hi) gload(kw + 1);
        const uint32_t* tab = Tb + buf * SM::TAB_WORDS;
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const uint32_t a = As[buf * BM + tr * TM + i];
            if (a == 0u) continue;
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                const int e = (a >> (4 * g)) & 15;
                const uint32_t* ent = tab + (g * 16 + e) * BNW;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int c = h * (CH / 2) + tc;
                    const uint4 v = *reinterpret_cast<const uint4*>(ent + m4r_chunk(c, e, CH) * 4);
                    acc[i][4 * h] |= v.x; acc[i][4 * h + 1] |= v.y; acc[i][4 * h + 2] |= v.z; acc[i][4 * h + 3] |= v.w;
                }
            }
        }
        if (kw + 1 < kw_hi) sstore(buf ^ 1);
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
            if (split) {
                for (int j = 0; j < 4; ++j)
                    if (gw + j < p.Nw && acc[i][g * 4 + j]) atomicOr(dst + j, acc[i][g * 4 + j]);
            } else if (gw + 4 <= p.Nw) {
                *reinterpret_cast<uint4*>(dst) = make_uint4(acc[i][g * 4], acc[i][g * 4 + 1],
                                                            acc[i][g * 4 + 2], acc[i][g * 4 + 3]);
            } else {
                for (int j = 0; j < 4; ++j)
                    if (gw + j < p.Nw) dst[j] = acc[i][g * 4 + j];
            }
        }
    }
}

template <typename Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) bool_m4r_gemm_kernel(const BitsArgs p) {
    extern __shared__ __align__(16) uint32_t m4r_smem[];
    pdl_wait();
    int mt = blockIdx.y;
    if (mt >= p.skip_tile0) mt += p.skip_tiles;
    const int nkw_all = (p.K + 31) / 32;
    const int kw_lo = blockIdx.z * p.kw_per;
    const int kw_hi = min(nkw_all, kw_lo + p.kw_per);
    m4r_tile<Cfg, false>(p, mt, blockIdx.x, kw_lo, kw_hi, p.kw_per < nkw_all, m4r_smem);
}

// smx_set_bits_m4r: the four-Russians bit GEMM (1, default) or the per-k
// predicate kernel (0).
static std::atomic<int> g_bits_m4r{1};

template <typename Cfg>
int launch_bits(const BitsArgs& a_in, cudaStream_t s) {
    BitsArgs a = a_in;
    const int mtiles = ceil_div(a.M, Cfg::BM) - a.skip_tiles;
    if (mtiles <= 0) return SMX_OK;
    const int ntiles = ceil_div(a.Nw, Cfg::BNW);
    const int nkw = ceil_div(a.K, 32);
    // Thin products (the 256-row pivot panels of Warshall) are K-latency
    // bound with a handful of CTAs: split K across CTAs and OR the partial
    // rows together with atomics.  Needs C pre-set (accumulate, or zeroed).
    int splits = 1;
    const int tiles = mtiles * ntiles;
    if (tiles < 2 * sm_count() && nkw >= 2) {
        splits = ceil_div(2 * sm_count(), tiles);
        if (splits > nkw) splits = nkw;
    }
    a.kw_per = ceil_div(nkw, splits);
    splits = nkw > 0 ? ceil_div(nkw, a.kw_per) : 1;
    if (splits > 1 && !a.accumulate) {
        cudaError_t e = cudaMemset2DAsync(a.C, (size_t)a.ldc * 4, 0, (size_t)a.Nw * 4, a.M, s);
        if (e != cudaSuccess) return (int)e;
    }
    dim3 grid(ntiles, mtiles, splits);
    smx::count_launch();
    if (g_bits_m4r.load(std::memory_order_relaxed)) {
        constexpr size_t smem = M4rSmem<Cfg>::BYTES;
        SMX_TRY(set_max_smem((const void*)bool_m4r_gemm_kernel<Cfg>, smem));
        const cudaError_t e = launch_kernel(bool_m4r_gemm_kernel<Cfg>, grid, dim3(Cfg::THREADS), smem, s, a);
        return e == cudaSuccess ? SMX_OK : (int)e;
    }
    const cudaError_t e = launch_kernel(bool_bits_gemm_kernel<Cfg>, grid, dim3(Cfg::THREADS), 0, s, a);
    return e == cudaSuccess ? SMX_OK : (int)e;
}

int bool_bits_gemm(const uint32_t* A, const uint32_t* B, uint32_t* C, int M, int Nw, int K,
                   long long lda, long long ldb, long long ldc, int accumulate, int skip_row0,
                   int skip_rows, cudaStream_t s) {
    if (M < 0 || Nw < 0 || K < 0) return SMX_E_ARG;
    if (M == 0 || Nw == 0) return SMX_OK;
    if (!aligned16(A) || !aligned16(B) || !aligned16(C)) return SMX_E_ALIGN;
    if ((ldb & 3) || (ldc & 3)) return SMX_E_ALIGN;
    if (lda * 32 < K || ldb < Nw || ldc < Nw) return SMX_E_ARG;
    BitsArgs a{A, B, C, M, Nw, K, lda, ldb, ldc, accumulate != 0, 0, 0, 0};
    const long long large_tiles = (long long)ceil_div(M, BitsLarge::BM) * ceil_div(Nw, BitsLarge::BNW);
    const bool large = large_tiles >= 2 * 148;
    const int bm = large ? BitsLarge::BM : BitsSmall::BM;
    if (skip_rows > 0) {
        if (skip_row0 % bm) return SMX_E_ARG;
        a.skip_tile0 = skip_row0 / bm;
        a.skip_tiles = ceil_div(skip_rows, bm);
        const int total = ceil_div(M, bm);
        if (a.skip_tile0 + a.skip_tiles > total) a.skip_tiles = total - a.skip_tile0;
    }
    return large ? launch_bits<BitsLarge>(a, s) : launch_bits<BitsSmall>(a, s);
}

// Warshall blocks: 256 vertices, or 512 for large n (kMaxWarshallBlock).
constexpr int kMaxWarshallBlock = 512;
#ifndef SMX_BOOL_BLOCK512_MIN_N
#define SMX_BOOL_BLOCK512_MIN_N 8192
#endif
constexpr int kBoolBlock512MinN = SMX_BOOL_BLOCK512_MIN_N;

template <int W>   // tile words per row: 8 (256 vertices) or 16 (512)
__global__ void __launch_bounds__(32 * W, 1) bool_pivot_kernel(uint32_t* P, int b, long long ld_w) {
    __shared__ __align__(16) PivotSmemT<W> sm;
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
    close_tile_bits<W>(w, b, sm);
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

static int launch_bool_pivot(uint32_t* P, int b, long long ld_w, cudaStream_t s) {
    count_launch();
    const cudaError_t e = b <= 128 ? launch_kernel(bool_pivot_kernel<4>, dim3(1), dim3(128), 0, s, P, b, ld_w)
                          : b <= kWarshallBlock
                              ? launch_kernel(bool_pivot_kernel<8>, dim3(1), dim3(256), 0, s, P, b, ld_w)
                              : launch_kernel(bool_pivot_kernel<16>, dim3(1), dim3(512), 0, s, P, b, ld_w);
    return e == cudaSuccess ? SMX_OK : (int)e;
}

// Block for an n-vertex closure.  Measured (ms, 256 / 512 blocks): n = 4096
// 0.33 / 0.46, 8192 1.79 / 1.51, 16384 10.1 / 10.1 -- halving the rounds pays
// once each round's phase 3 is long enough to hide the 512 pivot chain.
static int g_bool_block = 0;   // smx_set_bool_block: 0 = automatic, else 128 / 256 / 512
static int bool_block_for_n(int n) {
    if (g_bool_block) return g_bool_block;
    return n >= kBoolBlock512MinN ? 512 : kWarshallBlock;
}

// Column-panel snapshot of `cols` words for all rows (one thread per word).
__global__ void copy_words_kernel(const uint32_t* __restrict__ src, long long ld, uint32_t* __restrict__ dst,
                                  long long ldd, int rows, int cols) {
    pdl_wait();
    const long long total = (long long)rows * cols;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i / cols), c = (int)(i % cols);
        dst[r * ldd + c] = src[r * ld + c];
    }
}

int copy_words(const uint32_t* src, long long ld, uint32_t* dst, long long ldd, int rows, int cols,
               cudaStream_t s) {
    long long blocks = ((long long)rows * cols + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    count_launch();
    const cudaError_t e = launch_kernel(copy_words_kernel, dim3((unsigned)(blocks < 1 ? 1 : blocks)), dim3(256), 0,
                                        s, src, ld, dst, ldd, rows, cols);
    return e == cudaSuccess ? SMX_OK : (int)e;
}

// ---- persistent Warshall: the whole closure in one launch (n <= 8192) ---------
//
// The blocked schedule above is bound by its per-round chain at n = 4096
// (3a -> pivot -> row panel: three launches, ~15 us per round against ~4 us
// of phase-3 work).  Here one cooperative launch keeps every CTA resident and
// hands out work items from a global queue in schedule order; each item
// waits on device counters for exactly what it reads, so rounds overlap and
// no launch boundary sits on the chain:
//   RP(r)  row panel  T[K_r, :] |= P*_r . T[K_r, :]       waits pivot r
//   A3(r)  3a         T[K_r+1, :] |= T[K_r+1, K_r] . T[K_r, :]
//                                                          waits RP(r), 3b(r-1)
//   B3(r)  3b         T[X, :] |= T[X, K_r] . T[K_r, :], X = rows outside
//                     K_r u K_r+1                          waits RP(r), 3b(r-1)
//   pivot(r+1)        run by the CTA that completes the last A3(r) item
// Item g only waits on items with smaller indices (or the pivot run right
// after one of them), and all CTAs are co-resident, so the queue cannot
// deadlock.  Every read of T goes through L2 (m4r_tile<.., true>), partial
// products are OR-ed in with atomics where K is split, and items publish
// with __threadfence + a counter increment.  Exactness: the same in-place
// arguments as the blocked schedule (bits read after another item set them
// are real paths; P* . P* = P*).  tile: 64 rows x 2048 bits, 256 threads.
using BitsP = BitsCfg<64, 64, 2, 8, 1>;
constexpr int kPersistBlock = 256;
constexpr int kPersistMaxN = 8192;

struct PersistArgs {
    uint32_t* T;
    int n, nw;
    long long ld_w;
    int R, ntw;          // rounds; 2048-bit word tiles per row
    int ks_rp, ks_b;     // k-splits of the RP / A3 items and of the B3 items
    unsigned* ctr;       // [0] queue head, [1+r] pivot r done, [1+R+r] RP, [1+2R+r] A3, [1+3R+r] B3 done
    // development trace (smx_bool_persist_trace_arm; nullptr otherwise): per
    // item g, 4 u64 at [4 g]: start ns, dependencies met ns, end ns,
    // (cta << 32 | type << 16 | round); pivots in the last R slots
    unsigned long long* trace;
    int trace_cap;
};

__device__ __forceinline__ unsigned long long gtime_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_geq(const unsigned* p, unsigned v) {
    while (ld_acquire(p) < v) {
    }
}

__device__ __forceinline__ void persist_pivot(const PersistArgs& q, int k0, void* smem) {
    PivotSmemT<8>& sm = *reinterpret_cast<PivotSmemT<8>*>(smem);
    const int r = threadIdx.x;
    uint32_t w[8];
    const uint32_t* row = q.T + (long long)(k0 + r) * q.ld_w + k0 / 32;
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = __ldcg(row + i);
    __syncthreads();   // smem is reused from the last tile
    close_tile_bits<8>(w, kPersistBlock, sm);
    uint32_t* dst = q.T + (long long)(k0 + r) * q.ld_w + k0 / 32;
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[i] = w[i];
}

__global__ void __launch_bounds__(BitsP::THREADS, 1) bool_warshall_persistent_kernel(const PersistArgs q) {
    extern __shared__ __align__(16) uint32_t m4r_smem[];
    __shared__ int item;
    const int R = q.R, B = kPersistBlock;
    unsigned* piv = q.ctr + 1;
    unsigned* rp_done = q.ctr + 1 + R;
    unsigned* a_done = q.ctr + 1 + 2 * R;
    unsigned* b_done = q.ctr + 1 + 3 * R;
    const int tiles_k = B / BitsP::BM;                          // row tiles of one pivot block
    const int n_rp = tiles_k * q.ntw * q.ks_rp;
    const int rows_t = q.n / BitsP::BM;
    auto n_b = [&](int r) { return (rows_t - (r + 1 < R ? 2 : 1) * tiles_k) * q.ntw * q.ks_b; };
    auto n_a = [&](int r) { return r + 1 < R ? n_rp : 0; };
    const int nkw = B / 32;

    const bool tr = q.trace != nullptr && threadIdx.x == 0;
    if (blockIdx.x == 0) {   // pivot 0 before anything else
        if (tr) q.trace[4 * (q.trace_cap - R)] = gtime_ns();
        persist_pivot(q, 0, m4r_smem);
        if (tr) q.trace[4 * (q.trace_cap - R) + 2] = gtime_ns();
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicExch(&piv[0], 1u);
    }
    for (;;) {
        if (threadIdx.x == 0) item = (int)atomicAdd(&q.ctr[0], 1u);
        __syncthreads();
        int g = item;
        __syncthreads();
        const int g_all = g;
        unsigned long long t_start = tr ? gtime_ns() : 0;
        // queue order: RP(0) | A3(0) RP(1) B3(0) | A3(1) RP(2) B3(1) | ... | B3(R-1):
        // the chain's next row panel is handed out ahead of the bulk 3b
        // tiles, so CTAs are waiting for pivot r+1 when it lands
        int r = -1, type = -1;
        if (g < n_rp) { r = 0; type = 0; }
        else {
            g -= n_rp;
            for (int s = 0; s < R; ++s) {
                const int na = n_a(s), nr = s + 1 < R ? n_rp : 0, nb = n_b(s);
                if (g < na) { r = s; type = 1; break; }
                g -= na;
                if (g < nr) { r = s + 1; type = 0; break; }
                g -= nr;
                if (g < nb) { r = s; type = 2; break; }
                g -= nb;
            }
        }
        if (r < 0) return;
        const int k0 = r * B, k1 = k0 + B;
        // dependencies (thread 0 waits, the CTA follows)
        if (threadIdx.x == 0) {
            if (type == 0) wait_geq(&piv[r], 1u);
            else {
                wait_geq(&rp_done[r], (unsigned)n_rp);
                if (r > 0) wait_geq(&b_done[r - 1], (unsigned)n_b(r - 1));
            }
        }
        __syncthreads();
        unsigned long long t_ready = tr ? gtime_ns() : 0;
        const int ks = type == 2 ? q.ks_b : q.ks_rp;
        const int kc = g % ks, nt = (g / ks) % q.ntw, mi = g / (ks * q.ntw);
        const int kw_lo = kc * nkw / ks, kw_hi = (kc + 1) * nkw / ks;
        BitsArgs p{};
        p.Nw = q.nw; p.K = B; p.lda = p.ldb = p.ldc = q.ld_w; p.accumulate = 1;
        p.B = q.T + (long long)k0 * q.ld_w;
        int mt = mi;
        if (type == 0) {
            p.A = q.T + (long long)k0 * q.ld_w + k0 / 32; p.C = q.T + (long long)k0 * q.ld_w; p.M = B;
        } else if (type == 1) {
            p.A = q.T + (long long)k1 * q.ld_w + k0 / 32; p.C = q.T + (long long)k1 * q.ld_w; p.M = B;
        } else {
            p.A = q.T + k0 / 32; p.C = q.T; p.M = q.n;
            if (mt >= k0 / BitsP::BM) mt += (r + 1 < R ? 2 : 1) * tiles_k;   // skip K_r (u K_r+1)
        }
        m4r_tile<BitsP, true>(p, mt, nt, kw_lo, kw_hi, ks > 1, m4r_smem);
        __threadfence();
        __syncthreads();
        if (tr && g_all < q.trace_cap - R) {
            unsigned long long* e = q.trace + 4 * g_all;
            e[0] = t_start; e[1] = t_ready; e[2] = gtime_ns();
            e[3] = ((unsigned long long)blockIdx.x << 32) | ((unsigned long long)type << 16) | (unsigned)r;
        }
        if (type == 0) {
            if (threadIdx.x == 0) atomicAdd(&rp_done[r], 1u);
        } else if (type == 2) {
            if (threadIdx.x == 0) atomicAdd(&b_done[r], 1u);
        } else {
            __shared__ unsigned last;
            if (threadIdx.x == 0) last = atomicAdd(&a_done[r], 1u);
            __syncthreads();
            if (last + 1 == (unsigned)n_a(r)) {     // every A3(r) item is in: close pivot r+1
                __threadfence();
                if (tr) q.trace[4 * (q.trace_cap - R + r + 1)] = gtime_ns();
                persist_pivot(q, k1, m4r_smem);
                if (tr) q.trace[4 * (q.trace_cap - R + r + 1) + 2] = gtime_ns();
                __threadfence();
                __syncthreads();
                if (threadIdx.x == 0) atomicExch(&piv[r + 1], 1u);
            }
        }
    }
}

// Off by default: measured slower than the blocked schedule at every size
// (n = 2048 / 4096 / 8192: 0.156 / 0.30-0.40 / 1.33-1.96 ms against 0.128 /
// 0.250 / 0.85 ms; profiles/r02k_c2_persistent_trace.json).  The per-item
// timeline shows why: an item costs ~2.3 us of L2 round trips (operand
// loads through L2, atomics + fence) whatever its size, so the chain pivot
// (5 us) -> row panel -> 3a is no shorter than three PDL launches.
static std::atomic<int> g_bits_persistent{0};
static unsigned long long* g_persist_trace = nullptr;
static int g_persist_ks_rp = 8;
static int g_persist_trace_cap = 0;

inline size_t persist_ctr_bytes(int n) { return ((size_t)(1 + 4 * (n / kPersistBlock)) * 4 + 255) & ~size_t(255); }

// The persistent closure, when n fits it (n % 256 == 0, 512 <= n <= 8192).
static int bool_warshall_persistent(uint32_t* T, int n, long long ld_w, unsigned* ctr, cudaStream_t s) {
    constexpr size_t smem = M4rSmem<BitsP>::BYTES;
    static_assert(sizeof(PivotSmemT<8>) <= smem, "pivot smem aliases the tile tables");
    SMX_TRY(set_max_smem((const void*)bool_warshall_persistent_kernel, smem));
    int dev = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bool_warshall_persistent_kernel, BitsP::THREADS, smem);
    if (e != cudaSuccess) return (int)e;
    if (per_sm < 1) return SMX_E_ARG;
    const int grid = per_sm * sm_count();
    PersistArgs q{};
    q.T = T; q.n = n; q.nw = (n + 31) / 32; q.ld_w = ld_w; q.R = n / kPersistBlock;
    q.ntw = ceil_div(q.nw, BitsP::BNW);
    q.ks_rp = g_persist_ks_rp;
    const int b_tiles = (n / BitsP::BM - 2 * (kPersistBlock / BitsP::BM)) * q.ntw;
    q.ks_b = 1;
    while (q.ks_b < 8 && b_tiles * q.ks_b * 2 <= grid) q.ks_b *= 2;
    q.ctr = ctr;
    q.trace = g_persist_trace;
    q.trace_cap = g_persist_trace_cap;
    e = cudaMemsetAsync(ctr, 0, persist_ctr_bytes(n), s);
    if (e != cudaSuccess) return (int)e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(BitsP::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // every CTA resident: the queue's waits cannot deadlock
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    count_launch();
    e = cudaLaunchKernelEx(&cfg, bool_warshall_persistent_kernel, q);
    return e == cudaSuccess ? SMX_OK : (int)e;
}

inline size_t bits_ws_bytes(int n, long long ld_w) {
    const size_t rp = ((size_t)kMaxWarshallBlock * ld_w * 4 + 255) & ~size_t(255);
    const size_t cp = (size_t)n * (kMaxWarshallBlock / 32) * 4;
    return rp + ((cp + 255) & ~size_t(255)) + persist_ctr_bytes(n);
}

// -DSMX_DEV_BOOL_SKIP (tools/perf_c2_legs.py): timing experiments that leave
// out legs of the schedule by the mask in $SMX_DEV_BOOL_SKIP (1 = 3b, 2 =
// pivot, 4 = row panel, 8 = 3a).  Results are wrong; never in a normal build.
#ifdef SMX_DEV_BOOL_SKIP
#include <cstdlib>
static int dev_skip(int bit) {
    static const int mask = [] { const char* e = getenv("SMX_DEV_BOOL_SKIP"); return e ? atoi(e) : 0; }();
    return mask & bit;
}
#else
static constexpr int dev_skip(int) { return 0; }
#endif

// Pivot tile + pivot row panel of block [k0, k0 + bb).
static int bits_pivot_and_row_panel(uint32_t* T, int n, long long ld_w, uint32_t* RP, int k0, int bb,
                                    cudaStream_t s) {
    const int kw0 = k0 / 32, nw = (n + 31) / 32;
    uint32_t* rowK = T + (long long)k0 * ld_w;
    if (!dev_skip(2)) SMX_TRY(launch_bool_pivot(rowK + kw0, bb, ld_w, s));
    if (dev_skip(4)) return SMX_OK;
    PdlNext pdl;   // the row panel directly follows the pivot kernel
    // Row panel in place, no snapshot: T[K,:] |= P* . T[K,:] with P* = T[K,K]
    // closed.  A CTA may read rows K that another CTA has already OR-ed into;
    // those bits are paths through K, and P* . (T[K,:] | P* . T[K,:]) =
    // P* . T[K,:] because P* . P* = P*.  The P* tile itself is rewritten with
    // its own value.  So any interleaving gives the same result.
    (void)RP;
    return bool_bits_gemm(rowK + kw0, rowK, rowK, bb, nw, bb, ld_w, ld_w, ld_w, 1, 0, 0, s);
}

static int bool_warshall_schedule(uint32_t* T, int n, long long ld_w, uint32_t* RP, uint32_t* CP,
                                  cudaStream_t s);

// Same look-ahead schedule as fw_run_lookahead (fw.cu): pivot block r+1 is
// closed on the side stream while the bulk of round r's update runs.
int bool_warshall_bits(uint32_t* T, int n, long long ld_w, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (n < 0 || ld_w * 32 < n) return SMX_E_ARG;
    if (n == 0) return SMX_OK;
    if (!aligned16(T) || (ld_w & 3)) return SMX_E_ALIGN;
    if (n <= kWarshallBlock) return launch_bool_pivot(T, n, ld_w, s);
    if (ws == nullptr || ws_bytes < bits_ws_bytes(n, ld_w)) return SMX_E_WORKSPACE;
    uint32_t* RP = reinterpret_cast<uint32_t*>(ws);
    uint32_t* CP = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(ws) +
                                               (((size_t)kMaxWarshallBlock * ld_w * 4 + 255) & ~size_t(255)));
    unsigned* ctr = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(ws) + bits_ws_bytes(n, ld_w) -
                                                persist_ctr_bytes(n));
    const bool persist = g_bits_persistent.load() && n % kPersistBlock == 0 && n >= 2 * kPersistBlock &&
                         n <= kPersistMaxN && g_bits_m4r.load();
    GraphKey key;
    key.fn = 200;
    const unsigned long long kv[] = {(uintptr_t)T, (unsigned long long)n, (unsigned long long)ld_w,
                                     (uintptr_t)ws, ws_bytes, (unsigned long long)lookahead_enabled(),
                                     (unsigned long long)bool_block_for_n(n), (unsigned long long)g_bits_m4r.load(),
                                     (unsigned long long)persist};
    for (size_t i = 0; i < sizeof(kv) / sizeof(kv[0]); ++i) key.v[i] = kv[i];
    return run_graphed(key, s, false, [&](cudaStream_t st) -> int {
        if (persist) return bool_warshall_persistent(T, n, ld_w, ctr, st);
        return bool_warshall_schedule(T, n, ld_w, RP, CP, st);
    });
}

static int bool_warshall_schedule(uint32_t* T, int n, long long ld_w, uint32_t* RP, uint32_t* CP,
                                  cudaStream_t s) {
    // Phase 3 reads its A operand, the column panel T[:, K], straight from T:
    // the launch also ORs into T[:, K] (its j in K part), and a bit it reads
    // after another CTA set it is a real path through K, so the result is the
    // same for any interleaving (the row-panel argument of
    // bits_pivot_and_row_panel) -- no column-panel snapshot per round.
    (void)CP;
    const int nw = (n + 31) / 32;
    const int BLK = bool_block_for_n(n);
    const int R = (n + BLK - 1) / BLK;
    auto blk = [&](int r) { return n - r * BLK < BLK ? n - r * BLK : BLK; };

    if (!lookahead_enabled()) {
        for (int r = 0; r < R; ++r) {
            const int k0 = r * BLK, bb = blk(r), kw0 = k0 / 32;
            SMX_TRY(bits_pivot_and_row_panel(T, n, ld_w, RP, k0, bb, s));
            SMX_TRY(bool_bits_gemm(T + kw0, T + (long long)k0 * ld_w, T, n, nw, bb, ld_w, ld_w, ld_w, 1, k0, bb, s));
        }
        return SMX_OK;
    }
    SideStream* ss = nullptr;
    SMX_TRY(side_stream(&ss));
    cudaError_t e;
    SMX_TRY(bits_pivot_and_row_panel(T, n, ld_w, RP, 0, blk(0), s));
    for (int r = 0; r < R; ++r) {
        const int k0 = r * BLK, bb = blk(r), kw0 = k0 / 32;
        uint32_t* rowK = T + (long long)k0 * ld_w;
        if (r + 1 < R) {
            const int k1 = k0 + BLK, bb1 = blk(r + 1);
            // 3a: the next pivot block's rows
            if (!dev_skip(8))
                SMX_TRY(bool_bits_gemm(T + (long long)k1 * ld_w + kw0, rowK, T + (long long)k1 * ld_w, bb1, nw, bb,
                                       ld_w, ld_w, ld_w, 1, 0, 0, s));
            if ((e = cudaEventRecord(ss->fork, s)) != cudaSuccess) return (int)e;
            if ((e = cudaStreamWaitEvent(ss->side, ss->fork, 0)) != cudaSuccess) return (int)e;
            {
                PriorityScope ps(ss->priority);
                SMX_TRY(bits_pivot_and_row_panel(T, n, ld_w, RP, k1, bb1, ss->side));
            }
            if ((e = cudaEventRecord(ss->join, ss->side)) != cudaSuccess) return (int)e;
            // 3b: every other row (reads T[:, K_r] of rows outside K_r u K_{r+1}
            // only, which the side stream does not touch)
            if (!dev_skip(1))
                SMX_TRY(bool_bits_gemm(T + kw0, rowK, T, n, nw, bb, ld_w, ld_w, ld_w, 1, k0, bb + bb1, s));
            if ((e = cudaStreamWaitEvent(s, ss->join, 0)) != cudaSuccess) return (int)e;
        } else {
            SMX_TRY(bool_bits_gemm(T + kw0, rowK, T, n, nw, bb, ld_w, ld_w, ld_w, 1, k0, bb, s));
        }
    }
    return SMX_OK;
}

}  // namespace smx

using namespace smx;

extern "C" {

int smx_set_bits_m4r(int enable) {
    return g_bits_m4r.exchange(enable ? 1 : 0);
}

int smx_set_bool_block(int block) {
    if (block != 0 && block != 128 && block != 256 && block != 512) return SMX_E_ARG;
    const int old = g_bool_block;
    g_bool_block = block;
    return old;
}

int smx_set_bool_persistent(int enable) {
    return g_bits_persistent.exchange(enable ? 1 : 0);
}

// development: per-item trace of the persistent closure (see PersistArgs)
int smx_bool_persist_trace_arm(unsigned long long* buf, int cap_items) {
    if (cap_items < 0) {   // (development) k-split of the row-panel / 3a items: -1, -2, -4, -8
        g_persist_ks_rp = -cap_items;
        return SMX_OK;
    }
    g_persist_trace = buf;
    g_persist_trace_cap = buf ? cap_items : 0;
    return SMX_OK;
}

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
    return bool_warshall_bits(T, n, ld_w, ws, ws_bytes, as_stream(stream));
}

}  // extern "C"
