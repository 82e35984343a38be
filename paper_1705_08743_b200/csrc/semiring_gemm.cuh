// Saturated semiring GEMM on CUDA cores: C = (acc ? C : I) (+) A (x) B.
//
// Replaces the outer-product sweeps _mul_vector / _minplus_mul_vector
// (pkg/src/semimat/antidist.py:361-371, :412-422).  The reference folds one
// candidate row per k; here every (i, j, k) cell-update is computed densely
// (the reference's zero-skip is an optimisation only: a skipped A entry is
// the (x)-annihilator and (+)-neutral, so including it changes nothing).
//
// Tiling (B200-first): a CTA owns a BM x BN output tile held in registers,
// TM rows x TNW words per thread.  Per k-tile of BK, A and B are read from
// HBM/L2 with 16-byte vector loads into registers (prefetched one k-tile
// ahead), converted to the canonical distance form and stored to a
// double-buffered shared-memory stage:
//   As[k][row] = {splat(a), splat(S - a)}  (or just splat(a) for u8)
//   Bs[k][word] = lane word of B
// so the inner loop is nothing but LDS.128 broadcasts and the 1- or
// 2-instruction lane update of semiring.cuh (the paper's SSE inner loop,
// P:351-375, one 32-bit word = 2 lanes wide, 32 threads x 4 SMSPs deep).
// Arithmetic intensity: BM*BN*BK cells per (BM + BN)*BK*elem bytes staged;
// the kernel is bound by packed-integer issue, not HBM.
#pragma once
#include <type_traits>

#include "semiring.cuh"

namespace smx {

template <typename T>
struct GemmArgs {
    const T* A;
    const T* B;
    T* C;
    int M, N, K;
    long long lda, ldb, ldc;
    int anti;
    int accumulate;
    int skip_tile0;   // first M-tile (in units of BM) to skip
    int skip_tiles;   // number of M-tiles skipped
    int allow_bounded;  // permit the verified 1-instruction k-tiles
    // Optional "sparse-bounded" row/column certificates (lane_flags_kernel):
    // rowflags[i] = every lane of A row i (k < K) is S or < 2^(w-2);
    // colflags[j] = the same for B column j.  A CTA whose rows, columns and
    // C tile are all certified runs every k-tile with the 1-instruction
    // update in a shifted encoding (see semiring_gemm_kernel).
    const uint8_t* rowflags;
    const uint8_t* colflags;
};

// Process-wide switch for the bounded 1-instruction k-tiles (on by default;
// smx_set_bounded_fastpath(0) forces the general 2-instruction form, for
// measurement and tests -- results are identical either way).
int bounded_fastpath_enabled();

template <typename T, int BM_, int BNW_, int BK_, int TM_, int TNW_, int MINB_>
struct GemmCfg {
    static constexpr int MINB = MINB_;
    using L = Lane<T>;
    static constexpr int BM = BM_, BNW = BNW_, BK = BK_, TM = TM_, TNW = TNW_;
    static constexpr int CPW = L::kCellsPerWord;
    static constexpr int BN = BNW * CPW;            // output cells per tile row
    static constexpr int E = L::kCellsPerChunk;     // cells per 16-byte chunk
    static constexpr int WPC = L::kWordsPerChunk;   // canonical words per chunk
    static constexpr int TCOLS = BNW / TNW;
    static constexpr int THREADS = (BM / TM) * TCOLS;
    static constexpr int HW = TNW / 2;              // words per half-group
    static constexpr int A_CPR = BK / E;            // A chunks per tile row
    static constexpr int A_CHUNKS = BM * A_CPR;
    static constexpr int A_PT = (A_CHUNKS + THREADS - 1) / THREADS;
    static constexpr int B_CPR = BNW / WPC;
    static constexpr int B_CHUNKS = BK * B_CPR;
    static constexpr int B_PT = (B_CHUNKS + THREADS - 1) / THREADS;
    // A is staged as planes: splat(a) and (2-instruction form only) splat(S-a),
    // so the bounded / one-instruction loop reads TM rows with one LDS.128.
    static constexpr int APLANES = L::kOneInstr ? 1 : 2;
    static constexpr size_t SMEM = 2ull * APLANES * BK * BM * 4 + 2ull * BK * BNW * 4;
    static_assert(TM == 2 || TM == 4, "A fragment is one 8- or 16-byte load per plane");
    static_assert(BK % E == 0, "BK must hold whole chunks");
    static_assert(BNW % WPC == 0, "BNW must hold whole chunks");
    static_assert(HW == 2 || HW == 4, "half-group must be 2 or 4 words");
};

// --- C row-group load/store (HW canonical words starting at cell gc) -------
template <typename T, int HW>
__device__ __forceinline__ void load_c_group(const T* crow, int gc, int N, bool anti,
                                             uint32_t* w) {
    using L = Lane<T>;
    constexpr int CELLS = HW * L::kCellsPerWord;
    const uint32_t m = anti ? 0xFFFFFFFFu : 0u;
    if (gc + CELLS <= N) {
        if constexpr (std::is_same<T, uint8_t>::value) {
            if constexpr (HW == 4) {
                uint2 v = *reinterpret_cast<const uint2*>(crow + gc);
                v.x ^= m; v.y ^= m;
                w[0] = __byte_perm(v.x, 0u, 0x4140); w[1] = __byte_perm(v.x, 0u, 0x4342);
                w[2] = __byte_perm(v.y, 0u, 0x4140); w[3] = __byte_perm(v.y, 0u, 0x4342);
            } else {
                uint32_t v = *reinterpret_cast<const uint32_t*>(crow + gc) ^ m;
                w[0] = __byte_perm(v, 0u, 0x4140); w[1] = __byte_perm(v, 0u, 0x4342);
            }
        } else {
            if constexpr (HW == 4) {
                uint4 v = *reinterpret_cast<const uint4*>(crow + gc);
                w[0] = v.x ^ m; w[1] = v.y ^ m; w[2] = v.z ^ m; w[3] = v.w ^ m;
            } else {
                uint2 v = *reinterpret_cast<const uint2*>(crow + gc);
                w[0] = v.x ^ m; w[1] = v.y ^ m;
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < HW; ++i) w[i] = L::kIdentityWord;
        for (int c = 0; c < CELLS; ++c) {
            if (gc + c >= N) break;
            uint32_t v = static_cast<uint32_t>(crow[gc + c]);
            v = anti ? (L::kS - v) : v;
            if (L::kCellsPerWord == 2) {
                const int wi = c >> 1, sh = (c & 1) * 16;
                w[wi] = (w[wi] & ~(0xFFFFu << sh)) | (v << sh);
            } else {
                w[c] = v;
            }
        }
    }
}

template <typename T, int HW>
__device__ __forceinline__ void store_c_group(T* crow, int gc, int N, bool anti,
                                              const uint32_t* w) {
    using L = Lane<T>;
    constexpr int CELLS = HW * L::kCellsPerWord;
    if (gc + CELLS <= N) {
        uint32_t o[HW];
        words_to_store<T, HW>(w, anti, o);
        if constexpr (std::is_same<T, uint8_t>::value) {
            if constexpr (HW == 4) *reinterpret_cast<uint2*>(crow + gc) = make_uint2(o[0], o[1]);
            else *reinterpret_cast<uint32_t*>(crow + gc) = o[0];
        } else {
            if constexpr (HW == 4)
                *reinterpret_cast<uint4*>(crow + gc) = make_uint4(o[0], o[1], o[2], o[3]);
            else *reinterpret_cast<uint2*>(crow + gc) = make_uint2(o[0], o[1]);
        }
    } else {
        for (int c = 0; c < CELLS; ++c) {
            if (gc + c >= N) break;
            uint32_t v = word_cell<T>(w, c);
            v = anti ? (L::kS - v) : v;
            crow[gc + c] = static_cast<T>(v);
        }
    }
}

// Raw 16-byte chunk loads (conversion to canonical words happens at the smem
// store, so staging costs 4 registers per chunk for every element type).
// Out-of-range cells read as the storage encoding of the (+)-identity:
// 0 for anti-distance, S (all ones) for distance.
template <typename T>
__device__ __forceinline__ uint4 identity_chunk(bool anti) {
    const uint32_t v = anti ? 0u : 0xFFFFFFFFu;
    return make_uint4(v, v, v, v);
}

template <typename Cfg, typename T>
__device__ __forceinline__ uint4 load_a_chunk(const GemmArgs<T>& p, int row0, int k0, int c) {
    const int r = c / Cfg::A_CPR, kc = c % Cfg::A_CPR;
    const int grow = row0 + r, gk = k0 + kc * Cfg::E;
    if (c < Cfg::A_CHUNKS && grow < p.M && gk < p.K) {
        uint4 raw = __ldg(reinterpret_cast<const uint4*>(p.A + (long long)grow * p.lda + gk));
        if (gk + Cfg::E > p.K) {   // chunk straddles K: cells >= K are identity
            const int valid = p.K - gk;
            const uint32_t id = p.anti ? 0u : 0xFFFFFFFFu;
            uint32_t v[4] = {raw.x, raw.y, raw.z, raw.w};
            constexpr int CPU = 4 / sizeof(T);   // cells per 32-bit storage word
#pragma unroll
            for (int j = 0; j < Cfg::E; ++j) {
                if (j >= valid) {
                    const int wi = j / CPU, sh = (j % CPU) * 8 * sizeof(T);
                    const uint32_t m = (sizeof(T) == 4) ? 0xFFFFFFFFu : (((1u << (8 * sizeof(T))) - 1u) << sh);
                    v[wi] = (v[wi] & ~m) | (id & m);
                }
            }
            raw = make_uint4(v[0], v[1], v[2], v[3]);
        }
        return raw;
    }
    return identity_chunk<T>(p.anti);
}

template <typename Cfg, typename T>
__device__ __forceinline__ uint4 load_b_chunk(const GemmArgs<T>& p, int col0, int k0, int c) {
    const int kr = c / Cfg::B_CPR, wc = c % Cfg::B_CPR;
    const int gk = k0 + kr, gc = col0 + wc * Cfg::E;
    if (c < Cfg::B_CHUNKS && gk < p.K && gc < p.N)
        return __ldg(reinterpret_cast<const uint4*>(p.B + (long long)gk * p.ldb + gc));
    return identity_chunk<T>(p.anti);
}

// CERT: instantiate the sparse-bounded certificate logic (only the certified
// public products use it; the Floyd-Warshall instantiation carries none of
// its registers or branches).
template <typename Cfg, typename T, bool CERT>
__device__ __forceinline__ void semiring_gemm_tile(const GemmArgs<T>& p, int bx, int by) {
    using L = Lane<T>;
    constexpr int BM = Cfg::BM, BNW = Cfg::BNW, BK = Cfg::BK, TM = Cfg::TM, TNW = Cfg::TNW;
    constexpr int HW = Cfg::HW, WPC = Cfg::WPC, E = Cfg::E, CPW = Cfg::CPW, AP = Cfg::APLANES;

    extern __shared__ uint4 smem_raw[];
    uint32_t* As = reinterpret_cast<uint32_t*>(smem_raw);     // [2][AP][BK][BM]
    uint32_t* Bs = As + 2 * AP * BK * BM;                     // [2][BK][BNW]

    const int tid = threadIdx.x;
    int mt = by;
    if (mt >= p.skip_tile0) mt += p.skip_tiles;
    const int row0 = mt * BM;
    const int col0 = bx * Cfg::BN;
    const bool anti = p.anti != 0;
    const int tc = tid % Cfg::TCOLS, tr = tid / Cfg::TCOLS;

    // ---- accumulator init: C (accumulate) or the (+)-identity ------------
    uint32_t acc[TM][TNW];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int grow = row0 + tr * TM + i;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            uint32_t* w = &acc[i][g * HW];
            if (p.accumulate && grow < p.M) {
                const int gc = col0 + (g * (BNW / 2) + tc * HW) * CPW;
                load_c_group<T, HW>(p.C + (long long)grow * p.ldc, gc, p.N, anti, w);
            } else {
#pragma unroll
                for (int j = 0; j < HW; ++j) w[j] = L::kIdentityWord;
            }
        }
    }

    // ---- sparse-bounded CTA: all A rows / B columns certified (S or small)
    // and the C tile too -> whole K loop in the shifted 1-instruction form.
    bool sparse = false;
    if constexpr (!L::kOneInstr && CERT) {
        if (p.rowflags != nullptr && p.allow_bounded) {
            bool ok = true;
            for (int i = tid; i < BM; i += Cfg::THREADS)
                if (row0 + i < p.M && !p.rowflags[row0 + i]) ok = false;
            for (int j = tid; j < Cfg::BN; j += Cfg::THREADS)
                if (col0 + j < p.N && !p.colflags[col0 + j]) ok = false;
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TNW; ++j) ok = ok && L::cert_ok(acc[i][j]);
            sparse = __syncthreads_and(ok);
            if (sparse) {
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TNW; ++j) acc[i][j] = L::to_shifted(acc[i][j]);
            }
        }
    }

    uint4 a_st[Cfg::A_PT];
    uint4 b_st[Cfg::B_PT];

    auto gload = [&](int k0) {
#pragma unroll
        for (int i = 0; i < Cfg::A_PT; ++i) a_st[i] = load_a_chunk<Cfg>(p, row0, k0, tid + i * Cfg::THREADS);
#pragma unroll
        for (int i = 0; i < Cfg::B_PT; ++i) b_st[i] = load_b_chunk<Cfg>(p, col0, k0, tid + i * Cfg::THREADS);
    };
    // sstore returns whether every staged lane of this thread is below the
    // half range (L::kHalfMask clear): if that holds for the whole CTA, no
    // a + b of this k-tile can reach S and the 1-instruction update is exact.
    auto sstore = [&](int buf) -> bool {
        uint32_t hi = 0;
#pragma unroll
        for (int i = 0; i < Cfg::A_PT; ++i) {
            const int c = tid + i * Cfg::THREADS;
            if (c < Cfg::A_CHUNKS) {
                const int r = c / Cfg::A_CPR, kc = c % Cfg::A_CPR;
                uint32_t* dst = As + (buf * AP * BK + kc * E) * BM + r;
                uint32_t w[WPC];
                chunk_to_words<T>(a_st[i], anti, w);
                if (sparse) {
#pragma unroll
                    for (int q = 0; q < WPC; ++q) w[q] = L::to_shifted(w[q]);
#pragma unroll
                    for (int j = 0; j < E; ++j) dst[j * BM] = L::splat(word_cell<T>(w, j));
                    continue;
                }
#pragma unroll
                for (int q = 0; q < WPC; ++q) hi |= w[q];
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    const uint32_t v = word_cell<T>(w, j);
                    dst[j * BM] = L::splat(v);
                    if constexpr (AP == 2) dst[BK * BM + j * BM] = L::splat(L::kS - v);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < Cfg::B_PT; ++i) {
            const int c = tid + i * Cfg::THREADS;
            if (c < Cfg::B_CHUNKS) {
                const int kr = c / Cfg::B_CPR, wc = c % Cfg::B_CPR;
                uint4* dst = reinterpret_cast<uint4*>(Bs + (buf * BK + kr) * BNW + wc * WPC);
                uint32_t w[WPC];
                chunk_to_words<T>(b_st[i], anti, w);
#pragma unroll
                for (int q = 0; q < WPC; ++q) {
                    hi |= w[q];
                    if (sparse) w[q] = L::to_shifted(w[q]);
                }
#pragma unroll
                for (int q = 0; q < WPC / 4; ++q)
                    dst[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
            }
        }
        return (hi & L::kHalfMask) == 0u;
    };

    // One k-tile of updates.  BOUNDED selects the 1-instruction form
    // c = min(c, a + b) (VIADDMNMX alone), exact when the CTA verified that all
    // lanes of both staged tiles are < 2^(w-1), so a + b < S never wraps and
    // never needs the S clamp (see semiring.cuh).
    auto ktile = [&](int buf, auto bounded_tag) {
        constexpr bool BOUNDED = decltype(bounded_tag)::value;
        const uint32_t* Ab = As + buf * AP * BK * BM + tr * TM;   // plane 0: splat(a)
        const uint32_t* Bb = Bs + buf * BK * BNW + tc * HW;
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            uint32_t b[TNW];
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                const uint32_t* src = Bb + kk * BNW + g * (BNW / 2);
                if constexpr (HW == 4) {
                    const uint4 v = *reinterpret_cast<const uint4*>(src);
                    b[g * 4 + 0] = v.x; b[g * 4 + 1] = v.y; b[g * 4 + 2] = v.z; b[g * 4 + 3] = v.w;
                } else {
                    const uint2 v = *reinterpret_cast<const uint2*>(src);
                    b[g * 2 + 0] = v.x; b[g * 2 + 1] = v.y;
                }
            }
            uint32_t a[TM], sa[TM];
            auto load_rows = [&](const uint32_t* src, uint32_t* dst) {
                if constexpr (TM == 4) {
                    const uint4 v = *reinterpret_cast<const uint4*>(src);
                    dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;
                } else {
                    const uint2 v = *reinterpret_cast<const uint2*>(src);
                    dst[0] = v.x; dst[1] = v.y;
                }
            };
            load_rows(Ab + kk * BM, a);
            if constexpr (!L::kOneInstr && !BOUNDED) load_rows(Ab + BK * BM + kk * BM, sa);
#pragma unroll
            for (int i = 0; i < TM; ++i) {
#pragma unroll
                for (int j = 0; j < TNW; ++j) {
                    if constexpr (L::kOneInstr) acc[i][j] = L::step(acc[i][j], b[j], a[i], 0u);
                    else if constexpr (BOUNDED) acc[i][j] = L::step_bounded(acc[i][j], b[j], a[i]);
                    else acc[i][j] = L::step(acc[i][j], b[j], a[i], sa[i]);
                }
            }
        }
    };

    const int nkt = (p.K + BK - 1) / BK;
    bool bounded = false;
    if (nkt > 0) {
        gload(0);
        bounded = __syncthreads_and(sstore(0)) && p.allow_bounded;
    }
    for (int kt = 0; kt < nkt; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nkt) gload((kt + 1) * BK);
        if constexpr (L::kOneInstr) {
            ktile(buf, std::false_type{});
        } else {
            if (bounded || sparse) ktile(buf, std::true_type{});
            else ktile(buf, std::false_type{});
        }
        bool ok = true;
        if (kt + 1 < nkt) ok = sstore(buf ^ 1);
        bounded = __syncthreads_and(ok) && p.allow_bounded;
    }

    // ---- epilogue ---------------------------------------------------------
    if constexpr (!L::kOneInstr) {
        if (sparse) {
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TNW; ++j) acc[i][j] = L::from_shifted(acc[i][j]);
        }
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int grow = row0 + tr * TM + i;
        if (grow >= p.M) continue;
        T* crow = p.C + (long long)grow * p.ldc;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const int gc = col0 + (g * (BNW / 2) + tc * HW) * CPW;
            store_c_group<T, HW>(crow, gc, p.N, anti, &acc[i][g * HW]);
        }
    }
}

template <typename Cfg, typename T, bool CERT>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) semiring_gemm_kernel(const GemmArgs<T> p) {
    semiring_gemm_tile<Cfg, T, CERT>(p, blockIdx.x, blockIdx.y);
}

// Two independent products in one launch (blockIdx.z selects the problem;
// the grid covers the larger one and the other's spare CTAs exit): the
// pivot recursion's pairs P12 (+)= P11* (x) P12 | P21 (+)= P21 (x) P11* and
// P21 (+)= P22* (x) P21 | P12 (+)= P12 (x) P22* (fw.cu fw_pivot_2x2).  On the
// look-ahead side stream every launch waits for SM slots beside phase-3 CTAs,
// so two launches cost about twice one (profiles/r02w_pivot_steps_contended.json).
template <typename Cfg, typename T>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
semiring_gemm_pair_kernel(const GemmArgs<T> p0, const GemmArgs<T> p1) {
    const bool second = blockIdx.z != 0;
    const int M = second ? p1.M : p0.M, N = second ? p1.N : p0.N;
    const int st = second ? p1.skip_tiles : p0.skip_tiles;
    if ((int)blockIdx.x >= (N + Cfg::BN - 1) / Cfg::BN || (int)blockIdx.y >= (M + Cfg::BM - 1) / Cfg::BM - st) return;
    if (second) semiring_gemm_tile<Cfg, T, false>(p1, blockIdx.x, blockIdx.y);
    else semiring_gemm_tile<Cfg, T, false>(p0, blockIdx.x, blockIdx.y);
}

// Tile configurations.  "Large" is the throughput tile: 128 x 128 cells
// (u8/u16; 128 x 64 for u32), 256 threads with 4-row x 8-word thread tiles,
// 2 CTAs per SM so one CTA's C load / store overlaps the other's k-loop (a
// measured 15-20% over one 512-thread 128 x 256 CTA per SM, which left the
// prologue/epilogue exposed and quantised C3's 512 tiles into 4 waves).
// "Small" keeps >= 2 waves on 148 SMs for thin products such as the FW
// pivot row panel (128 x n).
// (u8 stages k-tiles of 32: its 1-instruction loop halves the compute per
// staged byte, and the longer k-tile measured +4% on C3 u8; u16 is best at 16.)
template <typename T> using LargeCfg = GemmCfg<T, 128, 64, (sizeof(T) == 1 ? 32 : 16), 4, 8, 2>;
template <typename T> using SmallCfg = GemmCfg<T, 64, 64, 16, 4, 4, 2>;
// "Lite": 128 threads with 2 x 4-word thread tiles (~8K registers, 12 KB
// smem per CTA) -- small enough to run beside two Large CTAs on one SM, for
// the look-ahead side stream's pivot row panel while phase 3 fills the GPU.
template <typename T> using LiteCfg = GemmCfg<T, 32, 32, 16, 2, 4, 4>;

template <typename T>
int launch_large(const GemmArgs<T>& a, cudaStream_t stream);

template <typename Cfg, typename T>
int launch_semiring_gemm(const GemmArgs<T>& a, cudaStream_t stream) {
    if (a.rowflags != nullptr) {
        auto kern = semiring_gemm_kernel<Cfg, T, true>;
        SMX_TRY(set_max_smem((const void*)kern, Cfg::SMEM));
        const int mtiles = ceil_div(a.M, Cfg::BM) - a.skip_tiles;
        const int ntiles = ceil_div(a.N, Cfg::BN);
        if (mtiles <= 0 || ntiles <= 0) return SMX_OK;
        smx::count_launch();
        const cudaError_t e = launch_kernel(kern, dim3(ntiles, mtiles), dim3(Cfg::THREADS), Cfg::SMEM, stream, a);
        return e == cudaSuccess ? SMX_OK : (int)e;
    }
    auto kern = semiring_gemm_kernel<Cfg, T, false>;
    SMX_TRY(set_max_smem((const void*)kern, Cfg::SMEM));
    const int mtiles = ceil_div(a.M, Cfg::BM) - a.skip_tiles;
    const int ntiles = ceil_div(a.N, Cfg::BN);
    if (mtiles <= 0 || ntiles <= 0) return SMX_OK;
    dim3 grid(ntiles, mtiles);
    smx::count_launch();
    const cudaError_t e = launch_kernel(kern, grid, dim3(Cfg::THREADS), Cfg::SMEM, stream, a);
    return e == cudaSuccess ? SMX_OK : (int)e;
}

// ---- sparse-bounded certificates -------------------------------------------
// rowflags[i] (A, over k < K) and colflags[j] (B, over k < K): 1 iff every
// lane in distance form is S or < 2^(w-2) (Lane<T>::cert_ok).  One warp per A
// row (coalesced along k); one thread per 16-byte column chunk of B walking
// down its K rows (coalesced across threads).
template <typename T>
__global__ void lane_rowflags_kernel(const T* __restrict__ A, int M, int K, long long lda, bool anti,
                                     uint8_t* __restrict__ flags) {
    using L = Lane<T>;
    constexpr int E = L::kCellsPerChunk;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= M) return;
    const T* row = A + warp * lda;
    bool ok = true;
    for (int k = lane * E; k < K; k += 32 * E) {
        uint4 raw = __ldg(reinterpret_cast<const uint4*>(row + k));
        if (k + E > K) {   // cells >= K: identity (S), which certifies
            T* cells = reinterpret_cast<T*>(&raw);
            const T id = anti ? T(0) : T(L::kS);
            for (int j = K - k; j < E; ++j) cells[j] = id;
        }
        uint32_t w[Lane<T>::kWordsPerChunk];
        chunk_to_words<T>(raw, anti, w);
#pragma unroll
        for (int q = 0; q < Lane<T>::kWordsPerChunk; ++q) ok = ok && L::cert_ok(w[q]);
    }
    ok = __all_sync(0xFFFFFFFFu, ok);
    if (lane == 0) flags[warp] = ok ? 1 : 0;
}

// Column flags start at 1 (memset); each thread checks one 16-byte column
// chunk over a 64-row slice of K and clears the flags that fail (concurrent
// writers only ever store 0, so the race is benign).
constexpr int kColFlagSlice = 64;

template <typename T>
__global__ void lane_colflags_kernel(const T* __restrict__ B, int N, int K, long long ldb, bool anti,
                                     uint8_t* __restrict__ flags) {
    using L = Lane<T>;
    constexpr int E = L::kCellsPerChunk, WPC = L::kWordsPerChunk, CPW = L::kCellsPerWord;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c0 = (int)t * E;
    if (c0 >= N) return;
    const int k0 = blockIdx.y * kColFlagSlice, k1 = min(K, k0 + kColFlagSlice);
    bool ok[WPC];
#pragma unroll
    for (int q = 0; q < WPC; ++q) ok[q] = true;
#pragma unroll 4
    for (int k = k0; k < k1; ++k) {
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(B + k * ldb + c0));
        uint32_t w[WPC];
        chunk_to_words<T>(raw, anti, w);
#pragma unroll
        for (int q = 0; q < WPC; ++q) ok[q] = ok[q] && L::cert_ok(w[q]);
    }
    // per-word verdicts cover CPW cells each (u16: a pair of columns)
#pragma unroll
    for (int q = 0; q < WPC; ++q)
#pragma unroll
        for (int l = 0; l < CPW; ++l) {
            const int c = c0 + q * CPW + l;
            if (c < N && !ok[q]) flags[c] = 0;
        }
}

template <typename T>
int launch_lane_flags(const T* A, int M, int K, long long lda, const T* B, int N, long long ldb, bool anti,
                      uint8_t* rowflags, uint8_t* colflags, cudaStream_t s) {
    const long long rt = (long long)M * 32;
    lane_rowflags_kernel<T><<<(unsigned)((rt + 255) / 256), 256, 0, s>>>(A, M, K, lda, anti, rowflags);
    SMX_LAUNCHED_OR_RETURN();
    cudaError_t e = cudaMemsetAsync(colflags, 1, (size_t)N, s);
    if (e != cudaSuccess) return (int)e;
    const long long ct = (N + Lane<T>::kCellsPerChunk - 1) / Lane<T>::kCellsPerChunk;
    dim3 grid((unsigned)((ct + 127) / 128), (unsigned)((K + kColFlagSlice - 1) / kColFlagSlice));
    lane_colflags_kernel<T><<<grid, 128, 0, s>>>(B, N, K, ldb, anti, colflags);
    SMX_RETURN_LAUNCH();
}

// Stream-ordered scratch for the certificates (cudaMallocAsync from the
// device's default pool, kept cached by a high release threshold).
int scratch_alloc(void** p, size_t bytes, cudaStream_t s);
int scratch_free(void* p, cudaStream_t s);

// Certify only products large enough to amortise the flag pass.
inline bool worth_certifying(int M, int N, int K) {
    return (long long)M * N >= (1LL << 20) && K >= 64;
}

// Validates and dispatches one product; used by every entry point.
// `certify`: compute the sparse-bounded row/column certificates first (the
// public product entry points).  Floyd-Warshall's phase-3 calls leave it off:
// their tiles are almost all finite-and-small after the first rounds, where
// the per-k-tile bounded vote already applies, and the extra pass and CTA
// prologue measured -7% on the closure.
template <typename T>
int semiring_gemm(const T* A, const T* B, T* C, int M, int N, int K, long long lda,
                  long long ldb, long long ldc, int kind, int accumulate, int skip_row0,
                  int skip_rows, cudaStream_t stream, bool certify = false) {
    if (M < 0 || N < 0 || K < 0 || (kind != SMX_ANTI && kind != SMX_DIST)) return SMX_E_ARG;
    if (M == 0 || N == 0) return SMX_OK;
    if (!aligned16(A) || !aligned16(B) || !aligned16(C)) return SMX_E_ALIGN;
    if (!ld_ok(lda, sizeof(T)) || !ld_ok(ldb, sizeof(T)) || !ld_ok(ldc, sizeof(T)))
        return SMX_E_ALIGN;
    if (lda < K || ldb < N || ldc < N) return SMX_E_ARG;
    GemmArgs<T> a{A, B, C, M, N, K, lda, ldb, ldc, kind == SMX_ANTI, accumulate != 0, 0, 0,
                  bounded_fastpath_enabled(), nullptr, nullptr};
    // sparse-bounded certificates for u16/u32 products worth it
    void* flags = nullptr;
    if (certify && !Lane<T>::kOneInstr && a.allow_bounded && worth_certifying(M, N, K)) {
        if (scratch_alloc(&flags, (size_t)M + N, stream) == SMX_OK) {
            uint8_t* rf = reinterpret_cast<uint8_t*>(flags);
            SMX_TRY(launch_lane_flags<T>(A, M, K, lda, B, N, ldb, a.anti, rf, rf + M, stream));
            a.rowflags = rf;
            a.colflags = rf + M;
        }
    }
    struct FreeOnExit {
        void* p; cudaStream_t s;
        ~FreeOnExit() { if (p) scratch_free(p, s); }
    } guard{flags, stream};
    if (skip_rows > 0) {
        // skip ranges are whole 128-row tiles of the large config (FW phase 3)
        if (skip_row0 % LargeCfg<T>::BM) return SMX_E_ARG;
        a.skip_tile0 = skip_row0 / LargeCfg<T>::BM;
        a.skip_tiles = ceil_div(skip_rows, LargeCfg<T>::BM);
        const int total = ceil_div(M, LargeCfg<T>::BM);
        if (a.skip_tile0 + a.skip_tiles > total) a.skip_tiles = total - a.skip_tile0;
        if (a.skip_tiles < 0) return SMX_E_ARG;
        return launch_large<T>(a, stream);
    }
    const long long large_tiles = (long long)ceil_div(M, LargeCfg<T>::BM) * ceil_div(N, LargeCfg<T>::BN);
    const long long slots = 2LL * sm_count();   // Large runs 2 CTAs per SM
    // (A wave-tail split -- Large tiles for the rows filling whole waves,
    // Small tiles for the rest, as a second launch -- measured 10% slower on
    // C3: the second launch only starts after the first drains.)
    if (large_tiles < slots) return launch_semiring_gemm<SmallCfg<T>>(a, stream);
    return launch_large<T>(a, stream);
}

template <typename T>
int launch_large(const GemmArgs<T>& a, cudaStream_t stream) {
    return launch_semiring_gemm<LargeCfg<T>>(a, stream);
}

// Two independent accumulating products with Lite tiles in one launch
// (semiring_gemm_pair_kernel); each as semiring_gemm_lite.
template <typename T>
int semiring_gemm_lite_pair(const T* A0, const T* B0, T* C0, int M0, int N0, int K0, const T* A1, const T* B1,
                            T* C1, int M1, int N1, int K1, long long ld, int kind, cudaStream_t stream) {
    using Cfg = LiteCfg<T>;
    if (M0 < 0 || N0 < 0 || K0 < 0 || M1 < 0 || N1 < 0 || K1 < 0 || (kind != SMX_ANTI && kind != SMX_DIST))
        return SMX_E_ARG;
    for (const void* q : {(const void*)A0, (const void*)B0, (const void*)C0, (const void*)A1, (const void*)B1,
                          (const void*)C1})
        if (!aligned16(q)) return SMX_E_ALIGN;
    if (!ld_ok(ld, sizeof(T))) return SMX_E_ALIGN;
    GemmArgs<T> a0{A0, B0, C0, M0, N0, K0, ld, ld, ld, kind == SMX_ANTI, 1, 0, 0, bounded_fastpath_enabled(),
                   nullptr, nullptr};
    GemmArgs<T> a1{A1, B1, C1, M1, N1, K1, ld, ld, ld, kind == SMX_ANTI, 1, 0, 0, bounded_fastpath_enabled(),
                   nullptr, nullptr};
    const int mt = ceil_div(M0 > M1 ? M0 : M1, Cfg::BM), nt = ceil_div(N0 > N1 ? N0 : N1, Cfg::BN);
    if (mt <= 0 || nt <= 0) return SMX_OK;
    auto kern = semiring_gemm_pair_kernel<Cfg, T>;
    SMX_TRY(set_max_smem((const void*)kern, Cfg::SMEM));
    smx::count_launch();
    const cudaError_t e = launch_kernel(kern, dim3(nt, mt, 2), dim3(Cfg::THREADS), Cfg::SMEM, stream, a0, a1);
    return e == cudaSuccess ? SMX_OK : (int)e;
}

// Accumulating product with the co-residable Lite tiles (no row skip).
template <typename T>
int semiring_gemm_lite(const T* A, const T* B, T* C, int M, int N, int K, long long lda, long long ldb,
                       long long ldc, int kind, cudaStream_t stream) {
    if (M < 0 || N < 0 || K < 0 || (kind != SMX_ANTI && kind != SMX_DIST)) return SMX_E_ARG;
    if (M == 0 || N == 0) return SMX_OK;
    if (!aligned16(A) || !aligned16(B) || !aligned16(C)) return SMX_E_ALIGN;
    if (!ld_ok(lda, sizeof(T)) || !ld_ok(ldb, sizeof(T)) || !ld_ok(ldc, sizeof(T))) return SMX_E_ALIGN;
    GemmArgs<T> a{A, B, C, M, N, K, lda, ldb, ldc, kind == SMX_ANTI, 1, 0, 0, bounded_fastpath_enabled(),
                  nullptr, nullptr};
    return launch_semiring_gemm<LiteCfg<T>>(a, stream);
}

}  // namespace smx
