// Warp-specialised u16 semiring GEMM over pre-packed operand tiles: the
// Floyd-Warshall phase-3 kernel (antidist.py:390-398 / :440-448 via fw.cu)
// and the large public u16 products (antidist.py:361-371 / :412-422).
//
// semiring_gemm_kernel (semiring_gemm.cuh) stages every k-tile through
// registers: each thread loads 16-byte chunks from global, converts them to
// the canonical form and splats A into shared memory, then the CTA votes on
// the k-tile's boundedness in a __syncthreads_and.  ncu on the n=32768 closure
// shows the ALU pipe 86% busy with long-scoreboard (0.84) and barrier (0.26)
// stalls left.  Phase 3 reuses each operand tile across a whole row or column
// of output tiles, so that per-tile conversion work is repeated 256 times.
//
// Here the conversion happens once per round (or once per product K-chunk),
// in two small pack kernels that write each 128 x BK A tile (splat words,
// [BK][BM]) and BK x 128 B tile (canonical words, [BK][BNW]) contiguously,
// together with a per-tile flag "every lane < 2^15" -- the bounded test,
// decided once per tile instead of voted per CTA.  Public products may
// instead be packed in the product-wide shifted encoding (cert_kernel).
// The GEMM runs one producer warp that streams tiles with 1-D bulk async
// copies (cp.async.bulk + mbarrier complete_tx) into a SMX_PACKED_STAGES ring
// of SMX_PACKED_BK-deep k-tiles (3 x 32 by default: 24 KB stages), and 8
// consumer warps that only wait, compute and arrive: no staging registers,
// no global loads and no CTA barrier in the k-loop.  The consumer's inner
// loop is the same LDS.128 + VIADDMNMX.U16x2 sequence (1 instruction per 2
// cells on bounded tiles, 2 otherwise; S - a of the general form is
// ~splat(a), 1 LOP per A value).  Measured: 95.9% ALU-pipe busy on a
// phase-3 launch at n = 32768 (profiles/r01g_ncu_fw32768_packed_3b.txt).
#pragma once
#include "semiring_gemm.cuh"

#ifndef SMX_PACKED_BK
#define SMX_PACKED_BK 32
#endif
#ifndef SMX_PACKED_STAGES
#define SMX_PACKED_STAGES 3
#endif
// C tile handling and residency.  Default: 3 CTAs per SM (72 registers,
// 73 KB of shared memory each) with C read from global in the epilogue -- the
// other two CTAs cover its latency.  SMX_PACKED_CSMEM=1 instead prefetches C
// into shared memory with bulk copies, which costs 32 KB and so the third CTA
// (2 CTAs/SM: 1.6% slower on the n=32768 closure).
#ifndef SMX_PACKED_CSMEM
#define SMX_PACKED_CSMEM 0
#endif
#ifndef SMX_PACKED_MINB
#define SMX_PACKED_MINB 3
#endif

namespace smx {

// T = uint16_t, or uint8_t widened to u16 lanes (Lane<uint8_t>: a + b <= 510
// cannot wrap and C starts <= 255, so every u8 tile takes the 1-instruction
// update).  The packed tiles hold the same u16x2 lane words for both.
// T = uint32_t: one cell per word (kernels.py:35), so the same 128 x 64-word
// tiles cover 128 x 64 cells; the update is VIADDMNMX (bounded / certified
// tiles) or IMNMX + VIADDMNMX (general), one or two instructions per cell.
template <typename T>
struct PackedCfg {
    static constexpr int BM = 128, BNW = 64, BK = SMX_PACKED_BK, TM = 4, TNW = 8, HW = 4;
    static constexpr int BN = Lane<T>::kCellsPerWord * BNW;   // cells
    static constexpr int TCOLS = BNW / TNW;            // 8
    static constexpr int CONSUMERS = (BM / TM) * TCOLS;  // 256
    static constexpr int THREADS = CONSUMERS + 32;     // + producer warp
    static constexpr int STAGES = SMX_PACKED_STAGES;
    static constexpr int A_TILE_WORDS = BK * BM;       // 4096 words = 16 KB
    static constexpr int B_TILE_WORDS = BK * BNW;      // 2048 words = 8 KB
    static constexpr int C_TILE_BYTES = BM * BN * (int)sizeof(T);
    static constexpr bool CSMEM = SMX_PACKED_CSMEM != 0;
    static constexpr int MINB = SMX_PACKED_MINB;
    static constexpr size_t SMEM =
        (size_t)STAGES * (A_TILE_WORDS + B_TILE_WORDS) * 4 + (CSMEM ? C_TILE_BYTES : 0) + 1024;
};
using PackedU16 = PackedCfg<uint16_t>;

template <typename T>
struct PackedArgsT {
    const uint32_t* Ap;    // [MT][KT][BK][BM] splat(canonical a)
    const uint32_t* Bp;    // [KT][NT][BK][BNW] canonical words
    const uint8_t* fA;     // [MT][KT]
    const uint8_t* fB;     // [KT][NT]
    T* C;
    int M, N, KT, NT;
    long long ldc;
    int anti, accumulate, allow_bounded;
    int row_tile0;                // first 128-row tile of the launch window
    int skip_tile0, skip_tiles;   // tiles skipped inside the window
    const int* cert;              // nullable: nonzero = operands packed in the shifted encoding
    int col_tile0;                // first output column tile of the launch (grid x counts from it)
    int mtiles;                   // row tiles of the launch (after the skipped ones)
    int backoff_ns;               // producer's free-slot wait (pk_mbar_wait_backoff)
};

// smx_set_packed_tiles_per_cta (abi.cu): output tiles per CTA of the packed
// GEMM (1 or 2).
int packed_tiles_per_cta();
// smx_set_packed_producer_backoff (abi.cu): see pk_mbar_wait_backoff.
int packed_producer_backoff();

// ---- pack kernels -----------------------------------------------------------
// Canonical (distance-form) lane value of one storage cell.
template <typename T>
__device__ __forceinline__ uint32_t canon_cell(T x, int anti) {
    return anti ? (Lane<T>::kS - (uint32_t)x) : (uint32_t)x;
}

// One CTA of 128 threads per A tile: thread r reads BK cells of row r (16-byte
// loads), writes BK splat words down column r of the tile.
template <typename T>
__global__ void __launch_bounds__(128) pack_a_kernel(const T* __restrict__ A, int M, int K, long long lda,
                                                    int anti, int KT, uint32_t* __restrict__ Ap,
                                                    uint8_t* __restrict__ fA, const int* __restrict__ cert,
                                                    int mt0 = 0) {
    using L = Lane<T>;
    using G = PackedCfg<T>;
    constexpr int BK = G::BK, E = L::kCellsPerChunk, WPC = L::kWordsPerChunk;
    const int kt = blockIdx.x, mt = mt0 + blockIdx.y, r = threadIdx.x;
    const int row = mt * G::BM + r, k0 = kt * BK;
    const bool sh = cert != nullptr && *cert != 0;
    uint32_t* dst = Ap + ((size_t)mt * KT + kt) * G::A_TILE_WORDS + r;
    uint32_t hi = 0;
#pragma unroll
    for (int q = 0; q < BK / E; ++q) {
        const int kq = k0 + q * E;
        uint32_t w[WPC];
        if (row < M && kq + E <= K) {
            chunk_to_words<T>(__ldg(reinterpret_cast<const uint4*>(A + (long long)row * lda + kq)), anti != 0, w);
        } else {
#pragma unroll
            for (int i = 0; i < WPC; ++i) w[i] = L::kIdentityWord;
            for (int j = 0; j < E; ++j) {
                if (row >= M || kq + j >= K) break;
                set_word_cell<T>(w, j, canon_cell<T>(A[(long long)row * lda + kq + j], anti));
            }
        }
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const uint32_t v = word_cell<T>(w, j);
            hi |= v;
            const uint32_t sw = L::splat(v);
            dst[(q * E + j) * G::BM] = sh ? L::to_shifted(sw) : sw;
        }
    }
    const int ok = __syncthreads_and((hi & L::kCellHalf) == 0u);
    if (r == 0) fA[(size_t)mt * KT + kt] = (uint8_t)ok;
}

// One CTA of 256 threads per B tile: each 16-byte chunk of a k-row becomes
// WPC canonical words; a k-row of the tile is 64 words.
template <typename T>
__global__ void __launch_bounds__(256) pack_b_kernel(const T* __restrict__ B, int K, int N, long long ldb,
                                                    int anti, int NT, uint32_t* __restrict__ Bp,
                                                    uint8_t* __restrict__ fB, const int* __restrict__ cert) {
    using L = Lane<T>;
    using G = PackedCfg<T>;
    constexpr int BK = G::BK, E = L::kCellsPerChunk, WPC = L::kWordsPerChunk;
    constexpr int CPR = G::BN / E;   // chunks per k-row
    const int nt = blockIdx.x, kt = blockIdx.y, t = threadIdx.x;
    const bool sh = cert != nullptr && *cert != 0;
    uint32_t hi = 0;
#pragma unroll
    for (int q = 0; q < (BK * CPR + 255) / 256; ++q) {
        const int ch = t + q * 256;
        if (ch >= BK * CPR) break;
        const int kk = ch / CPR, c = ch % CPR;
        const int k = kt * BK + kk, col = nt * G::BN + c * E;
        uint32_t w[WPC];
        if (k < K && col + E <= N) {
            chunk_to_words<T>(__ldg(reinterpret_cast<const uint4*>(B + (long long)k * ldb + col)), anti != 0, w);
        } else {
#pragma unroll
            for (int i = 0; i < WPC; ++i) w[i] = L::kIdentityWord;
            for (int j = 0; j < E; ++j) {
                if (k >= K || col + j >= N) break;
                set_word_cell<T>(w, j, canon_cell<T>(B[(long long)k * ldb + col + j], anti));
            }
        }
        uint32_t* dst = Bp + ((size_t)kt * NT + nt) * G::B_TILE_WORDS + kk * G::BNW + c * WPC;
#pragma unroll
        for (int i = 0; i < WPC; i += 4) {
            uint32_t o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                hi |= w[i + j] & L::kHalfMask;
                o[j] = sh ? L::to_shifted(w[i + j]) : w[i + j];
            }
            *reinterpret_cast<uint4*>(dst + i) = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
    const int ok = __syncthreads_and(hi == 0u);
    if (t == 0) fB[(size_t)kt * NT + nt] = (uint8_t)ok;
}

// ---- mbarrier / bulk-copy helpers --------------------------------------------
__device__ __forceinline__ uint32_t pk_smem(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void pk_mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(pk_smem(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void pk_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(pk_smem(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void pk_mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(pk_smem(bar)) : "memory");
}
__device__ __forceinline__ void pk_mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = pk_smem(bar);
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(addr), "r"(parity)
            : "memory");
    } while (!ok);
}
// 0xFFFF in each 16-bit lane whose sign bit is set (prmt's sign-replicate
// mode, selector msb; __byte_perm only takes the 3-bit byte indices).
__device__ __forceinline__ uint32_t pk_lane_sign_masks(uint32_t x) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %1, 0xbb99;" : "=r"(r) : "r"(x));
    return r;
}
// The producer's wait for a free ring slot.  It runs three stages ahead, so it
// always waits, and a bare try_wait loop issues SYNCS + BRA + YIELD every ~35
// cycles for the CTA's whole life (ncu at n = 8192: 11% of the kernel's warp
// instructions, on the consumers' issue slots).  ns > 0: try_wait with that
// suspend-time hint; ns < 0: nanosleep(-ns) between polls; 0: bare loop.
__device__ __forceinline__ void pk_mbar_wait_backoff(uint64_t* bar, uint32_t parity, int ns) {
    if (ns == 0) {
        pk_mbar_wait(bar, parity);
        return;
    }
    const uint32_t addr = pk_smem(bar);
    uint32_t ok = 0;
    for (;;) {
        if (ns > 0) {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(addr), "r"(parity), "r"((uint32_t)ns)
                : "memory");
        } else {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(addr), "r"(parity)
                : "memory");
        }
        if (ok) break;
        if (ns < 0) __nanosleep((unsigned)(-ns));
    }
}
__device__ __forceinline__ void pk_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            pk_smem(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(pk_smem(bar))
        : "memory");
}

// ---- the GEMM ------------------------------------------------------------------
// Accumulation order: the consumers start from the (+)-identity, run the K
// loop, and fold C in at the end (min is associative and commutative, so the
// result is bit-identical).  The producer prefetches an interior C tile into
// shared memory with row bulk copies while the K loop runs, so neither the C
// read latency nor the operand-flag reads sit on a warp's critical path.
// TPC: output tiles per CTA, walked in sequence through one continuous
// stage ring: the producer streams the next tile's first stages while the
// consumers fold and store the previous tile, so a tile's ring fill no longer
// sits between two tiles of the same CTA.  The tiles of a CTA are adjacent
// row tiles of one column tile (the same B tiles, hot in L2).
template <typename T, int TPC>
__global__ void __launch_bounds__(PackedCfg<T>::THREADS, PackedCfg<T>::MINB)
packed_gemm_kernel(const PackedArgsT<T> p) {
    using L = Lane<T>;
    using G = PackedCfg<T>;
    constexpr int BM = G::BM, BNW = G::BNW, BK = G::BK, TM = G::TM, TNW = G::TNW, HW = G::HW;
    constexpr int ST = G::STAGES;
    static_assert(TPC == 1 || !G::CSMEM, "the C-in-shared-memory variant runs one tile per CTA");

    extern __shared__ __align__(128) uint4 smem_raw[];
    uint32_t* As = reinterpret_cast<uint32_t*>(smem_raw);              // [ST][BK][BM]
    uint32_t* Bs = As + ST * G::A_TILE_WORDS;                          // [ST][BK][BNW]
    T* Cs = reinterpret_cast<T*>(Bs + ST * G::B_TILE_WORDS);   // [BM][BN] (raw C)
    uint64_t* full = reinterpret_cast<uint64_t*>(Cs + (G::CSMEM ? BM * G::BN : 0));
    uint64_t* empty = full + ST;
    uint64_t* cbar = empty + ST;
    uint32_t* flag = reinterpret_cast<uint32_t*>(cbar + 1);

    const int tid = threadIdx.x, lane = tid & 31;
    const int nt = p.col_tile0 + blockIdx.x;
    const int KT = p.KT;
    const int col0 = nt * G::BN;
    // this CTA's row tiles: compacted indices blockIdx.y * TPC + t of the
    // launch's p.mtiles (the skipped tiles excluded)
    int mts[TPC];
    int ntiles = 0;
#pragma unroll
    for (int t = 0; t < TPC; ++t) {
        const int idx = (int)blockIdx.y * TPC + t;
        int mt = p.row_tile0 + idx;
        if (mt >= p.skip_tile0) mt += p.skip_tiles;
        mts[t] = mt;
        if (idx < p.mtiles) ntiles = t + 1;
    }
    const bool c_async = G::CSMEM && p.accumulate && KT > 0 && mts[0] * BM + BM <= p.M && col0 + G::BN <= p.N;

    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            pk_mbar_init(&full[s], 1);
            pk_mbar_init(&empty[s], G::CONSUMERS / 32);
        }
        pk_mbar_init(cbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (tid >= G::CONSUMERS) {
        // ---- producer warp ----
        const int first = KT < ST ? KT : ST;
        auto issue = [&](int mt, int kt, int s) {
            pk_bulk_load(As + s * G::A_TILE_WORDS, p.Ap + ((size_t)mt * KT + kt) * G::A_TILE_WORDS,
                         G::A_TILE_WORDS * 4, &full[s]);
            pk_bulk_load(Bs + s * G::B_TILE_WORDS, p.Bp + ((size_t)kt * p.NT + nt) * G::B_TILE_WORDS,
                         G::B_TILE_WORDS * 4, &full[s]);
        };
        // The first ring fill goes out before the flag reads: a stage's
        // complete_tx may land before its expect_tx (the tx-count goes
        // transiently negative; the phase cannot complete until the arrive).
        if (lane == 0)
            for (int kt = 0; kt < first; ++kt) issue(mts[0], kt, kt);
        for (int t = 0; t < ntiles; ++t) {
            const int mt = mts[t];
            for (int kb = 0; kb < KT; kb += 32) {
                // bounded flags of 32 k-tiles in one round trip (one per lane)
                const int k = kb + lane;
                // (u8: always -- its update is the 1-instruction form)
                const bool f = k < KT && (L::kOneInstr || (p.allow_bounded &&
                               ((p.cert != nullptr && *p.cert != 0) ||
                                (p.fA[(size_t)mt * KT + k] != 0 && p.fB[(size_t)k * p.NT + nt] != 0))));
                const uint32_t fmask = __ballot_sync(0xFFFFFFFFu, f);
                if (lane == 0) {
                    const int kend = KT - kb < 32 ? KT : kb + 32;
                    for (int kt = kb; kt < kend; ++kt) {
                        const int g = t * KT + kt;          // position in the CTA's stage sequence
                        const int s = g % ST;
                        if (g >= ST) pk_mbar_wait_backoff(&empty[s], ((g / ST) - 1) & 1, p.backoff_ns);
                        flag[s] = (fmask >> (kt - kb)) & 1u;
                        pk_mbar_expect_tx(&full[s], (G::A_TILE_WORDS + G::B_TILE_WORDS) * 4);
                        if (g >= first) issue(mt, kt, s);
                        // the C tile goes behind the first ring fill, so the
                        // first operand tiles arrive first
                        if (c_async && g == first - 1) {
                            const int row0 = mt * BM;
                            pk_mbar_expect_tx(cbar, G::C_TILE_BYTES);
                            for (int r = 0; r < BM; ++r)
                                pk_bulk_load(Cs + r * G::BN, p.C + (long long)(row0 + r) * p.ldc + col0,
                                             G::BN * (int)sizeof(T), cbar);
                        }
                    }
                }
                __syncwarp();
            }
        }
        return;
    }

    const int tc = tid % G::TCOLS, tr = tid / G::TCOLS;
    const bool anti = p.anti != 0;

    for (int t = 0; t < ntiles; ++t) {
        const int row0 = mts[t] * BM;
        uint32_t acc[TM][TNW];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TNW; ++j) acc[i][j] = L::kIdentityWord;

        for (int kt = 0; kt < KT; ++kt) {
            const int g = t * KT + kt;
            const int s = g % ST;
            pk_mbar_wait(&full[s], (g / ST) & 1);
            const bool bounded = flag[s] != 0;
            const uint32_t* Ab = As + s * G::A_TILE_WORDS + tr * TM;
            const uint32_t* Bb = Bs + s * G::B_TILE_WORDS + tc * HW;
            if (bounded) {
#pragma unroll
                for (int kk = 0; kk < BK; ++kk) {
                    const uint4 b0 = *reinterpret_cast<const uint4*>(Bb + kk * BNW);
                    const uint4 b1 = *reinterpret_cast<const uint4*>(Bb + kk * BNW + BNW / 2);
                    const uint4 av = *reinterpret_cast<const uint4*>(Ab + kk * BM);
                    const uint32_t b[TNW] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                    const uint32_t a[TM] = {av.x, av.y, av.z, av.w};
#pragma unroll
                    for (int i = 0; i < TM; ++i)
#pragma unroll
                        for (int j = 0; j < TNW; ++j) acc[i][j] = L::step_bounded(acc[i][j], b[j], a[i]);
                }
            } else {
#pragma unroll
                for (int kk = 0; kk < BK; ++kk) {
                    const uint4 b0 = *reinterpret_cast<const uint4*>(Bb + kk * BNW);
                    const uint4 b1 = *reinterpret_cast<const uint4*>(Bb + kk * BNW + BNW / 2);
                    const uint4 av = *reinterpret_cast<const uint4*>(Ab + kk * BM);
                    const uint32_t b[TNW] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                    const uint32_t a[TM] = {av.x, av.y, av.z, av.w};
#pragma unroll
                    for (int i = 0; i < TM; ++i) {
                        const uint32_t sa = ~a[i];   // u16: splat(S - a), S = 0xFFFF per lane (u8: unused)
#pragma unroll
                        for (int j = 0; j < TNW; ++j) acc[i][j] = L::step(acc[i][j], b[j], a[i], sa);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) pk_mbar_arrive(&empty[s]);
        }

        // ---- fold C in and store ----
        // u16 accumulate launches (every phase-3 launch) fold in the storage
        // domain: storage = canonical ^ m (m = all ones for anti-distance), so
        // min over canonical lanes is max (anti) or min (dist) over storage
        // lanes and C needs no conversion either way.  The shifted encoding's
        // "lane >= S'" -> S is one add, one PRMT and one LOP3 per word: every
        // lane is <= 2 S' = 65534 after the first k-step, so lane + 1 cannot
        // carry into its neighbour and its sign bit is the test; PRMT 0xbb99
        // spreads the sign bits into lane masks.  (The generic form below
        // costs 7 instructions per word for from_shifted and 3 for the fold;
        // ncu at n = 8192: 4.3% of the ALU pipe's instructions.)
        const bool shifted = !L::kOneInstr && p.cert != nullptr && *p.cert != 0;
        bool done = false;
#ifndef SMX_PACKED_GENERIC_EPILOGUE   // (A/B and debugging: the generic fold below for every tile)
        if constexpr (std::is_same<T, uint16_t>::value && !G::CSMEM) {
            if (p.accumulate && KT > 0 && col0 + G::BN <= p.N) {
                const uint32_t m = anti ? 0xFFFFFFFFu : 0u;
                auto fold_rows = [&](auto sh) {
#pragma unroll
                    for (int i = 0; i < TM; ++i) {
                        const int grow = row0 + tr * TM + i;
                        if (grow >= p.M) continue;
                        T* crow = p.C + (long long)grow * p.ldc + col0;
#pragma unroll
                        for (int g = 0; g < 2; ++g) {
                            uint4* cp = reinterpret_cast<uint4*>(crow + (g * (BNW / 2) + tc * HW) * 2);
                            const uint4 v = *cp;
                            const uint32_t c[HW] = {v.x, v.y, v.z, v.w};
                            uint32_t o[HW];
#pragma unroll
                            for (int j = 0; j < HW; ++j) {
                                uint32_t x = acc[i][g * HW + j];
                                if (decltype(sh)::value) x |= pk_lane_sign_masks(x + 0x00010001u);
                                x ^= m;
                                o[j] = anti ? __vmaxu2(x, c[j]) : __vminu2(x, c[j]);
                            }
                            *cp = make_uint4(o[0], o[1], o[2], o[3]);
                        }
                    }
                };
                if (shifted) fold_rows(std::true_type{});
                else fold_rows(std::false_type{});
                done = true;
            }
        }
#endif
        if (!done) {
            if (shifted) {
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TNW; ++j) acc[i][j] = L::from_shifted(acc[i][j]);
            }
            if (c_async) pk_mbar_wait(cbar, 0);
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                const int grow = row0 + tr * TM + i;
                if (grow >= p.M) continue;
                T* crow = p.C + (long long)grow * p.ldc;
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    const int cc = (g * (BNW / 2) + tc * HW) * L::kCellsPerWord;   // cell offset in the tile
                    uint32_t* w = &acc[i][g * HW];
                    if (c_async || p.accumulate) {
                        uint32_t c[HW];
                        if (c_async) load_c_group<T, HW>(Cs + (tr * TM + i) * G::BN, cc, G::BN, anti, c);
                        else load_c_group<T, HW>(crow, col0 + cc, p.N, anti, c);
#pragma unroll
                        for (int j = 0; j < HW; ++j) w[j] = L::fold(w[j], c[j]);
                    }
                    store_c_group<T, HW>(crow, col0 + cc, p.N, anti, w);
                }
            }
        }
    }
}

// Workspace for one packed product of M x K by K x N (A tiles, B tiles, flags;
// the same for u8 and u16, which both pack u16x2 lane words; u32 B tiles
// cover half as many columns).
template <typename T>
inline size_t packed_ws_bytes_t(int M, int N, int K) {
    using G = PackedCfg<T>;
    const size_t MT = ceil_div(M, G::BM), NT = ceil_div(N, G::BN), KT = ceil_div(K, G::BK);
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    return al(MT * KT * G::A_TILE_WORDS * 4) + al(KT * NT * G::B_TILE_WORDS * 4) + al(MT * KT) + al(KT * NT);
}
inline size_t packed_ws_bytes(int M, int N, int K) { return packed_ws_bytes_t<uint16_t>(M, N, K); }
// A separate B-only block (B tiles + their flags): a second B operand beside
// the one in a packed workspace (the closure's double-buffered row panels).
template <typename T>
inline size_t packed_b_ws_bytes_t(int N, int K) {
    using G = PackedCfg<T>;
    const size_t NT = ceil_div(N, G::BN), KT = ceil_div(K, G::BK);
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    return al(KT * NT * G::B_TILE_WORDS * 4) + al(KT * NT);
}
inline size_t packed_b_ws_bytes_eb(int N, int K, int eb) {
    return eb == 4 ? packed_b_ws_bytes_t<uint32_t>(N, K) : packed_b_ws_bytes_t<uint16_t>(N, K);
}
inline size_t packed_u16_ws_bytes(int M, int N, int K) { return packed_ws_bytes(M, N, K); }
// by storage element bytes (1, 2: u16x2 lanes; 4: u32 lanes)
inline size_t packed_ws_bytes_eb(int M, int N, int K, int eb) {
    return eb == 4 ? packed_ws_bytes_t<uint32_t>(M, N, K) : packed_ws_bytes_t<uint16_t>(M, N, K);
}

// Views of a packed workspace laid out by packed_ws_bytes_t<T>(M, N, K).
struct PackedWs {
    uint32_t* Ap;
    uint32_t* Bp;
    uint8_t* fA;
    uint8_t* fB;
    int MT, NT, KT;
};
// wsb: a B-only block (packed_b_ws_bytes_t) that replaces the workspace's
// own B tiles and flags, or nullptr.
template <typename T>
inline PackedWs packed_views(void* ws, int M, int N, int K, void* wsb = nullptr) {
    using G = PackedCfg<T>;
    PackedWs v;
    v.MT = ceil_div(M, G::BM);
    v.NT = ceil_div(N, G::BN);
    v.KT = ceil_div(K, G::BK);
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    char* w = reinterpret_cast<char*>(ws);
    v.Ap = reinterpret_cast<uint32_t*>(w);
    w += al((size_t)v.MT * v.KT * G::A_TILE_WORDS * 4);
    v.Bp = reinterpret_cast<uint32_t*>(w);
    w += al((size_t)v.KT * v.NT * G::B_TILE_WORDS * 4);
    v.fA = reinterpret_cast<uint8_t*>(w);
    w += al((size_t)v.MT * v.KT);
    v.fB = reinterpret_cast<uint8_t*>(w);
    if (wsb != nullptr) {
        v.Bp = reinterpret_cast<uint32_t*>(wsb);
        v.fB = reinterpret_cast<uint8_t*>(wsb) + al((size_t)v.KT * v.NT * G::B_TILE_WORDS * 4);
    }
    return v;
}

template <typename T>
inline int packed_check(const void* A, const void* B, int M, int N, int K, long long lda, long long ldb, int kind,
                        void* ws, size_t ws_bytes) {
    if (M < 0 || N < 0 || K < 0 || (kind != SMX_ANTI && kind != SMX_DIST)) return SMX_E_ARG;
    if ((A && !aligned16(A)) || (B && !aligned16(B))) return SMX_E_ALIGN;
    if (!ld_ok(lda, sizeof(T)) || !ld_ok(ldb, sizeof(T))) return SMX_E_ALIGN;
    if (lda < K || ldb < N) return SMX_E_ARG;
    if (ws == nullptr || ws_bytes < packed_ws_bytes_t<T>(M, N, K)) return SMX_E_WORKSPACE;
    return SMX_OK;
}

// Pack A (M x K; A == nullptr skips it) and/or B (K x N; B == nullptr skips).
template <typename T>
inline int packed_pack(const T* A, const T* B, int M, int N, int K, long long lda, long long ldb, int kind, void* ws,
                       size_t ws_bytes, cudaStream_t s, const int* cert = nullptr, void* wsb = nullptr) {
    SMX_TRY(packed_check<T>(A, B, M, N, K, lda, ldb, kind, ws, ws_bytes));
    if (M == 0 || N == 0 || K == 0) return SMX_OK;
    const PackedWs v = packed_views<T>(ws, M, N, K, wsb);
    const int anti = kind == SMX_ANTI;
    if (A) {
        pack_a_kernel<T><<<dim3(v.KT, v.MT), 128, 0, s>>>(A, M, K, lda, anti, v.KT, v.Ap, v.fA, cert);
        SMX_LAUNCHED_OR_RETURN();
    }
    if (B) {
        pack_b_kernel<T><<<dim3(v.NT, v.KT), 256, 0, s>>>(B, K, N, ldb, anti, v.NT, v.Bp, v.fB, cert);
        SMX_LAUNCHED_OR_RETURN();
    }
    return SMX_OK;
}

// Pack only the A tiles of the 128-row tiles [tile0, tile0 + tiles) of an
// M x K operand (the workspace keeps the packed_ws_bytes(M, N, K) layout, so
// packed_run over the same row window reads them).  The host-streamed closure
// (fw.cu) packs just the rows it is about to update.
template <typename T>
inline int packed_pack_a_rows(const T* A, int M, int N, int K, long long lda, int kind, void* ws, size_t ws_bytes,
                              int tile0, int tiles, cudaStream_t s, const int* cert = nullptr) {
    SMX_TRY(packed_check<T>(A, nullptr, M, N, K, lda, lda, kind, ws, ws_bytes));   // (no B: ldb unused)
    if (M == 0 || N == 0 || K == 0) return SMX_OK;
    const PackedWs v = packed_views<T>(ws, M, N, K);
    if (tile0 < 0 || tile0 > v.MT) return SMX_E_ARG;
    if (tiles < 0 || tile0 + tiles > v.MT) tiles = v.MT - tile0;
    if (tiles == 0) return SMX_OK;
    pack_a_kernel<T><<<dim3(v.KT, tiles), 128, 0, s>>>(A, M, K, lda, kind == SMX_ANTI, v.KT, v.Ap, v.fA, cert,
                                                       tile0);
    SMX_RETURN_LAUNCH();
}

// C rows (+)= packed A (x) packed B over the 128-row tiles
// [row_tile0, row_tile0 + row_tiles) minus the rows [skip_row0, skip_row0 +
// skip_rows) (whole tiles, inside the window).  row_tiles < 0: to the end.
template <typename T>
inline int packed_run(T* C, int M, int N, int K, long long ldc, int kind, int accumulate, int row_tile0,
                      int row_tiles, int skip_row0, int skip_rows, void* ws, size_t ws_bytes, cudaStream_t s,
                      const int* cert = nullptr, int col_tile0 = 0, int col_tiles = -1, void* wsb = nullptr) {
    using G = PackedCfg<T>;
    if (M < 0 || N < 0 || K < 0 || (kind != SMX_ANTI && kind != SMX_DIST)) return SMX_E_ARG;
    if (M == 0 || N == 0) return SMX_OK;
    if (!aligned16(C) || !ld_ok(ldc, sizeof(T))) return SMX_E_ALIGN;
    if (ldc < N) return SMX_E_ARG;
    if (ws == nullptr || ws_bytes < packed_ws_bytes_t<T>(M, N, K)) return SMX_E_WORKSPACE;
    const PackedWs v = packed_views<T>(ws, M, N, K, wsb);
    if (row_tile0 < 0 || row_tile0 > v.MT) return SMX_E_ARG;
    if (row_tiles < 0 || row_tile0 + row_tiles > v.MT) row_tiles = v.MT - row_tile0;
    if (col_tile0 < 0 || col_tile0 > v.NT) return SMX_E_ARG;
    if (col_tiles < 0 || col_tile0 + col_tiles > v.NT) col_tiles = v.NT - col_tile0;
    if (col_tiles == 0) return SMX_OK;
    PackedArgsT<T> a{v.Ap, v.Bp, v.fA, v.fB, C, M, N, v.KT, v.NT, ldc, kind == SMX_ANTI, accumulate != 0,
                     bounded_fastpath_enabled(), row_tile0, v.MT, 0, cert, col_tile0};
    if (skip_rows > 0) {
        if (skip_row0 % G::BM) return SMX_E_ARG;
        a.skip_tile0 = skip_row0 / G::BM;
        a.skip_tiles = ceil_div(skip_rows, G::BM);
        if (a.skip_tile0 < row_tile0 || a.skip_tile0 > row_tile0 + row_tiles) return SMX_E_ARG;
        if (a.skip_tile0 + a.skip_tiles > row_tile0 + row_tiles) a.skip_tiles = row_tile0 + row_tiles - a.skip_tile0;
    }
    const int mtiles = row_tiles - a.skip_tiles;
    if (mtiles <= 0) return SMX_OK;
    a.mtiles = mtiles;
    a.backoff_ns = packed_producer_backoff();
    const int tpc = packed_tiles_per_cta();
    // launch_kernel: a launch on the look-ahead side stream (3a) carries the
    // side stream's priority into a captured graph (PriorityScope)
    // (a plain launch: carrying the side stream's priority into the replay
    // graph for the look-ahead's 3a measured no different, 17.51 vs 17.54 ms
    // at n = 8192)
    if (tpc == 2 && !G::CSMEM) {
        SMX_TRY(set_max_smem((const void*)packed_gemm_kernel<T, 2>, G::SMEM));
        packed_gemm_kernel<T, 2><<<dim3(col_tiles, (mtiles + 1) / 2), G::THREADS, G::SMEM, s>>>(a);
    } else {
        SMX_TRY(set_max_smem((const void*)packed_gemm_kernel<T, 1>, G::SMEM));
        packed_gemm_kernel<T, 1><<<dim3(col_tiles, mtiles), G::THREADS, G::SMEM, s>>>(a);
    }
    SMX_RETURN_LAUNCH();
}

// C (+)= A (x) B, rows [skip_row0, skip_row0 + skip_rows) left untouched
// (whole 128-row tiles).  ws: packed_ws_bytes(M, N, K).
template <typename T>
inline int semiring_gemm_packed(const T* A, const T* B, T* C, int M, int N, int K, long long lda, long long ldb,
                                long long ldc, int kind, int accumulate, int skip_row0, int skip_rows, void* ws,
                                size_t ws_bytes, cudaStream_t s) {
    if (A == nullptr || B == nullptr) return SMX_E_ARG;
    if (M == 0 || N == 0) return SMX_OK;
    SMX_TRY(packed_pack<T>(A, B, M, N, K, lda, ldb, kind, ws, ws_bytes, s));
    return packed_run<T>(C, M, N, K, ldc, kind, accumulate, 0, -1, skip_row0, skip_rows, ws, ws_bytes, s);
}

// u16 spellings used by fw.cu
inline int packed_u16_pack(const uint16_t* A, const uint16_t* B, int M, int N, int K, long long lda, long long ldb,
                           int kind, void* ws, size_t ws_bytes, cudaStream_t s, const int* cert = nullptr) {
    return packed_pack<uint16_t>(A, B, M, N, K, lda, ldb, kind, ws, ws_bytes, s, cert);
}
inline int packed_u16_run(uint16_t* C, int M, int N, int K, long long ldc, int kind, int accumulate, int row_tile0,
                          int row_tiles, int skip_row0, int skip_rows, void* ws, size_t ws_bytes, cudaStream_t s,
                          const int* cert = nullptr) {
    return packed_run<uint16_t>(C, M, N, K, ldc, kind, accumulate, row_tile0, row_tiles, skip_row0, skip_rows, ws,
                                ws_bytes, s, cert);
}
inline int semiring_gemm_packed_u16(const uint16_t* A, const uint16_t* B, uint16_t* C, int M, int N, int K,
                                    long long lda, long long ldb, long long ldc, int kind, int accumulate,
                                    int skip_row0, int skip_rows, void* ws, size_t ws_bytes, cudaStream_t s) {
    return semiring_gemm_packed<uint16_t>(A, B, C, M, N, K, lda, ldb, ldc, kind, accumulate, skip_row0, skip_rows,
                                          ws, ws_bytes, s);
}

// Global sparse-bounded certificate of a u16 / u32 operand (rows x cols, ld):
template <typename T>
__device__ __forceinline__ bool cert_operand(const T* __restrict__ X, int rows, int cols, long long ld, uint32_t m,
                                             long long i0, long long stride) {
    using L = Lane<T>;
    constexpr int E = 16 / (int)sizeof(T);
    const int cpr = (cols + E - 1) / E;
    const long long total = (long long)rows * cpr;
    bool ok = true;
    if (i0 >= total) return ok;
    // (row, chunk) walked incrementally: one division per thread, not per chunk
    long long r = i0 / cpr;
    int c = (int)(i0 - r * cpr);
    const long long dr = stride / cpr;
    const int dc = (int)(stride - dr * cpr);
    for (long long i = i0; i < total; i += stride) {
        uint4 w = __ldg(reinterpret_cast<const uint4*>(X + r * ld + (long long)c * E));
        w.x ^= m; w.y ^= m; w.z ^= m; w.w ^= m;
        if ((c + 1) * E > cols) {   // cells >= cols: identity (S), which certifies
            uint32_t e[4] = {w.x, w.y, w.z, w.w};
            for (int j = cols - c * E; j < E; ++j) set_word_cell<T>(e, j, L::kS);
            w = make_uint4(e[0], e[1], e[2], e[3]);
        }
        ok = ok && L::cert_ok(w.x) && L::cert_ok(w.y) && L::cert_ok(w.z) && L::cert_ok(w.w);
        c += dc;
        r += dr;
        if (c >= cpr) { c -= cpr; ++r; }
    }
    return ok;
}

// clears *cert if any lane in distance form is neither S nor < 2^14 (u16) /
// 2^30 (u32) (Lane::cert_ok).  Concurrent writers only store 0.  One launch
// covers both operands: blocks [0, gridDim.x / 2) read X, the rest Y.
template <typename T>
__global__ void __launch_bounds__(256) cert_kernel(const T* __restrict__ X, int xr, int xc, long long ldx,
                                                   const T* __restrict__ Y, int yr, int yc, long long ldy, int anti,
                                                   int* __restrict__ cert) {
    const uint32_t m = anti ? 0xFFFFFFFFu : 0u;
    const bool second = Y != nullptr && blockIdx.x >= gridDim.x / 2;
    const int nblk = Y != nullptr ? gridDim.x / 2 : gridDim.x;
    const int bx = second ? blockIdx.x - nblk : blockIdx.x;
    const long long i0 = (long long)bx * blockDim.x + threadIdx.x, stride = (long long)nblk * blockDim.x;
    const bool ok = second ? cert_operand<T>(Y, yr, yc, ldy, m, i0, stride)
                           : (X == nullptr || cert_operand<T>(X, xr, xc, ldx, m, i0, stride));
    if (!__all_sync(0xFFFFFFFFu, ok) && (threadIdx.x & 31) == 0) *cert = 0;
}

// Reset *cert and run the certificate over an operand pair (either may be
// nullptr) in one launch: the caller's packs and products then read *cert.
template <typename T>
inline int run_cert(const T* X, int xr, int xc, long long ldx, const T* Y, int yr, int yc, long long ldy, int anti,
                    int* cert, cudaStream_t s) {
    static_assert(sizeof(T) >= 2, "u8 is always the 1-instruction form");
    cudaError_t e = cudaMemsetAsync(cert, 0xFF, sizeof(int), s);
    if (e != cudaSuccess) return (int)e;
    if (X == nullptr && Y == nullptr) return SMX_OK;
    if (X == nullptr) { X = Y; xr = yr; xc = yc; ldx = ldy; Y = nullptr; }
    const int per = 4 * sm_count();
    cert_kernel<T><<<Y ? 2 * per : per, 256, 0, s>>>(X, xr, xc, ldx, Y, yr, yc, ldy, anti, cert);
    SMX_RETURN_LAUNCH();
}

// Public u16 product on the packed kernel.  K is processed in chunks so the
// packed operands stay <= ~384 MB of stream-ordered scratch; a certificate
// pass first decides, for the whole product, whether the operands can be
// packed in the shifted 1-instruction encoding (semiring.cuh, Lane<uint16_t>):
// then every k-tile runs VIADDMNMX alone, and results map back to S before C
// is folded in.  Otherwise tiles use the per-tile bounded flags.
template <typename T>
inline int semiring_gemm_packed_public(const T* A, const T* B, T* C, int M, int N, int K, long long lda,
                                       long long ldb, long long ldc, int kind, int accumulate, cudaStream_t s) {
    using G = PackedCfg<T>;
    if (M < 0 || N < 0 || K < 0 || (kind != SMX_ANTI && kind != SMX_DIST)) return SMX_E_ARG;
    if (M == 0 || N == 0) return SMX_OK;
    if (!aligned16(A) || !aligned16(B) || !aligned16(C)) return SMX_E_ALIGN;
    if (!ld_ok(lda, sizeof(T)) || !ld_ok(ldb, sizeof(T)) || !ld_ok(ldc, sizeof(T))) return SMX_E_ALIGN;
    if (lda < K || ldb < N || ldc < N) return SMX_E_ARG;
    long long kc = (384LL << 20) / ((long long)G::BM * ceil_div(M, G::BM) * 4 +
                                    (long long)G::BNW * ceil_div(N, G::BN) * 4);
    kc = kc / 256 * 256;
    if (kc < 256) kc = 256;
    if (kc > K) kc = K;
    const size_t ws_bytes = packed_ws_bytes_t<T>(M, N, (int)kc);
    void* scratch = nullptr;
    SMX_TRY(scratch_alloc(&scratch, ws_bytes + 256, s));
    struct FreeOnExit {
        void* p; cudaStream_t s;
        ~FreeOnExit() { scratch_free(p, s); }
    } guard{scratch, s};
    int* cert = reinterpret_cast<int*>(scratch);
    void* ws = reinterpret_cast<char*>(scratch) + 256;
    const int anti = kind == SMX_ANTI;
    const int* certp = nullptr;
    // (u8 needs no certificate: every u8 tile is the 1-instruction form)
    if constexpr (!Lane<T>::kOneInstr) {
        if (bounded_fastpath_enabled() && K > 0) {
            SMX_TRY(run_cert<T>(A, M, K, lda, B, K, N, ldb, anti, cert, s));
            certp = cert;
        }
    }
    if (K == 0) return packed_run<T>(C, M, N, 0, ldc, kind, accumulate, 0, -1, 0, 0, ws, ws_bytes, s);
    for (long long k0 = 0; k0 < K; k0 += kc) {
        const int kk = (int)(K - k0 < kc ? K - k0 : kc);
        SMX_TRY(packed_pack<T>(A + k0, B + k0 * ldb, M, N, kk, lda, ldb, kind, ws, ws_bytes, s, certp));
        SMX_TRY(packed_run<T>(C, M, N, kk, ldc, kind, k0 == 0 ? accumulate : 1, 0, -1, 0, 0, ws, ws_bytes, s,
                              certp));
    }
    return SMX_OK;
}

inline int semiring_gemm_packed_public_u16(const uint16_t* A, const uint16_t* B, uint16_t* C, int M, int N, int K,
                                           long long lda, long long ldb, long long ldc, int kind, int accumulate,
                                           cudaStream_t s) {
    return semiring_gemm_packed_public<uint16_t>(A, B, C, M, N, K, lda, ldb, ldc, kind, accumulate, s);
}

}  // namespace smx
