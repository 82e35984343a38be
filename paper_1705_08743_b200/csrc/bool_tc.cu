// Boolean product on the 5th-generation tensor cores: tcgen05.mma kind::i8
// with a count > 0 threshold, and the blocked Warshall closure built on it.
//
// BoolMatrix.__mul__ (pkg/src/semimat/boolmat.py:151-172) ORs row k of B into
// every row i with A[i,k] = 1.  Over 0/1 bytes that is exactly
//     C[i,j] = (sum_k A[i,k] * B[k,j]) > 0
// (SURVEY.md 0.1 fact 3), an unsigned 8-bit dense contraction with an int32
// accumulator that cannot overflow for K < 2^31.  So the Boolean product is
// run as a real GEMM on the tensor cores:
//   * TMA (cp.async.bulk.tensor, 128-byte swizzle) streams 128 x 128-byte A
//     and BN x 128-byte B^T tiles into a 4-stage shared-memory ring, tracked
//     by mbarriers (full/empty);
//   * one elected thread issues tcgen05.mma.cta_group::1.kind::i8 (M = 128,
//     N = BN, K = 32 per instruction) accumulating into TMEM, and
//     tcgen05.commit frees each ring slot when its MMAs retire;
//   * 4 epilogue warps read the accumulator with tcgen05.ld (32 lanes x 32
//     columns per instruction), threshold count > 0, and write either 0/1
//     bytes or the reference's packed-bit layout directly (one 32-bit word per
//     thread per 32 columns, LSB first -- boolmat.py:3-5), optionally OR-ing
//     into the existing output (Warshall phases 2/3).
// Ragged M, N, K come for free: TMA zero-fills out-of-bounds boxes and zero
// is the Boolean (+)-identity and (x)-annihilator.
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "bool_pivot.cuh"

namespace smx {

constexpr int kTcBM = 128;
constexpr int kTcBK = 128;        // bytes of K per stage = one 128-byte swizzle row
// TMA ring depth per tile width (192 KB of operand stages): deep enough that a
// short-K product (C1: 8 k-blocks) issues every load up front.
template <int BN> struct TcStages { static constexpr int value = BN <= 64 ? 8 : (BN <= 128 ? 6 : 4); };
constexpr int kTcThreads = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
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

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0,
                                            int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// K-major operand tile with 128-byte swizzle (rows of 128 bytes, 8-row core
// groups 1024 bytes apart): start>>4 | LBO(unused)=1 | SBO=1024>>4 |
// version 1 (sm_100) | layout SWIZZLE_128B (2).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
    return (uint64_t)((smem_addr & 0x3FFFFu) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
           (2ull << 61);
}

template <int BN>
__device__ __forceinline__ constexpr uint32_t idesc_i8() {
    // c_format S32 (2) @4 | a,b unsigned 8-bit (0) | K-major | N>>3 @17 | M>>4 @24
    return (2u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(kTcBM >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}

// kind::mxf4 (E2M1 operands, two per byte, UE8M0 scale per 32 elements of
// K, f32 accumulate): the same product on 0/1 operands (1.0 = 0b0010) at
// half the operand bytes and twice the MMA rate of kind::i8.  Block-scaled
// descriptor: a/b format E2M1 (1) @7/@10 | N>>3 @17 | scale UE8M0 @23 |
// M>>4 @24 | K = 64 per instruction (bit 31 clear) | scale-factor ids 0.
template <int BN>
__device__ __forceinline__ constexpr uint32_t idesc_f4() {
    return (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | (1u << 23) | ((uint32_t)(kTcBM >> 4) << 24);
}

__device__ __forceinline__ void umma_f4(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate, uint32_t tmem_sfa, uint32_t tmem_sfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(
            tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(tmem_sfa), "r"(tmem_sfb)
        : "memory");
}

// 8 TMEM columns of this warp's 32 lanes <- v
__device__ __forceinline__ void tmem_fill8(uint32_t taddr, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v)
                 : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 32 lanes x 64 columns in one tcgen05.ld, with its wait in the same asm
// statement (so no use of the registers can be scheduled before it).
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&r)[64]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr)
        : "memory");
}

struct TcArgs {
    uint8_t* C;          // bytes output (or nullptr)
    uint32_t* Cbits;     // packed output (or nullptr)
    int M, N, K;
    long long ldc;       // bytes, or u32 words for Cbits
    int accumulate;
    int skip_tile0, skip_tiles;
    int splits;          // split-K factor (gridDim.z); > 1 ORs into a pre-set output
    // batched products (pair kernel): products of batch_mt row tiles each are
    // stacked in A and C; product i's B^T rows start at i * bt_item_rows of
    // the stacked B^T operand (0 = one product)
    int batch_mt, bt_item_rows;
    // development trace (smx_tc_trace_arm; nullptr otherwise): per CTA,
    // globaltimer at entry and exit, and for CTA 0 clock64 at each phase
    unsigned long long* trace;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// F4: E2M1 nibble operands (kind::mxf4; a.K in bytes), TMEM columns
// [BN, 2 BN) hold the scale factors (all 1.0), as in the pair kernel below.
template <int BN, bool F4 = false>
__global__ void __launch_bounds__(kTcThreads, 1)
bool_i8_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const TcArgs p) {
    constexpr uint32_t A_BYTES = kTcBM * kTcBK;
    constexpr uint32_t B_BYTES = BN * kTcBK;
    extern __shared__ __align__(1024) uint8_t smem_dyn[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    constexpr int kTcStages = TcStages<BN>::value;
    uint8_t* sB = smem + kTcStages * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + kTcStages * B_BYTES);
    uint64_t* empty = full + kTcStages;
    uint64_t* accum = empty + kTcStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const bool tr0 = p.trace && cta == 0;
    if (p.trace && threadIdx.x == 0) p.trace[16 + 2 * cta] = gtimer();
    if (tr0 && threadIdx.x == 0) p.trace[0] = clock64();
    int mt = blockIdx.y;
    if (mt >= p.skip_tile0) mt += p.skip_tiles;
    const int m0 = mt * kTcBM, n0 = blockIdx.x * BN;
    // split-K: CTA z handles k-blocks [kb_lo, kb_hi); partial counts are
    // combined with atomicOr (OR is idempotent, so the merge is exact)
    const int nkb_all = (p.K + kTcBK - 1) / kTcBK;
    const int per = (nkb_all + p.splits - 1) / p.splits;
    const int kb_lo = blockIdx.z * per;
    const int kb_hi = min(nkb_all, kb_lo + per);
    const int nkb = kb_hi > kb_lo ? kb_hi - kb_lo : 0;

    // thread 0 issues the first ring fill before the TMEM allocation and the
    // CTA barrier (the loads only touch barriers it initialised itself)
    const int first_fill = nkb < kTcStages ? nkb : kTcStages;
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accum, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // Programmatic dependent launch: everything above ran while the
        // preceding kernel (e.g. the operand unpack) was still finishing; the
        // operands are read only after it completes.  A no-op without the
        // attribute.
        asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int kb = 0; kb < first_fill; ++kb) {
            mbar_expect_tx(&full[kb], A_BYTES + B_BYTES);
            tma_load_2d(&mapA, &full[kb], sA + kb * A_BYTES, (kb_lo + kb) * kTcBK, m0);
            tma_load_2d(&mapB, &full[kb], sB + kb * B_BYTES, (kb_lo + kb) * kTcBK, n0);
        }
    }
    constexpr uint32_t kTmemCols = F4 ? 2 * BN : BN;
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    if (tr0 && threadIdx.x == 0) p.trace[1] = clock64();
    if constexpr (F4) {
        // every warp sets its 32 lanes of the scale-factor columns to 1.0
        const uint32_t t = tmem + ((uint32_t)(warp * 32) << 16) + BN;
#pragma unroll
        for (int c = 0; c < BN; c += 8) tmem_fill8(t + c, 0x7F7F7F7Fu);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }

    if (threadIdx.x == 0) {
        // ---- TMA producer: the rest of the ring ----
        for (int kb = first_fill; kb < nkb; ++kb) {
            const int s = kb % kTcStages;
            const uint32_t ph = (kb / kTcStages) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
            tma_load_2d(&mapA, &full[s], sA + s * A_BYTES, (kb_lo + kb) * kTcBK, m0);
            tma_load_2d(&mapB, &full[s], sB + s * B_BYTES, (kb_lo + kb) * kTcBK, n0);
        }
        if (tr0) p.trace[2] = clock64();
    } else if (threadIdx.x == 32) {
        // ---- MMA issuer ----
        constexpr uint32_t idesc = F4 ? idesc_f4<BN>() : idesc_i8<BN>();
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % kTcStages;
            const uint32_t ph = (kb / kTcStages) & 1;
            mbar_wait(&full[s], ph);
            if (tr0 && (kb == 0 || kb == nkb - 1)) p.trace[kb == 0 ? 3 : 4] = clock64();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a0 = smem_u32(sA + s * A_BYTES), b0 = smem_u32(sB + s * B_BYTES);
#pragma unroll
            for (int k = 0; k < kTcBK / 32; ++k) {
                if constexpr (F4)
                    umma_f4(tmem, umma_desc_sw128(a0 + 32 * k), umma_desc_sw128(b0 + 32 * k), idesc,
                            (kb | k) != 0, tmem + BN, tmem + BN + BN / 2);
                else
                    umma_i8(tmem, umma_desc_sw128(a0 + 32 * k), umma_desc_sw128(b0 + 32 * k), idesc,
                            (kb | k) != 0);
            }
            umma_commit(&empty[s]);
        }
        umma_commit(accum);
    }
    __syncwarp();

    // ---- epilogue: TMEM -> threshold -> bytes or bits (F4: f32 counts,
    // nonzero exactly when positive) ----
    // a PDL-launched successor may start its prologue now (it reads nothing
    // of ours before its own griddepcontrol.wait)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    mbar_wait(accum, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tr0 && threadIdx.x == 0) p.trace[5] = clock64();
    const int row = m0 + warp * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(trow + c * 32, r);   // warp-collective: all lanes participate
        if (row >= p.M || nkb == 0) continue;
        const int col0 = n0 + c * 32;
        if (col0 >= p.N) continue;
        if (p.Cbits) {
            uint32_t word = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) word |= (r[j] != 0u ? 1u : 0u) << j;
            uint32_t* dst = p.Cbits + (long long)row * p.ldc + (col0 >> 5);
            if (p.splits > 1) atomicOr(dst, word);
            else *dst = p.accumulate ? (*dst | word) : word;
        } else if (p.splits > 1) {
            uint32_t w[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                w[q] = (r[4 * q] != 0u ? 1u : 0u) | (r[4 * q + 1] != 0u ? 0x100u : 0u) |
                       (r[4 * q + 2] != 0u ? 0x10000u : 0u) | (r[4 * q + 3] != 0u ? 0x1000000u : 0u);
            uint32_t* dst = reinterpret_cast<uint32_t*>(p.C + (long long)row * p.ldc + col0);
            const int nq = min(8, (p.N - col0 + 3) / 4);
            for (int q = 0; q < nq; ++q) {
                uint32_t v = w[q];
                const int valid = p.N - (col0 + 4 * q);
                if (valid < 4) v &= (1u << (8 * valid)) - 1u;
                if (v) atomicOr(dst + q, v);
            }
        } else {
            uint32_t w[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                w[q] = (r[4 * q] != 0u ? 1u : 0u) | (r[4 * q + 1] != 0u ? 0x100u : 0u) |
                       (r[4 * q + 2] != 0u ? 0x10000u : 0u) | (r[4 * q + 3] != 0u ? 0x1000000u : 0u);
            uint8_t* dst = p.C + (long long)row * p.ldc + col0;
            if (col0 + 32 <= p.N && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
                uint4* d4 = reinterpret_cast<uint4*>(dst);
                uint4 v0 = make_uint4(w[0], w[1], w[2], w[3]), v1 = make_uint4(w[4], w[5], w[6], w[7]);
                if (p.accumulate) {
                    const uint4 o0 = d4[0], o1 = d4[1];
                    v0.x |= o0.x; v0.y |= o0.y; v0.z |= o0.z; v0.w |= o0.w;
                    v1.x |= o1.x; v1.y |= o1.y; v1.z |= o1.z; v1.w |= o1.w;
                }
                d4[0] = v0;
                d4[1] = v1;
            } else {
                const uint8_t* wb = reinterpret_cast<const uint8_t*>(w);
                for (int j = 0; j < 32 && col0 + j < p.N; ++j)
                    dst[j] = p.accumulate ? (uint8_t)(dst[j] | wb[j]) : wb[j];
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tr0 && threadIdx.x == 0) p.trace[6] = clock64();
    if (p.trace && threadIdx.x == 0) p.trace[17 + 2 * cta] = gtimer();
    if (warp == 2) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols)
                     : "memory");
    }
}

// ---- split-K pair (small packed-bit products: C1) ------------------------------
//
// C1 (1024^3) has 128 output tiles of 128 x 64 in the kernel above: one per
// SM, each streaming 192 KB of operands for only 8 k-blocks, so the product
// is bound by the L2 -> SM operand stream (profiles/r02_tc_phases_c1.json:
// ~49 B/clk per SM, 3900 of the CTA's 6700 cycles), not by the tensor
// cores.  Here a cluster of two CTAs shares one 128 x 128 output tile and
// splits K in halves: each CTA streams (128 + 128) x K/2 bytes (128 KB at
// C1), and the whole product reads 16 MB instead of 24.
//
// Merge.  A partial count > 0 already proves the output bit (OR is
// idempotent), so each CTA thresholds its own half-K counts to bits and the
// pair only exchanges 1 KB of words: CTA r owns rows [64r, 64r + 64) of the
// tile and receives the partner's words of those rows by st.async into its
// shared memory (completing on a local mbarrier: no polling, no second
// barrier round trip), ORs them into its own and stores.  Eight warps run the
// epilogue: warps w and w + 4 read the same TMEM lanes (32 rows), columns
// [0, 64) and [64, 128).
constexpr int kPairBN = 128;
constexpr int kPairThreads = 256;
// Stage ring depth: a single product is one wave of CTAs, one per SM, and
// takes 6 stages of 32 KB (every k-block of C1 in flight at once); batched
// products run many waves, and 2 stages (~66 KB) let three CTAs share an SM
// so one CTA's loads and epilogue overlap the others' MMAs: 16 C1 products
// per launch 2.81 -> 1.43 us each with 2 stages (3 stages: 1.65 us;
// tools/perf_c1_batched.py, profiles/r04d_c1_batched_stages.json).
constexpr int kPairStagesSingle = 6;
constexpr int kPairStagesBatched = 2;
// A cluster of KS CTAs splits K; CTA r owns rows [r * 128 / KS, ...) of the
// tile and receives the other KS - 1 CTAs' words of them (one slot each).
template <int KS>
struct PairRecv {
    static constexpr int kRows = kTcBM / KS;                                   // rows owned per CTA
    static constexpr uint32_t kBytes = (KS - 1) * kRows * (kPairBN / 32) * 4;   // KS=2: 1 KB, KS=4: 1.5 KB
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_v2(uint32_t remote, uint32_t a, uint32_t b, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];"
                 ::"r"(remote), "r"(a), "r"(b), "r"(remote_bar) : "memory");
}
__device__ __forceinline__ uint32_t bits_of(const uint32_t (&r)[32]) {
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) word |= (r[j] != 0u ? 1u : 0u) << j;
    return word;
}

// (Tried: a cluster of four, 2 N-tiles x 2 K-halves, each CTA loading half
// of the shared A tile and multicasting it (TMA .multicast::cluster), so a
// CTA issues 96 KB instead of 128: no faster -- 3.79 against 3.49 us per
// launch, the same per-CTA timeline -- so the operand stream is bound where
// the bytes land, not where they are issued; removed.)
// F4: operands are E2M1 nibbles (bool_f4_gemm); one 128-byte k-block then
// holds 256 elements of K, and TMEM columns [128, 256) hold the scale
// factors, all 1.0 (UE8M0 127): a uniform fill, so their TMEM layout does
// not matter.
template <int KS, int kPairStages, bool F4 = false>
__global__ void __launch_bounds__(kPairThreads, 1)
bool_i8_gemm_pair_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                         const TcArgs p) {
    constexpr uint32_t A_BYTES = kTcBM * kTcBK;
    constexpr uint32_t B_BYTES = kPairBN * kTcBK;
    extern __shared__ __align__(1024) uint8_t smem_dyn[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + kPairStages * A_BYTES;
    using RV = PairRecv<KS>;
    uint32_t* recv = reinterpret_cast<uint32_t*>(sB + kPairStages * B_BYTES);   // [KS-1][rows][4] partner words
    uint64_t* full = reinterpret_cast<uint64_t*>(recv + RV::kBytes / 4);
    uint64_t* empty = full + kPairStages;
    uint64_t* accum = empty + kPairStages;
    uint64_t* recv_bar = accum + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv_bar + 1);
    constexpr uint32_t kTmemCols = F4 ? 2 * kPairBN : kPairBN;
    constexpr uint32_t kSfa = kPairBN, kSfb = kPairBN + 64;   // (F4) scale-factor columns

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();   // the K slice; owns rows [rank * RV::kRows, ...)
    const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const bool tr0 = p.trace && cta == 0;
    if (p.trace && threadIdx.x == 0) p.trace[16 + 2 * cta] = gtimer();
    if (tr0 && threadIdx.x == 0) p.trace[0] = clock64();
    const int m0 = blockIdx.y * kTcBM, n0 = blockIdx.x * kPairBN;
    // (batched: this CTA's product's B^T rows)
    const int nb0 = n0 + (p.batch_mt > 0 ? (int)(blockIdx.y / p.batch_mt) * p.bt_item_rows : 0);
    const int nkb_all = (p.K + kTcBK - 1) / kTcBK;
    const int per = (nkb_all + KS - 1) / KS;
    const int kb_lo = (int)rank * per;
    const int kb_hi = min(nkb_all, kb_lo + per);
    const int nkb = kb_hi > kb_lo ? kb_hi - kb_lo : 0;

    // Thread 0 initialises the barriers and issues the first ring fill right
    // away -- before the TMEM allocation and the CTA barrier -- so the first
    // operand stage is in flight while the rest of the CTA sets up (the
    // loads only touch barriers this thread initialised).  (Initialising
    // the barriers one per lane of warp 0 was slower: ~900 against ~350
    // cycles to the first load.)
    const int first_fill = nkb < kPairStages ? nkb : kPairStages;
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
        for (int s = 0; s < kPairStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accum, 1);
        mbar_init(recv_bar, 1);
        // the partner's 1 KB lands on recv_bar: expected before the cluster
        // barrier below, so no complete_tx can precede it
        mbar_expect_tx(recv_bar, RV::kBytes);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (tr0) p.trace[10] = clock64();
        // PDL: operands are read only after the preceding kernel in the
        // stream completes (a no-op without the launch attribute)
        asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int kb = 0; kb < first_fill; ++kb) {
            mbar_expect_tx(&full[kb], A_BYTES + B_BYTES);
            tma_load_2d(&mapA, &full[kb], sA + kb * A_BYTES, (kb_lo + kb) * kTcBK, m0);
            tma_load_2d(&mapB, &full[kb], sB + kb * B_BYTES, (kb_lo + kb) * kTcBK, nb0);
        }
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)), "n"(kTmemCols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        if (tr0 && lane == 0) p.trace[11] = clock64();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // publish the initialised barriers to the partner (waited on before the
    // first remote store, long after).  Relaxed: thread 0's
    // fence.mbarrier_init.release.cluster already orders the inits, and a
    // release arrive costs ~500 cycles of memory fence here.
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    if (tr0 && threadIdx.x == 0) p.trace[1] = clock64();
    if constexpr (F4) {
        // warps 4-7 (TMEM lanes 32 * (warp - 4) ...) set every scale factor to
        // 1.0 while the first operands are in flight; the MMA warp waits on
        // named barrier 1 for them
        if (warp >= 4) {
            const uint32_t t = tmem + ((uint32_t)((warp & 3) * 32) << 16) + kPairBN;
#pragma unroll
            for (int c = 0; c < kPairBN; c += 8) tmem_fill8(t + c, 0x7F7F7F7Fu);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            asm volatile("bar.arrive 1, 160;" ::: "memory");
        } else if (warp == 1) {
            asm volatile("bar.sync 1, 160;" ::: "memory");
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
    }

    if (threadIdx.x == 0) {
        // ---- TMA producer: the rest of the ring (K beyond the first fill)
        for (int kb = first_fill; kb < nkb; ++kb) {
            const int s = kb % kPairStages;
            const uint32_t ph = (kb / kPairStages) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
            tma_load_2d(&mapA, &full[s], sA + s * A_BYTES, (kb_lo + kb) * kTcBK, m0);
            tma_load_2d(&mapB, &full[s], sB + s * B_BYTES, (kb_lo + kb) * kTcBK, nb0);
        }
        if (tr0) p.trace[2] = clock64();
    } else if (threadIdx.x == 32) {
        // ---- MMA issuer ----
        constexpr uint32_t idesc = F4 ? idesc_f4<kPairBN>() : idesc_i8<kPairBN>();
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % kPairStages;
            const uint32_t ph = (kb / kPairStages) & 1;
            mbar_wait(&full[s], ph);
            if (tr0 && (kb == 0 || kb == nkb - 1)) p.trace[kb == 0 ? 3 : 4] = clock64();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a0 = smem_u32(sA + s * A_BYTES), b0 = smem_u32(sB + s * B_BYTES);
            // 32 bytes of K per instruction either way (i8: 32 elements, F4: 64)
#pragma unroll
            for (int k = 0; k < kTcBK / 32; ++k) {
                if constexpr (F4)
                    umma_f4(tmem, umma_desc_sw128(a0 + 32 * k), umma_desc_sw128(b0 + 32 * k), idesc,
                            (kb | k) != 0, tmem + kSfa, tmem + kSfb);
                else
                    umma_i8(tmem, umma_desc_sw128(a0 + 32 * k), umma_desc_sw128(b0 + 32 * k), idesc,
                            (kb | k) != 0);
            }
            umma_commit(&empty[s]);
        }
        umma_commit(accum);
    }
    __syncwarp();

    // ---- epilogue: this K slice's counts -> bits ----
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    mbar_wait(accum, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tr0 && threadIdx.x == 0) p.trace[5] = clock64();
    const int quad = warp & 3, chalf = warp >> 2;          // TMEM lanes 32*quad.., columns 64*chalf..
    const int trow = quad * 32 + lane;                      // row within the tile
    const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(chalf * 64);
    uint32_t w0 = 0, w1 = 0;
    {
        // counts of this CTA's K half are < 2^16 (K <= 65536, host-checked):
        // two counts per 16-bit lane pair (PRMT), clamped to 0/1 by one
        // VIMNMX.U16x2, placed at bits j and j + 16 by one shift-add:
        // 1.5 instructions per output bit instead of ~2.7
        // (F4: f32 counts; a positive count has a nonzero upper half, so the
        // same clamp runs on the upper halves)
        constexpr uint32_t sel = F4 ? 0x7632u : 0x5410u;
        uint32_t r[64];
        tmem_ld64(taddr, r);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            w0 += __vminu2(__byte_perm(r[j], r[j + 16], sel), 0x00010001u) << j;
            w1 += __vminu2(__byte_perm(r[32 + j], r[48 + j], sel), 0x00010001u) << j;
        }
    }
    if (nkb == 0) w0 = w1 = 0u;   // (K shorter than one k-block per CTA: TMEM was never written)
    if (tr0 && threadIdx.x == 0) p.trace[8] = clock64();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    // rows owned by another CTA go to it, into this CTA's slot there; words
    // [row][2*chalf, 2*chalf + 1]
    const uint32_t owner = (uint32_t)(trow / RV::kRows);   // the CTA that stores this row
    const int orow = trow % RV::kRows;
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (tr0 && threadIdx.x == 0) p.trace[9] = clock64();
    if (owner != rank) {
        const int slot = (int)rank < (int)owner ? (int)rank : (int)rank - 1;
        const uint32_t off = (uint32_t)(((slot * RV::kRows + orow) * 4 + 2 * chalf) * 4);
        st_async_v2(mapa_shared(smem_u32(recv) + off, owner), w0, w1, mapa_shared(smem_u32(recv_bar), owner));
    }
    // No second cluster barrier: every store into this CTA's shared memory
    // completes on recv_bar, which the owner threads wait on before the CTA
    // can exit, and this CTA stores into the partner only (the partner
    // waits on its own recv_bar likewise).
    if (tr0 && threadIdx.x == 0) p.trace[6] = clock64();
    if (owner == rank) {
        mbar_wait(recv_bar, 0);
#pragma unroll
        for (int sl = 0; sl < KS - 1; ++sl) {
            const uint2 o = *reinterpret_cast<const uint2*>(&recv[(sl * RV::kRows + orow) * 4 + 2 * chalf]);
            w0 |= o.x;
            w1 |= o.y;
        }
        const int row = m0 + trow, col0 = n0 + chalf * 64;
        if (row < p.M && col0 < p.N) {
            uint32_t* dst = p.Cbits + (long long)row * p.ldc + (col0 >> 5);
            const int left = p.N - col0;
            if (left < 32) w0 &= (1u << left) - 1u;
            if (left < 64 && left > 32) w1 &= (1u << (left - 32)) - 1u;
            if (p.accumulate) {
                dst[0] |= w0;
                if (left > 32) dst[1] |= w1;
            } else {
                dst[0] = w0;
                if (left > 32) dst[1] = w1;
            }
        }
    }
    __syncthreads();
    if (tr0 && threadIdx.x == 0) p.trace[7] = clock64();
    if (p.trace && threadIdx.x == 0) p.trace[17 + 2 * cta] = gtimer();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
}

// ---- host side ---------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// rows x cols bytes (K-major), box = box_rows x 128 bytes, 128-byte swizzle
static int make_map(CUtensorMap* map, const uint8_t* base, int rows, int cols, long long ld, int box_rows) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return SMX_E_DRIVER;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {(cuuint32_t)kTcBK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? SMX_OK : SMX_E_DRIVER;
}

template <int BN, bool F4 = false>
static int launch_tc(const uint8_t* A, const uint8_t* Bt, const TcArgs& a, long long lda, long long ldbt,
                     cudaStream_t s, bool pdl = false) {
    CUtensorMap mA, mB;
    SMX_TRY(make_map(&mA, A, a.M, a.K, lda, kTcBM));
    SMX_TRY(make_map(&mB, Bt, a.N, a.K, ldbt, BN));
    constexpr int kTcStages = TcStages<BN>::value;
    constexpr size_t smem = 1024 + kTcStages * (size_t)(kTcBM + BN) * kTcBK + 8 * (2 * kTcStages + 1) + 16;
    auto kern = bool_i8_gemm_kernel<BN, F4>;
    SMX_TRY(set_max_smem((const void*)kern, smem));
    const int mtiles = ceil_div(a.M, kTcBM) - a.skip_tiles;
    if (mtiles <= 0) return SMX_OK;
    TcArgs args = a;
    // split K only for long, thin products (few tiles, >= 16 k-blocks): at
    // C1's 1024^3 the extra zero-fill and atomics cost more than the
    // latency they hide (12.7 -> 17.2 us measured), so it stays off there
    const int tiles = mtiles * ceil_div(a.N, BN);
    const int nkb = ceil_div(a.K, kTcBK);
    int splits = 1;
    if (tiles < 148 / 2 && nkb >= 16) {
        splits = ceil_div(148, tiles);
        if (splits > nkb / 8) splits = nkb / 8;
    }
    args.splits = splits;
    if (splits > 1 && !a.accumulate) {
        // partial results are OR-ed in: start from an all-zero output
        const size_t row_bytes = a.Cbits ? (size_t)ceil_div(a.N, 32) * 4 : (size_t)a.N;
        const size_t pitch = a.Cbits ? (size_t)a.ldc * 4 : (size_t)a.ldc;
        void* base = a.Cbits ? (void*)a.Cbits : (void*)a.C;
        cudaError_t e = cudaMemset2DAsync(base, pitch, 0, row_bytes, a.M, s);
        if (e != cudaSuccess) return (int)e;
    }
    dim3 grid(ceil_div(a.N, BN), mtiles, splits);
    if (!pdl) {
        kern<<<grid, kTcThreads, smem, s>>>(mA, mB, args);
        SMX_RETURN_LAUNCH();
    }
    // overlap this kernel's launch and prologue (barriers, TMEM allocation,
    // descriptor prefetch) with the tail of the preceding kernel
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    count_launch();
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mA, mB, args);
    return e == cudaSuccess ? SMX_OK : (int)e;
}


// Split-K pair launch (packed-bit output, no row skip).  The caller has
// checked the shape (see bool_i8_gemm).
// (F4: a.K is the operand row length in BYTES, ceil(K / 2))
template <int KS, int kPairStages, bool F4 = false>
static int launch_tc_pair(const uint8_t* A, const uint8_t* Bt, const TcArgs& a, long long lda, long long ldbt,
                          cudaStream_t s, bool pdl, int bt_rows = -1) {
    CUtensorMap mA, mB;
    SMX_TRY(make_map(&mA, A, a.M, a.K, lda, kTcBM));
    SMX_TRY(make_map(&mB, Bt, bt_rows < 0 ? a.N : bt_rows, a.K, ldbt, kPairBN));
    constexpr size_t smem = 1024 + kPairStages * (size_t)(kTcBM + kPairBN) * kTcBK + PairRecv<KS>::kBytes +
                            8 * (2 * kPairStages + 2) + 16;
    auto kern = bool_i8_gemm_pair_kernel<KS, kPairStages, F4>;
    SMX_TRY(set_max_smem((const void*)kern, smem));
    TcArgs args = a;
    args.splits = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ceil_div(a.N, kPairBN), ceil_div(a.M, kTcBM), KS);
    cfg.blockDim = dim3(kPairThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = KS;
    int na = 1;
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    count_launch();
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mA, mB, args);
    return e == cudaSuccess ? SMX_OK : (int)e;
}

// Output tile width of smx_bool_gemm_i8: 0 = automatic (the widest tile that
// still gives every SM a tile), or force 64 / 128 / 256 (tuning switch;
// results are identical).
static int g_tc_tile_n = 0;
static int g_tc_pair = 1;
static int g_tc_batch_ks = 1;   // K slices per batched product (1: one CTA per tile, fastest measured)
static unsigned long long* g_tc_trace = nullptr;

int bool_i8_gemm(const uint8_t* A, const uint8_t* Bt, uint8_t* C, uint32_t* Cbits, int M, int N, int K,
                 long long lda, long long ldbt, long long ldc, int accumulate, int skip_row0, int skip_rows,
                 cudaStream_t s, bool pdl = false) {
    if (M < 0 || N < 0 || K < 1 || (C == nullptr) == (Cbits == nullptr)) return SMX_E_ARG;
    if (M == 0 || N == 0) return SMX_OK;
    if (!aligned16(A) || !aligned16(Bt) || (lda & 15) || (ldbt & 15)) return SMX_E_ALIGN;
    if (lda < K || ldbt < K) return SMX_E_ARG;
    if (Cbits ? ((long long)ldc * 32 < N) : (ldc < N)) return SMX_E_ARG;
    TcArgs a{C, Cbits, M, N, K, ldc, accumulate != 0, 0, 0, 1, 0, 0, g_tc_trace};
    if (skip_rows > 0) {
        if (skip_row0 % kTcBM) return SMX_E_ARG;
        a.skip_tile0 = skip_row0 / kTcBM;
        a.skip_tiles = ceil_div(skip_rows, kTcBM);
        const int total = ceil_div(M, kTcBM);
        if (a.skip_tile0 + a.skip_tiles > total) a.skip_tiles = total - a.skip_tile0;
    }
    // small packed-bit products (C1): split K across a CTA pair when one
    // wave of 128 x 64 tiles or fewer covers the output (smx_set_tc_pair:
    // 0 = off, 1 = automatic, 2 = always when the shape allows it)
    if (Cbits && skip_rows == 0 && g_tc_pair != 0 && K > kTcBK && K <= 65536) {
        const long long tiles64 = (long long)ceil_div(M, kTcBM) * ceil_div(N, 64);
        if (g_tc_pair >= 2 || (tiles64 <= 148 && g_tc_tile_n == 0))
        {
            if (g_tc_pair == 3) return launch_tc_pair<4, 2>(A, Bt, a, lda, ldbt, s, pdl);
            return launch_tc_pair<2, kPairStagesSingle>(A, Bt, a, lda, ldbt, s, pdl);
        }
    }
    if (g_tc_tile_n == 64) return launch_tc<64>(A, Bt, a, lda, ldbt, s, pdl);
    if (g_tc_tile_n == 128) return launch_tc<128>(A, Bt, a, lda, ldbt, s, pdl);
    if (g_tc_tile_n == 256) return launch_tc<256>(A, Bt, a, lda, ldbt, s, pdl);
    // widest tile that still gives every SM a tile
    const long long rows = ceil_div(M, kTcBM) - a.skip_tiles;
    if (rows * ceil_div(N, 256) >= 148) return launch_tc<256>(A, Bt, a, lda, ldbt, s, pdl);
    if (rows * ceil_div(N, 128) >= 148) return launch_tc<128>(A, Bt, a, lda, ldbt, s, pdl);
    return launch_tc<64>(A, Bt, a, lda, ldbt, s, pdl);
}

// Batched products on the split-K pair: `batch` products of M x K by K x N
// stacked in A (batch * M rows), B^T (batch * N rows) and the packed-bit
// C (batch * M rows), one launch; M and N multiples of 128 so no tile
// straddles two products.
int bool_i8_gemm_batched(const uint8_t* A, const uint8_t* Bt, uint32_t* Cbits, int batch, int M, int N, int K,
                         long long lda, long long ldbt, long long ldc, int accumulate, cudaStream_t s) {
    if (batch < 0 || M < 0 || N < 0 || K < 1 || Cbits == nullptr) return SMX_E_ARG;
    if (batch == 0 || M == 0 || N == 0) return SMX_OK;
    if (M % kTcBM || N % kPairBN || K <= kTcBK || K > 65536) return SMX_E_ARG;
    if (!aligned16(A) || !aligned16(Bt) || (lda & 15) || (ldbt & 15)) return SMX_E_ALIGN;
    if (lda < K || ldbt < K || (long long)ldc * 32 < N) return SMX_E_ARG;
    TcArgs a{nullptr, Cbits, batch * M, N, K, ldc, accumulate != 0, 0, 0, 1, M / kTcBM, N, g_tc_trace};
    if (g_tc_batch_ks == 4) return launch_tc_pair<4, 2>(A, Bt, a, lda, ldbt, s, /*pdl=*/true, batch * N);
    // (one CTA per tile: counts up to K must fit the 16-bit clamp)
    if (g_tc_batch_ks == 1 && K < 65536)
        return launch_tc_pair<1, 2>(A, Bt, a, lda, ldbt, s, /*pdl=*/true, batch * N);
    return launch_tc_pair<2, kPairStagesBatched>(A, Bt, a, lda, ldbt, s, /*pdl=*/true, batch * N);
}

// The same products on E2M1 nibble operands (kind::mxf4, the pair kernel):
// A is M rows of ceil(K / 2) bytes (lda bytes apart), B^T N rows likewise
// (unpack_nib_ab); packed-bit output.  Any M, N, K >= 1.
static int g_tc_f4 = 1;   // bool_mul_tc / bool_mul_tc_batched operands: 1 = E2M1 nibbles, 0 = bytes
static int g_tc_f4_batch_stages = 2;   // (experiment switch: ring depth of the batched nibble products)

int bool_f4_gemm(const uint8_t* A, const uint8_t* Bt, uint32_t* Cbits, int M, int N, int K, long long lda,
                 long long ldbt, long long ldc, int accumulate, cudaStream_t s, bool pdl) {
    if (M < 0 || N < 0 || K < 1 || Cbits == nullptr) return SMX_E_ARG;
    if (M == 0 || N == 0) return SMX_OK;
    const int kb = (K + 1) / 2;
    if (!aligned16(A) || !aligned16(Bt) || (lda & 15) || (ldbt & 15)) return SMX_E_ALIGN;
    if (lda < kb || ldbt < kb || (long long)ldc * 32 < N) return SMX_E_ARG;
    TcArgs a{nullptr, Cbits, M, N, kb, ldc, accumulate != 0, 0, 0, 1, 0, 0, g_tc_trace};
    // the same tile choice as bool_i8_gemm: the split-K pair for one wave of
    // 128 x 64 tiles or fewer, else the widest tile that gives every SM one
    const long long rows = ceil_div(M, kTcBM);
    if (g_tc_pair != 0 && (g_tc_pair >= 2 || (rows * ceil_div(N, 64) <= 148 && g_tc_tile_n == 0))) {
        if (g_tc_pair == 3) return launch_tc_pair<4, 2, true>(A, Bt, a, lda, ldbt, s, pdl);
        return launch_tc_pair<2, kPairStagesSingle, true>(A, Bt, a, lda, ldbt, s, pdl);
    }
    if (g_tc_tile_n == 64) return launch_tc<64, true>(A, Bt, a, lda, ldbt, s, pdl);
    if (g_tc_tile_n == 128) return launch_tc<128, true>(A, Bt, a, lda, ldbt, s, pdl);
    if (g_tc_tile_n == 256) return launch_tc<256, true>(A, Bt, a, lda, ldbt, s, pdl);
    if (rows * ceil_div(N, 256) >= 148) return launch_tc<256, true>(A, Bt, a, lda, ldbt, s, pdl);
    if (rows * ceil_div(N, 128) >= 148) return launch_tc<128, true>(A, Bt, a, lda, ldbt, s, pdl);
    return launch_tc<64, true>(A, Bt, a, lda, ldbt, s, pdl);
}

int bool_f4_gemm_batched(const uint8_t* A, const uint8_t* Bt, uint32_t* Cbits, int batch, int M, int N, int K,
                         long long lda, long long ldbt, long long ldc, int accumulate, cudaStream_t s) {
    if (batch < 0 || M < 0 || N < 0 || K < 1 || Cbits == nullptr) return SMX_E_ARG;
    if (batch == 0 || M == 0 || N == 0) return SMX_OK;
    if (M % kTcBM || N % kPairBN) return SMX_E_ARG;
    const int kb = (K + 1) / 2;
    if (!aligned16(A) || !aligned16(Bt) || (lda & 15) || (ldbt & 15)) return SMX_E_ALIGN;
    if (lda < kb || ldbt < kb || (long long)ldc * 32 < N) return SMX_E_ARG;
    TcArgs a{nullptr, Cbits, batch * M, N, kb, ldc, accumulate != 0, 0, 0, 1, M / kTcBM, N, g_tc_trace};
    const int ks = g_tc_batch_ks, st = g_tc_f4_batch_stages;
    if (ks == 1) return st == 3 ? launch_tc_pair<1, 3, true>(A, Bt, a, lda, ldbt, s, true, batch * N)
                                : launch_tc_pair<1, 2, true>(A, Bt, a, lda, ldbt, s, true, batch * N);
    if (ks == 4) return launch_tc_pair<4, 2, true>(A, Bt, a, lda, ldbt, s, true, batch * N);
    return st == 3 ? launch_tc_pair<2, 3, true>(A, Bt, a, lda, ldbt, s, true, batch * N)
                   : launch_tc_pair<2, 2, true>(A, Bt, a, lda, ldbt, s, true, batch * N);
}

// ---- Warshall on bytes with tensor-core phases 2/3 -----------------------------

constexpr int kTcWarshallBlock = 256;

// Pivot tile closure on bytes: each thread packs its row of 0/1 bytes to
// bits, the tile is closed by the bit-packed table pivot (bool_pivot.cuh),
// and the rows are unpacked back to bytes.
__global__ void __launch_bounds__(kWarshallBlock, 1)
bool_pivot_bytes_kernel(uint8_t* P, int b, long long ld) {
    constexpr int W = kWarshallBlock / 32;
    __shared__ __align__(16) PivotSmem sm;
    const int r = threadIdx.x;
    uint8_t* row = P + (long long)r * ld;
    const bool vec = b == kWarshallBlock && (reinterpret_cast<uintptr_t>(row) & 15) == 0;
    uint32_t w[W];
#pragma unroll
    for (int i = 0; i < W; ++i) {
        uint32_t v = 0;
        if (r < b) {
            if (vec) {
                const uint4* src = reinterpret_cast<const uint4*>(row + i * 32);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint4 x = src[h];
                    const uint32_t q[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t o = __vcmpne4(q[j], 0u) & 0x01010101u;   // 0/1 per byte
                        const uint32_t nib = (o & 1u) | ((o >> 7) & 2u) | ((o >> 14) & 4u) | ((o >> 21) & 8u);
                        v |= nib << (16 * h + 4 * j);
                    }
                }
            } else {
                for (int j = 0; j < 32; ++j) {
                    const int c = i * 32 + j;
                    if (c < b && row[c]) v |= 1u << j;
                }
            }
        }
        w[i] = v;
    }
    close_tile_bits(w, b, sm);
    if (r < b) {
        if (vec) {
#pragma unroll
            for (int i = 0; i < W; ++i) {
                uint4* dst = reinterpret_cast<uint4*>(row + i * 32);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t q[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t nib = (w[i] >> (16 * h + 4 * j)) & 0xFu;
                        q[j] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
                    }
                    dst[h] = make_uint4(q[0], q[1], q[2], q[3]);
                }
            }
        } else {
            for (int c = 0; c < b; ++c) row[c] = (w[c >> 5] >> (c & 31)) & 1u;
        }
    }
}

inline size_t tc_ws_bytes(int n, long long ld) {
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t rpt = al((size_t)n * kTcWarshallBlock);          // (row panel)^T, n x B
    const size_t cp = al((size_t)n * kTcWarshallBlock);           // column panel snapshot
    const size_t rp = al((size_t)kTcWarshallBlock * ld);          // row panel snapshot
    return rpt + cp + rp;
}

int transpose_bytes(const uint8_t* in, uint8_t* out, int rows, int cols, long long ld_in, long long ld_out,
                    cudaStream_t s);

int bool_warshall_i8(uint8_t* T, int n, long long ld, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (n < 0 || ld < n) return SMX_E_ARG;
    if (n == 0) return SMX_OK;
    if (!aligned16(T) || (ld & 15)) return SMX_E_ALIGN;
    if (n <= kTcWarshallBlock) {
        bool_pivot_bytes_kernel<<<1, kTcWarshallBlock, 0, s>>>(T, n, ld);
        SMX_RETURN_LAUNCH();
    }
    if (ws == nullptr || ws_bytes < tc_ws_bytes(n, ld)) return SMX_E_WORKSPACE;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    uint8_t* RPt = reinterpret_cast<uint8_t*>(ws);
    uint8_t* CP = RPt + al((size_t)n * kTcWarshallBlock);
    uint8_t* RP = CP + al((size_t)n * kTcWarshallBlock);
    constexpr long long B = kTcWarshallBlock;
    (void)RP;
    GraphKey key;
    key.fn = 301;
    const unsigned long long kv[] = {(uintptr_t)T, (unsigned long long)n, (unsigned long long)ld, (uintptr_t)ws,
                                     ws_bytes};
    for (size_t i = 0; i < sizeof(kv) / sizeof(kv[0]); ++i) key.v[i] = kv[i];
    return run_graphed(key, s, false, [&](cudaStream_t st) -> int {
        for (int k0 = 0; k0 < n; k0 += kTcWarshallBlock) {
            const int bb = n - k0 < kTcWarshallBlock ? n - k0 : kTcWarshallBlock;
            uint8_t* rowK = T + (long long)k0 * ld;
            count_launch();
            bool_pivot_bytes_kernel<<<1, kTcWarshallBlock, 0, st>>>(rowK + k0, bb, ld);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return (int)e;
            // phase 2 in place: T[K,:] |= P* . T[K,:]  (B^T = T[K,:]^T snapshot;
            // reading P* while it is rewritten with its own value is exact)
            SMX_TRY(transpose_bytes(rowK, RPt, bb, n, ld, B, st));
            SMX_TRY(bool_i8_gemm(rowK + k0, RPt, rowK, nullptr, bb, n, bb, ld, B, ld, 1, 0, 0, st));
            // phase 3: T[i,:] |= CP[i,:] . T[K,:]  for i outside K  (B^T = T[K,:]^T)
            SMX_TRY(transpose_bytes(rowK, RPt, bb, n, ld, B, st));
            e = cudaMemcpy2DAsync(CP, B, T + k0, ld, bb, n, cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return (int)e;
            SMX_TRY(bool_i8_gemm(CP, RPt, T, nullptr, n, n, bb, B, B, ld, 1, k0, bb, st));
        }
        return SMX_OK;
    });
}

int unpack_bits(const uint32_t* words, uint8_t* bytes, int rows, int cols, long long ld_w, long long ld,
                cudaStream_t s);
int unpack_bits_transposed(const uint32_t* words, uint8_t* out, int rows, int cols, long long ld_w,
                           long long ld_out, cudaStream_t s);
int unpack_bits_transposed_batched(const uint32_t* words, uint8_t* out, int batch, int rows, int cols, long long ld_w,
                                   long long ld_out, long long in_stride, long long out_stride, cudaStream_t s);
int unpack_ab(const uint32_t* a_words, uint8_t* a_bytes, int a_rows, int a_cols, long long a_ldw, long long a_ld,
              const uint32_t* b_words, uint8_t* bt, int b_rows, int b_cols, long long b_ldw, long long b_ldt,
              cudaStream_t s);
int unpack_nib_ab(const uint32_t* a_words, uint8_t* a_nib, int a_rows, int a_cols, long long a_ldw, long long a_ld,
                  const uint32_t* b_words, uint8_t* bt, int b_rows, int b_cols, long long b_ldw, long long b_ldt,
                  int batch, long long a_in, long long a_out, long long b_in, long long b_out, cudaStream_t s);

inline long long round16(long long x) { return (x + 15) & ~15LL; }

inline size_t bool_mul_ws_bytes(int M, int N, int K) {
    return (size_t)((M * round16(K) + 255) & ~255LL) + (size_t)N * round16(K);
}

// BoolMatrix.__mul__ on the reference's bit rows in one call: A bits ->
// bytes, B bits -> B^T bytes (fused transpose), tensor-core product with the
// packed-bit epilogue.  Workspace: M x K + N x K bytes (rows rounded to 16).
int bool_mul_tc(const uint32_t* A, const uint32_t* B, uint32_t* C, int M, int N, int K, long long lda_w,
                long long ldb_w, long long ldc_w, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (M < 0 || N < 0 || K < 1) return SMX_E_ARG;
    if (M == 0 || N == 0) return SMX_OK;
    if (ws == nullptr || ws_bytes < bool_mul_ws_bytes(M, N, K)) return SMX_E_WORKSPACE;
    uint8_t* a8 = reinterpret_cast<uint8_t*>(ws);
    uint8_t* bt8 = a8 + ((M * round16(K) + 255) & ~255LL);
    // E2M1 nibble operands (kind::mxf4) unless switched off
    const bool f4 = g_tc_f4 != 0;
    GraphKey key;
    key.fn = f4 ? 301 : 300;
    const unsigned long long kv[] = {(uintptr_t)A, (uintptr_t)B, (uintptr_t)C, (unsigned long long)M,
                                     (unsigned long long)N, (unsigned long long)K, (unsigned long long)lda_w,
                                     (unsigned long long)ldb_w, (unsigned long long)ldc_w, (uintptr_t)ws,
                                     ws_bytes};
    for (size_t i = 0; i < sizeof(kv) / sizeof(kv[0]); ++i) key.v[i] = kv[i];
    return run_graphed(key, s, false, [&](cudaStream_t st) -> int {
        const long long nw = (N + 31) / 32;
        if (f4) {
            const long long ldn = round16((K + 1) / 2);
            SMX_TRY(unpack_nib_ab(A, a8, M, K, lda_w, ldn, B, bt8, K, N, ldb_w, ldn, 1, 0, 0, 0, 0, st));
        } else {
            SMX_TRY(unpack_ab(A, a8, M, K, lda_w, round16(K), B, bt8, K, N, ldb_w, round16(K), st));
        }
        // words past ceil(N/32) in each output row are padding: keep them zero
        if (ldc_w > nw) {
            cudaError_t e = cudaMemset2DAsync(C + nw, ldc_w * 4, 0, (ldc_w - nw) * 4, M, st);
            if (e != cudaSuccess) return (int)e;
        }
        if (f4)
            return bool_f4_gemm(a8, bt8, C, M, N, K, round16((K + 1) / 2), round16((K + 1) / 2), ldc_w, 0, st,
                                /*pdl=*/ldc_w == nw);
        return bool_i8_gemm(a8, bt8, nullptr, C, M, N, K, round16(K), round16(K), ldc_w, 0, 0, 0, st,
                            /*pdl=*/ldc_w == nw);
    });
}

// Batched BoolMatrix products in one call: stacked bit rows in (A: batch x M
// rows, B: batch x K rows), stacked bit rows out (batch x M rows); A is
// unpacked in one launch, every B^T by one batched transpose launch, then one
// pair launch for every product.  Replayed as a graph on repeat calls.
inline size_t bool_mul_batched_ws_bytes(int batch, int M, int N, int K) {
    return (size_t)(((long long)batch * M * round16(K) + 255) & ~255LL) + (size_t)batch * N * round16(K);
}

int bool_mul_tc_batched(const uint32_t* A, const uint32_t* B, uint32_t* C, int batch, int M, int N, int K,
                        long long lda_w, long long ldb_w, long long ldc_w, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (batch < 0 || M < 0 || N < 0 || K < 1) return SMX_E_ARG;
    if (batch == 0 || M == 0 || N == 0) return SMX_OK;
    if (M % kTcBM || N % kPairBN || K <= kTcBK || K > 65536 || ldc_w * 32 != N) return SMX_E_ARG;
    if (ws == nullptr || ws_bytes < bool_mul_batched_ws_bytes(batch, M, N, K)) return SMX_E_WORKSPACE;
    uint8_t* a8 = reinterpret_cast<uint8_t*>(ws);
    uint8_t* bt8 = a8 + (((long long)batch * M * round16(K) + 255) & ~255LL);
    const bool f4 = g_tc_f4 != 0;
    GraphKey key;
    key.fn = f4 ? 303 : 302;
    const unsigned long long kv[] = {(uintptr_t)A, (uintptr_t)B, (uintptr_t)C, (unsigned long long)batch,
                                     (unsigned long long)M, (unsigned long long)N, (unsigned long long)K,
                                     (unsigned long long)lda_w, (unsigned long long)ldb_w,
                                     (unsigned long long)ldc_w, (uintptr_t)ws, ws_bytes};
    for (size_t i = 0; i < sizeof(kv) / sizeof(kv[0]); ++i) key.v[i] = kv[i];
    return run_graphed(key, s, false, [&](cudaStream_t st) -> int {
        if (f4) {
            // A as one stacked matrix (item 0 of a batch of B items)
            const long long ldn = round16((K + 1) / 2);
            SMX_TRY(unpack_nib_ab(A, a8, batch * M, K, lda_w, ldn, nullptr, nullptr, 0, 0, 1, 1, 1, 0, 0, 0, 0,
                                  st));
            SMX_TRY(unpack_nib_ab(nullptr, nullptr, 0, 0, 1, 1, B, bt8, K, N, ldb_w, ldn, batch, 0, 0,
                                  (long long)K * ldb_w, (long long)N * ldn, st));
            return bool_f4_gemm_batched(a8, bt8, C, batch, M, N, K, ldn, ldn, ldc_w, 0, st);
        }
        SMX_TRY(unpack_bits(A, a8, batch * M, K, lda_w, round16(K), st));
        SMX_TRY(unpack_bits_transposed_batched(B, bt8, batch, K, N, ldb_w, round16(K), (long long)K * ldb_w,
                                               (long long)N * round16(K), st));
        return bool_i8_gemm_batched(a8, bt8, C, batch, M, N, K, round16(K), round16(K), ldc_w, 0, st);
    });
}

}  // namespace smx

using namespace smx;

extern "C" {

size_t smx_bool_mul_tc_batched_workspace_bytes(int batch, int M, int N, int K) {
    if (batch <= 0 || M <= 0 || N <= 0 || K <= 0) return 0;
    return bool_mul_batched_ws_bytes(batch, M, N, K);
}

int smx_bool_mul_tc_batched(const uint32_t* A, const uint32_t* B, uint32_t* C, int batch, int M, int N, int K,
                            int lda_w, int ldb_w, int ldc_w, void* ws, size_t ws_bytes, void* stream) {
    return bool_mul_tc_batched(A, B, C, batch, M, N, K, lda_w, ldb_w, ldc_w, ws, ws_bytes, as_stream(stream));
}

int smx_bool_gemm_i8_batched(const uint8_t* A, const uint8_t* Bt, uint32_t* C_bits, int batch, int M, int N, int K,
                             int lda, int ldbt, int ldc, int accumulate, void* stream) {
    return bool_i8_gemm_batched(A, Bt, C_bits, batch, M, N, K, lda, ldbt, ldc, accumulate, as_stream(stream));
}

size_t smx_bool_mul_tc_workspace_bytes(int M, int N, int K) {
    if (M <= 0 || N <= 0 || K <= 0) return 0;
    return bool_mul_ws_bytes(M, N, K);
}

int smx_bool_mul_tc(const uint32_t* A, const uint32_t* B, uint32_t* C, int M, int N, int K, int lda_w,
                    int ldb_w, int ldc_w, void* ws, size_t ws_bytes, void* stream) {
    return bool_mul_tc(A, B, C, M, N, K, lda_w, ldb_w, ldc_w, ws, ws_bytes, as_stream(stream));
}

// development: trace buffer (device, >= 16 + 2 * CTAs u64) for the next
// plain-kernel products; nullptr disarms
int smx_tc_trace_arm(unsigned long long* buf) {
    g_tc_trace = buf;
    return SMX_OK;
}

int smx_bool_gemm_f4(const uint8_t* A, const uint8_t* Bt, uint32_t* C_bits, int M, int N, int K, int lda, int ldbt,
                     int ldc, int accumulate, void* stream) {
    return bool_f4_gemm(A, Bt, C_bits, M, N, K, lda, ldbt, ldc, accumulate, as_stream(stream), /*pdl=*/true);
}

int smx_bool_gemm_f4_batched(const uint8_t* A, const uint8_t* Bt, uint32_t* C_bits, int batch, int M, int N, int K,
                             int lda, int ldbt, int ldc, int accumulate, void* stream) {
    return bool_f4_gemm_batched(A, Bt, C_bits, batch, M, N, K, lda, ldbt, ldc, accumulate, as_stream(stream));
}

int smx_set_tc_f4(int enable) {
    if (enable != 0 && enable != 1) return SMX_E_ARG;
    const int old = g_tc_f4;
    g_tc_f4 = enable;
    return old;
}

int smx_set_tc_f4_batch_stages(int stages) {
    if (stages != 2 && stages != 3) return SMX_E_ARG;
    const int old = g_tc_f4_batch_stages;
    g_tc_f4_batch_stages = stages;
    return old;
}

int smx_set_tc_batch_ks(int ks) {
    if (ks != 1 && ks != 2 && ks != 4) return SMX_E_ARG;
    const int old = g_tc_batch_ks;
    g_tc_batch_ks = ks;
    return old;
}

int smx_set_tc_pair(int mode) {
    if (mode < 0 || mode > 3) return SMX_E_ARG;
    const int old = g_tc_pair;
    g_tc_pair = mode;
    return old;
}

int smx_set_tc_tile_n(int bn) {
    if (bn != 0 && bn != 64 && bn != 128 && bn != 256) return SMX_E_ARG;
    const int old = g_tc_tile_n;
    g_tc_tile_n = bn;
    return old;
}

int smx_bool_gemm_i8(const uint8_t* A, const uint8_t* Bt, uint8_t* C, uint32_t* C_bits, int M, int N, int K,
                     int lda, int ldbt, int ldc, int accumulate, void* stream) {
    // programmatic dependent launch: the kernel touches no memory before its
    // griddepcontrol.wait, so it may overlap its launch and prologue with
    // whatever kernel precedes it in the stream (back-to-back products)
    return bool_i8_gemm(A, Bt, C, C_bits, M, N, K, lda, ldbt, ldc, accumulate, 0, 0, as_stream(stream),
                        /*pdl=*/true);
}

size_t smx_bool_warshall_i8_workspace_bytes(int n, int ld) {
    if (n <= 0 || ld < n) return 0;
    return tc_ws_bytes(n, ld);
}

int smx_bool_warshall_i8(uint8_t* T, int n, int ld, void* ws, size_t ws_bytes, void* stream) {
    return bool_warshall_i8(T, n, ld, ws, ws_bytes, as_stream(stream));
}

}  // extern "C"
