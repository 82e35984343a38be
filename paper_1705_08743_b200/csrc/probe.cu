// Instruction-issue microbenchmark for the roofline denominator of the
// CUDA-core semiring kernels: the packed-integer issue peak
// is MEASURED on the box, not assumed.  Each thread runs 16 independent
// accumulator pairs of exactly the instruction pair the semiring inner loop
// uses (VIMNMX.U16x2 + VIADDMNMX.U16x2), or VIADDMNMX.U16x2 alone (the
// one-instruction form), so the result is the sustained issue rate of the
// same SASS mix on every SM.  bench.py also reports it per SM per clock
// against the nominal 64 lanes/clk/SM of the packed-integer pipe.  Mode 2
// issues the Boolean bit-GEMM's update instead, c = c | (a & b) on 32-bit
// words (one LOP3.LUT = 32 cell-updates): the ceiling of the bit-packed
// Warshall (C2) and bit products (inline PTX, so the compiler cannot fold
// the idempotent OR-of-AND chains across sweeps).
#include "common.cuh"

namespace smx {

template <int MODE>
__global__ void __launch_bounds__(256) int_issue_probe_kernel(uint32_t* sink, int iters, uint32_t seed) {
    // 32 accumulators in 16 independent pairs (c[i] reads c[i ^ 16]): every
    // SMSP has 8+ warps x 16 chains in flight, so latency never binds; 4
    // sweeps per iteration keep the loop and operand bookkeeping (3-4 ops)
    // under 3% of the issued instructions.
    uint32_t c[32];
    uint32_t a = seed * 3u + blockIdx.x, sa = ~a;
#pragma unroll
    for (int i = 0; i < 32; ++i) c[i] = seed + i * 0x01010101u + threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int rep = 0; rep < 4; ++rep) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const uint32_t o = c[i ^ 16];
                if (MODE == 1) c[i] = __viaddmin_u16x2(a, c[i], o);
                else if (MODE == 2)   // (a & b) | c as one LOP3.LUT (asm: no algebraic folding)
                    asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(c[i]) : "r"(c[i]), "r"(a), "r"(o));
                else c[i] = __viaddmin_u16x2(__vminu2(c[i], sa), a, o);
            }
        }
        a += 0x00010001u;
        sa = ~a;
    }
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) x ^= c[i];
    if (x == 0x9E3779B9u) sink[blockIdx.x * blockDim.x + threadIdx.x] = x;  // keep the work
}

}  // namespace smx

extern "C" int smx_int_issue_probe(uint32_t* sink, int blocks, int threads, int iters, int one_instr,
                                   long long* instr_per_thread, void* stream) {
    if (blocks <= 0 || threads <= 0 || threads > 256 || iters <= 0) return SMX_E_ARG;
    // semiring instructions per thread (the loop's 3-6 bookkeeping ops per
    // 128 or 256 semiring instructions are excluded); one_instr: 0 = the
    // VIMNMX + VIADDMNMX pair, 1 = VIADDMNMX alone, 2 = LOP3 (bit OR-of-AND)
    if (one_instr < 0 || one_instr > 2) return SMX_E_ARG;
    if (instr_per_thread) *instr_per_thread = (long long)iters * 4 * (one_instr ? 32 : 64);
    auto st = smx::as_stream(stream);
    if (one_instr == 1)
        smx::int_issue_probe_kernel<1><<<blocks, threads, 0, st>>>(sink, iters, 12345u);
    else if (one_instr == 2)
        smx::int_issue_probe_kernel<2><<<blocks, threads, 0, st>>>(sink, iters, 12345u);
    else
        smx::int_issue_probe_kernel<0><<<blocks, threads, 0, st>>>(sink, iters, 12345u);
    SMX_RETURN_LAUNCH();
}
