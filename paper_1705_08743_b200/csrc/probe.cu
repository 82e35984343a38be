// Instruction-issue microbenchmark for the roofline denominator of the
// CUDA-core semiring kernels: the packed-integer issue peak
// is MEASURED on the box, not assumed.  Each thread runs 16 independent
// accumulator chains of exactly the instruction pair the semiring inner loop
// uses (VIMNMX.U16x2 + VIADDMNMX.U16x2), or VIADDMNMX.U16x2 alone (the u8
// one-instruction form), so the result is the sustained issue rate of the
// same SASS mix on every SM.
#include "common.cuh"

namespace smx {

template <bool ONE>
__global__ void __launch_bounds__(256) int_issue_probe_kernel(uint32_t* sink, int iters, uint32_t seed) {
    uint32_t c[16];
    uint32_t b = seed ^ threadIdx.x, a = seed * 3u + blockIdx.x, sa = ~a;
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = seed + i * 0x01010101u + threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (ONE) c[i] = __viaddmin_u16x2(a, c[i], c[(i + 1) & 15]);
            else c[i] = __viaddmin_u16x2(__vminu2(c[i], sa), a, c[(i + 5) & 15]);
        }
        b += 1u;
        a ^= b;
        sa = ~a;
    }
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) x ^= c[i];
    if (x == 0x9E3779B9u) sink[blockIdx.x * blockDim.x + threadIdx.x] = x;  // keep the work
}

}  // namespace smx

extern "C" int smx_int_issue_probe(uint32_t* sink, int blocks, int threads, int iters, int one_instr,
                                   long long* instr_per_thread, void* stream) {
    if (blocks <= 0 || threads <= 0 || threads > 256 || iters <= 0) return SMX_E_ARG;
    // semiring instructions per thread (the 3 bookkeeping ALU ops per
    // iteration are excluded: they only dilute the measured rate by 3/35)
    if (instr_per_thread) *instr_per_thread = (long long)iters * (one_instr ? 16 : 32);
    if (one_instr)
        smx::int_issue_probe_kernel<true><<<blocks, threads, 0, smx::as_stream(stream)>>>(sink, iters, 12345u);
    else
        smx::int_issue_probe_kernel<false><<<blocks, threads, 0, smx::as_stream(stream)>>>(sink, iters, 12345u);
    SMX_RETURN_LAUNCH();
}
