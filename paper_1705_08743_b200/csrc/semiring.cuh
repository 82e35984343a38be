// Packed-SIMD semiring lane arithmetic for sm_100a CUDA cores.
//
// Every kernel computes in ONE canonical form, the plain-distance (min-plus)
// semiring: (+) = min, (x) = min(a + b, S).  Anti-distance operands
// (pkg/src/semimat/antidist.py:3-8: value a encodes distance S - a) are
// complemented when staged into shared memory and complemented back when the
// result is stored; complement at width is a bitwise NOT (scalars.py:46-52),
// and the anti-distance product max(a+b-S, 0) (scalars.py:36-43) is exactly
// the complement of min((S-a)+(S-b), S).  One code path therefore serves
// AntidistMatrix.__mul__ (antidist.py:226-250) and DistMatrix.__mul__
// (:311-329) bit-exactly.
//
// Per-cell update, all native sm_100a instructions (see profiles/sass_*.txt):
//   u16 : t = vmin.u16x2(b, S-a)          -> VIMNMX.U16x2
//         c = viaddmin.u16x2(t, a, c)      -> VIADDMNMX.U16x2
//         t + a <= S never wraps, so this is min(c, min(a+b, S)) exactly:
//         2 instructions per 2 cells.  This is the paper's saturating lane
//         trick (kernels.py:199-200 np_addsat = min(b, S-a) + a).
//   u8  : widened into u16x2 lanes; a + b <= 510 cannot wrap a 16-bit lane
//         and c starts <= 255, so c = viaddmin.u16x2(a, b, c) alone is exact:
//         1 instruction per 2 cells.
//   u32 : t = min(b, S-a) (IMNMX), c = viaddmin.u32(t, a, c) (VIADDMNMX):
//         2 instructions per cell.
#pragma once
#include "common.cuh"

namespace smx {

template <typename T> struct Lane;

template <> struct Lane<uint16_t> {
    static constexpr int kCellsPerWord = 2;
    static constexpr bool kOneInstr = false;
    static constexpr uint32_t kS = 0xFFFFu;
    static constexpr uint32_t kIdentityWord = 0xFFFFFFFFu;  // S in both lanes
    static constexpr int kCellsPerChunk = 8;                 // 16 B of global
    static constexpr int kWordsPerChunk = 4;
    __device__ __forceinline__ static uint32_t splat(uint32_t v) { return v * 0x10001u; }
    // (+) of two canonical words: lane-wise min
    __device__ __forceinline__ static uint32_t fold(uint32_t x, uint32_t y) { return __vminu2(x, y); }
    __device__ __forceinline__ static uint32_t step(uint32_t c, uint32_t b, uint32_t a,
                                                    uint32_t sa) {
        return __viaddmin_u16x2(__vminu2(b, sa), a, c);
    }
    // lanes below 2^15 on both sides: a + b <= 65534 < S, no clamp needed
    static constexpr uint32_t kHalfMask = 0x80008000u;
    static constexpr uint32_t kCellHalf = 0x8000u;    // the same test on one cell value
    __device__ __forceinline__ static uint32_t step_bounded(uint32_t c, uint32_t b, uint32_t a) {
        return __viaddmin_u16x2(a, b, c);
    }
    // Sparse-bounded certificate and shifted encoding: every lane is either
    // S (unreachable) or < 2^14.  Shifting S to S' = 2^15 - 1 makes every
    // sum <= 65534 (no wrap); finite + finite <= 32766 < S', anything with
    // an S' operand >= S', so "result >= S'" is exactly "unreachable".
    __device__ __forceinline__ static bool cert_ok(uint32_t w) {
        const uint32_t is_s = __vcmpeq2(w, 0xFFFFFFFFu);
        return ((w & ~is_s) & 0xC000C000u) == 0u;
    }
    __device__ __forceinline__ static uint32_t to_shifted(uint32_t w) {
        return w - (__vcmpeq2(w, 0xFFFFFFFFu) & 0x80008000u);
    }
    __device__ __forceinline__ static uint32_t from_shifted(uint32_t w) {
        return w | __vcmpgeu2(w, 0x7FFF7FFFu);
    }
};

template <> struct Lane<uint8_t> {
    static constexpr int kCellsPerWord = 2;
    static constexpr bool kOneInstr = true;
    static constexpr uint32_t kS = 0xFFu;
    static constexpr uint32_t kIdentityWord = 0x00FF00FFu;
    static constexpr int kCellsPerChunk = 16;
    static constexpr int kWordsPerChunk = 8;
    __device__ __forceinline__ static uint32_t splat(uint32_t v) { return v * 0x10001u; }
    __device__ __forceinline__ static uint32_t fold(uint32_t x, uint32_t y) { return __vminu2(x, y); }
    __device__ __forceinline__ static uint32_t step(uint32_t c, uint32_t b, uint32_t a,
                                                    uint32_t /*sa*/) {
        return __viaddmin_u16x2(a, b, c);
    }
    static constexpr uint32_t kHalfMask = 0u;   // always the 1-instruction form
    static constexpr uint32_t kCellHalf = 0u;
    __device__ __forceinline__ static uint32_t step_bounded(uint32_t c, uint32_t b, uint32_t a) {
        return __viaddmin_u16x2(a, b, c);
    }
    __device__ __forceinline__ static bool cert_ok(uint32_t) { return true; }
    __device__ __forceinline__ static uint32_t to_shifted(uint32_t w) { return w; }
    __device__ __forceinline__ static uint32_t from_shifted(uint32_t w) { return w; }
};

template <> struct Lane<uint32_t> {
    static constexpr int kCellsPerWord = 1;
    static constexpr bool kOneInstr = false;
    static constexpr uint32_t kS = 0xFFFFFFFFu;
    static constexpr uint32_t kIdentityWord = 0xFFFFFFFFu;
    static constexpr int kCellsPerChunk = 4;
    static constexpr int kWordsPerChunk = 4;
    __device__ __forceinline__ static uint32_t splat(uint32_t v) { return v; }
    __device__ __forceinline__ static uint32_t fold(uint32_t x, uint32_t y) { return min(x, y); }
    __device__ __forceinline__ static uint32_t step(uint32_t c, uint32_t b, uint32_t a,
                                                    uint32_t sa) {
        return __viaddmin_u32(min(b, sa), a, c);
    }
    static constexpr uint32_t kHalfMask = 0x80000000u;
    static constexpr uint32_t kCellHalf = 0x80000000u;
    __device__ __forceinline__ static uint32_t step_bounded(uint32_t c, uint32_t b, uint32_t a) {
        return __viaddmin_u32(a, b, c);
    }
    // as for u16 with 2^30 / S' = 2^31 - 1
    __device__ __forceinline__ static bool cert_ok(uint32_t w) { return w == kS || w < 0x40000000u; }
    __device__ __forceinline__ static uint32_t to_shifted(uint32_t w) { return w == kS ? 0x7FFFFFFFu : w; }
    __device__ __forceinline__ static uint32_t from_shifted(uint32_t w) { return w >= 0x7FFFFFFFu ? kS : w; }
};

// ---- chunk <-> canonical words ------------------------------------------
// A "chunk" is 16 bytes of global memory (one aligned vector access).
// Canonical words hold distance-form lanes (u16x2 for u8/u16, u32 for u32).

template <typename T>
__device__ __forceinline__ void chunk_to_words(uint4 raw, bool anti, uint32_t* w);

template <> __device__ __forceinline__ void chunk_to_words<uint16_t>(uint4 raw, bool anti,
                                                                     uint32_t* w) {
    const uint32_t m = anti ? 0xFFFFFFFFu : 0u;
    w[0] = raw.x ^ m; w[1] = raw.y ^ m; w[2] = raw.z ^ m; w[3] = raw.w ^ m;
}
template <> __device__ __forceinline__ void chunk_to_words<uint32_t>(uint4 raw, bool anti,
                                                                     uint32_t* w) {
    const uint32_t m = anti ? 0xFFFFFFFFu : 0u;
    w[0] = raw.x ^ m; w[1] = raw.y ^ m; w[2] = raw.z ^ m; w[3] = raw.w ^ m;
}
template <> __device__ __forceinline__ void chunk_to_words<uint8_t>(uint4 raw, bool anti,
                                                                    uint32_t* w) {
    const uint32_t m = anti ? 0xFFFFFFFFu : 0u;
    const uint32_t v[4] = {raw.x ^ m, raw.y ^ m, raw.z ^ m, raw.w ^ m};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        w[2 * i] = __byte_perm(v[i], 0u, 0x4140);      // bytes 0,1 -> u16 lanes
        w[2 * i + 1] = __byte_perm(v[i], 0u, 0x4342);  // bytes 2,3 -> u16 lanes
    }
}

// Lane value of cell j (0-based) of a chunk, in distance form.
template <typename T>
__device__ __forceinline__ uint32_t word_cell(const uint32_t* w, int j) {
    if (Lane<T>::kCellsPerWord == 2) return (w[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu;
    return w[j];
}

// Set cell j of a chunk's canonical words to the lane value v.
template <typename T>
__device__ __forceinline__ void set_word_cell(uint32_t* w, int j, uint32_t v) {
    if (Lane<T>::kCellsPerWord == 2) {
        const int s2 = (j & 1) * 16;
        w[j >> 1] = (w[j >> 1] & ~(0xFFFFu << s2)) | (v << s2);
    } else {
        w[j] = v;
    }
}

// Replace cells [valid, kCellsPerChunk) of a chunk by the (+)-identity S.
template <typename T>
__device__ __forceinline__ void mask_tail(uint32_t* w, int valid) {
    constexpr int CPW = Lane<T>::kCellsPerWord;
#pragma unroll
    for (int i = 0; i < Lane<T>::kWordsPerChunk; ++i) {
        if (CPW == 2) {
            const int c0 = 2 * i;
            if (c0 >= valid) w[i] = Lane<T>::kIdentityWord;
            else if (c0 + 1 >= valid)
                w[i] = (w[i] & 0xFFFFu) | (Lane<T>::kIdentityWord & 0xFFFF0000u);
        } else {
            if (i >= valid) w[i] = Lane<T>::kIdentityWord;
        }
    }
}

// ---- canonical words -> storage ------------------------------------------
// `nwords` words (a multiple of the per-type packing) to storage bytes.
template <typename T, int NW>
__device__ __forceinline__ void words_to_store(const uint32_t* w, bool anti, uint32_t* out);
// u16/u32: one storage word per canonical word
template <> __device__ __forceinline__ void words_to_store<uint16_t, 4>(const uint32_t* w,
                                                                       bool anti, uint32_t* o) {
    const uint32_t m = anti ? 0xFFFFFFFFu : 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = w[i] ^ m;
}
template <> __device__ __forceinline__ void words_to_store<uint16_t, 2>(const uint32_t* w,
                                                                       bool anti, uint32_t* o) {
    const uint32_t m = anti ? 0xFFFFFFFFu : 0u;
    o[0] = w[0] ^ m; o[1] = w[1] ^ m;
}
template <> __device__ __forceinline__ void words_to_store<uint32_t, 4>(const uint32_t* w,
                                                                       bool anti, uint32_t* o) {
    const uint32_t m = anti ? 0xFFFFFFFFu : 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = w[i] ^ m;
}
template <> __device__ __forceinline__ void words_to_store<uint32_t, 2>(const uint32_t* w,
                                                                       bool anti, uint32_t* o) {
    const uint32_t m = anti ? 0xFFFFFFFFu : 0u;
    o[0] = w[0] ^ m; o[1] = w[1] ^ m;
}
// u8: two u16x2 words -> one storage word of 4 bytes
template <> __device__ __forceinline__ void words_to_store<uint8_t, 4>(const uint32_t* w,
                                                                      bool anti, uint32_t* o) {
    const uint32_t m = anti ? 0xFFFFFFFFu : 0u;
    o[0] = __byte_perm(w[0], w[1], 0x6420) ^ m;
    o[1] = __byte_perm(w[2], w[3], 0x6420) ^ m;
}
template <> __device__ __forceinline__ void words_to_store<uint8_t, 2>(const uint32_t* w,
                                                                      bool anti, uint32_t* o) {
    const uint32_t m = anti ? 0xFFFFFFFFu : 0u;
    o[0] = __byte_perm(w[0], w[1], 0x6420) ^ m;
}

}  // namespace smx
