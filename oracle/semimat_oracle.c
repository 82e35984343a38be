/*
 * semimat CPU oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain-C restatement of the reference package's compute engines
 * (arxiv/paper_1705_08743, package `semimat`, pkg/src/semimat/), used only by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg as the checker.  The product path never links or calls this.
 *
 * Parity of this restatement with the reference is PINNED by
 * tests/test_oracle_golden.py against golden vectors produced by running the
 * reference itself (tests/golden/make_golden.py).
 *
 * Every engine follows the reference's outer-product sweep, including its
 * zero-skip (anti-distance skips A[i,k] == 0, min-plus skips A[i,k] == S,
 * Boolean skips clear bits).  The only restructuring is loop interchange to
 * row-outer order so rows can be split across OpenMP threads: each output
 * row folds the same candidate rows with the same associative, commutative
 * integer max/min/or, so the result is bit-identical to the k-outer order.
 *
 * All matrices are row-major with explicit leading dimensions (in elements).
 * `cols` is the padded width the reference operates on (it sweeps whole
 * padded rows, pkg/src/semimat/antidist.py:38-55).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_API __attribute__((visibility("default")))

static int orc_threads(int requested) {
#ifdef _OPENMP
    return requested > 0 ? requested : omp_get_max_threads();
#else
    (void)requested;
    return 1;
#endif
}

/* ---------------------------------------------------------------------------
 * Anti-distance product: _mul_vector, pkg/src/semimat/antidist.py:361-371.
 *   out starts at 0 (:362); for each k, rows with a[r,k] != 0 (:364-366)
 *   fold  max(b[k,:], gap) - gap  with gap = S - a[r,k]  (:367-368, the
 *   np_subsat rewrite of kernels.py:195-196) into out[r,:] by max (:369-370).
 * Min-plus product: _minplus_mul_vector, antidist.py:412-422.
 *   out starts at S (:413); rows with a[r,k] != S (:416) fold
 *   min(b[k,:], S - e) + e  (np_addsat, kernels.py:199-200) by min (:419-421).
 * ------------------------------------------------------------------------- */
#define DEFINE_MUL(T, SUF)                                                         \
ORC_API void orc_anti_mul_##SUF(const T* a, const T* b, T* out, int64_t rows,       \
                                int64_t inner, int64_t cols, int64_t lda,          \
                                int64_t ldb, int64_t ldo, uint32_t limit,          \
                                int threads) {                                     \
    const T S = (T)limit;                                                          \
    _Pragma("omp parallel for schedule(dynamic, 4) num_threads(orc_threads(threads))") \
    for (int64_t r = 0; r < rows; ++r) {                                           \
        T* o = out + r * ldo;                                                      \
        memset(o, 0, (size_t)cols * sizeof(T));                                    \
        const T* ar = a + r * lda;                                                 \
        for (int64_t k = 0; k < inner; ++k) {                                      \
            const T e = ar[k];                                                     \
            if (e == 0) continue;                                                  \
            const T gap = (T)(S - e);                                              \
            const T* bk = b + k * ldb;                                             \
            for (int64_t j = 0; j < cols; ++j) {                                   \
                const T x = bk[j];                                                 \
                const T cand = (T)((x > gap ? x : gap) - gap);                     \
                o[j] = o[j] > cand ? o[j] : cand;                                  \
            }                                                                      \
        }                                                                          \
    }                                                                              \
}                                                                                  \
ORC_API void orc_minplus_mul_##SUF(const T* a, const T* b, T* out, int64_t rows,    \
                                   int64_t inner, int64_t cols, int64_t lda,       \
                                   int64_t ldb, int64_t ldo, uint32_t limit,       \
                                   int threads) {                                  \
    const T S = (T)limit;                                                          \
    _Pragma("omp parallel for schedule(dynamic, 4) num_threads(orc_threads(threads))") \
    for (int64_t r = 0; r < rows; ++r) {                                           \
        T* o = out + r * ldo;                                                      \
        for (int64_t j = 0; j < cols; ++j) o[j] = S;                               \
        const T* ar = a + r * lda;                                                 \
        for (int64_t k = 0; k < inner; ++k) {                                      \
            const T e = ar[k];                                                     \
            if (e == S) continue;                                                  \
            const T room = (T)(S - e);                                             \
            const T* bk = b + k * ldb;                                             \
            for (int64_t j = 0; j < cols; ++j) {                                   \
                const T x = bk[j];                                                 \
                const T cand = (T)((x < room ? x : room) + e);                     \
                o[j] = o[j] < cand ? o[j] : cand;                                  \
            }                                                                      \
        }                                                                          \
    }                                                                              \
}

/* ---------------------------------------------------------------------------
 * Closures (Floyd-Warshall over the semiring), in place on t:
 *   _close_vector, antidist.py:390-398 and _minplus_close_vector, :440-448.
 * For each k in order, every row r whose column-k entry is non-identity is
 * folded with the candidate built from row k as it stood at the start of
 * step k (numpy materialises `cand` from t[k] before the scatter, :395-398),
 * and the column value is read before row r is rewritten (:392-394).  Row k
 * is therefore snapshotted once per step; rows are then independent.
 * ------------------------------------------------------------------------- */
#define DEFINE_CLOSE(T, SUF)                                                       \
ORC_API void orc_anti_close_##SUF(T* t, int64_t dim, int64_t cols, int64_t ld,      \
                                  uint32_t limit, int threads) {                   \
    const T S = (T)limit;                                                          \
    T* pivot = (T*)malloc((size_t)cols * sizeof(T));                               \
    const int nt = orc_threads(threads);                                           \
    for (int64_t k = 0; k < dim; ++k) {                                            \
        memcpy(pivot, t + k * ld, (size_t)cols * sizeof(T));                       \
        _Pragma("omp parallel for schedule(static) num_threads(nt)")               \
        for (int64_t r = 0; r < dim; ++r) {                                        \
            T* row = t + r * ld;                                                   \
            const T e = row[k];                                                    \
            if (e == 0) continue;                                                  \
            const T gap = (T)(S - e);                                              \
            for (int64_t j = 0; j < cols; ++j) {                                   \
                const T x = pivot[j];                                              \
                const T cand = (T)((x > gap ? x : gap) - gap);                     \
                row[j] = row[j] > cand ? row[j] : cand;                            \
            }                                                                      \
        }                                                                          \
    }                                                                              \
    free(pivot);                                                                   \
}                                                                                  \
ORC_API void orc_minplus_close_##SUF(T* t, int64_t dim, int64_t cols, int64_t ld,   \
                                     uint32_t limit, int threads) {                \
    const T S = (T)limit;                                                          \
    T* pivot = (T*)malloc((size_t)cols * sizeof(T));                               \
    const int nt = orc_threads(threads);                                           \
    for (int64_t k = 0; k < dim; ++k) {                                            \
        memcpy(pivot, t + k * ld, (size_t)cols * sizeof(T));                       \
        _Pragma("omp parallel for schedule(static) num_threads(nt)")               \
        for (int64_t r = 0; r < dim; ++r) {                                        \
            T* row = t + r * ld;                                                   \
            const T e = row[k];                                                    \
            if (e == S) continue;                                                  \
            const T room = (T)(S - e);                                             \
            for (int64_t j = 0; j < cols; ++j) {                                   \
                const T x = pivot[j];                                              \
                const T cand = (T)((x < room ? x : room) + e);                     \
                row[j] = row[j] < cand ? row[j] : cand;                            \
            }                                                                      \
        }                                                                          \
    }                                                                              \
    free(pivot);                                                                   \
}

DEFINE_MUL(uint8_t, u8)
DEFINE_MUL(uint16_t, u16)
DEFINE_MUL(uint32_t, u32)
DEFINE_CLOSE(uint8_t, u8)
DEFINE_CLOSE(uint16_t, u16)
DEFINE_CLOSE(uint32_t, u32)

/* ---------------------------------------------------------------------------
 * Boolean matrices on the reference's storage: uint64 blocks, bit j of a row
 * in block j>>6 at position j&63, LSB first (pkg/src/semimat/boolmat.py:3-5).
 *
 * Product, boolmat.py:151-172: p starts at 0 (:164); for each k, rows whose
 * column-k bit of a is set (:168-169) OR in row k of b (:170-171).
 * Closure, boolmat.py:174-189: the same sweep on a copy, in place, rows
 * folded with row k as it stood at the start of step k (`t[hit] |= t[k]`
 * evaluates t[k] before the scatter).
 * ------------------------------------------------------------------------- */
ORC_API void orc_bool_mul(const uint64_t* a, const uint64_t* b, uint64_t* p,
                          int64_t rows, int64_t inner, int64_t bwords,
                          int64_t lda, int64_t ldb, int64_t ldp, int threads) {
    _Pragma("omp parallel for schedule(dynamic, 8) num_threads(orc_threads(threads))")
    for (int64_t r = 0; r < rows; ++r) {
        uint64_t* pr = p + r * ldp;
        memset(pr, 0, (size_t)bwords * sizeof(uint64_t));
        const uint64_t* ar = a + r * lda;
        for (int64_t k = 0; k < inner; ++k) {
            if (!((ar[k >> 6] >> (k & 63)) & 1u)) continue;
            const uint64_t* bk = b + k * ldb;
            for (int64_t w = 0; w < bwords; ++w) pr[w] |= bk[w];
        }
    }
}

ORC_API void orc_bool_close(uint64_t* t, int64_t dim, int64_t bwords, int64_t ld,
                            int threads) {
    uint64_t* pivot = (uint64_t*)malloc((size_t)bwords * sizeof(uint64_t));
    const int nt = orc_threads(threads);
    for (int64_t k = 0; k < dim; ++k) {
        memcpy(pivot, t + k * ld, (size_t)bwords * sizeof(uint64_t));
        _Pragma("omp parallel for schedule(static) num_threads(nt)")
        for (int64_t r = 0; r < dim; ++r) {
            uint64_t* row = t + r * ld;
            if (!((row[k >> 6] >> (k & 63)) & 1u)) continue;
            for (int64_t w = 0; w < bwords; ++w) row[w] |= pivot[w];
        }
    }
    free(pivot);
}

ORC_API int orc_max_threads(void) { return orc_threads(0); }

/* ---------------------------------------------------------------------------
 * Cache-blocked restatement of the same closures (test infrastructure for the
 * full-size C5 pin, n = 32768, where the plain k-sweep above streams the whole
 * 2 GiB matrix once per k and would take hours on the build host).
 *
 * Same per-cell arithmetic as _close_vector / _minplus_close_vector
 * (antidist.py:390-398, :440-448; the np_subsat / np_addsat rewrites of
 * kernels.py:195-200) and the same zero / S skip; only the order of the
 * (i, j, k) updates changes, to the classic blocked three-phase schedule:
 *   1. the pivot tile T[K,K] by the plain in-place k-sweep;
 *   2. the pivot row panel T[K,J] and column panel T[I,K], k-sweep over K
 *      with the closed pivot tile;
 *   3. every other tile T[I,J] (+)= T[I,K] (x) T[K,J].
 * That this order is bit-identical to the reference's vertex-at-a-time sweep
 * is SURVEY.md 0.1 fact 2 (x -> min(x, S) is a semiring homomorphism from
 * (min,+) on [0,inf]); tests/test_oracle_golden.py checks it against the
 * plain sweep above and against the reference's own sha256 of the C4 n = 8192
 * closure, so it is pinned independently of the GPU path.
 * ------------------------------------------------------------------------- */
#define ORC_BLK 128
#define ORC_JT 2048

#define DEFINE_CLOSE_BLOCKED(T, SUF)                                               \
static void orc_fold_anti_##SUF(T* o, const T* x, T e, T S, int64_t n) {          \
    const T gap = (T)(S - e);                                                      \
    for (int64_t j = 0; j < n; ++j) {                                              \
        const T v = x[j];                                                          \
        const T cand = (T)((v > gap ? v : gap) - gap);                             \
        o[j] = o[j] > cand ? o[j] : cand;                                          \
    }                                                                              \
}                                                                                  \
static void orc_fold_minplus_##SUF(T* o, const T* x, T e, T S, int64_t n) {       \
    const T room = (T)(S - e);                                                     \
    for (int64_t j = 0; j < n; ++j) {                                              \
        const T v = x[j];                                                          \
        const T cand = (T)((v < room ? v : room) + e);                             \
        o[j] = o[j] < cand ? o[j] : cand;                                          \
    }                                                                              \
}                                                                                  \
/* k-outer sweep of rows [i0,i1) x cols [j0,j1) over pivots [k0,k1) */            \
static void orc_sweep_##SUF(T* t, int64_t ld, int64_t i0, int64_t i1, int64_t j0,  \
                            int64_t j1, int64_t k0, int64_t k1, T S, int anti) {   \
    for (int64_t k = k0; k < k1; ++k)                                              \
        for (int64_t i = i0; i < i1; ++i) {                                        \
            const T e = t[i * ld + k];                                             \
            if (anti ? e == 0 : e == S) continue;                                  \
            if (anti) orc_fold_anti_##SUF(t + i * ld + j0, t + k * ld + j0, e, S, j1 - j0); \
            else orc_fold_minplus_##SUF(t + i * ld + j0, t + k * ld + j0, e, S, j1 - j0); \
        }                                                                          \
}                                                                                  \
static void orc_close_blocked_##SUF(T* t, int64_t dim, int64_t cols, int64_t ld,    \
                                    uint32_t limit, int threads, int anti) {       \
    const T S = (T)limit;                                                          \
    const int nt = orc_threads(threads);                                           \
    const int64_t nb = (dim + ORC_BLK - 1) / ORC_BLK;                              \
    const int64_t njt = (cols + ORC_JT - 1) / ORC_JT;                              \
    for (int64_t kb = 0; kb < nb; ++kb) {                                          \
        const int64_t k0 = kb * ORC_BLK, k1 = k0 + ORC_BLK < dim ? k0 + ORC_BLK : dim; \
        orc_sweep_##SUF(t, ld, k0, k1, k0, k1, k0, k1, S, anti);                   \
        /* row panel T[K, outside K] (padding columns included) and column    \
         * panel T[outside K, K]; both read only the closed pivot tile and     \
         * their own tiles */                                                  \
        _Pragma("omp parallel for schedule(dynamic, 1) num_threads(nt)")          \
        for (int64_t x = 0; x < njt + nb; ++x) {                                  \
            if (x < njt) {                                                         \
                int64_t j0 = x * ORC_JT, j1 = j0 + ORC_JT < cols ? j0 + ORC_JT : cols; \
                if (j0 < k0) {                                                     \
                    int64_t e1 = j1 < k0 ? j1 : k0;                                \
                    orc_sweep_##SUF(t, ld, k0, k1, j0, e1, k0, k1, S, anti);       \
                }                                                                  \
                if (j1 > k1) {                                                     \
                    int64_t s0 = j0 > k1 ? j0 : k1;                                \
                    orc_sweep_##SUF(t, ld, k0, k1, s0, j1, k0, k1, S, anti);       \
                }                                                                  \
            } else {                                                               \
                int64_t ib = x - njt;                                              \
                if (ib == kb) continue;                                            \
                int64_t i0 = ib * ORC_BLK, i1 = i0 + ORC_BLK < dim ? i0 + ORC_BLK : dim; \
                orc_sweep_##SUF(t, ld, i0, i1, k0, k1, k0, k1, S, anti);           \
            }                                                                      \
        }                                                                          \
        /* everything else: T[I,J] (+)= T[I,K] (x) T[K,J], rows i-outer */       \
        _Pragma("omp parallel for schedule(dynamic, 1) num_threads(nt)")          \
        for (int64_t x = 0; x < nb * njt; ++x) {                                  \
            const int64_t ib = x / njt, jt = x % njt;                              \
            if (ib == kb) continue;                                                \
            const int64_t i0 = ib * ORC_BLK, i1 = i0 + ORC_BLK < dim ? i0 + ORC_BLK : dim; \
            const int64_t j0 = jt * ORC_JT, j1 = j0 + ORC_JT < cols ? j0 + ORC_JT : cols; \
            for (int64_t i = i0; i < i1; ++i) {                                    \
                T* row = t + i * ld;                                               \
                for (int64_t k = k0; k < k1; ++k) {                                \
                    const T e = row[k];                                            \
                    if (anti ? e == 0 : e == S) continue;                          \
                    /* skip the pivot columns: they are the column panel,      \
                     * already final */                                        \
                    if (j0 < k0) {                                                 \
                        int64_t e1 = j1 < k0 ? j1 : k0;                            \
                        if (anti) orc_fold_anti_##SUF(row + j0, t + k * ld + j0, e, S, e1 - j0); \
                        else orc_fold_minplus_##SUF(row + j0, t + k * ld + j0, e, S, e1 - j0); \
                    }                                                              \
                    if (j1 > k1) {                                                 \
                        int64_t s0 = j0 > k1 ? j0 : k1;                            \
                        if (anti) orc_fold_anti_##SUF(row + s0, t + k * ld + s0, e, S, j1 - s0); \
                        else orc_fold_minplus_##SUF(row + s0, t + k * ld + s0, e, S, j1 - s0); \
                    }                                                              \
                }                                                                  \
            }                                                                      \
        }                                                                          \
    }                                                                              \
}                                                                                  \
ORC_API void orc_anti_close_blocked_##SUF(T* t, int64_t dim, int64_t cols, int64_t ld, \
                                          uint32_t limit, int threads) {           \
    orc_close_blocked_##SUF(t, dim, cols, ld, limit, threads, 1);                  \
}                                                                                  \
ORC_API void orc_minplus_close_blocked_##SUF(T* t, int64_t dim, int64_t cols, int64_t ld, \
                                             uint32_t limit, int threads) {        \
    orc_close_blocked_##SUF(t, dim, cols, ld, limit, threads, 0);                  \
}

DEFINE_CLOSE_BLOCKED(uint8_t, u8)
DEFINE_CLOSE_BLOCKED(uint16_t, u16)
DEFINE_CLOSE_BLOCKED(uint32_t, u32)
