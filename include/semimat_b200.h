/*
 * semimat_b200 -- C ABI of the B200-native semiring kernels.
 *
 * Drop-in boundary for the hot path of arxiv/paper_1705_08743 (package
 * `semimat`).  The reference has no FFI: its "operator API" is the Python
 * class surface (pkg/src/semimat/__init__.py:10-27) and the private engines
 * that `kernels.use_vector()` selects (pkg/src/semimat/kernels.py:58-64).
 * Each entry point below replaces one of those engines; the Python classes in
 * paper_1705_08743_b200/ keep the reference's class API and call these.
 *
 * Conventions
 *   - All matrix pointers are DEVICE pointers, row-major, with leading
 *     dimensions in elements.  Base pointers must be 16-byte aligned and
 *     ld * sizeof(elem) a multiple of 16 (the reference pads every lane row to
 *     a whole 128-bit block, antidist.py:38-55, so its layout satisfies this).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *   - Every call is asynchronous on `stream`, allocates nothing persistent and
 *     returns 0 on success, a negative SMX_E* code for argument errors, or a
 *     positive cudaError_t from the launch.
 *   - kind: SMX_ANTI = anti-distance (0 = unreachable, S = distance 0;
 *     (+) = max, (x) = max(a+b-S,0)); SMX_DIST = plain distance (S =
 *     unreachable; (+) = min, (x) = min(a+b,S)).  S = 2^w - 1.
 *   - accumulate = 0: C = A (x) B          (the reference __mul__ contract,
 *                                           output starts at the (+)-identity)
 *     accumulate = 1: C = C (+) A (x) B    (Floyd-Warshall phases 2/3)
 */
#ifndef SEMIMAT_B200_H
#define SEMIMAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SMX_OK = 0,
    SMX_E_ARG = -1,      /* bad size / kind / flag */
    SMX_E_ALIGN = -2,    /* pointer or leading dimension not 16-byte aligned */
    SMX_E_WORKSPACE = -3,/* workspace missing or too small */
    SMX_E_DRIVER = -4,   /* driver entry point (TMA descriptor encode) unavailable */
    SMX_E_COMM = -5      /* the exchange (broadcast callback / NCCL) failed or is unavailable */
};
enum { SMX_ANTI = 0, SMX_DIST = 1 };

int smx_version(void);
const char* smx_error_string(int code);
/* Number of kernels this library has launched in the process so far. */
unsigned long long smx_launch_count(void);
/* Output tiles per CTA of the packed semiring GEMM (phase 3 and the large
 * products): 1 (default) or 2 adjacent row tiles walked through one
 * continuous operand ring.  Results are identical.  Returns the previous
 * setting. */
int smx_set_packed_tiles_per_cta(int tpc);
/* How the packed GEMM's producer warp waits for a free ring slot: 0 = a bare
 * mbarrier.try_wait loop, ns > 0 = try_wait with that suspend-time hint (ns),
 * ns < 0 = nanosleep(-ns) between polls (|ns| clamped to 100000).  Results are
 * identical.  Returns the previous setting. */
int smx_set_packed_producer_backoff(int ns);
/* The u16/u32 semiring kernels run a k-tile with the 1-instruction update
 * c = min(c, a + b) when the CTA has verified that every staged lane of that
 * k-tile is below 2^(w-1) (so a + b cannot reach S and the clamp is a
 * no-op); otherwise the general 2-instruction update.  The public products
 * (smx_semiring_gemm_u16/u32) additionally certify every A row and B column
 * as "S or < 2^(w-2)" in a first pass; a CTA whose rows, columns and C tile
 * are all certified runs its whole K loop with the 1-instruction update in
 * a shifted encoding (S -> 2^(w-1)-1, results >= that map back to S), which
 * covers sparse inputs with unreachable entries.  Results are identical;
 * this switch (default on) forces the general form.  Returns the old value. */
int smx_set_bounded_fastpath(int enable);

/* ---- saturated lane semiring products ---------------------------------
 * Replace _mul_vector (pkg/src/semimat/antidist.py:361-371, called from
 * AntidistMatrix.__mul__ :226-250) and _minplus_mul_vector (:412-422, called
 * from DistMatrix.__mul__ :311-329).  C is M x N, A is M x K, B is K x N. */
int smx_semiring_gemm_u8(const uint8_t* A, const uint8_t* B, uint8_t* C,
                         int M, int N, int K, int lda, int ldb, int ldc,
                         int kind, int accumulate, void* stream);
int smx_semiring_gemm_u16(const uint16_t* A, const uint16_t* B, uint16_t* C,
                          int M, int N, int K, int lda, int ldb, int ldc,
                          int kind, int accumulate, void* stream);
int smx_semiring_gemm_u32(const uint32_t* A, const uint32_t* B, uint32_t* C,
                          int M, int N, int K, int lda, int ldb, int ldc,
                          int kind, int accumulate, void* stream);

/* ---- Floyd-Warshall closures (blocked three-phase) ---------------------
 * Replace _close_vector (antidist.py:390-398, from AntidistMatrix.
 * transitive_close :252-261) and _minplus_close_vector (:440-448, from
 * DistMatrix.transitive_close :331-340).  In place on the n x n matrix T
 * (row stride ld >= n).  `workspace` is caller-owned device memory of at
 * least smx_fw_workspace_bytes(n, ld, elem_bytes) bytes. */
size_t smx_fw_workspace_bytes(int n, int ld, int elem_bytes);
int smx_fw_u8(uint8_t* T, int n, int ld, int kind, void* workspace, size_t ws_bytes,
              void* stream);
int smx_fw_u16(uint16_t* T, int n, int ld, int kind, void* workspace, size_t ws_bytes,
               void* stream);
int smx_fw_u32(uint32_t* T, int n, int ld, int kind, void* workspace, size_t ws_bytes,
               void* stream);

/* Host -> device copy of `bytes` from `src` (any host memory) into `dst`,
 * ordered on `stream`.  Page-locked sources (and copies under 8 MB) are one
 * cudaMemcpyAsync; larger pageable ones are staged through the library's
 * page-locked ring by a pool of memcpy threads (host_stage.cu: ~47 GB/s of
 * memcpy against ~11 GB/s for a pageable cudaMemcpy on the pool's hosts),
 * and the call returns once `src` has been read in full.  Used when a
 * host-backed matrix moves to HBM. */
int smx_copy_h2d(void* dst, const void* src, size_t bytes, void* stream);

/* Closure of a matrix held in HOST memory: the same result as
 * copying host_in (n x ld, row-major, the reference's padded layout) into T,
 * smx_fw_*, and copying T back into host_out -- the user-visible work of
 * AntidistMatrix(.., data).transitive_closure().data (antidist.py:263-273)
 * -- with the two PCIe copies overlapped with the closure: rows are copied
 * in group by group and enter the rounds as they arrive, and the last rows'
 * result is copied out chunk by chunk while the rest finishes (fw.cu,
 * fw_host_run).  T (device, n x ld) is the working matrix and holds the
 * closure afterwards too.  host_out may equal host_in.  Stream-ordered:
 * host_out is complete once `stream` reaches the end of the call.  Page-locked
 * host buffers give the overlap; a pageable host_in is staged through the
 * library's page-locked ring by a memcpy thread pool, overlapped the same way
 * (host_stage.cu); a pageable host_out (e.g. the caller's own array closed
 * in place) is staged back through the same ring, its copies overlapped with
 * the rest of the closure, and the call returns once every row is in it.
 * `workspace`: smx_fw_host_workspace_bytes(n, ld, elem_bytes) bytes. */
size_t smx_fw_host_workspace_bytes(int n, int ld, int elem_bytes);
int smx_fw_host_u8(const uint8_t* host_in, uint8_t* host_out, uint8_t* T, int n, int ld, int kind,
                   void* workspace, size_t ws_bytes, void* stream);
int smx_fw_host_u16(const uint16_t* host_in, uint16_t* host_out, uint16_t* T, int n, int ld,
                    int kind, void* workspace, size_t ws_bytes, void* stream);
/* Streamed schedule of smx_fw_host_*: 0 = never (copy in, close, copy out),
 * 1 = automatic (default: from n = 16384), 2 = whenever the closure has at
 * least 8 pivot blocks.  Results are identical.  Returns the previous mode
 * (or SMX_E_ARG). */
int smx_set_fw_host_stream(int mode);
int smx_fw_host_u32(const uint32_t* host_in, uint32_t* host_out, uint32_t* T, int n, int ld,
                    int kind, void* workspace, size_t ws_bytes, void* stream);

/* smx_fw_* overlap each pivot block's phase 1/2 with the previous round's
 * phase 3 on an internal high-priority side stream (forked from and joined
 * back into `stream` with events, so it is graph-capturable).  Passing 0
 * selects the plain serial schedule; results are identical.  Returns the
 * previous setting. */
int smx_set_fw_lookahead(int enable);
/* Pivot tiles of up to 128 vertices (u8/u16): 1 = the blocked kernel (32-
 * vertex sub-blocks, 7 barriers each; default), 0 = the register kernel (one
 * barrier per vertex).  Results are identical.  Returns the previous setting. */
int smx_set_fw_pivot_blocked(int enable);
/* Bit-packed Boolean GEMM (smx_bool_gemm_bits and the bit Warshall): 1 = the
 * four-Russians kernel (per 32 k, 8 nibble-table lookups; default), 0 = the
 * per-k predicate kernel.  Results are identical.  Returns the previous
 * setting. */
int smx_set_bits_m4r(int enable);
/* Bit Warshall for 512 <= n <= 8192, n a multiple of 256: 1 = one persistent
 * cooperative launch for the whole closure (a work queue of row panel / 3a /
 * 3b tiles synchronised by device counters, the pivot closed by the CTA that
 * finishes the last 3a tile); 0 (default, faster as measured) = the blocked
 * schedule of one launch per phase.  Results are identical.  Returns the
 * previous setting. */
int smx_set_bool_persistent(int enable);
/* Pivot block of the blocked bit Warshall: 0 = automatic (256, or 512 from
 * n = 8192), or force 128 / 256 / 512.  Results are identical.  Returns the
 * previous setting (or SMX_E_ARG). */
int smx_set_bool_block(int block);
/* Development trace of the persistent closure: buf (device, 4 * cap_items
 * u64) receives per work item start / dependencies-met / end globaltimer
 * stamps and (CTA, type, round); the last R slots hold the pivots.  NULL
 * disarms.  Graph replay is keyed without it: use with smx_set_graphs(0). */
int smx_bool_persist_trace_arm(unsigned long long* buf, int cap_items);
/* Graph replay of multi-launch calls (smx_fw_*, smx_bool_warshall_bits,
 * smx_bool_warshall_i8, smx_bool_mul_tc): the first call with a given
 * (entry, pointers, sizes, switches) launches eagerly, the second records its
 * launches into a CUDA graph, later identical calls replay it with one
 * cudaGraphLaunch on `stream` (16 graphs kept, LRU).
 * Calls on a stream that is itself being captured run eagerly into the
 * caller's capture.  1 = on (default), 0 = always launch eagerly.  Results
 * are identical.  Returns the previous setting. */
int smx_set_graphs(int enable);
/* Side-stream kernels of the look-ahead: 1 = the small-footprint pivot
 * (tile in shared memory) and row-panel tiles that fit beside phase-3 CTAs;
 * 0 (default) = the regular pivot and tiles.  Results are identical.
 * Returns the previous setting. */
int smx_set_fw_side_lite(int enable);
/* Look-ahead 3a (round r's update of the next pivot block's rows) in two
 * parts: the diagonal tile first with the pivot right behind it on the side
 * stream, the other columns on a second side stream beside the pivot.
 * 0 = never (one launch before the pivot), 1 = automatic (default;
 * currently never: it measured no net gain), 2 = always.
 * Results are identical.  Returns the previous setting. */
int smx_set_fw_split_3a(int mode);
/* Pivot tiles above 128 vertices close by a 2 x 2 blocked recursion; its two
 * independent panel products per half run as one launch (1, default) or as
 * two (0).  Results are identical.  Returns the previous setting. */
int smx_set_fw_pivot_pairs(int enable);
/* Row panel of the look-ahead closure on the packed kernel (the closed
 * pivot tile and the panel packed into the row-panel workspace region
 * first) or on the register-staged tiles: 0 = never, 1 = automatic (default:
 * n >= 8192, where it measured faster), 2 = always.  Results are identical.
 * Returns the previous setting. */
int smx_set_fw_packed_panel(int mode);
/* Packed row-panel buffers of the look-ahead closure: 2 (default) = double
 * buffered, the side stream packs the next round's row panel beside the
 * current phase 3; 1 = one buffer, packed on the main stream between the
 * phase-3 launches.  Results are identical.  Returns the previous setting. */
int smx_set_fw_panel_buffers(int count);
/* Pivot block of smx_fw_*: 0 = automatic (u16: 512 at n >= 16384, 256 at
 * n >= 8192; u8: 256 at n >= 8192; else 128), or force 128 / 256 / 512
 * (clamped to smx_fw_block: u8 256, u32 128).  Returns the previous setting
 * (or SMX_E_ARG). */
int smx_set_fw_block(int block);
/* Packed u8/u16 kernel: 1 (default) = smx_fw_u8/u16's phase 3, large
 * smx_semiring_gemm_u8/u16 products (M*N >= 2^22, K >= 256) and large
 * smx_semiring_gemm_skip u8/u16 updates pack their operands into canonical
 * tiles (with per-tile bounded flags, or for u16 products the product-wide
 * shifted encoding when a certificate pass allows it) and run the
 * warp-specialised bulk-copy kernel; 0 = the register-staged kernel.
 * Results are identical.  Returns the previous setting. */
int smx_set_fw_packed(int enable);

/* Measurement hook: arm a CUDA-event trace of up to max_launches phase-3
 * launches (the dominant kernel) of the following smx_fw_* calls; read back
 * each launch's duration (ms) and cell-updates; returns the count (< 0 on a
 * CUDA error).  Reading disarms the trace. */
int smx_fw_trace_arm(int max_launches);
/* Begin / end (ms) of every traced launch relative to the first one's
 * begin: the gaps between phase-3 launches.  Call before smx_fw_trace_read,
 * which disarms the trace.  Returns the count, or -(cudaError_t). */
int smx_fw_trace_offsets(float* begin_ms, float* end_ms, int cap);
int smx_fw_trace_read(float* ms, long long* cells, int cap);

/* Building blocks of the blocked FW, exported for the row-panel-sharded
 * multi-GPU driver (paper_1705_08743_b200/sharded.py).  elem_bytes in
 * {1,2,4}.  Pivot tile: b x b (b <= smx_fw_block(elem_bytes)), in place. */
int smx_fw_block(int elem_bytes);
/* The pivot block smx_fw_* uses for an n-vertex closure under the current
 * smx_set_fw_block setting (<= smx_fw_block(elem_bytes)). */
int smx_fw_block_for(int n, int elem_bytes);
int smx_fw_pivot(void* P, int b, int ld, int elem_bytes, int kind, void* stream);
/* C[rows, :] (+)= A (x) B over rows [0, M) except the row-tile range
 * [skip_row0, skip_row0 + skip_rows), which must be multiples of 128. */
int smx_semiring_gemm_skip(const void* A, const void* B, void* C, int M, int N, int K,
                           int lda, int ldb, int ldc, int elem_bytes, int kind,
                           int skip_row0, int skip_rows, void* stream);
/* The same product with an operand certificate first (u16): if every lane of
 * A and B is unreachable or < 2^14, all tiles run the 1-instruction shifted
 * encoding.  For the first rounds of a closure, whose operands are the
 * mostly unreachable input graph; same result. */
int smx_semiring_gemm_skip_certified(const void* A, const void* B, void* C, int M, int N, int K,
                                     int lda, int ldb, int ldc, int elem_bytes, int kind,
                                     int skip_row0, int skip_rows, void* stream);

/* ---- row-panel-sharded Floyd-Warshall, one call per rank
 * Rank `rank` of `world` holds rows [row0, row0 + rows) of the n x n matrix
 * (row stride ld) at T, where row0 = rank * per, per = ceil(n / world)
 * rounded up to whole `block`s (smx_fw_sharded_block).  Closes its rows in
 * place: per pivot block the owner closes the pivot tile and updates its row
 * panel, the panel (block x ld lanes) is broadcast with `bcast`, and every
 * rank folds it into its rows; pipelined so the owner's chain and the
 * broadcast of block r+1 run on a high-priority side stream beside round r.
 * The gathered panels equal smx_fw_*'s closure bit for bit.  Replaces the
 * reference's _close_vector / _minplus_close_vector (antidist.py:390-398,
 * :440-448) for a matrix spread over GPUs.
 *
 * bcast(buf, bytes, root, ctx, stream): broadcast `bytes` at device pointer
 * buf from rank `root` to every rank, ordered on `stream` (enqueue or
 * complete before returning); return 0 on success.  smx_nccl_broadcast is
 * one (ctx = an ncclComm_t); any other transport can be plugged in.
 * Workspace: smx_fw_sharded_workspace_bytes(rows, ld, elem_bytes, block). */
typedef int (*smx_bcast_fn)(void* buf, size_t bytes, int root, void* ctx, void* stream);
int smx_nccl_broadcast(void* buf, size_t bytes, int root, void* nccl_comm, void* stream);
/* ncclCommGetAsyncError on the communicator: 0 = healthy, SMX_E_COMM = an
 * asynchronous failure was recorded (smx_nccl_broadcast also checks it before
 * every broadcast, so a sharded closure on a failed communicator returns
 * SMX_E_COMM instead of hanging in the next collective). */
int smx_nccl_async_error(void* nccl_comm);
int smx_fw_sharded_block(int n, int world, int elem_bytes);
size_t smx_fw_sharded_workspace_bytes(int rows, int ld, int elem_bytes, int block);
int smx_fw_sharded(void* T, int n, int row0, int rows, int ld, int elem_bytes, int kind, int rank,
                   int world, int block, smx_bcast_fn bcast, void* ctx, void* workspace,
                   size_t ws_bytes, void* stream);
/* The survey's entry point: u16, NCCL.  Rank, world size and block come from
 * the communicator (ncclComm_t passed as void*; NCCL is loaded at run time,
 * the process's copy if one is loaded, e.g. torch's). */
int smx_fw_sharded_u16(uint16_t* Tpanel, int n, int row0, int rows, int ld, int kind, void* nccl_comm,
                       void* workspace, size_t ws_bytes, void* stream);

/* ---- Boolean products and Warshall closure ------------------------------
 * Replace BoolMatrix.__mul__ (pkg/src/semimat/boolmat.py:151-172) and
 * BoolMatrix.transitive_closure (:174-189).
 *
 * Byte layout (one byte per entry, 0/1): tcgen05 kind::i8 tensor-core GEMM
 * with a count>0 threshold.  Bt is B TRANSPOSED (N x K, K-major), K >= 1.
 * Output is written as 0/1 bytes to C (C_bits == NULL, ldc in bytes) or as
 * packed bits to C_bits (C == NULL, ldc in u32 words) in the reference's
 * LSB-first block layout (boolmat.py:3-5); accumulate ORs into the output. */
int smx_bool_gemm_i8(const uint8_t* A, const uint8_t* Bt, uint8_t* C, uint32_t* C_bits,
                     int M, int N, int K, int lda, int ldbt, int ldc, int accumulate,
                     void* stream);
/* `batch` Boolean products A_i (M x K) * B_i (K x N) in one call on the
 * tensor cores: A stacked as batch * M bit rows (lda_w words each), B as
 * batch * K rows, C as batch * M rows (ldc_w = N / 32).  M and N multiples
 * of 128, 128 < K <= 65536.  Workspace:
 * smx_bool_mul_tc_batched_workspace_bytes(batch, M, N, K) bytes. */
size_t smx_bool_mul_tc_batched_workspace_bytes(int batch, int M, int N, int K);
int smx_bool_mul_tc_batched(const uint32_t* A, const uint32_t* B, uint32_t* C, int batch, int M, int N, int K,
                            int lda_w, int ldb_w, int ldc_w, void* workspace, size_t ws_bytes, void* stream);
/* The same on unpacked operands: A (batch * M rows of 0/1 bytes), B^T
 * (batch * N rows), packed-bit C (batch * M rows); one split-K pair launch. */
int smx_bool_gemm_i8_batched(const uint8_t* A, const uint8_t* Bt, uint32_t* C_bits, int batch, int M, int N,
                             int K, int lda, int ldbt, int ldc, int accumulate, void* stream);
/* The same products on E2M1 nibble operands, tcgen05 kind::mxf4 (half the
 * operand bytes and twice the MMA rate of kind::i8; scale factors 1.0, f32
 * counts, count > 0 threshold): A is M rows of ceil(K / 2) bytes (lda bytes
 * apart, lda % 16 == 0), B^T N rows likewise, as smx_unpack_nibbles writes
 * them; packed-bit output (ldc in u32 words).  Any M, N, K >= 1 (batched: M
 * and N multiples of 128).  Bit-identical to smx_bool_gemm_i8. */
int smx_bool_gemm_f4(const uint8_t* A, const uint8_t* Bt, uint32_t* C_bits, int M, int N, int K, int lda,
                     int ldbt, int ldc, int accumulate, void* stream);
int smx_bool_gemm_f4_batched(const uint8_t* A, const uint8_t* Bt, uint32_t* C_bits, int batch, int M, int N,
                             int K, int lda, int ldbt, int ldc, int accumulate, void* stream);
/* Operands of smx_bool_mul_tc / smx_bool_mul_tc_batched on the split-K pair:
 * 1 = E2M1 nibbles, kind::mxf4 (default), 0 = bytes, kind::i8.  Results are
 * identical.  Returns the previous setting. */
int smx_set_tc_f4(int enable);
/* Output tile width (N) of the tensor-core Boolean GEMM: 0 = automatic (the
 * widest of 256 / 128 / 64 that still gives every SM a tile), or force 64,
 * 128 or 256.  Results are identical.  Returns the previous setting. */
int smx_set_tc_tile_n(int bn);
/* Split-K CTA cluster for small packed-bit products (the C1 shape): 0 = off,
 * 1 = automatic (a pair of CTAs on one wave of 128 x 64 tiles or fewer,
 * 128 < K <= 65536, automatic tile width), 2 = the pair whenever the shape
 * allows it (packed-bit output, no row skip, 128 < K <= 65536), 3 = as 2
 * with four CTAs per tile (a quarter of K each, two-stage rings, two or
 * three CTAs per SM).  Results are identical.  Returns the previous setting. */
int smx_set_tc_pair(int mode);
/* K slices per product of the batched tensor-core products (1, 2 or 4).
 * Results are identical.  Returns the previous setting. */
int smx_set_tc_batch_ks(int ks);
/* Ring depth (2 or 3 stages) of the batched nibble products.  Results are
 * identical.  Returns the previous setting. */
int smx_set_tc_f4_batch_stages(int stages);
/* Development trace of the plain tensor-core kernel: buf (device, >= 16 + 2 *
 * CTAs u64) receives clock64 phase stamps of CTA 0 in [0, 8) and globaltimer
 * entry/exit of every CTA from [16]; NULL disarms. */
int smx_tc_trace_arm(unsigned long long* buf);
/* BoolMatrix.__mul__ on packed bit rows in one call (unpack A, fused
 * bits -> B^T bytes, tcgen05 product with the packed-bit epilogue).  C rows
 * are fully written, padding words zeroed.  Workspace: see
 * smx_bool_mul_tc_workspace_bytes. */
size_t smx_bool_mul_tc_workspace_bytes(int M, int N, int K);
int smx_bool_mul_tc(const uint32_t* A, const uint32_t* B, uint32_t* C, int M, int N, int K,
                    int lda_w, int ldb_w, int ldc_w, void* workspace, size_t ws_bytes, void* stream);
/* Warshall closure in place on 0/1 bytes (n x n, ld bytes, 16-byte aligned
 * rows) with tensor-core phases 2/3. */
size_t smx_bool_warshall_i8_workspace_bytes(int n, int ld);
int smx_bool_warshall_i8(uint8_t* T, int n, int ld, void* workspace, size_t ws_bytes,
                         void* stream);
/* Bit-packed comparison variant on u32 words (the reference's uint64 blocks
 * reinterpreted little-endian): C = (acc ? C : 0) | A (x) B. */
int smx_bool_gemm_bits(const uint32_t* A, const uint32_t* B, uint32_t* C,
                       int M, int Nwords, int K, int lda_w, int ldb_w, int ldc_w,
                       int accumulate, void* stream);
/* Warshall closure in place on packed bits (n x n, ld in u32 words). */
size_t smx_bool_warshall_workspace_bytes(int n, int ld_w);
int smx_bool_warshall_bits(uint32_t* T, int n, int ld_w, void* workspace, size_t ws_bytes,
                           void* stream);

/* ---- layout helpers ---------------------------------------------------- */
/* bytes (rows x cols, ld bytes) <-> packed u32 words (ld_w words), zero pad bits */
int smx_pack_bits(const uint8_t* bytes, uint32_t* words, int rows, int cols, int ld,
                  int ld_w, void* stream);
int smx_unpack_bits(const uint32_t* words, uint8_t* bytes, int rows, int cols, int ld_w,
                    int ld, void* stream);
/* packed bits (rows x cols) -> 0/1 bytes of the TRANSPOSE (cols x rows, ld_out
 * bytes): the K-major B^T operand of smx_bool_gemm_i8 in one pass */
int smx_unpack_bits_transposed(const uint32_t* words, uint8_t* bytes_t, int rows, int cols,
                               int ld_w, int ld_out, void* stream);
/* packed bits -> the E2M1 nibble operands of smx_bool_gemm_f4 in one launch:
 * A (a_rows x a_cols bits; NULL skips A) -> a_rows rows of nibbles (a_ld
 * bytes apart), B (b_rows x b_cols bits) -> B^T, b_cols rows of nibbles
 * (b_ldt bytes apart).  Bit k of a row -> nibble k (byte k / 2, low nibble
 * first), 0 or 0b0010 (1.0); bytes past ceil(cols / 2) are not written. */
int smx_unpack_nibbles(const uint32_t* a_words, uint8_t* a_nib, int a_rows, int a_cols, int a_ldw, int a_ld,
                       const uint32_t* b_words, uint8_t* bt_nib, int b_rows, int b_cols, int b_ldw, int b_ldt,
                       void* stream);
/* out (cols x rows) = in^T for bytes */
int smx_transpose_u8(const uint8_t* in, uint8_t* out, int rows, int cols, int ld_in,
                     int ld_out, void* stream);

/* ---- entrywise algebra (antidist.py:128-156, boolmat.py:120-137) -------
 * Lane matrices: op 0 = min (&), 1 = max (|), 2 = |a-b| (^), 3 = S - a (~,
 * B unused); columns >= cols of every row are set to the pad value (S when
 * pad_is_limit, else 0).  Bits: op 0 = or, 1 = and, 2 = xor, 3 = not (B
 * unused); bits >= cols are cleared.  C may alias A or B. */
int smx_lane_entrywise(const void* A, const void* B, void* C, int rows, int cols, int ld,
                       int elem_bytes, int op, int pad_is_limit, void* stream);
int smx_bits_entrywise(const uint32_t* A, const uint32_t* B, uint32_t* C, int rows, int cols,
                       int ld_w, int op, void* stream);

/* ---- lane kernels (kernels.py:129-204) ---------------
 * The paper's 128-bit block primitives over a flat array of nlanes lanes
 * (nlanes * elem_bytes a multiple of 16): op 0 = subsat max(a-b,0),
 * 1 = addsat min(a+b,S), 2 = max, 3 = min, 4 = |a-b|, 5 = clonenot S-a (B
 * unused).  Replaces subsat/addsat/maxlanes/minlanes/absdiff/clonenot
 * (kernels.py:129-189) and np_subsat/np_addsat/np_absdiff (:195-204). */
int smx_lane_op(const void* A, const void* B, void* C, long long nlanes, int elem_bytes, int op,
                void* stream);

/* ---- Boolean bridge (antidist.py:213-224) -------------------------------
 * from_boolmat: lanes = S where the bit is set, else 0; padding lanes 0.
 * to_boolmat: bit = (lane > 0) for columns < cols; every other bit of the
 * ld_w words 0. */
int smx_lanes_from_bits(const uint32_t* words, int ld_w, void* out, int rows, int cols, int ld,
                        int elem_bytes, void* stream);
int smx_lanes_to_bits(const void* in, int ld, uint32_t* words, int ld_w, int rows, int cols,
                      int elem_bytes, void* stream);

/* ---- batched small matrices (one launch per batch) ----------------------
 * `batch` independent problems, each matrix `stride_*` elements (words for
 * bits, lanes for lane matrices) after the previous one.
 * Boolean product (boolmat.py:151-172) on packed rows: C = A (x) B, padding
 * words of C zeroed.  Boolean Warshall (boolmat.py:174-189), n <= 512, in
 * place.  Lane Floyd-Warshall (antidist.py:390-398, :440-448), n <= 128, in
 * place, padding lanes untouched. */
int smx_bool_mul_batched(const uint32_t* A, const uint32_t* B, uint32_t* C, int batch, int M, int N,
                         int K, int lda_w, int ldb_w, int ldc_w, long long stride_a,
                         long long stride_b, long long stride_c, void* stream);
int smx_bool_warshall_batched(uint32_t* T, int batch, int n, int ld_w, long long stride, void* stream);
int smx_fw_batched(void* T, int batch, int n, int ld, long long stride, int elem_bytes, int kind,
                   void* stream);

/* The first invalid edge of an edge list on the device (edges: m x 3 int64
 * rows (u, v, w)): a vertex outside [0, n) or a weight outside [0, limit].
 * *first (device, u64) receives its index, or m if every edge is valid; the
 * caller reports it with the reference's message (antidist.py:201-208). */
int smx_edges_first_invalid(const long long* edges, long long m, int n, long long limit,
                            unsigned long long* first, void* stream);
/* ---- construction (antidist.py:191-211, :294-309) ---------------------
 * Fill the n x ld matrix T with the (+)-identity (0 anti / S dist, padding
 * included) and fold m weighted edges edges[3*i .. 3*i+2] = (u, v, w) into it,
 * keeping the best parallel edge (anti: max of S - w; dist: min of w).
 * Edges must already be validated (0 <= u, v < n, 0 <= w <= S); `edges` is a
 * device array of int64. */
int smx_from_edges(const long long* edges, long long m, void* T, int n, int ld, int elem_bytes,
                   int kind, void* stream);

/* ---- measurement support (bench.py roofline denominators) -------------- */
/* Runs `iters` iterations of an independent VIMNMX.U16x2 + VIADDMNMX.U16x2
 * (or VIADDMNMX only when one_instr != 0) instruction stream on every
 * resident thread; writes a checksum to sink.  Instructions issued =
 * grid*block*iters*per_iter (returned via *instr_per_thread). */
int smx_int_issue_probe(uint32_t* sink, int blocks, int threads, int iters, int one_instr,
                        long long* instr_per_thread, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SEMIMAT_B200_H */
