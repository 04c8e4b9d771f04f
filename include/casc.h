/*
 * casc.h — C ABI of the B200-native cascaded FP64x2 GEMM (arXiv 2303.04353,
 * "Cascading GEMM": FP64x2 GEMM as ten cascading FP64 GEMMs).
 *
 *   C := A B  for FP64x2 (double-double) A (m x k), B (k x n), C (m x n)
 *   ("C := A B"; P:L228 fixed number of FP64 GEMMs, data-independent
 *   time; P:L39-45 FP64 for all O(n^3) work, cheap cancellation detection).
 *
 * Method (all of it runs in this library's sm_100a kernels):
 *   1. widths c0,c1,c2 from min(k, 256) (§3.3);
 *   2. per (row of A, 256-wide k panel) and (column of B, panel) power-of-two
 *      scales;
 *   3. Appendix A conditional-free split of every FP64x2 element into four
 *      FP64 slices A0..A3 / B0..B3, plus B4, B5, B6;
 *   4. per panel, the ten FP64 products of eqn:Gemm10 on the FP64
 *      tensor cores (DMMA) into four on-chip bins 0, 1, 2, 3-6;
 *   5. per panel, the FP64x2 combine bin 3-6 -> 2 -> 1 -> 0 (P:L946-949,
 *      P:L2506-2520), scaling by the row/column scales, and FP64x2 accumulation
 *      into C across panels;
 *   6. cancellation flag = OR over panels of (bin0 == 0) (§3.7, §4.4
 *      P:L3380-3382).
 *
 * Entry points (in this order below):
 *   the north-star call casc_gemm_fp64x2 (+ _ws, workspace sizing, finalize);
 *   host-resident operands casc_gemm_fp64x2_host; phases separately
 *   (casc_pack_a / casc_pack_b / casc_gemm_packed, used by the multi-GPU layer);
 *   inspection exports (casc_split_a/b, casc_debug_bins); the simple path
 *   (casc_gemm_fp64x2_simple, casc_slice_product); BLAS-style generality
 *   (casc_gemm_fp64x2_ex, casc_syrk_fp64x2, casc_trsm_fp64x2,
 *   casc_trsm_diag_inv); the INT8 cascade (casc_i8_*: GEMM, _ws, _ex, _host,
 *   SYRK, pack / packed GEMM, split and bins exports).
 *
 * Conventions (all entry points):
 *   - Matrices are row-major with a leading dimension (elements).  An FP64x2
 *     value is the unevaluated sum hi + lo of two binary64 arrays (SoA).
 *   - Unless stated otherwise, pointers are DEVICE pointers owned by the
 *     caller; the library reads inputs and writes outputs only.
 *   - Work is enqueued on `stream` (NULL = legacy default stream).  The library
 *     never synchronises the host except where stated (the teardown calls
 *     casc_finalize / casc_i8_finalize, and k == 0 of the host-operand
 *     entries); kernel faults surface at the caller's next synchronisation.
 *     Every call is re-entrant: concurrent calls on different streams or host
 *     threads share no device memory (workspaces are the caller's or
 *     stream-ordered allocations of the call).
 *   - Preconditions (not checked): inputs finite; pairs normalised
 *     (|lo| <= ulp(hi)/2).  Outside them results are computed but the
 *     paper's error bound is not guaranteed.  Any finite exponent range is
 *     handled exactly: the scalings by 2^-e (split) and 2^(e+f) (combine) are
 *     ldexp-exact, subnormal results and overflow to +-inf included (reading
 *     R16).
 *   - Return value: a casc_status.  No exception crosses the ABI.
 *   - Results are deterministic: the same inputs give the same bits on every
 *     call, every grid size and every number of GPUs.
 */
#ifndef CASC_H_
#define CASC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* An opaque CUDA stream handle (ABI-identical to cudaStream_t). */
typedef struct CUstream_st* casc_stream_t;

typedef enum {
  CASC_OK = 0,
  CASC_ERR_INVALID = 1,     /* negative size, ld too small, NULL with non-zero size, aliasing */
  CASC_ERR_CUDA = 2,        /* CUDA launch / runtime / allocation failure */
  CASC_ERR_UNSUPPORTED = 3  /* device is not sm_100 (B200) */
} casc_status;

/* Human-readable name of a status code (static string, never NULL). */
const char* casc_status_string(int status);

/* k_C, the rank-k update depth the digit budgets are tied to (§3.5 P:L1474-1484,
 * §4.2): A and B are split and combined per 256-wide k panel. */
#define CASC_KC 256

/* Split widths c[0..2] = (c0, c1, c2) for inner dimension k (host function).
 * §3.3 P:L916-945 with L = ceil(log2(min(k, 256))): greedy c0 (2c0 + L <= 53),
 * then c1 (c0 + c1 + L + 1 <= 53, 2c1 + L + 2 <= 53), then c2
 * (c0 + c2 + L + 2 <= 53).  k = 256 -> (22, 21, 21); k = 64 -> (23, 22, 22).
 * Returns CASC_ERR_INVALID if c is NULL or k < 0. */
int casc_select_widths(int64_t k, int* c);

/* ------------------------------------------------------------------------ */
/* The north-star entry point.                                               */
/* ------------------------------------------------------------------------ */

/* C := A B in cascaded FP64x2 (ten FP64 DMMA GEMMs per 256-wide k panel).
 *   m, n, k   >= 0.  m == 0 or n == 0: no-op.  k == 0: C := 0, flags := 0.
 *   A_hi, A_lo: m x k, leading dimension lda >= max(1, k).
 *   B_hi, B_lo: k x n, leading dimension ldb >= max(1, n).
 *   C_hi, C_lo: m x n outputs, leading dimension ldc >= max(1, n); must not
 *               overlap A or B (CASC_ERR_INVALID).  C_hi + C_lo is the result.
 *   flags:      m x n uint8 output (leading dimension n) or NULL.  flags[i*n+j]
 *               = 1 iff bin 0 of entry (i, j) was exactly zero in some panel
 *               (catastrophic cancellation suspected, §3.7); the library
 *               performs no correction.
 *   stream:     CUDA stream.
 * Takes a workspace of casc_workspace_bytes(m, n, k) bytes from the device's
 * stream-ordered pool for the duration of the call (cudaMallocAsync /
 * cudaFreeAsync on `stream`; the pool keeps it cached, casc_finalize returns
 * it).  No host synchronisation; re-entrant. */
int casc_gemm_fp64x2(int64_t m, int64_t n, int64_t k,
                     const double* A_hi, const double* A_lo, int64_t lda,
                     const double* B_hi, const double* B_lo, int64_t ldb,
                     double* C_hi, double* C_lo, int64_t ldc,
                     uint8_t* flags, casc_stream_t stream);

/* Bytes of device workspace needed by casc_gemm_fp64x2 for (m, n, k): the
 * packed A and B (each rounded up to 256 bytes), the small-problem split-mode
 * panel sums when that mode applies, and a 256-byte slot for the fused
 * kernel's per-launch tile-wave counter. */
size_t casc_workspace_bytes(int64_t m, int64_t n, int64_t k);

/* casc_gemm_fp64x2 with HOST-resident operands (BASELINE north star's call,
 * operands in host memory): A_hi/A_lo, B_hi/B_lo, C_hi/C_lo (row-major, lda /
 * ldb / ldc in elements) and flags (m x n, ld = n, nullable) are host
 * pointers; page-locked memory (cudaHostAlloc / cudaHostRegister) lets the
 * copies overlap the kernels, pageable memory works but serialises them.
 * Result: bitwise the casc_gemm_fp64x2 result of the same operands.
 * Pipeline over blocks of C = row slabs of A (slab_rows rows) x column slabs
 * of B (slab_cols columns; each 0 = 4096 for a dimension >= 8192, else half the
 * dimension but at least 1024; when m and n are both >= 8192 the default column
 * slab is the first 64-multiple >= 2048 that makes a block a whole number of
 * waves of 64 x 64 tiles (2368 on 148 SMs), and the FIRST row / column slab is
 * 1024 (a shorter exposed first copy); rounded up to a multiple of 64), row slab
 * outer: an internal H2D stream copies A_0, then the column slabs of B, then
 * the next row slabs of A ahead of their use; the caller's stream splits each
 * slab once and multiplies block after block; an internal D2H stream returns
 * each block of C (and flags) as soon as it is done.  So only the first A and
 * B slabs and the last C block are exposed.  Device memory (two staging slots
 * for A, B and C blocks, the packed B, one packed A slab) comes from the
 * device's stream-ordered pool and is returned at the end.  Stream-ordered:
 * the call returns once everything is enqueued; the host buffers must stay
 * valid and untouched until `stream` completes.  k == 0 synchronises `stream`
 * and zeroes C and flags on the host.  Errors as casc_gemm_fp64x2
 * (CASC_ERR_INVALID also for slab_rows or slab_cols < 0). */
int casc_gemm_fp64x2_host(int64_t m, int64_t n, int64_t k,
                          const double* A_hi, const double* A_lo, int64_t lda,
                          const double* B_hi, const double* B_lo, int64_t ldb,
                          double* C_hi, double* C_lo, int64_t ldc,
                          uint8_t* flags, int64_t slab_rows, int64_t slab_cols,
                          casc_stream_t stream);

/* Same as casc_gemm_fp64x2 with a caller-owned device workspace of at least
 * casc_workspace_bytes(m, n, k) bytes (256-byte aligned).  No allocation, no
 * host synchronisation, re-entrant. */
int casc_gemm_fp64x2_ws(int64_t m, int64_t n, int64_t k,
                        const double* A_hi, const double* A_lo, int64_t lda,
                        const double* B_hi, const double* B_lo, int64_t ldb,
                        double* C_hi, double* C_lo, int64_t ldc,
                        uint8_t* flags, void* workspace, size_t workspace_bytes,
                        casc_stream_t stream);

/* Teardown: wait for the current device and return the cached memory of its
 * default stream-ordered pool (the per-call workspaces of both cascades) to
 * the system (cudaMemPoolTrimTo).  Host-synchronising. */
int casc_finalize(void);

/* ------------------------------------------------------------------------ */
/* Split ("packed") interface: phase 1 and phases 2-3 as separate calls, used */
/* by the multi-GPU layer (each rank packs its rows of A and its column slab  */
/* of B; B's packed slabs are all-gathered; each rank multiplies its rows).   */
/* Packed buffers are opaque device byte arrays in the GEMM kernel's layout   */
/* (DESIGN.md §6): 64-row (A) / 64-column (B) blocks, each block contiguous,  */
/* so a contiguous range of blocks is a contiguous byte range.               */
/* ------------------------------------------------------------------------ */

/* Bytes of the packed A (m x k): 4 slices + per-(row, panel) exponents.
 * Equals ceil(m/64) * casc_packed_a_block_bytes(k). */
size_t casc_packed_a_bytes(int64_t m, int64_t k);
size_t casc_packed_a_block_bytes(int64_t k);
/* Bytes of the packed B (k x n): 7 slices + per-(column, panel) exponents.
 * Equals ceil(n/64) * casc_packed_b_block_bytes(k); a column slab of B whose
 * width is a multiple of 64 packs into exactly (width/64) blocks. */
size_t casc_packed_b_bytes(int64_t k, int64_t n);
size_t casc_packed_b_block_bytes(int64_t k);

/* Phase 1 for A: per (row, panel) scale exponent and the Appendix A split
 * into A0, A1, A2, A3 (A2 stored pre-multiplied by 2^(c0-c1), an exact
 * power-of-two alignment).  Widths come from k (the FULL inner
 * dimension).  packed_a: casc_packed_a_bytes(m, k) bytes, 16-byte aligned. */
int casc_pack_a(int64_t m, int64_t k, const double* A_hi, const double* A_lo, int64_t lda,
                void* packed_a, casc_stream_t stream);

/* Phase 1 for B: per (column, panel) scale exponent, split into B0..B3 and
 * the derived B4 = B2 + 2^-c2 B3, B5 = B1 + 2^-c1 B4, B6 = B0 + 2^-c0 B5
 * (one RNE add each), stored pre-aligned (B2 x 2^(c0-c1),
 * B4 x 2^(c2-c0), B5 x 2^(c1+c2-2c0)).  packed_b: casc_packed_b_bytes(k, n). */
int casc_pack_b(int64_t k, int64_t n, const double* B_hi, const double* B_lo, int64_t ldb,
                void* packed_b, casc_stream_t stream);

/* Phases 2-3: C := A B from packed operands (same m, n, k as packed).
 * Fused kernel: TMA bulk copies of the slice tiles into shared memory, the ten
 * products on DMMA into four register bins, per-panel FP64x2 combine and
 * detector.  flags as in casc_gemm_fp64x2 (leading dimension n). */
int casc_gemm_packed(int64_t m, int64_t n, int64_t k, const void* packed_a,
                     const void* packed_b, double* C_hi, double* C_lo, int64_t ldc,
                     uint8_t* flags, casc_stream_t stream);
/* casc_gemm_packed with the flags' leading dimension ldf >= n (CASC_ERR_INVALID
 * otherwise), so that a column block of C and of the flags can be computed on
 * its own: with packed_b pointing at the packed blocks of columns [c0, c1)
 * (c0 a multiple of 64: a byte range of the packed B, casc_pack_b) and C /
 * flags pointing at column c0, the result is bitwise the same block of the
 * full product (per-column scales are column-local).  The multi-GPU layer
 * multiplies its local column slab this way while the other slabs arrive. */
int casc_gemm_packed_ld(int64_t m, int64_t n, int64_t k, const void* packed_a,
                        const void* packed_b, double* C_hi, double* C_lo, int64_t ldc,
                        uint8_t* flags, int64_t ldf, casc_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Test / inspection entry points (same kernels as the product path).        */
/* ------------------------------------------------------------------------ */

/* Run casc_pack_a and export its result in the paper's normalisation:
 *   slices: 4 x m x k doubles, slices[t*m*k + i*k + p] = chi_t of A(i, p)
 *           (value ~ 2^e (chi0 + 2^-D0 chi1 + 2^-D1 chi2 + 2^-D2 chi3));
 *   e:      P x m int32 (P = ceil(k/256)), e[q*m + i] = scale exponent of row i
 *           in panel q (max |A_hi| over the panel in [2^(e-1), 2^e); 0 if zero).
 * Uses a temporary device allocation (cudaMallocAsync on `stream`). */
int casc_split_a(int64_t m, int64_t k, const double* A_hi, const double* A_lo, int64_t lda,
                 double* slices, int32_t* e, casc_stream_t stream);

/* As casc_split_a for B: slices 7 x k x n (B0..B6, paper normalisation, no
 * pre-alignment), f: P x n int32. */
int casc_split_b(int64_t k, int64_t n, const double* B_hi, const double* B_lo, int64_t ldb,
                 double* slices, int32_t* f, casc_stream_t stream);

/* Bins of one k panel `panel` (0 <= panel < ceil(k/256)) as computed by the
 * fused kernel, in the paper's reference scales (bin0: 1, bin1: sigma1,
 * bin2: sigma2, bin36: sigma3): bins[b*m*n + i*n + j], b = 0..3.  Bins 0-2 are
 * exact and therefore bit-comparable with any exact evaluation. */
int casc_debug_bins(int64_t m, int64_t n, int64_t k,
                    const double* A_hi, const double* A_lo, int64_t lda,
                    const double* B_hi, const double* B_lo, int64_t ldb,
                    int64_t panel, double* bins, casc_stream_t stream);

/* Test export of the device power-of-two scaling the split (2^-e) and the
 * combine (2^(e_i+f_j)) use: out[i] = x[i] 2^n[i] rounded once
 * to nearest-even for any int n[i] (bitwise C99 ldexp: subnormal results,
 * overflow to +-inf, signed zeros; reading R16).  x, n, out: device arrays of
 * `count` elements (out may equal x). */
int casc_debug_ldexp(int64_t count, const double* x, const int32_t* n, double* out,
                     casc_stream_t stream);

/* ------------------------------------------------------------------------ */
/* BLAS-style generality ("other level-3 BLAS").  */
/* ------------------------------------------------------------------------ */
typedef enum { CASC_OP_N = 0, CASC_OP_T = 1 } casc_op;

/* C := alpha (x) op(A) op(B) (+) beta (x) C, all FP64x2, op(X) = X or X^T.
 *   op(A) is m x k: A stored m x k (transa = CASC_OP_N, lda >= max(1,k)) or
 *     k x m (CASC_OP_T, lda >= max(1,m)); op(B) is k x n likewise.
 *   alpha = alpha_hi + alpha_lo, beta = beta_hi + beta_lo (normalised pairs).
 *   The product op(A) op(B) is the cascaded one of casc_gemm_fp64x2 (bitwise
 *   identical for the same operands); the update uses FP64x2 multiplication
 *   (TwoProd by FMA) and FP64x2 addition: C := (alpha (x) P) (+) (beta (x) C),
 *   DESIGN.md reading R21.  beta == 0: C is not read (may hold NaN).
 *   k == 0 or alpha == 0: A and B are not referenced, C := beta (x) C, flags := 0.
 *   flags: as casc_gemm_fp64x2 (of the product), or NULL.
 *   workspace: NULL (temporary stream-ordered allocation) or a caller buffer of
 *   casc_workspace_bytes(m, n, k) bytes.
 * Errors as casc_gemm_fp64x2; CASC_ERR_INVALID also for trans values other than
 * CASC_OP_N / CASC_OP_T. */
int casc_gemm_fp64x2_ex(int transa, int transb, int64_t m, int64_t n, int64_t k,
                        double alpha_hi, double alpha_lo,
                        const double* A_hi, const double* A_lo, int64_t lda,
                        const double* B_hi, const double* B_lo, int64_t ldb,
                        double beta_hi, double beta_lo,
                        double* C_hi, double* C_lo, int64_t ldc,
                        uint8_t* flags, void* workspace, size_t workspace_bytes,
                        casc_stream_t stream);

/* NEXT-4, level-3 BLAS on the cascaded GEMM ("All Level-3 BLAS
 * algorithms can be written in terms of GEMM"): symmetric rank-k update
 *   C := alpha (x) op(A) op(A)^T (+) beta (x) C   on one triangle of C,
 * op(A) = A (trans = CASC_OP_N, A stored n x k, lda >= max(1,k)) or A^T
 * (CASC_OP_T, A stored k x n, lda >= max(1,n)); uplo = CASC_LOWER / CASC_UPPER
 * selects the triangle (diagonal included) that is read (beta != 0) and
 * written; the other triangle of C_hi / C_lo and of flags is not touched.
 * The product is the cascaded GEMM of op(A) and op(A)^T: op(A) is split as the
 * A and as the B operand and the fused kernel runs only the triangle's 64 x 64 tiles
 * (half the work of the GEMM); every stored element is bitwise what
 * casc_gemm_fp64x2_ex(trans, !trans, ..., A, A, ...) stores there.  alpha,
 * beta, the update sequence (reading R21), k == 0 / alpha == 0, workspace
 * (>= casc_workspace_bytes(n, n, k) or NULL), flags (n x n, ld = n) and
 * errors as casc_gemm_fp64x2_ex. */
typedef enum { CASC_LOWER = 0, CASC_UPPER = 1 } casc_uplo;
int casc_syrk_fp64x2(int uplo, int trans, int64_t n, int64_t k,
                     double alpha_hi, double alpha_lo,
                     const double* A_hi, const double* A_lo, int64_t lda,
                     double beta_hi, double beta_lo,
                     double* C_hi, double* C_lo, int64_t ldc,
                     uint8_t* flags, void* workspace, size_t workspace_bytes,
                     casc_stream_t stream);

/* NEXT-4, SYR2K on the cascaded GEMM (reading R30): on the uplo
 * triangle, C := alpha (x) op(A) op(B)^T (+) beta (x) C, then
 * C := alpha (x) op(B) op(A)^T (+) C (two triangular launches of the fused
 * kernel, each half the tiles of a GEMM; the R21 update sequence, the second
 * with beta = 1); flags (n x n, ld n, nullable) = OR of the two products'
 * flags.  A and B are stored n x k (trans CASC_OP_N, lda / ldb >= max(1,k))
 * or k x n (CASC_OP_T).  k == 0 / alpha == 0: C := beta C on the triangle.
 * Stream-ordered temporary workspace; errors as casc_syrk_fp64x2. */
int casc_syr2k_fp64x2(int uplo, int trans, int64_t n, int64_t k,
                      double alpha_hi, double alpha_lo,
                      const double* A_hi, const double* A_lo, int64_t lda,
                      const double* B_hi, const double* B_lo, int64_t ldb,
                      double beta_hi, double beta_lo,
                      double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
                      casc_stream_t stream);

/* NEXT-4, TRSM on the cascaded GEMM (reading R27):
 * left side: solve op(A) X = alpha (x) B for X, op(A) = A (trans CASC_OP_N) or
 * A^T (CASC_OP_T), A m x m triangular (uplo CASC_LOWER / CASC_UPPER; diag
 * CASC_NONUNIT / CASC_UNIT: the diagonal is taken as 1 and not read), X
 * overwrites the m x n B (ldb >= max(1,n)); only A's triangle is read.
 * B := alpha (x) B; the 256 x 256 diagonal blocks of A are inverted in FP64x2
 * (casc_trsm_diag_inv; op(A_bb)^-1 = op(Inv_b)); then, block by block in the
 * order of op(A)'s triangle (ascending when op(A) is lower, descending when
 * upper), X_b = op(Inv_b) B_b and B_rest := B_rest - op(A)_rest,b X_b with
 * casc_gemm_fp64x2_ex.  Device memory for the inverses and one block of X comes
 * from the stream-ordered pool; no host synchronisation.  alpha == 0: X := 0,
 * A not read.  Errors as casc_gemm_fp64x2_ex (CASC_ERR_INVALID also for bad
 * uplo / trans / diag and for B overlapping A). */
typedef enum { CASC_NONUNIT = 0, CASC_UNIT = 1 } casc_diag;
int casc_trsm_fp64x2(int uplo, int trans, int diag, int64_t m, int64_t n,
                     double alpha_hi, double alpha_lo,
                     const double* A_hi, const double* A_lo, int64_t lda,
                     double* B_hi, double* B_lo, int64_t ldb, casc_stream_t stream);
/* NEXT-4, more level-3 BLAS on the cascaded GEMM (DESIGN.md
 * readings R28, R29).  side: CASC_LEFT / CASC_RIGHT. */
typedef enum { CASC_LEFT = 0, CASC_RIGHT = 1 } casc_side;
/* SYMM: C := alpha (x) A B (+) beta (x) C (side LEFT, A m x m) or
 * C := alpha (x) B A (+) beta (x) C (side RIGHT, A n x n), A symmetric and only
 * its `uplo` triangle read (lda >= max(1, dim A)); B, C m x n (ldb, ldc >=
 * max(1, n)); flags m x n (ld n) or NULL.  The symmetric A is expanded from its
 * triangle into a stream-ordered temporary, then casc_gemm_fp64x2_ex computes
 * the product: bitwise casc_gemm_fp64x2_ex of the full symmetric matrix.
 * alpha == 0: C := beta C, A and B not read.  Errors as casc_gemm_fp64x2_ex
 * (also bad side / uplo). */
int casc_symm_fp64x2(int side, int uplo, int64_t m, int64_t n,
                     double alpha_hi, double alpha_lo,
                     const double* A_hi, const double* A_lo, int64_t lda,
                     const double* B_hi, const double* B_lo, int64_t ldb,
                     double beta_hi, double beta_lo,
                     double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
                     casc_stream_t stream);
/* TRMM: B := alpha (x) op(A) B (side LEFT, A m x m) or B := alpha (x) B op(A)
 * (side RIGHT, A n x n), A triangular (uplo; diag CASC_UNIT: diagonal taken as
 * 1, not read), op(A) = A or A^T; B m x n overwritten.  The triangular A (other
 * triangle zero) is expanded into a stream-ordered temporary and the product is
 * the cascaded GEMM of it (each tile's k range stopped at the zero triangle:
 * about half the work), written back into B: the values of
 * casc_gemm_fp64x2_ex of the expanded matrix (the skipped terms are zeros).
 * alpha == 0: B := 0, A not read.  CASC_ERR_INVALID for bad enums, B
 * overlapping A. */
int casc_trmm_fp64x2(int side, int uplo, int trans, int diag, int64_t m, int64_t n,
                     double alpha_hi, double alpha_lo,
                     const double* A_hi, const double* A_lo, int64_t lda,
                     double* B_hi, double* B_lo, int64_t ldb, casc_stream_t stream);
/* Right-side TRSM: solve X op(A) = alpha (x) B, A n x n triangular, B m x n
 * (X overwrites B).  The blocked algorithm of casc_trsm_fp64x2 on column
 * blocks: X_b = B_b op(Inv_b), then B_c := B_c - X_b op(A)_(b,c) for the
 * blocks still to solve (super-blocks of 4 x 256 as the left side), every
 * product a casc_gemm_fp64x2_ex (op(A) read transposed by its split kernels,
 * no transposed copy of B).  Arguments and errors as casc_trsm_fp64x2. */
int casc_trsm_fp64x2_right(int uplo, int trans, int diag, int64_t m, int64_t n,
                           double alpha_hi, double alpha_lo,
                           const double* A_hi, const double* A_lo, int64_t lda,
                           double* B_hi, double* B_lo, int64_t ldb, casc_stream_t stream);
/* Test / inspection export of the TRSM's first step: the inverses of the
 * 256 x 256 diagonal blocks of the triangular A, inv_hi / inv_lo =
 * [ceil(m/256)][256][256] row-major FP64x2 (zeros outside the triangle and
 * beyond a ragged last block), by column substitution in the oracle's order. */
int casc_trsm_diag_inv(int uplo, int diag, int64_t m, const double* A_hi, const double* A_lo,
                       int64_t lda, double* inv_hi, double* inv_lo, casc_stream_t stream);

/* ------------------------------------------------------------------------ */
/* The paper's simple path (§4.2): phases as separate kernels.  */
/* ------------------------------------------------------------------------ */

/* C := A B exactly as casc_gemm_fp64x2 (same widths, split, combine and flag
 * semantics) but staged like §4.2: per 256-wide k panel, ten separate
 * slice-GEMM launches (DMMA) accumulate the products of eqn:Gemm10 into four
 * m x n bins in HBM, then a standalone HBM-bound epilogue kernel adds the bins
 * into C in FP64x2 (bin 3-6, 2, 1, 0) and applies Sigma, T.  Bins 0-2 and the
 * flags equal the fused path's bit for bit; C agrees within the error bound
 * (bin 3-6 is summed in another order).  Uses temporary device memory
 * (cudaMallocAsync on `stream`): packed slices + 32 m n bytes of bins.
 * Arguments and errors as casc_gemm_fp64x2. */
int casc_gemm_fp64x2_simple(int64_t m, int64_t n, int64_t k,
                            const double* A_hi, const double* A_lo, int64_t lda,
                            const double* B_hi, const double* B_lo, int64_t ldb,
                            double* C_hi, double* C_lo, int64_t ldc,
                            uint8_t* flags, casc_stream_t stream);

/* One slice GEMM of one k panel: out (m x n, leading dimension n) :=
 * sum_{p in panel} A_sa[i, p] B_sb[p, j] in the paper's normalisation
 * (sa in 0..3 = A0..A3, sb in 0..6 = B0..B6), computed by the simple path's
 * slice-GEMM kernel.  The six products A0B0, A0B1, A1B0, A0B2, A1B1, A2B0 are
 * exact and therefore bit-comparable.  CASC_ERR_INVALID for slice or
 * panel out of range. */
int casc_slice_product(int64_t m, int64_t n, int64_t k,
                       const double* A_hi, const double* A_lo, int64_t lda,
                       const double* B_hi, const double* B_lo, int64_t ldb,
                       int sa, int sb, int64_t panel, double* out, casc_stream_t stream);

/* ------------------------------------------------------------------------ */
/* NEXT-3: the INT8 cascade (paper §6 "FP64x2 in terms of INT8") */
/* ------------------------------------------------------------------------ */
/* The same product C := A B (FP64x2) computed from y int8 slices per operand
 * with the y(y+1)/2 products A_i B_j, i + j < y ("14 to 15 INT8 splits and
 * about 105 to 120 INT8 multiplies") on the INT8 tensor cores
 * (tcgen05.mma kind::i8, int32 accumulation in tensor memory).
 * DESIGN.md readings R22-R26 fix what the paper leaves open:
 *   R22 k panel 8192; scale exponent per (row, panel) / (column, panel);
 *   R23 X = rint(hi 2^(F-e)) + rint(lo 2^(F-e)), F = 6 + 8(y-1), slices = the
 *       balanced base-256 digits of X (d_0 in [-64, 64], d_t in [-128, 127]);
 *   R24 bin_s = sum_p sum_(i+j=s) dA_i dB_j (exact int32), s < y;
 *   R25 four bins at a time -> exact FP64x2 group value, scaled by
 *       2^(e+f-12-8(s+nb-1)); panel value T = FP64x2 sum of the groups, most
 *       significant first; C := C (+) T over panels (ascending);
 *   R26 flags[i*n+j] = 1 iff |T.hi| <= kp 2^(e+f-50) in some panel (the panel's
 *       product cancelled by at least ~50 bits against its operand scale).
 * The result is bitwise deterministic and bitwise equal to the CPU oracle of
 * the same readings (every step is exact integer work or a fixed sequence of
 * RNE FP64 operations). */
#define CASC_I8_KC 8192
#define CASC_I8_DEFAULT_SLICES 14

/* C := A B through y int8 slices, 3 <= y <= 15 (CASC_ERR_INVALID otherwise).
 * Arguments, aliasing rules, k == 0 / m == 0 / n == 0 behaviour and errors as
 * casc_gemm_fp64x2 (flags semantics: R26 above).  Takes a workspace of
 * casc_i8_workspace_bytes(m, n, k, y) bytes from the device's stream-ordered
 * pool for the duration of the call (as casc_gemm_fp64x2); no host
 * synchronisation, re-entrant. */
int casc_i8_gemm_fp64x2(int64_t m, int64_t n, int64_t k,
                        const double* A_hi, const double* A_lo, int64_t lda,
                        const double* B_hi, const double* B_lo, int64_t ldb,
                        double* C_hi, double* C_lo, int64_t ldc,
                        uint8_t* flags, int y, casc_stream_t stream);

/* As casc_i8_gemm_fp64x2 with a caller-owned device workspace (256-byte
 * aligned, >= casc_i8_workspace_bytes(m, n, k, y)); no host synchronisation
 * (small single-panel problems in split mode take a stream-ordered temporary,
 * see casc_i8_gemm_ws_bytes). */
int casc_i8_gemm_fp64x2_ws(int64_t m, int64_t n, int64_t k,
                           const double* A_hi, const double* A_lo, int64_t lda,
                           const double* B_hi, const double* B_lo, int64_t ldb,
                           double* C_hi, double* C_lo, int64_t ldc,
                           uint8_t* flags, int y, void* workspace, size_t workspace_bytes,
                           casc_stream_t stream);

/* casc_gemm_fp64x2_host for the INT8 cascade: host-resident operands streamed
 * in blocks (slab_rows, slab_cols: 0 = the casc_gemm_fp64x2_host default,
 * rounded up to multiples of 256), bitwise
 * the casc_i8_gemm_fp64x2 result; memory, ordering and errors as
 * casc_gemm_fp64x2_host (CASC_ERR_INVALID also for y outside [3, 15]). */
int casc_i8_gemm_fp64x2_host(int64_t m, int64_t n, int64_t k,
                             const double* A_hi, const double* A_lo, int64_t lda,
                             const double* B_hi, const double* B_lo, int64_t ldb,
                             double* C_hi, double* C_lo, int64_t ldc,
                             uint8_t* flags, int y, int64_t slab_rows, int64_t slab_cols,
                             casc_stream_t stream);

/* SYRK on the INT8 cascade (NEXT-4): casc_syrk_fp64x2's semantics (uplo,
 * trans, alpha, beta, untouched other triangle, flags n x n) through y int8
 * slices; only the pair tiles holding triangle elements run, and every
 * stored element is bitwise what casc_i8_gemm_fp64x2_ex(trans, !trans, ...,
 * A, A, ...) stores there.  Stream-ordered temporary workspace.  Errors as
 * casc_i8_gemm_fp64x2_ex. */
int casc_i8_syrk_fp64x2(int uplo, int trans, int64_t n, int64_t k,
                        double alpha_hi, double alpha_lo,
                        const double* A_hi, const double* A_lo, int64_t lda,
                        double beta_hi, double beta_lo,
                        double* C_hi, double* C_lo, int64_t ldc,
                        uint8_t* flags, int y, casc_stream_t stream);

/* TRSM on the INT8 cascade (NEXT-4): casc_trsm_fp64x2's semantics and blocked
 * algorithm (reading R27) with casc_i8_gemm_fp64x2_ex (y slices) as the GEMM;
 * bit-exact with its oracle.  Errors as casc_trsm_fp64x2 (CASC_ERR_INVALID also
 * for y outside [3, 15]). */
int casc_i8_trsm_fp64x2(int uplo, int trans, int diag, int64_t m, int64_t n,
                        double alpha_hi, double alpha_lo,
                        const double* A_hi, const double* A_lo, int64_t lda,
                        double* B_hi, double* B_lo, int64_t ldb, int y, casc_stream_t stream);

/* NEXT-4 on the INT8 cascade: C := alpha (x) op(A) op(B) (+) beta (x) C with the
 * semantics, argument layout and errors of casc_gemm_fp64x2_ex (reading R21),
 * the product computed through y int8 slices (bitwise the casc_i8_gemm_fp64x2
 * product of the same op(A), op(B)).  workspace: NULL (temporary stream-ordered
 * allocation) or >= casc_i8_workspace_bytes(m, n, k, y) bytes. */
int casc_i8_gemm_fp64x2_ex(int transa, int transb, int64_t m, int64_t n, int64_t k,
                           double alpha_hi, double alpha_lo,
                           const double* A_hi, const double* A_lo, int64_t lda,
                           const double* B_hi, const double* B_lo, int64_t ldb,
                           double beta_hi, double beta_lo,
                           double* C_hi, double* C_lo, int64_t ldc,
                           uint8_t* flags, int y, void* workspace, size_t workspace_bytes,
                           casc_stream_t stream);

/* Workspace bytes: packed A + packed B + casc_i8_gemm_ws_bytes(m, n) (each
 * part 256-byte aligned).  0 for empty problems or y out of range. */
size_t casc_i8_workspace_bytes(int64_t m, int64_t n, int64_t k, int y);

/* Split ("packed") interface of the INT8 cascade, phase 1 and phases 2-3 as
 * separate calls (timing, and the multi-GPU layer: each rank packs its rows of
 * A and its column slab of B; packed B slabs are all-gathered).
 * A packed operand is an opaque device byte array of 128-row (A) / 128-column
 * (B) blocks, each casc_i8_packed_block_bytes(k, y) bytes and contiguous: y
 * slices x ceil(k/128) chunks of 128 x 128 int8 in the tcgen05 shared-memory
 * layout (K-major, 128-byte swizzle), then the int32 scale exponents of the
 * block's 128 vectors per panel.  The number of blocks is rounded up to an
 * even count (the GEMM runs on CTA pairs); a column slab of B whose width is a
 * multiple of 256 packs into exactly width/128 blocks. */
size_t casc_i8_packed_block_bytes(int64_t k, int y);
/* Bytes of one packed operand: 2 ceil(rows/256) blocks (rows = m for A, n for B). */
size_t casc_i8_packed_bytes(int64_t rows, int64_t k, int y);
/* Phase 1 (R22, R23): scale exponents and int8 slices of A (is_b == 0: rows x k,
 * ld >= k) or of B's columns (is_b != 0: B is k x rows, ld >= rows) into
 * `packed` (casc_i8_packed_bytes(rows, k, y) bytes, 256-byte aligned). */
int casc_i8_pack(int64_t rows, int64_t k, const double* hi, const double* lo, int64_t ld,
                 int is_b, int y, void* packed, casc_stream_t stream);
/* Bytes of the GEMM's own scratch: 6 x 128 x 128 x 8 bytes per CTA (the FP64x2
 * C accumulator and the exact group values of the tile in flight; all CTA
 * pairs for problems small enough for split mode), then a wave-synchronisation
 * counter.  Split mode (a single k panel and few tiles: one work item per
 * (tile, k-block part), bitwise the same C) also takes a stream-ordered
 * temporary for the parts' exact partial products. */
size_t casc_i8_gemm_ws_bytes(int64_t m, int64_t n);
/* Phases 2-3 (R24-R26) from packed operands of the same m, n, k, y: the fused
 * tcgen05 kernel on CTA pairs.  ws: >= casc_i8_gemm_ws_bytes(m, n) bytes of
 * device scratch.  C, flags and errors as casc_i8_gemm_fp64x2. */
int casc_i8_gemm_packed(int64_t m, int64_t n, int64_t k, int y, const void* packed_a,
                        const void* packed_b, double* C_hi, double* C_lo, int64_t ldc,
                        uint8_t* flags, void* ws, size_t ws_bytes, casc_stream_t stream);
/* casc_i8_gemm_packed with the flags' leading dimension ldf >= n (column
 * blocks as casc_gemm_packed_ld; c0 a multiple of 256, the INT8 slab unit). */
int casc_i8_gemm_packed_ld(int64_t m, int64_t n, int64_t k, int y, const void* packed_a,
                           const void* packed_b, double* C_hi, double* C_lo, int64_t ldc,
                           uint8_t* flags, int64_t ldf, void* ws, size_t ws_bytes,
                           casc_stream_t stream);
/* Same as casc_finalize (kept for the INT8 cascade's API symmetry). */
int casc_i8_finalize(void);

/* Test export of the split (R22, R23) as computed by the GEMM's split kernels:
 *   is_b == 0: A (rows x k, leading dimension ld >= k); is_b != 0: B (k x rows,
 *   ld >= rows; "rows" are the columns of B).
 *   digits: y x rows x k int8, digits[(t*rows + r)*k + p] = slice t of element
 *           (r, p) of A, or (p, r) of B;
 *   e:      P x rows int32 (P = ceil(k/8192)), scale exponent of row/column r
 *           in panel q.
 * Uses a temporary device allocation (cudaMallocAsync on `stream`). */
int casc_i8_split(int64_t rows, int64_t k, const double* hi, const double* lo, int64_t ld,
                  int is_b, int y, int8_t* digits, int32_t* e, casc_stream_t stream);

/* Test export of the exact int32 bins (R24) of k panel `panel` as accumulated
 * in tensor memory by the GEMM kernel: bins[(s*m + i)*n + j], s = 0 .. y-1.
 * Bit-comparable with any exact evaluation.  CASC_ERR_INVALID for a panel out
 * of range. */
int casc_i8_debug_bins(int64_t m, int64_t n, int64_t k,
                       const double* A_hi, const double* A_lo, int64_t lda,
                       const double* B_hi, const double* B_lo, int64_t ldb,
                       int y, int64_t panel, int32_t* bins, casc_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Multi-GPU exchange over peer memory (north star: "B      */
/* slices broadcast over NVLink"; paper_2303_04353_b200/multigpu.py,        */
/* gather = "p2p").  Each rank exports the device buffer holding its packed  */
/* column slab of B; the other ranks map it and pull the slab with the copy  */
/* engines (no SM is used by the exchange; a slab's GEMM starts when that    */
/* slab has landed).  Host code; ordering between ranks is the caller's       */
/* (host-side barriers), no kernel waits on another rank.                     */
#define CASC_IPC_HANDLE_BYTES 64

/* cudaMalloc `bytes` (> 0) on the current device and export it:
 *   *ptr    the device pointer (owned by the caller; release with casc_ipc_free);
 *   handle  CASC_IPC_HANDLE_BYTES bytes of host memory receiving the
 *           cudaIpcMemHandle_t to send to the other ranks.
 * CASC_ERR_INVALID for NULL arguments or bytes == 0, CASC_ERR_CUDA if the
 * allocation or the export fails (*ptr = NULL then). */
int casc_ipc_alloc(size_t bytes, void** ptr, void* handle);
/* cudaFree of a casc_ipc_alloc buffer (NULL: no-op).  Host-synchronising as cudaFree. */
int casc_ipc_free(void* ptr);
/* Map another process's exported buffer into this process (current device,
 * peer access enabled lazily): *ptr = its base address here.  CASC_ERR_CUDA
 * if the handle cannot be opened (e.g. no peer access between the devices,
 * or a handle of this same process). */
int casc_ipc_open(const void* handle, void** ptr);
/* Unmap a casc_ipc_open pointer (NULL: no-op). */
int casc_ipc_close(void* ptr);
/* Enqueue a copy of `bytes` bytes from src to dst on `stream` (device, peer
 * or host pointers: cudaMemcpyDefault; a peer-mapped src is read over NVLink
 * by the copy engine).  bytes == 0 is a no-op; NULL with bytes > 0 is
 * CASC_ERR_INVALID. */
int casc_copy_async(void* dst, const void* src, size_t bytes, casc_stream_t stream);

/* Number of kernel launches the last successful call of the given entry point
 * family enqueued on this host thread (for launch accounting in bench.py). */
int casc_last_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* CASC_H_ */
