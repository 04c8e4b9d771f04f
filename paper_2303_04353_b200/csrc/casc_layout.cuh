// casc_layout.cuh — packed slice layout, tile shape and device helpers shared
// by the split kernels and the fused cascaded-GEMM kernel (product path only;
// nothing here is shared with oracle/).
//
// Packed layout.  The GEMM's CTA tile is 64 x 64 output elements
// computed by 8 MMA warps arranged 2 (m) x 4 (n), each warp a 32 x 16 sub-tile
// built from mma.sync.m8n8k4.f64 fragments (4 m-subtiles x 2 n-subtiles).
// The split kernels write every slice directly in FRAGMENT ORDER, so that:
//   * one pipeline stage (8 values of k) of a 64-row A block (4 slices) or a
//     64-column B block (7 slices) is ONE contiguous chunk -> one TMA bulk copy;
//   * inside shared memory each warp's fragment load for one (slice, subtile,
//     k4-step) is 32 consecutive doubles -> conflict-free 256-byte loads.
//
// A block (64 rows), per k4-step (4 values of k), 1024 doubles:
//   [slice s 0..3][mwarp 0..1][msub 0..3][lane 0..31]
//   element (row r in block, k) with g = r%8, ms = (r%32)/8, mw = r/32,
//   ks = k/4, c = k%4, lane = 4g + c (mma A fragment a0 = A[g][c]).
// B block (64 columns), per k4-step, 1792 doubles:
//   [slice s 0..6][nwarp 0..3][nsub 0..1][lane 0..31]
//   element (k, col j in block) with g = j%8, ns = (j%16)/8, nw = j/16,
//   lane = 4g + c (mma B fragment b0 = B[c][g]).
// After the kpad/4 k4-steps of slices (kpad = k rounded up to 8), each block
// holds its exponents: int32 [panel 0..P-1][64].
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace casc {

constexpr int KC = 256;          // k_C panel depth
constexpr int TM = 64;           // CTA tile rows
constexpr int TN = 64;           // CTA tile cols
#ifndef CASC_BK
#define CASC_BK 8
#endif
constexpr int BK = CASC_BK;      // k per pipeline stage (multiple of 4, divides 256)
constexpr int STAGES_PER_PANEL = KC / BK;
constexpr int A_SLICES = 4;
constexpr int B_SLICES = 7;
constexpr int A_KSTEP = A_SLICES * TM * 4;   // doubles per k4-step of an A block (1024)
constexpr int B_KSTEP = B_SLICES * TN * 4;   // doubles per k4-step of a B block (1792)
constexpr int A_STAGE = A_KSTEP * (BK / 4);  // doubles per stage (2048 = 16 KB)
constexpr int B_STAGE = B_KSTEP * (BK / 4);  // doubles per stage (3584 = 28 KB)

__host__ __device__ inline int64_t kpad_of(int64_t k) { return (k + BK - 1) / BK * BK; }
__host__ __device__ inline int64_t panels_of(int64_t k) { return (k + KC - 1) / KC; }
__host__ __device__ inline int64_t a_block_bytes(int64_t k) {
  return kpad_of(k) / 4 * A_KSTEP * 8 + panels_of(k) * TM * 4;
}
__host__ __device__ inline int64_t b_block_bytes(int64_t k) {
  return kpad_of(k) / 4 * B_KSTEP * 8 + panels_of(k) * TN * 4;
}
__host__ __device__ inline int64_t a_exp_offset(int64_t k) { return kpad_of(k) / 4 * A_KSTEP * 8; }
__host__ __device__ inline int64_t b_exp_offset(int64_t k) { return kpad_of(k) / 4 * B_KSTEP * 8; }

// Split widths and the derived constants used by the kernels.
struct Widths {
  int c0, c1, c2;
};

// ---------------------------------------------------------------- device math
// Every rounding operation is an explicit _rn intrinsic (never contracted into
// an FMA, never reassociated), so the split and combine are bit-reproducible.
__device__ __forceinline__ double pow2i(int n) {  // 2^n for n in [-1022, 1023], exact
  return __longlong_as_double((long long)(n + 1023) << 52);
}

// 2^n exactly for n in [-1074, 1023] (a subnormal double below -1022).
__device__ __forceinline__ double pow2_any(int n) {
  return n >= -1022 ? pow2i(n) : __longlong_as_double(1LL << (n + 1074));
}

// x 2^n rounded once to nearest-even for ANY int n, i.e. bitwise C99 ldexp(x, n)
// (the oracle scales with ldexp, reading R16): subnormal results on the
// 2^-1074 grid, overflow to +-inf, signed zeros kept.
//   n in [-1074, 1023]: one multiply by the exact power 2^n (IEEE multiplication
//               rounds the exact product once, also for a subnormal factor);
//   n > 1023:   factors 2^1023 (at most twice), then the rest; every factor is
//               >= 1, so a step is exact or overflows, and an intermediate
//               overflow means the result overflows too;
//   n < -1074:  y = x 2^(n+1074), then y 2^-1074.  y is exact whenever it is
//               normal; if not, |x 2^n| < 2^-2096 and both sides give +-0.
#ifdef CASC_LDEXP_NOINLINE  // timing experiment: the rare path as a call
static __device__ __noinline__
#else
static __device__ __forceinline__
#endif
double ldexp_rn_wide(double x, int n) {
  if (n >= -1074 && n <= 1023) return __dmul_rn(x, pow2_any(n));
  if (n > 1023) {
    x = __dmul_rn(x, pow2i(1023));
    n -= 1023;
    if (n > 1023) {
      x = __dmul_rn(x, pow2i(1023));
      n -= 1023;
    }
    return __dmul_rn(x, pow2i(n > 1023 ? 1023 : n));
  }
  const int s = n + 1074 < -1074 ? -1074 : n + 1074;  // clamped: the result is +-0 anyway
  return __dmul_rn(__dmul_rn(x, pow2_any(s)), __longlong_as_double(1LL));
}
// The same scaling as three exact powers of two applied in order,
// x 2^n = ((x s[0]) s[1]) s[2], for n in [-2148, 3069] (every e_i + f_j of
// binary64 operands, e, f in [-1073, 1024]) -- branch-free, for unrolled code:
//   n in [-1074, 1023]: (2^n, 1, 1)                      one rounding;
//   n > 1023:  (2^1023, 2^min(n-1023, 1023), 2^rest)     factors >= 1;
//   n < -1074: (2^(n+1074), 2^-1074, 1)                  as ldexp_rn_wide.
__device__ __forceinline__ void pow2_steps(int n, double s[3]) {
  const bool up = n > 1023, down = n < -1074;
  const int r = n - 1023, r2 = r < 1023 ? r : 1023;
  const int n0 = up ? 1023 : (down ? n + 1074 : n);
  const int n1 = up ? r2 : (down ? -1074 : 0);
  const int n2 = up ? r - r2 : 0;
  s[0] = pow2_any(n0 < -1074 ? -1074 : n0);
  s[1] = pow2_any(n1);
  s[2] = pow2i(n2);
}
__device__ __forceinline__ double ldexp_rn(double x, int n) {
  if ((unsigned)(n + 1022) <= 2045u) return __dmul_rn(x, pow2i(n));  // the common case
  return ldexp_rn_wide(x, n);
}

// Arguments of the fused cascaded-GEMM kernel (casc_gemm.cu).
struct GemmArgs {
  const uint8_t* pa;
  const uint8_t* pb;
  int64_t a_blk, b_blk;  // bytes per packed block
  int64_t a_exp, b_exp;  // byte offset of the exponents inside a block
  int64_t m, n;
  int mblocks, nblocks;
  int st_begin, st_end;  // stage range [begin, end) (a single panel in debug mode)
  int c0, D2;
  double* C_hi;
  double* C_lo;
  int64_t ldc;
  uint8_t* flags;  // m x n (ld ldf) or null
  int64_t ldf;
  double* dbg;     // debug: bins of the single panel, 4 x m x n (canonical scales)
  void* scratch;               // per launch (caller memory, gemm_scratch_bytes): the
                               // three below, set and zeroed by launch_gemm
  unsigned int* wave_counter;  // producers meet here at each tile wave (or null)
  unsigned int* wide_count;    // work items listed for the WIDE re-run
  unsigned int* wide_mask;     // per work item: the warps that met a wide scale
  unsigned int* wide_list;
  // NEXT-4 BLAS update at the tile's last panel: C := alpha (x) AB (+) beta (x) C
  int ab;        // 0: plain C := AB; 1: apply alpha; 2: apply alpha and beta (reads C)
  double alpha_hi, alpha_lo, beta_hi, beta_lo;
  // split mode (small problems): P > 0 -> one work item per (tile, panel), panel
  // sums to t_hi/t_lo [P][m][n] and flags to fbuf [P][m][n]; 0 -> off
  int split_p;
  double* t_hi;
  double* t_lo;
  uint8_t* fbuf;
  double un_b2;    // 2^(c1-c0): bin2' -> bin2 for the debug export
  // SYRK (NEXT-4, casc_syrk_fp64x2): 0 all tiles; 1 lower triangle (tiles with
  // nb <= mb, elements with row >= col stored); 2 upper (nb >= mb, row <= col)
  int tri;
  // 1: the caller zeroed the scratch head before the split launch that precedes
  // this one, and the product kernel is a programmatic dependent launch of it
  int pdl;
  // TRMM (NEXT-4, reading R28): one operand triangular, so a tile's k range
  // stops where that operand's rows / columns are zero.  0 none; 1 A lower
  // (row block mb: k < 64 (mb+1)); 2 A upper (k >= 64 mb); 3 B lower (column
  // block nb: k >= 64 nb); 4 B upper (k < 64 (nb+1)).  AB instantiations only.
  int band;
};

// scratch: [256-byte head: wave counter, WIDE count][WIDE warp masks, one u32
// per item][WIDE list, one u32 per item]; the head and the masks are zeroed
// per launch (gemm_scratch_zero_bytes)
constexpr int GEMM_SCRATCH_HEAD = 256;
cudaError_t launch_gemm(const GemmArgs& a, int num_sms, cudaStream_t st);
size_t gemm_scratch_bytes(int64_t work_items);
size_t gemm_scratch_zero_bytes(int64_t work_items);

// Arguments of the single slice-GEMM kernel of the simple path (casc_simple.cu).
struct SliceArgs {
  const uint8_t* pa;
  const uint8_t* pb;
  int64_t a_blk, b_blk;
  int64_t m, n;
  int mblocks, nblocks;
  int st_begin, st_end;  // stages of one panel
  int sa, sb;            // slice of A (0..3) and of B (0..6)
  double* out;           // m x n, leading dimension ldo
  int64_t ldo;
  int accumulate;        // out = out + scale * P  (else out = scale * P)
  double scale;          // exact power of two (un-alignment for the debug export)
};

cudaError_t launch_slice_gemm(const SliceArgs& a, int num_sms, cudaStream_t st);
cudaError_t launch_epilogue(const double* bins, const void* pa, const void* pb, int64_t k, int q,
                            int64_t m, int64_t n, double* C_hi, double* C_lo, int64_t ldc,
                            uint8_t* flags, int first, Widths w, int num_sms, cudaStream_t st);

}  // namespace casc
