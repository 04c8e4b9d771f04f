// casc_i8.cu — NEXT-3: the FP64x2 GEMM C := A B as a cascade
// of INT8 tensor-core GEMMs, the variant the paper proposes in §6 "FP64x2 in
// terms of INT8": the matrices are "converted into fixed point
// numbers which can be stored in integers", cascaded into ~14-15
// int8 splits, multiplied with the y(y+1)/2 products of the triangle i + j < y
// and accumulated in 32-bit integers.
// readings R22-R26 fix what the paper leaves open (the CPU oracle
// oracle/casc_i8_oracle.c follows the same readings with its own code):
//   R22  k panel of 8192; per (row, panel) / (column, panel) scale exponent e
//        (frexp exponent of max |hi|); every bin of a panel is an exact int32.
//   R23  X = rint(hi 2^(F-e)) + rint(lo 2^(F-e)), F = 6 + 8(y-1); slices = the
//        balanced base-256 digits of X (d_0 in [-64, 64], others [-128, 127]).
//   R24  bin_s = sum_p sum_(i+j=s) dA_i dB_j, s < y.
//   R25  (rev. 2) groups of four bins aligned at the least significant bin
//        (bins 0 .. r-1, r = (y-1) % 4 + 1, first) -> exact int64 group values
//        V_g; the panel's exact product S = sum_g V_g 2^(32(ng-1-g)) (192-bit)
//        is rounded to the nearest FP64x2 number T = (RN(x), RN(x - T.hi)),
//        x = S 2^(e+f-12-8(y-1)), with integer instructions only (subnormals
//        included); C = T over the first panel, C = C (+) T over the others.
//   R26  flag |= |T.hi| <= kp 2^(e+f-50).
//
// Phase 1 (HBM-bound):
//   i8_rowmax_kernel / i8_colmax_kernel  max |hi| per (row | column, panel) as
//                                        an atomicMax on the bit pattern;
//   i8_digits_kernel<A|B>                digits, written straight into the
//        tcgen05 shared-memory layout: per (slice, 128-row block, 128-byte k
//        block) one contiguous 16 KB chunk, K-major, 128-byte swizzle (row r at
//        (r/8)*1024 + (r%8)*128, 16-byte unit u at u ^ (r%8)), so the GEMM
//        moves every operand tile with ONE cp.async.bulk and points the MMA
//        descriptor at it.
// Phase 2+3: i8_gemm_kernel, persistent CTA pairs (cluster of 2, one pair per
// two SMs, 320 threads each); the pair computes a 256 x 128 C tile:
//   warp 8     TMA producer (both CTAs): 2-SM tensor copies
//              (cp.async.bulk.tensor.2d.cta_group::2) of the CTA's half of each
//              operand chunk (A: its 128 rows, 16 KB; B: its 64 of the chunk's
//              128 columns, 8 KB) into rings of 9 (A) + 10 (B) slots, completing on the
//              leader CTA's mbarriers; a soft wave synchronisation aligns the
//              producers of all CTAs at every (panel, group) sweep (L2 reuse);
//   warp 9     MMA issuer (leader CTA; also allocates TMEM): tcgen05.mma
//              .cta_group::2.kind::i8, M = 256, N = 128, K = 32, s8 x s8 -> s32,
//              the four bins of a group in tensor memory (4 x 128 = all 512
//              columns of each CTA); per 128-byte k block the group's operands
//              stream as a chain A_top .. A_s, B_0, A_(s-1), B_1, ... so every
//              chunk is loaded once and meets all (up to four) partners while
//              resident; commits are multicast to both CTAs;
//   warps 0-7  epilogue (both CTAs): tcgen05.ld of the int32 bins of the CTA's
//              128 rows (warp w reads TMEM lane quarter w%4, column half w/4)
//              into exact int64 group values (then TMEM is released), then once
//              per panel the exact panel product rounded to T (R25 rev. 2), C in a
//              per-CTA workspace, the detector, and the final store of C and the
//              flags.
// Producer and MMA warps have the highest warp ids: the sub-partition scheduler
// favours them over the epilogue warps they share an issue slot with.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/casc.h"
#include "casc_dd.cuh"
#include "casc_host.cuh"
#include "casc_ptx.cuh"

// DBG instantiation: the combine below its early `continue` is unreachable by design
#pragma nv_diag_suppress 128

namespace casc {
namespace i8 {

constexpr int KC8 = 8192;          // R22 panel depth
constexpr int KB = 128;            // k bytes per chunk (one 128-byte swizzle row)
constexpr int KBP = KC8 / KB;      // k blocks per panel (64)
constexpr int TR = 128;            // rows (A) / columns (B) per chunk = tile edge
constexpr int CHUNK = TR * KB;     // 16384 bytes
constexpr int YMIN = 3, YMAX = 15;
// C columns of a pair tile = the MMA's N (CASC_I8_TC, 128 or 64).  Tensor
// memory holds 512 / TC int32 accumulators of the tile, so with TC = 64 one
// sweep over k covers eight bins (two R25 value groups) instead of four, and
// every operand chunk is streamed that much less often (the data movement is
// what keeps the power-capped clock low: no operand loads at all runs at
// 1.70 GHz instead of 1.46 GHz).
#ifndef CASC_I8_TC
#define CASC_I8_TC 128
#endif
constexpr int TC = CASC_I8_TC;
static_assert(TC == 128 || TC == 64, "pair-tile columns: 128 or 64");
constexpr int CPB = TR / TC;       // pair-tile column blocks per 128-column packed block
constexpr int VG = 4;              // bins per R25 value group (exact int64 group values)
constexpr int NBIN = 512 / TC;     // bins per MMA group (tensor memory: 512 / TC accumulators)
constexpr int GPM = NBIN / VG;     // R25 value groups per MMA group
#ifndef CASC_I8_NSA
#define CASC_I8_NSA 9
#endif
#ifndef CASC_I8_NSB
#define CASC_I8_NSB (CASC_I8_TC == 64 ? 18 : 10)
#endif
constexpr int NSA = CASC_I8_NSA, NSB = CASC_I8_NSB;  // smem ring slots (A: 16 KB; B: TC/2 rows)
constexpr int NGMAX = (YMAX + VG - 1) / VG;  // R25 value groups per panel, at most
constexpr int64_t WS_PER_CTA = (int64_t)(2 + NGMAX) * TR * TC;  // doubles / int64 per CTA
// (320 threads: up to 204 registers each, room for the epilogue's 64 exact
// group values)
constexpr int THREADS = 320;
// warps 0-7 epilogue, warp 8 TMA producer, warp 9 MMA issuer + TMEM allocator.
// The warp scheduler of a sub-partition (warp id % 4) favours the highest warp
// id, so the producer and the MMA issuer win the issue slot over the epilogue
// warps they share a sub-partition with.
constexpr int PRODUCER_WARP = 8, MMA_WARP = 9, EPI_THREADS = 256;
#ifndef CASC_I8_SYNC_KB
#define CASC_I8_SYNC_KB 64  // k blocks between wave synchronisations (64 = once per sweep)
#endif
#ifndef CASC_I8_SUSPEND_NS
#define CASC_I8_SUSPEND_NS 1000000
#endif
#ifndef CASC_I8_EPI_SUB
#define CASC_I8_EPI_SUB 4
#endif
constexpr int EPI_SUB = CASC_I8_EPI_SUB;  // elements per phase-2 step of the epilogue
#ifndef CASC_I8_GROUP_M
#define CASC_I8_GROUP_M 6
#endif
constexpr int GROUP_M = CASC_I8_GROUP_M;  // tile raster: GROUP_M row-pair blocks sweep the columns
constexpr size_t SMEM = (size_t)NSA * CHUNK + (size_t)NSB * (TC / 2) * KB + 1024 + 1024;

struct Pack {
  int64_t R;    // 128-row blocks (even: the GEMM's CTA pairs take them two at a time)
  int64_t KBn;  // 128-byte k blocks
  int64_t P;    // k panels
  int y;
};
__host__ __device__ inline Pack pack_of(int64_t rows, int64_t k, int y) {
  return Pack{(rows + 2 * TR - 1) / (2 * TR) * 2, (k + KB - 1) / KB, (k + KC8 - 1) / KC8, y};
}
// A packed operand is R contiguous blocks of 128 rows (A) / columns (B), so a
// range of blocks (a row block of A, a column slab of B) is a contiguous byte
// range.  Block layout: [y slices][KBn k blocks] 16 KB chunks, then the int32
// scale exponents [P][128], then scratch u64 max |hi| bits [P][128].
__host__ __device__ inline int64_t al256(int64_t b) { return (b + 255) / 256 * 256; }
__host__ __device__ inline int64_t blk_exp_off(const Pack& g) {
  return (int64_t)g.y * g.KBn * CHUNK;
}
__host__ __device__ inline int64_t blk_max_off(const Pack& g) {
  return blk_exp_off(g) + al256(g.P * TR * 4);
}
__host__ __device__ inline int64_t blk_bytes(const Pack& g) {
  return al256(blk_max_off(g) + g.P * TR * 8);
}
__host__ __device__ inline int64_t packed_bytes(const Pack& g) { return g.R * blk_bytes(g); }
__host__ __device__ inline int64_t chunk_off(const Pack& g, int t, int64_t rb, int64_t kb) {
  return rb * blk_bytes(g) + ((int64_t)t * g.KBn + kb) * CHUNK;
}
__host__ __device__ inline int64_t exp_at(const Pack& g, int64_t r, int64_t q) {
  return (r / TR) * blk_bytes(g) + blk_exp_off(g) + (q * TR + r % TR) * 4;
}
__host__ __device__ inline int64_t max_at(const Pack& g, int64_t r, int64_t q) {
  return (r / TR) * blk_bytes(g) + blk_max_off(g) + (q * TR + r % TR) * 8;
}
// byte of (row r, k byte c) inside a chunk: K-major, 128-byte swizzle
__host__ __device__ inline uint32_t sw128(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((c >> 4) ^ (r & 7)) & 7) << 4) + (c & 15));
}

// ------------------------------------------------------------------ phase 1
__device__ __forceinline__ unsigned long long absbits(double x) {
  return (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
}

// max |A_hi| per (row, panel): warp = one row x 1024 k, 8 rows per block.
// kchunk (a multiple of 32 dividing 8192): k per warp; smaller for small
// problems so that the grid covers the SMs.
__global__ void __launch_bounds__(256) i8_rowmax_kernel(const double* __restrict__ hi, int64_t ld,
                                                        int64_t rows, int64_t k, Pack g,
                                                        uint8_t* __restrict__ packed, int kchunk) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + warp;
  const int64_t p0 = (int64_t)blockIdx.y * kchunk;
  if (r >= rows) return;
  unsigned long long m = 0;
  const double* row = hi + r * ld;
#pragma unroll 8
  for (int i = 0; i < kchunk / 32; ++i) {
    const int64_t p = p0 + i * 32 + lane;
    if (p < k) m = max(m, absbits(__ldg(row + p)));
  }
  for (int o = 16; o; o >>= 1) m = max(m, (unsigned long long)__shfl_xor_sync(~0u, m, o));
  if (lane == 0 && m)
    atomicMax(reinterpret_cast<unsigned long long*>(packed + max_at(g, r, p0 / KC8)), m);
}

// max |B_hi| per (column, panel): thread = one column x kchunk k (a divisor of
// 8192; smaller for small problems so that the grid covers the SMs).
__global__ void __launch_bounds__(256) i8_colmax_kernel(const double* __restrict__ hi, int64_t ld,
                                                        int64_t cols, int64_t k, Pack g,
                                                        uint8_t* __restrict__ packed, int kchunk) {
  const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t p0 = (int64_t)blockIdx.y * kchunk;
  if (j >= cols) return;
  unsigned long long m = 0;
#pragma unroll 8
  for (int i = 0; i < kchunk; ++i) {
    const int64_t p = p0 + i;
    if (p < k) m = max(m, absbits(__ldg(hi + p * ld + j)));
  }
  if (m) atomicMax(reinterpret_cast<unsigned long long*>(packed + max_at(g, j, p0 / KC8)), m);
}

// 2^n as a double for n in [-1022, 1023] (exact).
__device__ __forceinline__ double p2(int n) { return __longlong_as_double((long long)(n + 1023) << 52); }
// x * 2^n, exact whenever the result is a normal double (like ldexp).
__device__ __forceinline__ double mulp2(double x, int n) {
  if (n >= -1022 && n <= 1023) return __dmul_rn(x, p2(n));
  const int h = n / 2;
  return __dmul_rn(__dmul_rn(x, p2(h)), p2(n - h));
}
// ---- Reading R25 (rev. 2) on the integer pipe.  The panel value T is the FP64x2
// number nearest the exact panel product x = S 2^w (S an exact integer of up to
// ~150 bits): T.hi = RN(x), T.lo = RN(x - T.hi).  All of it is integer work:
// FP64 ALU instructions issued while the int8 MMAs run were measured ~5x slower
// than on an idle SM (they share a datapath), the integer pipe is not.
struct U192 {
  unsigned long long l0, l1, l2;  // little-endian limbs
};
__device__ __forceinline__ U192 u192_add(U192 a, U192 b) {
  U192 r;
  r.l0 = a.l0 + b.l0;
  const unsigned long long c0 = r.l0 < a.l0;
  const unsigned long long t = a.l1 + b.l1;
  const unsigned long long c1 = t < a.l1;
  r.l1 = t + c0;
  const unsigned long long c2 = c1 | (r.l1 < t);
  r.l2 = a.l2 + b.l2 + c2;
  return r;
}
__device__ __forceinline__ U192 u192_neg(U192 a) {
  U192 r{~a.l0, ~a.l1, ~a.l2};
  return u192_add(r, U192{1ull, 0ull, 0ull});
}
// V 2^(32 sh32), sign-extended to 192 bits (sh32 = 0 .. 3)
__device__ __forceinline__ U192 u192_from_shifted(long long v, int sh32) {
  const unsigned long long sx = v < 0 ? ~0ull : 0ull;
  const unsigned long long u = (unsigned long long)v;
  switch (sh32) {
    case 0: return U192{u, sx, sx};
    case 1: return U192{u << 32, (unsigned long long)(v >> 32), sx};
    case 2: return U192{0ull, u, sx};
    default: return U192{0ull, u << 32, (unsigned long long)(v >> 32)};
  }
}
__device__ __forceinline__ int u192_bitlen(const U192& a) {
  if (a.l2) return 192 - __clzll((long long)a.l2);
  if (a.l1) return 128 - __clzll((long long)a.l1);
  if (a.l0) return 64 - __clzll((long long)a.l0);
  return 0;
}
// bits [c, c + 64) of a (c >= 0)
__device__ __forceinline__ unsigned long long u192_shr64(const U192& a, int c) {
  if (c >= 192) return 0ull;
  const unsigned long long x = c < 64 ? a.l0 : c < 128 ? a.l1 : a.l2;
  const unsigned long long z = c < 64 ? a.l1 : c < 128 ? a.l2 : 0ull;
  const int b = c & 63;
  return b ? (x >> b) | (z << (64 - b)) : x;
}
// a mod 2^c (c >= 0)
__device__ __forceinline__ U192 u192_low(const U192& a, int c) {
  auto mask = [](int bits) { return bits >= 64 ? ~0ull : bits <= 0 ? 0ull : (1ull << bits) - 1; };
  return U192{a.l0 & mask(c), a.l1 & mask(c - 64), a.l2 & mask(c - 128)};
}
__device__ __forceinline__ bool u192_nonzero(const U192& a) { return (a.l0 | a.l1 | a.l2) != 0; }
// the double +-q 2^e2 for an integer q <= 2^54 whose value is representable
// (q 2^e2 on or above the 2^-1074 grid); overflow gives inf
__device__ __forceinline__ double make_double(bool neg, unsigned long long q, int e2) {
  unsigned long long bits = 0;
  if (q) {
    const int top = 63 - __clzll((long long)q);  // q in [2^top, 2^(top+1))
    int sh = 52 - top;                          // normalise to [2^52, 2^53)
    if (e2 - sh < -1074) sh = e2 + 1074;        // subnormal: e2 -> -1074
    q = sh >= 0 ? q << sh : q >> (-sh);         // exact (q even when shifted right)
    e2 -= sh;
    if (q >= (1ull << 52)) {                    // normal
      const int field = e2 + 1075;
      bits = field >= 2047 ? 0x7ff0000000000000ull
                           : ((unsigned long long)field << 52) | (q & 0xfffffffffffffull);
    } else {
      bits = q;                                 // subnormal (e2 == -1074)
    }
  }
  if (neg) bits |= 0x8000000000000000ull;
  return __longlong_as_double((long long)bits);
}
// RN(+-M 2^w) (ties to even, subnormals, RN(0) = +0); R, rneg: the exact
// remainder M 2^w - |RN| as a magnitude and a sign relative to the input's
__device__ __forceinline__ double rn_u192(const U192& M, int w, bool neg, U192& R, bool& rneg) {
  R = U192{0ull, 0ull, 0ull};
  rneg = false;
  const int len = u192_bitlen(M);
  if (len == 0) return 0.0;
  int c = len - 53;
  if (c < -1074 - w) c = -1074 - w;
  if (c <= 0) return make_double(neg, M.l0, w);  // exact: M < 2^53
  unsigned long long q = u192_shr64(M, c);
  const U192 low = u192_low(M, c);
  const bool guard = (u192_shr64(M, c - 1) & 1ull) != 0;
  const bool sticky = u192_nonzero(u192_low(M, c - 1));
  const bool up = guard && (sticky || (q & 1ull));
  if (up) {  // remainder 2^c - low, opposite sign
    U192 two_c{0ull, 0ull, 0ull};
    if (c < 64) two_c.l0 = 1ull << c;
    else if (c < 128) two_c.l1 = 1ull << (c - 64);
    else if (c < 192) two_c.l2 = 1ull << (c - 128);
    R = u192_add(two_c, u192_neg(low));
    rneg = true;
    ++q;
  } else {
    R = low;
  }
  return make_double(neg, q, w + c);
}

// T = (RN(x), RN(x - RN(x))) for x = S 2^w, S a signed 192-bit integer.  When
// w >= -1022 every nonzero result is normal and the rounding position is
// simply 53 bits below the leading bit: a 128-bit fast path (|S| < 2^145, so
// the cut c = len - 53 <= 92); otherwise the general rn_u192 (subnormal grid).
// Both give the same bits (tests/test_gpu_i8.py vs the big-integer oracle).
__device__ __forceinline__ void rn_pair(U192 S, int w, double& hi, double& lo) {
  const bool neg = (long long)S.l2 < 0;
  if (neg) S = u192_neg(S);
  if (w < -1022) {
    U192 R, R2;
    bool rneg, r2neg;
    hi = rn_u192(S, w, neg, R, rneg);
    lo = rn_u192(R, w, neg != rneg, R2, r2neg);
    return;
  }
  typedef unsigned __int128 u128;
  const int len = u192_bitlen(S);
  if (len <= 53) {  // exact (S = 0 gives +0)
    hi = make_double(neg, S.l0, w);
    lo = 0.0;
    return;
  }
  const int c = len - 53;
  unsigned long long q;
  u128 rem;
  if (c < 64) {  // len < 117: S.l2 == 0
    const u128 v = ((u128)S.l1 << 64) | S.l0;
    q = (unsigned long long)(v >> c);
    rem = v & (((u128)1 << c) - 1);
  } else {
    const u128 v = ((u128)S.l2 << 64) | S.l1;
    q = (unsigned long long)(v >> (c - 64));
    rem = ((u128)(S.l1 & ((1ull << (c - 64)) - 1)) << 64) | S.l0;
  }
  const u128 half = (u128)1 << (c - 1);
  const bool up = rem > half || (rem == half && (q & 1ull));
  const u128 R = up ? (((u128)1 << c) - rem) : rem;
  hi = make_double(neg, q + (up ? 1ull : 0ull), w + c);
  const bool lneg = neg != up;
  const unsigned long long Rh = (unsigned long long)(R >> 64), Rl = (unsigned long long)R;
  const int len2 = Rh ? 128 - __clzll((long long)Rh) : (Rl ? 64 - __clzll((long long)Rl) : 0);
  if (len2 == 0) {
    lo = 0.0;
  } else if (len2 <= 53) {
    lo = make_double(lneg, Rl, w);
  } else {
    const int c2 = len2 - 53;
    const unsigned long long q2 = (unsigned long long)(R >> c2);
    const u128 rem2 = R & (((u128)1 << c2) - 1);
    const u128 half2 = (u128)1 << (c2 - 1);
    const bool up2 = rem2 > half2 || (rem2 == half2 && (q2 & 1ull));
    lo = make_double(lneg, q2 + (up2 ? 1ull : 0ull), w + c2);
  }
}

// exact conversion of an integer-valued double (|w| < 2^126) to int128
__device__ __forceinline__ __int128 to_i128(double w) {
  if (fabs(w) < 9.0e18) return (__int128)__double2ll_rz(w);
  const unsigned long long b = (unsigned long long)__double_as_longlong(w);
  const int ex = (int)((b >> 52) & 0x7ff) - 1075;
  const __int128 mant = (__int128)((b & 0xfffffffffffffull) | 0x10000000000000ull);
  const __int128 v = mant << ex;
  return (b >> 63) ? -v : v;
}
__device__ __forceinline__ int scale_exp(unsigned long long bits) {
  if (!bits) return 0;
  int e;
  frexp(__longlong_as_double((long long)bits), &e);
  return e;
}

// 128-bit two's-complement integer as four 32-bit words (w[0] least significant)
struct U128 {
  uint32_t w[4];
};
// exact conversion of an integer-valued double (|x| < 2^113) to 128 bits
__device__ __forceinline__ U128 dbl_to_u128(double x) {
  U128 r{{0u, 0u, 0u, 0u}};
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  const int be = (int)((b >> 52) & 0x7ff);
  if (be == 0) return r;  // +-0 (an integer-valued double is never subnormal here)
  const int sh = be - 1075;  // value = mant * 2^sh, mant in [2^52, 2^53)
  unsigned long long mant = (b & 0xfffffffffffffull) | 0x10000000000000ull;
  unsigned long long lo, hi;
  if (sh <= 0) {
    lo = mant >> (-sh);  // exact: x is an integer
    hi = 0;
  } else if (sh < 64) {
    lo = mant << sh;
    hi = sh > 11 ? mant >> (64 - sh) : 0ull;
  } else {
    lo = 0;
    hi = mant << (sh - 64);
  }
  if (b >> 63) {  // negate (two's complement)
    lo = ~lo + 1ull;
    hi = ~hi + (lo == 0 ? 1ull : 0ull);
  }
  r.w[0] = (uint32_t)lo;
  r.w[1] = (uint32_t)(lo >> 32);
  r.w[2] = (uint32_t)hi;
  r.w[3] = (uint32_t)(hi >> 32);
  return r;
}
__device__ __forceinline__ U128 add_u128(const U128& a, const U128& b) {
  U128 r;
  asm("add.cc.u32 %0, %4, %8;\n\taddc.cc.u32 %1, %5, %9;\n\taddc.cc.u32 %2, %6, %10;\n\t"
      "addc.u32 %3, %7, %11;"
      : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
      : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]), "r"(b.w[1]),
        "r"(b.w[2]), "r"(b.w[3]));
  return r;
}

// Digits (R23) of 16 consecutive k of one vector, one 16-byte unit per slice.
// X = rint(hi 2^(F-e)) + rint(lo 2^(F-e)) exactly (128-bit); with K = 0x80 in
// each of the y-1 lowest byte positions, U = (X + K) xor K has the balanced
// base-256 digits of X as its bytes: d_t = byte (y-1-t) of U (adding 128 to a
// digit in [-128, 127] cannot carry; the top digit d_0 in [-64, 64] is the
// sign-extended remainder).  COLS = false: A rows (element (r, p) at
// hi[r*ld + p]); block = 32 rows x 128 k.  COLS = true: B columns (element (p, j)
// at hi[p*ld + j]); block = 128 columns x 32 k.  Padding rows / k get zero
// digits, so the packed operand is fully defined.
template <bool COLS>
__global__ void __launch_bounds__(256) i8_digits_kernel(const double* __restrict__ hi,
                                                        const double* __restrict__ lo, int64_t ld,
                                                        int64_t rows, int64_t k, Pack g,
                                                        uint8_t* __restrict__ packed) {
  const int t = threadIdx.x;
  const int64_t kb = blockIdx.y;
  int64_t r;
  int u0, du, nu;
  if (COLS) {
    r = (int64_t)blockIdx.x * 128 + (t & 127);
    u0 = 2 * blockIdx.z + (t >> 7);  // 16-k unit: grid.z = 4 pairs of units
    du = 0;
    nu = 1;
  } else {
    r = (int64_t)blockIdx.x * 32 + (t >> 3);
    u0 = t & 7;
    du = 8;
    nu = 1;
  }
  if (r >= g.R * TR) return;
  const int64_t q = kb / KBP;
  const int e =
      r < rows ? scale_exp(*reinterpret_cast<const unsigned long long*>(packed + max_at(g, r, q)))
               : 0;
  if ((kb % KBP) == 0 && (COLS ? u0 : t & 7) == 0)
    *reinterpret_cast<int32_t*>(packed + exp_at(g, r, q)) = e;
  const int y = g.y;
  const int F = 6 + 8 * (y - 1);
  const int s1 = min(F - e, 1023), s2 = F - e - s1;
  const double sc1 = p2(s1), sc2 = p2(s2);
  // K: 0x80 in byte positions 0 .. y-2
  U128 K{{0u, 0u, 0u, 0u}};
#pragma unroll
  for (int pos = 0; pos < 16; ++pos)
    if (pos < y - 1) K.w[pos >> 2] |= 0x80u << (8 * (pos & 3));
  const int rl = (int)(r % TR);
  const int64_t rb = r / TR;
  for (int iu = 0; iu < nu; ++iu) {
    const int u = u0 + iu * du;
    const int64_t p0 = kb * KB + u * 16;
    U128 U[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int64_t p = p0 + i;
      double h = 0.0, l = 0.0;
      if (r < rows && p < k) {
        const int64_t idx = COLS ? p * ld + r : r * ld + p;
        h = __ldg(hi + idx);
        l = __ldg(lo + idx);
      }
      U128 x = add_u128(dbl_to_u128(rint(__dmul_rn(__dmul_rn(h, sc1), sc2))),
                        dbl_to_u128(rint(__dmul_rn(__dmul_rn(l, sc1), sc2))));
      x = add_u128(x, K);
#pragma unroll
      for (int w = 0; w < 4; ++w) x.w[w] ^= K.w[w];
      U[i] = x;
    }
    const uint32_t off = sw128(rl, u * 16);
#pragma unroll
    for (int pos = 0; pos < 16; ++pos) {  // byte position pos holds slice y-1-pos
      if (pos >= y) break;
      const int sl = y - 1 - pos;
      const int wi = pos >> 2;
      const uint32_t sel = (uint32_t)(pos & 3);
      // gather byte `pos` of the 16 elements into 4 words (PRMT)
      uint32_t o[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const uint32_t a0 = U[4 * v + 0].w[wi], a1 = U[4 * v + 1].w[wi];
        const uint32_t a2 = U[4 * v + 2].w[wi], a3 = U[4 * v + 3].w[wi];
        const uint32_t lo2 = __byte_perm(a0, a1, sel | ((sel + 4) << 4));
        const uint32_t hi2 = __byte_perm(a2, a3, sel | ((sel + 4) << 4));
        o[v] = __byte_perm(lo2, hi2, 0x5410);
      }
      *reinterpret_cast<uint4*>(packed + chunk_off(g, sl, rb, kb) + off) =
          make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// zero the max |hi| scratch of every (block, panel) before the atomicMax passes
__global__ void i8_zero_max_kernel(Pack g, uint8_t* __restrict__ packed) {
  const int64_t total = g.R * g.P * TR;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x)
    *reinterpret_cast<unsigned long long*>(packed + max_at(g, x % (g.R * TR), x / (g.R * TR))) = 0;
}

// Debug export: packed chunks -> canonical digits D[t][r][p] (rows x k) and
// exponents E[q][r].
__global__ void i8_unpack_kernel(const uint8_t* __restrict__ packed, Pack g, int64_t rows,
                                 int64_t k, int8_t* __restrict__ D, int32_t* __restrict__ E) {
  const int64_t total = (int64_t)g.y * rows * k;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = x % k, r = (x / k) % rows;
    const int t = (int)(x / (k * rows));
    D[x] = (int8_t)packed[chunk_off(g, t, r / TR, p / KB) + sw128((int)(r % TR), (int)(p % KB))];
  }
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < g.P * rows;
       x += (int64_t)gridDim.x * blockDim.x)
    E[x] = *reinterpret_cast<const int32_t*>(packed + exp_at(g, x % rows, x / rows));
}

// ------------------------------------------------------------------ phase 2+3
struct GemmArgs {
  const uint8_t* pa;
  const uint8_t* pb;
  Pack ga, gb;
  int64_t m, n, k;
  double* C_hi;
  double* C_lo;
  int64_t ldc;
  uint8_t* flags;
  int64_t ldf;          // leading dimension of flags
  double* ws;           // per CTA: C hi, C lo, V[NGMAX] (WS_PER_CTA doubles)
  unsigned int* sync;   // wave-sync counter (zeroed before the launch) or null
  int32_t* dbg;         // debug: bins of panel dbg_panel (y x m x n int32) instead of C
  int64_t dbg_panel;
  // split mode (small single-panel problems): ks > 1 k-block parts per tile, one
  // work item per (tile, part); each item writes its exact partial panel product
  // S (192-bit) to split_ws [item][rank][limb][128 x 128] and a reduce kernel
  // sums the parts and rounds (bitwise the unsplit result: S is exact)
  int ks;
  unsigned long long* split_ws;
  // SYRK (NEXT-4): 0 every tile; 1 lower (pair tiles touching row >= col, only
  // those elements stored); 2 upper
  int tri;
  int ab;               // NEXT-4 update at the final store: 0 none, 1 alpha, 2 alpha and beta
  double ah, al, bh, bl;
};

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: s8 x s8 -> s32, K-major A and B, M = 256 (CTA pair), N = TC
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC >> 3) << 17) |
                           ((uint32_t)(256 >> 4) << 24);
constexpr int BHALF = (TC / 2) * KB;  // each CTA of the pair holds TC/2 of a B chunk's rows

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t leader_addr(const void* p) {  // same offset in CTA rank 0
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_C:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_C;\nbra WAIT_C;\nDONE_C:\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Blocking wait with a suspend-time hint: the thread sleeps until the phase
// completes (or the hint elapses) instead of spinning, so waiting warps do not
// steal issue slots from the MMA warp or burn power.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_S:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE_S;\nbra WAIT_S;\nDONE_S:\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "n"(CASC_I8_SUSPEND_NS)
      : "memory");
}
// warp-uniform wait: the loop condition is a warp vote, so control flow stays
// provably uniform and the scalar state can live in the uniform datapath
__device__ __forceinline__ void mbar_wait_uniform(uint64_t* bar, uint32_t parity) {
  while (!__all_sync(0xffffffffu, mbar_try(bar, parity))) {
  }
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster)
               : "memory");
}
// One elected lane: (leader only) arm the leader's barrier for both CTAs' bytes,
// then a 2-SM TMA of `rows` 128-byte rows at row coordinate y of `map` into this
// CTA's smem, completing on the LEADER's barrier (bar_cluster).
__device__ __forceinline__ void tma_pair_elect(void* dst, const CUtensorMap* map, int y,
                                               uint64_t* bar_local, uint32_t bar_cluster,
                                               uint32_t arm_bytes) {
  asm volatile(
      "{\n.reg .pred e, l;\nelect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 l, %4, 0;\n"
      "and.pred l, l, e;\n"
      "@l mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %4;\n"
      "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%5, %2}], [%6];\n"
      "}\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(y), "r"(smem_u32(bar_local)), "r"(arm_bytes),
      "r"(0), "r"(bar_cluster)
      : "memory");
}
// Four MMAs (K = 4 x 32 bytes, one 128-byte chunk) into accumulator tmem_d,
// issued by one elected lane of the (converged) leader MMA warp for the pair.
// acc == 0: the first overwrites the accumulator.
__device__ __forceinline__ void mma_i8_x4(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred e, p, t;\n.reg .b64 a1, a2, a3, b1, b2, b3;\n"
      "add.s64 a1, %1, 2;\nadd.s64 a2, %1, 4;\nadd.s64 a3, %1, 6;\n"
      "add.s64 b1, %2, 2;\nadd.s64 b2, %2, 4;\nadd.s64 b3, %2, 6;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %3, 0;\n"
      "setp.eq.b32 t, 0, 0;\n"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %4, p;\n"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], a1, b1, %4, t;\n"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], a2, b2, %4, t;\n"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], a3, b3, %4, t;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(acc), "n"(IDESC));
}
// tcgen05.commit (multicast to both CTAs of the pair) to one / two mbarriers
__device__ __forceinline__ void mma_commit1(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mma_commit2(uint64_t* bar0, uint64_t* bar1) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %2;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%1], %2;\n}\n" ::"r"(smem_u32(bar0)),
      "r"(smem_u32(bar1)), "h"((uint16_t)3)
      : "memory");
}

// timing studies only (wrong results): CASC_I8_NOWAIT, the MMAs do not wait for
// the epilogue to drain tensor memory; CASC_I8_NOTMA, no operand loads at all
// (the MMA issue rate on stale shared memory)
#ifdef CASC_I8_PROF  // timing study: MMA-issuer cycles spent in each kind of wait
__device__ unsigned long long g_i8prof[1024][64];
#define I8_PROF_WAIT(slot, stmt)                                    \
  do {                                                              \
    const long long t0_ = clock64();                                \
    stmt;                                                           \
    if ((threadIdx.x & 31) == 0)                                    \
      g_i8prof[blockIdx.x][slot] += (unsigned long long)(clock64() - t0_); \
  } while (0)
#else
#define I8_PROF_WAIT(slot, stmt) stmt
#endif
#ifdef CASC_I8_NOTMA
#define CASC_I8_WAITS_ON 0
#else
#define CASC_I8_WAITS_ON 1
#endif
// The MMAs of one 128-byte k block of a group (bins S .. S+NB-1), chain
// order: for B_j (j = 0 .. top) its partners A_i, i = top-j .. max(0, S-j).
// Everything except the ring positions is a compile-time constant.
// One 32-byte k step (kk) of A_i against its P partners B_j, issued by one
// elected lane: the A operand is read from shared memory once and held in the
// tensor core's A collector (collector::a::fill / use / lastuse) for the other
// P-1 MMAs.  d[u]: accumulator column of partner u; acc == 0: the MMAs
// overwrite (first k step of the panel).
template <int P>
__device__ __forceinline__ void mma_i8_astat(const uint32_t (&d)[4], uint64_t a,
                                             const uint64_t (&b)[4], uint32_t acc) {
  if constexpr (P == 1) {
    asm volatile(
        "{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %3, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %4, p;\n}\n" ::"r"(d[0]),
        "l"(a), "l"(b[0]), "r"(acc), "n"(IDESC));
  } else if constexpr (P == 2) {
    asm volatile(
        "{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %5, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::i8.collector::a::fill [%0], %2, %3, %6, p;\n"
        "@e tcgen05.mma.cta_group::2.kind::i8.collector::a::lastuse [%1], %2, %4, %6, p;\n}\n" ::"r"(
            d[0]),
        "r"(d[1]), "l"(a), "l"(b[0]), "l"(b[1]), "r"(acc), "n"(IDESC));
  } else if constexpr (P == 3) {
    asm volatile(
        "{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %7, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::i8.collector::a::fill [%0], %3, %4, %8, p;\n"
        "@e tcgen05.mma.cta_group::2.kind::i8.collector::a::use [%1], %3, %5, %8, p;\n"
        "@e tcgen05.mma.cta_group::2.kind::i8.collector::a::lastuse [%2], %3, %6, %8, p;\n}\n" ::"r"(
            d[0]),
        "r"(d[1]), "r"(d[2]), "l"(a), "l"(b[0]), "l"(b[1]), "l"(b[2]), "r"(acc), "n"(IDESC));
  } else {
    asm volatile(
        "{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %9, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::i8.collector::a::fill [%0], %4, %5, %10, p;\n"
        "@e tcgen05.mma.cta_group::2.kind::i8.collector::a::use [%1], %4, %6, %10, p;\n"
        "@e tcgen05.mma.cta_group::2.kind::i8.collector::a::use [%2], %4, %7, %10, p;\n"
        "@e tcgen05.mma.cta_group::2.kind::i8.collector::a::lastuse [%3], %4, %8, %10, p;\n}\n" ::"r"(
            d[0]),
        "r"(d[1]), "r"(d[2]), "r"(d[3]), "l"(a), "l"(b[0]), "l"(b[1]), "l"(b[2]), "l"(b[3]),
        "r"(acc), "n"(IDESC));
  }
}

// The MMAs of one 128-byte k block of a group (bins S .. S+NB-1, TOP = S+NB-1),
// A-stationary chain order: A_i for i = 0 .. TOP meets its partners B_j,
// j = TOP-i .. max(0, S-i), while they sit in shared memory (a window of up to
// four B chunks: B_TOP .. B_S first, then one new B_(S-i) per A_i), and for
// each 32-byte k step the A operand is fetched once into the collector.  The
// producer streams B_TOP .. B_S, A_0, B_(S-1), A_1, B_(S-2), A_2, ...
// Everything except the ring positions is a compile-time constant.
template <int S, int NB>
__device__ __forceinline__ void mma_chain(bool first_kb, uint32_t& aseq, uint32_t& bseq,
                                          uint32_t tmem, uint32_t a0, uint32_t b0,
                                          uint64_t* fullA, uint64_t* emptyA, uint64_t* fullB,
                                          uint64_t* emptyB) {
  constexpr int TOP = S + NB - 1;
  const uint32_t bbase = bseq;
#pragma unroll
  for (int i = 0; i <= TOP; ++i) {
    const uint32_t aq = aseq + i;
    const uint32_t as = aq % NSA;
    // B operands first used at this step: B_TOP..B_S at i = 0, B_(S-i) after
    if (!CASC_I8_WAITS_ON) {
    } else if (i == 0) {
#pragma unroll
      for (int u = 0; u < NB; ++u)
        I8_PROF_WAIT(16 + S, mbar_wait_uniform(&fullB[(bbase + u) % NSB], ((bbase + u) / NSB) & 1));
    } else if (S - i >= 0) {
      const uint32_t bq = bbase + NB + (i - 1);
      I8_PROF_WAIT(16 + S, mbar_wait_uniform(&fullB[bq % NSB], (bq / NSB) & 1));
    }
    if (CASC_I8_WAITS_ON) I8_PROF_WAIT(32 + S, mbar_wait_uniform(&fullA[as], (aq / NSA) & 1));
    tc_fence_after();
    const int jhi = TOP - i, jlo = (S - i > 0 ? S - i : 0);
    const uint64_t ad = sdesc(a0 + as * CHUNK);
    // partners of A_i in batches of up to four, each batch through the A
    // collector (A read from shared memory once per batch and 32-byte k step)
#pragma unroll
    for (int pb = 0; pb < (NB + 3) / 4; ++pb) {
      const int jtop = jhi - 4 * pb;  // this batch: j = jtop .. max(jlo, jtop - 3)
      if (jtop < jlo) break;
      uint32_t d[4];
      uint64_t bd[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = jtop - u;
        if (j >= jlo) {
          const uint32_t bq = j >= S ? bbase + (TOP - j) : bbase + NB + (S - 1 - j);
          bd[u] = sdesc(b0 + (bq % NSB) * BHALF);
          d[u] = tmem + (i + j - S) * TC;
        } else {
          bd[u] = 0;
          d[u] = 0;
        }
      }
      const int np = (jtop - jlo + 1) < 4 ? (jtop - jlo + 1) : 4;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        // at the panel's first k block every bin is first written at i = 0, kk = 0
        const uint32_t acc = (first_kb && i == 0 && kk == 0) ? 0u : 1u;
        const uint64_t bk[4] = {bd[0] + 2 * kk, bd[1] + 2 * kk, bd[2] + 2 * kk, bd[3] + 2 * kk};
#ifdef CASC_I8_NOMMA  // timing study only: no tensor-core work at all
        if (np > 0) continue;
#endif
        if (np == 4)
          mma_i8_astat<4>(d, ad + 2 * kk, bk, acc);
        else if (np == 3)
          mma_i8_astat<3>(d, ad + 2 * kk, bk, acc);
        else if (np == 2)
          mma_i8_astat<2>(d, ad + 2 * kk, bk, acc);
        else
          mma_i8_astat<1>(d, ad + 2 * kk, bk, acc);
      }
    }
    // A_i is done; B_(TOP-i) has met its last partner
    const int jr = TOP - i;
    const uint32_t rq = jr >= S ? bbase + i : bbase + NB + (S - 1 - jr);
    mma_commit2(&emptyA[as], &emptyB[rq % NSB]);
  }
  aseq += (uint32_t)(TOP + 1);
  bseq = bbase + (uint32_t)(S + NB);
}

__device__ __forceinline__ void mma_kblock(int s, int nb, bool first_kb, uint32_t& aseq,
                                           uint32_t& bseq, uint32_t tmem, uint32_t a0,
                                           uint32_t b0, uint64_t* fullA, uint64_t* emptyA,
                                           uint64_t* fullB, uint64_t* emptyB) {
#define CASC_I8_CHAIN(SS, NN)                                                             \
  if (s == SS && nb == NN) {                                                              \
    mma_chain<SS, NN>(first_kb, aseq, bseq, tmem, a0, b0, fullA, emptyA, fullB, emptyB); \
    return;                                                                               \
  }
  // (first bin, bins) of the MMA groups for y = 3 .. 15
#if CASC_I8_TC == 128  // one R25 value group each
  CASC_I8_CHAIN(0, 1) CASC_I8_CHAIN(0, 2) CASC_I8_CHAIN(0, 3) CASC_I8_CHAIN(0, 4)
  CASC_I8_CHAIN(1, 4) CASC_I8_CHAIN(2, 4) CASC_I8_CHAIN(3, 4) CASC_I8_CHAIN(4, 4)
  CASC_I8_CHAIN(5, 4) CASC_I8_CHAIN(6, 4) CASC_I8_CHAIN(7, 4) CASC_I8_CHAIN(8, 4)
  CASC_I8_CHAIN(9, 4) CASC_I8_CHAIN(10, 4) CASC_I8_CHAIN(11, 4)
#else  // two R25 value groups each: (0, r0 [+ 4]), then (r0 + 4, 4 | 8)
  CASC_I8_CHAIN(0, 3) CASC_I8_CHAIN(0, 4) CASC_I8_CHAIN(0, 5) CASC_I8_CHAIN(0, 6)
  CASC_I8_CHAIN(0, 7) CASC_I8_CHAIN(0, 8) CASC_I8_CHAIN(5, 4) CASC_I8_CHAIN(6, 4)
  CASC_I8_CHAIN(7, 4) CASC_I8_CHAIN(8, 4) CASC_I8_CHAIN(5, 8) CASC_I8_CHAIN(6, 8)
  CASC_I8_CHAIN(7, 8)
#endif
#undef CASC_I8_CHAIN
}

// epilogue workspace loads: coherent, no L1 allocation (keeps L1 / shared
// memory bandwidth for the tensor cores' operand reads)
template <typename T>
__device__ __forceinline__ T ld_na(const T* p) {
#ifdef CASC_I8_LD_PLAIN
  return *p;
#else
  if constexpr (sizeof(T) == 8) {
    unsigned long long v;
    asm volatile("ld.global.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
    T r;
    memcpy(&r, &v, 8);
    return r;
  } else {
    return *p;
  }
#endif
}

// named barrier 1 over the 256 epilogue threads
__device__ __forceinline__ void epi_bar_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(EPI_THREADS) : "memory");
}

// pair tile (256 rows x 128 columns) -> (row-pair block, column block), raster
// of GROUP_M row-pair blocks sweeping the column blocks
__device__ __forceinline__ void tile_of(int tile, int64_t RP, int64_t RB, int64_t& rp,
                                        int64_t& cb) {
  const int64_t per = (int64_t)GROUP_M * RB;
  const int64_t grp = tile / per;
  const int64_t first = grp * GROUP_M;
  const int64_t gs = min((int64_t)GROUP_M, RP - first);
  const int64_t rr = tile % per;
  rp = first + rr % gs;
  cb = rr / gs;
}

// (row-pair block, column block) -> pair tile (inverse of tile_of)
__device__ __forceinline__ int64_t tile_index(int64_t rp, int64_t cb, int64_t RP, int64_t RB) {
  const int64_t grp = rp / GROUP_M, first = grp * GROUP_M;
  const int64_t gs = min((int64_t)GROUP_M, RP - first);
  return grp * GROUP_M * RB + cb * gs + (rp - first);
}

// SYRK work list: the pair tiles (256 rows x TC columns) that hold elements of
// the triangle, row pair by row pair: lower cb < 2 CPB (rp + 1), upper cb >= 2 CPB rp
// (RB: pair-tile column blocks of TC columns; a row pair covers 256 / TC of them)
__device__ __forceinline__ int64_t tri_count(int tri, int64_t rp, int64_t RB) {
  return tri == 1 ? min(2 * CPB * (rp + 1), RB) : max(RB - 2 * CPB * rp, (int64_t)0);
}
__device__ __forceinline__ void tri_tile_of(int tile, int tri, int64_t RP, int64_t RB,
                                            int64_t& rp, int64_t& cb) {
  int64_t t = tile;
  for (rp = 0; rp < RP; ++rp) {
    const int64_t c = tri_count(tri, rp, RB);
    if (t < c) break;
    t -= c;
  }
  cb = tri == 1 ? t : 2 * CPB * rp + t;
}

// R25 value group g of a panel: bins s .. s + nb - 1 (bins 0 .. r0-1 first,
// then fours aligned at the least significant bin)
__device__ __forceinline__ void vgroup(int g, int r0, int& s, int& nb) {
  s = g ? r0 + (g - 1) * VG : 0;
  nb = g ? VG : r0;
}
// MMA group G: the value groups [g0, g1) (GPM of them), bins S .. S + NB - 1
// swept together over k (tensor memory holds them all)
__device__ __forceinline__ void mgroup(int G, int r0, int ngroups, int& S, int& NB, int& g0,
                                       int& g1) {
  g0 = G * GPM;
  g1 = min(ngroups, g0 + GPM);
  int s1, n1;
  vgroup(g1 - 1, r0, s1, n1);
  vgroup(g0, r0, S, NB);
  NB = s1 + n1 - S;
}

// The fused kernel on CTA pairs (cluster of 2, tcgen05 cta_group::2): the pair
// computes a 256 x 128 C tile; CTA r holds A rows 128r..128r+127 of it and
// rows 64r..64r+63 of every 128 x 128-byte B chunk; the leader (r = 0) issues
// the M = 256 MMAs for both, each CTA's tensor memory holds its 128 rows.
template <bool DBG, bool SPLITK, bool TRI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    i8_gemm_kernel(const GemmArgs p, const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapB) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + NSA * CHUNK;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + NSB * BHALF);
  uint64_t* fullA = bars;
  uint64_t* emptyA = fullA + NSA;
  uint64_t* fullB = emptyA + NSA;
  uint64_t* emptyB = fullB + NSB;
  uint64_t* tfull = emptyB + NSB;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);
  int32_t* sF = reinterpret_cast<int32_t*>(tempty + 2);  // column exponents [128]

  // warp index through a shuffle: provably warp-uniform, so role branches are
  // uniform and the MMA issuer's descriptors can live in uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSA; ++i) {
      mbar_init(&fullA[i], 1);
      mbar_init(&emptyA[i], 1);
    }
    for (int i = 0; i < NSB; ++i) {
      mbar_init(&fullB[i], 1);
      mbar_init(&emptyB[i], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * EPI_THREADS / 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  const int y = p.ga.y;
  // R25 groups: bins 0 .. r0-1, then fours (aligned at the least significant bin)
  const int r0 = (y - 1) % VG + 1;
  const int ngroups = 1 + (y - r0) / VG;
  const int nmg = (ngroups + GPM - 1) / GPM;  // MMA groups (sweeps over k) per panel
  const int64_t RA = p.ga.R, RB = p.gb.R * CPB, KBn = p.ga.KBn;
  const int64_t RP = RA / 2;
  const int P = (int)p.ga.P;
  int tiles = (int)(RP * RB);
  if (TRI) {
    tiles = 0;
    for (int64_t r = 0; r < RP; ++r) tiles += (int)tri_count(p.tri, r, RB);
  }
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // work items: tiles, or (tile, k-block part) in split mode (P == 1)
  const int ks = SPLITK ? p.ks : 1;
  const int items = tiles * ks;
  auto kb_range = [&](int item, int q, int64_t& kb0, int64_t& kb1) {
    kb0 = (int64_t)q * KBP;
    kb1 = min(kb0 + KBP, KBn);
    if (SPLITK) {
      const int64_t len = kb1 - kb0, part = item % ks;
      kb1 = kb0 + (part + 1) * len / ks;
      kb0 = kb0 + part * len / ks;
    }
  };

  if (warp == PRODUCER_WARP) {
    // ============================ TMA producer (both CTAs) ============================
    // all lanes run the loop; one elected lane arms / issues; the data of both
    // CTAs completes on the leader's full barriers
    uint32_t aseq = 0, bseq = 0;
    auto loadA = [&](int i, int64_t rb, int64_t kb) {
      const uint32_t s = aseq % NSA;
      mbar_wait_sleep(&emptyA[s], ((aseq / NSA) & 1) ^ 1);
      const int row = (int)(chunk_off(p.ga, i, rb, kb) / KB);
      tma_pair_elect(sA + s * CHUNK, &mapA, row, &fullA[s], leader_addr(&fullA[s]),
                     leader ? 2 * CHUNK : 0);
      ++aseq;
    };
    auto loadB = [&](int j, int64_t cb, int64_t kb) {
      const uint32_t s = bseq % NSB;
      mbar_wait_sleep(&emptyB[s], ((bseq / NSB) & 1) ^ 1);
      const int row = (int)(chunk_off(p.gb, j, cb / CPB, kb) / KB + (cb % CPB) * TC +
                            rank * (TC / 2));
      tma_pair_elect(sB + s * BHALF, &mapB, row, &fullB[s], leader_addr(&fullB[s]),
                     leader ? 2 * BHALF : 0);
      ++bseq;
    };
    const int full_waves = tiles / npairs;  // waves in which every pair has a tile
    uint32_t sweep = 0;
    for (int item = CASC_I8_WAITS_ON ? pair : items; item < items; item += npairs) {
      const int tile = item / ks;
      int64_t rp, cb;
      if (TRI)
        tri_tile_of(tile, p.tri, RP, RB, rp, cb);
      else
        tile_of(tile, RP, RB, rp, cb);
      const int64_t rb = 2 * rp + rank;
      const bool synced = p.sync && (tile / npairs) < full_waves;
      for (int q = 0; q < P; ++q) {
        int64_t kb0, kb1;
        kb_range(item, q, kb0, kb1);
        for (int go = 0; go < nmg; ++go) {
          int s, nb, g0_, g1_;
          mgroup(nmg - 1 - go, r0, ngroups, s, nb, g0_, g1_);  // the MMA issuer's order
          const int top = s + nb - 1;
          for (int64_t kb = kb0; kb < kb1; ++kb) {
            if (synced && (kb - kb0) % CASC_I8_SYNC_KB == 0) {
              // Soft wave synchronisation: the producers of all CTAs start each
              // (panel, group) sweep of a full tile wave, and every
              // CASC_I8_SYNC_KB k blocks of it, together, so the tiles in flight
              // stream the same slice chunks at the same time and hit them in L2
              // (bounded wait: never a hang, at worst an unsynchronised stretch).
              ++sweep;
              if (lane == 0) {
                atomicAdd(p.sync, 1u);
                const unsigned int target = sweep * gridDim.x;
                unsigned int v;
                for (int spin = 0; spin < 20000; ++spin) {
                  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.sync) : "memory");
                  if (v >= target) break;
                  __nanosleep(64);
                }
              }
              __syncwarp();
            }
            // A-stationary chain (mma_chain): B_top .. B_s, A_0, B_(s-1), A_1, ...
            for (int j = top; j >= s; --j) loadB(j, cb, kb);
            loadA(0, rb, kb);
            for (int i = 1; i <= top; ++i) {
              if (s - i >= 0) loadB(s - i, cb, kb);
              loadA(i, rb, kb);
            }
          }
        }
      }
    }
  } else if (warp == MMA_WARP) {
    if (leader) {
      // ============================ MMA issuer (leader CTA) ============================
      // All 32 lanes run the loop (warp-uniform control flow, so the scalar state
      // and the descriptors live in the uniform datapath); elect.sync inside the
      // issue blocks picks the one lane that issues each tcgen05 operation.
      uint32_t aseq = 0, bseq = 0, gcount = 0;
      const uint32_t a_base_addr = smem_u32(sA), b_base_addr = smem_u32(sB);
#ifdef CASC_I8_PROF
      const long long tstart = clock64();
      if (lane == 0)
        for (int x = 0; x < 64; ++x) g_i8prof[blockIdx.x][x] = 0;
#endif
      for (int item = pair; item < items; item += npairs) {
        for (int q = 0; q < P; ++q) {
          int64_t kb0_, kb1_;
          kb_range(item, q, kb0_, kb1_);
          const int kb0 = (int)kb0_, kb1 = (int)kb1_;
          // groups in reverse order (bins y-4 .. y-1 first): the short group
          // 0 .. r-1 (most significant, fewest products) ends the panel, so the
          // epilogue's once-per-panel phase 2 overlaps the longest group's MMAs
          // instead of delaying the drain of the shortest one
          for (int go = 0; go < nmg; ++go, ++gcount) {
            int s, nb, g0_, g1_;
            mgroup(nmg - 1 - go, r0, ngroups, s, nb, g0_, g1_);
#ifndef CASC_I8_NOWAIT
            I8_PROF_WAIT(s, mbar_wait_cluster(tempty, (gcount & 1) ^ 1));
#endif
            tc_fence_after();
            for (int kb = kb0; kb < kb1; ++kb)
              mma_kblock(s, nb, kb == kb0, aseq, bseq, tmem, a_base_addr, b_base_addr, fullA,
                         emptyA, fullB, emptyB);
            mma_commit1(tfull);
          }
        }
      }
#ifdef CASC_I8_PROF
      if (lane == 0 && (blockIdx.x % 16) == 0) {
        const unsigned long long* g = g_i8prof[blockIdx.x];
        printf("i8prof cta %d loads %llu round %llu phase2 %llu x %llu | total %lld | tempty %llu %llu %llu %llu | fullB %llu %llu %llu %llu"
               " | fullA %llu %llu %llu %llu\n", blockIdx.x, g[50], g[51], g[48], g[49], clock64() - tstart, g[0], g[2],
               g[6], g[10], g[16], g[18], g[22], g[26], g[32], g[34], g[38], g[42]);
      }
#endif
    }
  } else {
    // ============================ epilogue (both CTAs) ============================
    const int ew = warp;  // 0..7
    const int quarter = warp & 3, half = ew >> 2;
    const int lr = quarter * 32 + lane;       // tile row = TMEM lane
    const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t tempty_leader = leader_addr(tempty);
    // per-CTA workspace: C accumulator (hi, lo) of the tile, then the exact
    // group values V of the panel's groups [NGMAX][128 x 128]
    double* Ch = p.ws + (int64_t)blockIdx.x * WS_PER_CTA;
    double* Cl = Ch + TR * TC;
    long long* Vw = reinterpret_cast<long long*>(Cl + TR * TC);
    constexpr int CW = TC / 2;  // columns of the tile per epilogue thread
    uint32_t gcount = 0;
    for (int item = pair; item < items; item += npairs) {
      const int tile = item / ks;
      int64_t rp, cb;
      if (TRI)
        tri_tile_of(tile, p.tri, RP, RB, rp, cb);
      else
        tile_of(tile, RP, RB, rp, cb);
      const int64_t gi = (2 * rp + rank) * TR + lr;
      uint64_t fl = 0;  // detector bits of this thread's CW columns
      for (int q = 0; q < P; ++q) {
        const int64_t kp = min((int64_t)KC8, p.k - (int64_t)q * KC8);
        const int ei = *reinterpret_cast<const int32_t*>(p.pa + exp_at(p.ga, gi, q));
        // column exponents of this (tile, panel) -> shared memory
        epi_bar_sync();
        if (ew < TC / 32)
          sF[ew * 32 + lane] =
              *reinterpret_cast<const int32_t*>(p.pb + exp_at(p.gb, cb * TC + ew * 32 + lane, q));
        epi_bar_sync();
        for (int go = 0; go < nmg; ++go, ++gcount) {
          int S_, NB_, g0, g1;
          mgroup(nmg - 1 - go, r0, ngroups, S_, NB_, g0, g1);  // the MMA issuer's order
          const bool lastg = go + 1 == nmg;
          mbar_wait_sleep(tfull, gcount & 1);
          tc_fence_after();
          // Phase 1: drain this warp's part of TMEM into the exact group values
          // V = sum_u bin_(s+u) 2^(8(nb-1-u)) (int64, |V| < 2^56; R25) of each
          // value group of this MMA group, then release TMEM so that the MMAs of
          // the next group start at once.
          for (int grp = g0; grp < g1; ++grp) {
            int s, nb;
            vgroup(grp, r0, s, nb);
            const uint32_t tb = trow + (uint32_t)((s - S_) * TC);
#pragma unroll 2
            for (int cc = 0; cc < CW / 8; ++cc) {
              const int c0 = half * CW + cc * 8;
              uint32_t r0[8], r1[8], r2[8], r3[8];
              tmem_ld8(tb + 0 * TC + c0, r0);
              if (nb > 1) tmem_ld8(tb + 1 * TC + c0, r1);
              if (nb > 2) tmem_ld8(tb + 2 * TC + c0, r2);
              if (nb > 3) tmem_ld8(tb + 3 * TC + c0, r3);
              tmem_wait_ld();
              if (DBG && q == p.dbg_panel) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const int64_t gj = cb * TC + c0 + i;
                  if (gi < p.m && gj < p.n) {
                    const int64_t mn = p.m * p.n, o = gi * p.n + gj;
                    p.dbg[(int64_t)(s + 0) * mn + o] = (int32_t)r0[i];
                    if (nb > 1) p.dbg[(int64_t)(s + 1) * mn + o] = (int32_t)r1[i];
                    if (nb > 2) p.dbg[(int64_t)(s + 2) * mn + o] = (int32_t)r2[i];
                    if (nb > 3) p.dbg[(int64_t)(s + 3) * mn + o] = (int32_t)r3[i];
                  }
                }
              }
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                long long v = (int32_t)r0[i];
                if (nb > 1) v = v * 256 + (int32_t)r1[i];
                if (nb > 2) v = v * 256 + (int32_t)r2[i];
                if (nb > 3) v = v * 256 + (int32_t)r3[i];
                Vw[(int64_t)grp * TR * TC + (c0 + i) * TR + lr] = v;
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_leader);
          if (DBG) continue;
#ifdef CASC_I8_NO_EPI
          continue;
#endif
          if (!lastg) continue;
#ifdef CASC_I8_PROF
          const long long tp2 = clock64();
#endif
          // Phase 2, once per panel after its last group (overlaps the MMAs of
          // the next panel / tile): the FP64x2 panel sum T over the groups' exact
          // values, most significant first (R25), the detector (R26) and C.
#pragma unroll 1
          for (int cc = 0; cc < CW / EPI_SUB; ++cc) {
            const int c0 = half * CW + cc * EPI_SUB;
            double th[EPI_SUB], tl[EPI_SUB], xch[EPI_SUB], xcl[EPI_SUB];
            if (q > 0) {
#pragma unroll
              for (int i = 0; i < EPI_SUB; ++i) {
                xch[i] = ld_na(&Ch[(c0 + i) * TR + lr]);
                xcl[i] = ld_na(&Cl[(c0 + i) * TR + lr]);
              }
            }
            // all of this block's group values in flight at once (memory-level
            // parallelism: the loads are latency-bound under the operand traffic)
            long long xv[NGMAX][EPI_SUB];
#pragma unroll
            for (int g2 = 0; g2 < NGMAX; ++g2)
              if (g2 < ngroups) {
#pragma unroll
                for (int i = 0; i < EPI_SUB; ++i)
                  xv[g2][i] = ld_na(&Vw[(int64_t)g2 * TR * TC + (c0 + i) * TR + lr]);
              }
#ifdef CASC_I8_PROF
            long long tpa = clock64();
            if (xv[0][0] == 0x7fffffffffffffffll) tpa = 0;  // forces the loads to land
            if (lane == 0 && ew == 1) g_i8prof[blockIdx.x][50] += clock64() - tpa;
            tpa = clock64();
#endif
#pragma unroll
            for (int i = 0; i < EPI_SUB; ++i) {
              // R25 (rev. 2): S = sum_g V_g 2^(32 (ngroups-1-g)) exactly (the
              // groups are aligned at the least significant bin), then
              // T = (RN(S 2^w0), RN(S 2^w0 - T.hi)), w0 = e + f - 12 - 8(y-1)
              U192 S{0ull, 0ull, 0ull};
#pragma unroll
              for (int g2 = 0; g2 < NGMAX; ++g2)
                if (g2 < ngroups) S = u192_add(S, u192_from_shifted(xv[g2][i], ngroups - 1 - g2));
              if (SPLITK) {  // the exact partial S of this k-block part
                unsigned long long* sw =
                    p.split_ws + ((int64_t)(item * 2 + (int)rank) * 3) * TR * TC + (c0 + i) * TR + lr;
                sw[0] = S.l0;
                sw[TR * TC] = S.l1;
                sw[2 * TR * TC] = S.l2;
                continue;
              }
              rn_pair(S, ei + sF[c0 + i] - 12 - 8 * (y - 1), th[i], tl[i]);
            }
#ifdef CASC_I8_PROF
            if (th[0] == 12345.0) tpa = 0;
            if (lane == 0 && ew == 1) g_i8prof[blockIdx.x][51] += clock64() - tpa;
#endif
            if (SPLITK) continue;  // rounding, detector and C in i8_split_reduce_kernel
#pragma unroll
            for (int i = 0; i < EPI_SUB; ++i) {
              const int lc = c0 + i;
              const int fj = sF[lc];
              const int widx = lc * TR + lr;
              // R26 detector, then C (+)= T
              if (fabs(th[i]) <= mulp2((double)kp, ei + fj - 50)) fl |= 1ull << (lc - half * CW);
              double ch = th[i], cl = tl[i];
              if (q > 0) dd_add(xch[i], xcl[i], th[i], tl[i], ch, cl);
              if (q + 1 < P) {
                Ch[widx] = ch;
                Cl[widx] = cl;
              } else {
                const int64_t gj = cb * TC + lc;
                if (gi < p.m && gj < p.n && (!TRI || (p.tri == 1 ? gi >= gj : gi <= gj))) {
                  double* oh = p.C_hi + gi * p.ldc + gj;
                  double* ol = p.C_lo + gi * p.ldc + gj;
                  // NEXT-4 (reading R21): C := alpha (x) P (+) beta (x) C
                  if (p.ab)
                    apply_alpha_beta(ch, cl, p.ah, p.al, p.bh, p.bl, p.ab == 2 ? *oh : 0.0,
                                     p.ab == 2 ? *ol : 0.0, p.ab == 2);
                  *oh = ch;
                  *ol = cl;
                  if (p.flags) p.flags[gi * p.ldf + gj] = (uint8_t)((fl >> (lc - half * CW)) & 1);
                }
              }
            }
          }
#ifdef CASC_I8_PROF
          if (lane == 0 && ew == 1) g_i8prof[blockIdx.x][48] += clock64() - tp2;
          if (lane == 0 && ew == 1) g_i8prof[blockIdx.x][49] += 1;
#endif
        }
      }
    }
#ifdef CASC_I8_PROF
    if (lane == 0 && ew == 1 && (blockIdx.x % 16) == 0)
      printf("i8epi cta %d loads %llu round %llu phase2 %llu x %llu\n", blockIdx.x,
             g_i8prof[blockIdx.x][50], g_i8prof[blockIdx.x][51], g_i8prof[blockIdx.x][48],
             g_i8prof[blockIdx.x][49]);
#endif
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ------------------------------------------------------------------ launchers
cudaError_t pack(const double* hi, const double* lo, int64_t ld, int64_t rows, int64_t k, int y,
                 bool cols, void* packed, cudaStream_t st) {
  const Pack g = pack_of(rows, k, y);
  uint8_t* pk = static_cast<uint8_t*>(packed);
  i8_zero_max_kernel<<<256, 256, 0, st>>>(g, pk);
  // k per thread / warp of the max kernels: large enough to keep the atomics
  // few, small enough that small problems still fill the machine
  const int64_t elems = rows * k;
  if (cols) {
    const int kc = elems >= ((int64_t)1 << 26) ? 64 : 16;
    i8_colmax_kernel<<<dim3((unsigned)((rows + 255) / 256), (unsigned)((k + kc - 1) / kc)), 256,
                       0, st>>>(hi, ld, rows, k, g, pk, kc);
    i8_digits_kernel<true><<<dim3((unsigned)g.R, (unsigned)g.KBn, 4), 256, 0, st>>>(
        hi, lo, ld, rows, k, g, pk);
  } else {
    const int kc = elems >= ((int64_t)1 << 26) ? 1024 : 256;
    i8_rowmax_kernel<<<dim3((unsigned)((rows + 7) / 8), (unsigned)((k + kc - 1) / kc)), 256, 0,
                       st>>>(hi, ld, rows, k, g, pk, kc);
    i8_digits_kernel<false><<<dim3((unsigned)(g.R * 4), (unsigned)g.KBn), 256, 0, st>>>(
        hi, lo, ld, rows, k, g, pk);
  }
  return cudaGetLastError();
}

cudaError_t unpack(const void* packed, int64_t rows, int64_t k, int y, int8_t* D, int32_t* E,
                   cudaStream_t st) {
  const Pack g = pack_of(rows, k, y);
  i8_unpack_kernel<<<1024, 256, 0, st>>>(static_cast<const uint8_t*>(packed), g, rows, k, D, E);
  return cudaGetLastError();
}

int grid_for(int64_t m, int64_t n, int sms) {  // CTAs: 2 per pair, one pair per 2 SMs
  const int64_t tiles = ((m + 2 * TR - 1) / (2 * TR)) * ((n + TC - 1) / TC);
  const int64_t pairs = tiles < sms / 2 ? tiles : sms / 2;
  return (int)(2 * pairs);
}
// CTAs the GEMM scratch is sized for: small problems may run in split mode on
// every CTA pair (split_parts)
int ws_grid(int64_t m, int64_t n, int sms) {
  const int64_t tiles = ((m + 2 * TR - 1) / (2 * TR)) * ((n + TC - 1) / TC);
  return tiles < 2 * (int64_t)(sms / 2) ? 2 * (sms / 2) : grid_for(m, n, sms);
}
// per-CTA T / C scratch, then the wave-sync counter
size_t cta_ws_bytes(int grid) { return (size_t)grid * WS_PER_CTA * sizeof(double) + 256; }

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 2-D view of a packed operand's slices as 128-byte rows; `box_rows` rows per copy.
// The chunks are pre-swizzled, so the map copies bytes verbatim (SWIZZLE_NONE).
cudaError_t slice_map(CUtensorMap* map, const void* packed, const Pack& g, uint32_t box_rows) {
  static EncodeTiledFn enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc),
                                cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !enc)
      return cudaErrorNotSupported;
  }
  const uint64_t rows = (uint64_t)(packed_bytes(g) / KB);
  if (rows >= (1ull << 31)) return cudaErrorInvalidValue;  // int32 TMA coordinates
  cuuint64_t dims[2] = {(cuuint64_t)KB, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)KB};
  cuuint32_t box[2] = {(cuuint32_t)KB, box_rows};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(packed), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Split mode: C from the parts' exact partial products (P == 1): S = sum of the
// parts (192-bit, exact), T = (RN(S 2^w0), RN(S 2^w0 - T.hi)) (R25 rev. 2), the
// R26 detector, C = T, the R21 update -- the unsplit epilogue's steps on the
// same exact S, hence bitwise the same C and flags.
__global__ void __launch_bounds__(256) i8_split_reduce_kernel(const GemmArgs p) {
  const int64_t RP = p.ga.R / 2, RB = p.gb.R * CPB;
  const int y = p.ga.y;
  const int64_t mn = p.m * p.n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < mn;
       idx += (int64_t)gridDim.x * blockDim.x) {
    // consecutive threads: consecutive rows of one column (the workspace is
    // column-major per tile)
    const int64_t j = idx / p.m, i = idx - j * p.m;
    const int64_t rp = i / (2 * TR), rank = (i / TR) & 1, lr = i % TR;
    const int64_t cb = j / TC, col = j % TC;
    const int64_t tile = tile_index(rp, cb, RP, RB);
    U192 S{0ull, 0ull, 0ull};
    for (int part = 0; part < p.ks; ++part) {
      const unsigned long long* sw =
          p.split_ws + ((tile * p.ks + part) * 2 + rank) * 3 * TR * TC + col * TR + lr;
      S = u192_add(S, U192{sw[0], sw[TR * TC], sw[2 * TR * TC]});
    }
    const int ei = *reinterpret_cast<const int32_t*>(p.pa + exp_at(p.ga, i, 0));
    const int fj = *reinterpret_cast<const int32_t*>(p.pb + exp_at(p.gb, j, 0));
    double ch, cl;
    rn_pair(S, ei + fj - 12 - 8 * (y - 1), ch, cl);
    const uint8_t flag = fabs(ch) <= mulp2((double)p.k, ei + fj - 50) ? 1 : 0;
    double* oh = p.C_hi + i * p.ldc + j;
    double* ol = p.C_lo + i * p.ldc + j;
    if (p.ab)
      apply_alpha_beta(ch, cl, p.ah, p.al, p.bh, p.bl, p.ab == 2 ? *oh : 0.0,
                       p.ab == 2 ? *ol : 0.0, p.ab == 2);
    *oh = ch;
    *ol = cl;
    if (p.flags) p.flags[i * p.ldf + j] = flag;
  }
}

// Split plan: k-block parts per tile (1 = off) for single-panel problems whose
// tiles fill the CTA pairs' last wave badly; the smallest part count within 2%
// of the best wave efficiency.
int split_parts(int64_t m, int64_t n, int64_t k, int sms) {
  const char* env = getenv("CASC_I8_SPLIT");  // "0": never (tests compare both)
  if (env && env[0] == '0') return 1;
  if (k > KC8) return 1;
  const int64_t tiles = ((m + 2 * TR - 1) / (2 * TR)) * ((n + TC - 1) / TC);
  const int64_t np = sms / 2, kbn = (k + KB - 1) / KB;
  if (tiles >= 2 * np) return 1;
  auto eff = [&](int64_t ks) {
    const int64_t it = tiles * ks;
    return (double)it / (double)(((it + np - 1) / np) * np);
  };
  double best = eff(1);
  for (int64_t ks = 2; ks <= 16 && ks <= kbn && tiles * ks <= 4 * np; ++ks) best = max(best, eff(ks));
  for (int64_t ks = 1; ks <= 16 && ks <= kbn && tiles * ks <= 4 * np; ++ks)
    if (eff(ks) >= best - 0.02) return (int)ks;
  return 1;
}

cudaError_t gemm(const void* pa, const void* pb, int64_t m, int64_t n, int64_t k, int y,
                 double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags, double* ws, int grid,
                 int32_t* dbg, int64_t dbg_panel, cudaStream_t st, int ab = 0, double ah = 1.0,
                 double al = 0.0, double bh = 0.0, double bl = 0.0, int tri = 0,
                 int64_t ldf = -1) {
  GemmArgs a{};
  a.ldf = ldf < 0 ? n : ldf;
  a.tri = tri;
  a.ab = ab;
  a.ah = ah;
  a.al = al;
  a.bh = bh;
  a.bl = bl;
  a.pa = static_cast<const uint8_t*>(pa);
  a.pb = static_cast<const uint8_t*>(pb);
  a.ga = pack_of(m, k, y);
  a.gb = pack_of(n, k, y);
  a.m = m;
  a.n = n;
  a.k = k;
  a.C_hi = C_hi;
  a.C_lo = C_lo;
  a.ldc = ldc;
  a.flags = flags;
  a.ws = ws;
  a.dbg = dbg;
  a.dbg_panel = dbg_panel;
  // `grid`: the CTAs `ws` holds (ws_grid); the launch takes what the tiles need
  int sms = 0, dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return cudaErrorInvalidDevice;
  const int g0 = min(grid, grid_for(m, n, sms));
  const char* env = getenv("CASC_I8_WAVE_SYNC");  // "0": off (timing studies)
  if (!(env && env[0] == '0')) {
    a.sync = reinterpret_cast<unsigned int*>(reinterpret_cast<uint8_t*>(ws) +
                                             (size_t)grid * WS_PER_CTA * sizeof(double));
    cudaError_t e0 = cudaMemsetAsync(a.sync, 0, sizeof(unsigned int), st);
    if (e0 != cudaSuccess) return e0;
  }
  CUtensorMap mA, mB;
  cudaError_t e = slice_map(&mA, pa, a.ga, TR);
  if (e == cudaSuccess) e = slice_map(&mB, pb, a.gb, TC / 2);
  if (e != cudaSuccess) return e;
  if (dbg) {
    cudaFuncSetAttribute(i8_gemm_kernel<true, false, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    i8_gemm_kernel<true, false, false><<<g0, THREADS, SMEM, st>>>(a, mA, mB);
    return cudaGetLastError();
  }
  const int ks = tri ? 1 : split_parts(m, n, k, sms);
  if (ks > 1) {
    const int64_t tiles = ((m + 2 * TR - 1) / (2 * TR)) * ((n + TC - 1) / TC);
    const int64_t items = tiles * ks;
    const int g = (int)(2 * min(items, (int64_t)(sms / 2)));
    if (g > grid) return cudaErrorInvalidValue;  // ws sized for `grid` CTAs
    a.ks = ks;
    a.sync = nullptr;  // no wave synchronisation for a few waves
    if (cudaMallocAsync(reinterpret_cast<void**>(&a.split_ws),
                        (size_t)items * 2 * 3 * TR * TC * sizeof(unsigned long long),
                        st) != cudaSuccess)
      return cudaErrorMemoryAllocation;
    cudaFuncSetAttribute(i8_gemm_kernel<false, true, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    i8_gemm_kernel<false, true, false><<<g, THREADS, SMEM, st>>>(a, mA, mB);
    cudaError_t e2 = cudaGetLastError();
    if (e2 == cudaSuccess) {
      int64_t blocks = (m * n + 255) / 256;
      if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
      i8_split_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(a);
      e2 = cudaGetLastError();
    }
    cudaFreeAsync(a.split_ws, st);
    return e2;
  }
  if (tri) {
    cudaFuncSetAttribute(i8_gemm_kernel<false, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    i8_gemm_kernel<false, false, true><<<g0, THREADS, SMEM, st>>>(a, mA, mB);
    return cudaGetLastError();
  }
  cudaFuncSetAttribute(i8_gemm_kernel<false, false, false>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
  i8_gemm_kernel<false, false, false><<<g0, THREADS, SMEM, st>>>(a, mA, mB);
  return cudaGetLastError();
}

}  // namespace i8
}  // namespace casc

// ====================================================================== C ABI
namespace casc {
cudaError_t launch_scale_c_uplo(int64_t m, int64_t n, double bh, double bl, int use_beta,
                                double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
                                int num_sms, int uplo, cudaStream_t st);
cudaError_t launch_trsm_diag_inv(int uplo, int diag, int64_t m, const double* A_hi,
                                 const double* A_lo, int64_t lda, double* I_hi, double* I_lo,
                                 cudaStream_t st);
cudaError_t launch_scale_c(int64_t m, int64_t n, double bh, double bl, int use_beta, double* C_hi,
                           double* C_lo, int64_t ldc, uint8_t* flags, int num_sms,
                           cudaStream_t st);
namespace host {
int device_check(int* sms);
int validate_gemm(int64_t m, int64_t n, int64_t k, const double* A_hi, const double* A_lo,
                  int64_t lda, const double* B_hi, const double* B_lo, int64_t ldb, double* C_hi,
                  double* C_lo, int64_t ldc, uint8_t* flags);
int zero_c(int64_t m, int64_t n, double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
           cudaStream_t st);
int check_mat(const void* p, int64_t rows, int64_t cols, int64_t ld);
int current_sms();
void set_launches(int n);
bool trsm_overlap(int64_t m, int64_t n, const double* A_hi, const double* A_lo, int64_t lda,
                  const double* B_hi, const double* B_lo, int64_t ldb);
}  // namespace host
}  // namespace casc

namespace {
using namespace casc;
inline cudaStream_t S8(casc_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }
inline int st8(cudaError_t e) { return e == cudaSuccess ? CASC_OK : CASC_ERR_CUDA; }
inline size_t al256h(size_t b) { return (b + 255) / 256 * 256; }
}  // namespace

extern "C" {

size_t casc_i8_packed_bytes(int64_t rows, int64_t k, int y) {
  if (rows <= 0 || k <= 0 || y < i8::YMIN || y > i8::YMAX) return 0;
  return (size_t)i8::packed_bytes(i8::pack_of(rows, k, y));
}

size_t casc_i8_packed_block_bytes(int64_t k, int y) {
  if (k <= 0 || y < i8::YMIN || y > i8::YMAX) return 0;
  return (size_t)i8::blk_bytes(i8::pack_of(1, k, y));
}

size_t casc_i8_gemm_ws_bytes(int64_t m, int64_t n) {
  if (m <= 0 || n <= 0) return 0;
  return i8::cta_ws_bytes(i8::ws_grid(m, n, host::current_sms()));
}

size_t casc_i8_workspace_bytes(int64_t m, int64_t n, int64_t k, int y) {
  if (m <= 0 || n <= 0 || k <= 0 || y < i8::YMIN || y > i8::YMAX) return 0;
  return al256h(casc_i8_packed_bytes(m, k, y)) + al256h(casc_i8_packed_bytes(n, k, y)) +
         casc_i8_gemm_ws_bytes(m, n);
}

int casc_i8_pack(int64_t rows, int64_t k, const double* hi, const double* lo, int64_t ld,
                 int is_b, int y, void* packed, casc_stream_t stream) {
  host::set_launches(0);
  int r;
  if (rows < 0 || k < 0 || y < i8::YMIN || y > i8::YMAX) return CASC_ERR_INVALID;
  if (is_b) {
    if ((r = host::check_mat(hi, k, rows, ld)) || (r = host::check_mat(lo, k, rows, ld))) return r;
  } else {
    if ((r = host::check_mat(hi, rows, k, ld)) || (r = host::check_mat(lo, rows, k, ld))) return r;
  }
  if (rows == 0 || k == 0) return CASC_OK;
  if (!packed) return CASC_ERR_INVALID;
  if ((r = host::device_check(nullptr))) return r;
  const cudaError_t e = i8::pack(hi, lo, ld, rows, k, y, is_b != 0, packed, S8(stream));
  if (e == cudaSuccess) host::set_launches(3);
  return st8(e);
}

int casc_i8_gemm_packed_ld(int64_t m, int64_t n, int64_t k, int y, const void* packed_a,
                           const void* packed_b, double* C_hi, double* C_lo, int64_t ldc,
                           uint8_t* flags, int64_t ldf, void* ws, size_t ws_bytes,
                           casc_stream_t stream) {
  host::set_launches(0);
  int r;
  if (m < 0 || n < 0 || k < 0 || y < i8::YMIN || y > i8::YMAX) return CASC_ERR_INVALID;
  if ((r = host::check_mat(C_hi, m, n, ldc)) || (r = host::check_mat(C_lo, m, n, ldc))) return r;
  if (flags && ldf < (n > 1 ? n : 1)) return CASC_ERR_INVALID;
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = host::device_check(&sms))) return r;
  if (k == 0) {
    if (flags && ldf != n) {  // zero C, then the flags rows one by one (ld != n)
      if ((r = host::zero_c(m, n, C_hi, C_lo, ldc, nullptr, S8(stream)))) return r;
      return st8(cudaMemset2DAsync(flags, (size_t)ldf, 0, (size_t)n, (size_t)m, S8(stream)));
    }
    return host::zero_c(m, n, C_hi, C_lo, ldc, flags, S8(stream));
  }
  if (!packed_a || !packed_b || !ws || ws_bytes < casc_i8_gemm_ws_bytes(m, n))
    return CASC_ERR_INVALID;
  const cudaError_t e = i8::gemm(packed_a, packed_b, m, n, k, y, C_hi, C_lo, ldc, flags,
                                 static_cast<double*>(ws), i8::ws_grid(m, n, sms), nullptr, 0,
                                 S8(stream), 0, 1.0, 0.0, 0.0, 0.0, 0, ldf);
  if (e == cudaSuccess) host::set_launches(1);
  return st8(e);
}

int casc_i8_gemm_packed(int64_t m, int64_t n, int64_t k, int y, const void* packed_a,
                        const void* packed_b, double* C_hi, double* C_lo, int64_t ldc,
                        uint8_t* flags, void* ws, size_t ws_bytes, casc_stream_t stream) {
  return casc_i8_gemm_packed_ld(m, n, k, y, packed_a, packed_b, C_hi, C_lo, ldc, flags, n, ws,
                                ws_bytes, stream);
}

int casc_i8_gemm_fp64x2_ws(int64_t m, int64_t n, int64_t k, const double* A_hi,
                           const double* A_lo, int64_t lda, const double* B_hi,
                           const double* B_lo, int64_t ldb, double* C_hi, double* C_lo,
                           int64_t ldc, uint8_t* flags, int y, void* workspace,
                           size_t workspace_bytes, casc_stream_t stream) {
  host::set_launches(0);
  int r = host::validate_gemm(m, n, k, A_hi, A_lo, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, flags);
  if (r) return r;
  if (y < i8::YMIN || y > i8::YMAX) return CASC_ERR_INVALID;
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = host::device_check(&sms))) return r;
  const cudaStream_t st = S8(stream);
  if (k == 0) return host::zero_c(m, n, C_hi, C_lo, ldc, flags, st);
  const size_t need = casc_i8_workspace_bytes(m, n, k, y);
  if (!workspace || workspace_bytes < need) return CASC_ERR_INVALID;
  uint8_t* pa = static_cast<uint8_t*>(workspace);
  uint8_t* pb = pa + al256h(casc_i8_packed_bytes(m, k, y));
  double* ws = reinterpret_cast<double*>(pb + al256h(casc_i8_packed_bytes(n, k, y)));
  cudaError_t e = i8::pack(A_hi, A_lo, lda, m, k, y, false, pa, st);
  if (e == cudaSuccess) e = i8::pack(B_hi, B_lo, ldb, n, k, y, true, pb, st);
  if (e == cudaSuccess)
    e = i8::gemm(pa, pb, m, n, k, y, C_hi, C_lo, ldc, flags, ws, i8::ws_grid(m, n, sms), nullptr,
                 0, st);
  if (e == cudaSuccess) host::set_launches(7);
  return st8(e);
}

// Host-resident operands (casc.h), the row-slab pipeline of casc_host.cuh; slab
// starts are multiples of 256 rows (a CTA pair's tile).
int casc_i8_gemm_fp64x2_host(int64_t m, int64_t n, int64_t k, const double* A_hi,
                             const double* A_lo, int64_t lda, const double* B_hi,
                             const double* B_lo, int64_t ldb, double* C_hi, double* C_lo,
                             int64_t ldc, uint8_t* flags, int y, int64_t slab_rows,
                             int64_t slab_cols, casc_stream_t stream) {
  host::set_launches(0);
  int r = host::validate_gemm(m, n, k, A_hi, A_lo, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, flags);
  if (r) return r;
  if (y < i8::YMIN || y > i8::YMAX || slab_rows < 0 || slab_cols < 0) return CASC_ERR_INVALID;
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = host::device_check(&sms))) return r;
  const cudaStream_t st = S8(stream);
  if (k == 0) return casc::hostpipe::zero_host_c(m, n, C_hi, C_lo, ldc, flags, st);
  const int64_t blk = 2 * i8::TR;  // a CTA pair's rows; B slabs: two packed blocks
  auto fit = [&](int64_t v, int64_t lim) {
    v = (v + blk - 1) / blk * blk;
    const int64_t l = (lim + blk - 1) / blk * blk;
    return v < l ? v : l;
  };
  const int64_t sr = fit(slab_rows ? slab_rows : casc::hostpipe::default_slab(m), m);
  const int64_t sc = fit(slab_cols ? slab_cols : casc::hostpipe::default_slab(n), n);
  const int gmax = 2 * (sms / 2);  // every block's ws_grid fits
  double* gws = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&gws), i8::cta_ws_bytes(gmax), st) != cudaSuccess)
    return CASC_ERR_CUDA;
  int launches = 0;
  auto pack_b = [&](const double* bh, const double* bl, int64_t cols, void* pb) {
    const cudaError_t e = i8::pack(bh, bl, cols, cols, k, y, true, pb, st);
    launches += e == cudaSuccess ? 3 : 0;
    return st8(e);
  };
  auto pack_a = [&](const double* ah, const double* al, int64_t rows, void* pa) {
    const cudaError_t e = i8::pack(ah, al, k, rows, k, y, false, pa, st);
    launches += e == cudaSuccess ? 3 : 0;
    return st8(e);
  };
  auto gemm = [&](int64_t rows, int64_t cols, const void* pa, const void* pb, double* ch,
                  double* cl, uint8_t* fl) {
    const cudaError_t e = i8::gemm(pa, pb, rows, cols, k, y, ch, cl, cols, fl, gws,
                                   gmax, nullptr, 0, st);
    launches += e == cudaSuccess;
    return st8(e);
  };
  r = casc::hostpipe::run(m, n, k, A_hi, A_lo, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, flags, sr,
                          sc, casc_i8_packed_bytes(sc, k, y), casc_i8_packed_bytes(sr, k, y), st,
                          pack_b, pack_a, gemm);
  cudaFreeAsync(gws, st);
  host::set_launches(r == CASC_OK ? launches : 0);
  return r;
}

// TRSM on the INT8 cascade (NEXT-4, reading R27): casc_trsm_fp64x2's blocked solve
// with casc_i8_gemm_fp64x2_ex as the GEMM; bit-exact with orc_i8_casc_trsm.
int casc_i8_trsm_fp64x2(int uplo, int trans, int diag, int64_t m, int64_t n, double alpha_hi,
                        double alpha_lo, const double* A_hi, const double* A_lo, int64_t lda,
                        double* B_hi, double* B_lo, int64_t ldb, int y, casc_stream_t stream) {
  host::set_launches(0);
  if ((uplo != CASC_LOWER && uplo != CASC_UPPER) || (diag != CASC_NONUNIT && diag != CASC_UNIT) ||
      (trans != CASC_OP_N && trans != CASC_OP_T) || y < i8::YMIN || y > i8::YMAX)
    return CASC_ERR_INVALID;
  if (m < 0 || n < 0) return CASC_ERR_INVALID;
  int r;
  if ((r = host::check_mat(A_hi, m, m, lda)) || (r = host::check_mat(A_lo, m, m, lda))) return r;
  if ((r = host::check_mat(B_hi, m, n, ldb)) || (r = host::check_mat(B_lo, m, n, ldb))) return r;
  if (host::trsm_overlap(m, n, A_hi, A_lo, lda, B_hi, B_lo, ldb)) return CASC_ERR_INVALID;
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = host::device_check(&sms))) return r;
  const cudaStream_t st = S8(stream);
  const bool unit_alpha = (alpha_hi == 1.0 && alpha_lo == 0.0);
  const bool zero_alpha = (alpha_hi == 0.0 && alpha_lo == 0.0);
  if (!unit_alpha &&
      casc::launch_scale_c(m, n, alpha_hi, alpha_lo, zero_alpha ? 0 : 1, B_hi, B_lo, ldb, nullptr,
                           sms, st) != cudaSuccess)
    return CASC_ERR_CUDA;
  if (zero_alpha) return CASC_OK;
  const int64_t NB = 256, nblk = (m + NB - 1) / NB;
  const size_t inv_elems = (size_t)nblk * NB * NB, t_elems = (size_t)NB * n;
  double* buf = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&buf), (2 * inv_elems + 2 * t_elems) * 8, st) !=
      cudaSuccess)
    return CASC_ERR_CUDA;
  double* inv_hi = buf;
  double* inv_lo = buf + inv_elems;
  double* t_hi = inv_lo + inv_elems;
  double* t_lo = t_hi + t_elems;
  r = casc::launch_trsm_diag_inv(uplo, diag, m, A_hi, A_lo, lda, inv_hi, inv_lo, st) ==
              cudaSuccess
          ? CASC_OK
          : CASC_ERR_CUDA;
  const bool eff_lower = (uplo == CASC_LOWER) != (trans == CASC_OP_T);
  for (int64_t s = 0; s < nblk && r == CASC_OK; ++s) {
    const int64_t b = eff_lower ? s : nblk - 1 - s;
    const int64_t r0 = b * NB, nb = std::min(NB, m - r0), r1 = r0 + nb;
    r = casc_i8_gemm_fp64x2_ex(trans, CASC_OP_N, nb, n, nb, 1.0, 0.0, inv_hi + b * NB * NB,
                               inv_lo + b * NB * NB, NB, B_hi + r0 * ldb, B_lo + r0 * ldb, ldb,
                               0.0, 0.0, t_hi, t_lo, n, nullptr, y, nullptr, 0, stream);
    if (r) break;
    if (cudaMemcpy2DAsync(B_hi + r0 * ldb, ldb * 8, t_hi, n * 8, n * 8, nb,
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
        cudaMemcpy2DAsync(B_lo + r0 * ldb, ldb * 8, t_lo, n * 8, n * 8, nb,
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
      r = CASC_ERR_CUDA;
      break;
    }
    auto update = [&](int64_t R0, int64_t R1, int64_t C0, int64_t C1) {
      if (r != CASC_OK || R1 <= R0 || C1 <= C0) return;
      const int64_t off = trans ? C0 * lda + R0 : R0 * lda + C0;
      r = casc_i8_gemm_fp64x2_ex(trans, CASC_OP_N, R1 - R0, n, C1 - C0, -1.0, 0.0, A_hi + off,
                                 A_lo + off, lda, B_hi + C0 * ldb, B_lo + C0 * ldb, ldb, 1.0, 0.0,
                                 B_hi + R0 * ldb, B_lo + R0 * ldb, ldb, nullptr, y, nullptr, 0,
                                 stream);
    };
    const int64_t S0 = (b / 4) * 4 * NB, S1 = std::min(S0 + 4 * NB, m);
    if (eff_lower) {
      update(r1, S1, r0, r1);
      if (r1 == S1) update(S1, m, S0, S1);
    } else {
      update(S0, r0, r0, r1);
      if (r0 == S0) update(0, S0, S0, S1);
    }
  }
  cudaFreeAsync(buf, st);
  host::set_launches(0);
  return r;
}

// SYRK on the INT8 cascade (NEXT-4): the triangle's pair tiles only, every stored
// element bitwise the casc_i8_gemm_fp64x2_ex(trans, !trans, A, A) element.
int casc_i8_syrk_fp64x2(int uplo, int trans, int64_t n, int64_t k, double alpha_hi,
                        double alpha_lo, const double* A_hi, const double* A_lo, int64_t lda,
                        double beta_hi, double beta_lo, double* C_hi, double* C_lo, int64_t ldc,
                        uint8_t* flags, int y, casc_stream_t stream) {
  host::set_launches(0);
  if ((uplo != CASC_LOWER && uplo != CASC_UPPER) || (trans != CASC_OP_N && trans != CASC_OP_T))
    return CASC_ERR_INVALID;
  if (n < 0 || k < 0 || y < i8::YMIN || y > i8::YMAX) return CASC_ERR_INVALID;
  const int64_t ar = trans ? k : n, ac = trans ? n : k;
  const bool no_product = (k == 0) || (alpha_hi == 0.0 && alpha_lo == 0.0);
  int r;
  if (!no_product && ((r = host::check_mat(A_hi, ar, ac, lda)) ||
                      (r = host::check_mat(A_lo, ar, ac, lda))))
    return r;
  if ((r = host::check_mat(C_hi, n, n, ldc)) || (r = host::check_mat(C_lo, n, n, ldc))) return r;
  if (n == 0) return CASC_OK;
  int sms = 0;
  if ((r = host::device_check(&sms))) return r;
  const cudaStream_t st = S8(stream);
  const bool use_beta = !(beta_hi == 0.0 && beta_lo == 0.0);
  if (no_product) {
    const cudaError_t e = casc::launch_scale_c_uplo(n, n, beta_hi, beta_lo, use_beta, C_hi, C_lo,
                                                    ldc, flags, sms, uplo == CASC_LOWER ? 0 : 1,
                                                    st);
    if (e == cudaSuccess) host::set_launches(1);
    return st8(e);
  }
  const size_t need = casc_i8_workspace_bytes(n, n, k, y);
  void* ws = nullptr;
  if (cudaMallocAsync(&ws, need, st) != cudaSuccess) return CASC_ERR_CUDA;
  uint8_t* pa = static_cast<uint8_t*>(ws);
  uint8_t* pb = pa + al256h(casc_i8_packed_bytes(n, k, y));
  double* gws = reinterpret_cast<double*>(pb + al256h(casc_i8_packed_bytes(n, k, y)));
  // op(A) as the A operand; op(A)^T as the B operand: its columns are op(A)'s
  // rows, and A and B operands share the packed format, so one pack serves both
  cudaError_t e = i8::pack(A_hi, A_lo, lda, n, k, y, trans == CASC_OP_T, pa, st);
  (void)pb;
  const bool unit_alpha = (alpha_hi == 1.0 && alpha_lo == 0.0);
  const int ab = use_beta ? 2 : (unit_alpha ? 0 : 1);
  if (e == cudaSuccess)
    e = i8::gemm(pa, pa, n, n, k, y, C_hi, C_lo, ldc, flags, gws, i8::ws_grid(n, n, sms), nullptr,
                 0, st, ab, alpha_hi, alpha_lo, beta_hi, beta_lo, uplo == CASC_LOWER ? 1 : 2);
  cudaFreeAsync(ws, st);
  if (e == cudaSuccess) host::set_launches(4);
  return st8(e);
}

int casc_i8_gemm_fp64x2_ex(int transa, int transb, int64_t m, int64_t n, int64_t k,
                           double alpha_hi, double alpha_lo, const double* A_hi,
                           const double* A_lo, int64_t lda, const double* B_hi,
                           const double* B_lo, int64_t ldb, double beta_hi, double beta_lo,
                           double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags, int y,
                           void* workspace, size_t workspace_bytes, casc_stream_t stream) {
  host::set_launches(0);
  if ((transa != CASC_OP_N && transa != CASC_OP_T) || (transb != CASC_OP_N && transb != CASC_OP_T))
    return CASC_ERR_INVALID;
  if (m < 0 || n < 0 || k < 0 || y < i8::YMIN || y > i8::YMAX) return CASC_ERR_INVALID;
  // stored shapes: op(A) is m x k (A stored k x m if transposed), op(B) is k x n
  const int64_t ar = transa ? k : m, ac = transa ? m : k;
  const int64_t br = transb ? n : k, bc = transb ? k : n;
  const bool no_product = (k == 0) || (alpha_hi == 0.0 && alpha_lo == 0.0);
  int r;
  if (!no_product) {
    if ((r = host::check_mat(A_hi, ar, ac, lda)) || (r = host::check_mat(A_lo, ar, ac, lda)))
      return r;
    if ((r = host::check_mat(B_hi, br, bc, ldb)) || (r = host::check_mat(B_lo, br, bc, ldb)))
      return r;
  }
  if ((r = host::check_mat(C_hi, m, n, ldc)) || (r = host::check_mat(C_lo, m, n, ldc))) return r;
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = host::device_check(&sms))) return r;
  const cudaStream_t st = S8(stream);
  const bool use_beta = !(beta_hi == 0.0 && beta_lo == 0.0);
  if (no_product) {  // C := beta C (BLAS: A and B are not referenced)
    const cudaError_t e =
        casc::launch_scale_c(m, n, beta_hi, beta_lo, use_beta, C_hi, C_lo, ldc, flags, sms, st);
    if (e == cudaSuccess) host::set_launches(1);
    return st8(e);
  }
  const size_t need = casc_i8_workspace_bytes(m, n, k, y);
  void* ws = workspace;
  bool owned = false;
  if (!ws) {
    if (cudaMallocAsync(&ws, need, st) != cudaSuccess) return CASC_ERR_CUDA;
    owned = true;
  } else if (workspace_bytes < need) {
    return CASC_ERR_INVALID;
  }
  uint8_t* pa = static_cast<uint8_t*>(ws);
  uint8_t* pb = pa + al256h(casc_i8_packed_bytes(m, k, y));
  double* gws = reinterpret_cast<double*>(pb + al256h(casc_i8_packed_bytes(n, k, y)));
  // rows of op(A) are columns of a transposed A; columns of op(B) are rows of a
  // transposed B: the split kernels read either orientation directly
  cudaError_t e = i8::pack(A_hi, A_lo, lda, m, k, y, transa == CASC_OP_T, pa, st);
  if (e == cudaSuccess) e = i8::pack(B_hi, B_lo, ldb, n, k, y, transb != CASC_OP_T, pb, st);
  const bool unit_alpha = (alpha_hi == 1.0 && alpha_lo == 0.0);
  const int ab = use_beta ? 2 : (unit_alpha ? 0 : 1);
  if (e == cudaSuccess)
    e = i8::gemm(pa, pb, m, n, k, y, C_hi, C_lo, ldc, flags, gws, i8::ws_grid(m, n, sms),
                 nullptr, 0, st, ab, alpha_hi, alpha_lo, beta_hi, beta_lo);
  if (owned) cudaFreeAsync(ws, st);
  if (e == cudaSuccess) host::set_launches(7);
  return st8(e);
}

int casc_i8_gemm_fp64x2(int64_t m, int64_t n, int64_t k, const double* A_hi, const double* A_lo,
                        int64_t lda, const double* B_hi, const double* B_lo, int64_t ldb,
                        double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags, int y,
                        casc_stream_t stream) {
  int r = host::validate_gemm(m, n, k, A_hi, A_lo, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, flags);
  if (r) return r;
  if (y < i8::YMIN || y > i8::YMAX) return CASC_ERR_INVALID;
  if (m == 0 || n == 0) return CASC_OK;
  if ((r = host::device_check(nullptr))) return r;
  if (k == 0) return host::zero_c(m, n, C_hi, C_lo, ldc, flags, S8(stream));
  const size_t need = casc_i8_workspace_bytes(m, n, k, y);
  const cudaStream_t st = S8(stream);
  void* ws = nullptr;  // stream-ordered, per call (see casc_gemm_fp64x2)
  if (cudaMallocAsync(&ws, need, st) != cudaSuccess) return CASC_ERR_CUDA;
  r = casc_i8_gemm_fp64x2_ws(m, n, k, A_hi, A_lo, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, flags, y,
                             ws, need, stream);
  cudaFreeAsync(ws, st);
  return r;
}

int casc_i8_finalize(void) { return casc_finalize(); }

int casc_i8_split(int64_t rows, int64_t k, const double* hi, const double* lo, int64_t ld,
                  int is_b, int y, int8_t* digits, int32_t* e, casc_stream_t stream) {
  host::set_launches(0);
  int r;
  if (rows < 0 || k < 0 || y < i8::YMIN || y > i8::YMAX) return CASC_ERR_INVALID;
  if (is_b) {
    if ((r = host::check_mat(hi, k, rows, ld)) || (r = host::check_mat(lo, k, rows, ld))) return r;
  } else {
    if ((r = host::check_mat(hi, rows, k, ld)) || (r = host::check_mat(lo, rows, k, ld))) return r;
  }
  if (rows == 0 || k == 0) return CASC_OK;
  if (!digits || !e) return CASC_ERR_INVALID;
  if ((r = host::device_check(nullptr))) return r;
  const cudaStream_t st = S8(stream);
  void* buf = nullptr;
  if (cudaMallocAsync(&buf, casc_i8_packed_bytes(rows, k, y), st) != cudaSuccess)
    return CASC_ERR_CUDA;
  cudaError_t er = i8::pack(hi, lo, ld, rows, k, y, is_b != 0, buf, st);
  if (er == cudaSuccess) er = i8::unpack(buf, rows, k, y, digits, e, st);
  cudaFreeAsync(buf, st);
  return st8(er);
}

int casc_i8_debug_bins(int64_t m, int64_t n, int64_t k, const double* A_hi, const double* A_lo,
                       int64_t lda, const double* B_hi, const double* B_lo, int64_t ldb, int y,
                       int64_t panel, int32_t* bins, casc_stream_t stream) {
  host::set_launches(0);
  int r;
  if (m < 0 || n < 0 || k < 0 || y < i8::YMIN || y > i8::YMAX) return CASC_ERR_INVALID;
  if ((r = host::check_mat(A_hi, m, k, lda)) || (r = host::check_mat(A_lo, m, k, lda))) return r;
  if ((r = host::check_mat(B_hi, k, n, ldb)) || (r = host::check_mat(B_lo, k, n, ldb))) return r;
  if (m == 0 || n == 0 || k == 0) return CASC_OK;
  if (panel < 0 || panel >= (k + i8::KC8 - 1) / i8::KC8 || !bins) return CASC_ERR_INVALID;
  int sms = 0;
  if ((r = host::device_check(&sms))) return r;
  const cudaStream_t st = S8(stream);
  const size_t need = casc_i8_workspace_bytes(m, n, k, y);
  void* buf = nullptr;
  if (cudaMallocAsync(&buf, need, st) != cudaSuccess) return CASC_ERR_CUDA;
  uint8_t* pa = static_cast<uint8_t*>(buf);
  uint8_t* pb = pa + al256h(casc_i8_packed_bytes(m, k, y));
  double* ws = reinterpret_cast<double*>(pb + al256h(casc_i8_packed_bytes(n, k, y)));
  cudaError_t e = i8::pack(A_hi, A_lo, lda, m, k, y, false, pa, st);
  if (e == cudaSuccess) e = i8::pack(B_hi, B_lo, ldb, n, k, y, true, pb, st);
  if (e == cudaSuccess)
    e = i8::gemm(pa, pb, m, n, k, y, nullptr, nullptr, n, nullptr, ws, i8::ws_grid(m, n, sms),
                 bins, panel, st);
  cudaFreeAsync(buf, st);
  return st8(e);
}

}  // extern "C"
