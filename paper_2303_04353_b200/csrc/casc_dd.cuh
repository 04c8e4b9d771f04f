// casc_dd.cuh — double-double error-free transformations and the fl_casc bin
// combine shared by the fused kernel and the simple-path
// epilogue (product path only; the oracle has its own, independent code).
#pragma once
#include "casc_layout.cuh"

namespace casc {

// ------------------------------------------------------------ DD helpers
// Textbook EFTs with explicit _rn intrinsics (bit-reproducible, no FMA).
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
__device__ __forceinline__ void fast_two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  e = __dsub_rn(b, __dsub_rn(s, a));
}
__device__ __forceinline__ void dd_add_d(double& h, double& l, double x) {
  double s, e;
  two_sum(h, x, s, e);
  e = __dadd_rn(e, l);
  fast_two_sum(s, e, h, l);
}
__device__ __forceinline__ void dd_add(double xh, double xl, double yh, double yl, double& rh,
                                       double& rl) {
  double s1, s2, t1, t2;
  two_sum(xh, yh, s1, s2);
  two_sum(xl, yl, t1, t2);
  s2 = __dadd_rn(s2, t1);
  fast_two_sum(s1, s2, s1, s2);
  s2 = __dadd_rn(s2, t2);
  fast_two_sum(s1, s2, rh, rl);
}


// FP64x2 product (TwoProd by FMA; same sequence as the oracle's orc_dd_mul).
__device__ __forceinline__ void dd_mul(double xh, double xl, double yh, double yl, double& rh,
                                       double& rl) {
  const double p = __dmul_rn(xh, yh);
  double e = __fma_rn(xh, yh, -p);
  e = __dadd_rn(e, __dadd_rn(__dmul_rn(xh, yl), __dmul_rn(xl, yh)));
  fast_two_sum(p, e, rh, rl);
}

// FP64x2 long division (reading R27): q1 = x.hi / y.hi; r = x - q1 y;
// q2 = r.hi / y.hi; Fast2Sum(q1, q2).
__device__ __forceinline__ void dd_div(double xh, double xl, double yh, double yl, double& rh,
                                       double& rl) {
  const double q1 = __ddiv_rn(xh, yh);
  double ph, pl, sh, sl;
  dd_mul(q1, 0.0, yh, yl, ph, pl);
  dd_add(xh, xl, -ph, -pl, sh, sl);
  const double q2 = __ddiv_rn(sh, yh);
  fast_two_sum(q1, q2, rh, rl);
}

// BLAS-style update C := alpha (x) T (+) beta (x) C_old (NEXT-4, reading R21).
__device__ __forceinline__ void apply_alpha_beta(double& th, double& tl, double ah, double al,
                                                 double bh, double bl, double ch, double cl,
                                                 bool use_beta) {
  dd_mul(ah, al, th, tl, th, tl);
  if (use_beta) {
    double uh, ul;
    dd_mul(bh, bl, ch, cl, uh, ul);
    dd_add(th, tl, uh, ul, th, tl);
  }
}

// fl_casc of one element (reading R9), bins in the
// kernel's pre-aligned scales: T = TwoSum(2^-2c0 bin2', 2^-D2 bin36);
// T = T (+) 2^-c0 bin1; T = T (+) bin0; T = (ldexp(T.hi, escale), ldexp(T.lo, escale)).
// WIDE: e_i + f_j may lie outside [-1022, 1023] (then each limb is scaled
// ldexp-exactly, reading R16); otherwise 2^escale is one normal double.
template <bool WIDE = true>
__device__ __forceinline__ void combine_bins(double b0, double b1, double b2p, double b36,
                                             int c0, int D2, int escale, double& th,
                                             double& tl) {
  two_sum(__dmul_rn(b2p, pow2i(-2 * c0)), __dmul_rn(b36, pow2i(-D2)), th, tl);
  dd_add_d(th, tl, __dmul_rn(b1, pow2i(-c0)));
  dd_add_d(th, tl, b0);
#ifdef CASC_EXPERIMENT_POW2I  // timing experiment only: round-1 scaling (wrong outside the range)
  if (true) {
#else
  if (!WIDE) {
#endif
    const double sc = pow2i(escale);
    th = __dmul_rn(th, sc);
    tl = __dmul_rn(tl, sc);
  } else {
#if defined(CASC_WIDE_CALL)
    th = ldexp_rn_wide(th, escale);
    tl = ldexp_rn_wide(tl, escale);
#elif defined(CASC_WIDE_2STEP)
    const bool up = escale > 1023, down = escale < -1074;
    const int n0 = up ? 1023 : (down ? escale + 1074 : escale);
    const int n1 = up ? escale - 1023 : (down ? -1074 : 0);
    const double s0 = pow2_any(n0), s1 = pow2_any(n1);
    th = __dmul_rn(__dmul_rn(th, s0), s1);
    tl = __dmul_rn(__dmul_rn(tl, s0), s1);
#else
    double sc[3];
    pow2_steps(escale, sc);
    th = __dmul_rn(__dmul_rn(__dmul_rn(th, sc[0]), sc[1]), sc[2]);
    tl = __dmul_rn(__dmul_rn(__dmul_rn(tl, sc[0]), sc[1]), sc[2]);
#endif
  }
}

}  // namespace casc
