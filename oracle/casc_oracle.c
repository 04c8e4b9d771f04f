/*
 * casc_oracle.c — CPU ORACLE for the cascaded FP64x2 GEMM (arXiv 2303.04353).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library. The
 * product path (paper_2303_04353_b200/) never imports, links or executes it and
 * shares no code, header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct C (binary64, round-to-nearest-even, compiled
 * with -ffp-contract=off and no fast-math so every +, -, * is one IEEE op).
 * Loops are parallelised over output rows with OpenMP only; nothing is blocked,
 * fused or reordered beyond what the cited passage states.
 *
 * Citations: P:Lnnn = PAPER.md line, S:Lnnn = SPEC.md line, "reading Rn" =
 * the numbered reading in DESIGN.md §3 (SURVEY.md §8(c) ambiguity table).
 *
 * Three parts:
 *   ORACLE-CASCADE  orc_select_widths, orc_scale_exponent, orc_split_scalar,
 *                   orc_split_a_panel, orc_split_b_panel, orc_panel_bins,
 *                   orc_combine, orc_casc_gemm   — the paper's method, step by step.
 *   ORACLE-DD       orc_dd_gemm                  — triple-loop FP64x2 GEMM.
 *   ORACLE-EXACT    orc_exact_entries            — exact products via a fixed-point
 *                   superaccumulator (stands in for the paper's FP128x2 reference,
 *                   P:L3474).
 *
 * Pins: tests/test_oracle_*.py check every function here against Python
 * Fraction brute force, paper-printed values and closed-form bounds.
 * Parity unpinned: none (see DESIGN.md §4 for the pin of each function).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define KC 256 /* k_C, the rank-k update depth: P:L3131, reading R3 */

/* ------------------------------------------------------------------------- */
/* DD primitives. Textbook error-free transformations; the paper only says    */
/* "FP64x2 addition or quick two-sum arithmetic [Dekker1971]" */
/* ------------------------------------------------------------------------- */

/* Knuth TwoSum: s = fl(a+b), s + e = a + b exactly (6 adds, branch-free). */
void orc_two_sum(double a, double b, double* s, double* e) {
  double ss = a + b;
  double bb = ss - a;
  double err = (a - (ss - bb)) + (b - bb);
  *s = ss;
  *e = err;
}

/* Dekker Fast2Sum: valid when |a| >= |b| (or a == 0). */
void orc_fast_two_sum(double a, double b, double* s, double* e) {
  double ss = a + b;
  *e = b - (ss - a);
  *s = ss;
}

/* TwoProd with a correctly rounded FMA: p = fl(a*b), p + e = a*b exactly
 * ("emulating FP64x2 multiplication only requires 1 FMA and 1 multiply"). */
void orc_two_prod(double a, double b, double* p, double* e) {
  double pp = a * b;
  *e = fma(a, b, -pp);
  *p = pp;
}

/* DD + double: (s,e) = TwoSum(T.hi, x); e += T.lo; Fast2Sum(s, e). */
void orc_dd_add_d(double th, double tl, double x, double* rh, double* rl) {
  double s, e;
  orc_two_sum(th, x, &s, &e);
  e = e + tl;
  orc_fast_two_sum(s, e, rh, rl);
}

/* DD + DD (the "accurate" variant, two TwoSums). */
void orc_dd_add(double xh, double xl, double yh, double yl, double* rh, double* rl) {
  double s1, s2, t1, t2;
  orc_two_sum(xh, yh, &s1, &s2);
  orc_two_sum(xl, yl, &t1, &t2);
  s2 = s2 + t1;
  orc_fast_two_sum(s1, s2, &s1, &s2);
  s2 = s2 + t2;
  orc_fast_two_sum(s1, s2, rh, rl);
}

/* DD * DD: p = TwoProd(xh, yh); p.lo += xh*yl + xl*yh; renormalise. */
void orc_dd_mul(double xh, double xl, double yh, double yl, double* rh, double* rl) {
  double p, e;
  orc_two_prod(xh, yh, &p, &e);
  e = e + (xh * yl + xl * yh);
  orc_fast_two_sum(p, e, rh, rl);
}

/* ------------------------------------------------------------------------- */
/* a1. Split widths (§3.3; reading R3: widths from min(k, k_C)).  */
/*   2c0 + L <= 53;  c0 + c1 + L + 1 <= 53 and 2c1 + L + 2 <= 53;            */
/*   c0 + c2 + L + 2 <= 53;  L = ceil(log2 k_eff); greedy c0, then c1, c2.    */
/* ------------------------------------------------------------------------- */
static int ceil_log2(int64_t k) {
  int L = 0;
  while (((int64_t)1 << L) < k) L++;
  return L;
}

void orc_select_widths(int64_t k, int* c) {
  int64_t keff = k < KC ? k : KC;
  if (keff < 1) keff = 1;
  int L = ceil_log2(keff);
  int c0 = 0, c1 = 0, c2 = 0;
  while (2 * (c0 + 1) + L <= 53) c0++;
  while (c0 + (c1 + 1) + L + 1 <= 53 && 2 * (c1 + 1) + L + 2 <= 53) c1++;
  while (c0 + (c2 + 1) + L + 2 <= 53) c2++;
  c[0] = c0;
  c[1] = c1;
  c[2] = c2;
}

/* ------------------------------------------------------------------------- */
/* a2. Scale exponent of a vector ("smallest power of two greater      */
/* than" the max magnitude; P:L1139 ||x|| <= sigma <= 2||x||;   */
/* reading R1): e = frexp exponent of max |hi|, so max|hi| in [2^(e-1), 2^e). */
/* All-zero vector: e = 0.                                                    */
/* ------------------------------------------------------------------------- */
int orc_scale_exponent(const double* hi, int64_t n, int64_t stride) {
  double mx = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double a = fabs(hi[i * stride]);
    if (a > mx) mx = a;
  }
  if (mx == 0.0) return 0;
  int e;
  frexp(mx, &e);
  return e;
}

/* ------------------------------------------------------------------------- */
/* a3. Appendix A conditional-free split of one FP64x2 value. */
/* Each limb separately: v = limb * 2^-e; for t = 0,1,2:                      */
/*   s_t = (v + M_t) - M_t with M_t = 2^(53-c_t) + 2^(52-c_t) (readings R4,   */
/*   R5: one precomputed constant, "powers of two can be precomputed")*/
/*   v = (v - s_t) * 2^(c_t);  s_3 = v.   Then chi_t = s_t(hi) + s_t(lo).     */
/* Output chi[0..3] in the paper's normalisation: value ~ 2^e * (chi0 +       */
/* sigma1 chi1 + sigma2 chi2 + sigma3 chi3), sigma_t = 2^-D_(t-1)*/
/* ------------------------------------------------------------------------- */
static void split_limb(double x, int e, const int* c, double* s) {
  double v = ldexp(x, -e);
  for (int t = 0; t < 3; ++t) {
    double M = ldexp(1.0, 53 - c[t]) + ldexp(1.0, 52 - c[t]);
    double r = v + M;
    r = r - M;
    s[t] = r;
    v = (v - r) * ldexp(1.0, c[t]);
  }
  s[3] = v;
}

void orc_split_scalar(double hi, double lo, int e, const int* c, double* chi) {
  double sh[4], sl[4];
  split_limb(hi, e, c, sh);
  split_limb(lo, e, c, sl);
  for (int t = 0; t < 4; ++t) chi[t] = sh[t] + sl[t];
}

/* ------------------------------------------------------------------------- */
/* Panel splits (§3.4: rows of A and columns of B */
/* split conformally; reading R2: one scale per (row, k_C panel) and per      */
/* (column, k_C panel)).                                                      */
/*   A panel: rows 0..m-1, columns p0..p0+kp-1 of A (row-major, lda).         */
/*     out: S[t*m*kp + i*kp + p], t = 0..3 (canonical, unaligned); e[i].      */
/*   B panel: rows p0..p0+kp-1, columns 0..n-1 of B (row-major, ldb).         */
/*     out: S[t*kp*n + p*n + j], t = 0..6; f[j].                              */
/*     B4 = B2 + 2^-c2 B3; B5 = B1 + 2^-c1 B4; B6 = B0 + 2^-c0 B5 (P:L1403-    */
/*     1404; reading R7: nested, one RNE add each).                           */
/* ------------------------------------------------------------------------- */
void orc_split_a_panel(int64_t m, int64_t kp, const double* Ahi, const double* Alo,
                       int64_t lda, const int* c, double* S, int32_t* e) {
  for (int64_t i = 0; i < m; ++i) {
    int ei = orc_scale_exponent(Ahi + i * lda, kp, 1);
    e[i] = ei;
    for (int64_t p = 0; p < kp; ++p) {
      double chi[4];
      orc_split_scalar(Ahi[i * lda + p], Alo[i * lda + p], ei, c, chi);
      for (int t = 0; t < 4; ++t) S[(int64_t)t * m * kp + i * kp + p] = chi[t];
    }
  }
}

void orc_split_b_panel(int64_t kp, int64_t n, const double* Bhi, const double* Blo,
                       int64_t ldb, const int* c, double* S, int32_t* f) {
  const int64_t sz = kp * n;
  for (int64_t j = 0; j < n; ++j) {
    int fj = orc_scale_exponent(Bhi + j, kp, ldb);
    f[j] = fj;
    for (int64_t p = 0; p < kp; ++p) {
      double psi[4];
      orc_split_scalar(Bhi[p * ldb + j], Blo[p * ldb + j], fj, c, psi);
      double b4 = psi[2] + ldexp(psi[3], -c[2]); /* sigma3/sigma2 = 2^-c2 */
      double b5 = psi[1] + ldexp(b4, -c[1]);     /* sigma2/sigma1 = 2^-c1 */
      double b6 = psi[0] + ldexp(b5, -c[0]);     /* sigma1 = 2^-c0        */
      double out[7] = {psi[0], psi[1], psi[2], psi[3], b4, b5, b6};
      for (int t = 0; t < 7; ++t) S[t * sz + p * n + j] = out[t];
    }
  }
}

/* ------------------------------------------------------------------------- */
/* a5. Bins of one k_C panel (eqn:Gemm10 P:L1407-1440; bins P:L633-745;      */
/* reading R8: exact in-bin alignment factors).                               */
/*   bin0  = sum_p A0 B0                                     (ref scale 1)    */
/*   bin1  = sum_p (A0 B1 + A1 B0)                           (ref sigma1)     */
/*   bin2  = sum_p (A0 B2 + 2^(c1-c0) A1 B1 + A2 B0)         (ref sigma2)     */
/*   bin36 = sum_p (A0 B3 + 2^(c2-c0) A1 B4 + 2^(c2-c0) A2 B5 + A3 B6)        */
/*                                                           (ref sigma3)     */
/* Bins 0-2 are exact, so their order is irrelevant; bin36 is       */
/* evaluated in FP64 with p ascending and terms in the order written.         */
/* bins out: bins[b*m*n + i*n + j], b = 0..3.                                 */
/* ------------------------------------------------------------------------- */
void orc_panel_bins(int64_t m, int64_t n, int64_t kp, const double* SA, const double* SB,
                    const int* c, double* bins) {
  const int64_t sa = m * kp, sb = kp * n, sc = m * n;
#ifdef ORC_MUTATE_ALIGN
  /* Mutation canary: a deliberately wrong alignment factor. Only the
   * test suite builds this variant, to prove the bin identity test catches it. */
  const double f11 = ldexp(1.0, c[1] - c[0] + 1);
#else
  const double f11 = ldexp(1.0, c[1] - c[0]); /* sigma1^2/sigma2 */
#endif
  const double f36 = ldexp(1.0, c[2] - c[0]); /* sigma1 sigma2 / sigma3 */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      double b0 = 0, b1 = 0, b2 = 0, b36 = 0;
      for (int64_t p = 0; p < kp; ++p) {
        const double a0 = SA[0 * sa + i * kp + p], a1 = SA[1 * sa + i * kp + p];
        const double a2 = SA[2 * sa + i * kp + p], a3 = SA[3 * sa + i * kp + p];
        const double y0 = SB[0 * sb + p * n + j], y1 = SB[1 * sb + p * n + j];
        const double y2 = SB[2 * sb + p * n + j], y3 = SB[3 * sb + p * n + j];
        const double y4 = SB[4 * sb + p * n + j], y5 = SB[5 * sb + p * n + j];
        const double y6 = SB[6 * sb + p * n + j];
        b0 = b0 + a0 * y0;
        b1 = b1 + a0 * y1;
        b1 = b1 + a1 * y0;
        b2 = b2 + a0 * y2;
        b2 = b2 + f11 * (a1 * y1);
        b2 = b2 + a2 * y0;
        b36 = b36 + a0 * y3;
        b36 = b36 + f36 * (a1 * y4);
        b36 = b36 + f36 * (a2 * y5);
        b36 = b36 + a3 * y6;
      }
      bins[0 * sc + i * n + j] = b0;
      bins[1 * sc + i * n + j] = b1;
      bins[2 * sc + i * n + j] = b2;
      bins[3 * sc + i * n + j] = b36;
    }
  }
}

/* ------------------------------------------------------------------------- */
/* a6. Combine one element's bins (fl_casc: bin0 (+) (bin1 (+)  */
/* (bin2 (+) fl(bin3-6))) with (+) in FP64x2; order bin 6 -> bin 0, P:L948-   */
/* 949; Sigma, T applied after; reading R9 for the DD ops). */
/*   T = TwoSum(sigma2 bin2, sigma3 bin36); T = T (+) sigma1 bin1;            */
/*   T = T (+) bin0; T *= 2^(e+f).                                            */
/* ------------------------------------------------------------------------- */
void orc_combine(double bin0, double bin1, double bin2, double bin36, int escale,
                 const int* c, double* th, double* tl) {
  const int D0 = c[0], D1 = c[0] + c[1], D2 = c[0] + c[1] + c[2];
  double h, l;
  orc_two_sum(ldexp(bin2, -D1), ldexp(bin36, -D2), &h, &l);
  orc_dd_add_d(h, l, ldexp(bin1, -D0), &h, &l);
  orc_dd_add_d(h, l, bin0, &h, &l);
  *th = ldexp(h, escale);
  *tl = ldexp(l, escale);
}

/* ------------------------------------------------------------------------- */
/* ORACLE-CASCADE: C := A B staged as rank-k_C updates (§3.5 P:L1474- */
/* 1484, §4.2): for each panel q ascending: split A and B        */
/* panels, 10-product bins, combine, C (+)= T in FP64x2 (P:L2839;    */
/* reading R10), flag |= (bin0 == 0) (§3.7, §4.4;        */
/* reading R11). k == 0 gives C = 0, flags = 0 (reading R18).                 */
/* flags may be NULL. C is m x n row-major with ldc.                          */
/* ------------------------------------------------------------------------- */
void orc_casc_gemm(int64_t m, int64_t n, int64_t k, const double* Ahi, const double* Alo,
                   int64_t lda, const double* Bhi, const double* Blo, int64_t ldb, double* Chi,
                   double* Clo, int64_t ldc, uint8_t* flags, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  int c[3];
  orc_select_widths(k, c);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      Chi[i * ldc + j] = 0.0;
      Clo[i * ldc + j] = 0.0;
      if (flags) flags[i * n + j] = 0;
    }
  if (m == 0 || n == 0 || k == 0) return;
  const int64_t kpmax = k < KC ? k : KC;
  double* SA = (double*)malloc(sizeof(double) * 4 * m * kpmax);
  double* SB = (double*)malloc(sizeof(double) * 7 * kpmax * n);
  double* bins = (double*)malloc(sizeof(double) * 4 * m * n);
  int32_t* e = (int32_t*)malloc(sizeof(int32_t) * m);
  int32_t* f = (int32_t*)malloc(sizeof(int32_t) * n);
  for (int64_t p0 = 0; p0 < k; p0 += KC) {
    const int64_t kp = (k - p0) < KC ? (k - p0) : KC;
    orc_split_a_panel(m, kp, Ahi + p0, Alo + p0, lda, c, SA, e);
    orc_split_b_panel(kp, n, Bhi + p0 * ldb, Blo + p0 * ldb, ldb, c, SB, f);
    orc_panel_bins(m, n, kp, SA, SB, c, bins);
    const int64_t sc = m * n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j) {
        const double b0 = bins[0 * sc + i * n + j];
        double th, tl;
        orc_combine(b0, bins[1 * sc + i * n + j], bins[2 * sc + i * n + j],
                    bins[3 * sc + i * n + j], e[i] + f[j], c, &th, &tl);
        orc_dd_add(Chi[i * ldc + j], Clo[i * ldc + j], th, tl, &Chi[i * ldc + j],
                   &Clo[i * ldc + j]);
        if (flags && b0 == 0.0) flags[i * n + j] = 1;
      }
  }
  free(SA);
  free(SB);
  free(bins);
  free(e);
  free(f);
}

/* Rows [r0, r0+mr) of ORACLE-CASCADE, for bounded CPU-baseline samples and
 * sampled parity at full size: identical arithmetic, C rows only. */
void orc_casc_gemm_rows(int64_t r0, int64_t mr, int64_t n, int64_t k, const double* Ahi,
                        const double* Alo, int64_t lda, const double* Bhi, const double* Blo,
                        int64_t ldb, double* Chi, double* Clo, int64_t ldc, uint8_t* flags,
                        int nthreads) {
  orc_casc_gemm(mr, n, k, Ahi + r0 * lda, Alo + r0 * lda, lda, Bhi, Blo, ldb, Chi, Clo, ldc,
                flags, nthreads);
}

/* ------------------------------------------------------------------------- */
/* NEXT-4 (BLAS generality): C := alpha (x) op(A) op(B) (+)     */
/* beta (x) C (reading R21).  op() is a plain copy into row-major arrays; the */
/* product is ORACLE-CASCADE; the update is FP64x2 mul then FP64x2 add.       */
/* k == 0 or alpha == 0: C := beta (x) C (0 if beta == 0), flags := 0.        */
/* alpha == 1 and beta == 0: C := product (no update arithmetic).             */
/* ------------------------------------------------------------------------- */
void orc_casc_gemm_ex(int transa, int transb, int64_t m, int64_t n, int64_t k, double ah,
                      double al, const double* Ahi, const double* Alo, int64_t lda,
                      const double* Bhi, const double* Blo, int64_t ldb, double bh, double bl,
                      double* Chi, double* Clo, int64_t ldc, uint8_t* flags, int nthreads) {
  const int use_beta = !(bh == 0.0 && bl == 0.0);
  if (k == 0 || (ah == 0.0 && al == 0.0)) {
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j) {
        double rh = 0.0, rl = 0.0;
        if (use_beta) orc_dd_mul(bh, bl, Chi[i * ldc + j], Clo[i * ldc + j], &rh, &rl);
        Chi[i * ldc + j] = rh;
        Clo[i * ldc + j] = rl;
        if (flags) flags[i * n + j] = 0;
      }
    return;
  }
  double* a_h = (double*)calloc((size_t)(m * k), sizeof(double));
  double* a_l = (double*)calloc((size_t)(m * k), sizeof(double));
  double* b_h = (double*)calloc((size_t)(k * n), sizeof(double));
  double* b_l = (double*)calloc((size_t)(k * n), sizeof(double));
  double* p_h = (double*)malloc(sizeof(double) * m * n);
  double* p_l = (double*)malloc(sizeof(double) * m * n);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t p = 0; p < k; ++p) {
      const int64_t s = transa ? p * lda + i : i * lda + p;
      a_h[i * k + p] = Ahi[s];
      a_l[i * k + p] = Alo[s];
    }
  for (int64_t p = 0; p < k; ++p)
    for (int64_t j = 0; j < n; ++j) {
      const int64_t s = transb ? j * ldb + p : p * ldb + j;
      b_h[p * n + j] = Bhi[s];
      b_l[p * n + j] = Blo[s];
    }
  orc_casc_gemm(m, n, k, a_h, a_l, k, b_h, b_l, n, p_h, p_l, n, flags, nthreads);
  const int unit_alpha = (ah == 1.0 && al == 0.0);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double th = p_h[i * n + j], tl = p_l[i * n + j];
      if (!unit_alpha || use_beta) {
        orc_dd_mul(ah, al, th, tl, &th, &tl);
        if (use_beta) {
          double uh, ul;
          orc_dd_mul(bh, bl, Chi[i * ldc + j], Clo[i * ldc + j], &uh, &ul);
          orc_dd_add(th, tl, uh, ul, &th, &tl);
        }
      }
      Chi[i * ldc + j] = th;
      Clo[i * ldc + j] = tl;
    }
  free(a_h);
  free(a_l);
  free(b_h);
  free(b_l);
  free(p_h);
  free(p_l);
}

/* ------------------------------------------------------------------------- */
/* ORACLE-DD: plain triple-loop FP64x2 GEMM, the paper's accuracy comparator */
/* (§5.2 P:L3549 "a simple triple-nested loop in FP64x2 arithmetic";          */
/* S:L399-405). C := A B, loop order i, j, p; dd_mul then dd_add.             */
/* ------------------------------------------------------------------------- */
void orc_dd_gemm(int64_t m, int64_t n, int64_t k, const double* Ahi, const double* Alo,
                 int64_t lda, const double* Bhi, const double* Blo, int64_t ldb, double* Chi,
                 double* Clo, int64_t ldc, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double ch = 0.0, cl = 0.0;
      for (int64_t p = 0; p < k; ++p) {
        double ph, pl;
        orc_dd_mul(Ahi[i * lda + p], Alo[i * lda + p], Bhi[p * ldb + j], Blo[p * ldb + j], &ph,
                   &pl);
        orc_dd_add(ch, cl, ph, pl, &ch, &cl);
      }
      Chi[i * ldc + j] = ch;
      Clo[i * ldc + j] = cl;
    }
}

/* ------------------------------------------------------------------------- */
/* ORACLE-EXACT: fixed-point superaccumulator (Kulisch style,     */
/* S:L172-173). Value = sum_i dig[i] * 2^(32 i + SA_MINEXP); digits int64,    */
/* base 2^32, so each digit absorbs >= 2^30 additions before normalisation.   */
/* Covers every product of two finite doubles (exponents -2148 .. 2047).      */
/* ------------------------------------------------------------------------- */
#define SA_MINEXP (-2240)
#define SA_NDIG 140 /* 140 * 32 = 4480 bits: 2^-2240 .. 2^2240 */

typedef struct {
  int64_t d[SA_NDIG];
  int64_t nadd;
} superacc;

static void sa_clear(superacc* s) { memset(s, 0, sizeof(*s)); }

static void sa_normalize(superacc* s) {
  int64_t carry = 0;
  for (int i = 0; i < SA_NDIG; ++i) {
    int64_t v = s->d[i] + carry;
    int64_t lo = v & 0xFFFFFFFFLL;     /* in [0, 2^32) */
    carry = (v - lo) / 4294967296LL;   /* exact: v - lo is a multiple of 2^32 */
    s->d[i] = lo;
  }
  s->d[SA_NDIG - 1] += carry * 4294967296LL; /* top digit keeps the sign */
  s->nadd = 0;
}

static void sa_add_double(superacc* s, double x) {
  if (x == 0.0) return;
  int ex;
  double fr = frexp(fabs(x), &ex);                   /* |x| = fr * 2^ex, fr in [0.5,1) */
  uint64_t mant = (uint64_t)ldexp(fr, 53);            /* exact: 53-bit integer */
  int q = ex - 53;                                    /* |x| = mant * 2^q */
  if (q < -1074 - 53) {                               /* subnormal: mant has fewer bits */
    /* ldexp(fr,53) is still exact; q as computed remains correct */
  }
  int pos = q - SA_MINEXP;
  int di = pos / 32, sh = pos % 32;
  unsigned __int128 v = (unsigned __int128)mant << sh;
  int64_t p0 = (int64_t)(uint64_t)(v & 0xFFFFFFFFu);
  int64_t p1 = (int64_t)(uint64_t)((v >> 32) & 0xFFFFFFFFu);
  int64_t p2 = (int64_t)(uint64_t)((v >> 64) & 0xFFFFFFFFu);
  if (x > 0) {
    s->d[di] += p0; s->d[di + 1] += p1; s->d[di + 2] += p2;
  } else {
    s->d[di] -= p0; s->d[di + 1] -= p1; s->d[di + 2] -= p2;
  }
  if (++s->nadd >= (1LL << 29)) sa_normalize(s);
}

/* Add the exact product a*b (TwoProd: two doubles, exact). */
static void sa_add_prod(superacc* s, double a, double b) {
  double p, e;
  orc_two_prod(a, b, &p, &e);
  sa_add_double(s, p);
  sa_add_double(s, e);
}

/* Correctly rounded (RNE) double nearest to the accumulator (no overflow). */
static double sa_to_double(superacc* s) {
  sa_normalize(s);
  int neg = s->d[SA_NDIG - 1] < 0;
  int64_t dig[SA_NDIG];
  if (neg) {
    /* two's complement negate in base 2^32: value -> -value */
    int64_t carry = 1;
    for (int i = 0; i < SA_NDIG; ++i) {
      int64_t v = (~s->d[i] & 0xFFFFFFFFLL) + carry;
      carry = v >> 32;
      dig[i] = v & 0xFFFFFFFFLL;
    }
  } else {
    memcpy(dig, s->d, sizeof(dig));
  }
  int h = SA_NDIG - 1;
  while (h >= 0 && dig[h] == 0) --h;
  if (h < 0) return 0.0;
  int lo = h - 2 < 0 ? 0 : h - 2;
  unsigned __int128 v = 0;
  for (int i = h; i >= lo; --i) v = (v << 32) | (unsigned __int128)(uint64_t)dig[i];
  int sticky = 0;
  for (int i = lo - 1; i >= 0; --i)
    if (dig[i]) { sticky = 1; break; }
  /* v has >= 65 significant bits when h >= 2; setting bit 0 as a sticky bit is
   * exact for round-to-nearest to 53 bits. (__int128 -> double rounds RNE.) */
  v = (v << 1) | (unsigned __int128)sticky;
  double r = ldexp((double)v, 32 * lo + SA_MINEXP - 1);
  return neg ? -r : r;
}

/* For each requested entry (ii[t], jj[t]):
 *   exact C*_{ij} = sum_p (Ahi+Alo)(Bhi+Blo)  -> (ex_hi, ex_lo) RN double-double
 *   err  = RN( (Chi + Clo) - C*_{ij} )          (if Chi != NULL)
 *   absab = RN( sum_p |A_ip| |B_pj| )            (|A| = |Ahi + Alo| exactly)
 * Any output pointer may be NULL. */
void orc_exact_entries(int64_t k, const double* Ahi, const double* Alo, int64_t lda,
                       const double* Bhi, const double* Blo, int64_t ldb, int64_t nent,
                       const int64_t* ii, const int64_t* jj, const double* Chi,
                       const double* Clo, int64_t ldc, double* ex_hi, double* ex_lo,
                       double* err, double* absab, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < nent; ++t) {
    const int64_t i = ii[t], j = jj[t];
    superacc* s = (superacc*)malloc(sizeof(superacc));
    superacc* sa = (superacc*)malloc(sizeof(superacc));
    sa_clear(s);
    sa_clear(sa);
    for (int64_t p = 0; p < k; ++p) {
      const double ah = Ahi[i * lda + p], al = Alo[i * lda + p];
      const double bh = Bhi[p * ldb + j], bl = Blo[p * ldb + j];
      sa_add_prod(s, ah, bh);
      sa_add_prod(s, ah, bl);
      sa_add_prod(s, al, bh);
      sa_add_prod(s, al, bl);
      /* |a| |b| with a = ah + al exactly: sign of a is sign of ah (non-overlap). */
      const double sgna = (ah < 0) ? -1.0 : 1.0, sgnb = (bh < 0) ? -1.0 : 1.0;
      sa_add_prod(sa, sgna * ah, sgnb * bh);
      sa_add_prod(sa, sgna * ah, sgnb * bl);
      sa_add_prod(sa, sgna * al, sgnb * bh);
      sa_add_prod(sa, sgna * al, sgnb * bl);
    }
    if (absab) absab[t] = sa_to_double(sa);
    if (ex_hi || ex_lo || err) {
      superacc cp = *s;
      double h = sa_to_double(&cp);
      sa_add_double(&cp, -h);
      double l = sa_to_double(&cp);
      if (ex_hi) ex_hi[t] = h;
      if (ex_lo) ex_lo[t] = l;
    }
    if (err && Chi) {
      sa_add_double(s, -Chi[i * ldc + j]);
      sa_add_double(s, -Clo[i * ldc + j]);
      err[t] = -sa_to_double(s); /* (C_hi + C_lo) - exact */
    }
    free(s);
    free(sa);
  }
}

/* Exact sum of a list of doubles (RN double-double), for pins of the exact  */
/* bins and the DD primitives.                                               */
void orc_exact_sum(int64_t n, const double* x, double* rh, double* rl) {
  superacc* s = (superacc*)malloc(sizeof(superacc));
  sa_clear(s);
  for (int64_t i = 0; i < n; ++i) sa_add_double(s, x[i]);
  double h = sa_to_double(s);
  sa_add_double(s, -h);
  *rh = h;
  *rl = sa_to_double(s);
  free(s);
}

/* Exact dot product sum_p x_p y_p, RN double-double. */
void orc_exact_dot(int64_t n, const double* x, const double* y, double* rh, double* rl) {
  superacc* s = (superacc*)malloc(sizeof(superacc));
  sa_clear(s);
  for (int64_t i = 0; i < n; ++i) sa_add_prod(s, x[i], y[i]);
  double h = sa_to_double(s);
  sa_add_double(s, -h);
  *rh = h;
  *rl = sa_to_double(s);
  free(s);
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* NEXT-4, level-3 BLAS on the cascaded GEMM ("All Level-3 BLAS
 * algorithms can be written in terms of GEMM"): SYRK, C := alpha (x) op(A)
 * op(A)^T (+) beta (x) C on the lower (uplo 0) or upper (uplo 1) triangle,
 * diagonal included, by definition the triangle of orc_casc_gemm_ex with
 * B = A read the other way round; the other triangle of C and flags (n x n,
 * nullable) is left as it is.  A stored n x k (trans 0) or k x n (trans 1). */
void orc_casc_syrk(int uplo, int trans, int64_t n, int64_t k, double ah, double al,
                   const double* Ahi, const double* Alo, int64_t lda, double bh, double bl,
                   double* Chi, double* Clo, int64_t ldc, uint8_t* flags, int nthreads) {
  double* Th = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
  double* Tl = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
  uint8_t* Tf = (uint8_t*)calloc((size_t)(n * n + 1), 1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      Th[i * n + j] = Chi[i * ldc + j];
      Tl[i * n + j] = Clo[i * ldc + j];
    }
  orc_casc_gemm_ex(trans, !trans, n, n, k, ah, al, Ahi, Alo, lda, Ahi, Alo, lda, bh, bl, Th, Tl, n,
                   Tf, nthreads);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      if (uplo == 0 ? j > i : j < i) continue;
      Chi[i * ldc + j] = Th[i * n + j];
      Clo[i * ldc + j] = Tl[i * n + j];
      if (flags) flags[i * n + j] = Tf[i * n + j];
    }
  free(Th);
  free(Tl);
  free(Tf);
}

/* SYR2K (NEXT-4, reading R30): on one triangle,                              */
/*   C := alpha op(A) op(B)^T (+) beta C,  then  C := alpha op(B) op(A)^T (+) C, */
/* each the cascaded GEMM with the R21 update (the second with beta = 1);     */
/* flags = OR of the two products' flags.                                     */
void orc_casc_syr2k(int uplo, int trans, int64_t n, int64_t k, double ah, double al,
                    const double* Ahi, const double* Alo, int64_t lda, const double* Bhi,
                    const double* Blo, int64_t ldb, double bh, double bl, double* Chi,
                    double* Clo, int64_t ldc, uint8_t* flags, int nthreads) {
  double* Th = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
  double* Tl = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
  uint8_t* F1 = (uint8_t*)calloc((size_t)(n * n + 1), 1);
  uint8_t* F2 = (uint8_t*)calloc((size_t)(n * n + 1), 1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      Th[i * n + j] = Chi[i * ldc + j];
      Tl[i * n + j] = Clo[i * ldc + j];
    }
  orc_casc_gemm_ex(trans, !trans, n, n, k, ah, al, Ahi, Alo, lda, Bhi, Blo, ldb, bh, bl, Th, Tl, n,
                   F1, nthreads);
  orc_casc_gemm_ex(trans, !trans, n, n, k, ah, al, Bhi, Blo, ldb, Ahi, Alo, lda, 1.0, 0.0, Th, Tl,
                   n, F2, nthreads);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      if (uplo == 0 ? j > i : j < i) continue;
      Chi[i * ldc + j] = Th[i * n + j];
      Clo[i * ldc + j] = Tl[i * n + j];
      if (flags) flags[i * n + j] = F1[i * n + j] | F2[i * n + j];
    }
  free(Th);
  free(Tl);
  free(F1);
  free(F2);
}

/* ------------------------------------------------------------------------- */
/* NEXT-4, level-3 BLAS on the cascaded GEMM ("All Level-3 BLAS */
/* algorithms can be written in terms of GEMM ... integrating Phase 1 into    */
/* specific calls of say TRSM"): TRSM, reading R27.            */
/* ------------------------------------------------------------------------- */
#define TRSM_NB 256

/* DD / DD, long division: q1 = xh / yh; r = x - q1 y (DD); q2 = r.hi / yh;
 * Fast2Sum(q1, q2). */
void orc_dd_div(double xh, double xl, double yh, double yl, double* rh, double* rl) {
  const double q1 = xh / yh;
  double ph, pl, sh, sl;
  orc_dd_mul(q1, 0.0, yh, yl, &ph, &pl);
  orc_dd_add(xh, xl, -ph, -pl, &sh, &sl);
  const double q2 = sh / yh;
  orc_fast_two_sum(q1, q2, rh, rl);
}

/* Inverses of the diagonal blocks (TRSM_NB, the last one ragged) of the m x m
 * triangular A (uplo 0 lower / 1 upper; diag 0 non-unit / 1 unit): block b is
 * Inv[b][TRSM_NB][TRSM_NB] (row-major, zeros outside its triangle), column j by
 * substitution in FP64x2: lower y_j = 1 / a_jj, then for i > j
 * y_i = -(sum_{l=j}^{i-1} a_il y_l) / a_ii (l ascending); upper mirrored. */
void orc_trsm_diag_inv(int uplo, int diag, int64_t m, const double* Ahi, const double* Alo,
                       int64_t lda, double* Ihi, double* Ilo) {
  const int64_t nblk = (m + TRSM_NB - 1) / TRSM_NB;
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t r0 = b * TRSM_NB;
    const int nb = (int)((m - r0) < TRSM_NB ? (m - r0) : TRSM_NB);
    double* yh = Ihi + b * TRSM_NB * TRSM_NB;
    double* yl = Ilo + b * TRSM_NB * TRSM_NB;
    for (int i = 0; i < TRSM_NB * TRSM_NB; ++i) yh[i] = yl[i] = 0.0;
#define AH(i, l) Ahi[(r0 + (i)) * lda + r0 + (l)]
#define AL(i, l) Alo[(r0 + (i)) * lda + r0 + (l)]
    for (int j = 0; j < nb; ++j) {
      if (diag) {
        yh[j * TRSM_NB + j] = 1.0;
      } else {
        orc_dd_div(1.0, 0.0, AH(j, j), AL(j, j), &yh[j * TRSM_NB + j], &yl[j * TRSM_NB + j]);
      }
      const int step = uplo == 0 ? 1 : -1;
      for (int i = j + step; i >= 0 && i < nb; i += step) {
        double sh = 0.0, sl = 0.0;
        const int lo = uplo == 0 ? j : i + 1, hi = uplo == 0 ? i - 1 : j;
        for (int l = lo; l <= hi; ++l) {
          double ph, pl;
          orc_dd_mul(AH(i, l), AL(i, l), yh[l * TRSM_NB + j], yl[l * TRSM_NB + j], &ph, &pl);
          orc_dd_add(sh, sl, ph, pl, &sh, &sl);
        }
        if (diag) {
          yh[i * TRSM_NB + j] = -sh;
          yl[i * TRSM_NB + j] = -sl;
        } else {
          orc_dd_div(-sh, -sl, AH(i, i), AL(i, i), &yh[i * TRSM_NB + j], &yl[i * TRSM_NB + j]);
        }
      }
    }
#undef AH
#undef AL
  }
}

#define TRSM_SB 4 /* diagonal blocks per super-block of the trailing updates */
/* B[R0:R1) := B[R0:R1) - op(A)[R0:R1, C0:C1) X[C0:C1) (X = B's rows C0..C1-1),
 * with the cascaded GEMM (i8 = 0) or, when i8 = y > 0, the INT8 cascade. */
void orc_i8_casc_gemm_ex(int transa, int transb, int64_t m, int64_t n, int64_t k, double ah,
                         double al, const double* Ahi, const double* Alo, int64_t lda,
                         const double* Bhi, const double* Blo, int64_t ldb, double bh, double bl,
                         double* Chi, double* Clo, int64_t ldc, uint8_t* flags, int y,
                         int nthreads);
void orc_trsm_update(int trans, int64_t R0, int64_t R1, int64_t C0, int64_t C1, int64_t n,
                     const double* Ahi, const double* Alo, int64_t lda, double* Bhi, double* Blo,
                     int64_t ldb, int nthreads, int i8) {
  if (R1 <= R0 || C1 <= C0) return;
  const int64_t off = trans ? C0 * lda + R0 : R0 * lda + C0;
  if (i8)
    orc_i8_casc_gemm_ex(trans, 0, R1 - R0, n, C1 - C0, -1.0, 0.0, Ahi + off, Alo + off, lda,
                        Bhi + C0 * ldb, Blo + C0 * ldb, ldb, 1.0, 0.0, Bhi + R0 * ldb,
                        Blo + R0 * ldb, ldb, NULL, i8, nthreads);
  else
    orc_casc_gemm_ex(trans, 0, R1 - R0, n, C1 - C0, -1.0, 0.0, Ahi + off, Alo + off, lda,
                     Bhi + C0 * ldb, Blo + C0 * ldb, ldb, 1.0, 0.0, Bhi + R0 * ldb,
                     Blo + R0 * ldb, ldb, NULL, nthreads);
}

/* TRSM, left side: solve op(A) X = alpha B, op(A) = A (trans 0) or A^T (trans
 * 1); X overwrites the m x n B (ldb).  B := alpha (x) B; the diagonal blocks of
 * A are inverted (orc_trsm_diag_inv, op(A_bb)^-1 = op(Inv_b)); then block by
 * block in the order of op(A)'s triangle (ascending when op(A) is lower,
 * descending when upper): X_b = op(Inv_b) B_b, then the remaining rows of its
 * super-block of TRSM_SB blocks are updated with X_b and, after the super-
 * block's last block, the trailing rows with the whole super-block's X (k up
 * to 1024: fewer, deeper updates), all with the cascaded GEMM
 * (orc_casc_gemm_ex: alpha 1, beta 0, then alpha -1, beta 1). */
void orc_casc_trsm(int uplo, int trans, int diag, int64_t m, int64_t n, double ah, double al,
                   const double* Ahi, const double* Alo, int64_t lda, double* Bhi, double* Blo,
                   int64_t ldb, int nthreads) {
  if (m == 0 || n == 0) return;
  if (!(ah == 1.0 && al == 0.0))
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j) {
        double rh = 0.0, rl = 0.0;
        if (!(ah == 0.0 && al == 0.0))
          orc_dd_mul(ah, al, Bhi[i * ldb + j], Blo[i * ldb + j], &rh, &rl);
        Bhi[i * ldb + j] = rh;
        Blo[i * ldb + j] = rl;
      }
  if (ah == 0.0 && al == 0.0) return;
  const int eff_lower = (uplo == 0) != (trans == 1);
  const int64_t nblk = (m + TRSM_NB - 1) / TRSM_NB;
  double* Ihi = (double*)malloc(sizeof(double) * (size_t)(nblk * TRSM_NB * TRSM_NB));
  double* Ilo = (double*)malloc(sizeof(double) * (size_t)(nblk * TRSM_NB * TRSM_NB));
  double* Th = (double*)malloc(sizeof(double) * (size_t)(TRSM_NB * n));
  double* Tl = (double*)malloc(sizeof(double) * (size_t)(TRSM_NB * n));
  orc_trsm_diag_inv(uplo, diag, m, Ahi, Alo, lda, Ihi, Ilo);
  for (int64_t s = 0; s < nblk; ++s) {
    const int64_t b = eff_lower ? s : nblk - 1 - s;
    const int64_t r0 = b * TRSM_NB, nb = (m - r0) < TRSM_NB ? (m - r0) : TRSM_NB;
    const int64_t r1 = r0 + nb;
    /* X_b = op(Inv_b) B_b (into T, then back into B_b) */
    orc_casc_gemm_ex(trans, 0, nb, n, nb, 1.0, 0.0, Ihi + b * TRSM_NB * TRSM_NB,
                     Ilo + b * TRSM_NB * TRSM_NB, TRSM_NB, Bhi + r0 * ldb, Blo + r0 * ldb, ldb,
                     0.0, 0.0, Th, Tl, n, NULL, nthreads);
    for (int64_t i = 0; i < nb; ++i)
      for (int64_t j = 0; j < n; ++j) {
        Bhi[(r0 + i) * ldb + j] = Th[i * n + j];
        Blo[(r0 + i) * ldb + j] = Tl[i * n + j];
      }
    /* updates: inside the super-block (TRSM_SB blocks) with this block's X,
     * then, after its last block, the trailing rows with the whole super-block */
    const int64_t S0 = (b / TRSM_SB) * TRSM_SB * TRSM_NB;
    const int64_t S1 = S0 + TRSM_SB * TRSM_NB < m ? S0 + TRSM_SB * TRSM_NB : m;
    if (eff_lower) {
      orc_trsm_update(trans, r1, S1, r0, r1, n, Ahi, Alo, lda, Bhi, Blo, ldb, nthreads, 0);
      if (r1 == S1) orc_trsm_update(trans, S1, m, S0, S1, n, Ahi, Alo, lda, Bhi, Blo, ldb, nthreads, 0);
    } else {
      orc_trsm_update(trans, S0, r0, r0, r1, n, Ahi, Alo, lda, Bhi, Blo, ldb, nthreads, 0);
      if (r0 == S0) orc_trsm_update(trans, 0, S0, S0, S1, n, Ahi, Alo, lda, Bhi, Blo, ldb, nthreads, 0);
    }
  }
  free(Ihi);
  free(Ilo);
  free(Th);
  free(Tl);
}

/* ------------------------------------------------------------------------- */
/* NEXT-4, more level-3 BLAS as GEMMs ("All Level-3 BLAS         */
/* algorithms can be written in terms of GEMM"; R28, R29).          */
/* orc_expand: the dense n x n matrix of a stored triangle (uplo 0 lower / 1  */
/* upper): mode 0 symmetric (mirror), mode 1 triangular (other triangle 0;    */
/* unit: diagonal (1, 0), not read).                                          */
/* ------------------------------------------------------------------------- */
static void orc_expand(int64_t n, int uplo, int mode, int unit, const double* Ahi,
                       const double* Alo, int64_t lda, double* Fhi, double* Flo) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const int stored = uplo == 0 ? j <= i : j >= i;
      double h = 0.0, l = 0.0;
      if (mode == 1 && i == j && unit) {
        h = 1.0;
      } else if (stored) {
        h = Ahi[i * lda + j];
        l = Alo[i * lda + j];
      } else if (mode == 0) {
        h = Ahi[j * lda + i];
        l = Alo[j * lda + i];
      }
      Fhi[i * n + j] = h;
      Flo[i * n + j] = l;
    }
}

/* SYMM: C := alpha A B + beta C (side 0) or alpha B A + beta C (side 1), A     */
/* symmetric from its uplo triangle: the GEMM of the symmetric matrix.         */
void orc_casc_symm(int side, int uplo, int64_t m, int64_t n, double ah, double al,
                   const double* Ahi, const double* Alo, int64_t lda, const double* Bhi,
                   const double* Blo, int64_t ldb, double bh, double bl, double* Chi, double* Clo,
                   int64_t ldc, uint8_t* flags, int nthreads) {
  const int64_t ka = side == 0 ? m : n;
  double* F = (double*)malloc(sizeof(double) * 2 * (size_t)(ka * ka > 0 ? ka * ka : 1));
  orc_expand(ka, uplo, 0, 0, Ahi, Alo, lda, F, F + ka * ka);
  if (side == 0)
    orc_casc_gemm_ex(0, 0, m, n, m, ah, al, F, F + ka * ka, ka, Bhi, Blo, ldb, bh, bl, Chi, Clo,
                     ldc, flags, nthreads);
  else
    orc_casc_gemm_ex(0, 0, m, n, n, ah, al, Bhi, Blo, ldb, F, F + ka * ka, ka, bh, bl, Chi, Clo,
                     ldc, flags, nthreads);
  free(F);
}

/* TRMM: B := alpha op(A) B (side 0) or alpha B op(A) (side 1), A triangular:  */
/* the GEMM of the triangular matrix (other triangle zero), into B.            */
void orc_casc_trmm(int side, int uplo, int trans, int diag, int64_t m, int64_t n, double ah,
                   double al, const double* Ahi, const double* Alo, int64_t lda, double* Bhi,
                   double* Blo, int64_t ldb, int nthreads) {
  const int64_t ka = side == 0 ? m : n;
  double* F = (double*)malloc(sizeof(double) * 2 * (size_t)(ka * ka > 0 ? ka * ka : 1));
  double* T = (double*)malloc(sizeof(double) * 2 * (size_t)(m * n > 0 ? m * n : 1));
  orc_expand(ka, uplo, 1, diag, Ahi, Alo, lda, F, F + ka * ka);
  if (side == 0)
    orc_casc_gemm_ex(trans, 0, m, n, m, ah, al, F, F + ka * ka, ka, Bhi, Blo, ldb, 0.0, 0.0, T,
                     T + m * n, n, NULL, nthreads);
  else
    orc_casc_gemm_ex(0, trans, m, n, n, ah, al, Bhi, Blo, ldb, F, F + ka * ka, ka, 0.0, 0.0, T,
                     T + m * n, n, NULL, nthreads);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      Bhi[i * ldb + j] = T[i * n + j];
      Blo[i * ldb + j] = T[m * n + i * n + j];
    }
  free(F);
  free(T);
}

/* Right-side TRSM: X op(A) = alpha B  <=>  op(A)^T X^T = alpha B^T: the left   */
/* TRSM (orc_casc_trsm, reading R27) with the opposite transposition, on the   */
/* transposed right-hand sides (a mathematical identity, not the GPU's         */
/* column-block algorithm).                                                    */
void orc_casc_trsm_right(int uplo, int trans, int diag, int64_t m, int64_t n, double ah,
                         double al, const double* Ahi, const double* Alo, int64_t lda,
                         double* Bhi, double* Blo, int64_t ldb, int nthreads) {
  if (m == 0 || n == 0) return;
  double* T = (double*)malloc(sizeof(double) * 2 * (size_t)(m * n));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      T[j * m + i] = Bhi[i * ldb + j];
      T[m * n + j * m + i] = Blo[i * ldb + j];
    }
  orc_casc_trsm(uplo, !trans, diag, n, m, ah, al, Ahi, Alo, lda, T, T + m * n, m, nthreads);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      Bhi[i * ldb + j] = T[j * m + i];
      Blo[i * ldb + j] = T[m * n + j * m + i];
    }
  free(T);
}

/* ------------------------------------------------------------------------- */
/* Plain FP64x2 triangular solve, the textbook column-by-column substitution  */
/* with no blocking (the reference the blocked orc_casc_trsm is checked        */
/* against, independently of its block sizes): op(A) X = alpha B, left side;  */
/* for each column j, rows in the order of op(A)'s triangle:                  */
/*   x_i = (alpha b_i - sum_l op(A)_il x_l) / op(A)_ii   (l ascending),        */
/* every operation an FP64x2 one (orc_dd_mul, orc_dd_add, orc_dd_div).          */
/* ------------------------------------------------------------------------- */
void orc_dd_trsm_plain(int uplo, int trans, int diag, int64_t m, int64_t n, double ah, double al,
                       const double* Ahi, const double* Alo, int64_t lda, double* Bhi,
                       double* Blo, int64_t ldb) {
  const int lower = (uplo == 0) != (trans != 0); /* op(A) lower triangular */
  for (int64_t j = 0; j < n; ++j)
    for (int64_t t = 0; t < m; ++t) {
      const int64_t i = lower ? t : m - 1 - t;
      double sh, sl;
      orc_dd_mul(ah, al, Bhi[i * ldb + j], Blo[i * ldb + j], &sh, &sl);
      const int64_t l0 = lower ? 0 : i + 1, l1 = lower ? i : m;
      for (int64_t l = l0; l < l1; ++l) {
        const int64_t o = trans ? l * lda + i : i * lda + l; /* op(A)_il */
        double ph, pl;
        orc_dd_mul(Ahi[o], Alo[o], Bhi[l * ldb + j], Blo[l * ldb + j], &ph, &pl);
        orc_dd_add(sh, sl, -ph, -pl, &sh, &sl);
      }
      if (diag == 0)
        orc_dd_div(sh, sl, Ahi[i * lda + i], Alo[i * lda + i], &sh, &sl);
      Bhi[i * ldb + j] = sh;
      Blo[i * ldb + j] = sl;
    }
}

