/*
 * casc_i8_oracle.c — CPU ORACLE for the INT8 cascade of an FP64x2 GEMM
 * (NEXT-3; arXiv 2303.04353 §6 "FP64x2 in terms of INT8",
 * P:L3753-3754, and "FP64 in terms of INT8").
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library. The
 * product path (paper_2303_04353_b200/) never imports, links or executes it and
 * shares no code, header, table or constant generator with it.
 *
 * The paper only sketches this variant: the FP64x2 matrix is "converted into
 * fixed point numbers which can be stored in integers", cascaded into
 * "approximately 14 to 15 INT8 splits" with "about 105 to 120 INT8 multiplies"
 * (P:L3754), i.e. the y(y+1)/2 products A_i B_j with i + j < y, and "32-bit
 * accumulation" plays the role the 2^53 budget plays for the
 * FP64 cascade.  Everything the paper leaves open is fixed by the readings
 * R22-R26 in DESIGN.md §3; this file follows them step by step:
 *
 *   R22 panel      k_C8 = 8192: one scale exponent per (row, panel) of A and
 *                  (column, panel) of B, e = frexp exponent of max|hi| (the
 *                  FP64 cascade's R1), and every bin of a panel is an exact
 *                  int32 sum (y * 8192 * 2^14 < 2^31 for y <= 15).
 *   R23 slices     F = 6 + 8(y-1) fraction bits; X = rint(hi 2^(F-e)) +
 *                  rint(lo 2^(F-e)) (an exact integer, each limb rounded to
 *                  nearest-even); the slices are the balanced base-256 digits of
 *                  X: d_(y-1) .. d_1 in [-128, 127], d_0 in [-64, 64]; value of
 *                  slice t is d_t 2^(e - 6 - 8t).
 *   R24 products   bin_s = sum_p sum_(i+j=s) dA_i dB_j for s = 0 .. y-1 (the
 *                  paper's triangle of y(y+1)/2 products), exact.
 *   R25 combine    (revised twice; DESIGN.md §3 R25) the panel value T is the
 *                  FP64x2 number nearest the panel's exact product
 *                  x = sum_s bin_s 2^(e+f-12-8s):  T.hi = RN(x), T.lo = RN(x - T.hi)
 *                  (IEEE round to nearest even, subnormals included, RN(0) = +0);
 *                  then C = T over the first panel and C = DDadd(C, T) over the
 *                  following ones, in ascending order (FP64x2; the FP64
 *                  cascade's per-panel T of P:L3295).  Evaluated here with a plain
 *                  sign-magnitude big integer and ldexp of a <= 53-bit integer.
 *   R26 detector   flag |= (|T.hi| <= kp 2^(e+f-50)): the panel's exact-integer
 *                  product lost at least ~50 bits against its operand scale.
 *                  The paper's test "bin 0 is zero" asks whether the
 *                  exact leading 22 x 22-bit products cancel; balanced int8
 *                  slices are not symmetric under negation (the digit -128 has
 *                  no negative), so exact zeros of leading bins do not survive
 *                  x, -x pairs and the test is taken on the panel value instead.
 * Pins: tests/test_i8_oracle_pins.py (Fraction brute force; the all-diagonals
 * product equals the exact product of the reconstructed slices; the north-star
 * bound against ORACLE-EXACT; scaling neutrality; the detector cases).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define KC8 8192 /* reading R22 */

/* From casc_oracle.c (same library, same translation rules). */
void orc_two_sum(double a, double b, double* s, double* e);
void orc_dd_add(double xh, double xl, double yh, double yl, double* rh, double* rl);
int orc_scale_exponent(const double* hi, int64_t n, int64_t stride);

int orc_i8_panel(void) { return KC8; }

/* Reading R23: the y int8 slices of one FP64x2 value with scale exponent e. */
void orc_i8_split_scalar(double hi, double lo, int e, int y, int8_t* d) {
  const int F = 6 + 8 * (y - 1);
  __int128 X = (__int128)rint(ldexp(hi, F - e)) + (__int128)rint(ldexp(lo, F - e));
  for (int t = y - 1; t >= 1; --t) {
    int8_t b = (int8_t)(uint8_t)(X & 0xff); /* low byte as a signed digit */
    d[t] = b;
    X = (X - b) / 256; /* exact */
  }
  d[0] = (int8_t)X;
}

/* Split `rows` vectors of length kp: element (r, p) at x[r*ld + p*sk].
 * D is y x rows x kp (digit t of (r, p) at D[(t*rows + r)*kp + p]), ex[r] the
 * scale exponent of vector r (reading R1). */
void orc_i8_split_rows(int64_t rows, int64_t kp, const double* hi, const double* lo, int64_t ld,
                       int64_t sk, int y, int8_t* D, int32_t* ex) {
  int8_t d[16];
  for (int64_t r = 0; r < rows; ++r) {
    const int e = orc_scale_exponent(hi + r * ld, kp, sk);
    ex[r] = e;
    for (int64_t p = 0; p < kp; ++p) {
      orc_i8_split_scalar(hi[r * ld + p * sk], lo[r * ld + p * sk], e, y, d);
      for (int t = 0; t < y; ++t) D[((int64_t)t * rows + r) * kp + p] = d[t];
    }
  }
}

/* Reading R24: bins of one panel, exact (int64).  DA: y x m x kp, DB: y x n x kp.
 * nbins = y (the paper's triangle) or 2y-1 (every product, for the pins). */
void orc_i8_panel_bins(int64_t m, int64_t n, int64_t kp, int y, const int8_t* DA,
                       const int8_t* DB, int nbins, int64_t* bins) {
  for (int s = 0; s < nbins; ++s)
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j) {
        int64_t acc = 0;
        for (int a = 0; a < y; ++a) {
          const int b = s - a;
          if (b < 0 || b >= y) continue;
          const int8_t* x = DA + ((int64_t)a * m + i) * kp;
          const int8_t* z = DB + ((int64_t)b * n + j) * kp;
          for (int64_t p = 0; p < kp; ++p) acc += (int64_t)x[p] * (int64_t)z[p];
        }
        bins[((int64_t)s * m + i) * n + j] = acc;
      }
}

/* Reading R25: exact FP64x2 value of a group of nb <= 4 consecutive bins. */
void orc_i8_group_value(const int64_t* b, int nb, double* hi, double* lo) {
  int64_t V = 0;
  for (int u = 0; u < nb; ++u) V = V * 256 + b[u];
  const double h = (double)V; /* round to nearest even */
  *hi = h;
  *lo = (double)(V - (int64_t)h);
}

/* ---- Reading R25 (rev. 2): the FP64x2 number nearest an exact integer x 2^w.
 * Magnitudes are little-endian base-2^32 limbs, NL of them (> 160 bits). */
#define NL 8
static int big_bit(const uint32_t* M, int i) {
  return (i >= 0 && i < 32 * NL) ? (int)((M[i / 32] >> (i % 32)) & 1u) : 0;
}
static int big_bitlen(const uint32_t* M) { /* index of the top set bit + 1; 0 for M = 0 */
  for (int i = 32 * NL - 1; i >= 0; --i)
    if (big_bit(M, i)) return i + 1;
  return 0;
}
static int big_cmp(const uint32_t* a, const uint32_t* b) {
  for (int l = NL - 1; l >= 0; --l)
    if (a[l] != b[l]) return a[l] < b[l] ? -1 : 1;
  return 0;
}
static void big_sub(uint32_t* a, const uint32_t* b) { /* a -= b, requires a >= b */
  int64_t borrow = 0;
  for (int l = 0; l < NL; ++l) {
    int64_t d = (int64_t)a[l] - (int64_t)b[l] - borrow;
    borrow = d < 0;
    a[l] = (uint32_t)(d + (borrow ? ((int64_t)1 << 32) : 0));
  }
}
static void big_add_u64_shifted(uint32_t* a, uint64_t v, int sh) { /* a += v 2^sh */
  for (int i = 0; i < 64; ++i)
    if ((v >> i) & 1u) { /* add 2^(sh + i) */
      int j = sh + i;
      uint64_t carry = 1;
      for (int l = j / 32; l < NL && carry; ++l) {
        const uint64_t t = (uint64_t)a[l] + (carry << (l == j / 32 ? j % 32 : 0));
        a[l] = (uint32_t)t;
        carry = t >> 32;
      }
    }
}

/* RN(+-M 2^w) in IEEE double (ties to even; subnormals; overflow -> inf;
 * RN(0) = +0).  *R / *rneg receive the exact remainder M 2^w - |RN| as a
 * magnitude and a sign relative to the input's sign. */
static double rn_big(const uint32_t* M, int w, int neg, uint32_t* R, int* rneg) {
  memset(R, 0, sizeof(uint32_t) * NL);
  *rneg = 0;
  const int len = big_bitlen(M);
  if (len == 0) return 0.0;
  const int p = len - 1;                       /* x in [2^(p+w), 2^(p+w+1)) */
  int c = p - 52;                              /* keep 53 significant bits ... */
  if (c < -1074 - w) c = -1074 - w;            /* ... or the subnormal grid 2^-1074 */
  uint64_t q = 0;
  int up = 0;
  if (c <= 0) {
    for (int i = 0; i <= p; ++i) q |= (uint64_t)big_bit(M, i) << i; /* exact */
  } else {
    for (int i = c; i <= p; ++i) q |= (uint64_t)big_bit(M, i) << (i - c);
    const int guard = big_bit(M, c - 1);
    int sticky = 0;
    for (int i = 0; i < c - 1; ++i) sticky |= big_bit(M, i);
    up = guard && (sticky || (q & 1u));
    /* remainder: the bits below c, or 2^c minus them when rounded up */
    uint32_t low[NL];
    memset(low, 0, sizeof low);
    for (int i = 0; i < c && i < 32 * NL; ++i)
      if (big_bit(M, i)) low[i / 32] |= 1u << (i % 32);
    if (up) {
      uint32_t two_c[NL];
      memset(two_c, 0, sizeof two_c);
      if (c < 32 * NL) two_c[c / 32] = 1u << (c % 32);
      big_sub(two_c, low);
      memcpy(R, two_c, sizeof two_c);
      *rneg = 1;
    } else {
      memcpy(R, low, sizeof low);
    }
    q += (uint64_t)up;
  }
  const double v = ldexp((double)q, w + (c > 0 ? c : 0)); /* q <= 2^53: exact */
  return neg ? -v : v;
}

/* T of one element: bins b[0..y-1] (exact), x = sum_s b[s] 2^(w0 + 8(y-1-s)). */
void orc_i8_panel_value(const int64_t* b, int y, int w0, double* hi, double* lo) {
  uint32_t P[NL], N[NL], R[NL];
  memset(P, 0, sizeof P);
  memset(N, 0, sizeof N);
  for (int s = 0; s < y; ++s) {
    if (b[s] > 0) big_add_u64_shifted(P, (uint64_t)b[s], 8 * (y - 1 - s));
    if (b[s] < 0) big_add_u64_shifted(N, (uint64_t)(-b[s]), 8 * (y - 1 - s));
  }
  int neg = 0;
  if (big_cmp(P, N) >= 0) {
    big_sub(P, N);
  } else {
    big_sub(N, P);
    memcpy(P, N, sizeof P);
    neg = 1;
  }
  int rneg;
  *hi = rn_big(P, w0, neg, R, &rneg);
  uint32_t R2[NL];
  int r2neg;
  *lo = rn_big(R, w0, neg ^ rneg, R2, &r2neg);
}

/* ORACLE-I8CASCADE: C := A B (FP64x2) through y int8 slices per operand.
 * Row-major A (m x k, lda), B (k x n, ldb), C (m x n, ldc); flags m x n
 * (ld = n, nullable).  k == 0 gives C = 0, flags = 0. */
void orc_i8_casc_gemm(int64_t m, int64_t n, int64_t k, const double* Ahi, const double* Alo,
                      int64_t lda, const double* Bhi, const double* Blo, int64_t ldb, int y,
                      double* Chi, double* Clo, int64_t ldc, uint8_t* flags, int nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
  (void)nthreads;
#endif
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      Chi[i * ldc + j] = 0.0;
      Clo[i * ldc + j] = 0.0;
      if (flags) flags[i * n + j] = 0;
    }
  const int64_t P = (k + KC8 - 1) / KC8;
  for (int64_t q = 0; q < P; ++q) {
    const int64_t k0 = q * KC8;
    const int64_t kp = (k - k0 < KC8) ? k - k0 : KC8;
    int8_t* DA = (int8_t*)malloc((size_t)y * m * kp + 1);
    int8_t* DB = (int8_t*)malloc((size_t)y * n * kp + 1);
    int32_t* e = (int32_t*)malloc(sizeof(int32_t) * (m + 1));
    int32_t* f = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
    /* rows of A: stride 1 along k; columns of B: stride ldb along k */
    orc_i8_split_rows(m, kp, Ahi + k0, Alo + k0, lda, 1, y, DA, e);
    orc_i8_split_rows(n, kp, Bhi + k0 * ldb, Blo + k0 * ldb, 1, ldb, y, DB, f);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int64_t i = 0; i < m; ++i) {
      int64_t b[16];
      for (int64_t j = 0; j < n; ++j) {
        /* bins of element (i, j), exact (reading R24) */
        for (int s = 0; s < y; ++s) {
          int64_t acc = 0;
          for (int a = 0; a <= s; ++a) {
            const int8_t* x = DA + ((int64_t)a * m + i) * kp;
            const int8_t* z = DB + ((int64_t)(s - a) * n + j) * kp;
            for (int64_t p = 0; p < kp; ++p) acc += (int64_t)x[p] * (int64_t)z[p];
          }
          b[s] = acc;
        }
        /* reading R25 (rev. 2): T = the FP64x2 number nearest the exact panel
         * product */
        double th, tl;
        orc_i8_panel_value(b, y, e[i] + f[j] - 12 - 8 * (y - 1), &th, &tl);
        /* reading R26 */
        if (flags && fabs(th) <= ldexp((double)kp, e[i] + f[j] - 50)) flags[i * n + j] = 1;
        double ch = th, cl = tl; /* C = T_0, then C = DDadd(C, T_q) */
        if (q > 0) orc_dd_add(Chi[i * ldc + j], Clo[i * ldc + j], th, tl, &ch, &cl);
        Chi[i * ldc + j] = ch;
        Clo[i * ldc + j] = cl;
      }
    }
    free(DA);
    free(DB);
    free(e);
    free(f);
  }
}

/* NEXT-4 on the INT8 cascade: C := (alpha (x) P) (+) (beta (x) C), P = op(A) op(B)
 * through the INT8 cascade (reading R21; the same update sequence as the FP64
 * cascade's orc_casc_gemm_ex).  A stored m x k (transa = 0, lda) or k x m
 * (transa = 1); B stored k x n (transb = 0, ldb) or n x k (transb = 1).
 * beta == 0: C is not read; k == 0 or alpha == 0: C := beta (x) C, flags := 0. */
void orc_dd_mul(double xh, double xl, double yh, double yl, double* rh, double* rl);
void orc_i8_casc_gemm_ex(int transa, int transb, int64_t m, int64_t n, int64_t k, double ah,
                         double al, const double* Ahi, const double* Alo, int64_t lda,
                         const double* Bhi, const double* Blo, int64_t ldb, double bh, double bl,
                         double* Chi, double* Clo, int64_t ldc, uint8_t* flags, int y,
                         int nthreads) {
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
  double* p_h = (double*)calloc((size_t)(m * n), sizeof(double));
  double* p_l = (double*)calloc((size_t)(m * n), sizeof(double));
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
  orc_i8_casc_gemm(m, n, k, a_h, a_l, k, b_h, b_l, n, y, p_h, p_l, n, flags, nthreads);
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

/* NEXT-4 SYRK on the INT8 cascade: by definition the lower
 * (uplo 0) / upper (uplo 1) triangle of orc_i8_casc_gemm_ex(trans, !trans, A,
 * A); the other triangle of C and flags (n x n, nullable) is left as it is. */
void orc_i8_casc_syrk(int uplo, int trans, int64_t n, int64_t k, double ah, double al,
                      const double* Ahi, const double* Alo, int64_t lda, double bh, double bl,
                      double* Chi, double* Clo, int64_t ldc, uint8_t* flags, int y,
                      int nthreads) {
  double* Th = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
  double* Tl = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
  uint8_t* Tf = (uint8_t*)calloc((size_t)(n * n + 1), 1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      Th[i * n + j] = Chi[i * ldc + j];
      Tl[i * n + j] = Clo[i * ldc + j];
    }
  orc_i8_casc_gemm_ex(trans, !trans, n, n, k, ah, al, Ahi, Alo, lda, Ahi, Alo, lda, bh, bl, Th,
                      Tl, n, Tf, y, nthreads);
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

/* NEXT-4 TRSM on the INT8 cascade (reading R27 with the INT8 cascade as the
 * GEMM): the blocked solve of orc_casc_trsm with orc_i8_casc_gemm_ex (y slices)
 * for X_b = op(Inv_b) B_b and the updates; same diagonal-block inverses. */
#define I8_TRSM_NB 256
void orc_trsm_diag_inv(int uplo, int diag, int64_t m, const double* Ahi, const double* Alo,
                       int64_t lda, double* Ihi, double* Ilo);
void orc_trsm_update(int trans, int64_t R0, int64_t R1, int64_t C0, int64_t C1, int64_t n,
                     const double* Ahi, const double* Alo, int64_t lda, double* Bhi, double* Blo,
                     int64_t ldb, int nthreads, int i8);
void orc_i8_casc_trsm(int uplo, int trans, int diag, int64_t m, int64_t n, double ah, double al,
                      const double* Ahi, const double* Alo, int64_t lda, double* Bhi, double* Blo,
                      int64_t ldb, int y, int nthreads) {
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
  const int64_t nblk = (m + I8_TRSM_NB - 1) / I8_TRSM_NB;
  double* Ihi = (double*)malloc(sizeof(double) * (size_t)(nblk * I8_TRSM_NB * I8_TRSM_NB));
  double* Ilo = (double*)malloc(sizeof(double) * (size_t)(nblk * I8_TRSM_NB * I8_TRSM_NB));
  double* Th = (double*)malloc(sizeof(double) * (size_t)(I8_TRSM_NB * n));
  double* Tl = (double*)malloc(sizeof(double) * (size_t)(I8_TRSM_NB * n));
  orc_trsm_diag_inv(uplo, diag, m, Ahi, Alo, lda, Ihi, Ilo);
  for (int64_t s = 0; s < nblk; ++s) {
    const int64_t b = eff_lower ? s : nblk - 1 - s;
    const int64_t r0 = b * I8_TRSM_NB, nb = (m - r0) < I8_TRSM_NB ? (m - r0) : I8_TRSM_NB;
    const int64_t r1 = r0 + nb;
    orc_i8_casc_gemm_ex(trans, 0, nb, n, nb, 1.0, 0.0, Ihi + b * I8_TRSM_NB * I8_TRSM_NB,
                        Ilo + b * I8_TRSM_NB * I8_TRSM_NB, I8_TRSM_NB, Bhi + r0 * ldb,
                        Blo + r0 * ldb, ldb, 0.0, 0.0, Th, Tl, n, NULL, y, nthreads);
    for (int64_t i = 0; i < nb; ++i)
      for (int64_t j = 0; j < n; ++j) {
        Bhi[(r0 + i) * ldb + j] = Th[i * n + j];
        Blo[(r0 + i) * ldb + j] = Tl[i * n + j];
      }
    const int64_t S0 = (b / 4) * 4 * I8_TRSM_NB;
    const int64_t S1 = S0 + 4 * I8_TRSM_NB < m ? S0 + 4 * I8_TRSM_NB : m;
    if (eff_lower) {
      orc_trsm_update(trans, r1, S1, r0, r1, n, Ahi, Alo, lda, Bhi, Blo, ldb, nthreads, y);
      if (r1 == S1) orc_trsm_update(trans, S1, m, S0, S1, n, Ahi, Alo, lda, Bhi, Blo, ldb, nthreads, y);
    } else {
      orc_trsm_update(trans, S0, r0, r0, r1, n, Ahi, Alo, lda, Bhi, Blo, ldb, nthreads, y);
      if (r0 == S0) orc_trsm_update(trans, 0, S0, S0, S1, n, Ahi, Alo, lda, Bhi, Blo, ldb, nthreads, y);
    }
  }
  free(Ihi);
  free(Ilo);
  free(Th);
  free(Tl);
}
