// casc_split.cu — phase 1 of the cascaded FP64x2 GEMM: the split kernels.
//
// split_a_kernel / split_b_kernel turn each FP64x2 row segment of A (column
// segment of B) inside one 256-wide k panel into the paper's FP64 slices:
//   * scale exponent e = frexp exponent of max |hi| over the (row, panel)
//     ("smallest power of two greater than" the max; P:L1139;
//     P:L3862-3863; reading R1, R2);
//   * Appendix A conditional-free split, each limb separately:
//     v = limb 2^-e; s_t = (v + M_t) - M_t with M_t = 2^(53-c_t) + 2^(52-c_t);
//     v = (v - s_t) 2^(c_t); s_3 = v; chi_t = s_t(hi) + s_t(lo);
//   * for B also B4 = B2 + 2^-c2 B3, B5 = B1 + 2^-c1 B4, B6 = B0 + 2^-c0 B5
//     (reading R7);
//   * exact power-of-two pre-alignment so the GEMM can accumulate all ten
//     products straight into four bins: A2 x 2^(c0-c1),
//     B2 x 2^(c0-c1), B4 x 2^(c2-c0), B5 x 2^(c1+c2-2c0).
// Output goes straight into the GEMM's fragment-ordered packed layout
// (casc_layout.cuh).  HBM-bound: 16 B read and 32 B (A) / 56 B (B) written per
// element, all accesses in full 32-byte sectors, warp stores 256 B contiguous.
//
// One CTA = 256 threads = one 8-row (A) / 8-column (B) group x one panel.
// Thread (warp kq, lane = 4g + c) owns row/column g and k = 256q + 4(kq + 8 it) + c,
// it = 0..7, i.e. exactly the elements whose packed slots it writes.
#include <cuda_runtime.h>

#include "casc_layout.cuh"

namespace casc {

struct SplitConsts {
  double M[3];      // 2^(53-c_t) + 2^(52-c_t)
  double up[3];     // 2^(c_t)
  double b4f, b5f, b6f;              // 2^-c2, 2^-c1, 2^-c0
  double al_a2, al_b4, al_b5;        // 2^(c0-c1), 2^(c2-c0), 2^(c1+c2-2c0)
};

__host__ inline SplitConsts make_consts(Widths w) {
  SplitConsts s;
  const int c[3] = {w.c0, w.c1, w.c2};
  for (int t = 0; t < 3; ++t) {
    s.M[t] = ldexp(1.0, 53 - c[t]) + ldexp(1.0, 52 - c[t]);
    s.up[t] = ldexp(1.0, c[t]);
  }
  s.b4f = ldexp(1.0, -w.c2);
  s.b5f = ldexp(1.0, -w.c1);
  s.b6f = ldexp(1.0, -w.c0);
  s.al_a2 = ldexp(1.0, w.c0 - w.c1);
  s.al_b4 = ldexp(1.0, w.c2 - w.c0);
  s.al_b5 = ldexp(1.0, w.c1 + w.c2 - 2 * w.c0);
  return s;
}

// Appendix A, one limb.
// v = x 2^-e: one multiply by scale = 2^-e when that power is a normal double,
// else the exact ldexp (panel maxima >= 2^1023 or < 2^-1024; reading R16).
__device__ __forceinline__ void split_limb(double x, double scale, int ne, const SplitConsts& K,
                                           double s[4]) {
  double v = scale != 0.0 ? __dmul_rn(x, scale) : ldexp_rn_wide(x, ne);
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const double r = __dsub_rn(__dadd_rn(v, K.M[t]), K.M[t]);
    s[t] = r;
    v = __dmul_rn(__dsub_rn(v, r), K.up[t]);
  }
  s[3] = v;
}

// Max |hi| of the 8 rows (columns) g over the CTA's 256 k, then the exponent.
__device__ __forceinline__ int group_exponent(double mx, int g, int c, int kq) {
  __shared__ double smax[8][8];
  __shared__ int sexp[8];
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
  if (c == 0) smax[kq][g] = mx;
  __syncthreads();
  if (threadIdx.x < 8) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v = fmax(v, smax[w][threadIdx.x]);
    int e = 0;
    if (v != 0.0) frexp(v, &e);
    sexp[threadIdx.x] = e;
  }
  __syncthreads();
  return sexp[g];
}

// TRANS: A is given transposed (stored k x m, element (i, p) at A[p * lda + i]; BLAS op 'T')
template <bool TRANS>
__device__ __forceinline__ void split_a_body(
    const double* __restrict__ Ahi, const double* __restrict__ Alo, int64_t lda, int64_t m,
    int64_t k, const SplitConsts& K, uint8_t* __restrict__ packed, int64_t blk_bytes,
    int64_t exp_off, int64_t nks, int64_t rg) {
  const int t = threadIdx.x, lane = t & 31, kq = t >> 5;
  const int g = lane >> 2, c = lane & 3;
  // rg: 8-row group
  const int64_t mb = rg >> 3;
  const int within = (int)(rg & 7), mw = within >> 2, ms = within & 3;
  const int64_t row = rg * 8 + g;
  const int q = blockIdx.y;
  const int64_t k0 = (int64_t)q * KC;

  double h[8], l[8], mx = 0.0;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int64_t kk = k0 + 4 * (kq + 8 * it) + c;
    const bool ok = (row < m) && (kk < k);
    const int64_t off = TRANS ? kk * lda + row : row * lda + kk;
    h[it] = ok ? __ldg(Ahi + off) : 0.0;
    l[it] = ok ? __ldg(Alo + off) : 0.0;
    mx = fmax(mx, fabs(h[it]));
  }
  const int e = group_exponent(mx, g, c, kq);
  const double scale = (unsigned)(-e + 1022) <= 2045u ? pow2i(-e) : 0.0;  // 0: wide

  uint8_t* blk = packed + mb * blk_bytes;
  double* sl = reinterpret_cast<double*>(blk);
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int64_t ks = (int64_t)q * (KC / 4) + kq + 8 * it;
    if (ks >= nks) break;
    double sh[4], slo[4];
    split_limb(h[it], scale, -e, K, sh);
    split_limb(l[it], scale, -e, K, slo);
    double chi[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) chi[s] = __dadd_rn(sh[s], slo[s]);
    chi[2] = __dmul_rn(chi[2], K.al_a2);  // exact pre-alignment of A2
    double* dst = sl + ks * A_KSTEP + mw * 128 + ms * 32 + lane;
#pragma unroll
    for (int s = 0; s < 4; ++s) dst[s * 256] = chi[s];
  }
  if (kq == 0 && c == 0) {
    int32_t* ex = reinterpret_cast<int32_t*>(blk + exp_off);
    ex[q * TM + mw * 32 + ms * 8 + g] = e;
  }
}

// TRANS: B is given transposed (stored n x k, element (p, j) at B[j * ldb + p])
template <bool TRANS>
__device__ __forceinline__ void split_b_body(
    const double* __restrict__ Bhi, const double* __restrict__ Blo, int64_t ldb, int64_t n,
    int64_t k, const SplitConsts& K, uint8_t* __restrict__ packed, int64_t blk_bytes,
    int64_t exp_off, int64_t nks, int64_t cg) {
  const int t = threadIdx.x, lane = t & 31, kq = t >> 5;
  const int g = lane >> 2, c = lane & 3;
  // cg: 8-column group
  const int64_t nb = cg >> 3;
  const int within = (int)(cg & 7), nw = within >> 1, ns = within & 1;
  const int64_t col = cg * 8 + g;
  const int q = blockIdx.y;
  const int64_t k0 = (int64_t)q * KC;

  double h[8], l[8], mx = 0.0;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int64_t kk = k0 + 4 * (kq + 8 * it) + c;
    const bool ok = (col < n) && (kk < k);
    const int64_t off = TRANS ? col * ldb + kk : kk * ldb + col;
    h[it] = ok ? __ldg(Bhi + off) : 0.0;
    l[it] = ok ? __ldg(Blo + off) : 0.0;
    mx = fmax(mx, fabs(h[it]));
  }
  const int f = group_exponent(mx, g, c, kq);
  const double scale = (unsigned)(-f + 1022) <= 2045u ? pow2i(-f) : 0.0;  // 0: wide

  uint8_t* blk = packed + nb * blk_bytes;
  double* sl = reinterpret_cast<double*>(blk);
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int64_t ks = (int64_t)q * (KC / 4) + kq + 8 * it;
    if (ks >= nks) break;
    double sh[4], slo[4];
    split_limb(h[it], scale, -f, K, sh);
    split_limb(l[it], scale, -f, K, slo);
    double y[7];
#pragma unroll
    for (int s = 0; s < 4; ++s) y[s] = __dadd_rn(sh[s], slo[s]);
    y[4] = __dadd_rn(y[2], __dmul_rn(y[3], K.b4f));  // B4 = B2 + 2^-c2 B3
    y[5] = __dadd_rn(y[1], __dmul_rn(y[4], K.b5f));  // B5 = B1 + 2^-c1 B4
    y[6] = __dadd_rn(y[0], __dmul_rn(y[5], K.b6f));  // B6 = B0 + 2^-c0 B5
    y[2] = __dmul_rn(y[2], K.al_a2);                 // exact pre-alignments
    y[4] = __dmul_rn(y[4], K.al_b4);
    y[5] = __dmul_rn(y[5], K.al_b5);
    double* dst = sl + ks * B_KSTEP + nw * 64 + ns * 32 + lane;
#pragma unroll
    for (int s = 0; s < 7; ++s) dst[s * 256] = y[s];
  }
  if (kq == 0 && c == 0) {
    int32_t* ex = reinterpret_cast<int32_t*>(blk + exp_off);
    ex[q * TN + nw * 16 + ns * 8 + g] = f;
  }
}

template <bool TRANS>
__global__ void __launch_bounds__(256) split_a_kernel(
    const double* __restrict__ Ahi, const double* __restrict__ Alo, int64_t lda, int64_t m,
    int64_t k, SplitConsts K, uint8_t* __restrict__ packed, int64_t blk_bytes, int64_t exp_off,
    int64_t nks) {
  split_a_body<TRANS>(Ahi, Alo, lda, m, k, K, packed, blk_bytes, exp_off, nks, blockIdx.x);
}

template <bool TRANS>
__global__ void __launch_bounds__(256) split_b_kernel(
    const double* __restrict__ Bhi, const double* __restrict__ Blo, int64_t ldb, int64_t n,
    int64_t k, SplitConsts K, uint8_t* __restrict__ packed, int64_t blk_bytes, int64_t exp_off,
    int64_t nks) {
  split_b_body<TRANS>(Bhi, Blo, ldb, n, k, K, packed, blk_bytes, exp_off, nks, blockIdx.x);
}

// Both splits of one GEMM in ONE launch (the first ga row groups split A, the
// rest B's column groups): one launch and one tail instead of two, which
// matters for small problems.  Bitwise the two kernels above.
struct SplitABArgs {
  const double* Ahi;
  const double* Alo;
  int64_t lda, m;
  uint8_t* pa;
  int64_t a_blk, a_exp;
  const double* Bhi;
  const double* Blo;
  int64_t ldb, n;
  uint8_t* pb;
  int64_t b_blk, b_exp;
  int64_t k, nks, ga;
  SplitConsts K;
};
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) split_ab_kernel(const SplitABArgs a) {
  // the fused GEMM that follows may be scheduled now (PDL); it waits for this
  // grid's completion before it reads the packed slices
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if ((int64_t)blockIdx.x < a.ga)
    split_a_body<TA>(a.Ahi, a.Alo, a.lda, a.m, a.k, a.K, a.pa, a.a_blk, a.a_exp, a.nks,
                     blockIdx.x);
  else
    split_b_body<TB>(a.Bhi, a.Blo, a.ldb, a.n, a.k, a.K, a.pb, a.b_blk, a.b_exp, a.nks,
                     blockIdx.x - a.ga);
}

// ------------------------------------------------------------ debug export
// Packed -> canonical row-major slices in the paper's normalisation (undoing
// the exact pre-alignment), plus exponents [panel][row].  Test path only.
__global__ void unpack_a_kernel(const uint8_t* __restrict__ packed, int64_t m, int64_t k,
                                int64_t blk_bytes, int64_t exp_off, double un_a2,
                                double* __restrict__ out, int32_t* __restrict__ eout) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t P = panels_of(k);
  if (idx < m * k) {
    const int64_t i = idx / k, p = idx % k;
    const int64_t mb = i / TM, r = i % TM;
    const int g = r % 8, ms = (r % 32) / 8, mw = r / 32;
    const int64_t ks = p / 4;
    const int c = p % 4, lane = 4 * g + c;
    const double* sl = reinterpret_cast<const double*>(packed + mb * blk_bytes);
    for (int s = 0; s < 4; ++s) {
      double v = sl[ks * A_KSTEP + s * 256 + mw * 128 + ms * 32 + lane];
      if (s == 2) v = __dmul_rn(v, un_a2);
      out[s * m * k + i * k + p] = v;
    }
  }
  if (idx < P * m) {
    const int64_t q = idx / m, i = idx % m;
    const int32_t* ex = reinterpret_cast<const int32_t*>(packed + (i / TM) * blk_bytes + exp_off);
    eout[q * m + i] = ex[q * TM + i % TM];
  }
}

__global__ void unpack_b_kernel(const uint8_t* __restrict__ packed, int64_t k, int64_t n,
                                int64_t blk_bytes, int64_t exp_off, double un_b2, double un_b4,
                                double un_b5, double* __restrict__ out,
                                int32_t* __restrict__ fout) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t P = panels_of(k);
  if (idx < k * n) {
    const int64_t p = idx / n, j = idx % n;
    const int64_t nb = j / TN, cl = j % TN;
    const int g = cl % 8, ns = (cl % 16) / 8, nw = cl / 16;
    const int64_t ks = p / 4;
    const int c = p % 4, lane = 4 * g + c;
    const double* sl = reinterpret_cast<const double*>(packed + nb * blk_bytes);
    for (int s = 0; s < 7; ++s) {
      double v = sl[ks * B_KSTEP + s * 256 + nw * 64 + ns * 32 + lane];
      if (s == 2) v = __dmul_rn(v, un_b2);
      if (s == 4) v = __dmul_rn(v, un_b4);
      if (s == 5) v = __dmul_rn(v, un_b5);
      out[s * k * n + p * n + j] = v;
    }
  }
  if (idx < P * n) {
    const int64_t q = idx / n, j = idx % n;
    const int32_t* ex = reinterpret_cast<const int32_t*>(packed + (j / TN) * blk_bytes + exp_off);
    fout[q * n + j] = ex[q * TN + j % TN];
  }
}

// ------------------------------------------------------------ launchers
cudaError_t launch_split_a(const double* Ahi, const double* Alo, int64_t lda, int64_t m,
                           int64_t k, Widths w, void* packed, cudaStream_t st, bool trans) {
  const int64_t mpad = (m + TM - 1) / TM * TM;
  const int64_t P = panels_of(k);
  if (mpad == 0 || P == 0) return cudaSuccess;
  dim3 grid((unsigned)(mpad / 8), (unsigned)P);
  auto kern = trans ? split_a_kernel<true> : split_a_kernel<false>;
  kern<<<grid, 256, 0, st>>>(Ahi, Alo, lda, m, k, make_consts(w),
                                       static_cast<uint8_t*>(packed), a_block_bytes(k),
                                       a_exp_offset(k), kpad_of(k) / 4);
  return cudaGetLastError();
}

cudaError_t launch_split_b(const double* Bhi, const double* Blo, int64_t ldb, int64_t k,
                           int64_t n, Widths w, void* packed, cudaStream_t st, bool trans) {
  const int64_t npad = (n + TN - 1) / TN * TN;
  const int64_t P = panels_of(k);
  if (npad == 0 || P == 0) return cudaSuccess;
  dim3 grid((unsigned)(npad / 8), (unsigned)P);
  auto kern = trans ? split_b_kernel<true> : split_b_kernel<false>;
  kern<<<grid, 256, 0, st>>>(Bhi, Blo, ldb, n, k, make_consts(w),
                                       static_cast<uint8_t*>(packed), b_block_bytes(k),
                                       b_exp_offset(k), kpad_of(k) / 4);
  return cudaGetLastError();
}

cudaError_t launch_split_ab(const double* Ahi, const double* Alo, int64_t lda, int64_t m,
                            const double* Bhi, const double* Blo, int64_t ldb, int64_t n,
                            int64_t k, Widths w, void* pa, void* pb, cudaStream_t st, bool ta,
                            bool tb) {
  const int64_t mpad = (m + TM - 1) / TM * TM, npad = (n + TN - 1) / TN * TN;
  const int64_t P = panels_of(k);
  if ((mpad == 0 && npad == 0) || P == 0) return cudaSuccess;
  SplitABArgs a{Ahi, Alo, lda, m, static_cast<uint8_t*>(pa), a_block_bytes(k), a_exp_offset(k),
                Bhi, Blo, ldb, n, static_cast<uint8_t*>(pb), b_block_bytes(k), b_exp_offset(k),
                k, kpad_of(k) / 4, mpad / 8, make_consts(w)};
  dim3 grid((unsigned)(mpad / 8 + npad / 8), (unsigned)P);
  auto kern = ta ? (tb ? split_ab_kernel<true, true> : split_ab_kernel<true, false>)
                 : (tb ? split_ab_kernel<false, true> : split_ab_kernel<false, false>);
  kern<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_unpack_a(const void* packed, int64_t m, int64_t k, Widths w, double* out,
                            int32_t* eout, cudaStream_t st) {
  const int64_t tot = m * k > panels_of(k) * m ? m * k : panels_of(k) * m;
  if (tot == 0) return cudaSuccess;
  unpack_a_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
      static_cast<const uint8_t*>(packed), m, k, a_block_bytes(k), a_exp_offset(k),
      ldexp(1.0, w.c1 - w.c0), out, eout);
  return cudaGetLastError();
}

cudaError_t launch_unpack_b(const void* packed, int64_t k, int64_t n, Widths w, double* out,
                            int32_t* fout, cudaStream_t st) {
  const int64_t tot = k * n > panels_of(k) * n ? k * n : panels_of(k) * n;
  if (tot == 0) return cudaSuccess;
  unpack_b_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
      static_cast<const uint8_t*>(packed), k, n, b_block_bytes(k), b_exp_offset(k),
      ldexp(1.0, w.c1 - w.c0), ldexp(1.0, w.c0 - w.c2), ldexp(1.0, 2 * w.c0 - w.c1 - w.c2), out,
      fout);
  return cudaGetLastError();
}

}  // namespace casc
