// casc_blas.cu — BLAS-style generality around the cascaded GEMM:
// the degenerate updates of C := alpha op(A) op(B) + beta C that need no
// product (k == 0 or alpha == 0): C := beta (x) C in FP64x2, flags := 0.
// The general case runs in the fused kernel (alpha/beta applied at each tile's
// last panel, casc_gemm.cu) after transposed splits (casc_split.cu).
#include <cuda_runtime.h>

#include <algorithm>

#include "casc_dd.cuh"
#include "casc_layout.cuh"
#include "casc_ptx.cuh"

namespace casc {

// uplo: -1 every element; 0 / 1 only the lower / upper triangle (SYRK)
__global__ void __launch_bounds__(256) scale_c_kernel(int64_t m, int64_t n, double bh, double bl,
                                                      int use_beta, double* __restrict__ C_hi,
                                                      double* __restrict__ C_lo, int64_t ldc,
                                                      uint8_t* __restrict__ flags, int uplo) {
  const int64_t mn = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < mn;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / n, j = idx - (idx / n) * n;
    if ((uplo == 0 && j > i) || (uplo == 1 && j < i)) continue;
    double* ch = C_hi + i * ldc + j;
    double* cl = C_lo + i * ldc + j;
    if (use_beta) {
      double rh, rl;
      dd_mul(bh, bl, *ch, *cl, rh, rl);
      *ch = rh;
      *cl = rl;
    } else {
      *ch = 0.0;
      *cl = 0.0;
    }
    if (flags) flags[idx] = 0;
  }
}

// Split mode reduction (small problems, casc_gemm.cu item_coords): C := (0, 0)
// (+) T_0 (+) T_1 ... (+) T_{P-1} in panel order -- the same FP64x2 additions,
// in the same order, as the fused kernel's per-panel accumulation -- flags :=
// OR, then the optional BLAS update.  The panel sums are tile-major (the fused
// kernel's split-mode store): [q][tile mb*nblocks+nb][warp 0..7][element
// 0..15][lane 0..31], so consecutive threads read consecutive doubles.
__global__ void __launch_bounds__(256) split_reduce_kernel(
    int P, int64_t m, int64_t n, const double* __restrict__ t_hi,
    const double* __restrict__ t_lo, const uint8_t* __restrict__ fbuf,
    double* __restrict__ C_hi, double* __restrict__ C_lo, int64_t ldc,
    uint8_t* __restrict__ flags, int64_t ldf, int ab, double ah, double al, double bh, double bl) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the GEMM's panel sums are complete
  const int64_t nblocks = (n + TN - 1) / TN;
  const int64_t tot = (m + TM - 1) / TM * nblocks * (TM * TN);  // padded elements per panel
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x) {
    // the fused kernel's fragment coordinates of this slot
    const int64_t t = idx / (TM * TN);
    const int r = (int)(idx - t * (TM * TN));
    const int cw = r >> 9, e = (r >> 5) & 15, lane = r & 31;
    const int ms = e >> 2, ns = (e >> 1) & 1, ii = e & 1, g = lane >> 2, c = lane & 3;
    const int64_t i = (t / nblocks) * TM + (cw >> 2) * 32 + ms * 8 + g;
    const int64_t j = (t % nblocks) * TN + (cw & 3) * 16 + ns * 8 + 2 * c + ii;
    if (i >= m || j >= n) continue;
    double th = 0.0, tl = 0.0;  // C starts at (0, 0) (reading R10), as the fused kernel
    uint8_t fl = 0;
    for (int q = 0; q < P; ++q) {
      dd_add(th, tl, t_hi[q * tot + idx], t_lo[q * tot + idx], th, tl);
      fl |= fbuf[q * tot + idx];
    }
    double* ch = C_hi + i * ldc + j;
    double* cl = C_lo + i * ldc + j;
    if (ab) apply_alpha_beta(th, tl, ah, al, bh, bl, ab == 2 ? *ch : 0.0, ab == 2 ? *cl : 0.0,
                             ab == 2);
    *ch = th;
    *cl = tl;
    if (flags) flags[i * ldf + j] = fl;
  }
}

cudaError_t launch_split_reduce(int P, int64_t m, int64_t n, const double* t_hi,
                                const double* t_lo, const uint8_t* fbuf, double* C_hi,
                                double* C_lo, int64_t ldc, uint8_t* flags, int64_t ldf, int ab,
                                double ah, double al, double bh, double bl, int num_sms,
                                cudaStream_t st) {
  const int64_t tot = (m + TM - 1) / TM * ((n + TN - 1) / TN) * (TM * TN);
  if (m * n == 0) return cudaSuccess;
  int64_t blocks = (tot + 255) / 256;
  if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
  return launch_pdl(split_reduce_kernel, dim3((unsigned)blocks), dim3(256), 0, st, P, m, n, t_hi,
                    t_lo, fbuf, C_hi, C_lo, ldc, flags, ldf, ab, ah, al, bh, bl);
}

cudaError_t launch_scale_c_uplo(int64_t m, int64_t n, double bh, double bl, int use_beta,
                                double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
                                int num_sms, int uplo, cudaStream_t st) {
  const int64_t mn = m * n;
  if (mn == 0) return cudaSuccess;
  int64_t blocks = (mn + 255) / 256;
  if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
  scale_c_kernel<<<(unsigned)blocks, 256, 0, st>>>(m, n, bh, bl, use_beta, C_hi, C_lo, ldc, flags,
                                                   uplo);
  return cudaGetLastError();
}

cudaError_t launch_scale_c(int64_t m, int64_t n, double bh, double bl, int use_beta, double* C_hi,
                           double* C_lo, int64_t ldc, uint8_t* flags, int num_sms,
                           cudaStream_t st) {
  return launch_scale_c_uplo(m, n, bh, bl, use_beta, C_hi, C_lo, ldc, flags, num_sms, -1, st);
}

// ---------------------------------------------------------------- TRSM (NEXT-4)
// Inverses of the TRSM_NB diagonal blocks of the triangular A (reading R27):
// CTA b inverts block b, thread j computes column j by FP64x2 substitution in
// the oracle's order (orc_trsm_diag_inv): bitwise the same inverse.  The
// inverse is written to Inv[b][TRSM_NB][TRSM_NB] (zeros outside the triangle);
// each thread reads back only its own column.
constexpr int TRSM_NB = 256;

__global__ void __launch_bounds__(TRSM_NB) trsm_diag_inv_kernel(
    int uplo, int diag, int64_t m, const double* __restrict__ A_hi,
    const double* __restrict__ A_lo, int64_t lda, double* __restrict__ I_hi,
    double* __restrict__ I_lo) {
  const int64_t b = blockIdx.x, r0 = b * TRSM_NB;
  const int nb = (int)min((int64_t)TRSM_NB, m - r0);
  const int j = threadIdx.x;
  double* yh = I_hi + b * TRSM_NB * TRSM_NB + j;  // column j: element l at yh[l * TRSM_NB]
  double* yl = I_lo + b * TRSM_NB * TRSM_NB + j;
  for (int i = 0; i < TRSM_NB; ++i) yh[i * TRSM_NB] = yl[i * TRSM_NB] = 0.0;
  if (j >= nb) return;
  const double* ah = A_hi + r0 * lda + r0;
  const double* al = A_lo + r0 * lda + r0;
  if (diag) {
    yh[j * TRSM_NB] = 1.0;
  } else {
    double qh, ql;
    dd_div(1.0, 0.0, ah[j * lda + j], al[j * lda + j], qh, ql);
    yh[j * TRSM_NB] = qh;
    yl[j * TRSM_NB] = ql;
  }
  const int step = uplo == 0 ? 1 : -1;
  for (int i = j + step; i >= 0 && i < nb; i += step) {
    double sh = 0.0, sl = 0.0;
    const int lo = uplo == 0 ? j : i + 1, hi = uplo == 0 ? i - 1 : j;
    for (int l = lo; l <= hi; ++l) {
      double ph, pl;
      dd_mul(ah[i * lda + l], al[i * lda + l], yh[l * TRSM_NB], yl[l * TRSM_NB], ph, pl);
      dd_add(sh, sl, ph, pl, sh, sl);
    }
    if (diag) {
      yh[i * TRSM_NB] = -sh;
      yl[i * TRSM_NB] = -sl;
    } else {
      double qh, ql;
      dd_div(-sh, -sl, ah[i * lda + i], al[i * lda + i], qh, ql);
      yh[i * TRSM_NB] = qh;
      yl[i * TRSM_NB] = ql;
    }
  }
}

cudaError_t launch_trsm_diag_inv(int uplo, int diag, int64_t m, const double* A_hi,
                                 const double* A_lo, int64_t lda, double* I_hi, double* I_lo,
                                 cudaStream_t st) {
  const int64_t nblk = (m + TRSM_NB - 1) / TRSM_NB;
  if (nblk == 0) return cudaSuccess;
  trsm_diag_inv_kernel<<<(unsigned)nblk, TRSM_NB, 0, st>>>(uplo, diag, m, A_hi, A_lo, lda, I_hi,
                                                           I_lo);
  return cudaGetLastError();
}

// flags |= f2 on one triangle of an n x n flag matrix (SYR2K, reading R30)
__global__ void __launch_bounds__(256) or_flags_kernel(int64_t n, int uplo,
                                                       uint8_t* __restrict__ flags,
                                                       const uint8_t* __restrict__ f2) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / n, j = idx - (idx / n) * n;
    if (uplo == 0 ? j <= i : j >= i) flags[idx] |= f2[idx];
  }
}

cudaError_t launch_or_flags(int64_t n, int uplo, uint8_t* flags, const uint8_t* f2, int num_sms,
                            cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n * n + 255) / 256, (int64_t)num_sms * 8);
  or_flags_kernel<<<(unsigned)blocks, 256, 0, st>>>(n, uplo, flags, f2);
  return cudaGetLastError();
}

// Test export of the exact power-of-two scaling (casc_debug_ldexp)
__global__ void __launch_bounds__(256) ldexp_kernel(int64_t count, const double* __restrict__ x,
                                                    const int32_t* __restrict__ n,
                                                    double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = ldexp_rn(x[i], n[i]);
}

cudaError_t launch_ldexp(int64_t count, const double* x, const int32_t* n, double* out,
                         cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 8);
  ldexp_kernel<<<(unsigned)blocks, 256, 0, st>>>(count, x, n, out);
  return cudaGetLastError();
}

}  // namespace casc
