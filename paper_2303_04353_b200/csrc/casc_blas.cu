// casc_blas.cu — BLAS-style generality around the cascaded GEMM:
// the degenerate updates of C := alpha op(A) op(B) + beta C that need no
// product (k == 0 or alpha == 0): C := beta (x) C in FP64x2, flags := 0.
// The general case runs in the fused kernel (alpha/beta applied at each tile's
// last panel, casc_gemm.cu) after transposed splits (casc_split.cu).
#include <cuda_runtime.h>

#include "casc_dd.cuh"
#include "casc_layout.cuh"

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

// Split mode reduction (small problems, casc_gemm.cu item_coords): C := T_0 (+)
// T_1 (+) ... (+) T_{P-1} in panel order -- the same FP64x2 additions, in the
// same order, as the fused kernel's per-panel accumulation -- flags := OR, then
// the optional BLAS update.
__global__ void __launch_bounds__(256) split_reduce_kernel(
    int P, int64_t m, int64_t n, const double* __restrict__ t_hi,
    const double* __restrict__ t_lo, const uint8_t* __restrict__ fbuf,
    double* __restrict__ C_hi, double* __restrict__ C_lo, int64_t ldc,
    uint8_t* __restrict__ flags, int ab, double ah, double al, double bh, double bl) {
  const int64_t mn = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < mn;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double th = t_hi[idx], tl = t_lo[idx];
    uint8_t fl = fbuf[idx];
    for (int q = 1; q < P; ++q) {
      dd_add(th, tl, t_hi[q * mn + idx], t_lo[q * mn + idx], th, tl);
      fl |= fbuf[q * mn + idx];
    }
    const int64_t i = idx / n, j = idx - (idx / n) * n;
    double* ch = C_hi + i * ldc + j;
    double* cl = C_lo + i * ldc + j;
    if (ab) apply_alpha_beta(th, tl, ah, al, bh, bl, ab == 2 ? *ch : 0.0, ab == 2 ? *cl : 0.0,
                             ab == 2);
    *ch = th;
    *cl = tl;
    if (flags) flags[idx] = fl;
  }
}

cudaError_t launch_split_reduce(int P, int64_t m, int64_t n, const double* t_hi,
                                const double* t_lo, const uint8_t* fbuf, double* C_hi,
                                double* C_lo, int64_t ldc, uint8_t* flags, int ab, double ah,
                                double al, double bh, double bl, int num_sms, cudaStream_t st) {
  const int64_t mn = m * n;
  if (mn == 0) return cudaSuccess;
  int64_t blocks = (mn + 255) / 256;
  if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
  split_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(P, m, n, t_hi, t_lo, fbuf, C_hi, C_lo, ldc,
                                                        flags, ab, ah, al, bh, bl);
  return cudaGetLastError();
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

}  // namespace casc
