// casc_level3.cu — more level-3 BLAS on the cascaded GEMM (NEXT-4; the paper:
// "All Level-3 BLAS algorithms can be written in terms of GEMM"):
//   casc_symm_fp64x2        C := alpha A B + beta C  /  alpha B A + beta C, A symmetric
//   casc_trmm_fp64x2        B := alpha op(A) B  /  alpha B op(A), A triangular
//   casc_trsm_fp64x2_right  X op(A) = alpha B (the right-side TRSM, column blocks)
// The symmetric / triangular operand is expanded from its stored triangle into a
// stream-ordered temporary by one HBM-bound kernel (16 B read + 16 B written per
// element, < 0.1% of the GEMM at 16384), after which the work is the cascaded
// GEMM of casc_gemm_fp64x2_ex (transposes read directly by its split kernels).
// TRMM's GEMM is banded: each tile's k range stops at op(A)'s zero triangle
// (GemmArgs::band), about half the GEMM's work.
// Readings R28 (SYMM / TRMM), R29 (right-side TRSM) and R30 (SYR2K) in DESIGN.md.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/casc.h"
#include "casc_layout.cuh"

namespace casc {
cudaError_t launch_trsm_diag_inv(int uplo, int diag, int64_t m, const double* A_hi,
                                 const double* A_lo, int64_t lda, double* I_hi, double* I_lo,
                                 cudaStream_t st);
cudaError_t launch_scale_c(int64_t m, int64_t n, double bh, double bl, int use_beta, double* C_hi,
                           double* C_lo, int64_t ldc, uint8_t* flags, int num_sms,
                           cudaStream_t st);
namespace host {
int device_check(int* sms);
int check_mat(const void* p, int64_t rows, int64_t cols, int64_t ld);
void set_launches(int n);
bool trsm_overlap(int64_t m, int64_t n, const double* A_hi, const double* A_lo, int64_t lda,
                  const double* B_hi, const double* B_lo, int64_t ldb);
int gemm_ex_band(int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha_hi,
                 double alpha_lo, const double* A_hi, const double* A_lo, int64_t lda,
                 const double* B_hi, const double* B_lo, int64_t ldb, double* C_hi, double* C_lo,
                 int64_t ldc, casc_stream_t stream, int band);
}  // namespace host

// Expand the stored triangle of an n x n FP64x2 matrix into a dense one (ld n):
// mode 0 symmetric (the other triangle mirrored), mode 1 triangular (the other
// triangle zero; unit != 0: diagonal (1, 0), not read).
__global__ void __launch_bounds__(256) tri_expand_kernel(int64_t n, int uplo, int mode, int unit,
                                                         const double* __restrict__ A_hi,
                                                         const double* __restrict__ A_lo,
                                                         int64_t lda, double* __restrict__ F_hi,
                                                         double* __restrict__ F_lo) {
  const int64_t nn = n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < nn;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / n, j = idx - (idx / n) * n;
    const bool stored = uplo == CASC_LOWER ? j <= i : j >= i;
    double h, l;
    if (mode == 1 && i == j && unit) {
      h = 1.0;
      l = 0.0;
    } else if (stored) {
      h = A_hi[i * lda + j];
      l = A_lo[i * lda + j];
    } else if (mode == 0) {
      h = A_hi[j * lda + i];
      l = A_lo[j * lda + i];
    } else {
      h = 0.0;
      l = 0.0;
    }
    F_hi[idx] = h;
    F_lo[idx] = l;
  }
}

static cudaError_t expand(int64_t n, int uplo, int mode, int unit, const double* A_hi,
                          const double* A_lo, int64_t lda, double* F_hi, double* F_lo, int sms,
                          cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  int64_t blocks = (n * n + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  tri_expand_kernel<<<(unsigned)blocks, 256, 0, st>>>(n, uplo, mode, unit, A_hi, A_lo, lda, F_hi,
                                                      F_lo);
  return cudaGetLastError();
}
}  // namespace casc

namespace {
inline cudaStream_t S3(casc_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }
inline int st3(cudaError_t e) { return e == cudaSuccess ? CASC_OK : CASC_ERR_CUDA; }
inline bool overlap3(const void* a, size_t an, const void* b, size_t bn) {
  if (!a || !b || an == 0 || bn == 0) return false;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
  return a0 < b0 + bn && b0 < a0 + an;
}
inline size_t ext3(int64_t rows, int64_t cols, int64_t ld) {
  return (rows <= 0 || cols <= 0) ? 0 : size_t((rows - 1) * ld + cols) * sizeof(double);
}
}  // namespace

extern "C" {

int casc_symm_fp64x2(int side, int uplo, int64_t m, int64_t n, double alpha_hi, double alpha_lo,
                     const double* A_hi, const double* A_lo, int64_t lda, const double* B_hi,
                     const double* B_lo, int64_t ldb, double beta_hi, double beta_lo,
                     double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
                     casc_stream_t stream) {
  casc::host::set_launches(0);
  if ((side != CASC_LEFT && side != CASC_RIGHT) || (uplo != CASC_LOWER && uplo != CASC_UPPER))
    return CASC_ERR_INVALID;
  if (m < 0 || n < 0) return CASC_ERR_INVALID;
  const int64_t ka = side == CASC_LEFT ? m : n;  // A is ka x ka
  const bool no_product = ka == 0 || (alpha_hi == 0.0 && alpha_lo == 0.0);
  int r;
  if (!no_product) {
    if ((r = casc::host::check_mat(A_hi, ka, ka, lda)) ||
        (r = casc::host::check_mat(A_lo, ka, ka, lda)) ||
        (r = casc::host::check_mat(B_hi, m, n, ldb)) || (r = casc::host::check_mat(B_lo, m, n, ldb)))
      return r;
  }
  if ((r = casc::host::check_mat(C_hi, m, n, ldc)) || (r = casc::host::check_mat(C_lo, m, n, ldc)))
    return r;
  if (!no_product) {
    const void* ins[4] = {A_hi, A_lo, B_hi, B_lo};
    const size_t ine[4] = {ext3(ka, ka, lda), ext3(ka, ka, lda), ext3(m, n, ldb), ext3(m, n, ldb)};
    void* outs[3] = {C_hi, C_lo, flags};
    const size_t oute[3] = {ext3(m, n, ldc), ext3(m, n, ldc), flags ? (size_t)(m * n) : 0};
    for (int o = 0; o < 3; ++o)
      for (int i = 0; i < 4; ++i)
        if (overlap3(outs[o], oute[o], ins[i], ine[i])) return CASC_ERR_INVALID;
  }
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = casc::host::device_check(&sms))) return r;
  const cudaStream_t st = S3(stream);
  if (no_product)  // C := beta C through the GEMM entry's own k == 0 path
    return casc_gemm_fp64x2_ex(CASC_OP_N, CASC_OP_N, m, n, 0, alpha_hi, alpha_lo, nullptr,
                               nullptr, 1, nullptr, nullptr, n, beta_hi, beta_lo, C_hi, C_lo, ldc,
                               flags, nullptr, 0, stream);
  double* F = nullptr;  // the symmetric A, dense: hi | lo
  if (cudaMallocAsync(reinterpret_cast<void**>(&F), (size_t)2 * ka * ka * sizeof(double), st) !=
      cudaSuccess)
    return CASC_ERR_CUDA;
  cudaError_t e = casc::expand(ka, uplo, 0, 0, A_hi, A_lo, lda, F, F + ka * ka, sms, st);
  r = st3(e);
  if (r == CASC_OK) {
    r = side == CASC_LEFT
            ? casc_gemm_fp64x2_ex(CASC_OP_N, CASC_OP_N, m, n, m, alpha_hi, alpha_lo, F,
                                  F + ka * ka, ka, B_hi, B_lo, ldb, beta_hi, beta_lo, C_hi, C_lo,
                                  ldc, flags, nullptr, 0, stream)
            : casc_gemm_fp64x2_ex(CASC_OP_N, CASC_OP_N, m, n, n, alpha_hi, alpha_lo, B_hi, B_lo,
                                  ldb, F, F + ka * ka, ka, beta_hi, beta_lo, C_hi, C_lo, ldc,
                                  flags, nullptr, 0, stream);
  }
  const int gl = casc_last_launch_count();
  cudaFreeAsync(F, st);
  casc::host::set_launches(r == CASC_OK ? gl + 1 : 0);
  return r;
}

int casc_trmm_fp64x2(int side, int uplo, int trans, int diag, int64_t m, int64_t n,
                     double alpha_hi, double alpha_lo, const double* A_hi, const double* A_lo,
                     int64_t lda, double* B_hi, double* B_lo, int64_t ldb,
                     casc_stream_t stream) {
  casc::host::set_launches(0);
  if ((side != CASC_LEFT && side != CASC_RIGHT) || (uplo != CASC_LOWER && uplo != CASC_UPPER) ||
      (trans != CASC_OP_N && trans != CASC_OP_T) || (diag != CASC_NONUNIT && diag != CASC_UNIT))
    return CASC_ERR_INVALID;
  if (m < 0 || n < 0) return CASC_ERR_INVALID;
  const int64_t ka = side == CASC_LEFT ? m : n;
  int r;
  if ((r = casc::host::check_mat(A_hi, ka, ka, lda)) ||
      (r = casc::host::check_mat(A_lo, ka, ka, lda)) ||
      (r = casc::host::check_mat(B_hi, m, n, ldb)) || (r = casc::host::check_mat(B_lo, m, n, ldb)))
    return r;
  if (overlap3(B_hi, ext3(m, n, ldb), A_hi, ext3(ka, ka, lda)) ||
      overlap3(B_hi, ext3(m, n, ldb), A_lo, ext3(ka, ka, lda)) ||
      overlap3(B_lo, ext3(m, n, ldb), A_hi, ext3(ka, ka, lda)) ||
      overlap3(B_lo, ext3(m, n, ldb), A_lo, ext3(ka, ka, lda)) ||
      overlap3(B_hi, ext3(m, n, ldb), B_lo, ext3(m, n, ldb)))
    return CASC_ERR_INVALID;
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = casc::host::device_check(&sms))) return r;
  const cudaStream_t st = S3(stream);
  if (alpha_hi == 0.0 && alpha_lo == 0.0) {  // B := 0, A not read
    const cudaError_t e = casc::launch_scale_c(m, n, 0.0, 0.0, 0, B_hi, B_lo, ldb, nullptr, sms, st);
    casc::host::set_launches(e == cudaSuccess ? 1 : 0);
    return st3(e);
  }
  // the triangular A, dense (other triangle 0, unit diagonal 1), then T := alpha
  // op(A) B (or alpha B op(A)) with the cascaded GEMM, copied back into B
  double* F = nullptr;
  const size_t fa = (size_t)ka * ka, tb = (size_t)m * n;
  if (cudaMallocAsync(reinterpret_cast<void**>(&F), (2 * fa + 2 * tb) * sizeof(double), st) !=
      cudaSuccess)
    return CASC_ERR_CUDA;
  double* T = F + 2 * fa;
  r = st3(casc::expand(ka, uplo, 1, diag == CASC_UNIT, A_hi, A_lo, lda, F, F + fa, sms, st));
  int launches = 1;
  if (r == CASC_OK) {
    // each tile's k range stops at op(A)'s zero triangle (half the GEMM's work)
    const bool lower = (uplo == CASC_LOWER) != (trans == CASC_OP_T);  // op(A) lower
    r = side == CASC_LEFT
            ? casc::host::gemm_ex_band(trans, CASC_OP_N, m, n, m, alpha_hi, alpha_lo, F, F + fa,
                                       ka, B_hi, B_lo, ldb, T, T + tb, n, stream, lower ? 1 : 2)
            : casc::host::gemm_ex_band(CASC_OP_N, trans, m, n, n, alpha_hi, alpha_lo, B_hi, B_lo,
                                       ldb, F, F + fa, ka, T, T + tb, n, stream, lower ? 3 : 4);
    launches += casc_last_launch_count();
  }
  if (r == CASC_OK &&
      (cudaMemcpy2DAsync(B_hi, ldb * 8, T, n * 8, n * 8, m, cudaMemcpyDeviceToDevice, st) !=
           cudaSuccess ||
       cudaMemcpy2DAsync(B_lo, ldb * 8, T + tb, n * 8, n * 8, m, cudaMemcpyDeviceToDevice, st) !=
           cudaSuccess))
    r = CASC_ERR_CUDA;
  cudaFreeAsync(F, st);
  casc::host::set_launches(r == CASC_OK ? launches : 0);
  return r;
}

// Right side (reading R29): X op(A) = alpha B, A n x n triangular, B m x n.
// Column blocks of 256 in the order of op(A)'s triangle (ascending when op(A)
// is upper: X_b depends on the X_c left of it; descending when lower):
//   X_b = B_b op(Inv_b)          (Inv_b = A_bb^-1, casc_trsm_diag_inv)
//   B_c -= X_b op(A)_(b,c)       for the column blocks c still to solve,
// the updates of a super-block of 4 blocks applied at once after its last
// block (k up to 1024), as the left-side TRSM (reading R27).
int casc_trsm_fp64x2_right(int uplo, int trans, int diag, int64_t m, int64_t n, double alpha_hi,
                           double alpha_lo, const double* A_hi, const double* A_lo, int64_t lda,
                           double* B_hi, double* B_lo, int64_t ldb, casc_stream_t stream) {
  constexpr int64_t NB = 256, SB = 4;
  casc::host::set_launches(0);
  if ((uplo != CASC_LOWER && uplo != CASC_UPPER) || (diag != CASC_NONUNIT && diag != CASC_UNIT) ||
      (trans != CASC_OP_N && trans != CASC_OP_T))
    return CASC_ERR_INVALID;
  if (m < 0 || n < 0) return CASC_ERR_INVALID;
  int r;
  if ((r = casc::host::check_mat(A_hi, n, n, lda)) || (r = casc::host::check_mat(A_lo, n, n, lda)) ||
      (r = casc::host::check_mat(B_hi, m, n, ldb)) || (r = casc::host::check_mat(B_lo, m, n, ldb)))
    return r;
  if (overlap3(B_hi, ext3(m, n, ldb), A_hi, ext3(n, n, lda)) ||
      overlap3(B_hi, ext3(m, n, ldb), A_lo, ext3(n, n, lda)) ||
      overlap3(B_lo, ext3(m, n, ldb), A_hi, ext3(n, n, lda)) ||
      overlap3(B_lo, ext3(m, n, ldb), A_lo, ext3(n, n, lda)) ||
      overlap3(B_hi, ext3(m, n, ldb), B_lo, ext3(m, n, ldb)))
    return CASC_ERR_INVALID;
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = casc::host::device_check(&sms))) return r;
  const cudaStream_t st = S3(stream);
  int launches = 0;
  const bool unit_alpha = (alpha_hi == 1.0 && alpha_lo == 0.0);
  const bool zero_alpha = (alpha_hi == 0.0 && alpha_lo == 0.0);
  if (!unit_alpha) {  // B := alpha (x) B
    if (casc::launch_scale_c(m, n, alpha_hi, alpha_lo, zero_alpha ? 0 : 1, B_hi, B_lo, ldb,
                             nullptr, sms, st) != cudaSuccess)
      return CASC_ERR_CUDA;
    ++launches;
  }
  if (zero_alpha) {
    casc::host::set_launches(launches);
    return CASC_OK;
  }
  const int64_t nblk = (n + NB - 1) / NB;
  // T: the current super-block's X (m x SB*NB, ld SB*NB), the A operand of the
  // updates (a column block of B itself would overlap the updated columns' rows)
  const int64_t ldt = SB * NB;
  const size_t inv_elems = (size_t)nblk * NB * NB, t_elems = (size_t)m * ldt;
  double* buf = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&buf), (2 * inv_elems + 2 * t_elems) * 8, st) !=
      cudaSuccess)
    return CASC_ERR_CUDA;
  double* inv_hi = buf;
  double* inv_lo = buf + inv_elems;
  double* t_hi = inv_lo + inv_elems;
  double* t_lo = t_hi + t_elems;
  r = st3(casc::launch_trsm_diag_inv(uplo, diag, n, A_hi, A_lo, lda, inv_hi, inv_lo, st));
  ++launches;
  const bool eff_upper = (uplo == CASC_UPPER) != (trans == CASC_OP_T);  // op(A) upper
  // B_c -= X_K op(A)_(K, C): X_K = columns [K0, K1) of the solved super-block
  // starting at column S (held in T)
  auto update = [&](int64_t S, int64_t K0, int64_t K1, int64_t C0, int64_t C1) {
    if (r != CASC_OK || K1 <= K0 || C1 <= C0) return;
    // op(A)_(K, C) = A[K rows, C cols] (N) or A[C rows, K cols]^T (T)
    const int64_t off = trans == CASC_OP_N ? K0 * lda + C0 : C0 * lda + K0;
    r = casc_gemm_fp64x2_ex(CASC_OP_N, trans, m, C1 - C0, K1 - K0, -1.0, 0.0, t_hi + (K0 - S),
                            t_lo + (K0 - S), ldt, A_hi + off, A_lo + off, lda, 1.0, 0.0,
                            B_hi + C0, B_lo + C0, ldb, nullptr, nullptr, 0, stream);
    launches += casc_last_launch_count();
  };
  for (int64_t s = 0; s < nblk && r == CASC_OK; ++s) {
    const int64_t b = eff_upper ? s : nblk - 1 - s;
    const int64_t c0 = b * NB, nb = std::min(NB, n - c0), c1 = c0 + nb;
    const int64_t S0 = (b / SB) * SB * NB, S1 = std::min(S0 + SB * NB, n);
    // X_b = B_b op(Inv_b), into T's columns of block b and back into B's
    double* xh = t_hi + (c0 - S0);
    double* xl = t_lo + (c0 - S0);
    r = casc_gemm_fp64x2_ex(CASC_OP_N, trans, m, nb, nb, 1.0, 0.0, B_hi + c0, B_lo + c0, ldb,
                            inv_hi + b * NB * NB, inv_lo + b * NB * NB, NB, 0.0, 0.0, xh, xl,
                            ldt, nullptr, nullptr, 0, stream);
    launches += casc_last_launch_count();
    if (r) break;
    if (cudaMemcpy2DAsync(B_hi + c0, ldb * 8, xh, ldt * 8, nb * 8, m, cudaMemcpyDeviceToDevice,
                          st) != cudaSuccess ||
        cudaMemcpy2DAsync(B_lo + c0, ldb * 8, xl, ldt * 8, nb * 8, m, cudaMemcpyDeviceToDevice,
                          st) != cudaSuccess) {
      r = CASC_ERR_CUDA;
      break;
    }
    if (eff_upper) {
      update(S0, c0, c1, c1, S1);              // the super-block's remaining columns
      if (c1 == S1) update(S0, S0, S1, S1, n); // then the trailing columns, k = the super-block
    } else {
      update(S0, c0, c1, S0, c0);
      if (c0 == S0) update(S0, S0, S1, 0, S0);
    }
  }
  cudaFreeAsync(buf, st);
  casc::host::set_launches(r == CASC_OK ? launches : 0);
  return r;
}

}  // extern "C"
