// Host-resident operands: the row-slab pipeline shared by casc_gemm_fp64x2_host
// (FP64 cascade) and casc_i8_gemm_fp64x2_host (INT8 cascade); include/casc.h.
//
// Three streams: the caller's stream splits and multiplies, an internal H2D
// stream brings the slabs of A and B ahead of their use, an internal D2H
// stream returns each block of C as soon as it is done.  Two staging slots for
// A, B and C, events between the streams; device memory from the
// stream-ordered pool.  Blocks are bitwise the full product: an element of C
// depends only on its row of A and column of B, the scale exponents are per row
// of A / column of B, and slab starts are multiples of the packed block sizes.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "../../include/casc.h"

namespace casc {
namespace hostpipe {

struct Streams {
  cudaStream_t h2d = nullptr, d2h = nullptr;
};

inline int streams(Streams** out) {
  static Streams g[64];
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return CASC_ERR_CUDA;
  std::lock_guard<std::mutex> lk(mu);
  Streams& h = g[dev];
  if (!h.h2d && cudaStreamCreateWithFlags(&h.h2d, cudaStreamNonBlocking) != cudaSuccess)
    return CASC_ERR_CUDA;
  if (!h.d2h && cudaStreamCreateWithFlags(&h.d2h, cudaStreamNonBlocking) != cudaSuccess)
    return CASC_ERR_CUDA;
  *out = &h;
  return CASC_OK;
}

// Default slab extent along a dimension of `dim`: 4096 for large matrices; half
// the dimension (at least 1024) below 8192, so that the first blocks arrive
// early while each block still fills several waves of the GPU.
inline int64_t default_slab(int64_t dim) {
  if (dim >= 8192) return 4096;
  const int64_t h = (dim + 1) / 2;
  return h > 1024 ? h : 1024;
}

// k == 0: C := 0 and flags := 0 on the host, after the stream's prior work
inline int zero_host_c(int64_t m, int64_t n, double* C_hi, double* C_lo, int64_t ldc,
                       uint8_t* flags, cudaStream_t st) {
  if (cudaStreamSynchronize(st) != cudaSuccess) return CASC_ERR_CUDA;
  for (int64_t i = 0; i < m; ++i) {
    std::memset(C_hi + i * ldc, 0, sizeof(double) * n);
    std::memset(C_lo + i * ldc, 0, sizeof(double) * n);
  }
  if (flags) std::memset(flags, 0, (size_t)(m * n));
  return CASC_OK;
}

// Blocks of C: row slabs of A (height sr; the first one sr0 <= sr) x column
// slabs of B (width sc; the first one sc0 <= sc), row slab outer.  The H2D
// stream carries A_0, B_0 .. B_(J-1), A_1 .. A_(I-1) (two staging slots each),
// so the first block starts once A_0 and B_0 are in and the rest of B streams
// in under the first row of blocks; smaller first slabs shorten that exposed
// first copy.
// pack_b(dB_hi, dB_lo, cols, pB) / pack_a(dA_hi, dA_lo, rows, pA) /
// gemm(rows, cols, pA, pB, dC_hi, dC_lo, dFlags) enqueue on `st` (dense device
// operands: ld = cols for B and C, k for A) and return a casc status; bPBs /
// bPA are the packed sizes of one column slab of B / one row slab of A.
template <class PackB, class PackA, class Gemm>
int run(int64_t m, int64_t n, int64_t k, const double* A_hi, const double* A_lo, int64_t lda,
        const double* B_hi, const double* B_lo, int64_t ldb, double* C_hi, double* C_lo,
        int64_t ldc, uint8_t* flags, int64_t sr, int64_t sc, size_t bPBs, size_t bPA,
        cudaStream_t st, PackB pack_b, PackA pack_a, Gemm gemm, int64_t sr0 = 0,
        int64_t sc0 = 0) {
  Streams* hs = nullptr;
  int r = streams(&hs);
  if (r) return r;
  if (sr0 <= 0 || sr0 > sr) sr0 = sr;
  if (sc0 <= 0 || sc0 > sc) sc0 = sc;
  const int64_t I = m <= sr0 ? 1 : 1 + (m - sr0 + sr - 1) / sr;
  const int64_t J = n <= sc0 ? 1 : 1 + (n - sc0 + sc - 1) / sc;
  auto row0 = [&](int64_t i) { return i == 0 ? 0 : sr0 + (i - 1) * sr; };
  auto nrows = [&](int64_t i) { return std::min(i == 0 ? sr0 : sr, m - row0(i)); };
  auto col0 = [&](int64_t j) { return j == 0 ? 0 : sc0 + (j - 1) * sc; };
  auto ncols = [&](int64_t j) { return std::min(j == 0 ? sc0 : sc, n - col0(j)); };
  const int nA = I > 1 ? 2 : 1, nB = J > 1 ? 2 : 1, nC = I * J > 1 ? 2 : 1;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t bB = al(16 * (size_t)k * sc), bA = al(16 * (size_t)sr * k);
  const size_t bC = al(17 * (size_t)sr * sc);
  bPBs = al(bPBs);
  bPA = al(bPA);
  const size_t total = nB * bB + J * bPBs + nA * bA + bPA + nC * bC;
  cudaEvent_t ev_start, ev_done, ev_A[2], ev_packA[2], ev_B[2], ev_packB[2], ev_G[2], ev_D[2];
  cudaEvent_t* evs[] = {&ev_start, &ev_done, &ev_A[0], &ev_A[1], &ev_packA[0], &ev_packA[1],
                        &ev_B[0], &ev_B[1], &ev_packB[0], &ev_packB[1], &ev_G[0], &ev_G[1],
                        &ev_D[0], &ev_D[1]};
  int nev = 0;
  for (cudaEvent_t* x : evs) {
    if (cudaEventCreateWithFlags(x, cudaEventDisableTiming) != cudaSuccess) {
      for (int i = 0; i < nev; ++i) cudaEventDestroy(*evs[i]);
      return CASC_ERR_CUDA;
    }
    ++nev;
  }
  uint8_t* base = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&base), total, st) != cudaSuccess) {
    for (cudaEvent_t* x : evs) cudaEventDestroy(*x);
    return CASC_ERR_CUDA;
  }
  uint8_t* dBbuf = base;
  uint8_t* pB = dBbuf + nB * bB;
  uint8_t* dAbuf = pB + J * bPBs;
  uint8_t* pA = dAbuf + nA * bA;
  uint8_t* dCbuf = pA + bPA;
  cudaError_t e = cudaSuccess;
  int status = CASC_OK;
  auto ok = [&](cudaError_t x) {
    if (e == cudaSuccess) e = x;
  };
  auto okr = [&](int x) {
    if (status == CASC_OK) status = x;
  };
  // everything is ordered after the caller's prior work on `st`
  ok(cudaEventRecord(ev_start, st));
  ok(cudaStreamWaitEvent(hs->h2d, ev_start, 0));
  ok(cudaStreamWaitEvent(hs->d2h, ev_start, 0));
  // H2D items in stream order; item t waits for the pack that freed its slot
  int64_t packed_a = 0, packed_b = 0;  // packs enqueued so far
  int64_t next = 0;                    // next H2D item: 0 = A_0, 1..J = B_(t-1), then A_1..
  const int64_t nitems = I + J;
  auto pump = [&]() {
    for (; next < nitems; ++next) {
      const bool isB = next >= 1 && next <= J;
      if (isB) {
        const int64_t j = next - 1;
        const int sl = (int)(j % nB);
        if (j >= nB) {
          if (packed_b < j - nB + 1) return;  // slot still holds B_(j-2)
          ok(cudaStreamWaitEvent(hs->h2d, ev_packB[sl], 0));
        }
        const int64_t c0 = col0(j), cols = ncols(j);
        double* dB = reinterpret_cast<double*>(dBbuf + sl * bB);
        ok(cudaMemcpy2DAsync(dB, cols * 8, B_hi + c0, ldb * 8, cols * 8, k,
                             cudaMemcpyHostToDevice, hs->h2d));
        ok(cudaMemcpy2DAsync(dB + k * cols, cols * 8, B_lo + c0, ldb * 8, cols * 8, k,
                             cudaMemcpyHostToDevice, hs->h2d));
        ok(cudaEventRecord(ev_B[sl], hs->h2d));
      } else {
        const int64_t i = next == 0 ? 0 : next - J;
        const int sl = (int)(i % nA);
        if (i >= nA) {
          if (packed_a < i - nA + 1) return;  // slot still holds A_(i-2)
          ok(cudaStreamWaitEvent(hs->h2d, ev_packA[sl], 0));
        }
        const int64_t r0 = row0(i), rows = nrows(i);
        double* dA = reinterpret_cast<double*>(dAbuf + sl * bA);
        ok(cudaMemcpy2DAsync(dA, k * 8, A_hi + r0 * lda, lda * 8, k * 8, rows,
                             cudaMemcpyHostToDevice, hs->h2d));
        ok(cudaMemcpy2DAsync(dA + rows * k, k * 8, A_lo + r0 * lda, lda * 8, k * 8, rows,
                             cudaMemcpyHostToDevice, hs->h2d));
        ok(cudaEventRecord(ev_A[sl], hs->h2d));
      }
    }
  };
  pump();
  int64_t t = 0;  // block counter (C slots)
  for (int64_t i = 0; i < I && e == cudaSuccess && status == CASC_OK; ++i) {
    const int64_t r0 = row0(i), rows = nrows(i);
    double* dA = reinterpret_cast<double*>(dAbuf + (i % nA) * bA);
    ok(cudaStreamWaitEvent(st, ev_A[i % nA], 0));
    okr(pack_a(dA, dA + rows * k, rows, pA));
    ok(cudaEventRecord(ev_packA[i % nA], st));
    ++packed_a;
    pump();
    for (int64_t j = 0; j < J && e == cudaSuccess && status == CASC_OK; ++j, ++t) {
      const int64_t c0 = col0(j), cols = ncols(j);
      uint8_t* pBj = pB + j * bPBs;
      if (i == 0) {  // B_j arrives during the first row of blocks
        double* dB = reinterpret_cast<double*>(dBbuf + (j % nB) * bB);
        ok(cudaStreamWaitEvent(st, ev_B[j % nB], 0));
        okr(pack_b(dB, dB + k * cols, cols, pBj));
        ok(cudaEventRecord(ev_packB[j % nB], st));
        ++packed_b;
        pump();
      }
      const int sl = (int)(t % nC);
      double* dC = reinterpret_cast<double*>(dCbuf + sl * bC);
      uint8_t* dF = reinterpret_cast<uint8_t*>(dC + 2 * rows * cols);
      if (t >= nC) ok(cudaStreamWaitEvent(st, ev_D[sl], 0));  // C slot back on the host
      if (e != cudaSuccess || status != CASC_OK) break;
      okr(gemm(rows, cols, pA, pBj, dC, dC + rows * cols, flags ? dF : nullptr));
      ok(cudaEventRecord(ev_G[sl], st));
      // device -> host of this block of C (and flags) on the D2H stream
      ok(cudaStreamWaitEvent(hs->d2h, ev_G[sl], 0));
      ok(cudaMemcpy2DAsync(C_hi + r0 * ldc + c0, ldc * 8, dC, cols * 8, cols * 8, rows,
                           cudaMemcpyDeviceToHost, hs->d2h));
      ok(cudaMemcpy2DAsync(C_lo + r0 * ldc + c0, ldc * 8, dC + rows * cols, cols * 8, cols * 8,
                           rows, cudaMemcpyDeviceToHost, hs->d2h));
      if (flags)
        ok(cudaMemcpy2DAsync(flags + r0 * n + c0, n, dF, cols, cols, rows, cudaMemcpyDeviceToHost,
                             hs->d2h));
      ok(cudaEventRecord(ev_D[sl], hs->d2h));
    }
  }
  // the caller's stream completes after every copy; buffers go back to the pool
  cudaEventRecord(ev_done, hs->d2h);
  cudaStreamWaitEvent(st, ev_done, 0);
  cudaEventRecord(ev_done, hs->h2d);
  cudaStreamWaitEvent(st, ev_done, 0);
  cudaFreeAsync(base, st);
  for (cudaEvent_t* x : evs) cudaEventDestroy(*x);  // released once complete
  if (status != CASC_OK) return status;
  return e == cudaSuccess ? CASC_OK : CASC_ERR_CUDA;
}

}  // namespace hostpipe
}  // namespace casc
