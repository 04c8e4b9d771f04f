/* Standalone use of the C ABI (include/casc.h) from plain C, no Python:
 * C := A B for FP64x2 matrices with the ten-FP64-GEMM cascade, then the same
 * product with host-resident operands, then a check of a few entries against
 * a plain double-double dot product computed here.
 *
 * Build (CPU box or GPU box):
 *   gcc -O2 -std=c11 -Iinclude examples/c_api_demo.c \
 *       -Lpaper_2303_04353_b200 -lcasc -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2303_04353_b200 -o examples/c_api_demo
 * Run on a B200: ./examples/c_api_demo [n]   (prints "c_api_demo ok ...") */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "casc.h"

#define CK(x)                                                                      \
  do {                                                                             \
    int s_ = (x);                                                                  \
    if (s_) {                                                                      \
      fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, casc_status_string(s_)); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)
#define CU(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

/* error-free transformations for the host-side check */
static void two_sum(double a, double b, double* s, double* e) {
  *s = a + b;
  double bb = *s - a;
  *e = (a - (*s - bb)) + (b - bb);
}
static void dd_fma(double* h, double* l, double ah, double al, double bh, double bl) {
  double p = ah * bh, e = fma(ah, bh, -p) + (ah * bl + al * bh), s, t;
  two_sum(*h, p, &s, &t);
  t += e + *l;
  *h = s + t;
  *l = t - (*h - s);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 512;
  const size_t bytes = (size_t)n * n * sizeof(double);
  double *hA[2], *hB[2], *hC[2];
  for (int i = 0; i < 2; ++i) {
    CU(cudaMallocHost((void**)&hA[i], bytes));
    CU(cudaMallocHost((void**)&hB[i], bytes));
    CU(cudaMallocHost((void**)&hC[i], bytes));
  }
  uint64_t st = 12345;
  for (int64_t i = 0; i < n * n; ++i) {  /* hi in [-1,1), lo a tail below it */
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    const double u = (double)(st >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    const double v = (double)(st >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    hA[0][i] = u;
    hA[1][i] = u * 0x1.0p-54 * v;
    hB[0][i] = v;
    hB[1][i] = v * 0x1.0p-54 * u;
  }
  double *dA[2], *dB[2], *dC[2];
  for (int i = 0; i < 2; ++i) {
    CU(cudaMalloc((void**)&dA[i], bytes));
    CU(cudaMalloc((void**)&dB[i], bytes));
    CU(cudaMalloc((void**)&dC[i], bytes));
    CU(cudaMemcpy(dA[i], hA[i], bytes, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dB[i], hB[i], bytes, cudaMemcpyHostToDevice));
  }
  uint8_t* dF;
  CU(cudaMalloc((void**)&dF, (size_t)n * n));
  cudaStream_t s;
  CU(cudaStreamCreate(&s));
  /* device-resident operands */
  CK(casc_gemm_fp64x2(n, n, n, dA[0], dA[1], n, dB[0], dB[1], n, dC[0], dC[1], n, dF,
                      (casc_stream_t)s));
  CU(cudaStreamSynchronize(s));
  double* g[2];
  for (int i = 0; i < 2; ++i) {
    g[i] = (double*)malloc(bytes);
    CU(cudaMemcpy(g[i], dC[i], bytes, cudaMemcpyDeviceToHost));
  }
  /* host-resident operands (blocks streamed through the GPU): bitwise the same */
  CK(casc_gemm_fp64x2_host(n, n, n, hA[0], hA[1], n, hB[0], hB[1], n, hC[0], hC[1], n, NULL, 0, 0,
                           (casc_stream_t)s));
  CU(cudaStreamSynchronize(s));
  if (memcmp(g[0], hC[0], bytes) || memcmp(g[1], hC[1], bytes)) {
    fprintf(stderr, "host-operand result differs from the device result\n");
    return 1;
  }
  /* a few entries against a plain double-double dot product */
  double worst = 0.0;
  for (int t = 0; t < 16; ++t) {
    const int64_t i = (t * 7919) % n, j = (t * 104729) % n;
    double h = 0.0, l = 0.0, mag = 0.0;
    for (int64_t p = 0; p < n; ++p) {
      dd_fma(&h, &l, hA[0][i * n + p], hA[1][i * n + p], hB[0][p * n + j], hB[1][p * n + j]);
      mag += fabs(hA[0][i * n + p] * hB[0][p * n + j]);
    }
    const double err = fabs((g[0][i * n + j] - h) + (g[1][i * n + j] - l)) / mag;
    if (err > worst) worst = err;
  }
  printf("c_api_demo ok: n=%lld, host-operand entry bitwise, max |C - C_dd| / |A||B| = %.3e\n",
         (long long)n, worst);
  return worst < 0x1.0p-90 ? 0 : 1;
}
