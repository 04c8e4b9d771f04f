// Probe: confirm the f64 mma.sync fragment layouts assumed by the fused kernel.
// m8n8k4:  a0 = A[g][c], b0 = B[c][g], d{0,1} = D[g][2c+{0,1}]   (g = lane>>2, c = lane&3)
// m16n8k4: a{0,1} = A[g(+8)][c], b0 = B[c][g], d{0,1} = D[g][2c+i], d{2,3} = D[g+8][2c+i]
#include <cstdio>
#include <cmath>
__global__ void probe(double* out8, double* out16, const double* A, const double* B) {
  int l = threadIdx.x, g = l >> 2, c = l & 3;
  double d0 = 0, d1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(A[g * 4 + c]), "d"(B[c * 8 + g]));
  out8[g * 8 + 2 * c] = d0; out8[g * 8 + 2 * c + 1] = d1;
  double e0 = 0, e1 = 0, e2 = 0, e3 = 0;
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(e0), "+d"(e1), "+d"(e2), "+d"(e3)
               : "d"(A[g * 4 + c]), "d"(A[(g + 8) * 4 + c]), "d"(B[c * 8 + g]));
  out16[g * 8 + 2 * c] = e0; out16[g * 8 + 2 * c + 1] = e1;
  out16[(g + 8) * 8 + 2 * c] = e2; out16[(g + 8) * 8 + 2 * c + 1] = e3;
}
int main() {
  double hA[64], hB[32], r8[64], r16[128];
  for (int i = 0; i < 64; ++i) hA[i] = 1 + i * 0.5;
  for (int i = 0; i < 32; ++i) hB[i] = (i % 7) - 3 + 0.25 * i;
  double *dA, *dB, *o8, *o16;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&o8, sizeof r8); cudaMalloc(&o16, sizeof r16);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  probe<<<1, 32>>>(o8, o16, dA, dB);
  cudaMemcpy(r8, o8, sizeof r8, cudaMemcpyDeviceToHost); cudaMemcpy(r16, o16, sizeof r16, cudaMemcpyDeviceToHost);
  int bad8 = 0, bad16 = 0;
  for (int i = 0; i < 16; ++i) for (int j = 0; j < 8; ++j) {
    double s = 0; for (int k = 0; k < 4; ++k) s += hA[i * 4 + k] * hB[k * 8 + j];
    if (i < 8 && r8[i * 8 + j] != s) ++bad8;
    if (r16[i * 8 + j] != s) ++bad16;
  }
  printf("{\"mma_layout_m8n8k4_bad\": %d, \"mma_layout_m16n8k4_bad\": %d}\n", bad8, bad16);
  return (bad8 || bad16) ? 1 : 0;
}
