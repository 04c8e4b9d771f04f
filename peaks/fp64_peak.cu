// FP64 throughput microbenchmark for B200 (sm_100a): the roofline denominator
// R_fp64tc that MEASURED_PEAKS.json does not carry.
//
// Register-only loops, no memory traffic inside the timed region:
//   dmma : mma.sync.aligned.m8n8k4.row.col.f64 (SASS DMMA.8x8x4), 8 independent
//          accumulator chains per warp, 512 flops per instruction per warp.
//   dfma : plain fma.rn.f64, 8 independent chains per thread.
// Each is timed as a burst (best of 10 short launches) and sustained (launches
// back to back for ~4 s), CUDA events, grid = 148 SMs x blocks_per_sm.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
// Output: one JSON line.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__global__ void __launch_bounds__(256) dmma_loop(double* out, int iters, double seed) {
  int t = threadIdx.x;
  double a = seed + t * 1e-3, b = seed - t * 1e-3;
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) { c[j][0] = j; c[j][1] = -j; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[blockIdx.x * blockDim.x + t] = s;
}

__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters, double seed) {
  int t = threadIdx.x;
  double a = seed + t * 1e-9, b = 1.0 - 1e-12;
  double c[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = fma(c[j], b, a);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j];
  if (s == 12345.678) out[blockIdx.x * blockDim.x + t] = s;
}

// Plain DADD / DMUL chains (8 independent per thread): are they full rate like DFMA?
__global__ void __launch_bounds__(256) dadd_loop(double* out, int iters, double seed) {
  int t = threadIdx.x;
  double a = seed + t * 1e-9;
  double c[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = __dadd_rn(c[j], a);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j];
  if (s == 12345.678) out[blockIdx.x * blockDim.x + t] = s;
}
__global__ void __launch_bounds__(256) dmul_loop(double* out, int iters, double seed) {
  int t = threadIdx.x;
  double a = 1.0 + t * 1e-15;
  double c[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j] = seed + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = __dmul_rn(c[j], a);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j];
  if (s == 12345.678) out[blockIdx.x * blockDim.x + t] = s;
}

// Mixed: even warps run the DMMA loop, odd warps the DFMA loop.  If DMMA and
// DFMA use separate pipes, the time equals the slower half alone; if they share
// the FP64 datapath, it is the sum.
__global__ void __launch_bounds__(256) mixed_loop(double* out, int iters, double seed) {
  const int t = threadIdx.x;
  double s = 0;
  if ((t >> 5) & 1) {
    double a = seed + t * 1e-9, b = 1.0 - 1e-12;
    double c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = fma(c[j], b, a);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j];
  } else {
    double a = seed + t * 1e-3, b = seed - t * 1e-3;
    double c[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) { c[j][0] = j; c[j][1] = -j; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  }
  if (s == 12345.678) out[blockIdx.x * blockDim.x + t] = s;
}

struct Res { double burst, sustained; };

template <typename F>
static Res run(F launch, double flops_per_launch) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int i = 0; i < 3; ++i) launch();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  int n = (int)(4000.0 / best) + 1;
  CK(cudaEventRecord(e0));
  for (int r = 0; r < n; ++r) launch();
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
  float tot; CK(cudaEventElapsedTime(&tot, e0, e1));
  Res res;
  res.burst = flops_per_launch / (best * 1e-3) / 1e12;
  res.sustained = flops_per_launch * n / (tot * 1e-3) / 1e12;
  return res;
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out; CK(cudaMalloc(&out, sizeof(double) * 148 * 8 * 256 * 4));
  const int threads = 256, bps = 4, iters = 4096;
  const int grid = sms * bps;
  double dmma_flops = (double)grid * (threads / 32) * iters * 8 * 512.0;
  double dfma_flops = (double)grid * threads * iters * 8 * 2.0;
  Res rm = run([&] { dmma_loop<<<grid, threads>>>(out, iters, 1.0); }, dmma_flops);
  CK(cudaGetLastError());
  Res rf = run([&] { dfma_loop<<<grid, threads>>>(out, iters, 1.0); }, dfma_flops);
  CK(cudaGetLastError());
  double dadd_ops = (double)grid * threads * iters * 8;
  Res ra = run([&] { dadd_loop<<<grid, threads>>>(out, iters, 1.0); }, dadd_ops);
  Res rmu = run([&] { dmul_loop<<<grid, threads>>>(out, iters, 1.0); }, dadd_ops);
  printf("{\"dadd_gops\": %.1f, \"dmul_gops\": %.1f, \"dfma_gops\": %.1f}\n", ra.burst * 1e3,
         rmu.burst * 1e3, rf.burst * 1e3 / 2);
  // mixed: half the warps DMMA, half DFMA, each doing the same per-warp work as above
  double mixed_flops = 0.5 * dmma_flops + 0.5 * dfma_flops;
  Res rx = run([&] { mixed_loop<<<grid, threads>>>(out, iters, 1.0); }, mixed_flops);
  CK(cudaGetLastError());
  // time of each half alone at the rates measured above (ms per launch)
  double t_dmma_half = 0.5 * dmma_flops / (rm.burst * 1e12) * 1e3;
  double t_dfma_half = 0.5 * dfma_flops / (rf.burst * 1e12) * 1e3;
  double t_mixed = mixed_flops / (rx.burst * 1e12) * 1e3;
  printf("{\"mixed_ms\": %.3f, \"dmma_half_alone_ms\": %.3f, \"dfma_half_alone_ms\": %.3f, "
         "\"verdict\": \"%s\"}\n", t_mixed, t_dmma_half, t_dfma_half,
         t_mixed < 0.75 * (t_dmma_half + t_dfma_half) ? "DMMA and DFMA overlap (separate pipes)"
                                                        : "DMMA and DFMA share the FP64 datapath");
  printf("{\"sms\": %d, \"dmma_tflops_burst\": %.3f, \"dmma_tflops_sustained\": %.3f, "
         "\"dfma_tflops_burst\": %.3f, \"dfma_tflops_sustained\": %.3f, "
         "\"how\": \"register-only mma.sync m8n8k4 f64 (8 chains/warp) and fma.rn.f64 (8 chains/thread), "
         "grid %d x %d threads; burst = best of 10, sustained = back-to-back ~4 s; CUDA events\"}\n",
         sms, rm.burst, rm.sustained, rf.burst, rf.sustained, grid, threads);
  return 0;
}
