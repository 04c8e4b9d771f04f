// L2 -> shared-memory bandwidth probe for B200 (sm_100a), NEXT-3 groundwork:
// the INT8 cascade streams 16 KB slice chunks through TMA bulk copies
// (cp.async.bulk ... mbarrier::complete_tx), so its operand feed is bounded by
// what the TMA engines can pull from L2.  148 CTAs x 1 producer lane, a ring of
// NS 16 KB slots consumed as soon as they land.
//   mode 0: every CTA streams its own chunks of a buffer of `bytes` (distinct data);
//   mode 1: CTAs in groups of `share` stream the same chunk sequence (L2 reuse).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_probe l2_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

constexpr int CHUNK = 16384;
constexpr int NS = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(32) l2_stream(const uint8_t* buf, int64_t nchunks, int iters,
                                               int share, int* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[NS];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NS; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t group = share > 0 ? blockIdx.x / share : blockIdx.x;
  const int64_t ngroups = share > 0 ? (gridDim.x + share - 1) / share : gridDim.x;
  const int64_t per = nchunks / ngroups;
  int64_t c = group * per;
  for (int it = 0; it < iters; ++it) {
    const int s = it % NS;
    if (it >= NS) mbar_wait(&full[s], ((it / NS) - 1) & 1);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_u32(&full[s])),
                 "r"(CHUNK)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem + s * CHUNK)),
        "l"(buf + c * CHUNK), "r"(CHUNK), "r"(smem_u32(&full[s]))
        : "memory");
    if (++c >= (group + 1) * per) c = group * per;
  }
  for (int it = iters; it < iters + NS; ++it) {
    const int s = it % NS;
    if (it >= NS) mbar_wait(&full[s], ((it / NS) - 1) & 1);
  }
  if (smem[5] == 123 && out) out[blockIdx.x] = 1;
}

static void run(const uint8_t* buf, int64_t bytes, int share, int ctas_per_sm) {
  const int grid = 148 * ctas_per_sm;
  const int iters = 4000;
  const int smem = NS * CHUNK;
  CK(cudaFuncSetAttribute(l2_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  l2_stream<<<grid, 32, smem>>>(buf, bytes / CHUNK, 200, share, nullptr);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    l2_stream<<<grid, 32, smem>>>(buf, bytes / CHUNK, iters, share, nullptr);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  const double moved = (double)grid * iters * CHUNK;
  printf("{\"probe\": \"tma_stream\", \"buffer_mb\": %.0f, \"share\": %d, \"ctas_per_sm\": %d, "
         "\"GBps\": %.0f, \"B_per_clk_per_sm_at_1965\": %.1f}\n",
         bytes / 1e6, share, ctas_per_sm, moved / best / 1e6,
         moved / (best * 1e-3) / 148 / 1.965e9);
}

int main() {
  const int64_t big = 8ll << 30;
  uint8_t* buf;
  CK(cudaMalloc(&buf, big));
  CK(cudaMemset(buf, 1, big));
  run(buf, 64ll << 20, 0, 1);    // L2-resident, distinct per CTA
  run(buf, 64ll << 20, 0, 2);
  run(buf, big, 0, 1);           // HBM
  run(buf, 64ll << 20, 8, 1);    // groups of 8 CTAs on the same chunks
  run(buf, 64ll << 20, 16, 1);
  run(buf, big, 12, 1);          // HBM-sized, groups of 12 (the GEMM's sharing)
  return 0;
}
