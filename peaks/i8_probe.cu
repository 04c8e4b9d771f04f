// INT8 tensor-core probe for B200 (sm_100a): tcgen05.mma.kind::i8 with
// operands in shared memory (K-major, 128-byte swizzle) and an int32
// accumulator in tensor memory.  Two jobs (NEXT-3 groundwork):
//   1. correctness of the descriptor encodings (smem matrix descriptor,
//      instruction descriptor) against a CPU int32 GEMM, M=128, N in {128,256};
//   2. throughput: 148 persistent CTAs issue MMAs on smem-resident operands
//      (no memory traffic), burst (best of 5) and sustained (~3 s).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8_probe i8_probe.cu
// Output: JSON lines.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// smem matrix descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
  d |= (uint64_t)1 << 16;                           // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                 // SBO
  d |= (uint64_t)1 << 46;                           // version (sm_100)
  d |= (uint64_t)2 << 61;                           // SWIZZLE_128B
  return d;
}
// instruction descriptor: s8 x s8 -> s32, K-major A and B, M x N.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// byte offset of (row r, k byte c) inside a K-major SW128 tile of 128-byte rows
__host__ __device__ inline uint32_t sw128(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((c >> 4) ^ (r & 7)) & 7) << 4) + (c & 15));
}

// ---------------------------------------------------------------- correctness
// A: M x K (K contiguous), B: N x K (K contiguous), C: M x N int32. One CTA.
template <int N>
__global__ void __launch_bounds__(128) probe_correct(const int8_t* A, const int8_t* B, int32_t* C,
                                                     int K) {
  constexpr int M = 128;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;                // M x 128 B
  uint8_t* sb = smem + M * 128;      // N x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tbase)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) mbar_init(&bar, 1);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  uint32_t phase = 0;
  for (int kb = 0; kb < K / 128; ++kb) {
    for (int i = t; i < M * 128; i += 128) sa[sw128(i / 128, i % 128)] = A[(i / 128) * K + kb * 128 + i % 128];
    for (int i = t; i < N * 128; i += 128) sb[sw128(i / 128, i % 128)] = B[(i / 128) * K + kb * 128 + i % 128];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kk = 0; kk < 4; ++kk)
        mma_i8(tm, sdesc(smem_u32(sa) + 32 * kk), sdesc(smem_u32(sb) + 32 * kk), idesc_i8(M, N),
               (kb | kk) ? 1u : 0u);
      mma_commit(&bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  // row = 32*w + lane, columns in chunks of 8
  const int row = 32 * w + (t & 31);
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    tmem_ld8(tm + ((uint32_t)(32 * w) << 16) + c0, r);
    for (int j = 0; j < 8; ++j) C[row * N + c0 + j] = (int32_t)r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(256));
}

// ---------------------------------------------------------------- throughput
// Operands resident in smem (4 K-steps of 32 bytes); `iters` rounds of 4 MMAs
// alternating between two accumulators of N columns.
template <int N>
__global__ void __launch_bounds__(128) probe_tput(int32_t* out, int iters) {
  constexpr int M = 128;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;
  uint8_t* sb = smem + M * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < (M + N) * 128; i += 128) {  // random bytes (realistic bit activity)
    uint32_t h = (uint32_t)i * 0x9E3779B1u + blockIdx.x * 0x85EBCA6Bu;
    h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
    smem[i] = (uint8_t)h;
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tbase)),
                 "n"(2 * N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (t == 0) {
    const uint64_t a0 = sdesc(smem_u32(sa)), b0 = sdesc(smem_u32(sb));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_i8(tm + (it & 1) * N, a0 + 2 * kk, b0 + 2 * kk, idesc_i8(M, N), it > 1 ? 1u : 0u);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[8];
  tmem_ld8(tm + ((uint32_t)(32 * w) << 16), r);
  if (r[0] == 0x12345678u) out[blockIdx.x] = r[1];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(2 * N));
}

template <int N>
static bool run_correct(int K) {
  const int M = 128;
  std::vector<int8_t> A(M * K), B(N * K);
  uint64_t s = 12345 + N;
  auto rnd = [&]() { s = s * 6364136223846793005ULL + 1442695040888963407ULL; return (int8_t)(s >> 56); };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  std::vector<int32_t> C(M * N), R(M * N, 0);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int32_t acc = 0;
      for (int k = 0; k < K; ++k) acc += (int32_t)A[i * K + k] * (int32_t)B[j * K + k];
      R[i * N + j] = acc;
    }
  int8_t *dA, *dB;
  int32_t* dC;
  CK(cudaMalloc(&dA, M * K));
  CK(cudaMalloc(&dB, N * K));
  CK(cudaMalloc(&dC, M * N * 4));
  CK(cudaMemcpy(dA, A.data(), M * K, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), N * K, cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0, M * N * 4));
  const int smem = (M + N) * 128 + 1024;
  CK(cudaFuncSetAttribute(probe_correct<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe_correct<N><<<1, 128, smem>>>(dA, dB, dC, K);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(C.data(), dC, M * N * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < M * N; ++i) bad += C[i] != R[i];
  printf("{\"probe\": \"correct\", \"M\": %d, \"N\": %d, \"K\": %d, \"mismatches\": %d, \"c00\": %d, \"r00\": %d}\n",
         M, N, K, bad, C[0], R[0]);
  cudaFree(dA); cudaFree(dB); cudaFree(dC);
  return bad == 0;
}

template <int N>
static void run_tput(int blocks_per_sm) {
  const int M = 128;
  int32_t* out;
  CK(cudaMalloc(&out, 4096 * 4));
  const int smem = (M + N) * 128 + 1024;
  CK(cudaFuncSetAttribute(probe_tput<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = 148 * blocks_per_sm;
  const int iters = 20000;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  probe_tput<N><<<grid, 128, smem>>>(out, 100);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    probe_tput<N><<<grid, 128, smem>>>(out, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  const double ops = 2.0 * M * N * 128.0 * iters * grid;  // 4 MMAs of K=32 per iter
  // sustained: back to back for ~3 s
  int launches = (int)(5000.0 / best) + 1;
  CK(cudaEventRecord(e0));
  for (int r = 0; r < launches; ++r) probe_tput<N><<<grid, 128, smem>>>(out, iters);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms_all;
  CK(cudaEventElapsedTime(&ms_all, e0, e1));
  printf("{\"probe\": \"tput\", \"M\": %d, \"N\": %d, \"ctas_per_sm\": %d, \"burst_tops\": %.1f, "
         "\"sustained_tops\": %.1f, \"launches\": %d}\n",
         M, N, blocks_per_sm, ops / best / 1e9, ops * launches / ms_all / 1e9, launches);
  cudaFree(out);
}

int main() {
  bool ok = true;
  ok &= run_correct<256>(256);
  ok &= run_correct<128>(384);
  if (!ok) { printf("{\"probe\": \"abort\"}\n"); return 1; }
  run_tput<256>(1);
  run_tput<128>(1);
  run_tput<128>(2);
  return 0;
}
