// CTA-pair (cta_group::2) INT8 tensor-core probe for B200 (sm_100a), NEXT-3
// groundwork: one cluster of 2 CTAs computes a 256 x 128 int32 tile of
// A (256 x K) . B^T (B: 128 x K) with tcgen05.mma.cta_group::2.kind::i8
// (M = 256, N = 128, K = 32): CTA r holds A rows 128r .. 128r+127 and B rows
// 64r .. 64r+63 (its halves), loaded with cp.async.bulk.tensor.2d.cta_group::2
// signalling the leader CTA's mbarrier; the leader issues the MMAs and commits
// (multicast) to both CTAs.  Data is pre-swizzled in global memory (K-major,
// 128-byte swizzle), the tensor map copies it verbatim (SWIZZLE_NONE).
// Then a throughput run: 74 clusters, operands resident in smem.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8_pair_probe i8_pair_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) |
                           ((uint32_t)(256 >> 4) << 24);
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint32_t leader_addr(const void* p) {  // same offset in CTA rank 0
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* map, int x, int y,
                                     uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void commit_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %3, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %4, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(acc), "n"(IDESC));
}
__host__ __device__ inline uint32_t sw128(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((c >> 4) ^ (r & 7)) & 7) << 4) + (c & 15));
}

// A packed: per k block kb: 256 rows x 128 B pre-swizzled (two 16 KB chunks);
// B packed: per kb: 128 rows x 128 B (one 16 KB chunk).  Tensor maps see them
// as 2-D byte arrays with 128-byte rows.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_correct(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                 int32_t* C, int KB) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;           // 16 KB
  uint8_t* sb = smem + 16384;   // 8 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 24576);
  uint64_t* empty = full + 1;
  uint64_t* done = full + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(full + 3);
  const int t = threadIdx.x, w = t >> 5;
  const uint32_t rank = cta_rank();
  if (t == 0) {
    mbar_init(full, 1);
    mbar_init(empty, 1);
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = *tslot;
  const uint32_t full_l = leader_addr(full);
  for (int kb = 0; kb < KB; ++kb) {
    if (t == 0) {
      if (kb > 0) mbar_wait(empty, (kb - 1) & 1);
      if (rank == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full)),
                     "r"(2 * (16384 + 8192))
                     : "memory");
      tma2(sa, &mA, 0, kb * 256 + rank * 128, full_l);
      tma2(sb, &mB, 0, kb * 128 + rank * 64, full_l);
    }
    if (rank == 0 && t == 32) {
      mbar_wait(full, kb & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kk = 0; kk < 4; ++kk)
        mma2(tm, sdesc(smem_u32(sa)) + 2 * kk, sdesc(smem_u32(sb)) + 2 * kk, (kb | kk) ? 1u : 0u);
      commit_mc(empty);
      if (kb == KB - 1) commit_mc(done);
    }
  }
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = rank * 128 + 32 * w + (t & 31);
  for (int c0 = 0; c0 < 128; c0 += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(tm + ((uint32_t)(32 * w) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) C[row * 128 + c0 + j] = (int32_t)r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

// throughput: operands resident, leader issues `iters` x 4 MMAs into 4 accumulators of 128 cols
template <int NN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) pair_tput(int32_t* out, int iters) {
  constexpr uint32_t ID = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + 16384;
  uint64_t* done = reinterpret_cast<uint64_t*>(smem + 24576);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int t = threadIdx.x, w = t >> 5;
  const uint32_t rank = cta_rank();
  for (int i = t; i < 24576; i += 128) {  // random bytes (realistic bit activity)
    uint32_t h = (uint32_t)i * 0x9E3779B1u + blockIdx.x * 0x85EBCA6Bu;
    h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
    smem[i] = (uint8_t)h;
  }
  if (t == 0) {
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = *tslot;
  if (rank == 0 && t == 0) {
    const uint64_t a0 = sdesc(smem_u32(sa)), b0 = sdesc(smem_u32(sb));
    for (int it = 0; it < iters; ++it)
      for (int kk = 0; kk < 4; ++kk)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %3, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %4, p;\n}\n" ::"r"(tm + (it & 3) * 128), "l"(a0 + 2 * kk), "l"(b0 + 2 * kk), "r"(it > 3 ? 1u : 0u), "n"(ID));
    commit_mc(done);
  }
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tm + ((uint32_t)(32 * w) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (r == 0x12345678u) out[blockIdx.x] = 1;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

static CUtensorMap make_map(EncodeFn enc, void* base, uint64_t rows, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {128, rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {128, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { fprintf(stderr, "encode failed %d\n", (int)r); exit(1); }
  return m;
}

int main() {
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  const int M = 256, N = 128, K = 384, KB = K / 128;
  std::vector<int8_t> A(M * K), B(N * K);
  uint64_t s = 777;
  auto rnd = [&]() { s = s * 6364136223846793005ULL + 1442695040888963407ULL; return (int8_t)(s >> 56); };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  // packed, pre-swizzled: A per kb: 2 chunks of 128 rows; B per kb: 1 chunk
  std::vector<uint8_t> pA(M * K), pB(N * K);
  for (int kb = 0; kb < KB; ++kb) {
    for (int r = 0; r < M; ++r)
      for (int c = 0; c < 128; ++c)
        pA[(size_t)kb * M * 128 + (r / 128) * 16384 + sw128(r % 128, c)] = (uint8_t)A[r * K + kb * 128 + c];
    for (int r = 0; r < N; ++r)
      for (int c = 0; c < 128; ++c)
        pB[(size_t)kb * N * 128 + sw128(r, c)] = (uint8_t)B[r * K + kb * 128 + c];
  }
  std::vector<int32_t> R(M * N);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int32_t acc = 0;
      for (int k = 0; k < K; ++k) acc += (int32_t)A[i * K + k] * (int32_t)B[j * K + k];
      R[i * N + j] = acc;
    }
  uint8_t *dA, *dB;
  int32_t* dC;
  CK(cudaMalloc(&dA, pA.size()));
  CK(cudaMalloc(&dB, pB.size()));
  CK(cudaMalloc(&dC, M * N * 4));
  CK(cudaMemcpy(dA, pA.data(), pA.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, pB.data(), pB.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0, M * N * 4));
  CUtensorMap mA = make_map(enc, dA, (uint64_t)KB * M, 128);
  CUtensorMap mB = make_map(enc, dB, (uint64_t)KB * N, 64);
  const int smem = 24576 + 1024 + 2048;
  CK(cudaFuncSetAttribute(pair_correct, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  pair_correct<<<2, 128, smem>>>(mA, mB, dC, KB);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> C(M * N);
  CK(cudaMemcpy(C.data(), dC, M * N * 4, cudaMemcpyDeviceToHost));
  int bad = 0, first = -1;
  for (int i = 0; i < M * N; ++i)
    if (C[i] != R[i]) { ++bad; if (first < 0) first = i; }
  printf("{\"probe\": \"pair_correct\", \"mismatches\": %d, \"first\": %d, \"c0\": %d, \"r0\": %d, \"c_last\": %d, \"r_last\": %d}\n",
         bad, first, C[0], R[0], C[M * N - 1], R[M * N - 1]);
  if (bad) {
    // diagnose: compare against transposed / half-swapped B hypotheses
    int rows_ok = 0;
    for (int i = 0; i < M; ++i) { bool ok = true; for (int j = 0; j < N; ++j) ok &= C[i*N+j] == R[i*N+j]; rows_ok += ok; }
    printf("{\"rows_ok\": %d}\n", rows_ok);
  }
  auto run_t = [&](auto kern, int NN) {
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters = 20000;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  kern<<<148, 128, smem>>>(dC, 100);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    kern<<<148, 128, smem>>>(dC, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  const double ops = 2.0 * 256 * NN * 128.0 * iters * 74;
  const int launches = (int)(5000.0 / best) + 1;
  CK(cudaEventRecord(e0));
  for (int r = 0; r < launches; ++r) kern<<<148, 128, smem>>>(dC, iters);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms_all;
  CK(cudaEventElapsedTime(&ms_all, e0, e1));
  printf("{\"probe\": \"pair_tput\", \"M\": 256, \"N\": %d, \"data\": \"random\", \"burst_tops\": %.1f, \"sustained_tops\": %.1f, \"sustained_s\": %.2f}\n",
         NN, ops / best / 1e9, ops * launches / ms_all / 1e9, ms_all / 1e3);
  };
  run_t(pair_tput<128>, 128);
  run_t(pair_tput<64>, 64);
  return bad != 0;
}
