// casc_gemm.cu — phases 2 and 3 of the cascaded FP64x2 GEMM: the fused kernel.
//
// Per 64 x 64 C tile and per 256-wide k panel q (§3.5):
//   phase 2 (eqn:Gemm10), on the FP64 tensor cores (DMMA,
//   mma.sync.m8n8k4.f64; tcgen05 has no f64 kind on sm_100a), all ten
//   products accumulated straight into four register bins thanks to the exact
//   pre-alignment done by the split kernels:
//       bin0  += A0 B0                                   (exact)
//       bin1  += A0 B1 + A1 B0                           (exact)
//       bin2' += A0 B2' + A1 B1 + A2' B0                 (exact; = 2^(c0-c1) bin2)
//       bin36 += A0 B3 + A1 B4' + A2' B5'' + A3 B6        (FP64-rounded)
//   phase 3 (fl_casc; order bin 3-6 -> 2 -> 1 -> 0):
//       T = TwoSum(2^-2c0 bin2', 2^-D2 bin36); T = T (+) 2^-c0 bin1;
//       T = T (+) bin0; T *= 2^(e_i + f_j);  C (+)= T (FP64x2);
//       flag |= (bin0 == 0)  (§3.7, §4.4).
//
// Structure (Blackwell): persistent CTAs (one per SM), warp-specialised.
//   warp 8      producer: one elected lane issues TMA bulk copies
//               (cp.async.bulk ... mbarrier::complete_tx) of each stage's
//               A chunk (4 slices x 64 rows x 8 k = 16 KB) and B chunk
//               (7 slices x 64 cols x 8 k = 28 KB) into a 4-deep smem ring;
//   warps 0..7  MMA + epilogue: 2 (m) x 4 (n) warps, 32 x 16 outputs each,
//               4 bins x 8 m8n8 sub-tiles in registers; fragments are read
//               from smem as 32 consecutive doubles (fragment-ordered layout).
// The combine runs on the MMA warps at each panel end while the producer
// keeps prefetching; C is read-modified-written in global memory once per
// panel per element (16 B r + 16 B w per 2560 FMAs: negligible).
#include <cuda_runtime.h>

#include "casc_layout.cuh"

namespace casc {

constexpr int NSTAGE = 4;
constexpr int NCW = 8;                        // MMA / epilogue warps (warpgroups 1, 2)
constexpr int GEMM_THREADS = (NCW + 4) * 32;  // + producer warpgroup 0
// Register budget per thread after setmaxnreg: producer warpgroup 40,
// MMA warpgroups 232 (128*40 + 256*232 = 64512 <= 64K registers).
constexpr int PRODUCER_REGS = 40;
constexpr int MMA_REGS = 232;
constexpr int GROUP_M = 16;                  // tile raster grouping (L2 reuse)
constexpr size_t GEMM_SMEM =
    (size_t)NSTAGE * (A_STAGE + B_STAGE) * sizeof(double) + 2 * NSTAGE * sizeof(uint64_t);



// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// TMA engine 1-D bulk copy global -> shared, completion signalled on `bar`.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------ DD helpers
// Textbook EFTs with explicit _rn intrinsics (bit-reproducible, no FMA).
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
__device__ __forceinline__ void fast_two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  e = __dsub_rn(b, __dsub_rn(s, a));
}
__device__ __forceinline__ void dd_add_d(double& h, double& l, double x) {
  double s, e;
  two_sum(h, x, s, e);
  e = __dadd_rn(e, l);
  fast_two_sum(s, e, h, l);
}
__device__ __forceinline__ void dd_add(double xh, double xl, double yh, double yl, double& rh,
                                       double& rl) {
  double s1, s2, t1, t2;
  two_sum(xh, yh, s1, s2);
  two_sum(xl, yl, t1, t2);
  s2 = __dadd_rn(s2, t1);
  fast_two_sum(s1, s2, s1, s2);
  s2 = __dadd_rn(s2, t2);
  fast_two_sum(s1, s2, rh, rl);
}

__device__ __forceinline__ void tile_coords(int tile, int mblocks, int nblocks, int& mb,
                                            int& nb) {
  const int per_group = GROUP_M * nblocks;
  const int group = tile / per_group;
  const int first_m = group * GROUP_M;
  const int gsize = min(mblocks - first_m, GROUP_M);
  const int r = tile % per_group;
  mb = first_m + r % gsize;
  nb = r / gsize;
}

__global__ void __launch_bounds__(GEMM_THREADS, 1) casc_gemm_kernel(const GemmArgs p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  double* As = reinterpret_cast<double*>(smem);
  double* Bs = As + NSTAGE * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + NSTAGE * B_STAGE);
  uint64_t* empty = full + NSTAGE;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int ntiles = p.mblocks * p.nblocks;

  if (warp < 4) {
    // ===================== TMA producer (warpgroup 0) =====================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(PRODUCER_REGS));
    if (warp == 0 && lane == 0) {
      uint32_t it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int mb, nb;
        tile_coords(tile, p.mblocks, p.nblocks, mb, nb);
        const uint8_t* srcA = p.pa + mb * p.a_blk + (int64_t)p.st_begin * A_STAGE * 8;
        const uint8_t* srcB = p.pb + nb * p.b_blk + (int64_t)p.st_begin * B_STAGE * 8;
        for (int st = p.st_begin; st < p.st_end; ++st, ++it) {
          const uint32_t slot = it % NSTAGE, ph = (it / NSTAGE) & 1;
          mbar_wait(&empty[slot], ph ^ 1);
          mbar_arrive_expect_tx(&full[slot], (A_STAGE + B_STAGE) * 8);
          tma_bulk_g2s(As + slot * A_STAGE, srcA, A_STAGE * 8, &full[slot]);
          tma_bulk_g2s(Bs + slot * B_STAGE, srcB, B_STAGE * 8, &full[slot]);
          srcA += A_STAGE * 8;
          srcB += B_STAGE * 8;
        }
      }
    }
    return;
  }

  // ===================== MMA + epilogue warps (warpgroups 1, 2) =====================
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(MMA_REGS));
  const int cw = warp - 4;
  const int wm = cw >> 2, wn = cw & 3;
  const int g = lane >> 2, c = lane & 3;
  const double s_bin1 = pow2i(-p.c0), s_bin2 = pow2i(-2 * p.c0), s_bin36 = pow2i(-p.D2);

  double acc[4][4][2][2];  // [bin][msub][nsub][pair]
  uint32_t it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int mb, nb;
    tile_coords(tile, p.mblocks, p.nblocks, mb, nb);
    uint32_t flagbits = 0;
    for (int st = p.st_begin; st < p.st_end; ++st, ++it) {
      if (st == p.st_begin || (st % STAGES_PER_PANEL) == 0) {
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int ms = 0; ms < 4; ++ms)
#pragma unroll
            for (int ns = 0; ns < 2; ++ns) acc[b][ms][ns][0] = acc[b][ms][ns][1] = 0.0;
      }
      const uint32_t slot = it % NSTAGE, ph = (it / NSTAGE) & 1;
      mbar_wait(&full[slot], ph);
      const double* a_s = As + slot * A_STAGE + wm * 128 + lane;
      const double* b_s = Bs + slot * B_STAGE + wn * 64 + lane;
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk) {
        double a[4][4], b[7][2];
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int ms = 0; ms < 4; ++ms) a[s][ms] = a_s[kk * A_KSTEP + s * 256 + ms * 32];
#pragma unroll
        for (int s = 0; s < 7; ++s)
#pragma unroll
          for (int ns = 0; ns < 2; ++ns) b[s][ns] = b_s[kk * B_KSTEP + s * 256 + ns * 32];
        // ten products, eqn:Gemm10, sub-tile loop innermost
#define CASC_PROD(BIN, SA, SB)                      \
  _Pragma("unroll") for (int ms = 0; ms < 4; ++ms)  \
      _Pragma("unroll") for (int ns = 0; ns < 2; ++ns) dmma(acc[BIN][ms][ns], a[SA][ms], b[SB][ns]);
        CASC_PROD(0, 0, 0)  // bin0:  A0 B0
        CASC_PROD(1, 0, 1)  // bin1:  A0 B1
        CASC_PROD(2, 0, 2)  // bin2:  A0 B2'
        CASC_PROD(3, 0, 3)  // bin36: A0 B3
        CASC_PROD(1, 1, 0)  // bin1:  A1 B0
        CASC_PROD(2, 1, 1)  // bin2:  A1 B1
        CASC_PROD(3, 1, 4)  // bin36: A1 B4'
        CASC_PROD(2, 2, 0)  // bin2:  A2' B0
        CASC_PROD(3, 2, 5)  // bin36: A2' B5''
        CASC_PROD(3, 3, 6)  // bin36: A3 B6
#undef CASC_PROD
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);

      const bool panel_end = ((st + 1) % STAGES_PER_PANEL) == 0 || st + 1 == p.st_end;
      if (!panel_end) continue;
      // ------------------------------ phase 3: combine this panel
      const int q = st / STAGES_PER_PANEL;
      const int32_t* eA =
          reinterpret_cast<const int32_t*>(p.pa + mb * p.a_blk + p.a_exp) + q * TM;
      const int32_t* fB =
          reinterpret_cast<const int32_t*>(p.pb + nb * p.b_blk + p.b_exp) + q * TN;
      const bool first = (st + 1 - p.st_begin) <= STAGES_PER_PANEL;
#pragma unroll
      for (int ms = 0; ms < 4; ++ms) {
        const int rl = wm * 32 + ms * 8 + g;
        const int64_t row = (int64_t)mb * TM + rl;
        const int e = __ldg(eA + rl);
#pragma unroll
        for (int ns = 0; ns < 2; ++ns) {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int cl = wn * 16 + ns * 8 + 2 * c + i;
            const int64_t col = (int64_t)nb * TN + cl;
            const double b0 = acc[0][ms][ns][i], b1 = acc[1][ms][ns][i];
            const double b2 = acc[2][ms][ns][i], b36 = acc[3][ms][ns][i];
            flagbits |= (b0 == 0.0 ? 1u : 0u) << (ms * 4 + ns * 2 + i);
            if (row >= p.m || col >= p.n) continue;
            if (p.dbg) {
              const int64_t o = row * p.n + col, mn = p.m * p.n;
              p.dbg[o] = b0;
              p.dbg[mn + o] = b1;
              p.dbg[2 * mn + o] = __dmul_rn(b2, p.un_b2);
              p.dbg[3 * mn + o] = b36;
              continue;
            }
            const int f = __ldg(fB + cl);
            double th, tl;
            two_sum(__dmul_rn(b2, s_bin2), __dmul_rn(b36, s_bin36), th, tl);
            dd_add_d(th, tl, __dmul_rn(b1, s_bin1));
            dd_add_d(th, tl, b0);
            const double sc = pow2i(e + f);
            th = __dmul_rn(th, sc);
            tl = __dmul_rn(tl, sc);
            double* ch = p.C_hi + row * p.ldc + col;
            double* cl_ = p.C_lo + row * p.ldc + col;
            if (!first) dd_add(*ch, *cl_, th, tl, th, tl);
            *ch = th;
            *cl_ = tl;
          }
        }
      }
    }
    // ------------------------------ cancellation flags of this tile
    if (p.flags && !p.dbg) {
#pragma unroll
      for (int ms = 0; ms < 4; ++ms) {
        const int64_t row = (int64_t)mb * TM + wm * 32 + ms * 8 + g;
#pragma unroll
        for (int ns = 0; ns < 2; ++ns)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int64_t col = (int64_t)nb * TN + wn * 16 + ns * 8 + 2 * c + i;
            if (row < p.m && col < p.n)
              p.flags[row * p.n + col] = (flagbits >> (ms * 4 + ns * 2 + i)) & 1u;
          }
      }
    }
  }
}

cudaError_t launch_gemm(const GemmArgs& a, int num_sms, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(casc_gemm_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)GEMM_SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int ntiles = a.mblocks * a.nblocks;
  const int grid = ntiles < num_sms ? ntiles : num_sms;
  if (grid == 0 || a.st_end <= a.st_begin) return cudaSuccess;
  casc_gemm_kernel<<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(a);
  return cudaGetLastError();
}

}  // namespace casc
