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
//       T = T (+) bin0; T *= 2^(e_i + f_j) (ldexp per limb);
//       C (+)= T (FP64x2; C = (0, 0) before the first panel);
//       flag |= (bin0 == 0)  (§3.7, §4.4).
//
// Structure (Blackwell): persistent CTAs (one per SM), 384 threads,
// warp-specialised with setmaxnreg (producer 40 / MMA 232 registers).
//   warpgroup 0   producer: one elected lane issues TMA bulk copies
//                 (cp.async.bulk ... mbarrier::complete_tx) of each stage's
//                 A chunk (4 slices x 64 rows x 8 k = 16 KB) and B chunk
//                 (7 slices x 64 cols x 8 k = 28 KB) into a 4-deep smem ring,
//                 plus each panel's 64 + 64 scale exponents into an 8-deep ring;
//   warpgroups 1-2  8 MMA + epilogue warps, 2 (m) x 4 (n), 32 x 16 outputs each,
//                 4 bins x 8 m8n8 sub-tiles in registers; fragments are read
//                 from smem as 32 consecutive doubles (fragment-ordered layout).
// At each panel end the MMA warps combine their bins while the producer keeps
// prefetching; the FP64x2 C accumulator of the tile lives in TENSOR MEMORY
// (tcgen05.ld/st, 64 KB of the 256 KB) between panels and goes to global
// memory once, after the tile's last panel.
#include <cuda_runtime.h>

#include <cstdlib>

#include "casc_dd.cuh"
#include "casc_layout.cuh"
#include "casc_ptx.cuh"

// DBG instantiation: the combine below its early `continue` is unreachable by design
#pragma nv_diag_suppress 128

namespace casc {

#ifndef CASC_NSTAGE
#define CASC_NSTAGE 4
#endif
constexpr int NSTAGE = CASC_NSTAGE;  // smem ring depth
constexpr int NCW = 8;                        // MMA / epilogue warps (warpgroups 1, 2)
constexpr int GEMM_THREADS = (NCW + 4) * 32;  // + producer warpgroup 0
// Register budget per thread after setmaxnreg: producer warpgroup 40,
// MMA warpgroups 232 (128*40 + 256*232 = 64512 <= 64K registers).
constexpr int PRODUCER_REGS = 40;
constexpr int MMA_REGS = 232;
constexpr int GROUP_M = 16;                  // tile raster grouping (L2 reuse)
constexpr int EXP_RING = 8;  // > NSTAGE: a panel's exponents outlive the stages that carried them
constexpr size_t EXP_OFFSET =
    (size_t)NSTAGE * (A_STAGE + B_STAGE) * sizeof(double) + 2 * NSTAGE * sizeof(uint64_t) + 16;
// Longest wait of a producer at a tile-wave barrier (a cfg4 wave takes ~5.6 ms;
// the CTAs of a co-resident grid meet within microseconds).
constexpr uint64_t WAVE_WAIT_NS = 200000;
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr size_t GEMM_SMEM = EXP_OFFSET + (size_t)EXP_RING * (TM + TN) * sizeof(int32_t);



__device__ __forceinline__ void tile_coords(int tile, int mblocks, int nblocks, int& mb,
                                            int& nb, int gm = GROUP_M) {
  const int per_group = gm * nblocks;
  const int group = tile / per_group;
  const int first_m = group * gm;
  const int gsize = min(mblocks - first_m, gm);
  const int r = tile % per_group;
  mb = first_m + r % gsize;
  nb = r / gsize;
}

// Work item -> tile and stage range.  Normal mode: one item per 64x64 tile over
// all of its panels.  Split mode (small problems, p.split_p = P panels): one
// item per (tile, panel); its FP64x2 panel sum T_q goes to t_hi/t_lo[q] and a
// reduce kernel adds T_0 (+) T_1 (+) ... in panel order (bitwise the same
// sequence as the normal mode's C accumulation).
// SYRK: tile t of the row-major lower triangle -> (mb, nb), nb <= mb; the
// upper triangle is its transpose
__device__ __forceinline__ void tri_coords(int t, int tri, int& mb, int& nb) {
  int r = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
  while ((r + 1) * (r + 2) / 2 <= t) ++r;
  while (r * (r + 1) / 2 > t) --r;
  const int c = t - r * (r + 1) / 2;
  mb = tri == 2 ? c : r;
  nb = tri == 2 ? r : c;
}
template <bool TRI, bool BAND = false>
__device__ __forceinline__ void item_coords(const GemmArgs& p, int split_p, int item, int& mb,
                                            int& nb, int& s0, int& s1, int& q0) {
  if (TRI) {
    tri_coords(item, p.tri, mb, nb);
    s0 = p.st_begin;
    s1 = p.st_end;
    q0 = 0;
  } else if (split_p) {
    const int tile = item / split_p;
    q0 = item - tile * split_p;
    tile_coords(tile, p.mblocks, p.nblocks, mb, nb);
    s0 = q0 * STAGES_PER_PANEL;
    s1 = min(s0 + STAGES_PER_PANEL, p.st_end);
  } else {
    // TRMM (band): tile costs differ by row / column block; with 16 row blocks
    // per raster group the persistent CTA b only ever meets the row offsets
    // (b + 148 w) mod 16, i.e. 4 of the 16 (1.4% imbalance between CTAs); 17
    // is coprime with the grid and spreads every offset over every CTA (0.2%)
    tile_coords(item, p.mblocks, p.nblocks, mb, nb, (BAND && p.band) ? GROUP_M + 1 : GROUP_M);
    s0 = p.st_begin;
    s1 = p.st_end;
    q0 = 0;
    if (BAND && p.band) {  // the triangular operand's zero rows / columns: skip (TRMM)
      if (p.band == 1) s1 = min(s1, (mb + 1) * (TM / BK));
      if (p.band == 2) s0 = max(s0, mb * (TM / BK));
      if (p.band == 3) s0 = max(s0, nb * (TN / BK));
      if (p.band == 4) s1 = min(s1, (nb + 1) * (TN / BK));
    }
  }
}
// elements a SYRK stores (its triangle); everything for a GEMM
template <bool TRI>
__device__ __forceinline__ bool in_tri(const GemmArgs& p, int64_t row, int64_t col) {
  return !TRI || (p.tri == 1 ? row >= col : row <= col);
}
// work items of a launch
__host__ __device__ __forceinline__ int work_items(const GemmArgs& a) {
  if (a.tri) return a.mblocks * (a.mblocks + 1) / 2;
  return a.mblocks * a.nblocks * (a.split_p ? a.split_p : 1);
}

// DBG: debug export of one panel's bins instead of the combine (casc_debug_bins)
// AB:  BLAS update C := alpha AB + beta C at each tile's last panel (NEXT-4)
// SPLIT: split mode (small problems); a separate instantiation so the large-problem
//        kernel carries none of its indexing (measured 1.3% at 16384^3)
// TRI:  SYRK, one triangle of tiles (p.tri)
// WIDE: the re-run of the work items whose scales 2^(e_i + f_j) leave the
//       normal powers of two (reading R16), listed by the first launch
template <bool DBG, bool AB, bool SPLIT, bool TRI, bool WIDE>
__global__ void __launch_bounds__(GEMM_THREADS, 1) casc_gemm_kernel(const GemmArgs p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  double* As = reinterpret_cast<double*>(smem);
  double* Bs = As + NSTAGE * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + NSTAGE * B_STAGE);
  uint64_t* empty = full + NSTAGE;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(empty + NSTAGE);
  // ring of per-panel scale exponents [EXP_RING][A 64 | B 64] int32, filled by TMA
  int32_t* sexp = reinterpret_cast<int32_t*>(smem + EXP_OFFSET);

  // Programmatic dependent launch (PDL): the product launch lets its dependent
  // (the WIDE re-run) be scheduled at once, so that re-run's launch latency
  // hides in this grid's tail; the WIDE grid waits for this grid's completion
  // and memory (griddepcontrol.wait) before reading the list.
  if constexpr (WIDE) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (WIDE && *p.wide_count == 0) return;  // the common case: nothing to re-run
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // PDL: this launch may start in the split kernel's tail; nothing below reads
  // memory that kernel (or anything before it on the stream) writes before this
  // wait returns (a no-op without the launch attribute)
  if constexpr (!WIDE) asm volatile("griddepcontrol.wait;" ::: "memory");

  const int split_p = SPLIT ? p.split_p : 0;
  // work items (WIDE: the entries item * 8 + warp listed by the first launch)
  const int ntiles = WIDE ? (int)*p.wide_count
                          : (TRI ? p.mblocks * (p.mblocks + 1) / 2
                                 : p.mblocks * p.nblocks * (split_p ? split_p : 1));

  if (warp < 4) {
    // ===================== TMA producer (warpgroup 0) =====================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(PRODUCER_REGS));
    if (warp == 0 && lane == 0) {
      uint32_t it = 0, pc = 0;
      const int nwaves = (ntiles + gridDim.x - 1) / gridDim.x;
      for (int wave = 0; wave < nwaves; ++wave) {
        const int tile = blockIdx.x + wave * gridDim.x;
        if (!WIDE && p.wave_counter && wave > 0) {
          // Re-align all producers at every tile wave so that the tiles in flight
          // (a GROUP_M x ~9 block of C sharing A and B blocks) sweep k in step and
          // hit each other's slices in L2 instead of re-reading HBM.  A CTA without
          // a tile in this wave still arrives, so the count always completes.
          // The wait is bounded (WAVE_WAIT_NS): co-residency of the whole grid is
          // an optimisation here, never a correctness requirement, so the kernel
          // needs no cooperative launch and cannot hang when other work (another
          // stream, another process) holds some of the SMs.
          atomicAdd(p.wave_counter, 1u);
          if (tile < ntiles) {
            const unsigned int target = (unsigned int)wave * gridDim.x;
            const uint64_t t0 = globaltimer_ns();
            unsigned int v;
            for (;;) {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];"
                           : "=r"(v)
                           : "l"(p.wave_counter)
                           : "memory");
              if (v >= target || globaltimer_ns() - t0 > WAVE_WAIT_NS) break;
            }
          }
        }
        if (tile >= ntiles) continue;
        int mb, nb, s0, s1, q0;
        item_coords<TRI, AB && !SPLIT>(p, split_p, WIDE ? (int)p.wide_list[tile] : tile, mb,
                                       nb, s0, s1,
                         q0);
        const uint8_t* srcA = p.pa + mb * p.a_blk + (int64_t)s0 * A_STAGE * 8;
        const uint8_t* srcB = p.pb + nb * p.b_blk + (int64_t)s0 * B_STAGE * 8;
        for (int st = s0; st < s1; ++st, ++it) {
          const uint32_t slot = it % NSTAGE, ph = (it / NSTAGE) & 1;
          const bool pstart = (st == s0) || (st % STAGES_PER_PANEL) == 0;
          mbar_wait(&empty[slot], ph ^ 1);
          mbar_arrive_expect_tx(&full[slot],
                                (A_STAGE + B_STAGE) * 8 + (pstart ? (TM + TN) * 4 : 0));
          tma_bulk_g2s(As + slot * A_STAGE, srcA, A_STAGE * 8, &full[slot]);
          tma_bulk_g2s(Bs + slot * B_STAGE, srcB, B_STAGE * 8, &full[slot]);
          if (pstart) {  // this panel's row / column exponents ride along with its first stage
            const int q = st / STAGES_PER_PANEL;
            int32_t* dst = sexp + (pc % EXP_RING) * (TM + TN);
            tma_bulk_g2s(dst, p.pa + mb * p.a_blk + p.a_exp + q * TM * 4, TM * 4, &full[slot]);
            tma_bulk_g2s(dst + TM, p.pb + nb * p.b_blk + p.b_exp + q * TN * 4, TN * 4, &full[slot]);
            ++pc;
          }
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

  // The FP64x2 C accumulator of the current tile lives in TENSOR MEMORY between
  // panels: warp (wm, wn) owns lane quarter wn (= warp % 4) and columns
  // 64 wm .. 64 wm + 63, i.e. its 32 lanes x 16 elements x (hi, lo).  FP64 MMA
  // has no tcgen05 kind, so TMEM is otherwise idle; keeping C there frees the
  // registers and shared memory the DMMA pipeline needs.
  if (cw == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  named_bar_sync<NCW * 32>();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot + ((uint32_t)(wn * 32) << 16) + (uint32_t)(wm * 64);

  double acc[4][4][2][2];  // [bin][msub][nsub][pair]
  uint32_t it = 0, pc = 0;  // stage counter (smem ring), panel counter (exponent ring)
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int mb, nb, s0, s1, q0;
    const int item = WIDE ? (int)p.wide_list[tile] : tile;
    // WIDE: the warps of this item that met a wide scale in the first launch
    const unsigned int wmask = WIDE ? p.wide_mask[item] : 0u;
    item_coords<TRI, AB && !SPLIT>(p, split_p, item, mb, nb, s0, s1, q0);
    // Scales 2^(e_i + f_j) outside the normal powers of two (reading R16) are
    // rare; the combine of this kernel assumes one exact power of two per
    // element, and a warp that meets another scale in any panel of the item
    // stores no C (so C and beta C stay intact), sets its bit in the item's warp
    // mask and the item is listed once for the WIDE re-run, whose combine scales
    // ldexp-exactly and which stores the masked warps' elements.  Keeping that scaling out
    // of this kernel keeps its registers spill-free (measured: a warp-uniform
    // branch between the two scalings made ptxas spill in the k loop, -3%).
    bool wide_seen = false;
    // destination: C, or the panel-sum buffer T_q in split mode
    // Split mode writes the panel sums tile-major, [q][tile mb*nblocks+nb][warp][element
    // 0..15][lane]: every warp store is 256 contiguous bytes (split_reduce_kernel
    // reads the same layout)
    const int64_t toff = SPLIT ? (((int64_t)q0 * p.mblocks + mb) * p.nblocks + nb) * (TM * TN) +
                                     cw * 512 + lane
                               : 0;
    double* dst_hi = SPLIT ? p.t_hi + toff : p.C_hi;
    double* dst_lo = SPLIT ? p.t_lo + toff : p.C_lo;
    uint8_t* dst_fl = SPLIT ? p.fbuf + toff : p.flags;
    uint32_t flagbits = 0;
    for (int st = s0; st < s1; ++st, ++it) {
      if (st == s0 || (st % STAGES_PER_PANEL) == 0) {
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
        const double* ak = a_s + kk * A_KSTEP;
        const double* bk = b_s + kk * B_KSTEP;
        double a[4][4], b[7][2];
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int ms = 0; ms < 4; ++ms) a[s][ms] = ak[s * 256 + ms * 32];
#pragma unroll
        for (int s = 0; s < 7; ++s)
#pragma unroll
          for (int ns = 0; ns < 2; ++ns) b[s][ns] = bk[s * 256 + ns * 32];
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

      const bool panel_end = ((st + 1) % STAGES_PER_PANEL) == 0 || st + 1 == s1;
      if (!panel_end) continue;
      // this panel's scale exponents landed in smem with its first stage
      const int32_t* pex = sexp + (pc % EXP_RING) * (TM + TN);
      ++pc;
#ifdef CASC_EXPERIMENT_NO_COMBINE  // timing experiment only: combine the last panel alone
      if (st + 1 != s1) continue;
#endif
      // ------------------------------ phase 3: combine this panel
      const bool first = (st + 1 - s0) <= STAGES_PER_PANEL;  // first panel of the item
      const bool last = (st + 1 == s1);
#pragma unroll
      for (int ms = 0; ms < 4; ++ms)
#pragma unroll
        for (int ns = 0; ns < 2; ++ns)
#pragma unroll
          for (int i = 0; i < 2; ++i)
            flagbits |= (acc[0][ms][ns][i] == 0.0 ? 1u : 0u) << (ms * 4 + ns * 2 + i);
      if constexpr (DBG) {  // debug export of the single panel's bins (canonical scales)
#pragma unroll
        for (int ms = 0; ms < 4; ++ms)
#pragma unroll
          for (int ns = 0; ns < 2; ++ns)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int64_t row = (int64_t)mb * TM + wm * 32 + ms * 8 + g;
              const int64_t col = (int64_t)nb * TN + wn * 16 + ns * 8 + 2 * c + i;
              if (row >= p.m || col >= p.n) continue;
              const int64_t o = row * p.n + col, mn = p.m * p.n;
              p.dbg[o] = acc[0][ms][ns][i];
              p.dbg[mn + o] = acc[1][ms][ns][i];
              p.dbg[2 * mn + o] = __dmul_rn(acc[2][ms][ns][i], p.un_b2);
              p.dbg[3 * mn + o] = acc[3][ms][ns][i];
            }
        continue;
      }
      if constexpr (!WIDE) {  // this panel's scales: all normal powers of two for the warp?
        int emin = 1 << 30, emax = -(1 << 30), fmin = 1 << 30, fmax = -(1 << 30);
#pragma unroll
        for (int ms = 0; ms < 4; ++ms) {
          const int e = pex[wm * 32 + ms * 8 + g];
          emin = min(emin, e);
          emax = max(emax, e);
        }
#pragma unroll
        for (int ns = 0; ns < 2; ++ns)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int f = pex[TM + wn * 16 + ns * 8 + 2 * c + i];
            fmin = min(fmin, f);
            fmax = max(fmax, f);
          }
        wide_seen |= !__all_sync(0xffffffffu, emin + fmin >= -1022 && emax + fmax <= 1023);
      }
      const bool store_c = WIDE ? ((wmask >> cw) & 1u) != 0 : !wide_seen;
      // two halves (m-subtiles 0-1, 2-3): 8 elements = 32 TMEM columns each
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t cv[32];
        if (!first) {
          tmem_ld32(tmem + h * 32, cv);
          tmem_wait_ld();
        }
#pragma unroll
        for (int m2 = 0; m2 < 2; ++m2) {
          const int ms = 2 * h + m2;
          const int e = pex[wm * 32 + ms * 8 + g];
#pragma unroll
          for (int ns = 0; ns < 2; ++ns)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int x = (m2 * 4 + ns * 2 + i) * 4;
              double th, tl;
              combine_bins<WIDE>(
                  acc[0][ms][ns][i], acc[1][ms][ns][i], acc[2][ms][ns][i], acc[3][ms][ns][i],
                  p.c0, p.D2, e + pex[TM + wn * 16 + ns * 8 + 2 * c + i], th, tl);
              // C (+)= T with C = (0, 0) before the first panel (reading R10: the
              // FP64x2 addition also renormalises a T whose limbs were rounded
              // separately onto the subnormal grid, and turns -0 into +0, as the
              // oracle).  Split mode stores the raw panel value T_q; the reduction
              // adds (0, 0) (+) T_0 (+) T_1 ... in the same order.
              if constexpr (!SPLIT)
                dd_add(first ? 0.0 : __hiloint2double(cv[x + 1], cv[x]),
                       first ? 0.0 : __hiloint2double(cv[x + 3], cv[x + 2]), th, tl, th, tl);
              if (last) {
                const int64_t row = (int64_t)mb * TM + wm * 32 + ms * 8 + g;
                const int64_t col = (int64_t)nb * TN + wn * 16 + ns * 8 + 2 * c + i;
                if constexpr (SPLIT) {  // padded tile-major panel sums (reduced later)
                  if (store_c) {
                    dst_hi[(m2 * 4 + ns * 2 + i + h * 8) * 32] = th;
                    dst_lo[(m2 * 4 + ns * 2 + i + h * 8) * 32] = tl;
                  }
                } else if (store_c && row < p.m && col < p.n && in_tri<TRI>(p, row, col)) {
                  if (AB && p.ab)
                    apply_alpha_beta(th, tl, p.alpha_hi, p.alpha_lo, p.beta_hi, p.beta_lo,
                                     p.ab == 2 ? p.C_hi[row * p.ldc + col] : 0.0,
                                     p.ab == 2 ? p.C_lo[row * p.ldc + col] : 0.0, p.ab == 2);
                  dst_hi[row * p.ldc + col] = th;
                  dst_lo[row * p.ldc + col] = tl;
                }
              } else {
                cv[x] = __double2loint(th);
                cv[x + 1] = __double2hiint(th);
                cv[x + 2] = __double2loint(tl);
                cv[x + 3] = __double2hiint(tl);
              }
            }
        }
        if (!last) tmem_st32(tmem + h * 32, cv);
      }
      if (!last) tmem_wait_st();
    }
    if (!WIDE && wide_seen && lane == 0) {  // C of this warp's elements: the WIDE re-run
      // one list entry per item (the first of its warps to get here), a mask of
      // its warps: the re-run computes the item once and stores those warps
      if (atomicOr(&p.wide_mask[item], 1u << cw) == 0u)
        p.wide_list[atomicAdd(p.wide_count, 1u)] = (unsigned int)item;
    }
    // ------------------------------ cancellation flags of this tile
    // (independent of the scales: the first launch stores them for every warp)
    if (!DBG && !WIDE && dst_fl) {
#pragma unroll
      for (int ms = 0; ms < 4; ++ms) {
        const int64_t row = (int64_t)mb * TM + wm * 32 + ms * 8 + g;
#pragma unroll
        for (int ns = 0; ns < 2; ++ns)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int64_t col = (int64_t)nb * TN + wn * 16 + ns * 8 + 2 * c + i;
            if (row < p.m && col < p.n && in_tri<TRI>(p, row, col))
              dst_fl[SPLIT ? (int64_t)(ms * 4 + ns * 2 + i) * 32 : row * p.ldf + col] =
                  (flagbits >> (ms * 4 + ns * 2 + i)) & 1u;
          }
      }
    }
  }
  // ------------------------------ teardown: the allocating warp frees TMEM
  tc_fence_before();
  named_bar_sync<NCW * 32>();
  if (cw == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(*tmem_slot)
                 : "memory");
  }
}

template <bool DBG, bool AB, bool SPLIT, bool TRI = false, bool WIDE = false>
static cudaError_t launch_variant(GemmArgs& a, int grid, cudaStream_t st) {
  // per launch (the attribute is per device; the call is cheap and thread-safe)
  cudaError_t e = cudaFuncSetAttribute(casc_gemm_kernel<DBG, AB, SPLIT, TRI, WIDE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM);
  if (e != cudaSuccess) return e;
  if (!WIDE && !a.pdl) {
    casc_gemm_kernel<DBG, AB, SPLIT, TRI, WIDE><<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(a);
    return cudaGetLastError();
  }
  return launch_pdl(casc_gemm_kernel<DBG, AB, SPLIT, TRI, WIDE>, dim3(grid), dim3(GEMM_THREADS),
                    GEMM_SMEM, st, a);
}

// the product launch, then the WIDE re-run of what it listed (exits at once
// when the list is empty)
template <bool AB, bool SPLIT, bool TRI = false>
static cudaError_t launch_pair(GemmArgs& a, int grid, cudaStream_t st) {
  cudaError_t e = launch_variant<false, AB, SPLIT, TRI, false>(a, grid, st);
  if (e == cudaSuccess) e = launch_variant<false, AB, SPLIT, TRI, true>(a, grid, st);
  return e;
}

static bool wave_sync_on() {
  // default on: 10x less HBM traffic for the fused kernel at ~0.2% time cost
  // (profiles/r01c); CASC_WAVE_SYNC=0 turns it off
  const char* s = getenv("CASC_WAVE_SYNC");
  return !(s && s[0] == '0');
}

static size_t mask_bytes(int64_t items) {
  return ((size_t)items * sizeof(unsigned int) + 255) / 256 * 256;
}
size_t gemm_scratch_zero_bytes(int64_t items) { return GEMM_SCRATCH_HEAD + mask_bytes(items); }
size_t gemm_scratch_bytes(int64_t items) {
  return gemm_scratch_zero_bytes(items) + mask_bytes(items);
}

// a.scratch: gemm_scratch_bytes(work items) bytes of the caller's device memory,
// stream-ordered with this launch (wave counter, WIDE list count and entries).
cudaError_t launch_gemm(const GemmArgs& a_in, int num_sms, cudaStream_t st) {
  GemmArgs a = a_in;
  const int ntiles = work_items(a);
  const int grid = ntiles < num_sms ? ntiles : num_sms;
  if (grid == 0 || a.st_end <= a.st_begin) return cudaSuccess;
  if (a.dbg) {
    a.wave_counter = nullptr;
    a.pdl = 0;
    return launch_variant<true, false, false>(a, grid, st);
  }
  if (!a.scratch) return cudaErrorInvalidValue;
  a.wave_counter = reinterpret_cast<unsigned int*>(a.scratch);
  a.wide_count = a.wave_counter + 1;
  a.wide_mask = reinterpret_cast<unsigned int*>(static_cast<uint8_t*>(a.scratch) + GEMM_SCRATCH_HEAD);
  a.wide_list = reinterpret_cast<unsigned int*>(static_cast<uint8_t*>(a.scratch) +
                                                gemm_scratch_zero_bytes(ntiles));
  if (!a.pdl) {  // else zeroed by the caller before the split launch (PDL edge kept)
    cudaError_t e = cudaMemsetAsync(a.scratch, 0, gemm_scratch_zero_bytes(ntiles), st);
    if (e != cudaSuccess) return e;
  }
  // no wave barrier for few waves, split mode, or banded tiles of unequal length
  if (a.split_p || a.band || ntiles <= num_sms || !wave_sync_on()) a.wave_counter = nullptr;
  if (a.tri) return launch_pair<true, false, true>(a, grid, st);
  if (a.split_p)
    return a.ab ? launch_pair<true, true>(a, grid, st) : launch_pair<false, true>(a, grid, st);
  return (a.ab || a.band) ? launch_pair<true, false>(a, grid, st)
                          : launch_pair<false, false>(a, grid, st);
}

}  // namespace casc
