// casc_api.cu — host side of the C ABI declared in include/casc.h:
// argument validation, widths, workspace, kernel launches.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/casc.h"
#include "casc_host.cuh"
#include "casc_layout.cuh"

namespace casc {
cudaError_t launch_split_reduce(int P, int64_t m, int64_t n, const double* t_hi,
                                const double* t_lo, const uint8_t* fbuf, double* C_hi,
                                double* C_lo, int64_t ldc, uint8_t* flags, int64_t ldf, int ab,
                                double ah, double al, double bh, double bl, int num_sms,
                                cudaStream_t st);
cudaError_t launch_trsm_diag_inv(int uplo, int diag, int64_t m, const double* A_hi,
                                 const double* A_lo, int64_t lda, double* I_hi, double* I_lo,
                                 cudaStream_t st);
cudaError_t launch_scale_c_uplo(int64_t m, int64_t n, double bh, double bl, int use_beta,
                                double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
                                int num_sms, int uplo, cudaStream_t st);
cudaError_t launch_ldexp(int64_t count, const double* x, const int32_t* n, double* out,
                         cudaStream_t st);
cudaError_t launch_or_flags(int64_t n, int uplo, uint8_t* flags, const uint8_t* f2, int num_sms,
                            cudaStream_t st);
cudaError_t launch_scale_c(int64_t m, int64_t n, double bh, double bl, int use_beta, double* C_hi,
                           double* C_lo, int64_t ldc, uint8_t* flags, int num_sms,
                           cudaStream_t st);
cudaError_t launch_split_a(const double*, const double*, int64_t, int64_t, int64_t, Widths, void*,
                           cudaStream_t, bool trans = false);
cudaError_t launch_split_b(const double*, const double*, int64_t, int64_t, int64_t, Widths, void*,
                           cudaStream_t, bool trans = false);
cudaError_t launch_split_ab(const double* Ahi, const double* Alo, int64_t lda, int64_t m,
                            const double* Bhi, const double* Blo, int64_t ldb, int64_t n,
                            int64_t k, Widths w, void* pa, void* pb, cudaStream_t st, bool ta,
                            bool tb);
cudaError_t launch_unpack_a(const void*, int64_t, int64_t, Widths, double*, int32_t*,
                            cudaStream_t);
cudaError_t launch_unpack_b(const void*, int64_t, int64_t, Widths, double*, int32_t*,
                            cudaStream_t);
}  // namespace casc

namespace {

thread_local int g_launches = 0;

inline cudaStream_t S(casc_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// §3.3 P:L916-945 with L = ceil(log2 min(k, 256)) (reading R3).
casc::Widths widths_for(int64_t k) {
  int64_t keff = k < casc::KC ? k : casc::KC;
  if (keff < 1) keff = 1;
  int L = 0;
  while ((int64_t(1) << L) < keff) ++L;
  casc::Widths w{0, 0, 0};
  while (2 * (w.c0 + 1) + L <= 53) ++w.c0;
  while (w.c0 + (w.c1 + 1) + L + 1 <= 53 && 2 * (w.c1 + 1) + L + 2 <= 53) ++w.c1;
  while (w.c0 + (w.c2 + 1) + L + 2 <= 53) ++w.c2;
  return w;
}

struct DevInfo {
  int checked = 0;
  int ok = 0;
  int sms = 0;
};

int device_check(int* sms) {
  static DevInfo info[64];
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return CASC_ERR_CUDA;
  std::lock_guard<std::mutex> lk(mu);
  DevInfo& d = info[dev];
  if (!d.checked) {
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return CASC_ERR_CUDA;
    d.ok = (major == 10 && minor == 0);
    d.checked = 1;
    // Stream-ordered temporaries (split-mode sums, debug exports) come from the
    // default pool: keep freed blocks cached instead of unmapping them at every
    // synchronisation (measured 0.5 ms per call otherwise).
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  if (sms) *sms = d.sms;
  return d.ok ? CASC_OK : CASC_ERR_UNSUPPORTED;
}

inline bool ranges_overlap(const void* a, size_t an, const void* b, size_t bn) {
  if (!a || !b || an == 0 || bn == 0) return false;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
  return a0 < b0 + bn && b0 < a0 + an;
}
inline size_t extent(int64_t rows, int64_t cols, int64_t ld) {
  if (rows <= 0 || cols <= 0) return 0;
  return size_t((rows - 1) * ld + cols) * sizeof(double);
}

int check_mat(const void* p, int64_t rows, int64_t cols, int64_t ld) {
  if (rows < 0 || cols < 0) return CASC_ERR_INVALID;
  if (ld < (cols > 1 ? cols : 1)) return CASC_ERR_INVALID;
  if (rows > 0 && cols > 0 && !p) return CASC_ERR_INVALID;
  return CASC_OK;
}

// X (= B, overwritten) must not overlap the triangle A or itself (both TRSMs)
bool trsm_overlap(int64_t m, int64_t n, const double* A_hi, const double* A_lo, int64_t lda,
                  const double* B_hi, const double* B_lo, int64_t ldb) {
  const size_t ea = extent(m, m, lda), eb = extent(m, n, ldb);
  return ranges_overlap(B_hi, eb, A_hi, ea) || ranges_overlap(B_hi, eb, A_lo, ea) ||
         ranges_overlap(B_lo, eb, A_hi, ea) || ranges_overlap(B_lo, eb, A_lo, ea) ||
         ranges_overlap(B_hi, eb, B_lo, eb);
}

int cuda_status(cudaError_t e) { return e == cudaSuccess ? CASC_OK : CASC_ERR_CUDA; }

struct AlphaBeta {
  int ab = 0;  // 0 none, 1 alpha, 2 alpha and beta
  double ah = 1.0, al = 0.0, bh = 0.0, bl = 0.0;
};

// Split mode for small problems: when one work item per 64x64 tile leaves the
// last wave of the 148 SMs badly filled, use one item per (tile, k panel) and
// reduce the FP64x2 panel sums in panel order afterwards (bitwise the same
// result).  Returns P (> 1) or 0.
int split_plan(int64_t m, int64_t n, int64_t k, int sms) {
  const int64_t P = casc::panels_of(k);
  if (P < 2 || sms <= 0) return 0;
  const char* env = getenv("CASC_SPLIT_MODE");  // "0": never (tests compare both modes)
  if (env && env[0] == '0') return 0;
  const int64_t tiles = ((m + casc::TM - 1) / casc::TM) * ((n + casc::TN - 1) / casc::TN);
  if (tiles >= 2 * (int64_t)sms) return 0;  // enough waves already
  const int64_t units = tiles * P;
  const double eff_t = (double)tiles / (double)(((tiles + sms - 1) / sms) * sms);
  const double eff_s = (double)units / (double)(((units + sms - 1) / sms) * sms);
  if (eff_s < eff_t + 0.04) return 0;
  if ((double)P * (m + 63) * (n + 63) * 17.0 > (double)(1ull << 31)) return 0;
  return (int)P;
}
size_t split_bytes(int64_t m, int64_t n, int P) {  // tile-major panel sums + flags, padded tiles
  const int64_t padded = (m + casc::TM - 1) / casc::TM * ((n + casc::TN - 1) / casc::TN) *
                         (casc::TM * casc::TN);
  return P ? ((size_t)P * padded * 17 + 255) / 256 * 256 : 0;
}
// the fused kernel's per-launch scratch (wave counter, WIDE list) at the end of a
// workspace: sized for the most work items a call with (m, n, k) can have
size_t scratch_bytes_for(int64_t m, int64_t n, int P) {
  const int64_t tiles = ((m + casc::TM - 1) / casc::TM) * ((n + casc::TN - 1) / casc::TN);
  return casc::gemm_scratch_bytes(tiles * (P > 1 ? P : 1));
}

int current_sms() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 148;  // B200
  }
  return sms;
}

int gemm_packed_impl(int64_t m, int64_t n, int64_t k, const void* pa, const void* pb,
                     double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags, int sms,
                     cudaStream_t st, int st_begin, int st_end, double* dbg,
                     const AlphaBeta& abv = AlphaBeta(), void* split_ws = nullptr, int tri = 0,
                     void* scratch = nullptr, int64_t ldf = -1, bool pdl = false,
                     int band = 0) {
  const casc::Widths w = widths_for(k);
  casc::GemmArgs a{};
  a.ab = abv.ab;
  a.alpha_hi = abv.ah;
  a.alpha_lo = abv.al;
  a.beta_hi = abv.bh;
  a.beta_lo = abv.bl;
  a.pa = static_cast<const uint8_t*>(pa);
  a.pb = static_cast<const uint8_t*>(pb);
  a.a_blk = casc::a_block_bytes(k);
  a.b_blk = casc::b_block_bytes(k);
  a.a_exp = casc::a_exp_offset(k);
  a.b_exp = casc::b_exp_offset(k);
  a.m = m;
  a.n = n;
  a.mblocks = (int)((m + casc::TM - 1) / casc::TM);
  a.nblocks = (int)((n + casc::TN - 1) / casc::TN);
  a.st_begin = st_begin;
  a.st_end = st_end;
  a.c0 = w.c0;
  a.D2 = w.c0 + w.c1 + w.c2;
  a.C_hi = C_hi;
  a.C_lo = C_lo;
  a.ldc = ldc;
  a.flags = flags;
  a.ldf = ldf < 0 ? n : ldf;
  a.dbg = dbg;
  a.un_b2 = std::ldexp(1.0, w.c1 - w.c0);
  a.tri = tri;
  a.band = band;
  const int nst = (int)(casc::kpad_of(k) / casc::BK);
  const int P = (!dbg && !tri && !band && st_begin == 0 && st_end == nst)
                    ? split_plan(m, n, k, sms) : 0;
  // per-launch scratch of the fused kernel (wave counter, WIDE list): the caller's
  // workspace slot, else a stream-ordered allocation of this call (never shared
  // between launches or streams)
  const int64_t items = P ? (int64_t)a.mblocks * a.nblocks * P
                          : (tri ? (int64_t)a.mblocks * (a.mblocks + 1) / 2
                                 : (int64_t)a.mblocks * a.nblocks);
  bool own_scratch = false;
  if (!dbg && !scratch) {
    if (cudaMallocAsync(&scratch, casc::gemm_scratch_bytes(items), st) != cudaSuccess)
      return CASC_ERR_CUDA;
    own_scratch = true;
  }
  a.scratch = scratch;
  a.pdl = (pdl && !own_scratch && !dbg) ? 1 : 0;
  if (!P) {
    cudaError_t e = casc::launch_gemm(a, sms, st);
    if (own_scratch) cudaFreeAsync(scratch, st);
    if (e == cudaSuccess) g_launches += dbg ? 1 : 2;
    return cuda_status(e);
  }
  void* buf = split_ws;
  if (!buf && cudaMallocAsync(&buf, split_bytes(m, n, P), st) != cudaSuccess) {
    if (own_scratch) cudaFreeAsync(scratch, st);
    return CASC_ERR_CUDA;
  }
  const int64_t mn = (int64_t)a.mblocks * a.nblocks * (casc::TM * casc::TN);  // padded
  a.split_p = P;
  a.t_hi = static_cast<double*>(buf);
  a.t_lo = a.t_hi + (int64_t)P * mn;
  a.fbuf = reinterpret_cast<uint8_t*>(a.t_lo + (int64_t)P * mn);
  a.ab = 0;  // alpha / beta go to the reduction
  cudaError_t e = casc::launch_gemm(a, sms, st);
  if (e == cudaSuccess)
    e = casc::launch_split_reduce(P, m, n, a.t_hi, a.t_lo, a.fbuf, C_hi, C_lo, ldc, flags, a.ldf,
                                  abv.ab, abv.ah, abv.al, abv.bh, abv.bl, sms, st);
  if (!split_ws) cudaFreeAsync(buf, st);
  if (own_scratch) cudaFreeAsync(scratch, st);
  if (e == cudaSuccess) g_launches += 3;
  return cuda_status(e);
}


}  // namespace

extern "C" {

const char* casc_status_string(int status) {
  switch (status) {
    case CASC_OK: return "CASC_OK";
    case CASC_ERR_INVALID: return "CASC_ERR_INVALID: invalid argument";
    case CASC_ERR_CUDA: return "CASC_ERR_CUDA: CUDA runtime/launch/allocation error";
    case CASC_ERR_UNSUPPORTED: return "CASC_ERR_UNSUPPORTED: device is not sm_100 (B200)";
    default: return "CASC_ERR_UNKNOWN";
  }
}

int casc_select_widths(int64_t k, int* c) {
  if (!c || k < 0) return CASC_ERR_INVALID;
  const casc::Widths w = widths_for(k);
  c[0] = w.c0;
  c[1] = w.c1;
  c[2] = w.c2;
  return CASC_OK;
}

size_t casc_packed_a_block_bytes(int64_t k) { return k > 0 ? (size_t)casc::a_block_bytes(k) : 0; }
size_t casc_packed_b_block_bytes(int64_t k) { return k > 0 ? (size_t)casc::b_block_bytes(k) : 0; }
size_t casc_packed_a_bytes(int64_t m, int64_t k) {
  if (m <= 0 || k <= 0) return 0;
  return (size_t)((m + casc::TM - 1) / casc::TM) * casc_packed_a_block_bytes(k);
}
size_t casc_packed_b_bytes(int64_t k, int64_t n) {
  if (n <= 0 || k <= 0) return 0;
  return (size_t)((n + casc::TN - 1) / casc::TN) * casc_packed_b_block_bytes(k);
}
size_t casc_workspace_bytes(int64_t m, int64_t n, int64_t k) {
  const size_t a = (casc_packed_a_bytes(m, k) + 255) / 256 * 256;
  const size_t b = (casc_packed_b_bytes(k, n) + 255) / 256 * 256;
  const int P = (m > 0 && n > 0 && k > 0) ? split_plan(m, n, k, current_sms()) : 0;
  return a + b + split_bytes(m, n, P) + scratch_bytes_for(m, n, P);
}
// the fused kernel's scratch inside a workspace of casc_workspace_bytes(m, n, k) bytes
static void* ws_counter(void* ws, int64_t m, int64_t n, int64_t k) {
  const int P = (m > 0 && n > 0 && k > 0) ? split_plan(m, n, k, current_sms()) : 0;
  return static_cast<uint8_t*>(ws) + casc_workspace_bytes(m, n, k) - scratch_bytes_for(m, n, P);
}

int casc_last_launch_count(void) { return g_launches; }

int casc_pack_a(int64_t m, int64_t k, const double* A_hi, const double* A_lo, int64_t lda,
                void* packed_a, casc_stream_t stream) {
  g_launches = 0;
  int r;
  if ((r = check_mat(A_hi, m, k, lda)) || (r = check_mat(A_lo, m, k, lda))) return r;
  if (m > 0 && k > 0 && !packed_a) return CASC_ERR_INVALID;
  if ((r = device_check(nullptr))) return r;
  if (m == 0 || k == 0) return CASC_OK;
  cudaError_t e = casc::launch_split_a(A_hi, A_lo, lda, m, k, widths_for(k), packed_a, S(stream));
  if (e == cudaSuccess) ++g_launches;
  return cuda_status(e);
}

int casc_pack_b(int64_t k, int64_t n, const double* B_hi, const double* B_lo, int64_t ldb,
                void* packed_b, casc_stream_t stream) {
  g_launches = 0;
  int r;
  if ((r = check_mat(B_hi, k, n, ldb)) || (r = check_mat(B_lo, k, n, ldb))) return r;
  if (n > 0 && k > 0 && !packed_b) return CASC_ERR_INVALID;
  if ((r = device_check(nullptr))) return r;
  if (n == 0 || k == 0) return CASC_OK;
  cudaError_t e = casc::launch_split_b(B_hi, B_lo, ldb, k, n, widths_for(k), packed_b, S(stream));
  if (e == cudaSuccess) ++g_launches;
  return cuda_status(e);
}

static int zero_c(int64_t m, int64_t n, double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
                  cudaStream_t st, int64_t ldf = -1) {
  cudaError_t e = cudaMemset2DAsync(C_hi, ldc * sizeof(double), 0, n * sizeof(double), m, st);
  if (e == cudaSuccess)
    e = cudaMemset2DAsync(C_lo, ldc * sizeof(double), 0, n * sizeof(double), m, st);
  if (e == cudaSuccess && flags)
    e = cudaMemset2DAsync(flags, (size_t)(ldf < 0 ? n : ldf), 0, (size_t)n, (size_t)m, st);
  return cuda_status(e);
}

int casc_gemm_packed_ld(int64_t m, int64_t n, int64_t k, const void* packed_a,
                        const void* packed_b, double* C_hi, double* C_lo, int64_t ldc,
                        uint8_t* flags, int64_t ldf, casc_stream_t stream) {
  g_launches = 0;
  int r;
  if (m < 0 || n < 0 || k < 0) return CASC_ERR_INVALID;
  if ((r = check_mat(C_hi, m, n, ldc)) || (r = check_mat(C_lo, m, n, ldc))) return r;
  if (flags && ldf < (n > 1 ? n : 1)) return CASC_ERR_INVALID;
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = device_check(&sms))) return r;
  if (k == 0) return zero_c(m, n, C_hi, C_lo, ldc, flags, S(stream), ldf);
  if (!packed_a || !packed_b) return CASC_ERR_INVALID;
  const int nst = (int)(casc::kpad_of(k) / casc::BK);
  return gemm_packed_impl(m, n, k, packed_a, packed_b, C_hi, C_lo, ldc, flags, sms, S(stream), 0,
                          nst, nullptr, AlphaBeta(), nullptr, 0, nullptr, ldf);
}

int casc_gemm_packed(int64_t m, int64_t n, int64_t k, const void* packed_a, const void* packed_b,
                     double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
                     casc_stream_t stream) {
  return casc_gemm_packed_ld(m, n, k, packed_a, packed_b, C_hi, C_lo, ldc, flags, n, stream);
}

static int validate_gemm(int64_t m, int64_t n, int64_t k, const double* A_hi, const double* A_lo,
                         int64_t lda, const double* B_hi, const double* B_lo, int64_t ldb,
                         double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags) {
  int r;
  if (m < 0 || n < 0 || k < 0) return CASC_ERR_INVALID;
  if ((r = check_mat(A_hi, m, k, lda)) || (r = check_mat(A_lo, m, k, lda))) return r;
  if ((r = check_mat(B_hi, k, n, ldb)) || (r = check_mat(B_lo, k, n, ldb))) return r;
  if ((r = check_mat(C_hi, m, n, ldc)) || (r = check_mat(C_lo, m, n, ldc))) return r;
  const size_t ca = extent(m, k, lda), cb = extent(k, n, ldb), cc = extent(m, n, ldc);
  const void* ins[4] = {A_hi, A_lo, B_hi, B_lo};
  const size_t ine[4] = {ca, ca, cb, cb};
  void* outs[3] = {C_hi, C_lo, flags};
  const size_t oute[3] = {cc, cc, flags ? (size_t)(m * n) : 0};
  for (int o = 0; o < 3; ++o) {
    for (int i = 0; i < 4; ++i)
      if (ranges_overlap(outs[o], oute[o], ins[i], ine[i])) return CASC_ERR_INVALID;
    for (int o2 = o + 1; o2 < 3; ++o2)
      if (ranges_overlap(outs[o], oute[o], outs[o2], oute[o2])) return CASC_ERR_INVALID;
  }
  return CASC_OK;
}

int casc_gemm_fp64x2_ws(int64_t m, int64_t n, int64_t k, const double* A_hi, const double* A_lo,
                        int64_t lda, const double* B_hi, const double* B_lo, int64_t ldb,
                        double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags, void* workspace,
                        size_t workspace_bytes, casc_stream_t stream) {
  int r = validate_gemm(m, n, k, A_hi, A_lo, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, flags);
  if (r) return r;
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = device_check(&sms))) return r;
  if (k == 0) return zero_c(m, n, C_hi, C_lo, ldc, flags, S(stream));
  const size_t need = casc_workspace_bytes(m, n, k);
  if (!workspace || workspace_bytes < need) return CASC_ERR_INVALID;
  uint8_t* pa = static_cast<uint8_t*>(workspace);
  uint8_t* pb = pa + (casc_packed_a_bytes(m, k) + 255) / 256 * 256;
  const casc::Widths w = widths_for(k);
  // the fused kernel's scratch head is zeroed first, so that the split launch
  // and the product launch are adjacent (programmatic dependent launch)
  void* scr = ws_counter(workspace, m, n, k);
  {  // the launch's work items: one per tile, or per (tile, panel) in split mode
    const int Pz = split_plan(m, n, k, sms);
    const int64_t items = ((m + casc::TM - 1) / casc::TM) * ((n + casc::TN - 1) / casc::TN) *
                          (Pz ? Pz : 1);
    if (cudaMemsetAsync(scr, 0, casc::gemm_scratch_zero_bytes(items), S(stream)) != cudaSuccess)
      return CASC_ERR_CUDA;
  }
  // phase 1: both splits in one launch
  cudaError_t e = casc::launch_split_ab(A_hi, A_lo, lda, m, B_hi, B_lo, ldb, n, k, w, pa, pb,
                                        S(stream), false, false);
  if (e != cudaSuccess) return CASC_ERR_CUDA;
  const int nst = (int)(casc::kpad_of(k) / casc::BK);
  uint8_t* ps = pb + (casc_packed_b_bytes(k, n) + 255) / 256 * 256;  // split-mode buffer
  g_launches = 0;
  r = gemm_packed_impl(m, n, k, pa, pb, C_hi, C_lo, ldc, flags, sms, S(stream), 0, nst, nullptr,
                       AlphaBeta(), ps, 0, scr, -1, true);
  g_launches = (r == CASC_OK) ? g_launches + 1 : 0;  // + the split launch
  return r;
}

int casc_gemm_fp64x2(int64_t m, int64_t n, int64_t k, const double* A_hi, const double* A_lo,
                     int64_t lda, const double* B_hi, const double* B_lo, int64_t ldb,
                     double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
                     casc_stream_t stream) {
  int r = validate_gemm(m, n, k, A_hi, A_lo, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, flags);
  if (r) return r;
  if (m == 0 || n == 0 || k == 0)
    return casc_gemm_fp64x2_ws(m, n, k, A_hi, A_lo, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, flags,
                               nullptr, 0, stream);
  if ((r = device_check(nullptr))) return r;
  // Stream-ordered workspace of this call (the device's default pool keeps the
  // memory cached: release threshold set in device_check): no host
  // synchronisation, and concurrent calls on different streams never share it.
  const size_t need = casc_workspace_bytes(m, n, k);
  const cudaStream_t st = S(stream);
  void* ws = nullptr;
  if (cudaMallocAsync(&ws, need, st) != cudaSuccess) return CASC_ERR_CUDA;
  r = casc_gemm_fp64x2_ws(m, n, k, A_hi, A_lo, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, flags, ws,
                          need, stream);
  const int launches = g_launches;
  cudaFreeAsync(ws, st);
  g_launches = launches;
  return r;
}

// Host-resident operands (casc.h), the row-slab pipeline of casc_host.cuh.
int casc_gemm_fp64x2_host(int64_t m, int64_t n, int64_t k, const double* A_hi, const double* A_lo,
                          int64_t lda, const double* B_hi, const double* B_lo, int64_t ldb,
                          double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
                          int64_t slab_rows, int64_t slab_cols, casc_stream_t stream) {
  g_launches = 0;
  int r = validate_gemm(m, n, k, A_hi, A_lo, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, flags);
  if (r) return r;
  if (slab_rows < 0 || slab_cols < 0) return CASC_ERR_INVALID;
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = device_check(&sms))) return r;
  const cudaStream_t st = S(stream);
  if (k == 0) return casc::hostpipe::zero_host_c(m, n, C_hi, C_lo, ldc, flags, st);
  auto fit = [](int64_t v, int64_t blk, int64_t lim) {  // block multiple, at most lim rounded
    v = (v + blk - 1) / blk * blk;
    const int64_t l = (lim + blk - 1) / blk * blk;
    return v < l ? v : l;
  };
  int64_t dr = casc::hostpipe::default_slab(m), dc = casc::hostpipe::default_slab(n);
  if (m >= 8192 && n >= 8192) {
    // large operands: wave-aligned blocks, so that no block GEMM ends on a
    // partly filled wave of 64 x 64 tiles (16384^3 on 148 SMs: 4096 x 2368 =
    // 2368 tiles = 16 full waves; 4096 x 4096 would be 27.7 waves; measured
    // e2e 2532 -> 2499 ms, scripts/e2e_slabs.py)
    dr = 4096;
    const int64_t rb = dr / casc::TM;
    for (int64_t nb = 32; nb <= 96; ++nb)
      if ((rb * nb) % sms == 0) {
        dc = nb * casc::TN;
        break;
      }
  }
  const int64_t sr = fit(slab_rows ? slab_rows : dr, casc::TM, m);
  const int64_t sc = fit(slab_cols ? slab_cols : dc, casc::TN, n);
  const casc::Widths w = widths_for(k);
  const int nst = (int)(casc::kpad_of(k) / casc::BK);
  int launches = 0;
  auto pack_b = [&](const double* bh, const double* bl, int64_t cols, void* pb) {
    const cudaError_t e = casc::launch_split_b(bh, bl, cols, k, cols, w, pb, st);
    launches += e == cudaSuccess;
    return cuda_status(e);
  };
  auto pack_a = [&](const double* ah, const double* al, int64_t rows, void* pa) {
    const cudaError_t e = casc::launch_split_a(ah, al, k, rows, k, w, pa, st);
    launches += e == cudaSuccess;
    return cuda_status(e);
  };
  auto gemm = [&](int64_t rows, int64_t cols, const void* pa, const void* pb, double* ch,
                  double* cl, uint8_t* fl) {
    g_launches = 0;
    const int rr =
        gemm_packed_impl(rows, cols, k, pa, pb, ch, cl, cols, fl, sms, st, 0, nst, nullptr);
    launches += g_launches;
    return rr;
  };
  // large operands with the default blocks: first slabs of 1024 rows / columns,
  // so the exposed first copy is 0.5 GB instead of 1.6 GB at 16384^3
  const bool small_first = m >= 8192 && n >= 8192;
  const int64_t sr0 = (small_first && !slab_rows) ? fit(1024, casc::TM, m) : sr;
  const int64_t sc0 = (small_first && !slab_cols) ? fit(1024, casc::TN, n) : sc;
  r = casc::hostpipe::run(m, n, k, A_hi, A_lo, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, flags, sr,
                          sc, casc_packed_b_bytes(k, sc), casc_packed_a_bytes(sr, k), st, pack_b,
                          pack_a, gemm, sr0, sc0);
  g_launches = r == CASC_OK ? launches : 0;
  return r;
}

int casc_finalize(void) {
  // Return the cached stream-ordered memory of this device's default pool (the
  // workspaces of casc_gemm_fp64x2 / casc_i8_gemm_fp64x2) to the system.  A
  // teardown call: it waits for the device's work first.
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return CASC_ERR_CUDA;
  if (cudaDeviceSynchronize() != cudaSuccess) return CASC_ERR_CUDA;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return CASC_ERR_CUDA;
  return cuda_status(cudaMemPoolTrimTo(pool, 0));
}

int casc_split_a(int64_t m, int64_t k, const double* A_hi, const double* A_lo, int64_t lda,
                 double* slices, int32_t* e, casc_stream_t stream) {
  g_launches = 0;
  int r;
  if ((r = check_mat(A_hi, m, k, lda)) || (r = check_mat(A_lo, m, k, lda))) return r;
  if (m > 0 && k > 0 && (!slices || !e)) return CASC_ERR_INVALID;
  if ((r = device_check(nullptr))) return r;
  if (m == 0 || k == 0) return CASC_OK;
  void* tmp = nullptr;
  cudaStream_t st = S(stream);
  if (cudaMallocAsync(&tmp, casc_packed_a_bytes(m, k), st) != cudaSuccess) return CASC_ERR_CUDA;
  const casc::Widths w = widths_for(k);
  cudaError_t err = casc::launch_split_a(A_hi, A_lo, lda, m, k, w, tmp, st);
  if (err == cudaSuccess) err = casc::launch_unpack_a(tmp, m, k, w, slices, e, st);
  cudaFreeAsync(tmp, st);
  if (err == cudaSuccess) g_launches = 2;
  return cuda_status(err);
}

int casc_split_b(int64_t k, int64_t n, const double* B_hi, const double* B_lo, int64_t ldb,
                 double* slices, int32_t* f, casc_stream_t stream) {
  g_launches = 0;
  int r;
  if ((r = check_mat(B_hi, k, n, ldb)) || (r = check_mat(B_lo, k, n, ldb))) return r;
  if (n > 0 && k > 0 && (!slices || !f)) return CASC_ERR_INVALID;
  if ((r = device_check(nullptr))) return r;
  if (n == 0 || k == 0) return CASC_OK;
  void* tmp = nullptr;
  cudaStream_t st = S(stream);
  if (cudaMallocAsync(&tmp, casc_packed_b_bytes(k, n), st) != cudaSuccess) return CASC_ERR_CUDA;
  const casc::Widths w = widths_for(k);
  cudaError_t err = casc::launch_split_b(B_hi, B_lo, ldb, k, n, w, tmp, st);
  if (err == cudaSuccess) err = casc::launch_unpack_b(tmp, k, n, w, slices, f, st);
  cudaFreeAsync(tmp, st);
  if (err == cudaSuccess) g_launches = 2;
  return cuda_status(err);
}

int casc_debug_bins(int64_t m, int64_t n, int64_t k, const double* A_hi, const double* A_lo,
                    int64_t lda, const double* B_hi, const double* B_lo, int64_t ldb,
                    int64_t panel, double* bins, casc_stream_t stream) {
  g_launches = 0;
  int r;
  if (m < 0 || n < 0 || k < 0) return CASC_ERR_INVALID;
  if ((r = check_mat(A_hi, m, k, lda)) || (r = check_mat(A_lo, m, k, lda))) return r;
  if ((r = check_mat(B_hi, k, n, ldb)) || (r = check_mat(B_lo, k, n, ldb))) return r;
  if (panel < 0 || panel >= casc::panels_of(k)) return CASC_ERR_INVALID;
  if (m == 0 || n == 0) return CASC_OK;
  if (!bins) return CASC_ERR_INVALID;
  int sms = 0;
  if ((r = device_check(&sms))) return r;
  cudaStream_t st = S(stream);
  void* pa = nullptr;
  void* pb = nullptr;
  if (cudaMallocAsync(&pa, casc_packed_a_bytes(m, k), st) != cudaSuccess) return CASC_ERR_CUDA;
  if (cudaMallocAsync(&pb, casc_packed_b_bytes(k, n), st) != cudaSuccess) {
    cudaFreeAsync(pa, st);
    return CASC_ERR_CUDA;
  }
  const casc::Widths w = widths_for(k);
  cudaError_t err = casc::launch_split_a(A_hi, A_lo, lda, m, k, w, pa, st);
  if (err == cudaSuccess) err = casc::launch_split_b(B_hi, B_lo, ldb, k, n, w, pb, st);
  const int nst = (int)(casc::kpad_of(k) / casc::BK);
  const int s0 = (int)panel * casc::STAGES_PER_PANEL;
  const int s1 = s0 + casc::STAGES_PER_PANEL < nst ? s0 + casc::STAGES_PER_PANEL : nst;
  if (err == cudaSuccess)
    r = gemm_packed_impl(m, n, k, pa, pb, nullptr, nullptr, n, nullptr, sms, st, s0, s1, bins);
  else
    r = CASC_ERR_CUDA;
  cudaFreeAsync(pa, st);
  cudaFreeAsync(pb, st);
  if (r == CASC_OK) g_launches = 3;
  return r;
}

int casc_debug_ldexp(int64_t count, const double* x, const int32_t* n, double* out,
                     casc_stream_t stream) {
  g_launches = 0;
  if (count < 0 || (count > 0 && (!x || !n || !out))) return CASC_ERR_INVALID;
  int r;
  if ((r = device_check(nullptr))) return r;
  const cudaError_t e = casc::launch_ldexp(count, x, n, out, S(stream));
  if (e == cudaSuccess && count > 0) g_launches = 1;
  return cuda_status(e);
}

// ---------------------------------------------------------------- BLAS-style (NEXT-4)
static int gemm_ex_impl(int transa, int transb, int64_t m, int64_t n, int64_t k,
                        double alpha_hi, double alpha_lo, const double* A_hi, const double* A_lo,
                        int64_t lda, const double* B_hi, const double* B_lo, int64_t ldb,
                        double beta_hi, double beta_lo, double* C_hi, double* C_lo, int64_t ldc,
                        uint8_t* flags, void* workspace, size_t workspace_bytes,
                        casc_stream_t stream, int band);

int casc_gemm_fp64x2_ex(int transa, int transb, int64_t m, int64_t n, int64_t k,
                        double alpha_hi, double alpha_lo, const double* A_hi, const double* A_lo,
                        int64_t lda, const double* B_hi, const double* B_lo, int64_t ldb,
                        double beta_hi, double beta_lo, double* C_hi, double* C_lo, int64_t ldc,
                        uint8_t* flags, void* workspace, size_t workspace_bytes,
                        casc_stream_t stream) {
  return gemm_ex_impl(transa, transb, m, n, k, alpha_hi, alpha_lo, A_hi, A_lo, lda, B_hi, B_lo,
                      ldb, beta_hi, beta_lo, C_hi, C_lo, ldc, flags, workspace, workspace_bytes,
                      stream, 0);
}

}  // extern "C"

static int gemm_ex_impl(int transa, int transb, int64_t m, int64_t n, int64_t k,
                        double alpha_hi, double alpha_lo, const double* A_hi, const double* A_lo,
                        int64_t lda, const double* B_hi, const double* B_lo, int64_t ldb,
                        double beta_hi, double beta_lo, double* C_hi, double* C_lo, int64_t ldc,
                        uint8_t* flags, void* workspace, size_t workspace_bytes,
                        casc_stream_t stream, int band) {
  g_launches = 0;
  if ((transa != CASC_OP_N && transa != CASC_OP_T) || (transb != CASC_OP_N && transb != CASC_OP_T))
    return CASC_ERR_INVALID;
  if (m < 0 || n < 0 || k < 0) return CASC_ERR_INVALID;
  // stored shapes: op(A) is m x k (A stored k x m if transposed), op(B) is k x n
  const int64_t ar = transa ? k : m, ac = transa ? m : k;
  const int64_t br = transb ? n : k, bc = transb ? k : n;
  const bool no_product = (k == 0) || (alpha_hi == 0.0 && alpha_lo == 0.0);
  int r;
  if (!no_product) {
    if ((r = check_mat(A_hi, ar, ac, lda)) || (r = check_mat(A_lo, ar, ac, lda))) return r;
    if ((r = check_mat(B_hi, br, bc, ldb)) || (r = check_mat(B_lo, br, bc, ldb))) return r;
  }
  if ((r = check_mat(C_hi, m, n, ldc)) || (r = check_mat(C_lo, m, n, ldc))) return r;
  if (!no_product) {
    const size_t ea = extent(ar, ac, lda), eb = extent(br, bc, ldb), ec = extent(m, n, ldc);
    const void* ins[4] = {A_hi, A_lo, B_hi, B_lo};
    const size_t ine[4] = {ea, ea, eb, eb};
    void* outs[3] = {C_hi, C_lo, flags};
    const size_t oute[3] = {ec, ec, flags ? (size_t)(m * n) : 0};
    for (int o = 0; o < 3; ++o)
      for (int i = 0; i < 4; ++i)
        if (ranges_overlap(outs[o], oute[o], ins[i], ine[i])) return CASC_ERR_INVALID;
  }
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = device_check(&sms))) return r;
  cudaStream_t st = S(stream);
  const bool use_beta = !(beta_hi == 0.0 && beta_lo == 0.0);
  if (no_product) {  // C := beta C (BLAS: A and B are not referenced)
    cudaError_t e = casc::launch_scale_c(m, n, beta_hi, beta_lo, use_beta, C_hi, C_lo, ldc, flags,
                                         sms, st);
    if (e == cudaSuccess) g_launches = 1;
    return cuda_status(e);
  }
  const size_t need = casc_workspace_bytes(m, n, k);
  void* ws = workspace;
  bool owned = false;
  if (!ws) {
    if (cudaMallocAsync(&ws, need, st) != cudaSuccess) return CASC_ERR_CUDA;
    owned = true;
  } else if (workspace_bytes < need) {
    return CASC_ERR_INVALID;
  }
  uint8_t* pa = static_cast<uint8_t*>(ws);
  uint8_t* pb = pa + (casc_packed_a_bytes(m, k) + 255) / 256 * 256;
  const casc::Widths w = widths_for(k);
  cudaError_t e = casc::launch_split_ab(A_hi, A_lo, lda, m, B_hi, B_lo, ldb, n, k, w, pa, pb, st,
                                        transa == CASC_OP_T, transb == CASC_OP_T);
  AlphaBeta abv;
  const bool unit_alpha = (alpha_hi == 1.0 && alpha_lo == 0.0);
  abv.ab = use_beta ? 2 : (unit_alpha ? 0 : 1);
  abv.ah = alpha_hi;
  abv.al = alpha_lo;
  abv.bh = beta_hi;
  abv.bl = beta_lo;
  const int nst = (int)(casc::kpad_of(k) / casc::BK);
  uint8_t* ps = pb + (casc_packed_b_bytes(k, n) + 255) / 256 * 256;  // split-mode buffer
  g_launches = 0;
  r = (e == cudaSuccess) ? gemm_packed_impl(m, n, k, pa, pb, C_hi, C_lo, ldc, flags, sms, st, 0,
                                            nst, nullptr, abv, ps, 0, ws_counter(ws, m, n, k), -1,
                                            false, band)
                         : CASC_ERR_CUDA;
  if (owned) cudaFreeAsync(ws, st);
  g_launches = (r == CASC_OK) ? g_launches + 1 : 0;
  return r;
}

extern "C" {

// ---------------------------------------------------------------- SYRK (NEXT-4)
// C := alpha op(A) op(A)^T + beta C on one triangle (level-3 BLAS
// on the cascaded GEMM).  op(A) is split once as the A operand and, read
// transposed, as the B operand; the fused kernel runs only the triangle's
// tiles (half the work) and stores only the triangle's elements.
int casc_syrk_fp64x2(int uplo, int trans, int64_t n, int64_t k, double alpha_hi, double alpha_lo,
                     const double* A_hi, const double* A_lo, int64_t lda, double beta_hi,
                     double beta_lo, double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
                     void* workspace, size_t workspace_bytes, casc_stream_t stream) {
  g_launches = 0;
  if ((uplo != CASC_LOWER && uplo != CASC_UPPER) || (trans != CASC_OP_N && trans != CASC_OP_T))
    return CASC_ERR_INVALID;
  if (n < 0 || k < 0) return CASC_ERR_INVALID;
  const int64_t ar = trans ? k : n, ac = trans ? n : k;  // A as stored
  const bool no_product = (k == 0) || (alpha_hi == 0.0 && alpha_lo == 0.0);
  int r;
  if (!no_product && ((r = check_mat(A_hi, ar, ac, lda)) || (r = check_mat(A_lo, ar, ac, lda))))
    return r;
  if ((r = check_mat(C_hi, n, n, ldc)) || (r = check_mat(C_lo, n, n, ldc))) return r;
  if (!no_product) {
    const size_t ea = extent(ar, ac, lda), ec = extent(n, n, ldc);
    const void* ins[2] = {A_hi, A_lo};
    void* outs[3] = {C_hi, C_lo, flags};
    const size_t oute[3] = {ec, ec, flags ? (size_t)(n * n) : 0};
    for (int o = 0; o < 3; ++o)
      for (int i = 0; i < 2; ++i)
        if (ranges_overlap(outs[o], oute[o], ins[i], ea)) return CASC_ERR_INVALID;
  }
  if (n == 0) return CASC_OK;
  int sms = 0;
  if ((r = device_check(&sms))) return r;
  cudaStream_t st = S(stream);
  const bool use_beta = !(beta_hi == 0.0 && beta_lo == 0.0);
  if (no_product) {  // C := beta C on the triangle
    cudaError_t e = casc::launch_scale_c_uplo(n, n, beta_hi, beta_lo, use_beta, C_hi, C_lo, ldc,
                                              flags, sms, uplo == CASC_LOWER ? 0 : 1, st);
    if (e == cudaSuccess) g_launches = 1;
    return cuda_status(e);
  }
  const size_t need = casc_workspace_bytes(n, n, k);
  void* ws = workspace;
  bool owned = false;
  if (!ws) {
    if (cudaMallocAsync(&ws, need, st) != cudaSuccess) return CASC_ERR_CUDA;
    owned = true;
  } else if (workspace_bytes < need) {
    return CASC_ERR_INVALID;
  }
  uint8_t* pa = static_cast<uint8_t*>(ws);
  uint8_t* pb = pa + (casc_packed_a_bytes(n, k) + 255) / 256 * 256;
  const casc::Widths w = widths_for(k);
  // op(A) (n x k) as the A operand; op(A)^T (k x n) as the B operand: stored as A
  // itself, read transposed when trans == N
  cudaError_t e = casc::launch_split_ab(A_hi, A_lo, lda, n, A_hi, A_lo, lda, n, k, w, pa, pb, st,
                                        trans == CASC_OP_T, trans == CASC_OP_N);
  AlphaBeta abv;
  abv.ab = use_beta ? 2 : ((alpha_hi == 1.0 && alpha_lo == 0.0) ? 0 : 1);  // as casc_gemm_fp64x2_ex
  abv.ah = alpha_hi;
  abv.al = alpha_lo;
  abv.bh = beta_hi;
  abv.bl = beta_lo;
  const int nst = (int)(casc::kpad_of(k) / casc::BK);
  g_launches = 0;
  r = (e == cudaSuccess) ? gemm_packed_impl(n, n, k, pa, pb, C_hi, C_lo, ldc, flags, sms, st, 0,
                                            nst, nullptr, abv, nullptr,
                                            uplo == CASC_LOWER ? 1 : 2, ws_counter(ws, n, n, k))
                         : CASC_ERR_CUDA;
  if (owned) cudaFreeAsync(ws, st);
  g_launches = (r == CASC_OK) ? g_launches + 1 : 0;
  return r;
}

// ---------------------------------------------------------------- SYR2K (NEXT-4)
// C := alpha op(A) op(B)^T + alpha op(B) op(A)^T + beta C on one triangle
// (reading R30): two triangular launches of the fused kernel (half the tiles
// each), the second with beta = 1 on the first's result; flags ORed.
int casc_syr2k_fp64x2(int uplo, int trans, int64_t n, int64_t k, double alpha_hi, double alpha_lo,
                      const double* A_hi, const double* A_lo, int64_t lda, const double* B_hi,
                      const double* B_lo, int64_t ldb, double beta_hi, double beta_lo,
                      double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
                      casc_stream_t stream) {
  g_launches = 0;
  if ((uplo != CASC_LOWER && uplo != CASC_UPPER) || (trans != CASC_OP_N && trans != CASC_OP_T))
    return CASC_ERR_INVALID;
  if (n < 0 || k < 0) return CASC_ERR_INVALID;
  const int64_t ar = trans ? k : n, ac = trans ? n : k;  // A, B as stored
  const bool no_product = (k == 0) || (alpha_hi == 0.0 && alpha_lo == 0.0);
  int r;
  if (!no_product &&
      ((r = check_mat(A_hi, ar, ac, lda)) || (r = check_mat(A_lo, ar, ac, lda)) ||
       (r = check_mat(B_hi, ar, ac, ldb)) || (r = check_mat(B_lo, ar, ac, ldb))))
    return r;
  if ((r = check_mat(C_hi, n, n, ldc)) || (r = check_mat(C_lo, n, n, ldc))) return r;
  if (!no_product) {
    const void* ins[4] = {A_hi, A_lo, B_hi, B_lo};
    const size_t ine[4] = {extent(ar, ac, lda), extent(ar, ac, lda), extent(ar, ac, ldb),
                           extent(ar, ac, ldb)};
    void* outs[3] = {C_hi, C_lo, flags};
    const size_t oute[3] = {extent(n, n, ldc), extent(n, n, ldc), flags ? (size_t)(n * n) : 0};
    for (int o = 0; o < 3; ++o)
      for (int i = 0; i < 4; ++i)
        if (ranges_overlap(outs[o], oute[o], ins[i], ine[i])) return CASC_ERR_INVALID;
  }
  if (n == 0) return CASC_OK;
  int sms = 0;
  if ((r = device_check(&sms))) return r;
  const cudaStream_t st = S(stream);
  const bool use_beta = !(beta_hi == 0.0 && beta_lo == 0.0);
  if (no_product) {
    cudaError_t e = casc::launch_scale_c_uplo(n, n, beta_hi, beta_lo, use_beta, C_hi, C_lo, ldc,
                                              flags, sms, uplo == CASC_LOWER ? 0 : 1, st);
    if (e == cudaSuccess) g_launches = 1;
    return cuda_status(e);
  }
  const size_t need = casc_workspace_bytes(n, n, k);
  const size_t fbytes = flags ? (size_t)(n * n + 255) / 256 * 256 : 0;
  void* ws = nullptr;
  if (cudaMallocAsync(&ws, need + fbytes, st) != cudaSuccess) return CASC_ERR_CUDA;
  uint8_t* pa = static_cast<uint8_t*>(ws);
  uint8_t* pb = pa + (casc_packed_a_bytes(n, k) + 255) / 256 * 256;
  uint8_t* f2 = flags ? static_cast<uint8_t*>(ws) + need : nullptr;
  const casc::Widths w = widths_for(k);
  const int nst = (int)(casc::kpad_of(k) / casc::BK);
  const int tri = uplo == CASC_LOWER ? 1 : 2;
  int launches = 0;
  // 1) C := alpha op(A) op(B)^T (+) beta C on the triangle
  cudaError_t e = casc::launch_split_ab(A_hi, A_lo, lda, n, B_hi, B_lo, ldb, n, k, w, pa, pb, st,
                                        trans == CASC_OP_T, trans == CASC_OP_N);
  AlphaBeta abv;
  abv.ab = use_beta ? 2 : ((alpha_hi == 1.0 && alpha_lo == 0.0) ? 0 : 1);
  abv.ah = alpha_hi;
  abv.al = alpha_lo;
  abv.bh = beta_hi;
  abv.bl = beta_lo;
  g_launches = 0;
  r = (e == cudaSuccess) ? gemm_packed_impl(n, n, k, pa, pb, C_hi, C_lo, ldc, flags, sms, st, 0,
                                            nst, nullptr, abv, nullptr, tri,
                                            ws_counter(ws, n, n, k))
                         : CASC_ERR_CUDA;
  launches += 1 + g_launches;
  // 2) C := alpha op(B) op(A)^T (+) C, flags of this product into f2
  if (r == CASC_OK) {
    e = casc::launch_split_ab(B_hi, B_lo, ldb, n, A_hi, A_lo, lda, n, k, w, pa, pb, st,
                              trans == CASC_OP_T, trans == CASC_OP_N);
    AlphaBeta ab2 = abv;
    ab2.ab = 2;
    ab2.bh = 1.0;
    ab2.bl = 0.0;
    g_launches = 0;
    r = (e == cudaSuccess) ? gemm_packed_impl(n, n, k, pa, pb, C_hi, C_lo, ldc, f2, sms, st, 0,
                                              nst, nullptr, ab2, nullptr, tri,
                                              ws_counter(ws, n, n, k))
                           : CASC_ERR_CUDA;
    launches += 1 + g_launches;
  }
  if (r == CASC_OK && flags) {
    r = cuda_status(casc::launch_or_flags(n, uplo == CASC_LOWER ? 0 : 1, flags, f2, sms, st));
    ++launches;
  }
  cudaFreeAsync(ws, st);
  g_launches = r == CASC_OK ? launches : 0;
  return r;
}

// ---------------------------------------------------------------- TRSM (NEXT-4)
// Left side: op(A) X = alpha B, op(A) = A or A^T, X overwrites B (reading R27).
static constexpr int64_t kTrsmNb = 256;
static constexpr int64_t kTrsmSb = 4;  // diagonal blocks per super-block of the trailing updates

int casc_trsm_diag_inv(int uplo, int diag, int64_t m, const double* A_hi, const double* A_lo,
                       int64_t lda, double* inv_hi, double* inv_lo, casc_stream_t stream) {
  g_launches = 0;
  if ((uplo != CASC_LOWER && uplo != CASC_UPPER) || (diag != CASC_NONUNIT && diag != CASC_UNIT))
    return CASC_ERR_INVALID;
  int r;
  if ((r = check_mat(A_hi, m, m, lda)) || (r = check_mat(A_lo, m, m, lda))) return r;
  if (m > 0 && (!inv_hi || !inv_lo)) return CASC_ERR_INVALID;
  if ((r = device_check(nullptr))) return r;
  if (m == 0) return CASC_OK;
  const cudaError_t e =
      casc::launch_trsm_diag_inv(uplo, diag, m, A_hi, A_lo, lda, inv_hi, inv_lo, S(stream));
  if (e == cudaSuccess) g_launches = 1;
  return cuda_status(e);
}

int casc_trsm_fp64x2(int uplo, int trans, int diag, int64_t m, int64_t n, double alpha_hi,
                     double alpha_lo, const double* A_hi, const double* A_lo, int64_t lda,
                     double* B_hi, double* B_lo, int64_t ldb, casc_stream_t stream) {
  g_launches = 0;
  if ((uplo != CASC_LOWER && uplo != CASC_UPPER) || (diag != CASC_NONUNIT && diag != CASC_UNIT) ||
      (trans != CASC_OP_N && trans != CASC_OP_T))
    return CASC_ERR_INVALID;
  if (m < 0 || n < 0) return CASC_ERR_INVALID;
  int r;
  if ((r = check_mat(A_hi, m, m, lda)) || (r = check_mat(A_lo, m, m, lda))) return r;
  if ((r = check_mat(B_hi, m, n, ldb)) || (r = check_mat(B_lo, m, n, ldb))) return r;
  if (trsm_overlap(m, n, A_hi, A_lo, lda, B_hi, B_lo, ldb)) return CASC_ERR_INVALID;
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = device_check(&sms))) return r;
  const cudaStream_t st = S(stream);
  int launches = 0;
  const bool unit_alpha = (alpha_hi == 1.0 && alpha_lo == 0.0);
  const bool zero_alpha = (alpha_hi == 0.0 && alpha_lo == 0.0);
  if (!unit_alpha) {  // B := alpha (x) B
    const cudaError_t e = casc::launch_scale_c(m, n, alpha_hi, alpha_lo, zero_alpha ? 0 : 1, B_hi,
                                               B_lo, ldb, nullptr, sms, st);
    if (e != cudaSuccess) return CASC_ERR_CUDA;
    ++launches;
  }
  if (zero_alpha) {
    g_launches = launches;
    return CASC_OK;
  }
  const int64_t nblk = (m + kTrsmNb - 1) / kTrsmNb;
  const size_t inv_elems = (size_t)nblk * kTrsmNb * kTrsmNb, t_elems = (size_t)kTrsmNb * n;
  double* buf = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&buf), (2 * inv_elems + 2 * t_elems) * 8, st) !=
      cudaSuccess)
    return CASC_ERR_CUDA;
  double* inv_hi = buf;
  double* inv_lo = buf + inv_elems;
  double* t_hi = inv_lo + inv_elems;
  double* t_lo = t_hi + t_elems;
  cudaError_t e = casc::launch_trsm_diag_inv(uplo, diag, m, A_hi, A_lo, lda, inv_hi, inv_lo, st);
  r = e == cudaSuccess ? CASC_OK : CASC_ERR_CUDA;
  ++launches;
  // op(A) is lower when (uplo lower) xor (transposed); op(A_bb)^-1 = op(Inv_b)
  const bool eff_lower = (uplo == CASC_LOWER) != (trans == CASC_OP_T);
  for (int64_t s = 0; s < nblk && r == CASC_OK; ++s) {
    const int64_t b = eff_lower ? s : nblk - 1 - s;
    const int64_t r0 = b * kTrsmNb, nb = std::min(kTrsmNb, m - r0), r1 = r0 + nb;
    // X_b = op(Inv_b) B_b, into T and back into B_b
    r = casc_gemm_fp64x2_ex(trans, CASC_OP_N, nb, n, nb, 1.0, 0.0,
                            inv_hi + b * kTrsmNb * kTrsmNb, inv_lo + b * kTrsmNb * kTrsmNb,
                            kTrsmNb, B_hi + r0 * ldb, B_lo + r0 * ldb, ldb, 0.0, 0.0, t_hi, t_lo,
                            n, nullptr, nullptr, 0, stream);
    launches += g_launches;
    if (r) break;
    if (cudaMemcpy2DAsync(B_hi + r0 * ldb, ldb * 8, t_hi, n * 8, n * 8, nb,
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
        cudaMemcpy2DAsync(B_lo + r0 * ldb, ldb * 8, t_lo, n * 8, n * 8, nb,
                          cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
      r = CASC_ERR_CUDA;
      break;
    }
    // updates: the super-block's remaining rows with X_b, then, after its last
    // block, the trailing rows with the whole super-block's X (reading R27)
    auto update = [&](int64_t R0, int64_t R1, int64_t C0, int64_t C1) {
      if (r != CASC_OK || R1 <= R0 || C1 <= C0) return;
      const int64_t off = trans ? C0 * lda + R0 : R0 * lda + C0;
      r = casc_gemm_fp64x2_ex(trans, CASC_OP_N, R1 - R0, n, C1 - C0, -1.0, 0.0, A_hi + off,
                              A_lo + off, lda, B_hi + C0 * ldb, B_lo + C0 * ldb, ldb, 1.0, 0.0,
                              B_hi + R0 * ldb, B_lo + R0 * ldb, ldb, nullptr, nullptr, 0, stream);
      launches += g_launches;
    };
    const int64_t S0 = (b / kTrsmSb) * kTrsmSb * kTrsmNb;
    const int64_t S1 = std::min(S0 + kTrsmSb * kTrsmNb, m);
    g_launches = 0;
    if (eff_lower) {
      update(r1, S1, r0, r1);
      if (r1 == S1) update(S1, m, S0, S1);
    } else {
      update(S0, r0, r0, r1);
      if (r0 == S0) update(0, S0, S0, S1);
    }
    g_launches = 0;
    launches += g_launches;
  }
  cudaFreeAsync(buf, st);
  g_launches = r == CASC_OK ? launches : 0;
  return r;
}

// ---------------------------------------------------------------- simple path
// Ten products of eqn:Gemm10 in the order of the fused kernel: {bin, A slice, B slice}.
static const int kProducts[10][3] = {{0, 0, 0}, {1, 0, 1}, {1, 1, 0}, {2, 0, 2}, {2, 1, 1},
                                     {2, 2, 0}, {3, 0, 3}, {3, 1, 4}, {3, 2, 5}, {3, 3, 6}};

static int slice_args(int64_t m, int64_t n, int64_t k, const void* pa, const void* pb, int sa,
                      int sb, int64_t panel, double* out, int64_t ldo, int accumulate,
                      double scale, casc::SliceArgs& a) {
  const int nst = (int)(casc::kpad_of(k) / casc::BK);
  a.pa = static_cast<const uint8_t*>(pa);
  a.pb = static_cast<const uint8_t*>(pb);
  a.a_blk = casc::a_block_bytes(k);
  a.b_blk = casc::b_block_bytes(k);
  a.m = m;
  a.n = n;
  a.mblocks = (int)((m + casc::TM - 1) / casc::TM);
  a.nblocks = (int)((n + casc::TN - 1) / casc::TN);
  a.st_begin = (int)panel * casc::STAGES_PER_PANEL;
  a.st_end = a.st_begin + casc::STAGES_PER_PANEL < nst ? a.st_begin + casc::STAGES_PER_PANEL : nst;
  a.sa = sa;
  a.sb = sb;
  a.out = out;
  a.ldo = ldo;
  a.accumulate = accumulate;
  a.scale = scale;
  return CASC_OK;
}

int casc_gemm_fp64x2_simple(int64_t m, int64_t n, int64_t k, const double* A_hi,
                            const double* A_lo, int64_t lda, const double* B_hi,
                            const double* B_lo, int64_t ldb, double* C_hi, double* C_lo,
                            int64_t ldc, uint8_t* flags, casc_stream_t stream) {
  g_launches = 0;
  int r = validate_gemm(m, n, k, A_hi, A_lo, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, flags);
  if (r) return r;
  if (m == 0 || n == 0) return CASC_OK;
  int sms = 0;
  if ((r = device_check(&sms))) return r;
  cudaStream_t st = S(stream);
  if (k == 0) return zero_c(m, n, C_hi, C_lo, ldc, flags, st);
  void *pa = nullptr, *pb = nullptr, *bins = nullptr;
  const size_t bin_bytes = (size_t)4 * m * n * sizeof(double);
  if (cudaMallocAsync(&pa, casc_packed_a_bytes(m, k), st) != cudaSuccess) return CASC_ERR_CUDA;
  if (cudaMallocAsync(&pb, casc_packed_b_bytes(k, n), st) != cudaSuccess ||
      cudaMallocAsync(&bins, bin_bytes, st) != cudaSuccess) {
    cudaFreeAsync(pa, st);
    if (pb) cudaFreeAsync(pb, st);
    return CASC_ERR_CUDA;
  }
  const casc::Widths w = widths_for(k);
  cudaError_t e = casc::launch_split_a(A_hi, A_lo, lda, m, k, w, pa, st);
  if (e == cudaSuccess) e = casc::launch_split_b(B_hi, B_lo, ldb, k, n, w, pb, st);
  int launches = 2;
  const int64_t P = casc::panels_of(k);
  double* B = static_cast<double*>(bins);
  for (int64_t q = 0; q < P && e == cudaSuccess; ++q) {
    for (int t = 0; t < 10 && e == cudaSuccess; ++t) {
      const int bin = kProducts[t][0];
      const bool first_of_bin = (t == 0 || kProducts[t - 1][0] != bin);
      casc::SliceArgs a{};
      slice_args(m, n, k, pa, pb, kProducts[t][1], kProducts[t][2], q, B + bin * m * n, n,
                 first_of_bin ? 0 : 1, 1.0, a);
      e = casc::launch_slice_gemm(a, sms, st);
      ++launches;
    }
    if (e == cudaSuccess)
      e = casc::launch_epilogue(B, pa, pb, k, (int)q, m, n, C_hi, C_lo, ldc, flags, q == 0, w,
                                sms, st);
    ++launches;
  }
  cudaFreeAsync(bins, st);
  cudaFreeAsync(pa, st);
  cudaFreeAsync(pb, st);
  if (e != cudaSuccess) return CASC_ERR_CUDA;
  g_launches = launches;
  return CASC_OK;
}

int casc_slice_product(int64_t m, int64_t n, int64_t k, const double* A_hi, const double* A_lo,
                       int64_t lda, const double* B_hi, const double* B_lo, int64_t ldb, int sa,
                       int sb, int64_t panel, double* out, casc_stream_t stream) {
  g_launches = 0;
  int r;
  if (m < 0 || n < 0 || k < 0) return CASC_ERR_INVALID;
  if ((r = check_mat(A_hi, m, k, lda)) || (r = check_mat(A_lo, m, k, lda))) return r;
  if ((r = check_mat(B_hi, k, n, ldb)) || (r = check_mat(B_lo, k, n, ldb))) return r;
  if (sa < 0 || sa > 3 || sb < 0 || sb > 6) return CASC_ERR_INVALID;
  if (panel < 0 || panel >= casc::panels_of(k)) return CASC_ERR_INVALID;
  if (m == 0 || n == 0) return CASC_OK;
  if (!out) return CASC_ERR_INVALID;
  int sms = 0;
  if ((r = device_check(&sms))) return r;
  cudaStream_t st = S(stream);
  void *pa = nullptr, *pb = nullptr;
  if (cudaMallocAsync(&pa, casc_packed_a_bytes(m, k), st) != cudaSuccess) return CASC_ERR_CUDA;
  if (cudaMallocAsync(&pb, casc_packed_b_bytes(k, n), st) != cudaSuccess) {
    cudaFreeAsync(pa, st);
    return CASC_ERR_CUDA;
  }
  const casc::Widths w = widths_for(k);
  // undo the exact pre-alignment: paper normalisation of A2, B2, B4, B5
  int sh = 0;
  if (sa == 2) sh += w.c1 - w.c0;
  if (sb == 2) sh += w.c1 - w.c0;
  if (sb == 4) sh += w.c0 - w.c2;
  if (sb == 5) sh += 2 * w.c0 - w.c1 - w.c2;
  cudaError_t e = casc::launch_split_a(A_hi, A_lo, lda, m, k, w, pa, st);
  if (e == cudaSuccess) e = casc::launch_split_b(B_hi, B_lo, ldb, k, n, w, pb, st);
  if (e == cudaSuccess) {
    casc::SliceArgs a{};
    slice_args(m, n, k, pa, pb, sa, sb, panel, out, n, 0, std::ldexp(1.0, sh), a);
    e = casc::launch_slice_gemm(a, sms, st);
  }
  cudaFreeAsync(pa, st);
  cudaFreeAsync(pb, st);
  if (e != cudaSuccess) return CASC_ERR_CUDA;
  g_launches = 3;
  return CASC_OK;
}

}  // extern "C"

// Host helpers shared with the other entry-point files (casc_i8.cu).
namespace casc {
namespace host {
int device_check(int* sms) { return ::device_check(sms); }
int validate_gemm(int64_t m, int64_t n, int64_t k, const double* A_hi, const double* A_lo,
                  int64_t lda, const double* B_hi, const double* B_lo, int64_t ldb, double* C_hi,
                  double* C_lo, int64_t ldc, uint8_t* flags) {
  return ::validate_gemm(m, n, k, A_hi, A_lo, lda, B_hi, B_lo, ldb, C_hi, C_lo, ldc, flags);
}
int zero_c(int64_t m, int64_t n, double* C_hi, double* C_lo, int64_t ldc, uint8_t* flags,
           cudaStream_t st) {
  return ::zero_c(m, n, C_hi, C_lo, ldc, flags, st);
}
int check_mat(const void* p, int64_t rows, int64_t cols, int64_t ld) {
  return ::check_mat(p, rows, cols, ld);
}
int current_sms() { return ::current_sms(); }
bool trsm_overlap(int64_t m, int64_t n, const double* A_hi, const double* A_lo, int64_t lda,
                  const double* B_hi, const double* B_lo, int64_t ldb) {
  return ::trsm_overlap(m, n, A_hi, A_lo, lda, B_hi, B_lo, ldb);
}
// casc_gemm_fp64x2_ex with a banded (triangular) operand, GemmArgs::band (TRMM)
int gemm_ex_band(int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha_hi,
                 double alpha_lo, const double* A_hi, const double* A_lo, int64_t lda,
                 const double* B_hi, const double* B_lo, int64_t ldb, double* C_hi, double* C_lo,
                 int64_t ldc, casc_stream_t stream, int band) {
  return ::gemm_ex_impl(transa, transb, m, n, k, alpha_hi, alpha_lo, A_hi, A_lo, lda, B_hi, B_lo,
                        ldb, 0.0, 0.0, C_hi, C_lo, ldc, nullptr, nullptr, 0, stream, band);
}
void set_launches(int n) { g_launches = n; }
}  // namespace host
}  // namespace casc
