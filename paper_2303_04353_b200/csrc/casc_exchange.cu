// casc_exchange.cu — the multi-GPU exchange of B's packed slabs over peer
// memory (north star: "B slices broadcast over NVLink").
//
// Each rank exports the device buffer that holds its own packed column slab
// of B (cudaIpcGetMemHandle); every other rank maps it (cudaIpcOpenMemHandle,
// lazy peer access) and PULLS the slab with the copy engines
// (cudaMemcpyAsync, one copy per slab on internal copy streams of the caller),
// so the exchange uses no SM while the fused GEMM runs and each slab's GEMM
// can start as soon as that slab has landed (paper_2303_04353_b200/multigpu.py,
// gather = "p2p").  Ordering between ranks is host-side (the multigpu layer's
// CPU barriers); no kernel waits on another rank.  Host code only.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../include/casc.h"

namespace {
inline cudaStream_t S(casc_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }
inline int st(cudaError_t e) {
  if (e == cudaSuccess) return CASC_OK;
  cudaGetLastError();
  return CASC_ERR_CUDA;
}
}  // namespace

extern "C" {

int casc_ipc_alloc(size_t bytes, void** ptr, void* handle) {
  if (!ptr || !handle || bytes == 0) return CASC_ERR_INVALID;
  *ptr = nullptr;
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return st(cudaErrorMemoryAllocation);
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
    cudaFree(p);
    return st(cudaErrorInvalidValue);
  }
  static_assert(sizeof(h) == CASC_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle, &h, sizeof(h));
  *ptr = p;
  return CASC_OK;
}

int casc_ipc_free(void* ptr) {
  if (!ptr) return CASC_OK;
  return st(cudaFree(ptr));
}

int casc_ipc_open(const void* handle, void** ptr) {
  if (!handle || !ptr) return CASC_ERR_INVALID;
  *ptr = nullptr;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return st(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
}

int casc_ipc_close(void* ptr) {
  if (!ptr) return CASC_OK;
  return st(cudaIpcCloseMemHandle(ptr));
}

int casc_copy_async(void* dst, const void* src, size_t bytes, casc_stream_t stream) {
  if (bytes == 0) return CASC_OK;
  if (!dst || !src) return CASC_ERR_INVALID;
  return st(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, S(stream)));
}

}  // extern "C"
