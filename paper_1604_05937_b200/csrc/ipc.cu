// CUDA IPC for the fused halo: a rank exports its y window, the rank that
// computes the window's ghost columns maps it and adds into it with REDG
// over NVLink (strip kernel, y_peer).  Torch's caching allocator hands out
// pointers inside larger allocations, so the handle is taken on the
// allocation base and the window's byte offset travels with it.
#include <cuda.h>
#include <string.h>

#include "pm_common.cuh"

namespace {

typedef CUresult (*GetRangeFn)(CUdeviceptr *, size_t *, CUdeviceptr);

int allocation_base(const void *ptr, void **base) {
  static GetRangeFn fn = nullptr;
  if (!fn) {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    PM_CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f,
                                        cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f) {
      pm::set_error("cuMemGetAddressRange not available");
      return PM_ECUDA;
    }
    fn = reinterpret_cast<GetRangeFn>(f);
  }
  CUdeviceptr b = 0;
  size_t size = 0;
  if (fn(&b, &size, (CUdeviceptr)(uintptr_t)ptr) != CUDA_SUCCESS) {
    pm::set_error("pointer %p is not device memory", ptr);
    return PM_EINVAL;
  }
  *base = (void *)(uintptr_t)b;
  return PM_OK;
}

} // namespace

extern "C" int pm_ipc_export(const void *ptr, void *handle, int64_t *offset) {
  pm::clear_error();
  if (!ptr || !handle || !offset) {
    pm::set_error("pm_ipc_export: NULL argument");
    return PM_EINVAL;
  }
  void *base = nullptr;
  int rc = allocation_base(ptr, &base);
  if (rc) return rc;
  cudaIpcMemHandle_t h;
  PM_CUDA_TRY(cudaIpcGetMemHandle(&h, base));
  memcpy(handle, &h, sizeof h);
  *offset = (int64_t)((const char *)ptr - (const char *)base);
  return PM_OK;
}

extern "C" int pm_ipc_open(const void *handle, int64_t offset, void **ptr) {
  pm::clear_error();
  if (!handle || !ptr || offset < 0) {
    pm::set_error("pm_ipc_open: bad argument");
    return PM_EINVAL;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  void *base = nullptr;
  PM_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr = (char *)base + offset;
  return PM_OK;
}

extern "C" int pm_ipc_close(void *ptr, int64_t offset) {
  pm::clear_error();
  PM_CUDA_TRY(cudaIpcCloseMemHandle((char *)ptr - offset));
  return PM_OK;
}
