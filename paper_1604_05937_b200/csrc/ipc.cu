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
  // the fused halo adds into the mapping with fp64 atomics: the link must
  // carry them natively (NVLink does; a PCIe path may not) -- otherwise
  // refuse, and the caller falls back to the NCCL exchange
  cudaPointerAttributes pa;
  int here = 0;
  if (cudaPointerGetAttributes(&pa, base) == cudaSuccess &&
      cudaGetDevice(&here) == cudaSuccess && pa.device >= 0 &&
      pa.device != here) {
    int atomics = 0;
    if (cudaDeviceGetP2PAttribute(&atomics,
                                  cudaDevP2PAttrNativeAtomicSupported, here,
                                  pa.device) != cudaSuccess ||
        !atomics) {
      cudaIpcCloseMemHandle(base);
      pm::set_error("pm_ipc_open: no native peer atomics between devices %d "
                    "and %d",
                    here, pa.device);
      return PM_ECUDA;
    }
  }
  cudaGetLastError();
  *ptr = (char *)base + offset;
  return PM_OK;
}

// --- stream-ordered signalling between ranks (no host synchronisation) ---
// A rank raises a 32-bit flag -- its own or, through a mapping, a peer's
// -- with a one-thread kernel queued behind its preceding work (system-scope
// release: the preceding kernels' peer REDs are visible first), and makes
// its stream wait until a local flag reaches a value (cuStreamWaitValue32:
// the wait is done by the stream front end, no kernel spins).

namespace {

__global__ void k_signal(uint32_t *flag, uint32_t value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value)
               : "memory");
}

typedef CUresult (*WaitValueFn)(CUstream, CUdeviceptr, cuuint32_t,
                                unsigned int);

} // namespace

extern "C" int pm_stream_signal(uint32_t *flag, uint32_t value, void *stream) {
  pm::clear_error();
  if (!flag) {
    pm::set_error("pm_stream_signal: NULL flag");
    return PM_EINVAL;
  }
  k_signal<<<1, 1, 0, (cudaStream_t)stream>>>(flag, value);
  PM_LAUNCH_CHECK("k_signal");
  return PM_OK;
}

extern "C" int pm_stream_wait_geq(const uint32_t *flag, uint32_t value,
                                  void *stream) {
  pm::clear_error();
  static WaitValueFn fn = nullptr;
  if (!fn) {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    PM_CUDA_TRY(cudaGetDriverEntryPoint("cuStreamWaitValue32", &f,
                                        cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f) {
      pm::set_error("cuStreamWaitValue32 not available");
      return PM_ECUDA;
    }
    fn = reinterpret_cast<WaitValueFn>(f);
  }
  if (!flag) {
    pm::set_error("pm_stream_wait_geq: NULL flag");
    return PM_EINVAL;
  }
  const CUresult r = fn((CUstream)stream, (CUdeviceptr)(uintptr_t)flag,
                        (cuuint32_t)value, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) {
    pm::set_error("cuStreamWaitValue32 failed (%d)", (int)r);
    return PM_ECUDA;
  }
  return PM_OK;
}

extern "C" int pm_ipc_close(void *ptr, int64_t offset) {
  pm::clear_error();
  PM_CUDA_TRY(cudaIpcCloseMemHandle((char *)ptr - offset));
  return PM_OK;
}
