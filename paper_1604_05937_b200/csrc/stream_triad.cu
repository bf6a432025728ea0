// STREAM triad a = b + alpha * c on the device: the machine bandwidth
// reference of the perfbench module (SPEC.md "stream_triad", the paper's
// Table "Maximum STREAM triad"), B200 version: 16-byte loads / stores,
// a grid of a whole number of waves over the SMs.
#include "pm_common.cuh"

namespace {

__global__ void __launch_bounds__(256)
k_triad(double *__restrict__ a, const double *__restrict__ b,
        const double *__restrict__ c, double alpha, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n2 = n / 2;
  const double2 *b2 = reinterpret_cast<const double2 *>(b);
  const double2 *c2 = reinterpret_cast<const double2 *>(c);
  double2 *a2 = reinterpret_cast<double2 *>(a);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += stride) {
    const double2 u = __ldcs(b2 + i), v = __ldcs(c2 + i);
    __stcs(a2 + i, make_double2(u.x + alpha * v.x, u.y + alpha * v.y));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1))
    a[n - 1] = b[n - 1] + alpha * c[n - 1];
}

} // namespace

extern "C" int pm_stream_triad(double *a, const double *b, const double *c,
                               double alpha, int64_t n, void *stream) {
  pm::clear_error();
  if (n < 0) {
    pm::set_error("negative triad length");
    return PM_EINVAL;
  }
  if (((uintptr_t)a | (uintptr_t)b | (uintptr_t)c) & 15) {
    pm::set_error("triad arrays must be 16-byte aligned");
    return PM_EINVAL;
  }
  if (!n) return PM_OK;
  k_triad<<<pm::grid_for((n + 1) / 2, 256, 8), 256, 0,
            (cudaStream_t)stream>>>(a, b, c, alpha, n);
  PM_LAUNCH_CHECK("k_triad");
  return PM_OK;
}
