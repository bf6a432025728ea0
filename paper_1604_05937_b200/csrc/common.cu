// Error plumbing, device info and the host slot table.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "pm_common.cuh"

namespace pm {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

void clear_error() { g_err[0] = 0; }

int cuda_status(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return PM_OK;
  set_error("CUDA error in %s: %s (%s)", what, cudaGetErrorName(e),
            cudaGetErrorString(e));
  return PM_ECUDA;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) !=
            cudaSuccess ||
        n <= 0)
      n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

int make_slot_table(const int32_t *delta6, SlotTable *t) {
  if (!delta6) {
    set_error("delta6 is NULL");
    return PM_EINVAL;
  }
  int any = 0;
  for (int i = 0; i < 6; ++i) {
    if (delta6[i] < 0) {
      set_error("negative DoF count delta[%d]=%d", i, delta6[i]);
      return PM_EINVAL;
    }
    any |= delta6[i] != 0;
  }
  if (!any) {
    set_error("layout assigns no DoFs at all");
    return PM_EINVAL;
  }
  static const int n_local[3] = {3, 3, 1};
  int k = 0;
  for (int d = 0; d < 3; ++d) {
    const int lo = delta6[2 * d], conn = delta6[2 * d + 1];
    if (!lo && !conn) continue;
    for (int loc = 0; loc < n_local[d]; ++loc) {
      const int counts[3] = {lo, conn, lo};
      const int base[3] = {0, lo, lo + conn};
      for (int lev = 0; lev < 3; ++lev)
        for (int j = 0; j < counts[lev]; ++j) {
          if (k >= kMaxSlots) {
            set_error("layout has more than %d stencil slots", kMaxSlots);
            return PM_EINVAL;
          }
          t->kind[k] = (int8_t)d;
          t->local[k] = (int8_t)loc;
          t->level[k] = (int8_t)lev;
          t->within[k] = base[lev] + j;
          t->offset[k] = lo + conn;
          ++k;
        }
    }
  }
  t->k = k;
  return PM_OK;
}

} // namespace pm

extern "C" const char *pm_last_error(void) { return pm::g_err; }

extern "C" int pm_version(void) { return 1; }

extern "C" int pm_num_slots(const int32_t *delta6, int32_t *k_out) {
  pm::SlotTable t;
  int rc = pm::make_slot_table(delta6, &t);
  if (rc) return rc;
  if (k_out) *k_out = t.k;
  return PM_OK;
}

namespace pm {
static thread_local int g_overlap = 0;
bool launch_overlap() { return g_overlap != 0; }
} // namespace pm

extern "C" int pm_set_launch_overlap(int32_t on) {
  const int prev = pm::g_overlap;
  pm::g_overlap = on ? 1 : 0;
  return prev;
}

#ifndef PM_EXPERIMENTAL
#define PM_EXPERIMENTAL 0
#endif
// bit 0: built with the experimental schedules (PM_EXPERIMENTAL=1)
extern "C" int pm_build_flags(void) { return PM_EXPERIMENTAL ? 1 : 0; }

extern "C" int pm_device_info(int32_t *sm, int64_t *l2) {
  int dev = 0, n = 0, l2b = 0;
  PM_CUDA_TRY(cudaGetDevice(&dev));
  PM_CUDA_TRY(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  PM_CUDA_TRY(cudaDeviceGetAttribute(&l2b, cudaDevAttrL2CacheSize, dev));
  if (sm) *sm = n;
  if (l2) *l2 = l2b;
  return PM_OK;
}
