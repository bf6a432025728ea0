// Shared helpers for libprismesh_cuda.so: error reporting and launch sizing.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "prismesh_cuda.h"

namespace pm {

// Thread-local last-error message (read through pm_last_error()).
void set_error(const char *fmt, ...);
void clear_error();

// Map a CUDA status to PM_OK / PM_ECUDA, recording `what`.
int cuda_status(cudaError_t e, const char *what);

// Number of SMs of the current device (cached per device).
int sm_count();

// Grid size for a grid-stride loop over `n` items with `threads` per block:
// enough blocks to cover n, capped at `per_sm` resident blocks per SM.
inline unsigned grid_for(int64_t n, int threads, int per_sm = 16) {
  int64_t want = (n + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count() * per_sm;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (unsigned)want;
}

// Programmatic dependent launch of the DG stream kernel (thread-local,
// pm_set_launch_overlap): only for back-to-back applies whose inputs no
// preceding kernel writes.
bool launch_overlap();

constexpr int kMaxSlots = 64;

// Host-side restatement of the reference slot table (fspace.py:110-131):
// vertices 0-2, edges 0-2, cell; bottom copy, connecting entity, top copy.
struct SlotTable {
  int k;
  int8_t kind[kMaxSlots];    // 0 vertex, 1 edge, 2 cell
  int8_t local[kMaxSlots];   // index inside the family
  int8_t level[kMaxSlots];   // 0 bottom copy, 1 connecting, 2 top copy
  int32_t within[kMaxSlots]; // offset inside the column's layer block
  int32_t offset[kMaxSlots]; // vertical offset delta(d,0)+delta(d,1)
};

// Returns PM_OK or PM_EINVAL (negative counts, no DoFs, > kMaxSlots).
int make_slot_table(const int32_t *delta6, SlotTable *t);

} // namespace pm

#define PM_CUDA_TRY(expr)                                                    \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) return pm::cuda_status(_e, #expr);                \
  } while (0)

#define PM_LAUNCH_CHECK(what)                                                \
  do {                                                                       \
    cudaError_t _e = cudaGetLastError();                                     \
    if (_e != cudaSuccess) return pm::cuda_status(_e, what);                 \
  } while (0)
