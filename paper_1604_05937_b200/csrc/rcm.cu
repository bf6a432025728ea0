// Device Cuthill-McKee breadth-first walk, bit-exact
// with the reference's serial walk (pkg/src/prismesh/ordering.py:45-90,
// `_cuthill_mckee`): components in order of their smallest unvisited
// vertex, each started at its minimum-(degree, index) vertex, neighbours
// appended in the (degree, index) order of the pre-sorted CSR rows.
//
// The serial queue order is reproduced level by level without a sort:
// a vertex w of level k+1 is appended by the FIRST vertex of level k (in
// queue position) that has w as a neighbour, at that vertex's row rank.
// So per level:
//   1. every frontier position p atomicMin's its position into parent[w]
//      of each unvisited neighbour w;
//   2. p counts the neighbours whose parent is p (its children);
//   3. an exclusive scan of the counts over the frontier places p's
//      children right after those of p-1;
//   4. p writes its children in row order;
//   5. the new level is marked visited.
// Graphs of meshes have frontiers of O(sqrt(n)) vertices and O(sqrt(n))
// levels, so the walk runs in ONE thread block (no grid-wide barrier; the
// block's __syncthreads order the global-memory steps).  The component
// search before each walk (the reference's pass 1) is an unordered
// breadth-first flood with atomicCAS marks in the same block.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "pm_common.cuh"

namespace {

constexpr int kT = 1024;
constexpr int32_t kUnseen = 0, kWalked = 1, kFlooded = 2;

__global__ void k_fill_i32(int32_t *__restrict__ a, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

__global__ void __launch_bounds__(kT, 1)
k_cuthill_mckee(const int64_t *__restrict__ off, const int32_t *__restrict__ nb,
                int32_t n, int64_t *__restrict__ order,
                int32_t *__restrict__ mark, int32_t *__restrict__ parent,
                int32_t *__restrict__ cnt, int32_t *__restrict__ status) {
  using Scan = cub::BlockScan<int32_t, kT>;
  using Reduce = cub::BlockReduce<unsigned long long, kT>;
  __shared__ union {
    typename Scan::TempStorage scan;
    typename Reduce::TempStorage reduce;
  } tmp;
  __shared__ int32_t s_tail, s_int;
  __shared__ unsigned long long s_key;
  const int tid = threadIdx.x;
  int32_t pos = 0, scan = 0;
  while (pos < n) {
    // the smallest unvisited vertex (scan only moves forward)
    for (;; scan += kT) {
      if (tid == 0) s_int = INT32_MAX;
      __syncthreads();
      const int32_t v = scan + tid;
      if (v < n && mark[v] == kUnseen) atomicMin(&s_int, v);
      __syncthreads();
      const int32_t found = s_int;
      __syncthreads(); // everyone read s_int before it is reset
      if (found != INT32_MAX) {
        scan = found;
        break;
      }
    }
    // pass 1: flood the component of `scan` (queue in order[pos..]) and
    // take its minimum (degree, index) vertex
    if (tid == 0) {
      order[pos] = scan;
      mark[scan] = kFlooded;
      s_tail = pos + 1;
    }
    __syncthreads();
    int32_t h0 = pos, h1 = s_tail;
    while (h0 < h1) {
      for (int32_t p = h0 + tid; p < h1; p += kT) {
        const int32_t v = (int32_t)order[p];
        for (int64_t e = off[v]; e < off[v + 1]; ++e) {
          const int32_t w = nb[e];
          if (w < 0 || w >= n) {
            atomicOr(status, 1);
            continue;
          }
          if (atomicCAS(&mark[w], kUnseen, kFlooded) == kUnseen)
            order[atomicAdd(&s_tail, 1)] = w;
        }
      }
      __syncthreads();
      h0 = h1;
      h1 = s_tail;
      __syncthreads();
    }
    if (*status) return; // (uniform: read after the barrier)
    unsigned long long best = ~0ull;
    for (int32_t p = pos + tid; p < h1; p += kT) {
      const int32_t v = (int32_t)order[p];
      const unsigned long long key =
          ((unsigned long long)(off[v + 1] - off[v]) << 32) | (uint32_t)v;
      best = key < best ? key : best;
    }
    best = Reduce(tmp.reduce).Reduce(best, cub::Min());
    if (tid == 0) s_key = best;
    __syncthreads();
    const int32_t start = (int32_t)(s_key & 0xffffffffu);
    for (int32_t p = pos + tid; p < h1; p += kT) mark[order[p]] = kUnseen;
    __syncthreads();
    // pass 2: the ordered walk from `start`
    if (tid == 0) {
      order[pos] = start;
      mark[start] = kWalked;
    }
    __syncthreads();
    h0 = pos;
    h1 = pos + 1;
    while (h0 < h1) {
      // 1. first discoverer (lowest queue position) of every new vertex
      for (int32_t p = h0 + tid; p < h1; p += kT) {
        const int32_t v = (int32_t)order[p];
        for (int64_t e = off[v]; e < off[v + 1]; ++e) {
          const int32_t w = nb[e];
          if (mark[w] == kUnseen) atomicMin(&parent[w], p);
        }
      }
      __syncthreads();
      // 2. children per frontier position
      for (int32_t p = h0 + tid; p < h1; p += kT) {
        const int32_t v = (int32_t)order[p];
        int32_t c = 0;
        for (int64_t e = off[v]; e < off[v + 1]; ++e) {
          const int32_t w = nb[e];
          c += (mark[w] == kUnseen && parent[w] == p) ? 1 : 0;
        }
        cnt[p - h0] = c;
      }
      __syncthreads();
      // 3. exclusive scan over the frontier, kT positions at a time
      int32_t carry = 0;
      for (int32_t b = 0; b < h1 - h0; b += kT) {
        const int32_t i = b + tid;
        const int32_t c = i < h1 - h0 ? cnt[i] : 0;
        int32_t ex, total;
        Scan(tmp.scan).ExclusiveSum(c, ex, total);
        if (i < h1 - h0) cnt[i] = carry + ex;
        carry += total;
        __syncthreads();
      }
      // 4. children in row order (the row is sorted by (degree, index))
      for (int32_t p = h0 + tid; p < h1; p += kT) {
        const int32_t v = (int32_t)order[p];
        int64_t o = (int64_t)h1 + cnt[p - h0];
        for (int64_t e = off[v]; e < off[v + 1]; ++e) {
          const int32_t w = nb[e];
          if (mark[w] == kUnseen && parent[w] == p) order[o++] = w;
        }
      }
      __syncthreads();
      // 5. the new level is visited
      for (int32_t q = h1 + tid; q < h1 + carry; q += kT)
        mark[order[q]] = kWalked;
      __syncthreads();
      h0 = h1;
      h1 += carry;
    }
    pos = h1;
  }
}

} // namespace

extern "C" int pm_rcm_order_device(const int64_t *offsets,
                                   const int32_t *neighbours, int64_t n,
                                   int64_t *order, void *stream) {
  pm::clear_error();
  if (n < 0 || n >= INT32_MAX || (n > 0 && (!offsets || !neighbours ||
                                            !order))) {
    pm::set_error("pm_rcm_order_device: bad arguments (0 <= n < 2^31-1, "
                  "device pointers)");
    return PM_EINVAL;
  }
  if (n == 0) return PM_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int32_t *ws = nullptr;
  // mark, parent, counts (n each) and the status word
  PM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&ws),
                              sizeof(int32_t) * (3 * n + 1), s));
  int32_t *mark = ws, *parent = ws + n, *cnt = ws + 2 * n,
          *status = ws + 3 * n;
  int rc = PM_OK;
  cudaError_t e = cudaMemsetAsync(mark, 0, sizeof(int32_t) * n, s);
  if (e == cudaSuccess)
    e = cudaMemsetAsync(status, 0, sizeof(int32_t), s);
  if (e == cudaSuccess) {
    k_fill_i32<<<pm::grid_for(n, 256), 256, 0, s>>>(parent, n, INT32_MAX);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    k_cuthill_mckee<<<1, kT, 0, s>>>(offsets, neighbours, (int32_t)n, order,
                                     mark, parent, cnt, status);
    e = cudaGetLastError();
  }
  int32_t st = 0;
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&st, status, sizeof(int32_t), cudaMemcpyDeviceToHost,
                        s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(ws, s);
  if (e != cudaSuccess) {
    pm::set_error("pm_rcm_order_device: %s", cudaGetErrorString(e));
    rc = PM_ECUDA;
  } else if (st) {
    pm::set_error("pm_rcm_order_device: neighbour index out of range");
    rc = PM_EINVAL;
  }
  return rc;
}
