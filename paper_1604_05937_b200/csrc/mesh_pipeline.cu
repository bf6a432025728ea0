// Device base-mesh pipeline: the two host steps that
// dominate setup at 2048^2 (derive_edges, the cell re-sort of
// apply_ordering) as radix sorts on the GPU, bit-exact with the host
// restatements (mesh.py derive_edges, ordering.py apply_ordering).
//
// derive_edges (reference mesh.py:33-84): side k of cell c is the vertex
// pair opposite local vertex k, key (min << 32) | max at position k*C + c
// of the concatenated side list; edges are the sorted unique keys and
// cell_edges[c][k] the rank of its key (np.unique's inverse).  Here: one
// stable radix sort of (key, position), run heads, an inclusive scan for
// the edge ids and a scatter.  Topology errors are flagged on the device
// (the host validator then produces the reference's exact message).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "pm_common.cuh"

namespace {

enum : int32_t {
  kNegative = 1,    // negative vertex index
  kRange = 2,       // vertex index >= n_vertices
  kRepeated = 4,    // a cell with repeated vertices
  kDupCell = 8,     // two cells with the same vertex set
  kManyCells = 16,  // an edge shared by more than two cells
};

__device__ __forceinline__ void flag(int32_t *status, int32_t bit) {
  atomicOr(status, bit);
}

__global__ void k_side_keys(const int32_t *__restrict__ cells, int64_t C,
                            int64_t nv, uint64_t *__restrict__ keys,
                            int32_t *__restrict__ pos,
                            int32_t *__restrict__ status) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = cells[3 * c], b = cells[3 * c + 1], d = cells[3 * c + 2];
    if (a < 0 || b < 0 || d < 0) flag(status, kNegative);
    if (nv >= 0 && (a >= nv || b >= nv || d >= nv)) flag(status, kRange);
    if (a == b || b == d || a == d) flag(status, kRepeated);
    const int64_t v[3] = {a, b, d};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int64_t p = v[(k + 1) % 3], q = v[(k + 2) % 3];
      const uint64_t lo = (uint64_t)(p < q ? p : q), hi = (uint64_t)(p < q ? q : p);
      keys[k * C + c] = (lo << 32) | (hi & 0xffffffffull);
      pos[k * C + c] = (int32_t)(k * C + c);
    }
  }
}

__global__ void k_heads(const uint64_t *__restrict__ sk,
                        const int32_t *__restrict__ sp,
                        const int32_t *__restrict__ cells, int64_t C,
                        int64_t n, int32_t *__restrict__ head,
                        int32_t *__restrict__ status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool same = i > 0 && sk[i] == sk[i - 1];
    head[i] = same ? 0 : 1;
    if (i > 1 && sk[i] == sk[i - 2]) flag(status, kManyCells);
    if (same) {
      // two cells on one edge with the same opposite vertex: same vertex set
      const int64_t p1 = sp[i - 1], p2 = sp[i];
      const int64_t c1 = p1 % C, k1 = p1 / C, c2 = p2 % C, k2 = p2 / C;
      if (cells[3 * c1 + k1] == cells[3 * c2 + k2]) flag(status, kDupCell);
    }
  }
}

__global__ void k_scatter_edges(const uint64_t *__restrict__ sk,
                                const int32_t *__restrict__ sp,
                                const int32_t *__restrict__ head,
                                const int32_t *__restrict__ ids, int64_t C,
                                int64_t n, int32_t *__restrict__ edge_vertices,
                                int32_t *__restrict__ cell_edges) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = ids[i] - 1;
    const int64_t p = sp[i];
    cell_edges[3 * (p % C) + p / C] = e;
    if (head[i]) {
      edge_vertices[2 * (int64_t)e] = (int32_t)(sk[i] >> 32);
      edge_vertices[2 * (int64_t)e + 1] = (int32_t)(sk[i] & 0xffffffffull);
    }
  }
}

// apply_ordering's cell keys: new vertex numbers, the sorted triple
// (t0 < t1 < t2) as a 64-bit (t0, t1) key and the t2 key
__global__ void k_order_keys(const int32_t *__restrict__ cells, int64_t C,
                             const int64_t *__restrict__ fwd,
                             int32_t *__restrict__ mapped,
                             uint64_t *__restrict__ key01,
                             uint32_t *__restrict__ key2,
                             int32_t *__restrict__ idx) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x) {
    int64_t t[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      t[j] = fwd[cells[3 * c + j]];
      mapped[3 * c + j] = (int32_t)t[j];
    }
    if (t[0] > t[1]) { const int64_t s = t[0]; t[0] = t[1]; t[1] = s; }
    if (t[1] > t[2]) { const int64_t s = t[1]; t[1] = t[2]; t[2] = s; }
    if (t[0] > t[1]) { const int64_t s = t[0]; t[0] = t[1]; t[1] = s; }
    key01[c] = ((uint64_t)t[0] << 32) | (uint64_t)t[1];
    key2[c] = (uint32_t)t[2];
    idx[c] = (int32_t)c;
  }
}

__global__ void k_gather_u64(const uint64_t *__restrict__ src,
                             const int32_t *__restrict__ idx, int64_t n,
                             uint64_t *__restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

__global__ void k_gather_rows(const int32_t *__restrict__ mapped,
                              const int32_t *__restrict__ perm, int64_t C,
                              int32_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < C;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = perm[i];
#pragma unroll
    for (int j = 0; j < 3; ++j) out[3 * i + j] = mapped[3 * c + j];
  }
}

__global__ void k_degree(const int32_t *__restrict__ ev, int64_t ne,
                         int32_t *__restrict__ deg) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd(deg + ev[2 * e], 1);
    atomicAdd(deg + ev[2 * e + 1], 1);
  }
}

// both directions of every edge, keyed (row, degree(neighbour), neighbour)
__global__ void k_graph_keys(const int32_t *__restrict__ ev, int64_t ne,
                             const int32_t *__restrict__ deg,
                             uint64_t *__restrict__ keys) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = (uint32_t)ev[2 * e], b = (uint32_t)ev[2 * e + 1];
    keys[2 * e] = (a << 40) | ((uint64_t)deg[b] << 32) | b;
    keys[2 * e + 1] = (b << 40) | ((uint64_t)deg[a] << 32) | a;
  }
}

__global__ void k_graph_unpack(const uint64_t *__restrict__ keys, int64_t n,
                               int32_t *__restrict__ nbr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    nbr[i] = (int32_t)(keys[i] & 0xffffffffull);
}

__global__ void k_widen(const int32_t *__restrict__ a, int64_t n,
                        int64_t *__restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

__global__ void k_offsets(int64_t n, const int64_t *__restrict__ incl,
                          int64_t *__restrict__ offsets) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    offsets[i] = i == 0 ? 0 : incl[i - 1];
}

int bits_for(int64_t n) { // bits to hold values < n (n >= 1)
  int b = 0;
  while (b < 63 && ((int64_t)1 << b) < n) ++b;
  return b < 1 ? 1 : b;
}

// stream-ordered scratch, freed on every exit path
struct Scratch {
  cudaStream_t s;
  void *p[8] = {};
  int n = 0;
  explicit Scratch(cudaStream_t st) : s(st) {}
  template <class T> cudaError_t get(T **out, size_t count) {
    void *q = nullptr;
    const cudaError_t e = cudaMallocAsync(&q, count ? count * sizeof(T) : 1, s);
    if (e == cudaSuccess) p[n++] = q;
    *out = static_cast<T *>(q);
    return e;
  }
  ~Scratch() {
    for (int i = 0; i < n; ++i) cudaFreeAsync(p[i], s);
  }
};

} // namespace

extern "C" int pm_derive_edges(const int32_t *cell_vertices, int64_t n_cells,
                               int64_t n_vertices, int32_t *edge_vertices,
                               int32_t *cell_edges, int64_t *n_edges,
                               int32_t *status, void *stream) {
  pm::clear_error();
  if (n_cells < 0 || !n_edges || !status) {
    pm::set_error("pm_derive_edges: bad arguments");
    return PM_EINVAL;
  }
  if (3 * n_cells > INT32_MAX) {
    pm::set_error("pm_derive_edges: %lld cells exceed the int32 side index",
                  (long long)n_cells);
    return PM_EINVAL;
  }
  *n_edges = 0;
  *status = 0;
  if (!n_cells) return PM_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t C = n_cells, n = 3 * C;
  Scratch w(s);
  uint64_t *k0, *k1;
  int32_t *p0, *p1, *head, *ids, *d_status;
  PM_CUDA_TRY(w.get(&k0, n));
  PM_CUDA_TRY(w.get(&k1, n));
  PM_CUDA_TRY(w.get(&p0, n));
  PM_CUDA_TRY(w.get(&p1, n));
  PM_CUDA_TRY(w.get(&head, n));
  PM_CUDA_TRY(w.get(&ids, n));
  PM_CUDA_TRY(w.get(&d_status, 1));
  PM_CUDA_TRY(cudaMemsetAsync(d_status, 0, sizeof(int32_t), s));
  const unsigned g = pm::grid_for(C, 256);
  k_side_keys<<<g, 256, 0, s>>>(cell_vertices, C, n_vertices, k0, p0,
                                d_status);
  PM_LAUNCH_CHECK("k_side_keys");
  PM_CUDA_TRY(cudaMemcpyAsync(status, d_status, sizeof(int32_t),
                              cudaMemcpyDeviceToHost, s));
  PM_CUDA_TRY(cudaStreamSynchronize(s));
  if (*status) return PM_OK; // invalid cells: the caller reports
  // largest vertex id bounds the key bits
  const int64_t nv = n_vertices >= 0 ? n_vertices : ((int64_t)1 << 31);
  const int vb = bits_for(nv);
  cub::DoubleBuffer<uint64_t> keys(k0, k1);
  cub::DoubleBuffer<int32_t> vals(p0, p1);
  size_t tb = 0, tb2 = 0;
  PM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, vals, (int)n,
                                              0, 32 + vb, s));
  PM_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tb2, head, ids, (int)n, s));
  char *tmp;
  PM_CUDA_TRY(w.get(&tmp, tb > tb2 ? tb : tb2));
  PM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, vals, (int)n, 0,
                                              32 + vb, s));
  const unsigned gn = pm::grid_for(n, 256);
  k_heads<<<gn, 256, 0, s>>>(keys.Current(), vals.Current(), cell_vertices, C,
                             n, head, d_status);
  PM_LAUNCH_CHECK("k_heads");
  PM_CUDA_TRY(cub::DeviceScan::InclusiveSum(tmp, tb2, head, ids, (int)n, s));
  k_scatter_edges<<<gn, 256, 0, s>>>(keys.Current(), vals.Current(), head, ids,
                                     C, n, edge_vertices, cell_edges);
  PM_LAUNCH_CHECK("k_scatter_edges");
  int32_t last = 0;
  PM_CUDA_TRY(cudaMemcpyAsync(&last, ids + n - 1, sizeof(int32_t),
                              cudaMemcpyDeviceToHost, s));
  PM_CUDA_TRY(cudaMemcpyAsync(status, d_status, sizeof(int32_t),
                              cudaMemcpyDeviceToHost, s));
  PM_CUDA_TRY(cudaStreamSynchronize(s));
  *n_edges = last;
  return PM_OK;
}

// The vertex graph of the mesh (edge-adjacent vertices) as CSR with every
// row sorted by (degree, index): the input of the RCM breadth-first search
// (reference ordering.py rcm_order: mesh.vertex_neighbours + the row
// lexsort), which the host then walks (pm_rcm_order).
extern "C" int pm_vertex_graph_sorted(const int32_t *edge_vertices,
                                      int64_t n_edges, int64_t n_vertices,
                                      int64_t *offsets, int32_t *nbr,
                                      void *stream) {
  pm::clear_error();
  if (n_edges < 0 || n_vertices < 0 || n_vertices >= (1 << 24) ||
      2 * n_edges > INT32_MAX) {
    pm::set_error("pm_vertex_graph_sorted: sizes out of range (vertices "
                  "< 2^24, 2*edges < 2^31)");
    return PM_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (n_vertices == 0) return PM_OK;
  Scratch w(s);
  int32_t *deg;
  int64_t *deg64, *incl;
  uint64_t *k0, *k1;
  const int64_t n2 = 2 * n_edges;
  PM_CUDA_TRY(w.get(&deg, n_vertices));
  PM_CUDA_TRY(w.get(&deg64, n_vertices));
  PM_CUDA_TRY(w.get(&incl, n_vertices));
  PM_CUDA_TRY(w.get(&k0, n2));
  PM_CUDA_TRY(w.get(&k1, n2));
  PM_CUDA_TRY(cudaMemsetAsync(deg, 0, sizeof(int32_t) * n_vertices, s));
  if (n_edges) {
    k_degree<<<pm::grid_for(n_edges, 256), 256, 0, s>>>(edge_vertices,
                                                        n_edges, deg);
    PM_LAUNCH_CHECK("k_degree");
  }
  k_widen<<<pm::grid_for(n_vertices, 256), 256, 0, s>>>(deg, n_vertices,
                                                        deg64);
  PM_LAUNCH_CHECK("k_widen");
  size_t tb = 0, tb2 = 0;
  PM_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tb, deg64, incl,
                                            (int)n_vertices, s));
  cub::DoubleBuffer<uint64_t> keys(k0, k1);
  const int end_bit = 40 + bits_for(n_vertices);
  if (n2)
    PM_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tb2, keys, (int)n2, 0,
                                               end_bit, s));
  char *tmp;
  PM_CUDA_TRY(w.get(&tmp, tb > tb2 ? tb : tb2));
  PM_CUDA_TRY(cub::DeviceScan::InclusiveSum(tmp, tb, deg64, incl,
                                            (int)n_vertices, s));
  k_offsets<<<pm::grid_for(n_vertices + 1, 256), 256, 0, s>>>(
      n_vertices, incl, offsets);
  PM_LAUNCH_CHECK("k_offsets");
  if (n2) {
    k_graph_keys<<<pm::grid_for(n_edges, 256), 256, 0, s>>>(
        edge_vertices, n_edges, deg, k0);
    PM_LAUNCH_CHECK("k_graph_keys");
    PM_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp, tb2, keys, (int)n2, 0,
                                               end_bit, s));
    k_graph_unpack<<<pm::grid_for(n2, 256), 256, 0, s>>>(keys.Current(), n2,
                                                         nbr);
    PM_LAUNCH_CHECK("k_graph_unpack");
  }
  PM_CUDA_TRY(cudaStreamSynchronize(s));
  return PM_OK;
}

extern "C" int pm_reorder_cells(const int32_t *cell_vertices, int64_t n_cells,
                                const int64_t *forward, int64_t n_vertices,
                                int32_t *cells_out, int32_t *perm_out,
                                void *stream) {
  pm::clear_error();
  if (n_cells < 0 || n_vertices < 0 || n_vertices > INT32_MAX ||
      n_cells > INT32_MAX) {
    pm::set_error("pm_reorder_cells: bad sizes");
    return PM_EINVAL;
  }
  if (!n_cells) return PM_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t C = n_cells;
  Scratch w(s);
  int32_t *mapped, *i0, *i1;
  uint64_t *a0, *a1;
  uint32_t *b0, *b1;
  PM_CUDA_TRY(w.get(&mapped, 3 * C));
  PM_CUDA_TRY(w.get(&i0, C));
  PM_CUDA_TRY(w.get(&i1, C));
  PM_CUDA_TRY(w.get(&a0, C));
  PM_CUDA_TRY(w.get(&a1, C));
  PM_CUDA_TRY(w.get(&b0, C));
  PM_CUDA_TRY(w.get(&b1, C));
  const unsigned g = pm::grid_for(C, 256);
  k_order_keys<<<g, 256, 0, s>>>(cell_vertices, C, forward, mapped, a0, b0,
                                 i0);
  PM_LAUNCH_CHECK("k_order_keys");
  const int vb = bits_for(n_vertices > 0 ? n_vertices : 1);
  // lexsort((t2, t1, t0)): stable LSD passes, t2 first, then (t0, t1)
  cub::DoubleBuffer<uint32_t> kb(b0, b1);
  cub::DoubleBuffer<int32_t> iv(i0, i1);
  size_t t1 = 0, t2 = 0;
  PM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, t1, kb, iv, (int)C, 0,
                                              vb, s));
  cub::DoubleBuffer<uint64_t> ka(a1, a0);
  PM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, t2, ka, iv, (int)C, 0,
                                              32 + vb, s));
  char *tmp;
  PM_CUDA_TRY(w.get(&tmp, t1 > t2 ? t1 : t2));
  PM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, t1, kb, iv, (int)C, 0, vb,
                                              s));
  // (t0, t1) keys in the order of the first pass
  k_gather_u64<<<g, 256, 0, s>>>(a0, iv.Current(), C, a1);
  PM_LAUNCH_CHECK("k_gather_u64");
  cub::DoubleBuffer<uint64_t> kk(a1, a0);
  PM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, t2, kk, iv, (int)C, 0,
                                              32 + vb, s));
  k_gather_rows<<<g, 256, 0, s>>>(mapped, iv.Current(), C, cells_out);
  PM_LAUNCH_CHECK("k_gather_rows");
  if (perm_out)
    PM_CUDA_TRY(cudaMemcpyAsync(perm_out, iv.Current(), C * sizeof(int32_t),
                                cudaMemcpyDeviceToDevice, s));
  PM_CUDA_TRY(cudaStreamSynchronize(s));
  return PM_OK;
}
