// DG column loop with TMA bulk streaming (sm_100a cp.async.bulk).
//
// For a layout with DoFs only on the prism cells ((2,1) entities, e.g.
// DG1 x DG1) Algorithm 1 numbers cell c's column as one block of
// delta*layers values and the cell columns follow each other, so slot j of
// layer l is  map[c][j] + l*offset_j  with  map[c][j] = delta*layers*c + j
// and offset_j = delta: the whole field is a dense (cell, layer, slot)
// array.  Work unit = 256 consecutive cell-layers (one per thread) whose
// x block (256*delta doubles) arrives by one bulk copy into a S-stage
// shared-memory ring (mbarrier completion); each thread applies the element
// kernel in place and the block leaves by one bulk store.  Coordinates are
// gathered per cell-layer through the coordinate map + offsets.
#include "column_loop.cuh"
#include "pm_ptx.cuh"

#include <stdlib.h>

namespace pm {


// S pipeline stages, MINB resident CTAs per SM (register budget), T
// cell-layers per unit (= threads per CTA)
template <int D, int S, int MINB, int T = kStreamT>
__global__ void __launch_bounds__(T, MINB)
k_dg_stream(const MassMat<D> M, int64_t n_units, int64_t cl_begin, int layers,
            const int32_t *__restrict__ xmap,
            const int32_t *__restrict__ xoff,
            const double *__restrict__ coords,
            const double *__restrict__ x, double *__restrict__ y) {
  constexpr uint32_t BYTES = T * D * sizeof(double);
  extern __shared__ __align__(128) unsigned char smem[];
  double *buf = reinterpret_cast<double *>(smem);
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + S * BYTES);
  const int t = threadIdx.x;

  // the coordinate space (COORDS_LAYOUT) moves every slot up by 3 per
  // layer (Alg. 2); the device offsets array holds the same constants
  (void)xoff;
  constexpr int xo[18] = {3, 3, 3, 3, 3, 3, 3, 3, 3,
                          3, 3, 3, 3, 3, 3, 3, 3, 3};

  if (t == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // programmatic dependent launch (pm_set_launch_overlap): the next
  // kernel of the stream may start its prologue, loads and gathers while
  // this grid drains; it waits for this grid before its first store.  A
  // no-op when the launch carries no programmatic dependency.
  asm volatile("griddepcontrol.launch_dependents;");
  bool waited = false;

  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int64_t n_mine =
      first < n_units ? (n_units - first + stride - 1) / stride : 0;

  if (t == 0) {
    for (int64_t i = 0; i < S - 1 && i < n_mine; ++i) {
      const int64_t u = first + i * stride;
      mbar_arrive_expect_tx(&bar[i], BYTES);
      bulk_g2s(buf + i * T * D, x + (cl_begin + u * T) * D, BYTES, &bar[i]);
    }
  }

  // Coordinates are software-pipelined: the coordinate-map entries of unit
  // i+2 and the bottom-level (x,y,z) of the three vertices of unit i+1 are
  // in flight while unit i computes, so neither the map -> coordinate
  // dependency nor the gather latency is exposed.  The top level comes
  // from the next lane (same column, one layer up) or, on a column's last
  // layer / the warp's last lane, from an own (L1-resident) load.  In the
  // coordinate space slot 6a+3b+q sits 3b+q after slot 6a (COORDS_LAYOUT).
  const int lane = t & 31;
  struct Where {
    uint32_t c;
    int l;
  };
  auto where = [&](int64_t u) {
    const uint32_t g = (uint32_t)(cl_begin + u * T + t);
    const uint32_t c = g / (uint32_t)layers;
    return Where{c, (int)(g - c * (uint32_t)layers)};
  };
  auto load_map = [&](const Where &w, int32_t *lx) {
#pragma unroll
    for (int a = 0; a < 3; ++a) lx[a] = __ldg(xmap + (size_t)w.c * 18 + 6 * a);
  };
  auto load_xyz = [&](const Where &w, const int32_t *lx, double *dst) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int q = 0; q < 3; ++q)
        dst[3 * a + q] = __ldg(coords + lx[a] + q + 3 * w.l);
  };
  // lanes whose top level is not the next lane's bottom (warp edge, last
  // layer of a column) prefetch it too
  auto load_top = [&](const Where &w, const int32_t *lx, double *dst) {
    const uint32_t c_up = __shfl_down_sync(0xffffffffu, w.c, 1);
    const bool own = lane == 31 || w.l == layers - 1 || c_up != w.c;
    if (own) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int q = 0; q < 3; ++q)
          dst[3 * a + q] = __ldg(coords + lx[a] + 3 + q + 3 * w.l);
    }
    return own;
  };
  Where w0{0, 0}, w1{0, 0}, w2{0, 0};
  int32_t lx0[3] = {0, 0, 0}, lx1[3] = {0, 0, 0}, lx2[3] = {0, 0, 0};
  double cb[9], nb[9], ct[9], nt[9];
  bool own0 = false, own1 = false;
  if (n_mine > 0) {
    w0 = where(first);
    load_map(w0, lx0);
    load_xyz(w0, lx0, cb);
    own0 = load_top(w0, lx0, ct);
  }
  if (n_mine > 1) {
    w1 = where(first + stride);
    load_map(w1, lx1);
  }
  (void)xo;

  for (int64_t i = 0; i < n_mine; ++i) {
    const int s = (int)(i % S);
    const int64_t u = first + i * stride;
    double *b = buf + s * T * D;
    if (i + 1 < n_mine) {
      load_xyz(w1, lx1, nb);
      own1 = load_top(w1, lx1, nt);
    }
    if (i + 2 < n_mine) {
      w2 = where(u + 2 * stride);
      load_map(w2, lx2);
    }

    // top level of this cell-layer: the next lane's bottom, or prefetched
    double X[6], Y[6], Z[6];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double top[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const double up = __shfl_down_sync(0xffffffffu, cb[3 * a + q], 1);
        top[q] = own0 ? ct[3 * a + q] : up;
      }
      X[2 * a] = cb[3 * a], Y[2 * a] = cb[3 * a + 1], Z[2 * a] = cb[3 * a + 2];
      X[2 * a + 1] = top[0], Y[2 * a + 1] = top[1], Z[2 * a + 1] = top[2];
    }
    const double det = prism_abs_detj(X, Y, Z);

    mbar_wait(&bar[s], (uint32_t)((i / S) & 1));
    double xv[D], yv[D];
    if constexpr (D % 2 == 0) { // 16-byte shared accesses: conflict-free
      const double2 *b2 = reinterpret_cast<const double2 *>(b + t * D);
#pragma unroll
      for (int j = 0; j < D / 2; ++j) {
        const double2 v = b2[j];
        xv[2 * j] = v.x;
        xv[2 * j + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < D; ++j) xv[j] = b[t * D + j];
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < D; ++q) acc = fma(M.m[j * D + q], xv[q], acc);
      yv[j] = det * acc;
    }
    if constexpr (D % 2 == 0) {
      double2 *b2 = reinterpret_cast<double2 *>(b + t * D);
#pragma unroll
      for (int j = 0; j < D / 2; ++j) b2[j] = make_double2(yv[2 * j], yv[2 * j + 1]);
    } else {
#pragma unroll
      for (int j = 0; j < D; ++j) b[t * D + j] = yv[j];
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (t == 0) {
      if (!waited) { // the previous grid (same y) has finished
        asm volatile("griddepcontrol.wait;" ::: "memory");
        waited = true;
      }
      bulk_s2g(y + (cl_begin + u * T) * D, b, BYTES);
      bulk_commit();
      const int64_t nxt = i + S - 1;
      if (nxt < n_mine) {
        // stage of unit i-1: its store (one group back) must have read smem
        bulk_wait_read<1>();
        const int sn = (int)(nxt % S);
        mbar_arrive_expect_tx(&bar[sn], BYTES);
        bulk_g2s(buf + sn * T * D,
                 x + (cl_begin + (first + nxt * stride) * T) * D, BYTES,
                 &bar[sn]);
      }
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) cb[q] = nb[q], ct[q] = nt[q];
    own0 = own1;
    w0 = w1;
    w1 = w2;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lx0[a] = lx1[a];
      lx1[a] = lx2[a];
    }
  }
  if (t == 0) bulk_wait<0>();
}

template <int D, int S, int MINB, int T = kStreamT>
static int dg_stream_launch(const LoopArgs &a, const MassMat<D> &M,
                            int64_t n_units, int64_t cl_begin) {
  const size_t smem = S * T * D * sizeof(double) + S * sizeof(uint64_t);
  auto kern = k_dg_stream<D, S, MINB, T>;
  // the attribute and the occupancy are properties of the instantiation:
  // queried once (per device), not on every call
  static int cached_dev = -1, per_sm = 0;
  int dev = 0;
  PM_CUDA_TRY(cudaGetDevice(&dev));
  if (cached_dev != dev) {
    PM_CUDA_TRY(cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int nb = 0;
    PM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T,
                                                              smem));
    per_sm = nb < 1 ? 1 : nb;
    cached_dev = dev;
  }
  int64_t grid = (int64_t)sm_count() * per_sm;
  if (grid > n_units) grid = n_units;
  if (launch_overlap()) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = a.s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, M, n_units, cl_begin, a.layers,
                                   a.xmap, a.xoff, a.coords, a.x, a.y));
  } else {
    kern<<<(unsigned)grid, T, smem, a.s>>>(M, n_units, cl_begin, a.layers,
                                           a.xmap, a.xoff, a.coords, a.x,
                                           a.y);
  }
  PM_LAUNCH_CHECK("k_dg_stream");
  return PM_OK;
}

// Stream pipeline shape: 8 stages x 2 CTAs/SM (default; 14 bulk loads of
// 12 KB in flight per SM, no spills) or PM_STREAM_CFG=0: 6 stages x 3 CTAs
// (measured 68% vs 76% of HBM on C2, profiles/).
// Default by DoFs per cell-layer: 256-cell-layer units, 2 CTAs/SM for
// DG1 x DG1; 128-cell-layer units, 4 CTAs/SM for the smaller blocks
// (measured 3-4 % faster for D = 1, 2, 3 at lambda = 100).
static int stream_cfg(int D) {
  static int cfg = -2;
  if (cfg == -2) {
    const char *e = getenv("PM_STREAM_CFG");
    cfg = e ? atoi(e) : -1;
  }
  return cfg >= 0 ? cfg : (D >= 6 ? 1 : 2);
}

// The stream kernel never reads the field's cell map: it relies on the
// (2,1)-only layout being numbered by Alg. 1 (fspace.py:134-229), which
// makes the field a dense (cell, layer, slot) array: map[c][j] =
// c*k*layers + j, offsets[j] = k.  A caller-supplied map is checked once on
// the device (maps are immutable, fspace.py:159-174; the verdict is cached
// per (map, offsets, k, layers) and checked prefix); a map that is not dense, or an
// unchecked one met during stream capture, sends the launch to the
// map-reading kernels instead.
__global__ void k_dense_map_check(const int32_t *__restrict__ map,
                                  const int32_t *__restrict__ off,
                                  int64_t n_cells, int k, int layers,
                                  int *__restrict__ bad) {
  const int64_t n = n_cells * k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / k;
    const int j = (int)(i - c * k);
    if ((int64_t)map[i] != c * k * layers + j) atomicOr(bad, 1);
    if (i < k && off[i] != k) atomicOr(bad, 1);
  }
}

static int dense_map_ok(const LoopArgs &a, bool *ok) {
  struct Entry {
    const int32_t *map, *off;
    int64_t n_cells;
    int k, layers, dev;
    bool ok;
  };
  static Entry cache[32];
  static int next = 0;
  int dev = 0;
  PM_CUDA_TRY(cudaGetDevice(&dev));
  // an entry covers the map's first n_cells rows (the host path's chunks
  // are prefixes [0, cell_end) of one map)
  for (const Entry &e : cache)
    if (e.map == a.cmap && e.off == a.coff && e.k == a.k &&
        e.layers == a.layers && e.dev == dev &&
        (!e.ok || a.n_cells <= e.n_cells)) {
      *ok = e.ok;
      return PM_OK;
    }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  PM_CUDA_TRY(cudaStreamIsCapturing(a.s, &cs));
  if (cs != cudaStreamCaptureStatusNone) { // cannot synchronise: unchecked
    *ok = false;
    return PM_OK;
  }
  int *bad = nullptr;
  PM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&bad), sizeof(int),
                              a.s));
  int h = 1;
  cudaError_t err = cudaMemsetAsync(bad, 0, sizeof(int), a.s);
  if (err == cudaSuccess) {
    k_dense_map_check<<<grid_for(a.n_cells * a.k, 256, 4), 256, 0, a.s>>>(
        a.cmap, a.coff, a.n_cells, a.k, a.layers, bad);
    err = cudaGetLastError();
  }
  if (err == cudaSuccess)
    err = cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, a.s);
  if (err == cudaSuccess) err = cudaStreamSynchronize(a.s);
  cudaFreeAsync(bad, a.s);
  PM_CUDA_TRY(err);
  *ok = h == 0;
  cache[next] = {a.cmap, a.coff, a.n_cells, a.k, a.layers, dev, *ok};
  next = (next + 1) % 32;
  return PM_OK;
}

// cell-layers [cl_begin, n_cells*layers) of the DG field (cl_begin must be
// a multiple of the unit size so the bulk copies stay 16-byte aligned)
template <int D>
static int dg_stream_k(const LoopArgs &a, bool *handled, int64_t cl_begin) {
  *handled = false;
  bool dense = false;
  int rc0 = dense_map_ok(a, &dense);
  if (rc0 || !dense) return rc0; // the map-reading kernels take the launch
  const int64_t n_cl = a.n_cells * (int64_t)a.layers - cl_begin;
  const int cfg = stream_cfg(D);
  const int T = cfg == 2 ? 128 : cfg == 3 ? 512 : kStreamT;
  const int64_t n_units = n_cl / T;
  if ((reinterpret_cast<uintptr_t>(a.x) | reinterpret_cast<uintptr_t>(a.y)) &
      15)
    return PM_OK; // not aligned for bulk copies: caller picks another kernel
  if (n_cl > 0xFFFFFFFFll) return PM_OK;
  MassMat<D> M;
  for (int i = 0; i < D * D; ++i) M.m[i] = a.mref[i];
  if (n_units > 0) {
    int rc;
    switch (cfg) {
    case 0: rc = dg_stream_launch<D, 6, 3>(a, M, n_units, cl_begin); break;
    case 2:
      rc = dg_stream_launch<D, 8, 4, 128>(a, M, n_units, cl_begin);
      break;
    case 3:
      rc = dg_stream_launch<D, 4, 1, 512>(a, M, n_units, cl_begin);
      break;
    default: rc = dg_stream_launch<D, 8, 2>(a, M, n_units, cl_begin); break;
    }
    if (rc) return rc;
  }
  *handled = true;
  // ragged tail (< one unit): flattened generic kernel, plain stores
  if (n_units * T < n_cl)
    return launch_generic(a, false, cl_begin + n_units * T);
  return PM_OK;
}

int launch_dg_stream(const LoopArgs &a, bool *handled, int64_t cl_begin) {
  switch (a.k) {
  case 1: return dg_stream_k<1>(a, handled, cl_begin);
  case 2: return dg_stream_k<2>(a, handled, cl_begin);
  case 3: return dg_stream_k<3>(a, handled, cl_begin);
  case 6: return dg_stream_k<6>(a, handled, cl_begin);
  default:
    *handled = false;
    return PM_OK;
  }
}

} // namespace pm

// DG stream over the cell range [cell_begin, cell_end): the pipelined host
// path of kernels.mass_action launches one chunk per call.
extern "C" int pm_column_mass_dg_range(const int32_t *delta6, int32_t k,
                                       int64_t cell_begin, int64_t cell_end,
                                       int32_t layers, const int32_t *cell_map,
                                       const int32_t *offsets,
                                       const int32_t *coord_map,
                                       const int32_t *coord_offsets,
                                       const double *coords,
                                       const double *mref, const double *x,
                                       double *y, void *stream) {
  pm::clear_error();
  pm::LoopArgs a;
  int rc = pm::make_slot_table(delta6, &a.st);
  if (rc) return rc;
  const bool dg_only = !delta6[0] && !delta6[1] && !delta6[2] &&
                       !delta6[3] && !delta6[4];
  if (k != a.st.k || layers < 1 || cell_begin < 0 || cell_end < cell_begin ||
      !mref || !dg_only) {
    pm::set_error("bad arguments to pm_column_mass_dg_range");
    return PM_EINVAL;
  }
  if (cell_end == cell_begin) return PM_OK;
  if (((cell_begin * (int64_t)layers) % pm::kStreamT) != 0) {
    pm::set_error("cell_begin*layers must be a multiple of %d",
                  pm::kStreamT);
    return PM_EINVAL;
  }
  a.k = k;
  a.layers = layers;
  a.n_cells = cell_end;
  a.cells = nullptr;
  a.cmap = cell_map; // the ragged tail (generic kernel) addresses via the map
  a.coff = offsets;
  a.xmap = coord_map;
  a.xoff = coord_offsets;
  a.coords = coords;
  a.mref = mref;
  a.x = x;
  a.y = y;
  a.accumulate = 0;
  a.dg_only = true;
  a.hshared = false;
  a.s = (cudaStream_t)stream;
  bool handled = false;
  rc = pm::launch_dg_stream(a, &handled, cell_begin * (int64_t)layers);
  if (!rc && !handled) {
    pm::set_error("DG range needs 16-byte aligned fields");
    return PM_EINVAL;
  }
  return rc;
}
