// K0: column-innermost numbering -> bottom-layer cell maps and offsets,
// the extruded coordinate field, par-loop probes and the halo pack/unpack.
//
// Numbering (reference fspace.py:137-149, Alg. 1): base entities
// of dimension d own consecutive columns of
//     column_d = layers*(delta(d,0)+delta(d,1)) + delta(d,0)
// numbers, vertices first, then edges, then cells.  Slot j of cell c maps to
//     start[dim_j] + column[dim_j]*entity(c, j) + within_j
// (fspace.py:192-215) and moves up one layer by offset_j
// (fspace.py:218-229, Alg. 2).
#include "pm_common.cuh"

namespace {

struct MapArgs {
  int64_t start[3];
  int64_t column[3];
  int32_t k;
  int8_t kind[pm::kMaxSlots];
  int8_t local[pm::kMaxSlots];
  int32_t within[pm::kMaxSlots];
};

// One thread per (cell, slot); consecutive threads write consecutive map
// entries, so the int32 map store is fully coalesced.  The per-slot
// tables live in shared memory (lanes of a warp index different slots:
// from kernel parameters that would serialise the constant cache) and the
// (cell, slot) split is 32-bit when the map has < 2^31 entries.
template <typename I>
__global__ void __launch_bounds__(256)
k_build_cell_map(const MapArgs a, const int32_t *__restrict__ cv,
                 const int32_t *__restrict__ ce, int64_t n_cells,
                 int32_t *__restrict__ map) {
  __shared__ int8_t s_kind[pm::kMaxSlots], s_local[pm::kMaxSlots];
  __shared__ int64_t s_base[pm::kMaxSlots], s_col[pm::kMaxSlots];
  for (int j = threadIdx.x; j < a.k; j += blockDim.x) {
    const int kd = a.kind[j];
    s_kind[j] = (int8_t)kd;
    s_local[j] = a.local[j];
    s_base[j] = a.start[kd] + a.within[j];
    s_col[j] = a.column[kd];
  }
  __syncthreads();
  const I k = (I)a.k;
  const I total = (I)(n_cells * a.k);
  auto entry = [&](I c, int j) {
    const int kind = s_kind[j];
    int64_t ent;
    if (kind == 0)
      ent = __ldg(cv + 3 * (int64_t)c + s_local[j]);
    else if (kind == 1)
      ent = __ldg(ce + 3 * (int64_t)c + s_local[j]);
    else
      ent = c;
    const int64_t v = s_base[j] + s_col[j] * ent;
    return (int32_t)(uint32_t)(uint64_t)v; // numpy int64->int32 store wraps
  };
  // four consecutive entries per thread: one division, one 16-byte store
  for (I q = (I)(blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
       4 * q < total; q += (I)((int64_t)gridDim.x * blockDim.x)) {
    const I t = 4 * q;
    I c = t / k;
    int j = (int)(t - c * k);
    int32_t e[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      e[u] = t + u < total ? entry(c, j) : 0;
      if (++j == (int)k) j = 0, ++c;
    }
    if (t + 3 < total) {
      reinterpret_cast<int4 *>(map)[q] = make_int4(e[0], e[1], e[2], e[3]);
    } else {
      for (int u = 0; t + u < total; ++u) map[t + u] = e[u];
    }
  }
}

struct OffsetArgs {
  int32_t v[pm::kMaxSlots];
};

__global__ void k_offsets(const OffsetArgs a, int k, int32_t *__restrict__ dst) {
  int j = threadIdx.x;
  if (j < k) dst[j] = a.v[j];
}

// out[3*(i*(L+1)+l)+c]: one thread per output pair, one 16-byte store
// (out is 16-byte aligned), coalesced; 32-bit index split when the field
// has < 2^31 values.
template <typename I>
__global__ void __launch_bounds__(256)
k_extrude(const double *__restrict__ base, int64_t n_vertices, int layers,
          double h, double *__restrict__ out) {
  const I per = 3 * (I)(layers + 1);
  const I total = (I)(n_vertices * per);
  auto value = [&](I i, int r) {
    const int l = r / 3, c = r - 3 * l;
    return c < 2 ? __ldg(base + 2 * (int64_t)i + c) : (double)l * h;
  };
  for (I p = (I)(blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
       2 * p < total; p += (I)((int64_t)gridDim.x * blockDim.x)) {
    const I t = 2 * p;
    I i = t / per;
    int r = (int)(t - i * per);
    const double v0 = value(i, r);
    if (t + 1 < total) {
      if (++r == (int)per) r = 0, ++i;
      reinterpret_cast<double2 *>(out)[p] = make_double2(v0, value(i, r));
    } else {
      out[t] = v0;
    }
  }
}

// Probe 0: materialise every (cell, layer) DoF list via map + l*offset.
__global__ void __launch_bounds__(256)
k_probe_lists(int k, int64_t n_cells, int layers,
              const int32_t *__restrict__ map,
              const int32_t *__restrict__ off, int64_t *__restrict__ out) {
  const int64_t total = n_cells * layers * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cl = t / k;
    const int j = (int)(t - cl * k);
    const int64_t c = cl / layers;
    const int l = (int)(cl - c * layers);
    out[t] = (int64_t)__ldg(map + c * k + j) + (int64_t)l * __ldg(off + j);
  }
}

// Probe 1: counting kernel (+1 per slot per application).
__global__ void __launch_bounds__(256)
k_probe_count(int k, int64_t n_cells, int layers,
              const int32_t *__restrict__ map,
              const int32_t *__restrict__ off, double *__restrict__ out) {
  const int64_t total = n_cells * layers * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cl = t / k;
    const int j = (int)(t - cl * k);
    const int64_t c = cl / layers;
    const int l = (int)(cl - c * layers);
    atomicAdd(out + (int64_t)__ldg(map + c * k + j) +
                  (int64_t)l * __ldg(off + j),
              1.0);
  }
}

__global__ void __launch_bounds__(256)
k_halo_pack(const double *__restrict__ y, const int64_t *__restrict__ cols,
            int64_t n_cols, int col, double *__restrict__ buf) {
  const int64_t total = n_cols * col;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / col;
    buf[t] = y[__ldg(cols + i) + (t - i * col)];
  }
}

__global__ void __launch_bounds__(256)
k_halo_unpack_add(double *__restrict__ y, const int64_t *__restrict__ cols,
                  int64_t n_cols, int col, const double *__restrict__ buf) {
  const int64_t total = n_cols * col;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / col;
    y[__ldg(cols + i) + (t - i * col)] += buf[t];
  }
}

} // namespace

extern "C" int pm_build_cell_map(const int32_t *cell_vertices,
                                 const int32_t *cell_edges, int64_t n_cells,
                                 int64_t n_vertices, int64_t n_edges,
                                 const int32_t *delta6, int32_t layers,
                                 int32_t k, int32_t *cell_map,
                                 int32_t *offsets, int64_t *total_dofs,
                                 void *stream) {
  pm::clear_error();
  if (layers < 1) {
    pm::set_error("layer count must be >= 1, got %d", layers);
    return PM_EINVAL;
  }
  if (n_cells < 0 || n_vertices < 0 || n_edges < 0) {
    pm::set_error("negative entity count");
    return PM_EINVAL;
  }
  pm::SlotTable st;
  int rc = pm::make_slot_table(delta6, &st);
  if (rc) return rc;
  if (k != st.k) {
    pm::set_error("slot count mismatch: caller k=%d, layout has %d", k, st.k);
    return PM_EINVAL;
  }
  MapArgs a;
  const int64_t counts[3] = {n_vertices, n_edges, n_cells};
  int64_t acc = 0;
  for (int d = 0; d < 3; ++d) {
    a.start[d] = acc;
    a.column[d] = (int64_t)layers * (delta6[2 * d] + delta6[2 * d + 1]) +
                  delta6[2 * d];
    acc += a.column[d] * counts[d];
  }
  a.k = st.k;
  OffsetArgs o;
  for (int j = 0; j < st.k; ++j) {
    a.kind[j] = st.kind[j];
    a.local[j] = st.local[j];
    a.within[j] = st.within[j];
    o.v[j] = st.offset[j];
  }
  if (total_dofs) *total_dofs = acc;
  cudaStream_t s = (cudaStream_t)stream;
  if (n_cells > 0) {
    if (!cell_map || (st.kind[0] != 2 && !cell_vertices) ||
        (n_edges > 0 && !cell_edges)) {
      pm::set_error("NULL map / connectivity pointer");
      return PM_EINVAL;
    }
    const int64_t total = n_cells * st.k;
    if (reinterpret_cast<uintptr_t>(cell_map) & 15) {
      pm::set_error("cell map must be 16-byte aligned");
      return PM_EINVAL;
    }
    const unsigned g = pm::grid_for((total + 3) / 4, 256);
    if (total < ((int64_t)1 << 31))
      k_build_cell_map<uint32_t><<<g, 256, 0, s>>>(a, cell_vertices,
                                                  cell_edges, n_cells,
                                                  cell_map);
    else
      k_build_cell_map<int64_t><<<g, 256, 0, s>>>(a, cell_vertices,
                                                 cell_edges, n_cells,
                                                 cell_map);
    PM_LAUNCH_CHECK("k_build_cell_map");
  }
  if (offsets) {
    k_offsets<<<1, pm::kMaxSlots, 0, s>>>(o, st.k, offsets);
    PM_LAUNCH_CHECK("k_offsets");
  }
  return PM_OK;
}

extern "C" int pm_extrude_coordinates(const double *base_coords,
                                      int64_t n_vertices, int32_t layers,
                                      double layer_height, double *out,
                                      void *stream) {
  pm::clear_error();
  if (layers < 1) {
    pm::set_error("layer count must be >= 1, got %d", layers);
    return PM_EINVAL;
  }
  if (!(layer_height > 0)) {
    pm::set_error("layer height must be > 0, got %g", layer_height);
    return PM_EINVAL;
  }
  if (n_vertices == 0) return PM_OK;
  const int64_t total = n_vertices * 3 * (int64_t)(layers + 1);
  if (reinterpret_cast<uintptr_t>(out) & 15) {
    pm::set_error("coordinate field must be 16-byte aligned");
    return PM_EINVAL;
  }
  if (total < ((int64_t)1 << 31))
    k_extrude<uint32_t><<<pm::grid_for((total + 1) / 2, 256), 256, 0,
                          (cudaStream_t)stream>>>(base_coords, n_vertices,
                                                  layers, layer_height, out);
  else
    k_extrude<int64_t><<<pm::grid_for((total + 1) / 2, 256), 256, 0,
                         (cudaStream_t)stream>>>(base_coords, n_vertices,
                                                 layers, layer_height, out);
  PM_LAUNCH_CHECK("k_extrude");
  return PM_OK;
}

extern "C" int pm_column_probe(int32_t mode, int32_t k, int64_t n_cells,
                               int32_t layers, const int32_t *cell_map,
                               const int32_t *offsets, int64_t *out_i64,
                               double *out_f64, void *stream) {
  pm::clear_error();
  if (k < 1 || k > pm::kMaxSlots || layers < 1 || n_cells < 0) {
    pm::set_error("bad probe shape k=%d layers=%d", k, layers);
    return PM_EINVAL;
  }
  const int64_t total = n_cells * layers * (int64_t)k;
  if (total == 0) return PM_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0) {
    k_probe_lists<<<pm::grid_for(total, 256), 256, 0, s>>>(
        k, n_cells, layers, cell_map, offsets, out_i64);
  } else if (mode == 1) {
    k_probe_count<<<pm::grid_for(total, 256), 256, 0, s>>>(
        k, n_cells, layers, cell_map, offsets, out_f64);
  } else {
    pm::set_error("unknown probe mode %d", mode);
    return PM_EINVAL;
  }
  PM_LAUNCH_CHECK("k_probe");
  return PM_OK;
}

extern "C" int pm_halo_pack(const double *y, const int64_t *cols,
                            int64_t n_cols, int32_t col, double *buf,
                            void *stream) {
  pm::clear_error();
  if (n_cols < 0 || col < 1) {
    pm::set_error("bad halo shape");
    return PM_EINVAL;
  }
  const int64_t total = n_cols * col;
  if (!total) return PM_OK;
  k_halo_pack<<<pm::grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
      y, cols, n_cols, col, buf);
  PM_LAUNCH_CHECK("k_halo_pack");
  return PM_OK;
}

extern "C" int pm_halo_unpack_add(double *y, const int64_t *cols,
                                  int64_t n_cols, int32_t col,
                                  const double *buf, void *stream) {
  pm::clear_error();
  if (n_cols < 0 || col < 1) {
    pm::set_error("bad halo shape");
    return PM_EINVAL;
  }
  const int64_t total = n_cols * col;
  if (!total) return PM_OK;
  k_halo_unpack_add<<<pm::grid_for(total, 256), 256, 0,
                      (cudaStream_t)stream>>>(y, cols, n_cols, col, buf);
  PM_LAUNCH_CHECK("k_halo_unpack_add");
  return PM_OK;
}
