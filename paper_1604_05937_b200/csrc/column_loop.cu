// The column loop (Algorithm 3) driving
// the prism mass / residual kernel:
//
//   for every base cell c:        L = cell_map[c]            (once per column)
//     for l in 0 .. layers-1:     dof_j = L_j + l*offset_j   (direct addressing)
//       y[dof] (+)= |det J_{c,l}| * Mref * x[dof]
//
// |det J_{c,l}| = vol(prism)/vol(reference prism) is evaluated from the six
// prism vertices gathered out of the extruded coordinate field through the
// coordinate space's own map + offsets:
//     xm_a = (x_a,bot + x_a,top)/2, ym_a likewise,
//     A2   = (xm1-xm0)(ym2-ym0) - (xm2-xm0)(ym1-ym0)       (2 * area)
//     H    = ((z0t-z0b) + (z1t-z1b) + (z2t-z2b)) / 3       (mean height)
//     |det J| = |A2 * H|
// Mref is the reference-prism mass matrix pre-integrated on the host with
// the configured quadrature (exact for affine triangles x flat layers).
//
// Schedules implemented here:
//   generic  : one thread per cell-layer, flattened (c, l) index so lanes
//              walk up a column; DoFs private to a cell-layer are stored
//              directly, shared DoFs go through fp64 REDG atomics.
//   dg_column: DG spaces whose column block is contiguous
//              (delta only on (2,1)): one warp streams a cell column
//              through shared memory with 16-byte coalesced loads/stores.
#include "pm_common.cuh"
#include "column_loop.cuh"

namespace pm {

template <int K> struct MassMat {
  double m[K * K];
};

// -------------------------------------------------------------------------
// generic schedule
// -------------------------------------------------------------------------
template <int K, bool ATOMIC>
__global__ void __launch_bounds__(256)
k_mass_generic(const MassMat<K> M, uint32_t n_cl, int layers,
               const int32_t *__restrict__ cells,
               const int32_t *__restrict__ cmap,
               const int32_t *__restrict__ coff,
               const int32_t *__restrict__ xmap,
               const int32_t *__restrict__ xoff,
               const double *__restrict__ coords,
               const double *__restrict__ x, double *__restrict__ y,
               int accumulate) {
  int off[K];
#pragma unroll
  for (int j = 0; j < K; ++j) off[j] = __ldg(coff + j);
  int xo[18];
#pragma unroll
  for (int j = 0; j < 18; ++j) xo[j] = __ldg(xoff + j);

  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < n_cl;
       g += gridDim.x * blockDim.x) {
    const uint32_t ci = g / (uint32_t)layers;
    const int l = (int)(g - ci * (uint32_t)layers);
    const uint32_t c = cells ? (uint32_t)__ldg(cells + ci) : ci;
    const int32_t *xm = xmap + (size_t)c * 18;
    double X[6], Y[6], Z[6];
#pragma unroll
    for (int v = 0; v < 6; ++v) { // v = 2a + b
      const int s = 3 * v;        // coords slot 6a+3b
      X[v] = __ldg(coords + __ldg(xm + s) + l * xo[s]);
      Y[v] = __ldg(coords + __ldg(xm + s + 1) + l * xo[s + 1]);
      Z[v] = __ldg(coords + __ldg(xm + s + 2) + l * xo[s + 2]);
    }
    const double det = prism_abs_detj(X, Y, Z);

    const int32_t *cm = cmap + (size_t)c * K;
    int64_t idx[K];
    double xv[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      idx[j] = (int64_t)__ldg(cm + j) + (int64_t)l * off[j];
      xv[j] = __ldg(x + idx[j]);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) acc = fma(M.m[j * K + i], xv[i], acc);
      const double val = det * acc;
      if (ATOMIC)
        atomicAdd(y + idx[j], val);
      else
        y[idx[j]] = accumulate ? y[idx[j]] + val : val;
    }
  }
}

// -------------------------------------------------------------------------
// dg_column schedule: delta only on (2,1), so cell column c owns the
// contiguous block [map[c][0], map[c][0] + K*layers) and slot j of layer l
// sits at map[c][j] + l*K.  One warp per column: the block is streamed in
// chunks of 32 layers through shared memory with coalesced 16-byte
// accesses, each lane then applies the element kernel to one layer.
// -------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(256)
k_mass_dg_column(const MassMat<K> M, int64_t n_cells, int layers,
                 const int32_t *__restrict__ cmap,
                 const int32_t *__restrict__ xmap,
                 const int32_t *__restrict__ xoff,
                 const double *__restrict__ coords,
                 const double *__restrict__ x, double *__restrict__ y,
                 int accumulate) {
  constexpr int W = 32;
  // per warp: K*32 doubles of x staged (and reused for y)
  __shared__ double sx[8][K * W + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *buf = sx[warp];
  int xo[18];
#pragma unroll
  for (int j = 0; j < 18; ++j) xo[j] = __ldg(xoff + j);

  const int64_t warps_total = (int64_t)gridDim.x * 8;
  for (int64_t c = blockIdx.x * 8 + warp; c < n_cells; c += warps_total) {
    const int32_t *xm = xmap + c * 18;
    const int64_t base = __ldg(cmap + c * K); // slot 0 of layer 0
    for (int l0 = 0; l0 < layers; l0 += W) {
      const int nl = min(W, layers - l0);
      const int n = nl * K;
      const double *src = x + base + (int64_t)l0 * K;
      for (int t = lane; t < n; t += W) buf[t] = __ldg(src + t);
      __syncwarp();
      const int l = l0 + lane;
      double yv[K];
      if (lane < nl) {
        double X[6], Y[6], Z[6];
#pragma unroll
        for (int v = 0; v < 6; ++v) {
          const int s = 3 * v;
          X[v] = __ldg(coords + __ldg(xm + s) + l * xo[s]);
          Y[v] = __ldg(coords + __ldg(xm + s + 1) + l * xo[s + 1]);
          Z[v] = __ldg(coords + __ldg(xm + s + 2) + l * xo[s + 2]);
        }
        const double det = prism_abs_detj(X, Y, Z);
        double xv[K];
#pragma unroll
        for (int i = 0; i < K; ++i) xv[i] = buf[lane * K + i];
#pragma unroll
        for (int j = 0; j < K; ++j) {
          double acc = 0.0;
#pragma unroll
          for (int i = 0; i < K; ++i) acc = fma(M.m[j * K + i], xv[i], acc);
          yv[j] = det * acc;
        }
      }
      __syncwarp();
      if (lane < nl) {
#pragma unroll
        for (int j = 0; j < K; ++j) buf[lane * K + j] = yv[j];
      }
      __syncwarp();
      double *dst = y + base + (int64_t)l0 * K;
      for (int t = lane; t < n; t += W)
        dst[t] = accumulate ? dst[t] + buf[t] : buf[t];
      __syncwarp();
    }
  }
}

template <int K>
static int launch_mass(int share, const int32_t *cells, int64_t n_cells,
                       int layers,
                       const int32_t *cmap, const int32_t *coff,
                       const int32_t *xmap, const int32_t *xoff,
                       const double *coords, const double *mref,
                       const double *x, double *y, int accumulate,
                       int variant, cudaStream_t s) {
  MassMat<K> M;
  for (int i = 0; i < K * K; ++i) M.m[i] = mref[i];
  const int64_t n_cl = n_cells * (int64_t)layers;
  if (n_cl > 0xFFFFFFFFll) {
    set_error("too many cell-layers (%lld) for one launch", (long long)n_cl);
    return PM_EINVAL;
  }
  if (!cells && share == PM_SHARE_NONE &&
      (variant == PM_VARIANT_AUTO || variant == PM_VARIANT_COLUMN)) {
    k_mass_dg_column<K><<<grid_for(n_cells * 32, 256, 8), 256, 0, s>>>(
        M, n_cells, layers, cmap, xmap, xoff, coords, x, y, accumulate);
    PM_LAUNCH_CHECK("k_mass_dg_column");
    return PM_OK;
  }
  // A cell list (one colour of the base-mesh colouring) guarantees that no
  // two cell-layers of the launch share a DoF, so plain stores suffice.
  if (share == PM_SHARE_NONE || cells)
    k_mass_generic<K, false><<<grid_for(n_cl, 256), 256, 0, s>>>(
        M, (uint32_t)n_cl, layers, cells, cmap, coff, xmap, xoff, coords, x,
        y, accumulate);
  else
    k_mass_generic<K, true><<<grid_for(n_cl, 256), 256, 0, s>>>(
        M, (uint32_t)n_cl, layers, cells, cmap, coff, xmap, xoff, coords, x,
        y, accumulate);
  PM_LAUNCH_CHECK("k_mass_generic");
  return PM_OK;
}

} // namespace pm

namespace pm {
static int column_mass_dispatch(int32_t k, int32_t share,
                                const int32_t *cells, int64_t n_cells,
                                int32_t layers, const int32_t *cell_map,
                                const int32_t *offsets,
                                const int32_t *coord_map,
                                const int32_t *coord_offsets,
                                const double *coords, const double *mref,
                                const double *x, double *y, int32_t acc,
                                int32_t variant, cudaStream_t s) {
  switch (k) {
#define PM_K(KK)                                                             \
  case KK:                                                                   \
    return launch_mass<KK>(share, cells, n_cells, layers, cell_map, offsets, \
                           coord_map, coord_offsets, coords, mref, x, y, acc, \
                           variant, s);
    PM_K(1) PM_K(2) PM_K(3) PM_K(6) PM_K(18)
#undef PM_K
  default:
    set_error("unsupported slot count k=%d (built: 1,2,3,6,18)", k);
    return PM_EINVAL;
  }
}
} // namespace pm

extern "C" int pm_column_mass(int32_t k, int32_t share, int64_t n_cells,
                              int32_t layers, const int32_t *cell_map,
                              const int32_t *offsets,
                              const int32_t *coord_map,
                              const int32_t *coord_offsets,
                              const double *coords, const double *mref,
                              const double *x, double *y, int64_t n_dofs,
                              int32_t accumulate, int32_t variant,
                              const void *plan, void *stream) {
  pm::clear_error();
  (void)plan;
  if (layers < 1 || n_cells < 0 || n_dofs < 0) {
    pm::set_error("bad shape: layers=%d n_cells=%lld", layers,
                  (long long)n_cells);
    return PM_EINVAL;
  }
  if (share < PM_SHARE_NONE || share > PM_SHARE_HORIZONTAL) {
    pm::set_error("unknown sharing class %d", share);
    return PM_EINVAL;
  }
  if (!mref) {
    pm::set_error("mref is NULL");
    return PM_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (!accumulate && share != PM_SHARE_NONE && n_dofs > 0)
    PM_CUDA_TRY(cudaMemsetAsync(y, 0, (size_t)n_dofs * sizeof(double), s));
  if (n_cells == 0) return PM_OK;
  if (!cell_map || !offsets || !coord_map || !coord_offsets || !coords ||
      !x || !y) {
    pm::set_error("NULL device pointer");
    return PM_EINVAL;
  }
  return pm::column_mass_dispatch(k, share, nullptr, n_cells, layers,
                                  cell_map, offsets, coord_map, coord_offsets,
                                  coords, mref, x, y, accumulate ? 1 : 0,
                                  variant, s);
}

extern "C" int pm_column_mass_cells(int32_t k, const int32_t *cells,
                                    int64_t n_list, int32_t layers,
                                    const int32_t *cell_map,
                                    const int32_t *offsets,
                                    const int32_t *coord_map,
                                    const int32_t *coord_offsets,
                                    const double *coords, const double *mref,
                                    const double *x, double *y,
                                    void *stream) {
  pm::clear_error();
  if (layers < 1 || n_list < 0 || !mref) {
    pm::set_error("bad arguments to pm_column_mass_cells");
    return PM_EINVAL;
  }
  if (n_list == 0) return PM_OK;
  if (!cells || !cell_map || !offsets || !coord_map || !coord_offsets ||
      !coords || !x || !y) {
    pm::set_error("NULL device pointer");
    return PM_EINVAL;
  }
  return pm::column_mass_dispatch(k, PM_SHARE_HORIZONTAL, cells, n_list,
                                  layers, cell_map, offsets, coord_map,
                                  coord_offsets, coords, mref, x, y, 1,
                                  PM_VARIANT_AUTO, (cudaStream_t)stream);
}
