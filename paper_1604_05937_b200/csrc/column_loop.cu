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
// This file: the C entry point, schedule dispatch and the `generic`
// schedule (one thread per cell-layer on a flattened (c, l) index, fp64
// REDG for shared DoFs).  dg_stream.cu: DG fields streamed with TMA bulk
// copies.  column_warp.cu: warp-per-column, lanes = layers.
#include "column_loop.cuh"

namespace pm {

template <int K, bool ATOMIC>
__global__ void __launch_bounds__(256)
k_mass_generic(const MassMat<K> M, uint32_t cl_begin, uint32_t n_cl,
               int layers, const int32_t *__restrict__ cells,
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

  for (uint32_t g = cl_begin + blockIdx.x * blockDim.x + threadIdx.x;
       g < n_cl; g += gridDim.x * blockDim.x) {
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

template <int K>
static int generic_k(const LoopArgs &a, bool atomic, int64_t cl_begin) {
  MassMat<K> M;
  for (int i = 0; i < K * K; ++i) M.m[i] = a.mref[i];
  const int64_t n_cl = a.n_cells * (int64_t)a.layers;
  if (n_cl > 0xFFFFFFFFll) {
    set_error("too many cell-layers (%lld) for one launch", (long long)n_cl);
    return PM_EINVAL;
  }
  const int64_t todo = n_cl - cl_begin;
  if (todo <= 0) return PM_OK;
  if (atomic)
    k_mass_generic<K, true><<<grid_for(todo, 256), 256, 0, a.s>>>(
        M, (uint32_t)cl_begin, (uint32_t)n_cl, a.layers, a.cells, a.cmap,
        a.coff, a.xmap, a.xoff, a.coords, a.x, a.y, a.accumulate);
  else
    k_mass_generic<K, false><<<grid_for(todo, 256), 256, 0, a.s>>>(
        M, (uint32_t)cl_begin, (uint32_t)n_cl, a.layers, a.cells, a.cmap,
        a.coff, a.xmap, a.xoff, a.coords, a.x, a.y, a.accumulate);
  PM_LAUNCH_CHECK("k_mass_generic");
  return PM_OK;
}

int launch_generic(const LoopArgs &a, bool atomic, int64_t cl_begin) {
  switch (a.k) {
  case 1: return generic_k<1>(a, atomic, cl_begin);
  case 2: return generic_k<2>(a, atomic, cl_begin);
  case 3: return generic_k<3>(a, atomic, cl_begin);
  case 6: return generic_k<6>(a, atomic, cl_begin);
  case 18: return generic_k<18>(a, atomic, cl_begin);
  default:
    set_error("unsupported slot count k=%d (built: 1,2,3,6,18)", a.k);
    return PM_EINVAL;
  }
}

} // namespace pm

extern "C" int pm_column_mass(const int32_t *delta6, int32_t k,
                              int64_t n_cells, int32_t layers,
                              const int32_t *cell_map, const int32_t *offsets,
                              const int32_t *coord_map,
                              const int32_t *coord_offsets,
                              const double *coords, const double *mref,
                              const double *mtri, const double *mline,
                              const double *x, double *y, int64_t n_dofs,
                              int32_t accumulate, int32_t variant,
                              const int32_t *cells, int64_t n_list,
                              void *stream) {
  pm::clear_error();
  pm::LoopArgs a;
  int rc = pm::make_slot_table(delta6, &a.st);
  if (rc) return rc;
  if (k != a.st.k) {
    pm::set_error("slot count mismatch: k=%d, layout has %d", k, a.st.k);
    return PM_EINVAL;
  }
  if (layers < 1 || n_cells < 0 || n_dofs < 0 || n_list < 0) {
    pm::set_error("bad shape: layers=%d n_cells=%lld", layers,
                  (long long)n_cells);
    return PM_EINVAL;
  }
  if (!mref) {
    pm::set_error("mref is NULL");
    return PM_EINVAL;
  }
  a.k = k;
  a.layers = layers;
  a.cells = cells;
  a.n_cells = cells ? n_list : n_cells;
  a.cmap = cell_map;
  a.coff = offsets;
  a.xmap = coord_map;
  a.xoff = coord_offsets;
  a.coords = coords;
  a.mref = mref;
  a.mtri = mtri;
  a.mline = mline;
  a.x = x;
  a.y = y;
  a.accumulate = accumulate ? 1 : 0;
  a.s = (cudaStream_t)stream;
  a.dg_only = delta6[0] == 0 && delta6[1] == 0 && delta6[2] == 0 &&
              delta6[3] == 0 && delta6[4] == 0;
  a.hshared = delta6[0] || delta6[1] || delta6[2] || delta6[3];

  if (variant == PM_VARIANT_COLORED && !cells) {
    pm::set_error("the coloured variant needs a cell list (one colour)");
    return PM_EINVAL;
  }
  // Overwrite mode: DoFs that receive REDG need a zeroed field first.
  const bool needs_zero =
      !a.accumulate && a.hshared &&
      (variant == PM_VARIANT_ATOMIC || variant == PM_VARIANT_COLUMN ||
       variant == PM_VARIANT_AUTO);
  const bool generic_needs_zero =
      !a.accumulate && !a.dg_only &&
      (variant == PM_VARIANT_ATOMIC ||
       (variant == PM_VARIANT_AUTO && !pm::column_supports(delta6)));
  if ((needs_zero || generic_needs_zero) && n_dofs > 0)
    PM_CUDA_TRY(cudaMemsetAsync(y, 0, (size_t)n_dofs * sizeof(double), a.s));
  if (a.n_cells == 0) return PM_OK;
  if (!cell_map || !offsets || !coord_map || !coord_offsets || !coords ||
      !x || !y) {
    pm::set_error("NULL device pointer");
    return PM_EINVAL;
  }
  switch (variant) {
  case PM_VARIANT_AUTO:
    if (a.dg_only && !cells && !a.accumulate) {
      bool handled = false;
      rc = pm::launch_dg_stream(a, &handled);
      if (rc || handled) return rc;
    }
    if (!cells && !a.accumulate) { // vertical-only cell columns
      bool handled = false;
      rc = pm::launch_cell_stream(a, delta6, &handled);
      if (rc || handled) return rc;
    }
    if (pm::column_supports(delta6)) return pm::launch_column(a, delta6, false);
    return pm::launch_generic(a, !a.dg_only, 0);
  case PM_VARIANT_STREAM: {
    bool handled = false;
    if (!a.dg_only || cells || a.accumulate) {
      pm::set_error("stream variant needs a DG (2,1) layout, all cells, "
                    "overwrite mode");
      return PM_EINVAL;
    }
    rc = pm::launch_dg_stream(a, &handled);
    if (!rc && !handled) {
      pm::set_error("stream variant: field not 16-byte aligned");
      return PM_EINVAL;
    }
    return rc;
  }
  case PM_VARIANT_ATOMIC:
    return pm::launch_generic(a, !a.dg_only, 0);
  case PM_VARIANT_COLUMN:
    return pm::launch_column(a, delta6, false);
  case PM_VARIANT_COLORED:
    return pm::launch_column(a, delta6, true);
  default:
    pm::set_error("unknown variant %d", variant);
    return PM_EINVAL;
  }
}
