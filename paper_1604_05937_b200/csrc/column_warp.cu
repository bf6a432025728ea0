// Warp-per-column schedule: the paper's Algorithm 3 mapped onto a warp.
//
// A segment of W lanes (W = 8, 16 or 32) owns one base-cell column; lane
// `sl` handles layer l0+sl of the current W-layer chunk, so every slot's
// DoFs  L_j + l*offset_j  are consecutive across the segment (coalesced
// gathers along the column).  The bottom-layer lists L (field and
// coordinates) are loaded once per column.  Vertical sharing is carried in
// registers: a top-copy value is the next lane's bottom-copy value
// (shfl.down), a top-copy contribution is added to the next lane's bottom
// contribution (shfl.up) and across chunks through a per-segment carry, so
// each vertically shared DoF is written exactly once per column.  DoFs
// shared between columns (vertex / edge DoFs of CG spaces) are combined
// with fp64 REDG atomics, or -- in the coloured schedule, where no two
// columns of a launch share a DoF -- with plain read-add-stores.
#include "column_layout.cuh"

#include <stdlib.h>

namespace pm {

template <int K> struct ColumnArgs {
  KronMat M;
};

enum { kStorePlain = 0, kStoreAtomic = 1, kStoreRmw = 2 };

__device__ __forceinline__ void put(double *p, double v, int how) {
  if (how == kStoreAtomic)
    atomicAdd(p, v);
  else if (how == kStoreRmw)
    *p += v;
  else
    *p = v;
}

template <class LY, int W, bool COLORED, int K = LY::K>
__global__ void __launch_bounds__(256)
k_column(const ColumnArgs<K> A, int64_t n_cells, int layers,
         const int32_t *__restrict__ cells, const int32_t *__restrict__ cmap,
         const int32_t *__restrict__ coff, const int32_t *__restrict__ xmap,
         const int32_t *__restrict__ xoff, const double *__restrict__ coords,
         const double *__restrict__ x, double *__restrict__ y,
         int accumulate) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int SEGS = 32 / W;
  constexpr typename LY::Tab T = LY::make(); // folded at compile time
  const int lane = threadIdx.x & 31;
  const int sl = lane % W; // layer inside the chunk
  const int seg = lane / W;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  // Per-slot vertical offsets (Algorithm 2) are constants of the layout:
  // folded at compile time here; the device-built offsets array (K0) is
  // bit-checked against the same closed form by the tests.  The coordinate
  // space (COORDS_LAYOUT) has offset 3 on every slot.
  (void)coff;
  (void)xoff;

  // How each slot's contribution reaches y.
  int how[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (T.hshare[j])
      how[j] = COLORED ? kStoreRmw : kStoreAtomic;
    else
      how[j] = (accumulate || COLORED) ? kStoreRmw : kStorePlain;
  }

  for (int64_t cb = warp * SEGS; cb < n_cells; cb += n_warps * SEGS) {
    const int64_t ci = cb + seg;
    const bool cell_ok = ci < n_cells;
    const int64_t c = cell_ok ? (cells ? (int64_t)__ldg(cells + ci) : ci) : 0;
    // bottom-layer lists, loaded once per column
    // DoF numbers fit int32 (checked by the host), so all address
    // arithmetic along the column stays 32-bit.
    int32_t L[K];
#pragma unroll
    for (int j = 0; j < K; ++j) L[j] = cell_ok ? __ldg(cmap + c * K + j) : 0;
    // coordinate map: slot 6a+3b+q of vertex a sits `3b+q` after slot 6a
    int32_t LX[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
      LX[a] = cell_ok ? __ldg(xmap + c * 18 + 6 * a) : 0;

    double carry[K]; // top contribution of the chunk's last layer
#pragma unroll
    for (int j = 0; j < K; ++j) carry[j] = 0.0;

    for (int l0 = 0; l0 < layers; l0 += W) {
      const int nl = min(W, layers - l0);
      const int last = nl - 1;
      const int l = l0 + sl;
      const bool act = cell_ok && sl < nl;
      const bool own_top = act && sl == last; // loads its own top values

      // ---- gather the field: bottom / connecting slots directly, top
      //      copies from the next lane (or directly on the last lane)
      double xv[K];
#pragma unroll
      for (int j = 0; j < K; ++j)
        xv[j] = (act && T.level[j] != 2)
                    ? __ldg(x + L[j] + l * T.offset[j])
                    : 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (T.level[j] == 2) {
          const double up = __shfl_down_sync(FULL, xv[T.pair[j]], 1, W);
          xv[j] = own_top ? __ldg(x + L[j] + l * T.offset[j]) : up;
        }
      }
      // ---- geometry: the six prism vertices (bottom comps direct, top
      //      comps from the next lane)
      double P[18]; // slot 6a + 3b + comp
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int sb = 6 * a + q, st = 6 * a + 3 + q;
          const double bot = act ? __ldg(coords + LX[a] + q + 3 * l) : 0.0;
          const double up = __shfl_down_sync(FULL, bot, 1, W);
          P[sb] = bot;
          P[st] = own_top ? __ldg(coords + LX[a] + 3 + q + 3 * l) : up;
        }
      double X[6], Y[6], Z[6];
#pragma unroll
      for (int v = 0; v < 6; ++v) {
        X[v] = P[3 * v];
        Y[v] = P[3 * v + 1];
        Z[v] = P[3 * v + 2];
      }
      const double det = act ? prism_abs_detj(X, Y, Z) : 0.0;

      // ---- element kernel
      double yv[K];
      kron_apply<LY>(A.M, xv, det, yv);

      // ---- vertical combine: top(l-1) joins bottom(l)
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (T.level[j] == 2) {
          const int b = T.pair[j];
          const double below = __shfl_up_sync(FULL, yv[j], 1, W);
          yv[b] += (sl == 0) ? carry[j] : below;
          carry[j] = __shfl_sync(FULL, yv[j], last, W);
        }
      }
      // ---- scatter: every bottom / connecting DoF of the chunk once
      if (act) {
#pragma unroll
        for (int j = 0; j < K; ++j)
          if (T.level[j] != 2)
            put(y + L[j] + l * T.offset[j], yv[j], how[j]);
      }
    }
    // the column's top level (layers-1's top copies)
    const int nl_last = layers - ((layers - 1) / W) * W;
    if (cell_ok && sl == nl_last - 1) {
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (T.level[j] == 2)
          put(y + L[j] + (layers - 1) * T.offset[j], carry[j], how[j]);
    }
  }
}

template <class LY>
static int column_k(const LoopArgs &a, bool colored) {
  constexpr int K = LY::K;
  ColumnArgs<K> A;
  if (!a.mtri || !a.mline) {
    set_error("the column kernel needs the Kronecker factors mtri/mline");
    return PM_EINVAL;
  }
  for (int i = 0; i < LY::NH * LY::NH; ++i) A.M.t[i] = a.mtri[i];
  for (int i = 0; i < LY::NV * LY::NV; ++i) A.M.l[i] = a.mline[i];
  // segment width: smallest lane waste for this layer count
  // (PM_COLUMN_W=8|16|32 overrides, a tuning knob)
  int W = 32;
  static int forced = -1;
  if (forced < 0) {
    const char *e = getenv("PM_COLUMN_W");
    forced = e ? atoi(e) : 0;
  }
  if (forced == 8 || forced == 16 || forced == 32) {
    W = forced;
  } else {
    double best = 1e30;
    for (int w : {32, 16, 8}) {
      const int chunks = (a.layers + w - 1) / w;
      // measured (profiles/r01): small segments win -- more cells per warp
      const double waste = (double)(chunks * w) / a.layers + 0.005 * chunks;
      if (waste < best - 1e-9) {
        best = waste;
        W = w;
      }
    }
  }
  const int segs = 32 / W;
  const int64_t warps = (a.n_cells + segs - 1) / segs;
  const unsigned grid = grid_for(warps * 32, 256, 8);
#define PM_COL(WW)                                                           \
  do {                                                                       \
    if (colored)                                                             \
      k_column<LY, WW, true><<<grid, 256, 0, a.s>>>(                         \
          A, a.n_cells, a.layers, a.cells, a.cmap, a.coff, a.xmap, a.xoff,   \
          a.coords, a.x, a.y, a.accumulate);                                 \
    else                                                                     \
      k_column<LY, WW, false><<<grid, 256, 0, a.s>>>(                        \
          A, a.n_cells, a.layers, a.cells, a.cmap, a.coff, a.xmap, a.xoff,   \
          a.coords, a.x, a.y, a.accumulate);                                 \
  } while (0)
  if (W == 32)
    PM_COL(32);
  else if (W == 16)
    PM_COL(16);
  else
    PM_COL(8);
#undef PM_COL
  PM_LAUNCH_CHECK("k_column");
  return PM_OK;
}

bool column_supports(const int32_t *d) {
#define PM_MATCH(a, b, c, e, f, g)                                           \
  if (Layout<a, b, c, e, f, g>::matches(d)) return true;
  PM_LAYOUTS(PM_MATCH)
#undef PM_MATCH
  return false;
}

int launch_column(const LoopArgs &a, const int32_t *delta6, bool colored) {
#define PM_DISPATCH(a_, b_, c_, e_, f_, g_)                                  \
  if (Layout<a_, b_, c_, e_, f_, g_>::matches(delta6))                       \
    return column_k<Layout<a_, b_, c_, e_, f_, g_>>(a, colored);
  PM_LAYOUTS(PM_DISPATCH)
#undef PM_DISPATCH
  set_error("layout not built into the column kernel");
  return PM_EINVAL;
}

} // namespace pm
