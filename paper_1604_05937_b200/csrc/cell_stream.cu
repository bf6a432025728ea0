// Column loop for the vertical-only cell layouts (DoFs on the prism cells'
// level copies only: DG0 x CG1, DG1 x CG1 — delta(2,0) = D0 > 0, nothing
// else).  Algorithm 1 numbers cell c's column as (layers+1)*D0 consecutive
// values, level l at c*(layers+1)*D0 + l*D0, so consecutive cell-layers
// (cell-major) address one contiguous range and a level is shared only by
// the two cell-layers of its own column below and above it.
//
// Work unit = T consecutive cell-layers, one per thread; units overlap by
// one cell-layer, so every level shared by two cell-layers has both inside
// one unit.  The unit's level range arrives by one cp.async.bulk (TMA) of
// its 16-byte aligned superset into an S-stage ring (the per-unit size
// varies: column tops add a level each); coordinates are gathered through
// the coordinate map and prefetched one unit ahead (as in the DG stream
// kernel).  Each cell-layer's bottom / top contributions go to two shared
// arrays, and the unit's owned levels (bottom level of every cell-layer but
// the overlap one, plus column tops) are written once with coalesced plain
// stores: no atomics, no zeroing, deterministic.
#include "column_loop.cuh"
#include "pm_ptx.cuh"

#include <stdlib.h>

namespace pm {

template <int D0, int S, int T = 256>
__global__ void __launch_bounds__(T, 2)
k_cell_stream(const MassMat<2 * D0> M, int64_t n_units, int64_t n_cl,
              int layers, int stage_doubles, int ybuf_doubles,
              const int32_t *__restrict__ xmap,
              const double *__restrict__ coords,
              const double *__restrict__ x, double *__restrict__ y) {
  constexpr int K = 2 * D0;
  extern __shared__ __align__(128) unsigned char smem[];
  double *ring = reinterpret_cast<double *>(smem);
  double *ybuf = ring + (size_t)S * stage_doubles;        // 2 x (Yb, Yt)
  uint64_t *bar = reinterpret_cast<uint64_t *>(ybuf + 4 * ybuf_doubles);
  // per stage: the unit's first level and alignment shift (thread 0 writes
  // them when it issues the stage's copy; read after the next barrier)
  int64_t *st_L0 = reinterpret_cast<int64_t *>(bar + S);
  int *st_sh = reinterpret_cast<int *>(st_L0 + S);
  const int t = threadIdx.x, lane = t & 31;
  const uint32_t lp1 = (uint32_t)layers + 1;

  if (t == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int64_t n_mine =
      first < n_units ? (n_units - first + stride - 1) / stride : 0;
  // all indices fit 32 bits (the launcher checks n_cl < 2^31); 32-bit
  // divisions are a handful of instructions, 64-bit ones ~100
  const uint32_t lay = (uint32_t)layers, ncl = (uint32_t)n_cl;
  auto g0_of = [&](int64_t u) { return (uint32_t)u * (uint32_t)(T - 1); };
  auto level_of = [&](uint32_t g) -> int64_t { // global level of g's bottom
    const uint32_t c = g / lay;
    return (int64_t)c * lp1 + (g - c * lay);
  };
  // unit u: levels [L0, L1] -> aligned byte range of x, element shift
  struct Range {
    int64_t a0; // first double of the aligned copy
    uint32_t bytes;
    int sh;     // L0*D0 - a0
    int64_t L0;
  };
  auto range_of = [&](int64_t u) {
    const uint32_t g0 = g0_of(u);
    const uint32_t g1 = (g0 + T < ncl ? g0 + T : ncl) - 1;
    const int64_t L0 = level_of(g0), L1 = level_of(g1) + 1;
    const int64_t e0 = L0 * D0, e1 = (L1 + 1) * D0; // [e0, e1) doubles
    const int64_t a0 = e0 & ~(int64_t)1;
    const int64_t a1 = (e1 + 1) & ~(int64_t)1;
    return Range{a0, (uint32_t)((a1 - a0) * 8), (int)(e0 - a0), L0};
  };
  auto issue = [&](int64_t i) {
    const int s = (int)(i % S);
    const Range r = range_of(first + i * stride);
    st_L0[s] = r.L0;
    st_sh[s] = r.sh;
    mbar_arrive_expect_tx(&bar[s], r.bytes);
    bulk_g2s(ring + (size_t)s * stage_doubles, x + r.a0, r.bytes, &bar[s]);
  };
  if (t == 0)
    for (int64_t i = 0; i < S - 1 && i < n_mine; ++i) issue(i);
  __syncthreads(); // stage ranges visible

  // coordinates: map row and bottom (x,y,z) of the three vertices one unit
  // ahead; the top level from the next lane, or prefetched when the next
  // lane is another column / another warp
  struct Where {
    uint32_t g;
    uint32_t c;
    int l;
    bool ok;
  };
  auto where = [&](int64_t u) {
    const uint32_t g = g0_of(u) + t;
    const bool ok = g < ncl;
    const uint32_t gg = ok ? g : ncl - 1;
    const uint32_t c = gg / lay;
    return Where{gg, c, (int)(gg - c * lay), ok};
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
  // map rows two units ahead, coordinates one unit ahead: neither the
  // map -> coordinate dependency nor the gather latency is exposed
  Where w0{0, 0, 0, false}, w1{0, 0, 0, false}, w2{0, 0, 0, false};
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

  for (int64_t i = 0; i < n_mine; ++i) {
    const int s = (int)(i % S);
    const int64_t u = first + i * stride;
    if (i + 1 < n_mine) {
      load_xyz(w1, lx1, nb);
      own1 = load_top(w1, lx1, nt);
    }
    if (i + 2 < n_mine) {
      w2 = where(u + 2 * stride);
      load_map(w2, lx2);
    }
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

    const int64_t rL0 = st_L0[s];
    const int rsh = st_sh[s];
    mbar_wait(&bar[s], (uint32_t)((i / S) & 1));
    const double *xs = ring + (size_t)s * stage_doubles + rsh;
    double *Yb = ybuf + (size_t)(i & 1) * 2 * ybuf_doubles, *Yt = Yb + ybuf_doubles;
    const int64_t Lg = (int64_t)w0.c * lp1 + w0.l; // level of g's bottom
    const int ll = (int)(Lg - rL0); // local level of the bottom
    if (w0.ok) {
      double xv[K], yv[K];
#pragma unroll
      for (int j = 0; j < K; ++j) xv[j] = xs[ll * D0 + j]; // bottom, top
#pragma unroll
      for (int j = 0; j < K; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < K; ++q) acc = fma(M.m[j * K + q], xv[q], acc);
        yv[j] = det * acc;
      }
#pragma unroll
      for (int j = 0; j < D0; ++j) {
        Yb[ll * D0 + j] = yv[j];
        Yt[(ll + 1) * D0 + j] = yv[D0 + j];
        if (w0.l == 0) Yt[ll * D0 + j] = 0.0;                 // column bottom
        if (w0.l == layers - 1) Yb[(ll + 1) * D0 + j] = 0.0;  // column top
      }
    }
    __syncthreads(); // stage s read, Yb / Yt complete
    if (t == 0 && i + S - 1 < n_mine) issue(i + S - 1);
    // owned levels: every bottom but the overlap cell-layer's, column tops
    if (w0.ok && (t > 0 || u == 0)) {
      double *yo = y + Lg * D0;
#pragma unroll
      for (int j = 0; j < D0; ++j)
        yo[j] = Yb[ll * D0 + j] + Yt[ll * D0 + j];
      if (w0.l == layers - 1)
#pragma unroll
        for (int j = 0; j < D0; ++j) yo[D0 + j] = Yt[(ll + 1) * D0 + j];
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) cb[q] = nb[q], ct[q] = nt[q];
    own0 = own1;
    w0 = w1;
    w1 = w2;
#pragma unroll
    for (int a = 0; a < 3; ++a) lx0[a] = lx1[a], lx1[a] = lx2[a];
  }
}

template <int D0>
static int cell_stream_launch(const LoopArgs &a) {
  constexpr int T = 256, S = 6, K = 2 * D0;
  const int64_t n_cl = a.n_cells * (int64_t)a.layers;
  const int64_t n_units = n_cl <= 1 ? 1 : (n_cl - 1 + T - 2) / (T - 1);
  // levels per unit: T cell-layers + one top per column started + 1
  const int lv = T + (T - 1) / a.layers + 2;
  const int stage = ((lv * D0 + 2) + 1) & ~1; // + alignment shift, even
  const int ybufd = lv * D0;
  const size_t smem = sizeof(double) * ((size_t)S * stage + 4 * ybufd) +
                      S * (2 * sizeof(uint64_t) + sizeof(int));
  MassMat<K> M;
  for (int i = 0; i < K * K; ++i) M.m[i] = a.mref[i];
  auto kern = k_cell_stream<D0, S, T>;
  PM_CUDA_TRY(cudaFuncSetAttribute(
      kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  PM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T,
                                                            smem));
  if (per_sm < 1) {
    set_error("cell stream kernel does not fit an SM (%zu B smem)", smem);
    return PM_EINVAL;
  }
  int64_t grid = (int64_t)sm_count() * per_sm;
  if (grid > n_units) grid = n_units;
  kern<<<(unsigned)grid, T, smem, a.s>>>(M, n_units, n_cl, a.layers, stage,
                                         ybufd, a.xmap, a.coords, a.x, a.y);
  PM_LAUNCH_CHECK("k_cell_stream");
  return PM_OK;
}

// Vertical-only cell layouts, all cells, overwrite mode (AUTO).  x must be
// 16-byte aligned and readable up to the next 16-byte boundary past its
// end (the last unit copies an aligned superset).
int launch_cell_stream(const LoopArgs &a, const int32_t *delta6,
                       bool *handled) {
  *handled = false;
  const char *env = getenv("PM_CELL_STREAM"); // 0: the column kernel
  if (env && atoi(env) == 0) return PM_OK;
  const bool vert_cells = !delta6[0] && !delta6[1] && !delta6[2] &&
                          !delta6[3] && delta6[4] > 0 && !delta6[5];
  // short columns: many column ends per unit, the column kernel is faster
  // (measured at lambda = 5: 0.031 vs 0.045 ms; lambda >= 20: 6-15 % slower)
  if (!vert_cells || a.cells || a.accumulate || a.layers < 16 ||
      (reinterpret_cast<uintptr_t>(a.x) & 15) ||
      a.n_cells * (int64_t)a.layers > 0x7FFFFFFFll)
    return PM_OK;
  int rc = PM_OK;
  switch (delta6[4]) {
  case 1: rc = cell_stream_launch<1>(a); break;
  case 3: rc = cell_stream_launch<3>(a); break;
  default: return PM_OK;
  }
  if (!rc) *handled = true;
  return rc;
}

} // namespace pm
