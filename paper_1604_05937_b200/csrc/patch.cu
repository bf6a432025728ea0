// Patch-owner schedule for CG column loops (PM_VARIANT_PATCH).
//
// Plan (paper_1604_05937_b200/schedule.py): compact Morton patches of base
// cells; every vertex / edge is owned by the lowest patch touching it;
// patch p visits all cells incident to its owned entities (halo included),
// grouped by the global greedy colouring.
//
// One CTA per patch (persistent).  Per W-layer chunk:
//   phase A  (one colour at a time): W-lane segments run the column kernel
//            body of column_warp.cu on each visited cell -- gathers along
//            the column, |det J| from the coordinate field, Mref, vertical
//            combine in registers -- and add the per-level results into a
//            shared-memory accumulator Acc[entity][channel][level].  Cells
//            of one colour share no entity, so the adds are plain
//            read-modify-writes (no atomics); lanes hit consecutive levels.
//   phase B  owned entity columns are written once, coalesced, with plain
//            stores; the chunk's top level is carried to the next chunk.
// Every DoF is produced by one CTA in a fixed order: bitwise deterministic,
// no zeroing pass, no fp64 atomics.
#include "column_layout.cuh"

namespace pm {

struct PatchDev {
  const int32_t *cell_ptr, *cells, *color_ptr, *ent_ptr, *owned, *ents;
  const uint16_t *lents;
  int32_t n_colors, n0;
  int32_t max_local, max_owned;
  int64_t start0, column0, start1, column1; // Alg. 1 closed form
};

template <class LY, int W, int K = LY::K>
__global__ void __launch_bounds__(256)
k_patch(const KronMat M, const PatchDev P, int64_t n_patches, int layers,
        const int32_t *__restrict__ cmap, const int32_t *__restrict__ xmap,
        const double *__restrict__ coords, const double *__restrict__ x,
        double *__restrict__ y) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int SEGS = 32 / W;
  constexpr typename LY::Tab T = LY::make();
  constexpr int CH = LY::CH0 > LY::CH1 ? LY::CH0 : LY::CH1;
  constexpr int E = LY::has_edges ? 6 : 3;
  constexpr int STRIDE = W + 1; // levels l0 .. l0+W
  extern __shared__ double sm[];
  double *acc = sm;
  double *carry = sm + (size_t)P.max_local * CH * STRIDE;

  const int lane = threadIdx.x & 31;
  const int sl = lane % W, seg = lane / W;
  const int warp = threadIdx.x >> 5;
  const int n_warps = blockDim.x >> 5;
  const int nc = P.n_colors;

  for (int64_t p = blockIdx.x; p < n_patches; p += gridDim.x) {
    const int eb = __ldg(P.ent_ptr + p);
    const int n_loc = __ldg(P.ent_ptr + p + 1) - eb;
    const int n_own = __ldg(P.owned + p);
    const int n_acc = n_loc * CH * STRIDE;
    for (int i = threadIdx.x; i < n_acc; i += blockDim.x) acc[i] = 0.0;
    for (int i = threadIdx.x; i < n_own * CH; i += blockDim.x) carry[i] = 0.0;
    __syncthreads();

    for (int l0 = 0; l0 < layers; l0 += W) {
      const int nl = min(W, layers - l0);
      const int last = nl - 1;
      const int l = l0 + sl;
      // ---------------- phase A: colours one after the other
      for (int col = 0; col < nc; ++col) {
        const int lo = __ldg(P.color_ptr + p * (nc + 1) + col);
        const int hi = __ldg(P.color_ptr + p * (nc + 1) + col + 1);
        for (int ib = lo + warp * SEGS; ib < hi; ib += n_warps * SEGS) {
          const int ci = ib + seg;
          const bool ok = ci < hi;
          const int64_t c = ok ? __ldg(P.cells + ci) : 0;
          int32_t L[K];
#pragma unroll
          for (int j = 0; j < K; ++j) L[j] = ok ? __ldg(cmap + c * K + j) : 0;
          int32_t LX[3];
#pragma unroll
          for (int a = 0; a < 3; ++a)
            LX[a] = ok ? __ldg(xmap + c * 18 + 6 * a) : 0;
          int lent[E];
#pragma unroll
          for (int q = 0; q < E; ++q)
            lent[q] = ok ? (int)__ldg(P.lents + (size_t)ci * E + q) : 0;
          const bool act = ok && sl < nl;
          const bool own_top = act && sl == last;

          double xv[K];
#pragma unroll
          for (int j = 0; j < K; ++j)
            xv[j] = (act && T.level[j] != 2)
                        ? __ldg(x + L[j] + l * T.offset[j])
                        : 0.0;
#pragma unroll
          for (int j = 0; j < K; ++j)
            if (T.level[j] == 2) {
              const double up = __shfl_down_sync(FULL, xv[T.pair[j]], 1, W);
              xv[j] = own_top ? __ldg(x + L[j] + l * T.offset[j]) : up;
            }
          double Pc[18];
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              const double bot =
                  act ? __ldg(coords + LX[a] + q + 3 * l) : 0.0;
              const double up = __shfl_down_sync(FULL, bot, 1, W);
              Pc[6 * a + q] = bot;
              Pc[6 * a + 3 + q] =
                  own_top ? __ldg(coords + LX[a] + 3 + q + 3 * l) : up;
            }
          double X[6], Y[6], Z[6];
#pragma unroll
          for (int v = 0; v < 6; ++v) {
            X[v] = Pc[3 * v];
            Y[v] = Pc[3 * v + 1];
            Z[v] = Pc[3 * v + 2];
          }
          const double det = act ? prism_abs_detj(X, Y, Z) : 0.0;
          double yv[K];
          kron_apply<LY>(M, xv, det, yv);
          // vertical combine inside the chunk; the chunk's top level goes
          // to accumulator level `nl` (carried by phase B)
#pragma unroll
          for (int j = 0; j < K; ++j)
            if (T.level[j] == 2) {
              const double below = __shfl_up_sync(FULL, yv[j], 1, W);
              if (sl > 0) yv[T.pair[j]] += below;
            }
          if (act) {
#pragma unroll
            for (int j = 0; j < K; ++j) {
              if (T.level[j] == 2) {
                if (sl == last)
                  acc[(lent[T.pos[j]] * CH + T.ch[j]) * STRIDE + nl] += yv[j];
              } else {
                acc[(lent[T.pos[j]] * CH + T.ch[j]) * STRIDE + sl] += yv[j];
              }
            }
          }
        }
        __syncthreads();
      }
      // ---------------- phase B: owned entity columns, written once
      const int n_streams = n_own * CH;
      for (int sb = warp * SEGS; sb < n_streams; sb += n_warps * SEGS) {
        const int s = sb + seg;
        if (s >= n_streams) continue;
        const int i = s / CH, ch = s - i * CH;
        const int code = __ldg(P.ents + eb + i);
        const bool edge = code >= P.n0;
        const int ch_d = edge ? LY::CH1 : LY::CH0;
        if (ch >= ch_d) continue;
        const int lv_d = edge ? LY::LV1 : LY::LV0;
        const int64_t origin =
            edge ? P.start1 + P.column1 * (int64_t)(code - P.n0)
                 : P.start0 + P.column0 * (int64_t)code;
        const double *a = acc + (size_t)(i * CH + ch) * STRIDE;
        if (ch < lv_d) { // level copy: levels l0 .. l0+nl-1 (+ carry)
          double v = sl < nl ? a[sl] : 0.0;
          if (sl == 0) {
            v += carry[s];
            const double top = a[nl];
            carry[s] = top;
            if (l0 + nl == layers)
              y[origin + (int64_t)layers * ch_d + ch] = top;
          }
          if (sl < nl) y[origin + (int64_t)(l0 + sl) * ch_d + ch] = v;
        } else if (sl < nl) { // connecting entity: one value per layer
          y[origin + (int64_t)(l0 + sl) * ch_d + ch] = a[sl];
        }
      }
      __syncthreads();
      for (int i = threadIdx.x; i < n_acc; i += blockDim.x) acc[i] = 0.0;
      __syncthreads();
    }
  }
}

template <class LY>
static int patch_k(const LoopArgs &a, const PatchDev &P, int64_t n_patches,
                   int W) {
  constexpr int CH = LY::CH0 > LY::CH1 ? LY::CH0 : LY::CH1;
  if (!a.mtri || !a.mline) {
    set_error("the patch kernel needs the Kronecker factors mtri/mline");
    return PM_EINVAL;
  }
  KronMat M;
  for (int i = 0; i < LY::NH * LY::NH; ++i) M.t[i] = a.mtri[i];
  for (int i = 0; i < LY::NV * LY::NV; ++i) M.l[i] = a.mline[i];
  const size_t smem =
      sizeof(double) * ((size_t)P.max_local * CH * (W + 1) +
                        (size_t)P.max_owned * CH);
  if (smem > 227 * 1024) {
    set_error("patch plan needs %zu bytes of shared memory", smem);
    return PM_EINVAL;
  }
#define PM_PATCH(WW)                                                         \
  do {                                                                       \
    auto kern = k_patch<LY, WW>;                                             \
    PM_CUDA_TRY(cudaFuncSetAttribute(                                        \
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));      \
    int per_sm = 0;                                                          \
    PM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, \
                                                              256, smem));   \
    if (per_sm < 1) per_sm = 1;                                              \
    int64_t grid = (int64_t)sm_count() * per_sm;                             \
    if (grid > n_patches) grid = n_patches;                                  \
    kern<<<(unsigned)grid, 256, smem, a.s>>>(M, P, n_patches, a.layers,      \
                                             a.cmap, a.xmap, a.coords, a.x,  \
                                             a.y);                           \
  } while (0)
  if (W == 32)
    PM_PATCH(32);
  else if (W == 16)
    PM_PATCH(16);
  else if (W == 8)
    PM_PATCH(8);
  else {
    set_error("patch chunk width must be 8, 16 or 32 (got %d)", W);
    return PM_EINVAL;
  }
#undef PM_PATCH
  PM_LAUNCH_CHECK("k_patch");
  return PM_OK;
}

// Only layouts whose DoFs all live on vertex / edge columns (P1, P2,
// 3-vector P1, CG1 x DGk).
#define PM_PATCH_LAYOUTS(X)                                                  \
  X(1, 0, 0, 0, 0, 0)                                                        \
  X(0, 1, 0, 0, 0, 0)                                                        \
  X(0, 2, 0, 0, 0, 0)                                                        \
  X(1, 1, 1, 1, 0, 0)                                                        \
  X(3, 0, 0, 0, 0, 0)

int launch_patch(const LoopArgs &a, const int32_t *delta6,
                 const PatchDev &P, int64_t n_patches, int W) {
#define PM_DISPATCH(a_, b_, c_, e_, f_, g_)                                  \
  if (Layout<a_, b_, c_, e_, f_, g_>::matches(delta6))                       \
    return patch_k<Layout<a_, b_, c_, e_, f_, g_>>(a, P, n_patches, W);
  PM_PATCH_LAYOUTS(PM_DISPATCH)
#undef PM_DISPATCH
  set_error("layout not supported by the patch schedule");
  return PM_EINVAL;
}

} // namespace pm

extern "C" int pm_column_mass_patch(
    const int32_t *delta6, int32_t k, int64_t n_vertices, int64_t n_edges,
    int32_t layers, const int32_t *cell_map, const int32_t *coord_map,
    const double *coords, const double *mref, const double *mtri,
    const double *mline, const double *x, double *y, int64_t n_patches, int32_t n_colors, int32_t chunk, int32_t max_local,
    int32_t max_owned, const int32_t *cell_ptr, const int32_t *cells,
    const int32_t *color_ptr, const int32_t *ent_ptr, const int32_t *owned,
    const int32_t *ents, const uint16_t *lents, void *stream) {
  pm::clear_error();
  pm::LoopArgs a;
  int rc = pm::make_slot_table(delta6, &a.st);
  if (rc) return rc;
  if (k != a.st.k || layers < 1 || n_patches < 0 || n_colors < 1 ||
      max_local < 0 || max_owned < 0 || !mref) {
    pm::set_error("bad arguments to pm_column_mass_patch");
    return PM_EINVAL;
  }
  if (n_patches == 0) return PM_OK;
  if (!cell_map || !coord_map || !coords || !x || !y || !cell_ptr ||
      !cells || !color_ptr || !ent_ptr || !owned || !ents || !lents) {
    pm::set_error("NULL device pointer");
    return PM_EINVAL;
  }
  a.k = k;
  a.layers = layers;
  a.cmap = cell_map;
  a.xmap = coord_map;
  a.coords = coords;
  a.mref = mref;
  a.mtri = mtri;
  a.mline = mline;
  a.x = x;
  a.y = y;
  a.s = (cudaStream_t)stream;
  pm::PatchDev P;
  P.cell_ptr = cell_ptr;
  P.cells = cells;
  P.color_ptr = color_ptr;
  P.ent_ptr = ent_ptr;
  P.owned = owned;
  P.ents = ents;
  P.lents = lents;
  P.n_colors = n_colors;
  P.n0 = (int32_t)n_vertices;
  P.max_local = max_local;
  P.max_owned = max_owned;
  P.column0 = (int64_t)layers * (delta6[0] + delta6[1]) + delta6[0];
  P.column1 = (int64_t)layers * (delta6[2] + delta6[3]) + delta6[2];
  P.start0 = 0;
  P.start1 = P.column0 * n_vertices;
  (void)n_edges;
  return pm::launch_patch(a, delta6, P, n_patches, chunk);
}
