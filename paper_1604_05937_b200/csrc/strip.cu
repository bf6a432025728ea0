// Strip-patch schedule for vertex-column CG layouts (PM_VARIANT_STRIP):
// P1, 3-vector P1, CG1 x DG0, CG1 x DG1.
//
// Plan (schedule.py + pm_build_strips): compact Morton patches; every vertex
// owned by the lowest patch touching it; patch p visits all cells incident
// to its owned vertices, walked as edge-connected strips.
//
// One CTA per patch (persistent).  Per W-layer chunk:
//   stage   : every local vertex column of the chunk (field levels
//             l0..l0+W and coordinates) is copied once into shared memory
//             with coalesced loads -- the only global reads of the kernel.
//   strips  : a W-lane segment walks a strip, lane = layer.  A 3-vertex
//             window of (field, x, y, z at levels l and l+1) lives in
//             registers; each step loads ONE new vertex (the one opposite
//             the shared edge) from shared memory, applies the sum-factorised
//             element kernel to the cell-layer and accumulates into the
//             window's per-vertex accumulators.  When a vertex leaves the
//             window its partial column (vertically combined through
//             shfl.up) goes to a private Y slot -- no atomics, no colours.
//   gather  : every owned vertex column sums its ~2 Y slots and is written
//             once with coalesced stores; the chunk's top level is carried.
// Deterministic (fixed slot order), no zeroing pass.
#include "column_layout.cuh"

#include <type_traits>

namespace pm {

__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

struct StripDev {
  const int32_t *ent_ptr, *owned, *ents;
  const int32_t *patch_strip_ptr, *strip_step_ptr;
  const uint16_t *step_v;
  const uint8_t *step_slot, *step_flags;
  const int32_t *step_y;
  const int32_t *patch_y_count, *own_base, *own_y_ptr, *own_y;
  int32_t max_local, max_y, max_owned;
  int32_t max_steps, max_strips, max_oy; // per-patch maxima (smem sizing)
  int64_t column0; // Alg. 1 vertex column length
};

// 256 threads per CTA, two CTAs per SM (one stages while the other walks
// its strips)
template <class LY> constexpr int strip_threads() { return 256; }
// the 3-vector window needs ~170 registers: one CTA per SM there
template <class LY> constexpr int strip_min_blocks() {
  return LY::CH0 > 2 ? 1 : 2;
}

template <class LY, int W, int K = LY::K>
__global__ void __launch_bounds__(strip_threads<LY>(), strip_min_blocks<LY>())
k_strip(const KronMat M, const StripDev P, int64_t n_patches, int layers,
        const double *__restrict__ coords, const double *__restrict__ x,
        double *__restrict__ y) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int SEGS = 32 / W;
  constexpr typename LY::Tab T = LY::make();
  constexpr int LV = LY::LV0;        // level-copy DoFs per vertex level
  constexpr int CH = LY::CH0;        // DoFs per vertex layer block
  constexpr int LVA = LV > 0 ? LV : 1; // array extent
  constexpr int FS = W * CH + LV;    // staged field values per vertex
  constexpr int CS = 3 * (W + 1);    // staged coordinates per vertex
  constexpr int YS = W + 1;          // levels per Y slot channel
  extern __shared__ double sm[];
  double *sF = sm;                                   // [max_local][FS]
  double *sC = sF + (size_t)P.max_local * FS;        // [max_local][CS]
  double *sY = sC + (size_t)P.max_local * CS;        // [max_y][CH][YS]
  double *sCarry = sY + (size_t)P.max_y * CH * YS;   // [max_owned][LV]
  // per-patch plan records, staged once per patch
  int2 *sStep = reinterpret_cast<int2 *>(sCarry + (size_t)P.max_owned * LVA);
  int *sSPtr = reinterpret_cast<int *>(sStep + P.max_steps);   // strips+1
  int *sOPtr = sSPtr + P.max_strips + 1;                       // owned+1
  int *sOY = sOPtr + P.max_owned + 1;                          // y entries
  int *sEnt = sOY + P.max_oy;                                  // local ents
  __shared__ int sCounter[1];

  const int lane = threadIdx.x & 31;
  const int sl = lane % W, seg = lane / W;
  const int warp = threadIdx.x >> 5;
  const int n_warps = blockDim.x >> 5;
  const int64_t cstride = 3 * (int64_t)(layers + 1);

  for (int64_t p = blockIdx.x; p < n_patches; p += gridDim.x) {
    const int eb = __ldg(P.ent_ptr + p);
    const int n_loc = __ldg(P.ent_ptr + p + 1) - eb;
    const int n_own = __ldg(P.owned + p);
    const int sb = __ldg(P.patch_strip_ptr + p);
    const int n_strips = __ldg(P.patch_strip_ptr + p + 1) - sb;
    const int obase = __ldg(P.own_base + p);
    for (int i = threadIdx.x; i < n_own * LV; i += blockDim.x) sCarry[i] = 0.0;
    // plan records of this patch -> shared memory (one dependent global
    // round trip per patch instead of one per strip step)
    const int kb = __ldg(P.strip_step_ptr + sb);
    const int n_steps = __ldg(P.strip_step_ptr + sb + n_strips) - kb;
    for (int i = threadIdx.x; i < n_steps; i += blockDim.x) {
      const int kk = kb + i;
      sStep[i] = make_int2((int)__ldg(P.step_v + kk) |
                               ((int)__ldg(P.step_slot + kk) << 16) |
                               ((int)__ldg(P.step_flags + kk) << 24),
                           __ldg(P.step_y + kk));
    }
    for (int i = threadIdx.x; i <= n_strips; i += blockDim.x)
      sSPtr[i] = __ldg(P.strip_step_ptr + sb + i) - kb;
    const int ob = __ldg(P.own_y_ptr + obase);
    for (int i = threadIdx.x; i <= n_own; i += blockDim.x)
      sOPtr[i] = __ldg(P.own_y_ptr + obase + i) - ob;
    const int n_oy = __ldg(P.own_y_ptr + obase + n_own) - ob;
    for (int i = threadIdx.x; i < n_oy; i += blockDim.x)
      sOY[i] = __ldg(P.own_y + ob + i);
    for (int i = threadIdx.x; i < n_loc; i += blockDim.x)
      sEnt[i] = __ldg(P.ents + eb + i);
    __syncthreads();

    for (int l0 = 0; l0 < layers; l0 += W) {
      const int nl = min(W, layers - l0);
      // ---------------- stage: local vertex columns of the chunk
      {
        // warp per vertex column segment (contiguous, coalesced), copied
        // with cp.async so every copy of the chunk is in flight at once
        const int fl = nl * CH + LV, cl = 3 * (nl + 1);
        for (int v = warp; v < n_loc; v += n_warps) {
          const int64_t g = sEnt[v];
          const double *fx = x + g * P.column0 + (int64_t)l0 * CH;
          const double *fc = coords + g * cstride + 3 * (int64_t)l0;
#pragma unroll
          for (int r = 0; r < (FS + 31) / 32; ++r) {
            const int e = lane + 32 * r;
            if (e < fl) cp_async8(sF + v * FS + e, fx + e);
          }
#pragma unroll
          for (int r = 0; r < (CS + 31) / 32; ++r) {
            const int e = lane + 32 * r;
            if (e < cl) cp_async8(sC + v * CS + e, fc + e);
          }
        }
        cp_async_wait_all();
      }
      if (threadIdx.x == 0) sCounter[0] = 0;
      __syncthreads();

      // ---------------- strips: segments grab strips dynamically (the
      // planner orders them longest first), which balances the warps
      const bool lane_ok = sl < nl;
      for (;;) {
        int s0 = 0;
        if (lane == 0) s0 = atomicAdd(sCounter, SEGS);
        s0 = __shfl_sync(FULL, s0, 0);
        if (s0 >= n_strips) break;
        const int si = s0 + seg;
        const bool has = si < n_strips;
        const int k0 = has ? sSPtr[si] : 0;
        const int k1 = has ? sSPtr[si + 1] : 0;
        int len = k1 - k0, maxlen = len;
#pragma unroll
        for (int o = W; o < 32; o <<= 1)
          maxlen = max(maxlen, __shfl_xor_sync(FULL, maxlen, o));
        // window: per slot a, field at l (CH) and l+1 (LV), coords l, l+1
        double fb[3][CH], ft[3][LVA], cb[3][3], ct[3][3];
        double ab[3][CH], at[3][LVA]; // accumulators: bottom/conn, top
        int ysl[3] = {-1, -1, -1};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
#pragma unroll
          for (int c = 0; c < CH; ++c) fb[a][c] = 0.0, ab[a][c] = 0.0;
#pragma unroll
          for (int c = 0; c < LVA; ++c) ft[a][c] = 0.0, at[a][c] = 0.0;
#pragma unroll
          for (int q = 0; q < 3; ++q) cb[a][q] = 0.0, ct[a][q] = 0.0;
        }
        // partial column of window slot A -> its Y slot (lanes = levels;
        // top contributions shifted up one lane).  `doit`: the slot held a
        // residency of this segment's strip.
        auto flush = [&](auto A_, bool doit) {
          constexpr int A = decltype(A_)::value;
          const int ly = doit ? ysl[A] : -1;
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            double v = ab[A][c];
            if (c < LV) { // every lane takes part in the shuffle
              const double below = __shfl_up_sync(FULL, at[A][c], 1, W);
              if (sl > 0) v += below;
            }
            if (ly >= 0) {
              double *row = sY + ((size_t)ly * CH + c) * YS;
              if (lane_ok) row[sl] = v;
              if (c < LV && sl == nl - 1) row[nl] = at[A][c];
            }
          }
          if (doit) { // the residency is closed: clear its accumulators
#pragma unroll
            for (int c = 0; c < CH; ++c) ab[A][c] = 0.0;
#pragma unroll
            for (int c = 0; c < LVA; ++c) at[A][c] = 0.0;
          }
        };
        // one strip step into the compile-time window slot A
        auto step = [&](auto A_, int k) {
          constexpr int A = decltype(A_)::value;
          const bool act = k < len;
          flush(A_, act);
          if (!act) return;
          const int2 rec = sStep[k0 + k];
          const int v = rec.x & 0xffff;
          ysl[A] = rec.y;
          const double *f = sF + v * FS + sl * CH;
          const double *cc = sC + v * CS + 3 * sl;
          // lanes past the chunk read stale (finite or not) staged data:
          // their results never reach an active lane or a store
#pragma unroll
          for (int c = 0; c < CH; ++c) fb[A][c] = f[c];
#pragma unroll
          for (int c = 0; c < LV; ++c) ft[A][c] = f[CH + c];
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            cb[A][q] = cc[q];
            ct[A][q] = cc[3 + q];
          }
          if (k < 2) return; // window not full yet
          // the cell-layer in window order (symmetric element)
          double X[6], Y[6], Z[6];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            X[2 * a] = cb[a][0], Y[2 * a] = cb[a][1], Z[2 * a] = cb[a][2];
            X[2 * a + 1] = ct[a][0], Y[2 * a + 1] = ct[a][1];
            Z[2 * a + 1] = ct[a][2];
          }
          const double det = prism_abs_detj(X, Y, Z);
          double xv[K], yv[K];
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const int a = T.pos[j];
            xv[j] = T.level[j] == 2 ? ft[a][T.ch[j]] : fb[a][T.ch[j]];
          }
          kron_apply<LY>(M, xv, det, yv);
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const int a = T.pos[j];
            if (T.level[j] == 2)
              at[a][T.ch[j]] += yv[j];
            else
              ab[a][T.ch[j]] += yv[j];
          }
        };
        using S0 = std::integral_constant<int, 0>;
        using S1 = std::integral_constant<int, 1>;
        using S2 = std::integral_constant<int, 2>;
        // sequential strips: the replaced slot cycles 0, 1, 2, 0, ...
        for (int k = 0; k < maxlen; k += 3) {
          step(S0{}, k);
          step(S1{}, k + 1);
          step(S2{}, k + 2);
        }
        // strip end: the three remaining residencies
        flush(S0{}, has);
        flush(S1{}, has);
        flush(S2{}, has);
      }
      __syncthreads();

      // ---------------- gather: owned vertex columns written once
      const int n_streams = n_own * CH;
      for (int s0 = warp * SEGS; s0 < n_streams; s0 += n_warps * SEGS) {
        const int s = s0 + seg;
        if (s >= n_streams) continue;
        const int i = s / CH, c = s - i * CH;
        const int y0 = sOPtr[i], y1 = sOPtr[i + 1];
        double v = 0.0, top = 0.0;
        for (int q = y0; q < y1; ++q) {
          const double *row = sY + ((size_t)sOY[q] * CH + c) * YS;
          if (sl < nl) v += row[sl];
          if (c < LV && sl == 0) top += row[nl];
        }
        const int64_t origin = (int64_t)sEnt[i] * P.column0;
        if (c < LV) {
          if (sl == 0) {
            v += sCarry[i * LV + c];
            sCarry[i * LV + c] = top;
            if (l0 + nl == layers)
              y[origin + (int64_t)layers * CH + c] = top;
          }
        }
        if (sl < nl) y[origin + (int64_t)(l0 + sl) * CH + c] = v;
      }
      __syncthreads();
    }
  }
}

template <class LY>
static int strip_k(const LoopArgs &a, const StripDev &P, int64_t n_patches,
                   int W, int threads) {
  constexpr int LV = LY::LV0, CH = LY::CH0;
  if (!a.mtri || !a.mline) {
    set_error("the strip kernel needs the Kronecker factors mtri/mline");
    return PM_EINVAL;
  }
  KronMat M;
  for (int i = 0; i < LY::NH * LY::NH; ++i) M.t[i] = a.mtri[i];
  for (int i = 0; i < LY::NV * LY::NV; ++i) M.l[i] = a.mline[i];
  constexpr int LVA = LV > 0 ? LV : 1;
  const size_t smem =
      sizeof(double) * ((size_t)P.max_local * (W * CH + LV + 3 * (W + 1)) +
                        (size_t)P.max_y * CH * (W + 1) +
                        (size_t)P.max_owned * LVA) +
      sizeof(int2) * (size_t)P.max_steps +
      sizeof(int) * ((size_t)P.max_strips + 1 + P.max_owned + 1 + P.max_oy +
                     P.max_local);
  if (smem > 227 * 1024) {
    set_error("strip plan needs %zu bytes of shared memory", smem);
    return PM_EINVAL;
  }
  threads = strip_threads<LY>();
#define PM_STRIP(WW)                                                         \
  do {                                                                       \
    auto kern = k_strip<LY, WW>;                                             \
    PM_CUDA_TRY(cudaFuncSetAttribute(                                        \
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));      \
    int per_sm = 0;                                                          \
    PM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(               \
        &per_sm, kern, threads, smem));                                      \
    if (per_sm < 1) {                                                        \
      set_error("strip kernel does not fit (%zu B smem, %d threads)", smem,  \
                threads);                                                    \
      return PM_EINVAL;                                                      \
    }                                                                        \
    int64_t grid = (int64_t)sm_count() * per_sm;                             \
    if (grid > n_patches) grid = n_patches;                                  \
    kern<<<(unsigned)grid, threads, smem, a.s>>>(M, P, n_patches, a.layers,  \
                                                 a.coords, a.x, a.y);        \
  } while (0)
  if (W == 32)
    PM_STRIP(32);
  else if (W == 16)
    PM_STRIP(16);
  else if (W == 8)
    PM_STRIP(8);
  else {
    set_error("strip chunk width must be 8, 16 or 32 (got %d)", W);
    return PM_EINVAL;
  }
#undef PM_STRIP
  PM_LAUNCH_CHECK("k_strip");
  return PM_OK;
}

#define PM_STRIP_LAYOUTS(X)                                                  \
  X(1, 0, 0, 0, 0, 0)                                                        \
  X(0, 1, 0, 0, 0, 0)                                                        \
  X(0, 2, 0, 0, 0, 0)                                                        \
  X(3, 0, 0, 0, 0, 0)

bool strip_supports(const int32_t *d) {
#define PM_MATCH(a_, b_, c_, e_, f_, g_)                                     \
  if (Layout<a_, b_, c_, e_, f_, g_>::matches(d)) return true;
  PM_STRIP_LAYOUTS(PM_MATCH)
#undef PM_MATCH
  return false;
}

} // namespace pm

extern "C" int pm_column_mass_strip(
    const int32_t *delta6, int32_t k, int32_t layers, const double *coords,
    const double *mref, const double *mtri, const double *mline,
    const double *x, double *y, int64_t n_patches, int32_t chunk,
    int32_t threads, int32_t max_local, int32_t max_y, int32_t max_owned,
    int32_t max_steps, int32_t max_strips, int32_t max_oy,
    const int32_t *ent_ptr, const int32_t *owned, const int32_t *ents,
    const int32_t *patch_strip_ptr, const int32_t *strip_step_ptr,
    const uint16_t *step_v, const uint8_t *step_slot,
    const uint8_t *step_flags, const int32_t *step_y,
    const int32_t *patch_y_count, const int32_t *own_base,
    const int32_t *own_y_ptr, const int32_t *own_y, void *stream) {
  pm::clear_error();
  pm::LoopArgs a;
  int rc = pm::make_slot_table(delta6, &a.st);
  if (rc) return rc;
  if (k != a.st.k || layers < 1 || n_patches < 0 || !mref) {
    pm::set_error("bad arguments to pm_column_mass_strip");
    return PM_EINVAL;
  }
  if (!pm::strip_supports(delta6)) {
    pm::set_error("layout not supported by the strip schedule");
    return PM_EINVAL;
  }
  if (n_patches == 0) return PM_OK;
  if (!coords || !x || !y || !ent_ptr || !owned || !ents ||
      !patch_strip_ptr || !strip_step_ptr || !step_v || !step_slot ||
      !step_flags || !step_y || !own_base || !own_y_ptr || !own_y) {
    pm::set_error("NULL device pointer");
    return PM_EINVAL;
  }
  (void)patch_y_count;
  a.k = k;
  a.layers = layers;
  a.coords = coords;
  a.mref = mref;
  a.mtri = mtri;
  a.mline = mline;
  a.x = x;
  a.y = y;
  a.s = (cudaStream_t)stream;
  pm::StripDev P;
  P.ent_ptr = ent_ptr;
  P.owned = owned;
  P.ents = ents;
  P.patch_strip_ptr = patch_strip_ptr;
  P.strip_step_ptr = strip_step_ptr;
  P.step_v = step_v;
  P.step_slot = step_slot;
  P.step_flags = step_flags;
  P.step_y = step_y;
  P.patch_y_count = patch_y_count;
  P.own_base = own_base;
  P.own_y_ptr = own_y_ptr;
  P.own_y = own_y;
  P.max_local = max_local;
  P.max_y = max_y;
  P.max_owned = max_owned;
  P.max_steps = max_steps;
  P.max_strips = max_strips;
  P.max_oy = max_oy;
  P.column0 = (int64_t)layers * (delta6[0] + delta6[1]) + delta6[0];
#define PM_DISPATCH(a_, b_, c_, e_, f_, g_)                                  \
  if (pm::Layout<a_, b_, c_, e_, f_, g_>::matches(delta6))                   \
    return pm::strip_k<pm::Layout<a_, b_, c_, e_, f_, g_>>(a, P, n_patches,  \
                                                           chunk, threads);
  PM_STRIP_LAYOUTS(PM_DISPATCH)
#undef PM_DISPATCH
  return PM_EINVAL;
}
