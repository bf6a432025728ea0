// Strip-REDG schedule with TMA bulk-copy prefetch (vertex-column layouts).
//
// Same algorithm as k_strip_red (strip_red.cu): sequential strips, a 3-vertex
// register window per W-lane segment, one coalesced fp64 REDG per departing
// vertex.  The difference is how each step's vertex column chunk reaches
// shared memory: lane 0 of the segment issues two cp.async.bulk copies
// (field chunk, coordinate chunk) that complete on the ring slot's mbarrier,
// instead of every lane issuing 8-byte cp.async copies.  The copies never
// touch the LSU / L1 data path (SASS: UBLKCP).  Bulk copies need 16-byte
// aligned sources and sizes, so a chunk is fetched from the 16-byte boundary
// at or below its start with its size rounded up; the at most 8 bytes past
// the end of a field are fetched only if they lie inside the field's valid
// range, otherwise the last double is copied by lane 0 with a plain load.
#include "column_layout.cuh"
#include "pm_ptx.cuh"

#include <type_traits>

namespace pm {

constexpr int kSbDepth = 3;

template <class LY, int W> constexpr int sb_fs() { return W * LY::CH0 + LY::LV0; }
// entry: field part then coordinate part, each with a 2-double margin for
// the alignment shift and rounding, both 16-byte aligned
template <class LY, int W> constexpr int sb_fpart() {
  return ((sb_fs<LY, W>() + 3) / 2) * 2;
}
template <class LY, int W> constexpr int sb_cpart() {
  return ((3 * (W + 1) + 3) / 2) * 2;
}
template <class LY, int W> constexpr int sb_entry() {
  return sb_fpart<LY, W>() + sb_cpart<LY, W>();
}
template <class LY> constexpr int sb_min_blocks() {
  return LY::CH0 > 2 ? 1 : 2;
}

__device__ __forceinline__ void sb_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

template <class LY, int W, int K = LY::K>
__global__ void __launch_bounds__(256, sb_min_blocks<LY>())
k_strip_bulk(const KronMat M, const int32_t *__restrict__ strip_ptr,
             const int32_t *__restrict__ steps, int64_t n_strips, int layers,
             const double *__restrict__ coords, const double *__restrict__ x,
             double *__restrict__ y, int64_t x_lo, int64_t x_hi,
             int64_t c_lo, int64_t c_hi) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int SEGS = 32 / W;
  constexpr typename LY::Tab T = LY::make();
  constexpr int LV = LY::LV0, CH = LY::CH0;
  constexpr int LVA = LV > 0 ? LV : 1;
  constexpr int FP = sb_fpart<LY, W>(), ES = sb_entry<LY, W>();
  const int lane = threadIdx.x & 31;
  const int sl = lane % W, seg = lane / W;
  const int wid = threadIdx.x >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t col = (int64_t)layers * CH + LV;
  const int64_t ccol = 3 * (int64_t)(layers + 1);

  extern __shared__ __align__(16) double sb_smem[];
  const int n_slots = (blockDim.x >> 5) * SEGS * kSbDepth;
  double *zero = sb_smem + (size_t)n_slots * ES;
  uint64_t *bars = reinterpret_cast<uint64_t *>(zero + ES);
  for (int i = threadIdx.x; i < ES; i += blockDim.x) zero[i] = 0.0;
  if (sl == 0)
    for (int d = 0; d < kSbDepth; ++d)
      mbar_init(&bars[(wid * SEGS + seg) * kSbDepth + d], 1);
  fence_mbar_init();
  __syncthreads();
  uint32_t phase = 0; // bit d: parity of ring slot d's next completion

  const int n_chunks = (layers + W - 1) / W;
  const int64_t n_items = n_strips * n_chunks;
  for (int64_t i0 = warp * SEGS; i0 < n_items; i0 += n_warps * SEGS) {
    const int64_t item = i0 + seg;
    const bool has = item < n_items;
    const int64_t si = has ? item / n_chunks : 0;
    const int l0 = has ? (int)(item % n_chunks) * W : 0;
    const int k0 = has ? __ldg(strip_ptr + si) : 0;
    const int len = has ? __ldg(strip_ptr + si + 1) - k0 : 0;
    int maxlen = len;
#pragma unroll
    for (int o = W; o < 32; o <<= 1)
      maxlen = max(maxlen, __shfl_xor_sync(FULL, maxlen, o));
    const int nl = has ? min(W, layers - l0) : 0;
    const int l = l0 + sl;
    const bool lane_ok = sl < nl;
    const int fl = nl * CH + LV, cl = 3 * (nl + 1);

    double fb[3][CH], ft[3][LVA], cb[3][3], ct[3][3];
    double ab[3][CH], at[3][LVA];
    int64_t vo[3] = {0, 0, 0};
    bool live[3] = {false, false, false};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int c = 0; c < CH; ++c) fb[a][c] = 0.0, ab[a][c] = 0.0;
#pragma unroll
      for (int c = 0; c < LVA; ++c) ft[a][c] = 0.0, at[a][c] = 0.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) cb[a][q] = 0.0, ct[a][q] = 0.0;
    }
    int vbuf = (has && sl < len) ? __ldg(steps + k0 + sl) : 0;
    int vbase = 0;
    int rv[kSbDepth];
    int rsh[kSbDepth]; // (field shift) | (coord shift << 1)
    auto entry = [&](int slot) {
      return sb_smem + (size_t)((wid * SEGS + seg) * kSbDepth + slot) * ES;
    };
    auto bar = [&](int slot) {
      return &bars[(wid * SEGS + seg) * kSbDepth + slot];
    };
    auto fetch = [&](int k, int slot) {
      if (k - vbase >= W) {
        vbase += W;
        vbuf = (has && vbase + sl < len) ? __ldg(steps + k0 + vbase + sl)
                                         : 0;
      }
      const int v = __shfl_sync(FULL, vbuf, (k - vbase) & (W - 1), W);
      int shifts = 0;
      if (sl == 0) {
        uint64_t *b = bar(slot);
        if (k < len) {
          const int64_t fs = (int64_t)v * col + (int64_t)l0 * CH;
          const int64_t cs = (int64_t)v * ccol + 3 * (int64_t)l0;
          const int fa = (int)(fs & 1), ca = (int)(cs & 1);
          const uint32_t fbytes = (uint32_t)(((fl + fa) + 1) & ~1) * 8u;
          const uint32_t cbytes = (uint32_t)(((cl + ca) + 1) & ~1) * 8u;
          const bool fin = fs - fa >= x_lo && fs - fa + fbytes / 8 <= x_hi;
          const bool cin = cs - ca >= c_lo && cs - ca + cbytes / 8 <= c_hi;
          uint32_t tx = (fin ? fbytes : ((fl + fa) & ~1) * 8u) +
                        (cin ? cbytes : ((cl + ca) & ~1) * 8u);
          double *e = entry(slot);
          fence_proxy_async_smem(); // generic reads of the slot came first
          if (!fin)
            for (int i = (fl + fa) & ~1; i < fl + fa; ++i)
              e[i] = x[fs - fa + i];
          if (!cin)
            for (int i = (cl + ca) & ~1; i < cl + ca; ++i)
              e[FP + i] = coords[cs - ca + i];
          mbar_arrive_expect_tx(b, tx);
          const uint32_t fb_ = fin ? fbytes : ((fl + fa) & ~1) * 8u;
          const uint32_t cb_ = cin ? cbytes : ((cl + ca) & ~1) * 8u;
          if (fb_) bulk_g2s(e, x + (fs - fa), fb_, b);
          if (cb_) bulk_g2s(e + FP, coords + (cs - ca), cb_, b);
          shifts = fa | (ca << 1);
        } else {
          sb_arrive(b);
        }
      }
      shifts = __shfl_sync(FULL, shifts, 0, W);
      rv[slot] = v;
      rsh[slot] = shifts;
    };
#pragma unroll
    for (int d = 0; d < kSbDepth; ++d) fetch(d, d);

    auto flush = [&](auto A_) {
      constexpr int A = decltype(A_)::value;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        double v = ab[A][c];
        if (c < LV) {
          const double below = __shfl_up_sync(FULL, at[A][c], 1, W);
          if (sl > 0) v += below;
        }
        if (live[A] && lane_ok) {
          double *yp = y + vo[A] + (int64_t)l * CH + c;
          atomicAdd(yp, v);
          if (c < LV && sl == nl - 1) atomicAdd(yp + CH, at[A][c]);
        }
        ab[A][c] = 0.0;
      }
#pragma unroll
      for (int c = 0; c < LVA; ++c) at[A][c] = 0.0;
    };
    auto step = [&](auto A_, int k) {
      constexpr int A = decltype(A_)::value;
      flush(A_);
      const bool act = k < len;
      mbar_wait(bar(A), (phase >> A) & 1u);
      phase ^= 1u << A;
      const int64_t vcol = (int64_t)rv[A];
      const double *e = act ? entry(A) : zero;
      const int fsh = act ? (rsh[A] & 1) : 0, csh = act ? (rsh[A] >> 1) : 0;
      const double *ef = e + fsh, *ec = e + (act ? FP : 0) + csh;
#pragma unroll
      for (int c = 0; c < CH; ++c) fb[A][c] = ef[sl * CH + c];
#pragma unroll
      for (int c = 0; c < LV; ++c) ft[A][c] = ef[(sl + 1) * CH + c];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        cb[A][q] = ec[3 * sl + q];
        ct[A][q] = ec[3 * (sl + 1) + q];
      }
      vo[A] = vcol * col;
      live[A] = act;
      __syncwarp(); // every lane has read the slot before it is refilled
      fetch(k + kSbDepth, A);
      if (k < 2) return;
      double X[6], Y[6], Z[6];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        X[2 * a] = cb[a][0], Y[2 * a] = cb[a][1], Z[2 * a] = cb[a][2];
        X[2 * a + 1] = ct[a][0], Y[2 * a + 1] = ct[a][1];
        Z[2 * a + 1] = ct[a][2];
      }
      const double det = (act && lane_ok) ? prism_abs_detj(X, Y, Z) : 0.0;
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
    for (int k = 0; k < maxlen; k += 3) {
      step(S0{}, k);
      step(S1{}, k + 1);
      step(S2{}, k + 2);
    }
    flush(S0{});
    flush(S1{});
    flush(S2{});
    // drain: the kSbDepth prefetches past the loop must complete before
    // their slots are reused by the next item (or the CTA exits)
    const int kk = ((maxlen + 2) / 3) * 3;
#pragma unroll
    for (int d = 0; d < kSbDepth; ++d) {
      const int slot = (kk + d) % 3;
      mbar_wait(bar(slot), (phase >> slot) & 1u);
      phase ^= 1u << slot;
    }
  }
}

template <class LY>
int strip_bulk_k(const LoopArgs &a, const int32_t *strip_ptr,
                 const int32_t *steps, int64_t n_strips, int W, int64_t x_lo,
                 int64_t x_hi, int64_t c_lo, int64_t c_hi) {
  KronMat M;
  for (int i = 0; i < LY::NH * LY::NH; ++i) M.t[i] = a.mtri[i];
  for (int i = 0; i < LY::NV * LY::NV; ++i) M.l[i] = a.mline[i];
  const int segs = 32 / W;
  const int64_t items = n_strips * ((a.layers + W - 1) / W);
  const int64_t warps = (items + segs - 1) / segs;
  const unsigned grid = grid_for(warps * 32, 256, 8);
#define PM_SB(WW)                                                            \
  do {                                                                       \
    const size_t smem =                                                      \
        sizeof(double) * ((size_t)8 * (32 / WW) * kSbDepth + 1) *            \
            sb_entry<LY, WW>() +                                             \
        sizeof(uint64_t) * 8 * (32 / WW) * kSbDepth;                         \
    PM_CUDA_TRY(cudaFuncSetAttribute(                                        \
        k_strip_bulk<LY, WW>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
        (int)smem));                                                         \
    k_strip_bulk<LY, WW><<<grid, 256, smem, a.s>>>(                          \
        M, strip_ptr, steps, n_strips, a.layers, a.coords, a.x, a.y, x_lo,   \
        x_hi, c_lo, c_hi);                                                   \
  } while (0)
  if (W == 32)
    PM_SB(32);
  else if (W == 16)
    PM_SB(16);
  else if (W == 8)
    PM_SB(8);
  else {
    set_error("strip chunk width must be 8, 16 or 32 (got %d)", W);
    return PM_EINVAL;
  }
#undef PM_SB
  PM_LAUNCH_CHECK("k_strip_bulk");
  return PM_OK;
}

int launch_strip_bulk(const LoopArgs &a, const int32_t *delta6,
                      const int32_t *strip_ptr, const int32_t *steps,
                      int64_t n_strips, int W, int64_t x_lo, int64_t x_hi,
                      int64_t c_lo, int64_t c_hi) {
#define PM_DISPATCH(a_, b_, c_, e_, f_, g_)                                  \
  if (Layout<a_, b_, c_, e_, f_, g_>::matches(delta6))                       \
    return strip_bulk_k<Layout<a_, b_, c_, e_, f_, g_>>(                     \
        a, strip_ptr, steps, n_strips, W, x_lo, x_hi, c_lo, c_hi);
  PM_DISPATCH(1, 0, 0, 0, 0, 0)
  PM_DISPATCH(0, 1, 0, 0, 0, 0)
  PM_DISPATCH(0, 2, 0, 0, 0, 0)
  PM_DISPATCH(3, 0, 0, 0, 0, 0)
#undef PM_DISPATCH
  set_error("layout not supported by the bulk strip schedule");
  return PM_EINVAL;
}

} // namespace pm

extern "C" int pm_column_mass_strip_bulk(
    const int32_t *delta6, int32_t k, int32_t layers, const double *coords,
    const double *mref, const double *mtri, const double *mline,
    const double *x, double *y, int64_t x_lo, int64_t x_hi, int64_t c_lo,
    int64_t c_hi, int32_t accumulate, int64_t n_strips, int32_t chunk,
    const int32_t *strip_ptr, const int32_t *steps, void *stream) {
  pm::clear_error();
  pm::LoopArgs a;
  int rc = pm::make_slot_table(delta6, &a.st);
  if (rc) return rc;
  if (k != a.st.k || layers < 1 || n_strips < 0 || !mref || !mtri ||
      !mline || x_hi < x_lo || c_hi < c_lo) {
    pm::set_error("bad arguments to pm_column_mass_strip_bulk");
    return PM_EINVAL;
  }
  a.k = k;
  a.layers = layers;
  a.coords = coords;
  a.mref = mref;
  a.mtri = mtri;
  a.mline = mline;
  a.x = x;
  a.y = y;
  a.s = (cudaStream_t)stream;
  if (!accumulate && x_hi > x_lo)
    PM_CUDA_TRY(cudaMemsetAsync(y + x_lo, 0,
                                (size_t)(x_hi - x_lo) * sizeof(double), a.s));
  if (n_strips == 0) return PM_OK;
  if (!coords || !x || !y || !strip_ptr || !steps) {
    pm::set_error("NULL device pointer");
    return PM_EINVAL;
  }
  return pm::launch_strip_bulk(a, delta6, strip_ptr, steps, n_strips, chunk,
                               x_lo, x_hi, c_lo, c_hi);
}
