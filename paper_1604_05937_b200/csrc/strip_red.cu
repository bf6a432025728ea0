// Global-strip schedule for vertex-column CG layouts (PM_VARIANT_STRIPRED):
// P1, 3-vector P1, CG1 x DG0, CG1 x DG1.
//
// The base cells are walked as sequential strips (consecutive cells share
// the edge of the two youngest window vertices, schedule.build_global_
// strips), so every step brings exactly one new vertex into a 3-vertex
// register window and the replaced window slot cycles 0,1,2 (compile-time
// after a 3-way unroll).  A W-lane segment owns a strip, lane = layer of the
// current W-layer chunk:
//   * the new vertex's field and (x,y,z) at the lane's level are loaded
//     straight from global memory, prefetched one step ahead (the strip's
//     vertex ids are fetched W at a time and handed out by shfl);
//   * the level above comes from the next lane (shfl.down);
//   * the cell-layer contribution (sum-factorised Mtri (x) Mline) goes into
//     per-window-vertex accumulators in registers;
//   * when a vertex leaves the window its partial column is added to y with
//     one coalesced fp64 REDG per channel (top contributions shifted one
//     lane up; the chunk's top level by the last lane).
// One vertex load and one partial flush per cell instead of three gathers
// and three scatters per cell-layer.  Needs y zeroed first (overwrite mode).
#include "column_layout.cuh"
#include "pm_ptx.cuh"

#include <cstdlib>
#include <type_traits>

namespace pm {

__device__ __forceinline__ void sr_cp8(double *dst, const double *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void sr_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N> __device__ __forceinline__ void sr_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void sr_mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}

// ring entry per segment: the vertex's chunk of the field column
// (W*CH + LV values) and of the coordinate column (3*(W+1) values)
template <class LY, int W> constexpr int sr_fs() { return W * LY::CH0 + LY::LV0; }
template <class LY, int W> constexpr int sr_entry() {
  return sr_fs<LY, W>() + 3 * (W + 1);
}
// bulk (TMA) ring entries: both parts start 16-byte aligned and leave room
// for the 8-byte alignment shift and the rounding to 16-byte sizes
template <class LY, int W> constexpr int srb_fpart() {
  return ((sr_fs<LY, W>() + 3) / 2) * 2;
}
template <class LY, int W> constexpr int srb_entry() {
  return srb_fpart<LY, W>() + ((3 * (W + 1) + 3) / 2) * 2;
}
// steps in flight per segment: 3 (ring slot = window slot) or 6 (ring slot
// k % 6, window slot k % 3; compile-time PM_SR_DEPTH)
#ifndef PM_SR_DEPTH
#define PM_SR_DEPTH 3
#endif
constexpr int kSrDepth = PM_SR_DEPTH;
// PM_EXPERIMENTAL = 1: also compile the store-first patch-strip kernels
// (stream mode, schedule "pstrip"; slower than the global strips on every
// config, profiles/README.md)
#ifndef PM_EXPERIMENTAL
#define PM_EXPERIMENTAL 0
#endif
static_assert(kSrDepth == 3 || kSrDepth == 6, "ring depth 3 or 6");
// PM_SR_CELLSUM = 1 (default, scalar vertex columns): with the invariant
// triangle factor
// (Mtri = ta I + tb J) a window vertex's contribution from cell j is
// dta_j z_h + d_j, d_j = dtb_j (z_0 + z_1 + z_2): the same d_j for all
// three window vertices, and z_h fixed while h is in the window.  A vertex
// lives in exactly the three cells formed while it is in the window, the
// last three cells when it leaves, so instead of three accumulators
// updated every step (3 DADD + 3 DFMA per channel) the kernel keeps the
// last three cells' dta and d in a 3-slot ring (slot = cell % 3) and
// forms z_h (dta_k + dta_k+1 + dta_k+2) + (d_k + d_k+1 + d_k+2) once, when
// the vertex leaves.
#ifndef PM_SR_CELLSUM
#define PM_SR_CELLSUM 1
#endif


// Padded ring entries of the strip kernel (a chunk of CW = W*L levels):
// the field part and the coordinate part are whole rows of W values, so
// every lane issues every copy (cp.async with a 0/8-byte source size:
// lanes past the chunk zero-fill their row slot instead of being
// predicated off).
template <class LY, int CW> constexpr int sr_fsz() {
  return CW * LY::CH0 + LY::LV0;
}
#ifndef PM_SR16
#define PM_SR16 0
#endif
// PM_SR16: 16-byte cp.async.cg rows (L1 bypassed) of the 16-byte aligned
// superset of each chunk (per-vertex shift 0/1), W lanes x 2 doubles
constexpr int kSrVec = PM_SR16 ? 2 : 1; // doubles per lane per row
template <class LY, int W, int L> constexpr int sr_frows() {
  return (sr_fsz<LY, W * L>() + (kSrVec - 1) + kSrVec * W - 1) / (kSrVec * W);
}
template <class LY, int W, int L> constexpr int sr_crows() {
  return (3 * (W * L + 1) + (kSrVec - 1) + kSrVec * W - 1) / (kSrVec * W);
}
// PM_SR_PACK: the coordinate chunk follows the field chunk directly in the
// ring entry (one row straddles both), so a step copies
// ceil((fsz + 3 (CW + 1)) / W) rows instead of a row-rounded field part
// plus a row-rounded coordinate part (P1 at W = 32: 5 copies instead of 6;
// measured C5a -3 %, config-4 P1 -2..3 %; 3-vector P1 +1.5 %, so scalar
// vertex columns only)
#ifndef PM_SR_PACK
#define PM_SR_PACK 1
#endif
template <class LY> constexpr bool sr_pack() {
  return PM_SR_PACK && !PM_SR16 && LY::CH0 == 1;
}
template <class LY, int W, int L> constexpr int sr_prows() {
  return (sr_fsz<LY, W * L>() + 3 * (W * L + 1) + W - 1) / W;
}
template <class LY, int W, int L> constexpr int sr_pentry() {
  return sr_pack<LY>() ? sr_prows<LY, W, L>() * W
                 : (sr_frows<LY, W, L>() + sr_crows<LY, W, L>()) * kSrVec * W;
}
constexpr int kSrIds = 64; // strip vertex ids staged per segment
#ifndef PM_SR_VTHREADS
#define PM_SR_VTHREADS 384
#endif
// CTA size: 256 threads, 384 for the 3-vector layouts (12 warps at <= 168
// registers instead of 8 at 182)
#ifndef PM_SR_STHREADS
#define PM_SR_STHREADS 256 // CTA size of the scalar / 2-channel strip kernel
#endif
static_assert(PM_SR_STHREADS == 128 || PM_SR_STHREADS == 256 ||
                  PM_SR_STHREADS == 512,
              "PM_SR_STHREADS: 128, 256 or 512 (2 CTAs of 256 per SM at most)");
template <class LY> constexpr int sr_threads() {
  return LY::CH0 > 2 ? PM_SR_VTHREADS : PM_SR_STHREADS;
}
// Multi-channel layouts (3-vector P1: CH = 3) flush through a per-segment
// staging row of the chunk's (W + 1) * CH values, so the REDs run over
// consecutive addresses (lane-contiguous) instead of at a CH * 8-byte
// stride: a third of the L2 reduction sector operations
#ifndef PM_SR_TROW
#define PM_SR_TROW 1
#endif
// 1: ring copies zero-fill the unused tail of each row (every lane writes);
// 0: lanes past the chunk copy nothing (measured: C5a -1 %, C4 P1 -3 %,
// C5b +2 %: kept at 1)
#ifndef PM_SR_ZFILL
#define PM_SR_ZFILL 1
#endif
template <class LY, int W, int L> constexpr int sr_trow() {
  return (PM_SR_TROW && L == 1 && LY::CH0 > 1) ? (W + 1) * LY::CH0 : 0;
}
// PM_SR_DEFER = 1: the staged row's REDs are issued one flush later, from
// the other of two staging rows, after the next row was staged: the row's
// LDS results are ready by then (without it every RED waited on its LDS,
// 15 % of the C5b warp stall samples, ncu source page)
#ifndef PM_SR_DEFER
#define PM_SR_DEFER 1
#endif
constexpr int kSrTrowBufs = PM_SR_DEFER ? 2 : 1;
template <class LY, int W, int L> constexpr size_t sr_smem() {
  return sizeof(double) *
             ((size_t)(sr_threads<LY>() / 32) * kSrDepth * (32 / W) + 1) *
             sr_pentry<LY, W, L>() +
         sizeof(int) * (sr_threads<LY>() / 32) * (32 / W) * kSrIds +
         sizeof(double) * (sr_threads<LY>() / 32) * (32 / W) *
             sr_trow<LY, W, L>() * kSrTrowBufs;
}

__device__ __forceinline__ void sr_cp16z(double *dst, const double *src,
                                         int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void sr_cp8z(double *dst, const double *src,
                                        int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}

// Flush of a partial column element: mode 0 = nothing, 1 = add (REDG),
// 3 = store (the first residency of a patch-interior entity, pm_build_patch_
// strips).  Bit 0 = live, bit 1 = store, so `mode & mask` demotes a store
// to an add (mask 1) or drops the element (mask 0).
constexpr int kPutAdd = 1, kPutStore = 3;
__device__ __forceinline__ void sr_put(double *p, double v, int mode) {
  asm volatile("{\n\t.reg .pred ps, pr;\n\t"
               "setp.eq.s32 ps, %2, 3;\n\t"
               "setp.eq.s32 pr, %2, 1;\n\t"
               "@ps st.global.f64 [%0], %1;\n\t"
               "@pr red.global.add.f64 [%0], %1;\n\t}" ::"l"(p),
               "d"(v), "r"(mode)
               : "memory");
}
// predicated REDG, system scope (the fused halo's adds into a peer's window
// over NVLink, and the owner's own adds into it, are ordered at system
// scope; red.global defaults to .gpu)
__device__ __forceinline__ void sr_red_sys(double *p, double v, bool on) {
  asm volatile("{\n\t.reg .pred q;\n\t"
               "setp.ne.b32 q, %2, 0;\n\t"
               "@q red.sys.global.add.f64 [%0], %1;\n\t}" ::"l"(p),
               "d"(v), "r"((int)on)
               : "memory");
}
// predicated REDG (no branch around it)
__device__ __forceinline__ void sr_red(double *p, double v, bool on) {
  asm volatile("{\n\t.reg .pred q;\n\t"
               "setp.ne.b32 q, %2, 0;\n\t"
               "@q red.global.add.f64 [%0], %1;\n\t}" ::"l"(p),
               "d"(v), "r"((int)on)
               : "memory");
}
constexpr int kIdMask = PM_STEP_NOCELL - 1; // entity id of a step record

// element `v` of a column family with a stride in bytes (one IMAD.WIDE)
template <class T>
__device__ __forceinline__ T *col_at(T *base, int v, int stride_bytes) {
  using C = typename std::conditional<std::is_const<T>::value, const char,
                                      char>::type;
  return reinterpret_cast<T *>(reinterpret_cast<C *>(base) +
                               (int64_t)v * stride_bytes);
}

template <class LY, int L> constexpr int sr_blocks() {
  return (LY::CH0 > 2 || L > 1) ? 1 : 512 / PM_SR_STHREADS;
}

// The element kernel split along the window: y = det (Mtri (x) Mline) x.
// The interval stage z = Mline x only involves one vertex column, so it is
// applied once when the vertex enters the window (not in each of its three
// cells); per cell only the triangle stage runs, with det folded into the
// accumulation: acc[h] = fma(det, sum_g Mtri[h][g] z[g], acc[h]).
// L consecutive levels per lane (lane sl: levels l0 + L*sl + j, j < L):
// the level between two of them is read once, and the per-step overhead
// (ids, ring wait, addressing, loop) is paid once per L cell-layers.
template <class LY, int W, bool SYM, int L, bool PEER = false,
          bool STREAM = false, int K = LY::K>
__global__ void __launch_bounds__(sr_threads<LY>(), sr_blocks<LY, L>())
k_strip_red(const KronMat M, const int32_t *__restrict__ item_ptr,
            const int32_t *__restrict__ strip_ptr,
            const int32_t *__restrict__ steps, int64_t n_groups, int layers,
            int lbeg, int lend,
            const double *__restrict__ coords, const double *__restrict__ x,
            double *__restrict__ y, double *__restrict__ y_peer,
            int ghost_end, int store) {
  constexpr unsigned FULL = 0xffffffffu;
  // step ids carry flag bits only in STREAM mode
  constexpr int IDM = STREAM ? kIdMask : -1;
  constexpr int SEGS = 32 / W;
  constexpr int CW = W * L; // levels per chunk
  constexpr int LV = LY::LV0;
  constexpr int CH = LY::CH0;
  constexpr int LVA = LV > 0 ? LV : 1;
  constexpr int NC = LY::NC, NV = LY::NV, NH = LY::NH;
  // (component c, interval function v) of a vertex layer block: level
  // copies bottom fb[c] (v = 0) / top ft[c] (v = 1), or, without level
  // copies, connecting channel v*NC + c (the slot table of fspace.py)
  static_assert(NH == 3 && NC * NV == CH + LV, "vertex-column layout");
  static_assert(LV == 0 || (LV == NC && NV == 2 && CH == LV), "strip layout");
  constexpr int FR = sr_frows<LY, W, L>(), CR = sr_crows<LY, W, L>();
  // coordinate part offset in a ring entry
  constexpr bool kSrPack = sr_pack<LY>();
  constexpr int FP = kSrPack ? sr_fsz<LY, CW>() : FR * kSrVec * W;
  constexpr int PR = sr_prows<LY, W, L>(); // rows of a packed entry
  constexpr int ES = sr_pentry<LY, W, L>();
  const int lane = threadIdx.x & 31;
  const int sl = lane % W, seg = lane / W;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // column lengths in bytes fit 32 bits: a column origin is one IMAD.WIDE
  const int colb = 8 * (layers * CH + LV); // vertex column
  const int ccolb = 8 * 3 * (layers + 1);  // coordinate column
  extern __shared__ double sr_ring[];
  double *const ring =
      sr_ring + (size_t)(threadIdx.x >> 5) * kSrDepth * SEGS * ES;
  constexpr int NWARP = sr_threads<LY>() / 32;
  const double *const sr_zero =
      sr_ring + (size_t)NWARP * kSrDepth * SEGS * ES;
  int *const sid = reinterpret_cast<int *>(sr_ring + (size_t)(NWARP * kSrDepth *
                                                              SEGS + 1) * ES) +
                   ((threadIdx.x >> 5) * SEGS + seg) * kSrIds;
  constexpr int TR = sr_trow<LY, W, L>();
  // deferred REDs of the staged rows (non-stream strips only)
  constexpr bool DEFER = TR > 0 && PM_SR_DEFER && !STREAM;
  double *const trow0 =
      reinterpret_cast<double *>(reinterpret_cast<int *>(
          sr_ring + (size_t)(NWARP * kSrDepth * SEGS + 1) * ES) +
                                 NWARP * SEGS * kSrIds) +
      ((threadIdx.x >> 5) * SEGS + seg) * TR * kSrTrowBufs;
  // the zero block (and, without zero-filling copies, the whole ring)
  for (int i = threadIdx.x; i < (PM_SR_ZFILL ? 1 : NWARP * kSrDepth * SEGS + 1) * ES;
       i += blockDim.x)
    sr_ring[(size_t)(PM_SR_ZFILL ? NWARP * kSrDepth * SEGS * ES : 0) + i] = 0.0;
  __syncthreads();

  // work item = (group, layer chunk), chunk fastest: the chunks of a group
  // run side by side, so the sectors two chunks of a vertex column share
  // are fetched once (neighbouring groups are still close in time).  A
  // group is one global strip (item_ptr == NULL) or the strips of a patch
  // (item_ptr[p] .. item_ptr[p+1]), walked one after the other.
  // this launch covers levels [lbeg, lend) (a mixed-width chunk plan runs
  // one launch per width); column strides stay those of all `layers`
  const int n_chunks = (lend - lbeg + CW - 1) / CW;
  const int64_t n_items = n_groups * n_chunks;
  for (int64_t i0 = warp * SEGS; i0 < n_items; i0 += n_warps * SEGS) {
    const int64_t item = i0 + seg;
    const bool has = item < n_items;
    const int64_t gi = has ? item / n_chunks : 0;
    const int l0 = has ? lbeg + (int)(item % n_chunks) * CW : 0;
    // the group's steps are one contiguous range; in STREAM mode (patch
    // strips) its strips follow each other without a window refill: the
    // three fill steps of a strip flush the previous strip's vertices
    const int64_t gs = item_ptr ? __ldg(item_ptr + gi) : gi;
    const int64_t ge = item_ptr ? __ldg(item_ptr + gi + 1) : gi + 1;
    const int k0 = has ? __ldg(strip_ptr + gs) : 0;
    const int len = has ? __ldg(strip_ptr + ge) - k0 : 0;
    int maxlen = len;
#pragma unroll
    for (int o = W; o < 32; o <<= 1)
      maxlen = max(maxlen, __shfl_xor_sync(FULL, maxlen, o));
    const int nl = has ? min(CW, lend - l0) : 0;
    const int lb = L * sl; // the lane's first level in the chunk
    // store-first flushes (STREAM): the chunk's bottom level is shared with
    // the chunk below (its top), so lane 0 of an upper chunk always adds,
    // and so does the top lane unless the chunk ends the column (the zero
    // pass clears those levels).  Masks of the flush mode (sr_put): this
    // lane's values, its bottom level copy, the chunk's top level copy.
    const int mmask = lb < nl ? kPutStore : 0;
    const int bmask = lb >= nl                        ? 0
                      : (L == 1 && (sl > 0 || l0 == 0)) ? kPutStore
                                                          : kPutAdd;
    const int tmask = lb + L - 1 != nl - 1               ? 0
                      : (L == 1 && l0 + nl == layers) ? kPutStore
                                                       : kPutAdd;
    // source sizes of the lane's copies (8 inside the chunk, else 0)
    int fz[FR], cz[CR], pz[PR];
#pragma unroll
    for (int r = 0; r < PR; ++r) { // packed rows: field, then coordinates
      const int i = sl + W * r;
      pz[r] = i < FP ? (i < nl * CH + LV ? 8 : 0)
                     : (i - FP < 3 * (nl + 1) ? 8 : 0);
    }
#pragma unroll
    for (int r = 0; r < FR; ++r) fz[r] = sl + W * r < nl * CH + LV ? 8 : 0;
#pragma unroll
    for (int r = 0; r < CR; ++r) cz[r] = sl + W * r < 3 * (nl + 1) ? 8 : 0;
    // the segment's chunk of every column (copies), the lane's first
    // element of it (flushes)
    const double *xl = x + (int64_t)l0 * CH + sl;
    const double *cl0 = coords + 3 * (int64_t)l0 + sl;
    double *yl = y + ((int64_t)l0 + lb) * CH;
    // fused halo: a ghost vertex's partial columns go straight to its
    // owner's window (peer memory over NVLink) instead of a local window
    // that a later exchange would ship
    double *ylg = PEER ? y_peer + ((int64_t)l0 + lb) * CH : yl;
    // window vertex: interval-stage values z[j][c][v] at the lane's cell
    // layers and the geometry the Jacobian needs, derived once on entry:
    // xm, ym (mid-layer), dz; per-vertex accumulators acc[j][c][v]
    double zv[3][L][NC][NV], gm[3][L][3], acc[3][L][NC][NV];
    // PM_SR_CELLSUM: the last three cells' dta (tr) and d (dr), ring slot
    // = the window slot of the step that formed the cell
    // (scalar columns: measured -1..3 % on P1; the 3-vector columns lose
    // 2.5 % -- the flush's dependent sums lengthen its critical path)
    constexpr bool CSUM = SYM && PM_SR_CELLSUM && NC == 1;
    double tr[CSUM ? 3 : 1][L], dr[CSUM ? 3 : 1][L][NC][NV];
#pragma unroll
    for (int a = 0; a < (CSUM ? 3 : 1); ++a)
#pragma unroll
      for (int j = 0; j < L; ++j) {
        tr[a][j] = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int v = 0; v < NV; ++v) dr[a][j][c][v] = 0.0;
      }
    double *yc[3] = {yl, yl, yl}; // lane's first element of the column
    bool live[3] = {false, false, false}, st[3] = {false, false, false};
    // DEFER: staging row in use, the previously staged row's chunk origin
    // and liveness (its REDs are still to be issued)
    int tb = 0;
    double *pbase = y;
    bool plive = false;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int j = 0; j < L; ++j) {
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int v = 0; v < NV; ++v)
            zv[a][j][c][v] = 0.0, acc[a][j][c][v] = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) gm[a][j][q] = 0.0;
      }
    // the strip's vertex ids, staged kSrIds at a time (one broadcast LDS
    // per step)
    auto load_ids = [&](int base) {
#pragma unroll
      for (int r = 0; r < kSrIds / W; ++r) {
        const int i = base + sl + W * r;
        sid[sl + W * r] = i < len ? __ldg(steps + k0 + i) : 0;
      }
      __syncwarp();
    };
    __syncwarp(); // the previous item's last id reads are done
    load_ids(0);
    // per-warp shared-memory prefetch ring, kSrDepth steps deep: the
    // segment copies its vertex's chunk of the field and coordinate
    // columns contiguously (coalesced cp.async); lanes then read their
    // own levels (and the level above) out of shared memory.
    auto entry = [&](int slot) {
      return ring + (size_t)(slot * SEGS + seg) * ES;
    };
    int rv[kSrDepth];
#if PM_SR16
    int rsh[kSrDepth];
    const int fbytes = 8 * (nl * CH + LV) - 16 * sl;
    const int cbytes = 8 * 3 * (nl + 1) - 16 * sl;
    const double *xs = xl - sl, *cs = cl0 - sl;
#endif
    auto fetch = [&](int k, int slot) {
      if ((k & (kSrIds - 1)) == 0 && k > 0) { // warp-uniform
        __syncwarp();
        load_ids(k);
      }
      const int v = sid[k & (kSrIds - 1)];
#if PM_SR16
      const double *fp = col_at(xs, v & IDM, colb);
      const double *cp = col_at(cs, v & IDM, ccolb);
      const int fsh = (int)(reinterpret_cast<uintptr_t>(fp) >> 3) & 1;
      const int csh = (int)(reinterpret_cast<uintptr_t>(cp) >> 3) & 1;
      if (k < len) {
        double *e = entry(slot) + 2 * sl;
        const double *fa = fp - fsh + 2 * sl, *ca = cp - csh + 2 * sl;
#pragma unroll
        for (int r = 0; r < FR; ++r)
          sr_cp16z(e + 2 * W * r, fa + 2 * W * r,
                   min(max(fbytes + 8 * fsh - 16 * W * r, 0), 16));
#pragma unroll
        for (int r = 0; r < CR; ++r)
          sr_cp16z(e + FP + 2 * W * r, ca + 2 * W * r,
                   min(max(cbytes + 8 * csh - 16 * W * r, 0), 16));
      }
      rsh[slot] = fsh | (csh << 1);
#else
      if (k < len) {
        const double *fp = col_at(xl, v & IDM, colb);
        const double *cp = col_at(cl0, v & IDM, ccolb);
        double *e = entry(slot) + sl;
        if constexpr (kSrPack) {
#pragma unroll
          for (int r = 0; r < PR; ++r) {
            if (W * (r + 1) <= FP) // field row
              sr_cp8z(e + W * r, fp + W * r, pz[r]);
            else if (W * r >= FP) // coordinate row
              sr_cp8z(e + W * r, cp + (W * r - FP), pz[r]);
            else // the row that straddles both parts
              sr_cp8z(e + W * r,
                      sl + W * r < FP ? fp + W * r : cp + (W * r - FP),
                      pz[r]);
          }
        } else {
#if PM_SR_ZFILL
#pragma unroll
        for (int r = 0; r < FR; ++r) sr_cp8z(e + W * r, fp + W * r, fz[r]);
#pragma unroll
        for (int r = 0; r < CR; ++r)
          sr_cp8z(e + FP + W * r, cp + W * r, cz[r]);
#else
        // lanes past the chunk copy nothing (the last row of each part is
        // mostly empty: 1 of 33 field / 3 of 99 coordinate values at W =
        // 32); they read stale ring values, finite since the ring starts
        // zeroed, and are never flushed
#pragma unroll
        for (int r = 0; r < FR; ++r)
          if (fz[r]) sr_cp8(e + W * r, fp + W * r);
#pragma unroll
        for (int r = 0; r < CR; ++r)
          if (cz[r]) sr_cp8(e + FP + W * r, cp + W * r);
#endif
        }
      }
#endif
      sr_commit(); // one group per step (possibly empty)
      return v;
    };
#pragma unroll
    for (int d = 0; d < kSrDepth; ++d) rv[d] = fetch(d, d);

    auto flush = [&](auto A_) {
      constexpr int A = decltype(A_)::value;
      double *const trow = trow0 + (DEFER ? tb * TR : 0);
      constexpr int NR = TR > 0 ? (TR + W - 1) / W : 1;
      double pv[NR];
      if constexpr (DEFER) { // the previous row's values (staged, synced)
        const double *prow = trow0 + (tb ^ 1) * TR;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const int i = sl + W * r;
          pv[r] = prow[i < TR ? i : 0];
        }
      }
      if constexpr (CSUM) {
        // the leaving vertex's cells are the last three: all ring slots
#pragma unroll
        for (int j = 0; j < L; ++j) {
          const double t = tr[0][j] + tr[1][j] + tr[2][j];
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < NV; ++v)
              acc[A][j][c][v] =
                  fma(zv[A][j][c][v], t,
                      dr[0][j][c][v] + dr[1][j][c][v] + dr[2][j][c][v]);
        }
      }
      // back to the vertex column's layer blocks: per level j the bottom /
      // connecting channels vb[j], the top copies of the lane's last level
      // vt (added by the lane above, or by the chunk's last lane)
      double vb[L][CH], vt[LVA];
#pragma unroll
      for (int j = 0; j < L; ++j)
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const double a = acc[A][j][c][v];
            if (LV == 0)
              vb[j][v * NC + c] = a;
            else if (v == 0)
              vb[j][c] = a + (j > 0 ? vb[j][c] : 0.0);
            else if (j + 1 < L)
              vb[j + 1][c < LVA ? c : 0] = a; // summed when j+1 is visited
            else
              vt[c < LVA ? c : 0] = a;
            acc[A][j][c][v] = 0.0;
          }
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        double v0 = vb[0][c];
        if (c < LV) {
          const double below = __shfl_up_sync(FULL, vt[c < LV ? c : 0], 1, W);
          if (sl > 0) v0 += below;
        }
        if constexpr (STREAM && TR == 0) { // store-first patch strips
          const int put = !live[A] ? 0 : st[A] ? kPutStore : kPutAdd;
#pragma unroll
          for (int j = 0; j < L; ++j)
            sr_put(yc[A] + j * CH + c, j ? vb[j][c] : v0,
                   put & (j > 0 || c >= LV ? mmask : bmask));
          if (c < LV)
            sr_put(yc[A] + L * CH + c, vt[c < LV ? c : 0], put & tmask);
        } else if constexpr (TR > 0) { // staged, added / stored below
          // (lanes past the chunk stay out: their slot is the chunk top)
          if (sl < nl) trow[sl * CH + c] = v0;
          if (c < LV && sl == nl - 1)
            trow[(sl + 1) * CH + c] = vt[c < LV ? c : 0];
        } else {
#pragma unroll
          for (int j = 0; j < L; ++j)
            (PEER ? sr_red_sys : sr_red)(yc[A] + j * CH + c, j ? vb[j][c] : v0,
                   live[A] && lb + j < nl);
          if (c < LV)
            (PEER ? sr_red_sys : sr_red)(yc[A] + L * CH + c, vt[c < LV ? c : 0],
                   live[A] && lb + L - 1 == nl - 1);
        }
        if (live[A]) {
          if (c < LV && L > 1 && lb < nl && lb + L - 1 > nl - 1) {
            // partial chunk ending inside this lane: its top is the level
            // after the last valid one
#pragma unroll
            for (int j = 0; j + 1 < L; ++j)
              if (lb + j == nl - 1)
                atomicAdd(yc[A] + (j + 1) * CH + c, vb[j + 1][c]);
          }
        }
      }
      if constexpr (TR > 0) { // the staged chunk, lane-contiguous REDs
        if constexpr (!DEFER) __syncwarp();
        double *const base = yc[A] - sl * CH; // the chunk's first value
        const int n = nl * CH + LV;
        if constexpr (STREAM) {
          // store-first: the chunk's bottom / top level copies are shared
          // with the chunks below / above (zeroed, always added)
          const int put = !live[A] ? 0 : st[A] ? kPutStore : kPutAdd;
          const int lo = l0 > 0 ? LV : 0, hi = l0 + nl < layers ? n - LV : n;
#pragma unroll
          for (int r = 0; r < (TR + W - 1) / W; ++r) {
            const int i = sl + W * r;
            sr_put(base + i, trow[i < TR ? i : 0],
                   i >= n ? 0 : (i < lo || i >= hi) ? (put & kPutAdd) : put);
          }
        } else if constexpr (DEFER) {
          // the previous row's REDs now; this row's at the next flush (the
          // step's own __syncwarp orders the STS above before those LDS)
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            const int i = sl + W * r;
            (PEER ? sr_red_sys : sr_red)(pbase + i, pv[r], plive && i < n);
          }
          pbase = base;
          plive = live[A];
          tb ^= 1;
        } else {
#pragma unroll
          for (int r = 0; r < (TR + W - 1) / W; ++r) {
            const int i = sl + W * r;
            (PEER ? sr_red_sys : sr_red)(base + i, trow[i < TR ? i : 0],
                                         live[A] && i < n);
          }
        }
        if constexpr (!DEFER)
          __syncwarp(); // row reads done before the next flush stages
      }
    };

    // one strip step into window slot A; FILL: the first three steps (the
    // window fills, nothing to flush, no cell before the third vertex)
    auto step = [&](auto A_, auto R_, auto FILL_, int k) {
      constexpr int A = decltype(A_)::value; // window slot (k % 3)
      constexpr int R = decltype(R_)::value; // ring slot (k % kSrDepth)
      constexpr bool FILL = decltype(FILL_)::value;
      if (!FILL) flush(A_);
      const bool act = k < len;
      // the vertex of ring slot A (step k) enters window slot A
      sr_wait<kSrDepth - 1>(); // this lane's copies of step k landed
      __syncwarp();            // ... and the other lanes' ones
      // steps past this segment's strip read a zero block instead of the
      // (stale, possibly non-finite) ring slot; lanes past the chunk read
      // zero-filled values and are never flushed.
      const double *e = act ? entry(R) : sr_zero;
#if PM_SR16
      const int sh = act ? rsh[R] : 0;
      const double *ef = e + (sh & 1), *ec = e + FP + (sh >> 1);
#else
      const double *ef = e, *ec = e + FP;
#endif
      double f[L + 1][CH], g[L + 1][3];
#pragma unroll
      for (int j = 0; j <= L; ++j) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
          f[j][c] = (j < L || c < LV) ? ef[(lb + j) * CH + c] : 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) g[j][q] = ec[3 * (lb + j) + q];
      }
#pragma unroll
      for (int j = 0; j < L; ++j) {
        // bottom + top sums (2 xm, 2 ym) and the height; the factors 1/4
        // and 1/3 of |det J| live in the Kronecker factors (kron_fold12)
        gm[A][j][0] = g[j][0] + g[j + 1][0];
        gm[A][j][1] = g[j][1] + g[j + 1][1];
        gm[A][j][2] = g[j + 1][2] - g[j][2];
      }
      __syncwarp(); // reads done before the slot is refilled
      const int va = rv[R] & IDM;
      const int rv_cell = rv[R]; // before the slot is refilled
      yc[A] = col_at(PEER && va < ghost_end ? ylg : yl, va, colb);
      live[A] = act;
      st[A] = L == 1 && store && (rv[R] & PM_STEP_STORE);
      // interval stage of the entering vertex
#pragma unroll
      for (int j = 0; j < L; ++j)
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NV; ++w) {
              const double xw = LV == 0 ? f[j][w * NC + c]
                                : w == 0 ? f[j][c]
                                         : f[j + 1][c];
              s = fma(M.l[v * NV + w], xw, s);
            }
            zv[A][j][c][v] = s;
          }
      // refill ring slot A with the step kSrDepth ahead
      rv[R] = fetch(k + kSrDepth, R);
      if (FILL && A < 2) return; // window not full yet
#pragma unroll
      for (int j = 0; j < L; ++j) {
        // past the strip's end the window still holds two live vertices:
        // the step contributes nothing
        const double dj = prism_abs_detj_12(
            gm[0][j][0], gm[0][j][1], gm[0][j][2], gm[1][j][0], gm[1][j][1],
            gm[1][j][2], gm[2][j][0], gm[2][j][1], gm[2][j][2]);
        // (with L > 1 a lane's upper level may lie past a partial chunk;
        // its accumulator feeds the chunk's top level, so it must stay 0)
        const double det =
            (act && !(STREAM && (rv_cell & PM_STEP_NOCELL)) &&
             (L == 1 || lb + j < nl))
                ? dj
                : 0.0;
        // triangle stage, det folded into the accumulation
        if constexpr (CSUM) { // Mtri = ta I + tb J, cell ring slot A
          tr[A][j] = det * M.ta;
          const double dtb = det * M.tb;
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < NV; ++v)
              dr[A][j][c][v] = dtb * (zv[0][j][c][v] + zv[1][j][c][v] +
                                      zv[2][j][c][v]);
        } else if constexpr (SYM) { // Mtri = ta I + tb J
          const double dta = det * M.ta, dtb = det * M.tb;
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              const double d = dtb * (zv[0][j][c][v] + zv[1][j][c][v] +
                                      zv[2][j][c][v]);
#pragma unroll
              for (int h = 0; h < 3; ++h)
                acc[h][j][c][v] =
                    fma(dta, zv[h][j][c][v], acc[h][j][c][v] + d);
            }
        } else {
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
              for (int h = 0; h < 3; ++h) {
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < 3; ++q)
                  s = fma(M.t[h * 3 + q], zv[q][j][c][v], s);
                acc[h][j][c][v] = fma(det, s, acc[h][j][c][v]);
              }
        }
      }
    };
    using S0 = std::integral_constant<int, 0>;
    using S1 = std::integral_constant<int, 1>;
    using S2 = std::integral_constant<int, 2>;
    using TF = std::true_type;
    using FF = std::false_type;
    using S3 = std::integral_constant<int, 3>;
    using S4 = std::integral_constant<int, 4>;
    using S5 = std::integral_constant<int, 5>;
    int kb = 0;
    if constexpr (!STREAM) {
      step(S0{}, S0{}, TF{}, 0);
      step(S1{}, S1{}, TF{}, 1);
      step(S2{}, S2{}, TF{}, 2);
      kb = 3;
    }
    if constexpr (kSrDepth == 3) {
      for (int k = kb; k < maxlen; k += 3) {
        step(S0{}, S0{}, FF{}, k);
        step(S1{}, S1{}, FF{}, k + 1);
        step(S2{}, S2{}, FF{}, k + 2);
      }
    } else if constexpr (!STREAM) { // ring slots 3,4,5,0,1,2 from k = 3
      for (int k = kb; k < maxlen; k += 6) {
        step(S0{}, S3{}, FF{}, k);
        step(S1{}, S4{}, FF{}, k + 1);
        step(S2{}, S5{}, FF{}, k + 2);
        step(S0{}, S0{}, FF{}, k + 3);
        step(S1{}, S1{}, FF{}, k + 4);
        step(S2{}, S2{}, FF{}, k + 5);
      }
    } else {
      for (int k = kb; k < maxlen; k += 6) {
        step(S0{}, S0{}, FF{}, k);
        step(S1{}, S1{}, FF{}, k + 1);
        step(S2{}, S2{}, FF{}, k + 2);
        step(S0{}, S3{}, FF{}, k + 3);
        step(S1{}, S4{}, FF{}, k + 4);
        step(S2{}, S5{}, FF{}, k + 5);
      }
    }
    // the last window: vertex k in slot 1 / 2 has no cell k+... past the
    // loop, so the ring slots of cells it was not in are cleared first
    auto clear_cell = [&](auto A_) {
      constexpr int A = decltype(A_)::value;
      if constexpr (CSUM) {
#pragma unroll
        for (int j = 0; j < L; ++j) {
          tr[A][j] = 0.0;
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < NV; ++v) dr[A][j][c][v] = 0.0;
        }
      }
    };
    flush(S0{});
    clear_cell(S0{});
    __syncwarp(); // (DEFER: each flush's staged row before the next's LDS)
    flush(S1{});
    clear_cell(S1{});
    __syncwarp();
    flush(S2{});
    clear_cell(S2{});
    if constexpr (DEFER) { // the last staged row
      __syncwarp();
      const double *prow = trow0 + (tb ^ 1) * TR;
#pragma unroll
      for (int r = 0; r < (TR + W - 1) / W; ++r) {
        const int i = sl + W * r;
        (PEER ? sr_red_sys : sr_red)(pbase + i, prow[i < TR ? i : 0],
                                     plive && i < nl * CH + LV);
      }
      __syncwarp(); // row reads done before the next item stages
    }
    sr_wait<0>(); // no copy in flight into the ring across items
  }
  if constexpr (PEER) __threadfence_system(); // peer REDs land before exit
}

// CTAs per SM in the strip kernels' grid-stride grid (PM_STRIP_GRID tuning
// knob; default `def`)
static int strip_grid_cap(int def) {
  const char *e = getenv("PM_STRIP_GRID");
  const int v = e ? atoi(e) : 0;
  return v > 0 ? v : def;
}

// levels per lane (PM_STRIP_L tuning knob: 1 or 2)
static int strip_levels() {
  const char *e = getenv("PM_STRIP_L");
  return e && atoi(e) == 2 ? 2 : 1;
}

template <class LY, int W, bool SYM, int L, bool PEER = false,
          bool STREAM = false>
static int strip_red_launch(const LoopArgs &a, const KronMat &M,
                            const int32_t *strip_ptr, const int32_t *steps,
                            int64_t n_strips) {
  const int segs = 32 / W;
  const int64_t items =
      n_strips * ((a.lend - a.lbeg + W * L - 1) / (W * L));
  const int64_t warps = (items + segs - 1) / segs;
  constexpr int T = sr_threads<LY>();
  const unsigned grid = grid_for(warps * 32, T, strip_grid_cap(8));
  const size_t smem = sr_smem<LY, W, L>();
  static int cached_dev = -1; // attribute set once per device
  int dev = 0;
  PM_CUDA_TRY(cudaGetDevice(&dev));
  if (cached_dev != dev) {
    PM_CUDA_TRY(cudaFuncSetAttribute(
        k_strip_red<LY, W, SYM, L, PEER, STREAM>,
        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cached_dev = dev;
  }
  k_strip_red<LY, W, SYM, L, PEER, STREAM><<<grid, T, smem, a.s>>>(
      M, a.item_ptr, strip_ptr, steps, n_strips, a.layers, a.lbeg, a.lend,
      a.coords, a.x, a.y,
      a.y_peer, (int)a.ghost_end, a.store);
  PM_LAUNCH_CHECK("k_strip_red");
  return PM_OK;
}

template <class LY, int W>
static int strip_red_w(const LoopArgs &a, const KronMat &M, bool sym,
                       int L, const int32_t *strip_ptr, const int32_t *steps,
                       int64_t n_strips) {
  if (a.y_peer) { // fused halo
    if (sym)
      return strip_red_launch<LY, W, true, 1, true>(a, M, strip_ptr, steps,
                                                    n_strips);
    return strip_red_launch<LY, W, false, 1, true>(a, M, strip_ptr, steps,
                                                   n_strips);
  }
  if (a.item_ptr) { // store-first patch strips: one level per lane
#if PM_EXPERIMENTAL
    if (sym)
      return strip_red_launch<LY, W, true, 1, false, true>(a, M, strip_ptr,
                                                           steps, n_strips);
    return strip_red_launch<LY, W, false, 1, false, true>(a, M, strip_ptr,
                                                          steps, n_strips);
#else
    set_error("patch strips are experimental: rebuild with PM_EXPERIMENTAL=1");
    return PM_EINVAL;
#endif
  }
  if constexpr (LY::CH0 <= 2 && W <= 16) {
    if (L == 2 && sym)
      return strip_red_launch<LY, W, true, 2>(a, M, strip_ptr, steps,
                                              n_strips);
  }
  if (sym)
    return strip_red_launch<LY, W, true, 1>(a, M, strip_ptr, steps, n_strips);
  return strip_red_launch<LY, W, false, 1>(a, M, strip_ptr, steps, n_strips);
}

template <class LY>
static int strip_red_k1(const LoopArgs &a, const int32_t *strip_ptr,
                        const int32_t *steps, int64_t n_strips, int W);

template <class LY>
static int strip_red_k(const LoopArgs &a0, const int32_t *strip_ptr,
                       const int32_t *steps, int64_t n_strips, int chunk) {
  LoopArgs a = a0; // one launch over all levels (lbeg / lend: strip_red_k1)
  a.lbeg = 0;
  a.lend = a0.layers;
  return strip_red_k1<LY>(a, strip_ptr, steps, n_strips, chunk);
}

template <class LY>
static int strip_red_k1(const LoopArgs &a, const int32_t *strip_ptr,
                        const int32_t *steps, int64_t n_strips, int W) {
  if (!a.mtri || !a.mline) {
    set_error("the strip kernel needs the Kronecker factors mtri/mline");
    return PM_EINVAL;
  }
  KronMat M;
  for (int i = 0; i < LY::NH * LY::NH; ++i) M.t[i] = a.mtri[i];
  for (int i = 0; i < LY::NV * LY::NV; ++i) M.l[i] = a.mline[i];
  const bool sym = kron_sym3(M);
  kron_fold12(M);
  const int L = strip_levels();
  switch (W) {
  case 32: return strip_red_w<LY, 32>(a, M, sym, L, strip_ptr, steps, n_strips);
  case 16: return strip_red_w<LY, 16>(a, M, sym, L, strip_ptr, steps, n_strips);
  case 8: return strip_red_w<LY, 8>(a, M, sym, L, strip_ptr, steps, n_strips);
  default:
    set_error("strip chunk width must be 8, 16 or 32 (got %d)", W);
    return PM_EINVAL;
  }
}


// ---------------------------------------------------------------------------
// Vertex + edge layouts (P2 x P2): the window also holds the three edges,
// edge slot a opposite window vertex a.  A step replacing vertex slot s
// keeps edge slot s (the shared edge) and brings in the two new edges for
// slots s+1, s+2, so each cell costs one vertex + two edge column loads and
// three partial flushes (against six gathers / six scatters per cell-layer
// for the column kernel).
// ---------------------------------------------------------------------------
template <class LY, int W> constexpr int sre_fs0() { return W * LY::CH0 + LY::LV0; }
template <class LY, int W> constexpr int sre_fs1() { return W * LY::CH1 + LY::LV1; }
template <class LY, int W> constexpr int sre_trow() {
  return PM_SR_TROW ? (W + 1) * (LY::NV - 1) : 0;
}
template <class LY, int W> constexpr int sre_entry() {
  return sre_fs0<LY, W>() + 3 * (W + 1) + 2 * sre_fs1<LY, W>();
}

// CTA size of the P2 kernel: 384 threads (12 warps at <= 168 registers)
// with the block-structured triangle factor, 256 with a general one (it
// spills at 168: measured 8 % slower)
template <bool SYM> constexpr int sre_threads() { return SYM ? 384 : 256; }

template <class LY, int W, bool SYM, bool STREAM = false, int K = LY::K>
__global__ void __launch_bounds__(sre_threads<SYM>(), 1)
k_strip_red_e(const KronMat M, const int32_t *__restrict__ item_ptr,
              const int32_t *__restrict__ strip_ptr,
              const int32_t *__restrict__ steps,
              const int32_t *__restrict__ steps_e, int64_t n_groups,
              int layers, int lbeg, int lend, int64_t e_start,
              const double *__restrict__ coords,
              const double *__restrict__ x, double *__restrict__ y,
              int store) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int IDM = STREAM ? kIdMask : -1; // flag bits only in STREAM mode
  constexpr int SEGS = 32 / W;
  constexpr int LV0 = LY::LV0, CH0 = LY::CH0, LV1 = LY::LV1, CH1 = LY::CH1;
  constexpr int NV = LY::NV;
  static_assert(LY::NH == 6 && LY::NC == 1 && LV0 == 1 && LV1 == 1 &&
                    CH0 == NV - 1 && CH1 == NV - 1,
                "P2-type layout: level copies + NV-2 connecting functions");
  constexpr int kSreWarps = sre_threads<SYM>() / 32;
  constexpr int FS0 = sre_fs0<LY, W>(), FS1 = sre_fs1<LY, W>();
  constexpr int ES = sre_entry<LY, W>();
  constexpr int OC = FS0, OE1 = FS0 + 3 * (W + 1), OE2 = OE1 + FS1;
  const int lane = threadIdx.x & 31;
  const int sl = lane % W, seg = lane / W;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // column lengths in bytes fit 32 bits: a column origin is one IMAD.WIDE
  const int col0 = 8 * (layers * CH0 + LV0);
  const int col1 = 8 * (layers * CH1 + LV1);
  const int ccol = 8 * 3 * (layers + 1);
  extern __shared__ double sr_ring[];
  double *ring =
      sr_ring + (size_t)(threadIdx.x >> 5) * kSrDepth * SEGS * ES;
  const double *sr_zero = sr_ring + (size_t)kSreWarps * kSrDepth * SEGS * ES;
  // the strip's vertex and edge ids, staged kSrIds steps at a time
  int *const sid = reinterpret_cast<int *>(
                       sr_ring + (size_t)(kSreWarps * kSrDepth * SEGS + 1) * ES) +
                   ((threadIdx.x >> 5) * SEGS + (threadIdx.x & 31) / W) * 3 *
                       kSrIds;
  // flush staging row (see sr_trow): the entity chunk's (W + 1) * (NV - 1)
  // values, added with lane-contiguous REDs (level copies and mid values
  // alternate in the column: per-lane REDs run at a 16-byte stride)
  constexpr int TR = sre_trow<LY, W>();
  // PM_SR_DEFER: two staging rows, REDs one flush late (see k_strip_red)
  constexpr bool DEFER = TR > 0 && PM_SR_DEFER && !STREAM;
  double *const trow0 =
      reinterpret_cast<double *>(
          reinterpret_cast<int *>(sr_ring + (size_t)(kSreWarps * kSrDepth *
                                                         SEGS + 1) * ES) +
          kSreWarps * SEGS * 3 * kSrIds) +
      ((threadIdx.x >> 5) * SEGS + (threadIdx.x & 31) / W) * TR *
          kSrTrowBufs;
  // the zero block; in STREAM mode the whole ring (dead edge slots read
  // stale ring entries, which must be finite)
  for (int i = threadIdx.x; i < (STREAM ? kSreWarps * kSrDepth * SEGS + 1 : 1) * ES;
       i += blockDim.x)
    sr_ring[(size_t)(STREAM ? 0 : kSreWarps * kSrDepth * SEGS * ES) + i] = 0.0;
  __syncthreads();

  // items = (group, chunk) as in k_strip_red: a group is one global strip
  // or the strips of a patch
  const int n_chunks = (lend - lbeg + W - 1) / W; // levels [lbeg, lend)
  const int64_t n_items = n_groups * n_chunks;
  for (int64_t i0 = warp * SEGS; i0 < n_items; i0 += n_warps * SEGS) {
    const int64_t item = i0 + seg;
    const bool has = item < n_items;
    const int64_t gi = has ? item / n_chunks : 0;
    const int l0 = has ? lbeg + (int)(item % n_chunks) * W : 0;
    // one contiguous step range per group; STREAM (patch strips): strips
    // follow each other, every step in normal form (fill steps bring the
    // first cell's edges with -1 = none, see pm_build_patch_strips)
    const int64_t gs = item_ptr ? __ldg(item_ptr + gi) : gi;
    const int64_t ge = item_ptr ? __ldg(item_ptr + gi + 1) : gi + 1;
    const int k0 = has ? __ldg(strip_ptr + gs) : 0;
    const int len = has ? __ldg(strip_ptr + ge) - k0 : 0;
    int maxlen = len;
#pragma unroll
    for (int o = W; o < 32; o <<= 1)
      maxlen = max(maxlen, __shfl_xor_sync(FULL, maxlen, o));
    const int nl = has ? min(W, lend - l0) : 0;
    // store-first: the chunk's bottom level copy is shared with the chunk
    // below, its top with the chunk above (both cleared by the zero pass)
    const bool lane_ok = sl < nl;
    // flush-mode masks (sr_put): mid values, bottom and top level copies
    const int mmask = lane_ok ? kPutStore : 0;
    const int bmask = !lane_ok ? 0 : (sl > 0 || l0 == 0) ? kPutStore : kPutAdd;
    const int tmask = sl != nl - 1 ? 0 : l0 + nl == layers ? kPutStore : kPutAdd;
    const int fl0 = nl * CH0 + LV0, fl1 = nl * CH1 + LV1, cl = 3 * (nl + 1);
    // the segment's chunk of every column (copies) and the lane's element
    // (flushes)
    const double *xv0 = x + (int64_t)l0 * CH0;
    const double *xe0 = x + e_start + (int64_t)l0 * CH1;
    const double *cc0 = coords + 3 * (int64_t)l0;
    double *yv0 = y + ((int64_t)l0 + sl) * CH0;
    double *ye0 = y + e_start + ((int64_t)l0 + sl) * CH1;

    // window: per vertex / edge the interval stage z[v] = (Mline x)[v] at
    // the lane's cell-layer, per vertex the Jacobian geometry (xm, ym, dz);
    // accumulators per entity and interval function
    double zv[3][NV], ze[3][NV], gm[3][3], av[3][NV], ae[3][NV];
    double *yvc[3] = {yv0, yv0, yv0}, *yec[3] = {ye0, ye0, ye0};
    // flush mode per window slot (sr_put: 0 empty, 1 add, 3 store first)
    int vm[3] = {0, 0, 0}, em[3] = {0, 0, 0};
    // DEFER: staging row in use, the previous row's origin and mode
    int tb = 0, pm_ = 0;
    double *pbase = y;
    auto mode = [&](bool live, int id) {
      return !live ? 0 : (store && (id & PM_STEP_STORE)) ? kPutStore : kPutAdd;
    };
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int v = 0; v < NV; ++v)
        zv[a][v] = 0.0, ze[a][v] = 0.0, av[a][v] = 0.0, ae[a][v] = 0.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) gm[a][q] = 0.0;
    }
    auto load_ids = [&](int base) {
#pragma unroll
      for (int r = 0; r < kSrIds / W; ++r) {
        const int j = sl + W * r, i = base + j;
        const bool ok = i < len;
        sid[j] = ok ? __ldg(steps + k0 + i) : 0;
        sid[kSrIds + 2 * j] = ok ? __ldg(steps_e + 2 * (k0 + i)) : 0;
        sid[kSrIds + 2 * j + 1] = ok ? __ldg(steps_e + 2 * (k0 + i) + 1) : 0;
      }
      __syncwarp();
    };
    __syncwarp(); // the previous item's last id reads are done
    load_ids(0);
    auto entry = [&](int slot) {
      return ring + (size_t)(slot * SEGS + seg) * ES;
    };
    int rv[kSrDepth], re1[kSrDepth], re2[kSrDepth];
    auto seg_copy = [&](double *dst, const double *src, int n, int cap) {
#pragma unroll
      for (int r = 0; r < (cap + W - 1) / W; ++r) {
        const int i = sl + W * r;
        if (i < n) sr_cp8(dst + i, src + i);
      }
    };
    auto fetch = [&](int k, int slot) {
      if ((k & (kSrIds - 1)) == 0 && k > 0) { // warp-uniform
        __syncwarp();
        load_ids(k);
      }
      const int j = k & (kSrIds - 1);
      const int v = sid[j];
      const int e1 = sid[kSrIds + 2 * j], e2 = sid[kSrIds + 2 * j + 1];
      if (k < len) {
        double *en = entry(slot);
        seg_copy(en, col_at(xv0, v & IDM, col0), fl0, FS0);
        seg_copy(en + OC, col_at(cc0, v & IDM, ccol), cl, 3 * (W + 1));
        if (!STREAM || e1 >= 0)
          seg_copy(en + OE1, col_at(xe0, e1 & IDM, col1), fl1, FS1);
        if (STREAM ? e2 >= 0 : k >= 3)
          seg_copy(en + OE2, col_at(xe0, e2 & IDM, col1), fl1, FS1);
      }
      sr_commit();
      rv[slot] = v, re1[slot] = e1, re2[slot] = e2;
    };
#pragma unroll
    for (int d = 0; d < kSrDepth; ++d) fetch(d, d);

    // flush an entity residency: accumulators back to the layer block
    // (bottom copy v = 0, connecting v = 1..NV-2, top copy v = NV-1 added
    // one lane up; the chunk's top level by the last lane)
    auto flush = [&](double (&acc)[NV], double *yp, int m) {
      double *const trow = trow0 + (DEFER ? tb * TR : 0);
      constexpr int NR = TR > 0 ? (TR + W - 1) / W : 1;
      double pv[NR];
      if constexpr (DEFER) { // the previous row (staged, synced)
        const double *prow = trow0 + (tb ^ 1) * TR;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const int i = sl + W * r;
          pv[r] = prow[i < TR ? i : 0];
        }
      }
      const double below = __shfl_up_sync(FULL, acc[NV - 1], 1, W);
      if constexpr (STREAM && TR == 0) { // store-first patch strips
        sr_put(yp, sl > 0 ? acc[0] + below : acc[0], m & bmask);
#pragma unroll
        for (int v = 1; v < NV - 1; ++v) sr_put(yp + v, acc[v], m & mmask);
        sr_put(yp + (NV - 1), acc[NV - 1], m & tmask);
      } else if constexpr (TR > 0) {
        // (lanes past the chunk stay out: their first slot is the top)
        if (lane_ok) {
          trow[sl * (NV - 1)] = sl > 0 ? acc[0] + below : acc[0];
#pragma unroll
          for (int v = 1; v < NV - 1; ++v) trow[sl * (NV - 1) + v] = acc[v];
        }
        if (sl == nl - 1) trow[(sl + 1) * (NV - 1)] = acc[NV - 1];
        double *const base = yp - sl * (NV - 1); // the chunk's first value
        const int n = nl * (NV - 1) + 1;
        if constexpr (DEFER) {
          // the previous row's REDs; this row's at the next flush, after
          // the barrier below orders this STS before those LDS
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            const int i = sl + W * r;
            sr_red(pbase + i, pv[r], pm_ && i < n);
          }
          pbase = base;
          pm_ = m;
          tb ^= 1;
          __syncwarp();
        } else {
        __syncwarp();
        if constexpr (STREAM) { // store-first (m = 3): shared level copies add
          const int lo = l0 > 0 ? 1 : 0, hi = l0 + nl < layers ? n - 1 : n;
#pragma unroll
          for (int r = 0; r < (TR + W - 1) / W; ++r) {
            const int i = sl + W * r;
            sr_put(base + i, trow[i < TR ? i : 0],
                   i >= n ? 0 : (i < lo || i >= hi) ? (m & kPutAdd) : m);
          }
        } else {
#pragma unroll
          for (int r = 0; r < (TR + W - 1) / W; ++r) {
            const int i = sl + W * r;
            sr_red(base + i, trow[i < TR ? i : 0], m && i < n);
          }
        }
        __syncwarp(); // row reads done before the next flush stages
        }
      } else if (m && lane_ok) {
        atomicAdd(yp, sl > 0 ? acc[0] + below : acc[0]);
#pragma unroll
        for (int v = 1; v < NV - 1; ++v) atomicAdd(yp + v, acc[v]);
        if (sl == nl - 1) atomicAdd(yp + (NV - 1), acc[NV - 1]);
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[v] = 0.0;
    };
    // interval stage of an entering entity from its layer block in the ring
    auto enter = [&](double (&z)[NV], const double *src) {
      double b[NV];
#pragma unroll
      for (int v = 0; v < NV - 1; ++v) b[v] = src[sl * (NV - 1) + v];
      b[NV - 1] = src[(sl + 1) * (NV - 1)];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NV; ++w) s = fma(M.l[v * NV + w], b[w], s);
        z[v] = s;
      }
    };
    // one strip step into vertex slot A; FILL: edge slot A, else the edge
    // slots A+1, A+2
    auto step = [&](auto A_, auto R_, auto FILL_, int k) {
      constexpr int A = decltype(A_)::value; // window slot (k % 3)
      constexpr int R = decltype(R_)::value; // ring slot (k % kSrDepth)
      constexpr bool FILL = decltype(FILL_)::value;
      constexpr int B1 = (A + 1) % 3, B2 = (A + 2) % 3;
      flush(av[A], yvc[A], vm[A]);
      if (FILL) {
        flush(ae[A], yec[A], em[A]);
      } else {
        flush(ae[B1], yec[B1], em[B1]);
        flush(ae[B2], yec[B2], em[B2]);
      }
      const bool act = k < len;
      sr_wait<kSrDepth - 1>();
      __syncwarp();
      // past the strip's end: read the zero block (contribution exactly 0)
      const double *en = act ? entry(R) : sr_zero;
      enter(zv[A], en);
      {
        const double *g = en + OC + 3 * sl;
        gm[A][0] = g[0] + g[3]; // bottom + top sums and the height:
        gm[A][1] = g[1] + g[4]; // 12 |det J| (prism_abs_detj_12)
        gm[A][2] = g[5] - g[2];
      }
      yvc[A] = col_at(yv0, rv[R] & IDM, col0);
      vm[A] = mode(act, rv[R]);
      if (FILL) {
        enter(ze[A], en + OE1);
        yec[A] = col_at(ye0, re1[R] & IDM, col1);
        em[A] = mode(act, re1[R]);
      } else {
        // STREAM: an edge id -1 (fill steps) leaves the slot dead: nothing
        // flushed; its stale ring values (finite: the ring starts zeroed)
        // only meet NOCELL steps (det = 0)
        enter(ze[B1], en + OE1);
        yec[B1] = col_at(ye0, re1[R] & IDM, col1);
        em[B1] = mode(act && (!STREAM || re1[R] >= 0), re1[R]);
        enter(ze[B2], en + OE2);
        yec[B2] = col_at(ye0, re2[R] & IDM, col1);
        em[B2] = mode(act && (!STREAM || re2[R] >= 0), re2[R]);
      }
      const int rv_cell = rv[R]; // before the slot is refilled
      __syncwarp();
      fetch(k + kSrDepth, R);
      if (FILL && A < 2) return; // window not full yet
      // lanes past the chunk are never flushed; past the strip's end the
      // window still holds live entities: no contribution
      const double dj = prism_abs_detj_12(gm[0][0], gm[0][1], gm[0][2],
                                           gm[1][0], gm[1][1], gm[1][2],
                                           gm[2][0], gm[2][1], gm[2][2]);
      const double det =
          (act && !(STREAM && (rv_cell & PM_STEP_NOCELL))) ? dj : 0.0;
      // triangle stage (h: vertices 0-2, edges 3-5), det folded into the
      // accumulation
      if constexpr (SYM) { // block form a I + b J (KronMat::p)
        const double da1 = det * M.p[0], da2 = det * M.p[1];
        const double dc1 = det * M.p[2], dc2 = det * M.p[3];
        const double dbm = det * M.p[4], db2 = det * M.p[5];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double sv = zv[0][v] + zv[1][v] + zv[2][v];
          const double se = ze[0][v] + ze[1][v] + ze[2][v];
          const double tv = fma(da2, sv, db2 * se);
          const double te = fma(db2, sv, dc2 * se);
#pragma unroll
          for (int h = 0; h < 3; ++h) {
            av[h][v] = fma(da1, zv[h][v], fma(dbm, ze[h][v], av[h][v] + tv));
            ae[h][v] = fma(dbm, zv[h][v], fma(dc1, ze[h][v], ae[h][v] + te));
          }
        }
      } else {
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int h = 0; h < 6; ++h) {
            double s = 0.0;
#pragma unroll
            for (int g = 0; g < 3; ++g) s = fma(M.t[h * 6 + g], zv[g][v], s);
#pragma unroll
            for (int g = 0; g < 3; ++g)
              s = fma(M.t[h * 6 + 3 + g], ze[g][v], s);
            if (h < 3)
              av[h][v] = fma(det, s, av[h][v]);
            else
              ae[h - 3][v] = fma(det, s, ae[h - 3][v]);
          }
      }
    };
    using S0 = std::integral_constant<int, 0>;
    using S1 = std::integral_constant<int, 1>;
    using S2 = std::integral_constant<int, 2>;
    using TF = std::true_type;
    using FF = std::false_type;
    using S3 = std::integral_constant<int, 3>;
    using S4 = std::integral_constant<int, 4>;
    using S5 = std::integral_constant<int, 5>;
    int kb = 0;
    if constexpr (!STREAM) {
      step(S0{}, S0{}, TF{}, 0);
      step(S1{}, S1{}, TF{}, 1);
      step(S2{}, S2{}, TF{}, 2);
      kb = 3;
    }
    if constexpr (kSrDepth == 3) {
      for (int k = kb; k < maxlen; k += 3) {
        step(S0{}, S0{}, FF{}, k);
        step(S1{}, S1{}, FF{}, k + 1);
        step(S2{}, S2{}, FF{}, k + 2);
      }
    } else if constexpr (!STREAM) { // ring slots 3,4,5,0,1,2 from k = 3
      for (int k = kb; k < maxlen; k += 6) {
        step(S0{}, S3{}, FF{}, k);
        step(S1{}, S4{}, FF{}, k + 1);
        step(S2{}, S5{}, FF{}, k + 2);
        step(S0{}, S0{}, FF{}, k + 3);
        step(S1{}, S1{}, FF{}, k + 4);
        step(S2{}, S2{}, FF{}, k + 5);
      }
    } else {
      for (int k = kb; k < maxlen; k += 6) {
        step(S0{}, S0{}, FF{}, k);
        step(S1{}, S1{}, FF{}, k + 1);
        step(S2{}, S2{}, FF{}, k + 2);
        step(S0{}, S3{}, FF{}, k + 3);
        step(S1{}, S4{}, FF{}, k + 4);
        step(S2{}, S5{}, FF{}, k + 5);
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      flush(av[a], yvc[a], vm[a]);
      flush(ae[a], yec[a], em[a]);
    }
    if constexpr (DEFER) { // the last staged row (synced by its flush)
      const double *prow = trow0 + (tb ^ 1) * TR;
      const int n = nl * (NV - 1) + 1;
#pragma unroll
      for (int r = 0; r < (TR + W - 1) / W; ++r) {
        const int i = sl + W * r;
        sr_red(pbase + i, prow[i < TR ? i : 0], pm_ && i < n);
      }
      pm_ = 0;
      __syncwarp(); // row reads done before the next item stages
    }
    sr_wait<0>(); // no copy in flight into the ring across items
  }
}

template <class LY>
static int strip_red_e_k1(const LoopArgs &a, const int32_t *strip_ptr,
                          const int32_t *steps, const int32_t *steps_e,
                          int64_t n_strips, int W, int64_t e_start);

template <class LY>
static int strip_red_e_k(const LoopArgs &a0, const int32_t *strip_ptr,
                         const int32_t *steps, const int32_t *steps_e,
                         int64_t n_strips, int chunk, int64_t e_start) {
  LoopArgs a = a0;
  a.lbeg = 0;
  a.lend = a0.layers;
  return strip_red_e_k1<LY>(a, strip_ptr, steps, steps_e, n_strips, chunk,
                            e_start);
}

template <class LY>
static int strip_red_e_k1(const LoopArgs &a, const int32_t *strip_ptr,
                          const int32_t *steps, const int32_t *steps_e,
                          int64_t n_strips, int W, int64_t e_start) {
  if (!a.mtri || !a.mline) {
    set_error("the strip kernel needs the Kronecker factors mtri/mline");
    return PM_EINVAL;
  }
  if (!steps_e) {
    set_error("edge layouts need the strips' edge records (steps_e)");
    return PM_EINVAL;
  }
  KronMat M;
  for (int i = 0; i < LY::NH * LY::NH; ++i) M.t[i] = a.mtri[i];
  for (int i = 0; i < LY::NV * LY::NV; ++i) M.l[i] = a.mline[i];
  const int segs = 32 / W;
  const int64_t items = n_strips * ((a.lend - a.lbeg + W - 1) / W);
  const int64_t warps = (items + segs - 1) / segs;
  const bool sym = kron_sym6(M);
  kron_fold12(M);
#define PM_SRE(WW)                                                           \
  do {                                                                       \
    if (sym)                                                                 \
      PM_SRE2(WW, true);                                                     \
    else                                                                     \
      PM_SRE2(WW, false);                                                    \
  } while (0)
#if PM_EXPERIMENTAL
#define PM_SRE2(WW, SS)                                                      \
  do {                                                                       \
    if (a.item_ptr)                                                          \
      PM_SRE3(WW, SS, true);                                                 \
    else                                                                     \
      PM_SRE3(WW, SS, false);                                                \
  } while (0)
#else
#define PM_SRE2(WW, SS)                                                      \
  do {                                                                       \
    if (a.item_ptr) {                                                        \
      set_error("patch strips are experimental: rebuild with "              \
                "PM_EXPERIMENTAL=1");                                        \
      return PM_EINVAL;                                                      \
    }                                                                        \
    PM_SRE3(WW, SS, false);                                                  \
  } while (0)
#endif
#define PM_SRE3(WW, SS, ST)                                                  \
  do {                                                                       \
    constexpr int T = sre_threads<SS>(), NW = T / 32;                        \
    const unsigned grid = grid_for(warps * 32, T, strip_grid_cap(4));        \
    const size_t smem = sizeof(double) * (NW * kSrDepth * (32 / WW) + 1) *   \
                            sre_entry<LY, WW>() +                            \
                        sizeof(int) * NW * (32 / WW) * 3 * kSrIds +          \
                        sizeof(double) * NW * (32 / WW) * sre_trow<LY, WW>() *  \
                            kSrTrowBufs;                                     \
    static int attr_dev = -1; /* attribute set once per device */           \
    int dev_ = 0;                                                            \
    PM_CUDA_TRY(cudaGetDevice(&dev_));                                       \
    if (attr_dev != dev_) {                                                  \
      PM_CUDA_TRY(cudaFuncSetAttribute(                                      \
          k_strip_red_e<LY, WW, SS, ST>,                                     \
          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));          \
      attr_dev = dev_;                                                       \
    }                                                                        \
    k_strip_red_e<LY, WW, SS, ST><<<grid, T, smem, a.s>>>(                   \
        M, a.item_ptr, strip_ptr, steps, steps_e, n_strips, a.layers,        \
        a.lbeg, a.lend, e_start, a.coords, a.x, a.y, a.store);                               \
  } while (0)
  if (W == 32)
    PM_SRE(32);
  else if (W == 16)
    PM_SRE(16);
  else if (W == 8)
    PM_SRE(8);
  else {
    set_error("strip chunk width must be 8, 16 or 32 (got %d)", W);
    return PM_EINVAL;
  }
#undef PM_SRE
#undef PM_SRE2
#undef PM_SRE3
  PM_LAUNCH_CHECK("k_strip_red_e");
  return PM_OK;
}

#define PM_STRIPRED_LAYOUTS(X)                                               \
  X(1, 0, 0, 0, 0, 0)                                                        \
  X(0, 1, 0, 0, 0, 0)                                                        \
  X(0, 2, 0, 0, 0, 0)                                                        \
  X(3, 0, 0, 0, 0, 0)

// Zero pass of the store-first patch strips: the columns of the entities
// several patches touch (warp per entity, coalesced) ...
__global__ void k_zero_entities(double *__restrict__ y,
                                const int32_t *__restrict__ zero_list,
                                int64_t n_zero, int64_t n_vertices, int colv,
                                int cole, int64_t e_start) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n_zero; i += n_warps) {
    const int64_t e = __ldg(zero_list + i);
    double *col = e < n_vertices ? y + e * colv
                                 : y + e_start + (e - n_vertices) * cole;
    const int n = e < n_vertices ? colv : cole;
    for (int j = lane; j < n; j += 32) col[j] = 0.0;
  }
}

// ... and every column's level copies on the layer-chunk boundaries (the
// top of one chunk item, the bottom of the next: both add)
__global__ void k_zero_chunk_levels(double *__restrict__ y, int64_t n_vertices,
                                    int64_t n_edges, int colv, int cole,
                                    int64_t e_start, int ch0, int lv0, int ch1,
                                    int lv1, int cw, int nb) {
  const int64_t nv = n_vertices * nb * lv0, ne = n_edges * nb * lv1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nv + ne;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t < nv) {
      const int64_t ent = t / (nb * lv0);
      const int r = (int)(t - ent * nb * lv0);
      y[ent * colv + (int64_t)(r / lv0 + 1) * cw * ch0 + r % lv0] = 0.0;
    } else {
      const int64_t u = t - nv, ent = u / (nb * lv1);
      const int r = (int)(u - ent * nb * lv1);
      y[e_start + ent * cole + (int64_t)(r / lv1 + 1) * cw * ch1 + r % lv1] =
          0.0;
    }
  }
}

// ---------------------------------------------------------------------------
// DG layouts along strips (pm_column_mass_strip_dg): the DG stream kernel
// gathers every cell-layer's six prism vertices' coordinates through the
// coordinate map, which dominates its L1 traffic when a cell-layer holds
// few DoFs (DG0 x DG0: one).  Walking the cells as the CG strips do, a step
// brings one new vertex's coordinate chunk (the window keeps the other two)
// and the formed cell's field chunk, both by cp.async into the per-warp
// ring; the element kernel runs per lane (= layer) and the cell's D values
// per cell-layer are stored directly: every DoF belongs to one cell-layer,
// so there is no accumulation, no output zeroing and no atomics.
// step_cells[i] = the cell step i forms (-1 on a strip's two fill steps,
// pm_strip_step_cells).
// ---------------------------------------------------------------------------
template <int D, int W> constexpr int sd_crows() {
  return (3 * (W + 1) + W - 1) / W;
}
template <int D, int W> constexpr int sd_entry() {
  return (sd_crows<D, W>() + D) * W;
}
constexpr int kSdThreads = 256;

template <int D, int W>
__global__ void __launch_bounds__(kSdThreads, 3)
k_strip_dg(const MassMat<D> M, const int32_t *__restrict__ strip_ptr,
           const int32_t *__restrict__ steps,
           const int32_t *__restrict__ step_cells, int64_t n_strips,
           int layers, const double *__restrict__ coords,
           const double *__restrict__ x, double *__restrict__ y) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int SEGS = 32 / W;
  constexpr int CR = sd_crows<D, W>(), ES = sd_entry<D, W>();
  constexpr int CP = D * W; // coordinate part offset in an entry
  constexpr int NWARP = kSdThreads / 32;
  const int lane = threadIdx.x & 31;
  const int sl = lane % W, seg = lane / W;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int ccolb = 8 * 3 * (layers + 1); // coordinate column bytes
  extern __shared__ double sd_ring[];
  double *const ring =
      sd_ring + (size_t)(threadIdx.x >> 5) * kSrDepth * SEGS * ES;
  const double *const zero = sd_ring + (size_t)NWARP * kSrDepth * SEGS * ES;
  int *const sid = reinterpret_cast<int *>(sd_ring + (size_t)(NWARP * kSrDepth *
                                                              SEGS + 1) * ES) +
                   ((threadIdx.x >> 5) * SEGS + seg) * 2 * kSrIds;
  int *const scid = sid + kSrIds;
  for (int i = threadIdx.x; i < ES; i += blockDim.x)
    sd_ring[(size_t)NWARP * kSrDepth * SEGS * ES + i] = 0.0;
  __syncthreads();

  const int n_chunks = (layers + W - 1) / W;
  const int64_t n_items = n_strips * n_chunks;
  for (int64_t i0 = warp * SEGS; i0 < n_items; i0 += n_warps * SEGS) {
    const int64_t item = i0 + seg;
    const bool has = item < n_items;
    const int64_t s = has ? item / n_chunks : 0;
    const int l0 = has ? (int)(item % n_chunks) * W : 0;
    const int k0 = has ? __ldg(strip_ptr + s) : 0;
    const int len = has ? __ldg(strip_ptr + s + 1) - k0 : 0;
    int maxlen = len;
#pragma unroll
    for (int o = W; o < 32; o <<= 1)
      maxlen = max(maxlen, __shfl_xor_sync(FULL, maxlen, o));
    const int nl = has ? min(W, layers - l0) : 0;
    int cz[CR];
#pragma unroll
    for (int r = 0; r < CR; ++r) cz[r] = sl + W * r < 3 * (nl + 1) ? 8 : 0;
    const double *cl0 = coords + 3 * (int64_t)l0 + sl;
    double gm[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int q = 0; q < 3; ++q) gm[a][q] = 0.0;
    auto load_ids = [&](int base) {
#pragma unroll
      for (int r = 0; r < kSrIds / W; ++r) {
        const int i = base + sl + W * r;
        sid[sl + W * r] = i < len ? __ldg(steps + k0 + i) : 0;
        scid[sl + W * r] = i < len ? __ldg(step_cells + k0 + i) : -1;
      }
      __syncwarp();
    };
    __syncwarp();
    load_ids(0);
    auto entry = [&](int slot) {
      return ring + (size_t)(slot * SEGS + seg) * ES;
    };
    int rc[kSrDepth]; // the cell of each ring slot's step
    auto fetch = [&](int k, int slot) {
      if ((k & (kSrIds - 1)) == 0 && k > 0) { // warp-uniform
        __syncwarp();
        load_ids(k);
      }
      const int v = sid[k & (kSrIds - 1)];
      const int c = scid[k & (kSrIds - 1)];
      if (k < len) {
        double *e = entry(slot) + sl;
        const double *cp = col_at(cl0, v, ccolb);
#pragma unroll
        for (int r = 0; r < CR; ++r) sr_cp8z(e + CP + W * r, cp + W * r, cz[r]);
        if (c >= 0) { // the cell's chunk: D values per layer, contiguous
          const double *fp = x + ((int64_t)c * layers + l0) * D + sl;
#pragma unroll
          for (int r = 0; r < D; ++r)
            sr_cp8z(e + W * r, fp + W * r, sl + W * r < nl * D ? 8 : 0);
        }
      }
      sr_commit();
      return c;
    };
#pragma unroll
    for (int d = 0; d < kSrDepth; ++d) rc[d] = fetch(d, d);

    auto step = [&](auto A_, auto R_, int k) {
      constexpr int A = decltype(A_)::value; // window slot (k % 3)
      constexpr int R = decltype(R_)::value; // ring slot (k % kSrDepth)
      const bool act = k < len;
      sr_wait<kSrDepth - 1>();
      __syncwarp();
      const double *e = act ? entry(R) : zero;
      const double *ec = e + CP;
      double g0[3], g1[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        g0[q] = ec[3 * sl + q];
        g1[q] = ec[3 * (sl + 1) + q];
      }
      gm[A][0] = g0[0] + g1[0];
      gm[A][1] = g0[1] + g1[1];
      gm[A][2] = g1[2] - g0[2];
      const int c = rc[R];
      double xf[D];
#pragma unroll
      for (int d = 0; d < D; ++d) xf[d] = e[sl * D + d];
      __syncwarp(); // reads done before the slot is refilled
      rc[R] = fetch(k + kSrDepth, R);
      if (act && c >= 0 && sl < nl) {
        const double det = prism_abs_detj_12(gm[0][0], gm[0][1], gm[0][2],
                                             gm[1][0], gm[1][1], gm[1][2],
                                             gm[2][0], gm[2][1], gm[2][2]);
        double *yp = y + ((int64_t)c * layers + l0 + sl) * D;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          double sacc = 0.0;
#pragma unroll
          for (int j = 0; j < D; ++j) sacc = fma(M.m[i * D + j], xf[j], sacc);
          yp[i] = det * sacc;
        }
      }
    };
    using S0 = std::integral_constant<int, 0>;
    using S1 = std::integral_constant<int, 1>;
    using S2 = std::integral_constant<int, 2>;
    for (int k = 0; k < maxlen; k += 3) {
      step(S0{}, S0{}, k);
      step(S1{}, S1{}, k + 1);
      step(S2{}, S2{}, k + 2);
    }
    sr_wait<0>(); // no copy in flight into the ring across items
  }
}

template <int D, int W>
static int strip_dg_launch(const MassMat<D> &M, const int32_t *strip_ptr,
                           const int32_t *steps, const int32_t *step_cells,
                           int64_t n_strips, int layers, const double *coords,
                           const double *x, double *y, cudaStream_t s) {
  constexpr int SEGS = 32 / W, NW = kSdThreads / 32;
  const size_t smem =
      sizeof(double) * ((size_t)NW * kSrDepth * SEGS + 1) * sd_entry<D, W>() +
      sizeof(int) * NW * SEGS * 2 * kSrIds;
  static int cached_dev = -1;
  int dev = 0;
  PM_CUDA_TRY(cudaGetDevice(&dev));
  if (cached_dev != dev) {
    PM_CUDA_TRY(cudaFuncSetAttribute(
        k_strip_dg<D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
        (int)smem));
    cached_dev = dev;
  }
  const int64_t items = n_strips * ((layers + W - 1) / W);
  const int64_t warps = (items + SEGS - 1) / SEGS;
  const unsigned grid = grid_for(warps * 32, kSdThreads, strip_grid_cap(8));
  k_strip_dg<D, W><<<grid, kSdThreads, smem, s>>>(
      M, strip_ptr, steps, step_cells, n_strips, layers, coords, x, y);
  PM_LAUNCH_CHECK("k_strip_dg");
  return PM_OK;
}

template <int D>
static int strip_dg_w(const double *mref, int W, const int32_t *strip_ptr,
                      const int32_t *steps, const int32_t *step_cells,
                      int64_t n_strips, int layers, const double *coords,
                      const double *x, double *y, cudaStream_t s) {
  MassMat<D> M; // 12 |det J| from the strip geometry: fold 1/12 in
  for (int i = 0; i < D * D; ++i) M.m[i] = mref[i] * (1.0 / 12.0);
  switch (W) {
  case 32: return strip_dg_launch<D, 32>(M, strip_ptr, steps, step_cells,
                                         n_strips, layers, coords, x, y, s);
  case 16: return strip_dg_launch<D, 16>(M, strip_ptr, steps, step_cells,
                                         n_strips, layers, coords, x, y, s);
  case 8: return strip_dg_launch<D, 8>(M, strip_ptr, steps, step_cells,
                                       n_strips, layers, coords, x, y, s);
  default:
    set_error("strip chunk width must be 8, 16 or 32 (got %d)", W);
    return PM_EINVAL;
  }
}

// Cell columns with level DoFs (DoFs on (2,0) only: DG0 x CG1, DG1 x CG1),
// along strips: as k_strip_dg, but a cell column holds D0 values per LEVEL
// (layers + 1 levels), the level between two layers shared by both.  Lane
// l of a W-layer chunk computes cell-layer l0 + l from its bottom and top
// levels; its top contribution reaches level l0 + l + 1 by shfl.up, so each
// chunk-interior level is stored once.  The chunk's bottom level (shared
// with the chunk below) and top level (with the chunk above) are added
// (REDG) into levels zeroed first (pm_column_mass_strip_dgv zeroes only
// those, k_zero_cell_levels); a column's first and last level are stored.
template <int D0, int W> constexpr int sv_frows() {
  return (D0 * (W + 1) + W - 1) / W;
}
template <int D0, int W> constexpr int sv_entry() {
  return (sv_frows<D0, W>() + sd_crows<D0, W>()) * W;
}

template <int D0, int W>
__global__ void __launch_bounds__(kSdThreads, 3)
k_strip_dgv(const MassMat<2 * D0> M, const int32_t *__restrict__ strip_ptr,
            const int32_t *__restrict__ steps,
            const int32_t *__restrict__ step_cells, int64_t n_strips,
            int layers, const double *__restrict__ coords,
            const double *__restrict__ x, double *__restrict__ y) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int SEGS = 32 / W, K = 2 * D0;
  constexpr int FR = sv_frows<D0, W>(), CR = sd_crows<D0, W>();
  constexpr int ES = sv_entry<D0, W>(), CP = FR * W;
  constexpr int NWARP = kSdThreads / 32;
  const int lane = threadIdx.x & 31;
  const int sl = lane % W, seg = lane / W;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int ccolb = 8 * 3 * (layers + 1);
  const int64_t fcol = (int64_t)D0 * (layers + 1); // cell column length
  extern __shared__ double sd_ring[];
  double *const ring =
      sd_ring + (size_t)(threadIdx.x >> 5) * kSrDepth * SEGS * ES;
  const double *const zero = sd_ring + (size_t)NWARP * kSrDepth * SEGS * ES;
  int *const sid = reinterpret_cast<int *>(sd_ring + (size_t)(NWARP * kSrDepth *
                                                              SEGS + 1) * ES) +
                   ((threadIdx.x >> 5) * SEGS + seg) * 2 * kSrIds;
  int *const scid = sid + kSrIds;
  for (int i = threadIdx.x; i < ES; i += blockDim.x)
    sd_ring[(size_t)NWARP * kSrDepth * SEGS * ES + i] = 0.0;
  __syncthreads();

  const int n_chunks = (layers + W - 1) / W;
  const int64_t n_items = n_strips * n_chunks;
  for (int64_t i0 = warp * SEGS; i0 < n_items; i0 += n_warps * SEGS) {
    const int64_t item = i0 + seg;
    const bool has = item < n_items;
    const int64_t s = has ? item / n_chunks : 0;
    const int l0 = has ? (int)(item % n_chunks) * W : 0;
    const int k0 = has ? __ldg(strip_ptr + s) : 0;
    const int len = has ? __ldg(strip_ptr + s + 1) - k0 : 0;
    int maxlen = len;
#pragma unroll
    for (int o = W; o < 32; o <<= 1)
      maxlen = max(maxlen, __shfl_xor_sync(FULL, maxlen, o));
    const int nl = has ? min(W, layers - l0) : 0;
    int cz[CR], fz[FR];
#pragma unroll
    for (int r = 0; r < CR; ++r) cz[r] = sl + W * r < 3 * (nl + 1) ? 8 : 0;
#pragma unroll
    for (int r = 0; r < FR; ++r) fz[r] = sl + W * r < D0 * (nl + 1) ? 8 : 0;
    const double *cl0 = coords + 3 * (int64_t)l0 + sl;
    // bottom level of the chunk: shared with the chunk below unless the
    // column starts here; top level: with the chunk above unless it ends
    const bool bot_add = l0 > 0, top_add = l0 + nl < layers;
    double gm[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int q = 0; q < 3; ++q) gm[a][q] = 0.0;
    auto load_ids = [&](int base) {
#pragma unroll
      for (int r = 0; r < kSrIds / W; ++r) {
        const int i = base + sl + W * r;
        sid[sl + W * r] = i < len ? __ldg(steps + k0 + i) : 0;
        scid[sl + W * r] = i < len ? __ldg(step_cells + k0 + i) : -1;
      }
      __syncwarp();
    };
    __syncwarp();
    load_ids(0);
    auto entry = [&](int slot) {
      return ring + (size_t)(slot * SEGS + seg) * ES;
    };
    int rc[kSrDepth];
    auto fetch = [&](int k, int slot) {
      if ((k & (kSrIds - 1)) == 0 && k > 0) { // warp-uniform
        __syncwarp();
        load_ids(k);
      }
      const int v = sid[k & (kSrIds - 1)];
      const int c = scid[k & (kSrIds - 1)];
      if (k < len) {
        double *e = entry(slot) + sl;
        const double *cp = col_at(cl0, v, ccolb);
#pragma unroll
        for (int r = 0; r < CR; ++r) sr_cp8z(e + CP + W * r, cp + W * r, cz[r]);
        if (c >= 0) {
          const double *fp = x + (int64_t)c * fcol + (int64_t)l0 * D0 + sl;
#pragma unroll
          for (int r = 0; r < FR; ++r) sr_cp8z(e + W * r, fp + W * r, fz[r]);
        }
      }
      sr_commit();
      return c;
    };
#pragma unroll
    for (int d = 0; d < kSrDepth; ++d) rc[d] = fetch(d, d);

    auto step = [&](auto A_, auto R_, int k) {
      constexpr int A = decltype(A_)::value;
      constexpr int R = decltype(R_)::value;
      const bool act = k < len;
      sr_wait<kSrDepth - 1>();
      __syncwarp();
      const double *e = act ? entry(R) : zero;
      const double *ec = e + CP;
      double g0[3], g1[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        g0[q] = ec[3 * sl + q];
        g1[q] = ec[3 * (sl + 1) + q];
      }
      gm[A][0] = g0[0] + g1[0];
      gm[A][1] = g0[1] + g1[1];
      gm[A][2] = g1[2] - g0[2];
      const int c = rc[R];
      double xv[K]; // bottom level (D0), top level (D0) of the lane's layer
#pragma unroll
      for (int d = 0; d < D0; ++d) {
        xv[d] = e[sl * D0 + d];
        xv[D0 + d] = e[(sl + 1) * D0 + d];
      }
      __syncwarp();
      rc[R] = fetch(k + kSrDepth, R);
      // warp-uniform: every lane of the segment takes part in the shuffle
      const bool cell = act && c >= 0;
      if (__any_sync(FULL, cell)) {
        const double det = prism_abs_detj_12(gm[0][0], gm[0][1], gm[0][2],
                                             gm[1][0], gm[1][1], gm[1][2],
                                             gm[2][0], gm[2][1], gm[2][2]);
        const double dd = (cell && sl < nl) ? det : 0.0;
        double out[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          double sacc = 0.0;
#pragma unroll
          for (int j = 0; j < K; ++j) sacc = fma(M.m[i * K + j], xv[j], sacc);
          out[i] = dd * sacc;
        }
        double *col = y + (int64_t)(cell ? c : 0) * fcol;
#pragma unroll
        for (int d = 0; d < D0; ++d) {
          // level l0 + sl: own bottom part + the lane below's top part
          const double below = __shfl_up_sync(FULL, out[D0 + d], 1, W);
          double *p = col + (int64_t)(l0 + sl) * D0 + d;
          if (cell && sl < nl) {
            if (sl > 0)
              *p = out[d] + below;
            else if (bot_add)
              atomicAdd(p, out[d]);
            else
              *p = out[d];
          }
          if (cell && sl == nl - 1) { // the chunk's top level
            double *pt = p + D0;
            if (top_add)
              atomicAdd(pt, out[D0 + d]);
            else
              *pt = out[D0 + d];
          }
        }
      }
    };
    using S0 = std::integral_constant<int, 0>;
    using S1 = std::integral_constant<int, 1>;
    using S2 = std::integral_constant<int, 2>;
    for (int k = 0; k < maxlen; k += 3) {
      step(S0{}, S0{}, k);
      step(S1{}, S1{}, k + 1);
      step(S2{}, S2{}, k + 2);
    }
    sr_wait<0>();
  }
}

// zero the chunk-boundary levels (l = W, 2W, ... < layers) of every cell
// column with level DoFs: the two chunks meeting there add into them
__global__ void k_zero_cell_levels(double *__restrict__ y, int64_t n_cells,
                                   int layers, int d0, int w, int nb) {
  const int64_t n = n_cells * nb * d0;
  const int64_t fcol = (int64_t)d0 * (layers + 1);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / (nb * d0);
    const int r = (int)(t - c * nb * d0);
    y[c * fcol + (int64_t)(r / d0 + 1) * w * d0 + r % d0] = 0.0;
  }
}

template <int D0, int W>
static int strip_dgv_launch(const double *mref, const int32_t *strip_ptr,
                            const int32_t *steps, const int32_t *step_cells,
                            int64_t n_strips, int64_t n_cells, int layers,
                            const double *coords, const double *x, double *y,
                            cudaStream_t s) {
  constexpr int SEGS = 32 / W, NW = kSdThreads / 32, K = 2 * D0;
  MassMat<K> M;
  for (int i = 0; i < K * K; ++i) M.m[i] = mref[i] * (1.0 / 12.0);
  const int nb = (layers + W - 1) / W - 1; // interior chunk boundaries
  if (nb > 0 && n_cells > 0) {
    k_zero_cell_levels<<<grid_for(n_cells * nb * D0, 256, 4), 256, 0, s>>>(
        y, n_cells, layers, D0, W, nb);
    PM_LAUNCH_CHECK("k_zero_cell_levels");
  }
  const size_t smem =
      sizeof(double) * ((size_t)NW * kSrDepth * SEGS + 1) * sv_entry<D0, W>() +
      sizeof(int) * NW * SEGS * 2 * kSrIds;
  static int cached_dev = -1;
  int dev = 0;
  PM_CUDA_TRY(cudaGetDevice(&dev));
  if (cached_dev != dev) {
    PM_CUDA_TRY(cudaFuncSetAttribute(
        k_strip_dgv<D0, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
        (int)smem));
    cached_dev = dev;
  }
  const int64_t items = n_strips * ((layers + W - 1) / W);
  const int64_t warps = (items + SEGS - 1) / SEGS;
  const unsigned grid = grid_for(warps * 32, kSdThreads, strip_grid_cap(8));
  k_strip_dgv<D0, W><<<grid, kSdThreads, smem, s>>>(
      M, strip_ptr, steps, step_cells, n_strips, layers, coords, x, y);
  PM_LAUNCH_CHECK("k_strip_dgv");
  return PM_OK;
}

template <int D0>
static int strip_dgv_w(const double *mref, int W, const int32_t *strip_ptr,
                       const int32_t *steps, const int32_t *step_cells,
                       int64_t n_strips, int64_t n_cells, int layers,
                       const double *coords, const double *x, double *y,
                       cudaStream_t s) {
  switch (W) {
  case 32: return strip_dgv_launch<D0, 32>(mref, strip_ptr, steps, step_cells,
                                           n_strips, n_cells, layers, coords,
                                           x, y, s);
  case 16: return strip_dgv_launch<D0, 16>(mref, strip_ptr, steps, step_cells,
                                           n_strips, n_cells, layers, coords,
                                           x, y, s);
  case 8: return strip_dgv_launch<D0, 8>(mref, strip_ptr, steps, step_cells,
                                         n_strips, n_cells, layers, coords,
                                         x, y, s);
  default:
    set_error("strip chunk width must be 8, 16 or 32 (got %d)", W);
    return PM_EINVAL;
  }
}

} // namespace pm

static int strip_red_entry(
    const int32_t *delta6, int32_t k, int32_t layers, const double *coords,
    const double *mref, const double *mtri, const double *mline,
    const double *x, double *y, int64_t n_dofs, int32_t accumulate,
    int64_t n_strips, int32_t chunk, const int32_t *strip_ptr,
    const int32_t *steps, const int32_t *steps_e, int64_t n_vertices,
    double *y_peer, int64_t ghost_end, void *stream,
    const int32_t *item_ptr = nullptr, int64_t n_zero = 0,
    const int32_t *zero_list = nullptr) {
  pm::clear_error();
  pm::LoopArgs a;
  a.item_ptr = item_ptr;
  a.y_peer = y_peer;
  a.ghost_end = y_peer ? ghost_end : 0;
  if (y_peer && (ghost_end < 0 || ghost_end > INT32_MAX ||
                 pm::Layout<1, 1, 1, 1, 0, 0>::matches(delta6))) {
    pm::set_error("the fused halo needs a vertex-column layout and an int32 "
                  "ghost vertex bound");
    return PM_EINVAL;
  }
  int rc = pm::make_slot_table(delta6, &a.st);
  if (rc) return rc;
  if (k != a.st.k || layers < 1 || n_strips < 0 || !mref || n_dofs < 0) {
    pm::set_error("bad arguments to pm_column_mass_strip_red");
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
  if (item_ptr && !accumulate && n_dofs > 0 && chunk > 0) {
    // store-first patch strips: only the shared columns and the chunk
    // boundary levels need zeroing
    const int ch0 = delta6[0] + delta6[1], lv0 = delta6[0];
    const int ch1 = delta6[2] + delta6[3], lv1 = delta6[2];
    const int colv = layers * ch0 + lv0, cole = layers * ch1 + lv1;
    const int64_t e_start = (int64_t)colv * n_vertices;
    const int64_t n_edges = cole > 0 ? (n_dofs - e_start) / cole : 0;
    if (n_zero < 0 || (n_zero > 0 && !zero_list) || e_start > n_dofs ||
        e_start + n_edges * cole != n_dofs) {
      pm::set_error("pm_column_mass_patch_strips: bad zero list / sizes");
      return PM_EINVAL;
    }
    if (n_zero > 0) {
      pm::k_zero_entities<<<pm::grid_for(n_zero * 32, 256, 4), 256, 0, a.s>>>(
          y, zero_list, n_zero, n_vertices, colv, cole, e_start);
      PM_LAUNCH_CHECK("k_zero_entities");
    }
    const int nb = (layers + chunk - 1) / chunk - 1;
    const int64_t nlev = (n_vertices * lv0 + n_edges * lv1) * nb;
    if (nlev > 0) {
      pm::k_zero_chunk_levels<<<pm::grid_for(nlev, 256, 4), 256, 0, a.s>>>(
          y, n_vertices, n_edges, colv, cole, e_start, ch0, lv0, ch1, lv1,
          chunk, nb);
      PM_LAUNCH_CHECK("k_zero_chunk_levels");
    }
    a.store = 1;
  } else if (!accumulate && n_dofs > 0) {
    PM_CUDA_TRY(cudaMemsetAsync(y, 0, (size_t)n_dofs * sizeof(double), a.s));
  }
  if (n_strips == 0) return PM_OK;
  if (!coords || !x || !y || !strip_ptr || !steps) {
    pm::set_error("NULL device pointer");
    return PM_EINVAL;
  }
#define PM_DISPATCH(a_, b_, c_, e_, f_, g_)                                  \
  if (pm::Layout<a_, b_, c_, e_, f_, g_>::matches(delta6))                   \
    return pm::strip_red_k<pm::Layout<a_, b_, c_, e_, f_, g_>>(              \
        a, strip_ptr, steps, n_strips, chunk);
  PM_STRIPRED_LAYOUTS(PM_DISPATCH)
#undef PM_DISPATCH
  if (pm::Layout<1, 1, 1, 1, 0, 0>::matches(delta6)) {
    const int64_t col0 = (int64_t)layers * 2 + 1;
    return pm::strip_red_e_k<pm::Layout<1, 1, 1, 1, 0, 0>>(
        a, strip_ptr, steps, steps_e, n_strips, chunk, col0 * n_vertices);
  }
  pm::set_error("layout not supported by the strip schedule");
  return PM_EINVAL;
}

extern "C" int pm_column_mass_strip_red(
    const int32_t *delta6, int32_t k, int32_t layers, const double *coords,
    const double *mref, const double *mtri, const double *mline,
    const double *x, double *y, int64_t n_dofs, int32_t accumulate,
    int64_t n_strips, int32_t chunk, const int32_t *strip_ptr,
    const int32_t *steps, const int32_t *steps_e, int64_t n_vertices,
    void *stream) {
  return strip_red_entry(delta6, k, layers, coords, mref, mtri, mline, x, y,
                         n_dofs, accumulate, n_strips, chunk, strip_ptr,
                         steps, steps_e, n_vertices, nullptr, 0, stream);
}

extern "C" int pm_column_mass_strip_red_peer(
    const int32_t *delta6, int32_t k, int32_t layers, const double *coords,
    const double *mref, const double *mtri, const double *mline,
    const double *x, double *y, int64_t n_dofs, int32_t accumulate,
    int64_t n_strips, int32_t chunk, const int32_t *strip_ptr,
    const int32_t *steps, int64_t n_vertices, double *y_peer,
    int64_t ghost_vertex_end, void *stream) {
  return strip_red_entry(delta6, k, layers, coords, mref, mtri, mline, x, y,
                         n_dofs, accumulate, n_strips, chunk, strip_ptr,
                         steps, nullptr, n_vertices, y_peer,
                         ghost_vertex_end, stream);
}

extern "C" int pm_column_mass_patch_strips(
    const int32_t *delta6, int32_t k, int32_t layers, const double *coords,
    const double *mref, const double *mtri, const double *mline,
    const double *x, double *y, int64_t n_dofs, int32_t accumulate,
    int64_t n_patches, int32_t chunk, const int32_t *item_ptr,
    const int32_t *strip_ptr, const int32_t *steps, const int32_t *steps_e,
    int64_t n_vertices, int64_t n_zero, const int32_t *zero_list,
    void *stream) {
  if (!item_ptr && n_patches > 0) {
    pm::clear_error();
    pm::set_error("pm_column_mass_patch_strips: NULL item_ptr");
    return PM_EINVAL;
  }
  if (pm::strip_levels() != 1) {
    pm::clear_error();
    pm::set_error("store-first patch strips run one level per lane "
                  "(unset PM_STRIP_L)");
    return PM_EINVAL;
  }
  return strip_red_entry(delta6, k, layers, coords, mref, mtri, mline, x, y,
                         n_dofs, accumulate, n_patches, chunk, strip_ptr,
                         steps, steps_e, n_vertices, nullptr, 0, stream,
                         item_ptr, n_zero, zero_list);
}

extern "C" int pm_column_mass_strip_dg(
    const int32_t *delta6, int32_t k, int64_t n_cells, int32_t layers,
    const double *coords,
    const double *mref, const double *x, double *y, int64_t n_strips,
    int32_t chunk, const int32_t *strip_ptr, const int32_t *steps,
    const int32_t *step_cells, void *stream) {
  pm::clear_error();
  const bool cells_only = delta6 && !delta6[0] && !delta6[1] && !delta6[2] &&
                          !delta6[3];
  const bool dg_only = cells_only && !delta6[4] && delta6[5] == k;
  const bool levels_only = cells_only && !delta6[5] && 2 * delta6[4] == k;
  if (levels_only && layers >= 1 && n_strips >= 0 && mref) {
    if (n_strips == 0) return PM_OK;
    if (!coords || !x || !y || !strip_ptr || !steps || !step_cells) {
      pm::set_error("NULL device pointer");
      return PM_EINVAL;
    }
    if (n_cells < 0) {
      pm::set_error("pm_column_mass_strip_dg: n_cells < 0");
      return PM_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    switch (delta6[4]) {
    case 1: return pm::strip_dgv_w<1>(mref, chunk, strip_ptr, steps,
                                      step_cells, n_strips, n_cells, layers,
                                      coords, x, y, s);
    case 3: return pm::strip_dgv_w<3>(mref, chunk, strip_ptr, steps,
                                      step_cells, n_strips, n_cells, layers,
                                      coords, x, y, s);
    default:
      pm::set_error("pm_column_mass_strip_dg: %d DoFs per cell level (1 or "
                    "3 compiled)", delta6[4]);
      return PM_EINVAL;
    }
  }
  if (!dg_only || layers < 1 || n_strips < 0 || !mref) {
    pm::set_error("pm_column_mass_strip_dg: a DG layout (DoFs on the prism "
                  "cells only, k = delta(2,1)) and layers >= 1");
    return PM_EINVAL;
  }
  if (n_strips == 0) return PM_OK;
  if (!coords || !x || !y || !strip_ptr || !steps || !step_cells) {
    pm::set_error("NULL device pointer");
    return PM_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  switch (k) {
  case 1: return pm::strip_dg_w<1>(mref, chunk, strip_ptr, steps, step_cells,
                                   n_strips, layers, coords, x, y, s);
  case 2: return pm::strip_dg_w<2>(mref, chunk, strip_ptr, steps, step_cells,
                                   n_strips, layers, coords, x, y, s);
  case 3: return pm::strip_dg_w<3>(mref, chunk, strip_ptr, steps, step_cells,
                                   n_strips, layers, coords, x, y, s);
  case 6: return pm::strip_dg_w<6>(mref, chunk, strip_ptr, steps, step_cells,
                                   n_strips, layers, coords, x, y, s);
  default:
    pm::set_error("pm_column_mass_strip_dg: %d DoFs per cell-layer (1, 2, 3 "
                  "or 6 compiled)", k);
    return PM_EINVAL;
  }
}
