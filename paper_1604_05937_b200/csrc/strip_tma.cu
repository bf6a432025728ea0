// Run-strip schedule for vertex-column CG layouts with level DoFs (P1 and
// 3-vector P1): the strip-REDG walk of strip_red.cu, fed by bulk copies
// (cp.async.bulk, the 1-D TMA path) of WHOLE vertex columns, several columns
// per copy.
//
// On a level-ordered base mesh (RCM, ordering.py:45-90) a sequential strip
// that follows the band between two BFS levels (pm_build_run_strips) takes
// its even vertices from one run of consecutive ids and its odd vertices
// from another.  Under Alg. 1 (fspace.py:141-147) consecutive vertex ids are
// consecutive columns of the field, so the 3 steps of one side of a granule
// (= 6 strip steps) are ONE contiguous slab of the field and one of the
// coordinate field: 4 bulk copies per granule instead of 5-6 cp.async rows
// per step and warp, which is what bound the cp.async ring (L1 data pipe
// 84 %, profiles/README.md).  Granules whose ids are not consecutive fall
// back to one copy per column (any strip plan is valid input; only the
// speed depends on the runs).
//
// A group of NCH warps walks a strip in lock step out of a shared ring of
// 2 stages (one granule each).  Scalar columns take two 32-layer chunks per
// warp (NQ = 2: for 64 layers one warp per strip and no cross-warp
// protocol), otherwise one chunk per warp.  The warp of a group that
// releases a granule last (shared-memory counter) refills its stage with
// the granule 2 ahead, completion by mbarrier transaction bytes; it also
// writes each step's smem offsets and vertex id into a per-stage table (one
// broadcast LDS.128 per step for the consumers); the ids a refill needs are
// loaded a granule earlier.
//
// The strip loop: granule positions are template arguments (6 = lcm of the
// 3-slot window and the 2 sides), the ring values of step k+1 are read in
// the middle of step k, and for scalar columns there is NO predicated RED
// and NO guard in it -- ptxas compiles a predicated red into a branch, each
// branch ends a scheduling block, and in ~40-instruction blocks the fp64
// chains cannot overlap the next step's reads (C5a 2.96 -> 2.33 ms).  The
// one top value per flush is parked in shared memory and added once per
// granule; bottom values are added by every lane (a partial last chunk's
// dead lanes add 0.0 to a level of their own column); whole granules run
// unguarded, head and tail guarded.  Element kernel and window as
// k_strip_red (one level per lane, symmetric triangle factor ta I + tb J).
#include "column_layout.cuh"
#include "column_loop.cuh"
#include "pm_ptx.cuh"

#include <cstdlib>
#include <type_traits>

// CTA size caps (registers per thread = 65536 / cap): scalar / 3-vector
#ifndef PM_TMA_MAXT_S
#define PM_TMA_MAXT_S 512
#endif
#ifndef PM_TMA_MAXT_S2 // scalar columns, two chunks per warp
#define PM_TMA_MAXT_S2 256
#endif
#ifndef PM_TMA_MAXT_V
#define PM_TMA_MAXT_V 256
#endif
// 1: also compile the half-granule rings (4 stages of 3 steps, PM_TMA_NS=4)
#ifndef PM_TMA_HALF
#define PM_TMA_HALF 0
#endif
// 1: the branch-free flush for 3-vector columns too (measured slower)
#ifndef PM_TMA_VFULL
#define PM_TMA_VFULL 0
#endif


namespace pm {

namespace {

struct alignas(16) StmaEntry {
  uint32_t foff, coff; // byte offsets of the column starts in dynamic smem
  int32_t vid;
  int32_t pad;
};

__device__ __forceinline__ void stma_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile(
      "mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void stma_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void stma_red(double *p, double v, bool on) {
  asm volatile("{\n\t.reg .pred q;\n\t"
               "setp.ne.b32 q, %2, 0;\n\t"
               "@q red.global.add.f64 [%0], %1;\n\t}" ::"l"(p),
               "d"(v), "r"((int)on)); // y is never read: no memory clobber
}
__device__ __forceinline__ void stma_red_all(double *p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v));
}
// release this warp's reads of a stage / acquire the other warps' (one
// acq_rel atomic instead of two block fences around a relaxed one)
__device__ __forceinline__ int stma_count(int *p) {
  int old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
               : "=r"(old)
               : "r"(smem_u32(p))
               : "memory");
  return old;
}
__device__ __forceinline__ void stma_group_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

constexpr uint32_t stma_up16(uint32_t b) { return (b + 15u) & ~15u; }

// smem carve-up (bytes), shared by the kernel and the launcher
struct StmaSmem {
  uint32_t off_tab, bars, cnt, tops, trow, ring, zero, total;
};
__host__ __device__ inline StmaSmem stma_smem(int NC, int G2, int NS,
                                              int ngrp, int nwarp,
                                              uint32_t Pf, uint32_t Pc) {
  StmaSmem s;
  uint32_t o = 0;
  s.off_tab = o, o += (uint32_t)ngrp * NS * G2 * 16;
  s.bars = o, o += (uint32_t)ngrp * NS * 8;
  s.cnt = o, o += stma_up16((uint32_t)ngrp * NS * 4);
  s.tops = o, o += (uint32_t)nwarp * G2 * NC * 16;
  s.trow = o, o += NC > 1 ? (uint32_t)nwarp * 2 * (33 * NC + 1) * 8 : 0;
  o = (o + 127u) & ~127u;
  s.ring = o, o += (uint32_t)ngrp * NS * G2 * (Pf + Pc);
  s.zero = o;
  o += 2048; // lanes past a partial chunk read past their column (never used)
  s.total = o;
  return s;
}

template <int NC, int NQ, int NS, int NCH, int MAXT, bool FULL, int G2>
__global__ void __launch_bounds__(MAXT, 1)
k_strip_tma(const KronMat M, const int32_t *__restrict__ strip_ptr,
            const int32_t *__restrict__ steps, int64_t n_strips, int layers,
            const double *__restrict__ coords, const double *__restrict__ x,
            double *__restrict__ y, int ngrp, uint32_t Pf, uint32_t Pc,
            int64_t n_vertices) {
  static_assert(NC == 1 || NQ == 1, "two chunks per warp: scalar columns");
  constexpr unsigned FULL_MASK = 0xffffffffu;
  constexpr int CH = NC, NV = 2;
  // granule = G2 strip steps: the first step's side brings NA columns, the
  // other side NB (G2 = 3: 2 + 1, sides swapping from granule to granule)
  static_assert(G2 == 3 || G2 == 6, "granule = whole window cycles");
  constexpr int NA = (G2 + 1) / 2, NB = G2 / 2;
  constexpr int TR = NC > 1 ? 33 * NC : 0; // staged chunk row
  constexpr int TRP = 33 * NC + 1;         // row pitch (doubles)
  constexpr int NR = NC > 1 ? (TR + 31) / 32 : 1;
  constexpr bool CSUM = NC == 1;
  extern __shared__ __align__(128) unsigned char stma_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nwarp = blockDim.x >> 5;
  const int grp = wib / NCH, chunk = wib % NCH;
  const StmaSmem L = stma_smem(NC, G2, NS, ngrp, nwarp, Pf, Pc);
  StmaEntry *const tab =
      reinterpret_cast<StmaEntry *>(stma_raw + L.off_tab) + grp * NS * G2;
  uint64_t *const full = reinterpret_cast<uint64_t *>(stma_raw + L.bars) +
                         grp * NS;
  int *const cnt = reinterpret_cast<int *>(stma_raw + L.cnt) + grp * NS;
  double *const trow0 =
      reinterpret_cast<double *>(stma_raw + L.trow) + wib * 2 * TRP;
  // scalar columns: the one top value per flush (the chunk's last lane) is
  // parked here and added once per granule by 2G lanes, so the strip loop
  // has no predicated RED (ptxas turns those into branches, which end its
  // scheduling blocks: measured 2.96 -> 2.32 ms on C5a without them)
  constexpr int NT = G2 * NC; // parked values per warp and granule
  double *const topv = reinterpret_cast<double *>(stma_raw + L.tops) +
                       wib * 2 * NT;
  double **const topa = reinterpret_cast<double **>(topv + NT);
  const uint32_t SB = G2 * (Pf + Pc); // stage bytes
  const uint32_t ring_off = L.ring + (uint32_t)grp * NS * SB;

  if (threadIdx.x < (unsigned)(ngrp * NS)) {
    mbar_init(reinterpret_cast<uint64_t *>(stma_raw + L.bars) + threadIdx.x, 1);
    reinterpret_cast<int *>(stma_raw + L.cnt)[threadIdx.x] = 0;
  }
  fence_mbar_init();
  __syncthreads();

  const int colf = (layers + 1) * NC; // doubles per field column
  const int colc = (layers + 1) * 3;  // doubles per coordinate column
  const int sl = lane;
  const int l0 = chunk * 32 * NQ; // first level of this warp's chunks
  // lane predicates of the flushes: bottom values of live cell-layers, the
  // top value of the last chunk's last cell-layer (the top of chunk 0 of
  // two goes into chunk 1's lane 0: the launcher picks NQ = 2 only when
  // every warp's second chunk is non-empty)
  bool pb[NQ], pt;
  int nlq[NQ], boff[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    nlq[q] = max(0, min(32, layers - (l0 + 32 * q)));
    pb[q] = sl < nlq[q];
    boff[q] = 32 * q * CH;
  }
  // Lanes past a partial last chunk are not predicated off (no branches in
  // the strip loop): they add 0.0 inside their own column, at level
  // (their level) mod (levels per column) -- distinct levels for columns of
  // 32 levels or more, always in bounds.  (FULL: no such lanes.)
  if (!pb[NQ - 1])
    boff[NQ - 1] = ((l0 + 32 * (NQ - 1) + sl) % (layers + 1) - (l0 + sl)) * CH;
  pt = sl == nlq[NQ - 1] - 1;
  const int nl = nlq[0]; // (NC > 1: NQ == 1)
  const double *const x_end = x + n_vertices * colf;
  const double *const c_end = coords + n_vertices * colc;

  // Refill: stage `st` <- granule `g` of the strip (steps k0 + 2G g ..).
  // One converged warp; lane t < 2G looks after step 2G g + t, whose id `v`
  // the caller loaded (a granule ahead).
  auto refill = [&](int st, int g, int len, int v) {
    const int t = lane, k = G2 * g + t;
    const bool valid = t < G2 && k < len;
    const int side = t & 1, j = t >> 1;
    const int vfirst = __shfl_sync(FULL_MASK, v, side);
    const unsigned sidemask = 0x55555555u << side;
    const unsigned bad = __ballot_sync(FULL_MASK, valid && v != vfirst + j);
    const unsigned vmask = __ballot_sync(FULL_MASK, valid);
    const bool consec = !(bad & sidemask);
    const int nside = __popc(vmask & sidemask);
    // (`side` is relative to the granule's first step)
    const uint32_t side_base = ring_off + (uint32_t)st * SB +
                               (uint32_t)side * NA * (Pf + Pc);
    const uint32_t ncol = side ? NB : NA; // column slots of this side
    uint64_t *const bar = full + st;
    if (valid) {
      const int vb = consec ? vfirst : v; // first column of the copy
      const int nb = consec ? nside : 1;  // columns in the copy
      const bool issue = !consec || j == 0;
      const double *fs = x + (int64_t)vb * colf;
      const double *cs = coords + (int64_t)vb * colc;
      const uint32_t fsh = (uint32_t)(reinterpret_cast<uintptr_t>(fs) >> 3) & 1;
      const uint32_t csh = (uint32_t)(reinterpret_cast<uintptr_t>(cs) >> 3) & 1;
      // consecutive columns lie back to back, single ones at the padded pitch
      const uint32_t fdst = side_base + (consec ? 0u : (uint32_t)j * Pf);
      const uint32_t cdst = side_base + ncol * Pf + (consec ? 0u : (uint32_t)j * Pc);
      StmaEntry e;
      // (the lane's first value: level l0 + lane is added by the readers)
      e.foff = fdst + 8 * fsh + (consec ? (uint32_t)j * 8 * colf : 0u);
      e.coff = cdst + 8 * csh + (consec ? (uint32_t)j * 8 * colc : 0u);
      e.vid = v;
      e.pad = 0;
      tab[st * G2 + t] = e;
      if (issue) {
        uint32_t fbytes = stma_up16(8 * ((uint32_t)nb * colf + fsh));
        uint32_t cbytes = stma_up16(8 * ((uint32_t)nb * colc + csh));
        const double *fa = fs - fsh, *ca = cs - csh;
        // the 16-byte rounding may reach one double past the arrays' end:
        // copy 16 bytes fewer and bring the last double by hand
        if (fa + fbytes / 8 > x_end) {
          fbytes -= 16;
          *reinterpret_cast<double *>(stma_raw + fdst + fbytes) =
              __ldg(fa + fbytes / 8);
        }
        if (ca + cbytes / 8 > c_end) {
          cbytes -= 16;
          *reinterpret_cast<double *>(stma_raw + cdst + cbytes) =
              __ldg(ca + cbytes / 8);
        }
        stma_expect_tx(bar, fbytes + cbytes);
        if (fbytes) bulk_g2s(stma_raw + fdst, fa, fbytes, bar);
        if (cbytes) bulk_g2s(stma_raw + cdst, ca, cbytes, bar);
      }
    }
    __syncwarp();
    if (lane == 0) stma_arrive(bar);
  };

  const int64_t n_groups = (int64_t)gridDim.x * ngrp;
  uint32_t gc = 0; // granules consumed so far (identical in a group's warps)
  for (int64_t s = (int64_t)blockIdx.x * ngrp + grp; s < n_strips;
       s += n_groups) {
    const int k0 = __ldg(strip_ptr + s);
    const int len = __ldg(strip_ptr + s + 1) - k0;
    const int ngran = (len + G2 - 1) / G2;
    auto ids = [&](int g) { // the lane's step id of granule g
      const int kk = G2 * g + lane;
      return (lane < G2 && kk < len) ? __ldg(steps + k0 + kk) : 0;
    };
    // every warp of the group is done with the previous strip's stages
    if constexpr (NCH > 1)
      stma_group_sync(1 + grp, NCH * 32);
    else
      __syncwarp();
    if (chunk == 0) {
      for (int i = 0; i < NS && i < ngran; ++i)
        refill((int)((gc + i) % NS), i, len, ids(i));
    }
    // ids of granule NS (refilled at the first release of this strip)
    int vpre = ids(NS);
    double zv[NQ][3][NC][NV], gm[NQ][3][3], acc[CSUM ? 1 : 3][NC][NV];
    double tr[CSUM ? NQ : 1][3], dr[CSUM ? NQ : 1][3][NC][NV];
#pragma unroll
    for (int q = 0; q < (CSUM ? NQ : 1); ++q)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        tr[q][a] = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int v = 0; v < NV; ++v) dr[q][a][c][v] = 0.0;
      }
    double *yc[3] = {y, y, y};
    int tb = 0;
    double *pbase = y;
    bool plive = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          if (!CSUM) acc[a][c][v] = 0.0;
#pragma unroll
          for (int q = 0; q < NQ; ++q) zv[q][a][c][v] = 0.0;
        }
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int w = 0; w < 3; ++w) gm[q][a][w] = 0.0;
    }
    int cur_st = 0;
    if constexpr (NC == 1 || FULL) {
      if (lane < NT) topv[lane] = 0.0, topa[lane] = y;
      if constexpr (NC > 1) {
        // the first flush adds the (empty) previous row: zeros to y[0..]
        for (int i = lane; i < 2 * TRP; i += 32) trow0[i] = 0.0;
        plive = true;
      }
      __syncwarp();
    }

    // the vertex of window slot A leaves: its partial column goes to y
    auto flush = [&](auto A_, auto TS_) __attribute__((always_inline)) {
      constexpr int A = decltype(A_)::value;
      constexpr int TS = decltype(TS_)::value; // parked-top slot, -1: add now
      if constexpr (NC > 1) {
        // staged rows: the previous flush's STS before this one's LDS, its
        // LDS before this one's STS
        __syncwarp();
        double *const trow = trow0 + tb * TRP;
        const double *prow = trow0 + (tb ^ 1) * TRP;
        double pv[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const int i = sl + 32 * r;
          pv[r] = prow[i < TR ? i : 0];
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const double vt = acc[A][c][1];
          double v0 = acc[A][c][0];
          acc[A][c][0] = 0.0, acc[A][c][1] = 0.0;
          const double below = __shfl_up_sync(FULL_MASK, vt, 1);
          if (sl > 0) v0 += below;
          if (sl < nl) trow[sl * CH + c] = v0;
          if (sl == nl - 1) trow[(sl + 1) * CH + c] = vt;
        }
        // the previous row's REDs now (lane-contiguous); this row's at the
        // next flush
        double *const base = yc[A] - sl * CH;
        const int n = nl * CH + CH;
        if constexpr (FULL && TS >= 0) {
          // whole chunks: rows 0 .. NR-2 are all live (32 (NR-1) values of
          // the 33 CH); the CH values of the chunk's top level are parked
          // and added once per granule (no predicated RED in the loop)
          static_assert(32 * (NR - 1) + CH == TR, "row split");
#pragma unroll
          for (int r = 0; r + 1 < NR; ++r)
            stma_red_all(pbase + sl + 32 * r, pv[r]);
          if (sl < CH) {
            topv[TS * CH + sl] = pv[NR - 1];
            topa[TS * CH + sl] = pbase + 32 * (NR - 1) + sl;
          }
        } else {
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            const int i = sl + 32 * r;
            stma_red(pbase + i, pv[r], plive & (i < n));
          }
        }
        pbase = base;
        plive = true;
        tb ^= 1;
      } else {
        double a0[NQ], a1[NQ], rot[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const double t = tr[q][0] + tr[q][1] + tr[q][2];
          a0[q] = fma(zv[q][A][0][0], t,
                      dr[q][0][0][0] + dr[q][1][0][0] + dr[q][2][0][0]);
          a1[q] = fma(zv[q][A][0][1], t,
                      dr[q][0][0][1] + dr[q][1][0][1] + dr[q][2][0][1]);
          // the top value of the lane below (lane 0: of lane 31)
          rot[q] = __shfl_sync(FULL_MASK, a1[q], (sl + 31) & 31);
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const double below = sl > 0 ? rot[q] : (q > 0 ? rot[q - 1] : 0.0);
          const double v = a0[q] + below;
          if (FULL || q < NQ - 1)
            stma_red_all(yc[A] + boff[q], v);
          else
            stma_red_all(yc[A] + boff[q], pb[q] ? v : 0.0);
        }
        if constexpr (TS >= 0) {
          if (pt) {
            topv[TS] = a1[NQ - 1];
            topa[TS] = yc[A] + 32 * (NQ - 1) + 1;
          }
        } else {
          stma_red(yc[A] + 32 * (NQ - 1) + 1, a1[NQ - 1], pt);
        }
      }
    };
    // the parked top values of the last granule's flushes
    auto add_tops = [&]() __attribute__((always_inline)) {
      if constexpr (NC == 1 || FULL) {
        __syncwarp();
        if (lane < NT) {
          stma_red_all(topa[lane], topv[lane]);
          topv[lane] = 0.0;
        }
        __syncwarp();
      } else {
        __syncwarp();
      }
    };

    // Software pipeline: the column values of step k+1 are read out of the
    // ring (into F) in the middle of step k, after step k's own values were
    // consumed and before its cell arithmetic.  P = k mod 2G is a template
    // argument: granule boundaries and table slots are compile-time.
    double Ff[NQ][2][CH], Fg[NQ][2][3];
    int Fva = 0;
    auto prefetch = [&](auto P_, int k) __attribute__((always_inline)) {
      constexpr int P = decltype(P_)::value;
      if constexpr (P == 0) { // granule boundary
        const int g = k / G2;
        if (g > 0) {
          // release granule g-1 (its last values are in registers); the
          // last warp of the group to do so refills its stage with
          // granule g-1+NS
          // (the refill first: its round trip to HBM is the critical path
          // of the ring; the parked tops are added behind it)
          __syncwarp();
          bool last = true;
          if constexpr (NCH > 1) {
            int l = 0;
            if (lane == 0) {
              l = stma_count(cnt + cur_st) == NCH - 1;
              if (l) cnt[cur_st] = 0;
            }
            last = __shfl_sync(FULL_MASK, l, 0);
          }
          if (last && g - 1 + NS < ngran) refill(cur_st, g - 1 + NS, len, vpre);
          // ids of the granule the NEXT release refills (any warp of the
          // group may be the one): loaded a granule ahead of their use
          vpre = ids(g + NS);
          add_tops();
        }
        const uint32_t gg = gc + (uint32_t)g;
        cur_st = (int)(gg % NS);
        mbar_wait(full + cur_st, (gg / NS) & 1);
      }
      const int4 e = *reinterpret_cast<const int4 *>(tab + cur_st * G2 + P);
      Fva = e.z;
      const double *ef = reinterpret_cast<const double *>(stma_raw + e.x) +
                         (l0 + sl) * CH;
      const double *ec = reinterpret_cast<const double *>(stma_raw + e.y) +
                         3 * (l0 + sl);
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
#pragma unroll
          for (int c = 0; c < CH; ++c)
            Ff[q][j][c] = ef[(32 * q + j) * CH + c];
#pragma unroll
          for (int w = 0; w < 3; ++w) Fg[q][j][w] = ec[3 * (32 * q + j) + w];
        }
    };

    // one strip step: the vertex of step k enters window slot A = P mod 3
    auto step = [&](auto P_, auto FILL_, auto GUARD_, int k) __attribute__((always_inline)) {
      constexpr int P = decltype(P_)::value;
      constexpr int A = P % 3;
      constexpr bool FILL = decltype(FILL_)::value;
      constexpr bool GUARD = decltype(GUARD_)::value;
      using AC = std::integral_constant<int, A>;
      if constexpr (!FILL) flush(AC{}, P_);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        gm[q][A][0] = Fg[q][0][0] + Fg[q][1][0];
        gm[q][A][1] = Fg[q][0][1] + Fg[q][1][1];
        gm[q][A][2] = Fg[q][1][2] - Fg[q][0][2];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int v = 0; v < NV; ++v)
            zv[q][A][c][v] = fma(M.l[v * NV + 1], Ff[q][1][c],
                                 fma(M.l[v * NV + 0], Ff[q][0][c], 0.0));
      }
      yc[A] = y + (int64_t)Fva * colf + (l0 + sl) * CH;
      if (!GUARD || k + 1 < len)
        prefetch(std::integral_constant<int, (P + 1) % G2>{}, k + 1);
      if constexpr (FILL && A < 2) return;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const double det = prism_abs_detj_12(
            gm[q][0][0], gm[q][0][1], gm[q][0][2], gm[q][1][0], gm[q][1][1],
            gm[q][1][2], gm[q][2][0], gm[q][2][1], gm[q][2][2]);
        if constexpr (CSUM) {
          tr[q][A] = det * M.ta;
          const double dtb = det * M.tb;
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < NV; ++v)
              dr[q][A][c][v] =
                  dtb * (zv[q][0][c][v] + zv[q][1][c][v] + zv[q][2][c][v]);
        } else {
          const double dta = det * M.ta, dtb = det * M.tb;
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              const double d =
                  dtb * (zv[q][0][c][v] + zv[q][1][c][v] + zv[q][2][c][v]);
#pragma unroll
              for (int h = 0; h < 3; ++h)
                acc[h][c][v] = fma(dta, zv[q][h][c][v], acc[h][c][v] + d);
            }
        }
      }
    };
    using TF = std::true_type;
    using FF = std::false_type;
#define PM_P(N_) std::integral_constant<int, N_> {}
    // (loop period 6 = lcm of the window's 3 slots and the granule; the
    // position of step kb + i in its granule is i % G2)
    prefetch(PM_P(0), 0);
    step(PM_P(0), TF{}, TF{}, 0);
    step(PM_P(1 % G2), TF{}, TF{}, 1);
    step(PM_P(2 % G2), TF{}, TF{}, 2);
    // granule 0's cells, whole periods followed by at least one more step
    // (no guards: one scheduling block per step), then the guarded tail
    if (3 < len) step(PM_P(3 % G2), FF{}, TF{}, 3);
    if (4 < len) step(PM_P(4 % G2), FF{}, TF{}, 4);
    if (5 < len) step(PM_P(5 % G2), FF{}, TF{}, 5);
    int kb = 6;
    for (; kb + 6 < len; kb += 6) {
      step(PM_P(0), FF{}, FF{}, kb);
      step(PM_P(1 % G2), FF{}, FF{}, kb + 1);
      step(PM_P(2 % G2), FF{}, FF{}, kb + 2);
      step(PM_P(3 % G2), FF{}, FF{}, kb + 3);
      step(PM_P(4 % G2), FF{}, FF{}, kb + 4);
      step(PM_P(5 % G2), FF{}, FF{}, kb + 5);
    }
    for (; kb < len; kb += 6) {
      step(PM_P(0), FF{}, TF{}, kb);
      if (kb + 1 < len) step(PM_P(1 % G2), FF{}, TF{}, kb + 1);
      if (kb + 2 < len) step(PM_P(2 % G2), FF{}, TF{}, kb + 2);
      if (kb + 3 < len) step(PM_P(3 % G2), FF{}, TF{}, kb + 3);
      if (kb + 4 < len) step(PM_P(4 % G2), FF{}, TF{}, kb + 4);
      if (kb + 5 < len) step(PM_P(5 % G2), FF{}, TF{}, kb + 5);
    }
    add_tops();
#undef PM_P
    // the last window, oldest vertex first; a vertex that entered at step
    // j is in the cells formed at steps j, j+1, j+2 only: the ring slots of
    // cells that were never formed are cleared before its flush
    auto clear_cell = [&](auto A_) {
      constexpr int A = decltype(A_)::value;
      if constexpr (CSUM) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          tr[q][A] = 0.0;
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < NV; ++v) dr[q][A][c][v] = 0.0;
        }
      }
    };
    auto fin = [&](auto A1_, auto A2_, auto A3_) {
      using NOW = std::integral_constant<int, -1>;
      flush(A1_, NOW{});
      clear_cell(A1_);
      flush(A2_, NOW{});
      clear_cell(A2_);
      flush(A3_, NOW{});
    };
    using S0 = std::integral_constant<int, 0>;
    using S1 = std::integral_constant<int, 1>;
    using S2 = std::integral_constant<int, 2>;
    switch (len % 3) {
    case 0: fin(S0{}, S1{}, S2{}); break;
    case 1: fin(S1{}, S2{}, S0{}); break;
    default: fin(S2{}, S0{}, S1{}); break;
    }
    if constexpr (NC > 1) { // the last staged row
      __syncwarp();
      const double *prow = trow0 + (tb ^ 1) * TRP;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int i = sl + 32 * r;
        stma_red(pbase + i, prow[i < TR ? i : 0], plive & (i < nl * CH + CH));
      }
      __syncwarp();
    }
    gc += (uint32_t)ngran;
  }
}

template <int NC, int NQ, int NCH, int G2>
int stma_launch(const KronMat &M, const int32_t *strip_ptr,
                const int32_t *steps, int64_t n_strips, int layers,
                const double *coords, const double *x, double *y,
                int64_t n_vertices, cudaStream_t s) {
  // ring: 2 stages of 6 steps, or 4 stages of 3 (the same shared memory,
  // 9 instead of 6 steps of prefetch distance, smaller copies)
  constexpr int NS = 12 / G2;
  constexpr int MAXT = NC > 1 ? PM_TMA_MAXT_V
                              : (NQ > 1 ? PM_TMA_MAXT_S2 : PM_TMA_MAXT_S);
  const uint32_t Pf = stma_up16(8u * (layers + 1) * NC + 8);
  const uint32_t Pc = stma_up16(8u * (layers + 1) * 3 + 8);
  int dev = 0, smem_max = 0;
  PM_CUDA_TRY(cudaGetDevice(&dev));
  PM_CUDA_TRY(cudaDeviceGetAttribute(
      &smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  int ngrp = MAXT / 32 / NCH;
  if (ngrp > 15) ngrp = 15;
  if (const char *e = getenv("PM_TMA_GROUPS")) {
    const int v = atoi(e);
    if (v > 0 && v < ngrp) ngrp = v;
  }
  while (ngrp > 0 &&
         stma_smem(NC, G2, NS, ngrp, ngrp * NCH, Pf, Pc).total >
             (uint32_t)smem_max)
    --ngrp;
  if (ngrp < 1) {
    set_error("pm_column_mass_strip_tma: %d layers do not fit the column "
              "ring in shared memory", layers);
    return PM_EINVAL;
  }
  const StmaSmem L = stma_smem(NC, G2, NS, ngrp, ngrp * NCH, Pf, Pc);
  // FULL: every 32-layer chunk is whole (no lanes past a column's end)
  // (3-vector columns: the branch-free flush measured slower, C5b 7.18 vs
  // 6.02 ms, so they keep the predicated REDs; PM_TMA_VFULL=1 compiles it)
  const bool full = (NC == 1 || PM_TMA_VFULL) && layers % 32 == 0;
  auto kern = full ? k_strip_tma<NC, NQ, NS, NCH, MAXT,
                                 NC == 1 || PM_TMA_VFULL, G2>
                   : k_strip_tma<NC, NQ, NS, NCH, MAXT, false, G2>;
  static int cached_dev[2] = {-1, -1};
  if (cached_dev[full] != dev) {
    PM_CUDA_TRY(cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
    cached_dev[full] = dev;
  }
  int64_t want = (n_strips + ngrp - 1) / ngrp;
  const int64_t cap = sm_count();
  const unsigned grid = (unsigned)(want < cap ? (want < 1 ? 1 : want) : cap);
  kern<<<grid, ngrp * NCH * 32, L.total, s>>>(M, strip_ptr, steps, n_strips,
                                              layers, coords, x, y, ngrp, Pf,
                                              Pc, n_vertices);
  PM_LAUNCH_CHECK("k_strip_tma");
  return PM_OK;
}

// warps per group (32-layer chunks / chunks per warp) and ring depth
template <int NC, int NQ>
int stma_nch(int nch, [[maybe_unused]] int ns, const KronMat &M, const int32_t *strip_ptr,
             const int32_t *steps, int64_t n_strips, int layers,
             const double *coords, const double *x, double *y,
             int64_t n_vertices, cudaStream_t s) {
#if PM_TMA_HALF
#define PM_STMA_CASE(N_)                                                     \
  case N_:                                                                   \
    return ns == 4 ? stma_launch<NC, NQ, N_, 3>(M, strip_ptr, steps,         \
                                                n_strips, layers, coords, x, \
                                                y, n_vertices, s)            \
                   : stma_launch<NC, NQ, N_, 6>(M, strip_ptr, steps,         \
                                                n_strips, layers, coords, x, \
                                                y, n_vertices, s);
#else
#define PM_STMA_CASE(N_)                                                     \
  case N_:                                                                   \
    return stma_launch<NC, NQ, N_, 6>(M, strip_ptr, steps, n_strips, layers, \
                                      coords, x, y, n_vertices, s);
#endif
  switch (nch) {
    PM_STMA_CASE(1)
    PM_STMA_CASE(2)
    PM_STMA_CASE(3)
    PM_STMA_CASE(4)
  default:
    set_error("pm_column_mass_strip_tma: at most %d layers (got %d)",
              128 * NQ, layers);
    return PM_EINVAL;
  }
#undef PM_STMA_CASE
}

} // namespace
} // namespace pm

extern "C" int pm_column_mass_strip_tma(
    const int32_t *delta6, int32_t k, int32_t layers, const double *coords,
    const double *mtri, const double *mline, const double *x, double *y,
    int64_t n_dofs, int32_t accumulate, int64_t n_strips,
    const int32_t *strip_ptr, const int32_t *steps, int64_t n_vertices,
    void *stream) {
  pm::clear_error();
  const bool p1 = delta6 && delta6[0] == 1 && !delta6[1] && !delta6[2] &&
                  !delta6[3] && !delta6[4] && !delta6[5];
  const bool vp1 = delta6 && delta6[0] == 3 && !delta6[1] && !delta6[2] &&
                   !delta6[3] && !delta6[4] && !delta6[5];
  if (!p1 && !vp1) {
    pm::set_error("pm_column_mass_strip_tma: P1 or 3-vector P1 columns only");
    return PM_EINVAL;
  }
  const int nc = p1 ? 1 : 3;
  if (k != 6 * nc || layers < 1 || n_strips < 0 || n_vertices < 0 ||
      n_dofs != n_vertices * (int64_t)(layers + 1) * nc || !mtri || !mline) {
    pm::set_error("bad arguments to pm_column_mass_strip_tma");
    return PM_EINVAL;
  }
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(coords)) &
      15) {
    pm::set_error("pm_column_mass_strip_tma: x and coords must be 16-byte "
                  "aligned");
    return PM_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  pm::KronMat M;
  for (int i = 0; i < 9; ++i) M.t[i] = mtri[i];
  for (int i = 0; i < 4; ++i) M.l[i] = mline[i];
  if (!pm::kron_sym3(M)) {
    pm::set_error("pm_column_mass_strip_tma: the triangle factor must be "
                  "invariant under vertex permutations (ta I + tb J)");
    return PM_EINVAL;
  }
  pm::kron_fold12(M);
  if (!accumulate && n_dofs > 0)
    PM_CUDA_TRY(cudaMemsetAsync(y, 0, (size_t)n_dofs * sizeof(double), s));
  if (n_strips == 0) return PM_OK;
  if (!coords || !x || !y || !strip_ptr || !steps) {
    pm::set_error("NULL device pointer");
    return PM_EINVAL;
  }
  // ring shape: 2 stages of 6 steps; builds with -DPM_TMA_HALF=1 also hold
  // 4 stages of 3 steps (PM_TMA_NS=4: the same shared memory, 9 instead of
  // 6 steps of prefetch distance, smaller copies; measured slower, C5a 2.98
  // vs 2.36 ms, C5b 7.19 vs 6.27)
  int ns = 2;
  if (const char *e = getenv("PM_TMA_NS")) ns = atoi(e) == 4 ? 4 : 2;
  // two 32-layer chunks per warp for scalar columns when every warp's
  // second chunk is non-empty (PM_TMA_NQ=1: one chunk per warp)
  bool two = nc == 1 && layers > 32 && (layers - 1) % 64 >= 32;
  if (const char *e = getenv("PM_TMA_NQ")) two = two && atoi(e) != 1;
  const int nch = two ? (layers + 63) / 64 : (layers + 31) / 32;
  if (nc == 3)
    return pm::stma_nch<3, 1>(nch, ns, M, strip_ptr, steps, n_strips, layers,
                              coords, x, y, n_vertices, s);
  return two ? pm::stma_nch<1, 2>(nch, ns, M, strip_ptr, steps, n_strips,
                                  layers, coords, x, y, n_vertices, s)
             : pm::stma_nch<1, 1>(nch, ns, M, strip_ptr, steps, n_strips,
                                  layers, coords, x, y, n_vertices, s);
}
