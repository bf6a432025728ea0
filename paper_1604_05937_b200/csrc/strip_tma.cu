// Run-strip schedule for vertex-column CG layouts with level DoFs (P1 and
// 3-vector P1): the strip-REDG walk of strip_red.cu, fed by bulk copies
// (cp.async.bulk, the 1-D TMA path) of WHOLE vertex columns, several columns
// per copy.
//
// On a level-ordered base mesh (RCM, ordering.py:45-90) a sequential strip
// that follows the band between two BFS levels (pm_build_run_strips) takes
// its even vertices from one run of consecutive ids and its odd vertices
// from another.  Under Alg. 1 (fspace.py:141-147) consecutive vertex ids are
// consecutive columns of the field, so G strip steps of one side are ONE
// contiguous slab of the field and one of the coordinate field.  A group of
// NCH warps (one per 32-layer chunk of the column) walks a strip in lock
// step out of a shared ring of NS stages, each stage = a granule of 2G
// steps (G columns per side): 4 bulk copies per granule instead of
// 5-6 cp.async rows per step and warp, which is what bound the cp.async
// ring (L1 data pipe 84 %, profiles/README.md).  Granules whose ids are not
// consecutive fall back to one copy per column (any strip plan is valid
// input; only the speed depends on the runs).
//
// The warp of a group that releases a granule last refills its stage with
// the granule NS ahead (smem counter), completion by mbarrier transaction
// bytes; the refilling warp also writes each step's smem offsets and vertex
// id into a per-stage table (one broadcast LDS.128 per step for the
// consumers).  Element kernel, window and flushes as k_strip_red (one level
// per lane, symmetric triangle factor ta I + tb J).
#include "column_layout.cuh"
#include "column_loop.cuh"
#include "pm_ptx.cuh"

#include <cstdlib>
#include <type_traits>

// CTA size caps (registers per thread = 65536 / cap): scalar / 3-vector
#ifndef PM_TMA_MAXT_S
#define PM_TMA_MAXT_S 512
#endif
#ifndef PM_TMA_MAXT_V
#define PM_TMA_MAXT_V 384
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
__device__ __forceinline__ void stma_group_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

constexpr uint32_t stma_up16(uint32_t b) { return (b + 15u) & ~15u; }

// smem carve-up (bytes), shared by the kernel and the launcher
struct StmaSmem {
  uint32_t off_tab, bars, cnt, trow, ring, zero, total;
};
__host__ __device__ inline StmaSmem stma_smem(int NC, int G, int NS, int ngrp,
                                              int nwarp, uint32_t Pf,
                                              uint32_t Pc) {
  StmaSmem s;
  uint32_t o = 0;
  s.off_tab = o, o += (uint32_t)ngrp * NS * 2 * G * 16;
  s.bars = o, o += (uint32_t)ngrp * NS * 8;
  s.cnt = o, o += stma_up16((uint32_t)ngrp * NS * 4);
  s.trow = o, o += NC > 1 ? (uint32_t)nwarp * 2 * (33 * NC + 1) * 8 : 0;
  o = (o + 127u) & ~127u;
  s.ring = o, o += (uint32_t)ngrp * NS * 2 * G * (Pf + Pc);
  s.zero = o, o += (Pf > Pc ? Pf : Pc);
  o += 1024; // lanes past a partial chunk read past their column (never used)
  s.total = o;
  return s;
}

template <int NC, int G, int NS, int NCH, int MAXT>
__global__ void __launch_bounds__(MAXT, 1)
k_strip_tma(const KronMat M, const int32_t *__restrict__ strip_ptr,
            const int32_t *__restrict__ steps, int64_t n_strips, int layers,
            const double *__restrict__ coords, const double *__restrict__ x,
            double *__restrict__ y, int ngrp, uint32_t Pf, uint32_t Pc,
            int64_t n_vertices) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int CH = NC, NV = 2;
  constexpr int G2 = 2 * G;
  constexpr int TR = NC > 1 ? 33 * NC : 0;     // staged chunk row
  constexpr int TRP = 33 * NC + 1;             // row pitch (doubles)
  constexpr int NR = NC > 1 ? (TR + 31) / 32 : 1;
  extern __shared__ __align__(128) unsigned char stma_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nwarp = blockDim.x >> 5;
  const int grp = wib / NCH, chunk = wib % NCH;
  const StmaSmem L = stma_smem(NC, G, NS, ngrp, nwarp, Pf, Pc);
  StmaEntry *const tab =
      reinterpret_cast<StmaEntry *>(stma_raw + L.off_tab) + grp * NS * G2;
  uint64_t *const full = reinterpret_cast<uint64_t *>(stma_raw + L.bars) +
                         grp * NS;
  int *const cnt = reinterpret_cast<int *>(stma_raw + L.cnt) + grp * NS;
  double *const trow0 =
      reinterpret_cast<double *>(stma_raw + L.trow) + wib * 2 * TRP;
  const uint32_t SB = G2 * (Pf + Pc); // stage bytes
  const uint32_t ring_off = L.ring + (uint32_t)grp * NS * SB;
  const uint32_t zero_off = L.zero;

  for (uint32_t i = threadIdx.x; i < (L.total - L.zero) / 8; i += blockDim.x)
    reinterpret_cast<double *>(stma_raw + L.zero)[i] = 0.0;
  if (threadIdx.x < (unsigned)(ngrp * NS)) {
    mbar_init(reinterpret_cast<uint64_t *>(stma_raw + L.bars) + threadIdx.x, 1);
    reinterpret_cast<int *>(stma_raw + L.cnt)[threadIdx.x] = 0;
  }
  fence_mbar_init();
  __syncthreads();

  const int colf = (layers + 1) * NC; // doubles per field column
  const int colc = (layers + 1) * 3;  // doubles per coordinate column
  const int l0 = chunk * 32;
  const int nl = min(32, layers - l0); // cell-layers of this warp's chunk
  const int sl = lane;
  const double *const x_end = x + n_vertices * colf;
  const double *const c_end = coords + n_vertices * colc;

  // Refill: stage `st` <- granule `g` of the strip (steps k0 + 2G g ..).
  // One converged warp; lane t < 2G looks after step 2G g + t.
  // `v`: the lane's step id, loaded by the caller (a granule ahead).
  auto refill = [&](int st, int g, int k0, int len, int v) {
    const int t = lane, k = G2 * g + t;
    const bool valid = t < G2 && k < len;
    const int side = t & 1, j = t >> 1;
    const int vfirst = __shfl_sync(FULL, v, side);
    const unsigned sidemask = 0x55555555u << side;
    const unsigned bad = __ballot_sync(FULL, valid && v != vfirst + j);
    const unsigned vmask = __ballot_sync(FULL, valid);
    const bool consec = !(bad & sidemask);
    const int nside = __popc(vmask & sidemask);
    const uint32_t side_base = ring_off + (uint32_t)st * SB +
                               (uint32_t)side * G * (Pf + Pc);
    uint64_t *const bar = full + st;
    if (valid) {
      const int vb = consec ? vfirst : v;      // first column of the copy
      const int jb = consec ? 0 : j;           // its slot in the side
      const int nb = consec ? nside : 1;       // columns in the copy
      const bool issue = !consec || j == 0;
      const double *fs = x + (int64_t)vb * colf;
      const double *cs = coords + (int64_t)vb * colc;
      const uint32_t fsh = (uint32_t)(reinterpret_cast<uintptr_t>(fs) >> 3) & 1;
      const uint32_t csh = (uint32_t)(reinterpret_cast<uintptr_t>(cs) >> 3) & 1;
      // consecutive columns lie back to back, single ones at the padded pitch
      const uint32_t fdst = side_base + (consec ? 0u : (uint32_t)jb * Pf);
      const uint32_t cdst = side_base + G * Pf + (consec ? 0u : (uint32_t)jb * Pc);
      StmaEntry e;
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
    // every warp of the group is done with the previous strip's stages
    if constexpr (NCH > 1)
      stma_group_sync(1 + grp, NCH * 32);
    else
      __syncwarp();
    if (chunk == 0) {
      for (int i = 0; i < NS && i < ngran; ++i) {
        const int kk = G2 * i + lane;
        refill((int)((gc + i) % NS), i, k0, len,
               (lane < G2 && kk < len) ? __ldg(steps + k0 + kk) : 0);
      }
    }
    // ids of granule NS (refilled at the first release of this strip)
    int vpre = 0;
    {
      const int kk = G2 * NS + lane;
      vpre = (lane < G2 && kk < len) ? __ldg(steps + k0 + kk) : 0;
    }
    double zv[3][NC][NV], gm[3][3], acc[3][NC][NV];
    constexpr bool CSUM = NC == 1;
    double tr[CSUM ? 3 : 1], dr[CSUM ? 3 : 1][NC][NV];
#pragma unroll
    for (int a = 0; a < (CSUM ? 3 : 1); ++a) {
      tr[a] = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int v = 0; v < NV; ++v) dr[a][c][v] = 0.0;
    }
    double *yc[3] = {y, y, y};
    bool live[3] = {false, false, false};
    int tb = 0;
    double *pbase = y;
    bool plive = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int v = 0; v < NV; ++v) zv[a][c][v] = 0.0, acc[a][c][v] = 0.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) gm[a][q] = 0.0;
    }
    int cur_st = 0;

    auto flush = [&](auto A_) {
      constexpr int A = decltype(A_)::value;
      double *const trow = trow0 + tb * TRP;
      double pv[NR];
      if constexpr (NC > 1) { // the previous row's values (staged, synced)
        const double *prow = trow0 + (tb ^ 1) * TRP;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const int i = sl + 32 * r;
          pv[r] = prow[i < TR ? i : 0];
        }
      }
      if constexpr (CSUM) {
        const double t = tr[0] + tr[1] + tr[2];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int v = 0; v < NV; ++v)
            acc[A][c][v] = fma(zv[A][c][v], t,
                               dr[0][c][v] + dr[1][c][v] + dr[2][c][v]);
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double vt = acc[A][c][1];
        double v0 = acc[A][c][0];
        acc[A][c][0] = 0.0, acc[A][c][1] = 0.0;
        const double below = __shfl_up_sync(FULL, vt, 1);
        if (sl > 0) v0 += below;
        if constexpr (NC > 1) {
          if (sl < nl) trow[sl * CH + c] = v0;
          if (sl == nl - 1) trow[(sl + 1) * CH + c] = vt;
        } else {
          stma_red(yc[A] + c, v0, live[A] & (sl < nl));
          stma_red(yc[A] + CH + c, vt, live[A] & (sl == nl - 1));
        }
      }
      if constexpr (NC > 1) {
        // the previous row's REDs now (lane-contiguous); this row's at the
        // next flush (a __syncwarp of the step orders its STS before that)
        double *const base = yc[A] - sl * CH;
        const int n = nl * CH + CH;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const int i = sl + 32 * r;
          stma_red(pbase + i, pv[r], plive & (i < n));
        }
        pbase = base;
        plive = live[A];
        tb ^= 1;
      }
    };

    // Software pipeline: the column values of step k+1 are read out of the
    // ring (into F) in the middle of step k, after step k's own values were
    // consumed and before its cell arithmetic, so the two dependent LDS
    // (table entry, then the values) overlap ~40 fp64 instructions.
    double Ff[2][CH], Fg[2][3];
    int Fva = 0;
    bool Fact = false;
    auto prefetch = [&](int k) {
      const bool act = k < len;
      if (act && (k & (G2 - 1)) == 0) { // granule boundary (warp-uniform)
        const int g = k / G2;
        if (g > 0) {
          // release granule g-1 (its last values are in registers); the
          // last warp of the group to do so refills its stage with
          // granule g-1+NS
          __syncwarp();
          bool last = true;
          if constexpr (NCH > 1) {
            int l = 0;
            if (lane == 0) {
              __threadfence_block();
              l = atomicAdd(cnt + cur_st, 1) == NCH - 1;
              if (l) cnt[cur_st] = 0;
            }
            last = __shfl_sync(FULL, l, 0);
          }
          if (last && g - 1 + NS < ngran) {
            if constexpr (NCH > 1) __threadfence_block();
            refill(cur_st, g - 1 + NS, k0, len, vpre);
          }
          // ids of the granule the NEXT release refills (any warp of the
          // group may be the one): loaded a granule ahead of their use
          {
            const int kk = G2 * (g + NS) + lane;
            vpre = (lane < G2 && kk < len) ? __ldg(steps + k0 + kk) : 0;
          }
        }
        const uint32_t gg = gc + (uint32_t)g;
        cur_st = (int)(gg % NS);
        mbar_wait(full + cur_st, (gg / NS) & 1);
      }
      if constexpr (NC > 1)
        __syncwarp(); // the staged row's STS before the next flush's LDS
      const int4 e = *reinterpret_cast<const int4 *>(
          tab + cur_st * G2 + (k & (G2 - 1)));
      const uint32_t fo = act ? (uint32_t)e.x : zero_off;
      const uint32_t co = act ? (uint32_t)e.y : zero_off;
      Fva = act ? e.z : 0;
      Fact = act;
      const double *ef = reinterpret_cast<const double *>(stma_raw + fo) +
                         (l0 + sl) * CH;
      const double *ec = reinterpret_cast<const double *>(stma_raw + co) +
                         3 * (l0 + sl);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int c = 0; c < CH; ++c) Ff[j][c] = ef[j * CH + c];
#pragma unroll
        for (int q = 0; q < 3; ++q) Fg[j][q] = ec[3 * j + q];
      }
    };

    auto step = [&](auto A_, auto FILL_, int k) {
      constexpr int A = decltype(A_)::value;
      constexpr bool FILL = decltype(FILL_)::value;
      if (!FILL) flush(A_);
      const bool act = Fact;
      gm[A][0] = Fg[0][0] + Fg[1][0];
      gm[A][1] = Fg[0][1] + Fg[1][1];
      gm[A][2] = Fg[1][2] - Fg[0][2];
      yc[A] = y + (int64_t)Fva * colf + (l0 + sl) * CH;
      live[A] = act;
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int v = 0; v < NV; ++v)
          zv[A][c][v] = fma(M.l[v * NV + 1], Ff[1][c],
                            fma(M.l[v * NV + 0], Ff[0][c], 0.0));
      prefetch(k + 1);
      if (FILL && A < 2) return;
      const double dj = prism_abs_detj_12(gm[0][0], gm[0][1], gm[0][2],
                                          gm[1][0], gm[1][1], gm[1][2],
                                          gm[2][0], gm[2][1], gm[2][2]);
      const double det = act ? dj : 0.0;
      if constexpr (CSUM) {
        tr[A] = det * M.ta;
        const double dtb = det * M.tb;
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int v = 0; v < NV; ++v)
            dr[A][c][v] = dtb * (zv[0][c][v] + zv[1][c][v] + zv[2][c][v]);
      } else {
        const double dta = det * M.ta, dtb = det * M.tb;
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const double d = dtb * (zv[0][c][v] + zv[1][c][v] + zv[2][c][v]);
#pragma unroll
            for (int h = 0; h < 3; ++h)
              acc[h][c][v] = fma(dta, zv[h][c][v], acc[h][c][v] + d);
          }
      }
    };
    using S0 = std::integral_constant<int, 0>;
    using S1 = std::integral_constant<int, 1>;
    using S2 = std::integral_constant<int, 2>;
    using TF = std::true_type;
    using FF = std::false_type;
    prefetch(0);
    step(S0{}, TF{}, 0);
    step(S1{}, TF{}, 1);
    step(S2{}, TF{}, 2);
    for (int k = 3; k < len; k += 3) {
      step(S0{}, FF{}, k);
      step(S1{}, FF{}, k + 1);
      step(S2{}, FF{}, k + 2);
    }
    auto clear_cell = [&](auto A_) {
      constexpr int A = decltype(A_)::value;
      if constexpr (CSUM) {
        tr[A] = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int v = 0; v < NV; ++v) dr[A][c][v] = 0.0;
      }
    };
    flush(S0{});
    clear_cell(S0{});
    __syncwarp();
    flush(S1{});
    clear_cell(S1{});
    __syncwarp();
    flush(S2{});
    clear_cell(S2{});
    if constexpr (NC > 1) { // the last staged row
      __syncwarp();
      const double *prow = trow0 + (tb ^ 1) * TRP;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int i = sl + 32 * r;
        stma_red(pbase + i, prow[i < TR ? i : 0], plive && i < nl * CH + CH);
      }
      __syncwarp();
    }
    gc += (uint32_t)ngran;
  }
}

template <int NC, int G, int NCH, int NS>
int stma_launch(const KronMat &M, const int32_t *strip_ptr,
                const int32_t *steps, int64_t n_strips, int layers,
                const double *coords, const double *x, double *y,
                int64_t n_vertices, cudaStream_t s) {
  constexpr int MAXT = NC > 1 ? PM_TMA_MAXT_V : PM_TMA_MAXT_S;
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
         stma_smem(NC, G, NS, ngrp, ngrp * NCH, Pf, Pc).total >
             (uint32_t)smem_max)
    --ngrp;
  if (ngrp < 1) {
    set_error("pm_column_mass_strip_tma: %d layers do not fit the column "
              "ring in shared memory", layers);
    return PM_EINVAL;
  }
  const StmaSmem L = stma_smem(NC, G, NS, ngrp, ngrp * NCH, Pf, Pc);
  auto kern = k_strip_tma<NC, G, NS, NCH, MAXT>;
  static int cached_dev = -1;
  if (cached_dev != dev) {
    PM_CUDA_TRY(cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
    cached_dev = dev;
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

template <int NC, int G>
int stma_nch(int nch, int ns, const KronMat &M, const int32_t *strip_ptr,
             const int32_t *steps, int64_t n_strips, int layers,
             const double *coords, const double *x, double *y,
             int64_t n_vertices, cudaStream_t s) {
#define PM_STMA_CASE(N_)                                                     \
  case N_:                                                                   \
    return ns == 2 ? stma_launch<NC, G, N_, 2>(M, strip_ptr, steps, n_strips, \
                                               layers, coords, x, y,         \
                                               n_vertices, s)                \
                   : stma_launch<NC, G, N_, 3>(M, strip_ptr, steps, n_strips, \
                                               layers, coords, x, y,         \
                                               n_vertices, s);
  switch (nch) {
    PM_STMA_CASE(1)
    PM_STMA_CASE(2)
    PM_STMA_CASE(3)
    PM_STMA_CASE(4)
  default:
    set_error("pm_column_mass_strip_tma: at most 128 layers (got %d)", layers);
    return PM_EINVAL;
  }
#undef PM_STMA_CASE
}

template <int NC>
int stma_g(int g, int nch, int ns, const KronMat &M, const int32_t *strip_ptr,
           const int32_t *steps, int64_t n_strips, int layers,
           const double *coords, const double *x, double *y,
           int64_t n_vertices, cudaStream_t s) {
  if (g == 2)
    return stma_nch<NC, 2>(nch, ns, M, strip_ptr, steps, n_strips, layers, coords, x, y, n_vertices, s);
  return stma_nch<NC, 4>(nch, ns, M, strip_ptr, steps, n_strips, layers, coords, x, y, n_vertices, s);
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
  const int nch = (layers + 31) / 32;
  int g = 4;
  if (const char *e = getenv("PM_TMA_G")) g = atoi(e) == 2 ? 2 : 4;
  int ns = 3;
  if (const char *e = getenv("PM_TMA_NS")) ns = atoi(e) == 2 ? 2 : 3;
  return nc == 1 ? pm::stma_g<1>(g, nch, ns, M, strip_ptr, steps, n_strips, layers,
                                 coords, x, y, n_vertices, s)
                 : pm::stma_g<3>(g, nch, ns, M, strip_ptr, steps, n_strips, layers,
                                 coords, x, y, n_vertices, s);
}
