// Band-tile schedule for the vertex-column CG layouts (PM_VARIANT_TILE):
// P1, 3-vector P1, CG1 x DG0, CG1 x DG1.
//
// A persistent grid claims the tiles of pm_tiles_build (csrc/tile_plan.cpp)
// in index order through one atomic ticket.  Per tile:
//   1. one thread stages every vertex run of the tile -- whole columns of
//      the field and of the coordinate field, each run ONE contiguous byte
//      range under the reference numbering -- into shared memory with one
//      cp.async.bulk per run and array (TMA; no LSU / L1 traffic), completed
//      on an mbarrier;
//   2. meanwhile the CTA zeroes the output columns this tile touches first
//      and publishes that (flags[t] = epoch, release), then waits for the
//      tiles that zero its other vertices (always claimed earlier, so they
//      are running and never wait on this one): y needs no memset, and the
//      zeroed lines are still in L2 when the partial columns are added;
//   3. the warps walk the tile's sequential strips out of shared memory,
//      W lanes per segment, lane = layer of a W-layer chunk, exactly the
//      window / element kernel of k_strip_red (strip_red.cu): interval stage
//      once per entering vertex, triangle stage with |det J| folded into
//      the accumulation, one coalesced fp64 REDG per departing vertex.
// Tiles run in the mesh's cell order, i.e. along the RCM front: a vertex
// column is staged by the tiles of its two bands shortly one after the
// other (the second time from L2), and its output lines stay in L2 between
// zeroing and the last add.
#include "column_layout.cuh"
#include "pm_ptx.cuh"

#include <type_traits>

// Experimental schedule (slower than the strip kernels on every config,
// profiles/r02_tile_experiments.md): compiled only with PM_EXPERIMENTAL=1
// (build_native: PM_EXPERIMENTAL=1 in the environment); otherwise the entry
// points below report that and the library stays lean.
#ifndef PM_EXPERIMENTAL
#define PM_EXPERIMENTAL 0
#endif
#if PM_EXPERIMENTAL

namespace pm {

struct TilePlanDev {
  const int32_t *blob; // per-tile records (pm_tiles_blob)
  const int64_t *off;  // tile t = blob[off[t] .. off[t+1])
  // first-touch runs again, compact, for the zeroing warp
  const int32_t *zero_ptr, *zero_v0, *zero_n;
  int32_t *ctl;   // [1] CTAs done, [2] epoch (starts at 1)
  int32_t *flags; // per tile: epoch of its finished zeroing
  int32_t n_tiles;
  int32_t area_c;     // byte offset of the coordinate area in a data buffer
  int32_t data_bytes; // field area + coordinate area of one buffer
  int32_t max_slots;
  int32_t max_words;  // longest tile record
};

#ifndef PM_TILE_STAGES
#define PM_TILE_STAGES 4
#endif
#ifndef PM_TILE_LEAD
#define PM_TILE_LEAD 16
#endif
// Tiles are dealt statically: CTA c takes tiles c, c + G, c + 2G, ... (G =
// grid size), so every CTA knows its sequence and all CTAs sweep the tile
// order (the RCM front) together.  Warps 0 .. S-1 each own one tile
// buffer (stage) and stage the CTA's tiles i = b, b + S, ... into it;
// warp S zeroes the first-touch columns of the CTA's tiles and publishes
// them, running up to PM_TILE_LEAD tiles ahead of the walk (no buffer
// needed, so its fence / flag round trips are off the critical path); the
// other warps walk.
#ifndef PM_TILE_ZERO_BATCH
#define PM_TILE_ZERO_BATCH 16
#endif
constexpr int kTileStages = PM_TILE_STAGES;
constexpr int kTileLead = PM_TILE_LEAD;
// CTA work queue of warp items (a warp item = 32 / W consecutive (strip,
// chunk) items of one staged tile): slot = (sequence + 1) << 32 | item
constexpr int kTileQueue = 256;
constexpr int kTileZeroBatch = PM_TILE_ZERO_BATCH;
static_assert(kTileZeroBatch >= 1 && kTileZeroBatch <= 32, "zero batch");
// experiments only (wrong results): bit 0 = no dependency waits, bit 1 = no
// walk, bit 2 = no bulk copies
#ifndef PM_TILE_ABLATE
#define PM_TILE_ABLATE 0
#endif
// PM_TILE_TRACE: globaltimer stamps of CTAs 0..7 (experiments, pm_tile_trace)
#ifndef PM_TILE_TRACE
#define PM_TILE_TRACE 0
#endif
#if PM_TILE_TRACE
constexpr int kTrRounds = 256;
__device__ unsigned long long g_tile_trace[8][kTileStages + 2][kTrRounds][4];
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TL_STAMP(role, r, k)                                                 \
  do {                                                                       \
    if (blockIdx.x < 8 && lane == 0 && (r) < kTrRounds)                      \
      g_tile_trace[blockIdx.x][role][r][k] = tl_now();                       \
  } while (0)
#else
#define TL_STAMP(role, r, k)                                                 \
  do {                                                                       \
  } while (0)
#endif
static_assert(kTileStages >= 2 && kTileStages <= 4, "2..4 tile stages");
// CTA size: S producers and the zeroing warp, then walking warps up to 16
// warps in all (12 for the 3-vector layout, whose walk needs ~170
// registers): the walk is latency-bound, every resident warp counts
__host__ __device__ constexpr int tl_threads(int ch0) {
  return 32 * (ch0 > 2 ? 12 : 16);
}

// flush staging row per consumer segment (multi-channel columns:
// lane-contiguous REDs, as sr_trow in strip_red.cu)
__host__ __device__ constexpr int tl_trow(int ch0, int W) {
  return ch0 > 1 ? (W + 1) * ch0 : 0;
}
// shared memory: [barriers (full[S], empty[S], rec[2 S]), counters | work
// queue | 2 S tile records (a stage's next record arrives while it is
// walked) |
// S slot tables (int4 per slot) | flush rows | S data buffers]
__host__ __device__ constexpr int tl_meta_bytes(int max_words) {
  return (4 * max_words + 15) & ~15;
}
__host__ __device__ constexpr int tl_queue_off() { return 256; }
__host__ __device__ constexpr int tl_meta_off() {
  return tl_queue_off() + 8 * kTileQueue;
}
__host__ __device__ constexpr int tl_tab_off(int max_words) {
  return tl_meta_off() + 2 * kTileStages * tl_meta_bytes(max_words);
}
__host__ __device__ constexpr int tl_trow_off(int max_words, int max_slots) {
  return tl_tab_off(max_words) + kTileStages * 16 * max_slots;
}
__host__ __device__ constexpr int tl_data_off(int ch0, int W, int max_words,
                                              int max_slots) {
  return (tl_trow_off(max_words, max_slots) +
          8 * (tl_threads(ch0) / 32 - kTileStages - 1) * (32 / W) *
              tl_trow(ch0, W) +
          127) &
         ~127;
}

__device__ __forceinline__ void tl_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::
                   "r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n"
               " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
               " selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok)
               : "r"(smem_u32(bar)), "r"(parity)
               : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tl_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// flags: relaxed stores after one fence (a batch of tiles per fence),
// relaxed polls followed by one fence (no L1 invalidation per poll)
__device__ __forceinline__ void tl_st_relaxed(int32_t *p, int32_t v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v)
               : "memory");
}
__device__ __forceinline__ int32_t tl_ld_acquire(const int32_t *p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ int32_t tl_ld_relaxed(const int32_t *p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void tl_red(double *p, double v, bool on) {
  // no "memory" clobber: nothing in the kernel reads y back, so the
  // shared-memory loads of later steps may move above the REDs
  asm volatile("{\n\t.reg .pred q;\n\t"
               "setp.ne.b32 q, %2, 0;\n\t"
               "@q red.global.add.f64 [%0], %1;\n\t}" ::"l"(p),
               "d"(v), "r"((int)on));
}

// Bulk-copy geometry of one run [v0, v0 + n) of a column family with `colb`
// bytes per column at `base` (valid bytes: `limit`): 16-byte aligned source
// `src`, copied bytes `bytes` (0: nothing by bulk copy), the run's first
// column at `lead` bytes into the copy, and the tail [tail_from, end) of
// the last column that the bulk copy cannot take (a field ending 8 bytes
// past a 16-byte boundary) and a thread copies.
struct TlSpan {
  uintptr_t src;
  uint32_t bytes, lead;
  uintptr_t tail_from, end;
};
__device__ __forceinline__ TlSpan tl_span(const void *base, int64_t limit,
                                          int v0, int n, int colb) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(base) + (int64_t)v0 * colb;
  const uintptr_t end = a + (int64_t)n * colb;
  const uintptr_t lim = reinterpret_cast<uintptr_t>(base) + limit;
  TlSpan s;
  s.src = a & ~(uintptr_t)15;
  uintptr_t e = (end + 15) & ~(uintptr_t)15;
  if (e > lim) e -= 16;
  s.bytes = e > s.src ? (uint32_t)(e - s.src) : 0u;
  s.lead = (uint32_t)(a - s.src);
  s.tail_from = s.src + s.bytes;
  s.end = end;
  return s;
}

template <class LY, int W>
__global__ void __launch_bounds__(tl_threads(LY::CH0), 1)
k_tile(const KronMat M, const TilePlanDev P, int layers,
       const double *__restrict__ coords, const double *__restrict__ x,
       double *__restrict__ y, int64_t x_bytes, int64_t c_bytes) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NT = tl_threads(LY::CH0), NS = kTileStages;
  constexpr int SEGS = 32 / W, NCW = NT / 32 - NS - 1;
  constexpr int LV = LY::LV0, CH = LY::CH0, LVA = LV > 0 ? LV : 1;
  constexpr int NC = LY::NC, NV = LY::NV, NH = LY::NH;
  static_assert(NH == 3 && NC * NV == CH + LV, "vertex-column layout");
  static_assert(LV == 0 || (LV == NC && NV == 2 && CH == LV), "tile layout");
  constexpr int TR = tl_trow(LY::CH0, W);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col = layers * CH + LV; // doubles per vertex column
  const int colb = 8 * col;
  const int ccolb = 24 * (layers + 1);
  extern __shared__ __align__(128) unsigned char tl_sm[];
  uint64_t *const full = reinterpret_cast<uint64_t *>(tl_sm);
  uint64_t *const empty = full + NS;
  const int mbytes = tl_meta_bytes(P.max_words);
  auto meta_of = [&](int b, int r) { // stage b, round r
    return reinterpret_cast<int32_t *>(tl_sm + tl_meta_off() +
                                       (2 * b + (r & 1)) * mbytes);
  };
  uint64_t *const rec = empty + NS; // [2 S]: records landed
  int4 *const tab0 = reinterpret_cast<int4 *>(tl_sm + tl_tab_off(P.max_words));
  unsigned char *const data0 =
      tl_sm + tl_data_off(LY::CH0, W, P.max_words, P.max_slots);
  // tiles of this CTA walked so far (raised by the producers when a stage
  // comes back empty, read by the zeroing warp to bound its lead); the
  // work queue's head / tail, producers done, per stage its warp items and
  // how many are finished
  volatile int *const walked = reinterpret_cast<volatile int *>(tl_sm + 224);
  int *const q_head = reinterpret_cast<int *>(tl_sm + 128);
  int *const q_tail = reinterpret_cast<int *>(tl_sm + 132);
  int *const prod_done = reinterpret_cast<int *>(tl_sm + 136);
  int *const s_nitems = reinterpret_cast<int *>(tl_sm + 144); // [NS <= 4]
  int *const s_done = reinterpret_cast<int *>(tl_sm + 160);   // [NS <= 4]
  unsigned long long *const queue =
      reinterpret_cast<unsigned long long *>(tl_sm + tl_queue_off());
  if (tid == 0) {
    for (int b = 0; b < NS; ++b) {
      mbar_init(full + b, 1);
      mbar_init(empty + b, 1); // the warp finishing the stage's last item
      mbar_init(rec + 2 * b, 1);
      mbar_init(rec + 2 * b + 1, 1);
    }
    fence_mbar_init();
    *walked = 0;
    *q_head = 0;
    *q_tail = 0;
    *prod_done = 0;
  }
  for (int k = tid; k < kTileQueue; k += NT) queue[k] = 0ull;
  const int epoch = *reinterpret_cast<volatile int32_t *>(P.ctl + 2);
  const int G = gridDim.x, c0 = blockIdx.x;
  const int nchunks = (layers + W - 1) / W;
  __syncthreads();

  if (warp < NS) {
    // ================= producer of stage b = warp =========================
    // Round r stages the CTA's tile i = r S + b.  The tile's record arrives
    // by bulk copy one round ahead (its offsets two rounds ahead), the data
    // copies go out as soon as the stage is free, and the dependency flags
    // are checked while they are in flight.
    const int b = warp;
    unsigned char *datab = data0 + b * P.data_bytes;
    auto tile_of = [&](int r) { return c0 + (int64_t)G * (r * NS + b); };
    // record offsets of the next round (lane 0)
    int64_t nw0 = 0, nw1 = 0;
    auto fetch_off = [&](int r) {
      if (lane == 0 && tile_of(r) < P.n_tiles) {
        nw0 = __ldg(P.off + tile_of(r));
        nw1 = __ldg(P.off + tile_of(r) + 1);
      }
    };
    auto fetch_rec = [&](int r) { // bulk copy of round r's record
      if (lane == 0 && tile_of(r) < P.n_tiles) {
        const uint32_t bytes = (uint32_t)(4 * (nw1 - nw0));
        mbar_arrive_expect_tx(rec + 2 * b + (r & 1), bytes);
        bulk_g2s(meta_of(b, r), P.blob + nw0, bytes, rec + 2 * b + (r & 1));
      }
    };
    fetch_off(0);
    fetch_rec(0);
    fetch_off(1);
    for (int r = 0; tile_of(r) < P.n_tiles; ++r) {
      const int t = (int)tile_of(r);
      const int32_t *meta = meta_of(b, r);
      TL_STAMP(b, r, 0);
      if (r > 0) {
        // (back off between polls: a spinning producer steals issue slots)
        while (!mbar_try(empty + b, (r - 1) & 1)) __nanosleep(64);
        if (lane == 0) atomicMax((int *)walked, (r - 1) * NS + b + 1);
      }
      TL_STAMP(b, r, 1);
      // the next round's record buffer was this stage's round r-1 record,
      // free now: fetch it (offsets were loaded a round ago), then the
      // offsets of the round after
      fetch_rec(r + 1);
      fetch_off(r + 2);
      mbar_wait(rec + 2 * b + (r & 1), (r >> 1) & 1);
      const int nr = meta[0], nz = meta[1], nd = meta[2];
      const int32_t *runs = meta + 8, *dp = runs + 4 * nr + 2 * nz;
      if (lane == 0) { // whole vertex columns, one bulk copy per run/array
        uint32_t total = 0;
        for (int q = 0; q < nr; ++q)
          total += tl_span(x, x_bytes, runs[4 * q], runs[4 * q + 1], colb).bytes +
                   tl_span(coords, c_bytes, runs[4 * q], runs[4 * q + 1], ccolb)
                       .bytes;
        if (PM_TILE_ABLATE & 4) total = 0;
        tl_expect_tx(full + b, total);
        for (int q = 0; q < nr && !(PM_TILE_ABLATE & 4); ++q) {
          const TlSpan sf =
              tl_span(x, x_bytes, runs[4 * q], runs[4 * q + 1], colb);
          const TlSpan sc =
              tl_span(coords, c_bytes, runs[4 * q], runs[4 * q + 1], ccolb);
          if (sf.bytes)
            bulk_g2s(datab + runs[4 * q + 2],
                     reinterpret_cast<const void *>(sf.src), sf.bytes,
                     full + b);
          if (sc.bytes)
            bulk_g2s(datab + P.area_c + runs[4 * q + 3],
                     reinterpret_cast<const void *>(sc.src), sc.bytes,
                     full + b);
        }
      }
      // slot table: offsets (doubles from data0) of each slot's columns
      {
        int4 *tab = tab0 + b * P.max_slots;
        const int nslots = meta[5];
        const int dbase = b * (P.data_bytes >> 3);
        for (int s = lane; s < nslots; s += 32) {
          int q = 0, base = 0;
          while (base + runs[4 * q + 1] <= s) base += runs[4 * q + 1], ++q;
          const int v0 = runs[4 * q], v = v0 + (s - base);
          const uint32_t lf = (uint32_t)(
              (reinterpret_cast<uintptr_t>(x) + (int64_t)v0 * colb) & 15);
          const uint32_t lc = (uint32_t)(
              (reinterpret_cast<uintptr_t>(coords) + (int64_t)v0 * ccolb) & 15);
          const int fo =
              dbase + ((runs[4 * q + 2] + (int)lf + (s - base) * colb) >> 3);
          const int co = dbase + ((P.area_c + runs[4 * q + 3] + (int)lc +
                                   (s - base) * ccolb) >> 3);
          tab[s] = make_int4(fo, co, v, 0);
        }
      }
      // this tile's columns zeroed by their first tiles (own one included;
      // lower tile indices, published by zeroing warps that run ahead)
      // (acquire loads, no fence: a fence would also wait for the bulk
      // copies this lane just issued)
      for (int d0 = 0; d0 <= nd && !(PM_TILE_ABLATE & 1); d0 += 32) {
        const int d = d0 + lane < nd ? dp[d0 + lane] : t; // deps, then t
        while (!__all_sync(FULL, tl_ld_acquire(P.flags + d) == epoch))
          __nanosleep(64);
      }
      __syncwarp();
      if (lane == 0) {
        // the rare field tail a bulk copy cannot take (disjoint bytes)
        bool any = false;
        for (int q = 0; q < nr; ++q) {
          const TlSpan sf =
              tl_span(x, x_bytes, runs[4 * q], runs[4 * q + 1], colb);
          const TlSpan sc =
              tl_span(coords, c_bytes, runs[4 * q], runs[4 * q + 1], ccolb);
          for (uintptr_t a = sf.tail_from; a < sf.end; a += 8, any = true)
            *reinterpret_cast<double *>(datab + runs[4 * q + 2] + (a - sf.src)) =
                *reinterpret_cast<const double *>(a);
          for (uintptr_t a = sc.tail_from; a < sc.end; a += 8, any = true)
            *reinterpret_cast<double *>(datab + P.area_c + runs[4 * q + 3] +
                                        (a - sc.src)) =
                *reinterpret_cast<const double *>(a);
        }
        if (any) fence_proxy_async_smem();
        tl_arrive(full + b); // release: slot table, tail
      }
      // the tile's warp items into the work queue (walking warps wait on
      // full[b] before they touch the stage)
      {
        const int nwi = (meta[3] * nchunks + SEGS - 1) / SEGS;
        int pos = 0;
        if (lane == 0) {
          s_done[b] = 0;
          s_nitems[b] = nwi;
          pos = atomicAdd(q_tail, nwi);
        }
        pos = __shfl_sync(FULL, pos, 0);
        __syncwarp();
        for (int k = lane; k < nwi; k += 32) {
          const unsigned item = (unsigned)b | ((unsigned)(r & 1) << 2) |
                                ((unsigned)k << 3);
          reinterpret_cast<volatile unsigned long long *>(
              queue)[(pos + k) % kTileQueue] =
              ((unsigned long long)(pos + k + 1) << 32) | item;
        }
      }
      __syncwarp();
      TL_STAMP(b, r, 2);
      TL_STAMP(b, r, 3);
    }
    // the last producer to finish tells every walking warp to stop
    __syncwarp();
    if (lane == 0 && atomicAdd(prod_done, 1) == NS - 1) {
      const int pos = atomicAdd(q_tail, NCW);
      for (int k = 0; k < NCW; ++k)
        reinterpret_cast<volatile unsigned long long *>(
            queue)[(pos + k) % kTileQueue] =
            ((unsigned long long)(pos + k + 1) << 32) | 0xffffffffu;
    }
  } else if (warp == NS) {
    // ================= zeroing warp: first-touch columns, published =======
    // kTileZeroBatch tiles at a time: lane j fetches tile j's run range and
    // its first two runs in parallel (no dependent round trip per tile),
    // then the warp stores the zeros, fences once and raises the flags
    constexpr int ZB = kTileZeroBatch;
    for (int i = 0; c0 + (int64_t)G * i < P.n_tiles; i += ZB) {
      TL_STAMP(NS + 1, i / ZB, 0);
      while (i - *walked > kTileLead) __nanosleep(512);
      TL_STAMP(NS + 1, i / ZB, 1);
      const int64_t tj = c0 + (int64_t)G * (i + lane);
      const bool tv = lane < ZB && tj < P.n_tiles;
      int zp0 = 0, zp1 = 0, v0a = 0, na = 0, v0b = 0, nb = 0;
      if (tv) {
        zp0 = __ldg(P.zero_ptr + tj);
        zp1 = __ldg(P.zero_ptr + tj + 1);
        if (zp1 > zp0) v0a = __ldg(P.zero_v0 + zp0), na = __ldg(P.zero_n + zp0);
        if (zp1 > zp0 + 1)
          v0b = __ldg(P.zero_v0 + zp0 + 1), nb = __ldg(P.zero_n + zp0 + 1);
      }
      auto zero_run = [&](int v0, int nv) {
        // 16-byte stores over the aligned middle, 8-byte ends
        double *yd = y + (int64_t)v0 * col;
        const int n = nv * col;
        const int head = (int)((reinterpret_cast<uintptr_t>(yd) >> 3) & 1);
        if (lane == 0 && head && n > 0) yd[0] = 0.0;
        double2 *ya = reinterpret_cast<double2 *>(yd + head);
        const int n2 = (n - head) >> 1;
        for (int k = lane; k < n2; k += 32) ya[k] = make_double2(0.0, 0.0);
        if (lane == 0 && n > head && ((n - head) & 1)) yd[n - 1] = 0.0;
      };
      for (int j = 0; j < ZB; ++j) {
        const int z0 = __shfl_sync(FULL, zp0, j), z1 = __shfl_sync(FULL, zp1, j);
        if (z1 > z0) zero_run(__shfl_sync(FULL, v0a, j), __shfl_sync(FULL, na, j));
        if (z1 > z0 + 1)
          zero_run(__shfl_sync(FULL, v0b, j), __shfl_sync(FULL, nb, j));
        for (int z = z0 + 2; z < z1; ++z) // rare: more than two runs
          zero_run(__ldg(P.zero_v0 + z), __ldg(P.zero_n + z));
      }
      __syncwarp();
      TL_STAMP(NS + 1, i / ZB, 2);
      __threadfence(); // cumulative: the warp's zero stores, then the flags
      TL_STAMP(NS + 1, i / ZB, 3);
      if (tv) tl_st_relaxed(P.flags + tj, epoch);
      __syncwarp();
    }
  } else {
    // ================= consumers: walk the staged tiles' strips ===========
    const int sl = lane % W, seg = lane / W;
    const int cw = warp - NS - 1;
    double *trow = reinterpret_cast<double *>(
                       tl_sm + tl_trow_off(P.max_words, P.max_slots)) +
                   (cw * SEGS + seg) * TR;
    const double *data = reinterpret_cast<const double *>(data0);
    for (int qi = 0;; ++qi) {
      // next warp item of the CTA queue
      int k = 0;
      if (lane == 0) k = atomicAdd(q_head, 1);
      k = __shfl_sync(FULL, k, 0);
      unsigned long long e;
      while (true) {
        e = reinterpret_cast<volatile unsigned long long *>(
            queue)[k % kTileQueue];
        if ((int)(e >> 32) == k + 1) break;
        __nanosleep(32);
      }
      const unsigned wi = (unsigned)e;
      if (wi == 0xffffffffu) break;
      const int b = wi & 3, rp = (wi >> 2) & 1, wk = wi >> 3;
      if (cw == 0) TL_STAMP(NS, qi, 0);
      mbar_wait(full + b, rp);
      if (cw == 0) TL_STAMP(NS, qi, 1);
      const int32_t *meta = meta_of(b, rp);
      const int nr = meta[0], nz = meta[1], nd = meta[2], ns = meta[3];
      const int32_t *strips = meta + 8 + 4 * nr + 2 * nz + nd;
      const int16_t *steps =
          reinterpret_cast<const int16_t *>(strips + 2 * ns);
      const int4 *tab = tab0 + b * P.max_slots;
      const int n_items = ns * nchunks;
      if (!(PM_TILE_ABLATE & 2)) {
        const int item = wk * SEGS + seg;
        const bool has = item < n_items;
        const int si = has ? item / nchunks : 0;
        const int l0 = has ? (item % nchunks) * W : 0;
        const int16_t *stp = steps + strips[2 * si];
        const int len = has ? strips[2 * si + 1] : 0;
        int maxlen = len;
#pragma unroll
        for (int o = W; o < 32; o <<= 1)
          maxlen = max(maxlen, __shfl_xor_sync(FULL, maxlen, o));
        const int nl = has ? min(W, layers - l0) : 0;
        // lanes past the chunk read (finite) data of the column's last layer
        const int lc = min(l0 + sl, layers - 1);
        double *yl = y + (int64_t)(l0 + sl) * CH;
        double zv[3][NC][NV], gm[3][3], acc[3][NC][NV];
        double *yc[3] = {yl, yl, yl};
        bool live[3] = {false, false, false};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < NV; ++v) zv[a][c][v] = 0.0, acc[a][c][v] = 0.0;
#pragma unroll
          for (int q = 0; q < 3; ++q) gm[a][q] = 0.0;
        }
        // software pipeline: step k's data is in registers when step k
        // starts, the slot entry of step k+1 and the slot id of step k+2
        // too (every strip has >= 3 steps; segments without item: slot 0)
        double fc[2][CH], gc[2][3], fn[2][CH], gn[2][3];
        auto load = [&](const int4 &e, double (&f)[2][CH], double (&g)[2][3]) {
          const double *ef = data + e.x, *ec = data + e.y;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
#pragma unroll
            for (int c = 0; c < CH; ++c)
              f[j][c] = (j == 0 || c < LV) ? ef[(lc + j) * CH + c] : 0.0;
#pragma unroll
            for (int q = 0; q < 3; ++q) g[j][q] = ec[3 * (lc + j) + q];
          }
        };
        const int4 e0 = tab[len > 0 ? stp[0] : 0];
        int4 en = tab[len > 1 ? stp[1] : 0];
        int sid2 = len > 2 ? stp[2] : 0;
        load(e0, fc, gc);
        int gid = e0.z;

        auto flush = [&](auto A_) {
          constexpr int A = decltype(A_)::value;
          double vb[CH], vt[LVA];
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              const double a = acc[A][c][v];
              if (LV == 0)
                vb[v * NC + c] = a;
              else if (v == 0)
                vb[c] = a;
              else
                vt[c < LVA ? c : 0] = a;
              acc[A][c][v] = 0.0;
            }
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            double v0 = vb[c];
            if (c < LV) {
              const double below =
                  __shfl_up_sync(FULL, vt[c < LV ? c : 0], 1, W);
              if (sl > 0) v0 += below;
            }
            if constexpr (TR > 0) {
              if (sl < nl) trow[sl * CH + c] = v0;
              if (c < LV && sl == nl - 1)
                trow[(sl + 1) * CH + c] = vt[c < LV ? c : 0];
            } else {
              tl_red(yc[A] + c, v0, live[A] && sl < nl);
              if (c < LV)
                tl_red(yc[A] + CH + c, vt[c < LV ? c : 0],
                       live[A] && sl == nl - 1);
            }
          }
          if constexpr (TR > 0) { // lane-contiguous REDs of the staged chunk
            __syncwarp();
            double *const base = yc[A] - sl * CH;
            const int n = nl * CH + LV;
#pragma unroll
            for (int r = 0; r < (TR + W - 1) / W; ++r) {
              const int i = sl + W * r;
              tl_red(base + i, trow[i < TR ? i : 0], live[A] && i < n);
            }
            __syncwarp();
          }
        };

        auto step = [&](auto A_, auto FILL_, int k) {
          constexpr int A = decltype(A_)::value;
          constexpr bool FILL = decltype(FILL_)::value;
          if (!FILL) flush(A_);
          const bool act = k < len;
          // next step's data, the slot entry after it, the id after that
          load(en, fn, gn);
          const int gid_n = en.z;
          en = tab[sid2];
          sid2 = k + 3 < len ? stp[k + 3] : 0;
          // bottom + top sums of x, y and the height (1/4, 1/3 of |det J|
          // live in the folded Kronecker factors, kron_fold12)
          gm[A][0] = gc[0][0] + gc[1][0];
          gm[A][1] = gc[0][1] + gc[1][1];
          gm[A][2] = gc[1][2] - gc[0][2];
          yc[A] = yl + (int64_t)gid * col;
          live[A] = act;
          // interval stage of the entering vertex
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              double s = 0.0;
#pragma unroll
              for (int w = 0; w < NV; ++w) {
                const double xw = LV == 0 ? fc[0][w * NC + c]
                                  : w == 0 ? fc[0][c]
                                           : fc[1][c];
                s = fma(M.l[v * NV + w], xw, s);
              }
              zv[A][c][v] = s;
            }
#pragma unroll
          for (int j = 0; j < 2; ++j) {
#pragma unroll
            for (int c = 0; c < CH; ++c) fc[j][c] = fn[j][c];
#pragma unroll
            for (int q = 0; q < 3; ++q) gc[j][q] = gn[j][q];
          }
          gid = gid_n;
          if (FILL && A < 2) return; // window not full yet
          const double dj = prism_abs_detj_12(gm[0][0], gm[0][1], gm[0][2],
                                              gm[1][0], gm[1][1], gm[1][2],
                                              gm[2][0], gm[2][1], gm[2][2]);
          const double det = act ? dj : 0.0;
          const double dta = det * M.ta, dtb = det * M.tb;
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              const double d =
                  dtb * (zv[0][c][v] + zv[1][c][v] + zv[2][c][v]);
#pragma unroll
              for (int h = 0; h < 3; ++h)
                acc[h][c][v] = fma(dta, zv[h][c][v], acc[h][c][v] + d);
            }
        };
        using S0 = std::integral_constant<int, 0>;
        using S1 = std::integral_constant<int, 1>;
        using S2 = std::integral_constant<int, 2>;
        using TF = std::true_type;
        using FF = std::false_type;
        step(S0{}, TF{}, 0);
        step(S1{}, TF{}, 1);
        step(S2{}, TF{}, 2);
        for (int k = 3; k < maxlen; k += 3) {
          step(S0{}, FF{}, k);
          step(S1{}, FF{}, k + 1);
          step(S2{}, FF{}, k + 2);
        }
        flush(S0{});
        flush(S1{});
        flush(S2{});
      }
      __syncwarp();
      if (cw == 0) TL_STAMP(NS, qi, 2);
      // the warp finishing the stage's last item frees it
      if (lane == 0 && atomicAdd(s_done + b, 1) == s_nitems[b] - 1)
        tl_arrive(empty + b);
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(P.ctl + 1, 1) == (int)gridDim.x - 1) {
      P.ctl[1] = 0;
      __threadfence();
      atomicAdd(P.ctl + 2, 1);
    }
  }
}

template <class LY, int W>
static int tile_launch(const KronMat &M, const TilePlanDev &P, int layers,
                       const double *coords, const double *x, double *y,
                       int64_t x_bytes, int64_t c_bytes, cudaStream_t s) {
  constexpr int NT = tl_threads(LY::CH0);
  const int smem = tl_data_off(LY::CH0, W, P.max_words, P.max_slots) +
                   kTileStages * P.data_bytes;
  auto kern = k_tile<LY, W>;
  // attribute and occupancy per (kernel, smem size): cached, not per call
  static int cached_smem = -1, cached_blocks = 0, cached_dev = -1;
  int dev = 0;
  PM_CUDA_TRY(cudaGetDevice(&dev));
  if (cached_smem != smem || cached_dev != dev) {
    PM_CUDA_TRY(cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int nb = 0;
    PM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &nb, kern, NT, smem));
    if (nb < 1) {
      set_error("tile kernel: %d bytes of shared memory per CTA do not fit",
                smem);
      return PM_EINVAL;
    }
    cached_smem = smem;
    cached_blocks = nb;
    cached_dev = dev;
  }
  int64_t grid = (int64_t)sm_count() * cached_blocks;
  if (grid > P.n_tiles) grid = P.n_tiles;
  if (grid < 1) return PM_OK;
  kern<<<(unsigned)grid, NT, smem, s>>>(M, P, layers, coords, x, y,
                                                  x_bytes, c_bytes);
  PM_LAUNCH_CHECK("k_tile");
  return PM_OK;
}

template <class LY>
static int tile_w(const double *mtri, const double *mline,
                  const TilePlanDev &P, int layers, const double *coords,
                  const double *x, double *y, int64_t x_bytes,
                  int64_t c_bytes, int W, cudaStream_t s) {
  KronMat M{};
  for (int i = 0; i < 9; ++i) M.t[i] = mtri[i];
  for (int i = 0; i < LY::NV * LY::NV; ++i) M.l[i] = mline[i];
  if (!kron_sym3(M)) {
    set_error("pm_column_mass_tile: the triangle factor is not invariant "
              "under vertex permutations (a I + b J)");
    return PM_EINVAL;
  }
  kron_fold12(M);
  switch (W) {
  case 32: return tile_launch<LY, 32>(M, P, layers, coords, x, y, x_bytes, c_bytes, s);
  case 16: return tile_launch<LY, 16>(M, P, layers, coords, x, y, x_bytes, c_bytes, s);
  case 8: return tile_launch<LY, 8>(M, P, layers, coords, x, y, x_bytes, c_bytes, s);
  default:
    set_error("tile chunk width must be 8, 16 or 32 (got %d)", W);
    return PM_EINVAL;
  }
}

} // namespace pm

// bytes of shared memory in front of the data buffers, the buffer count
// and the CTA size (pm_column_mass_tile's CTA = offset + stages * data_bytes)
extern "C" int pm_tile_smem_layout(const int32_t *delta6, int32_t max_words,
                                   int32_t max_slots, int32_t width,
                                   int32_t *stages, int32_t *threads) {
  if (stages) *stages = pm::kTileStages;
  if (threads) *threads = pm::tl_threads(delta6[0] + delta6[1]);
  return pm::tl_data_off(delta6[0] + delta6[1], width, max_words, max_slots);
}

extern "C" int pm_column_mass_tile(const int32_t *delta6, int32_t layers,
                                   const double *coords, int64_t n_coords,
                                   const double *mtri, const double *mline,
                                   const double *x, double *y, int64_t n_dofs,
                                   const int32_t *blob, const int64_t *off,
                                   const int32_t *zero_ptr,
                                   const int32_t *zero_v0,
                                   const int32_t *zero_n, int32_t *ctl,
                                   int32_t *flags,
                                   int32_t n_tiles, int32_t area_c,
                                   int32_t data_bytes, int32_t max_slots,
                                   int32_t max_words, int32_t width,
                                   void *stream) {
  using namespace pm;
  clear_error();
  if (!delta6 || !coords || !x || !y || !blob || !off || !zero_ptr ||
      !zero_v0 || !zero_n || !ctl || !flags ||
      !mtri || !mline || layers < 1 || n_tiles < 0 || n_dofs < 0 ||
      n_coords < 0 || max_slots < 1 || max_words < 1 || data_bytes < 0 ||
      area_c < 0 || (area_c & 15) || (data_bytes & 127)) {
    set_error("pm_column_mass_tile: bad arguments");
    return PM_EINVAL;
  }
  TilePlanDev P;
  P.blob = blob;
  P.off = off;
  P.zero_ptr = zero_ptr;
  P.zero_v0 = zero_v0;
  P.zero_n = zero_n;
  P.ctl = ctl;
  P.flags = flags;
  P.n_tiles = n_tiles;
  P.area_c = area_c;
  P.data_bytes = data_bytes;
  P.max_slots = max_slots;
  P.max_words = max_words;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t xb = 8 * n_dofs, cb = 8 * n_coords;
  using L1 = Layout<1, 0, 0, 0, 0, 0>;
  using LV3 = Layout<3, 0, 0, 0, 0, 0>;
  using LD0 = Layout<0, 1, 0, 0, 0, 0>;
  using LD1 = Layout<0, 2, 0, 0, 0, 0>;
  if (L1::matches(delta6))
    return tile_w<L1>(mtri, mline, P, layers, coords, x, y, xb, cb, width, s);
  if (LV3::matches(delta6))
    return tile_w<LV3>(mtri, mline, P, layers, coords, x, y, xb, cb, width, s);
  if (LD0::matches(delta6))
    return tile_w<LD0>(mtri, mline, P, layers, coords, x, y, xb, cb, width, s);
  if (LD1::matches(delta6))
    return tile_w<LD1>(mtri, mline, P, layers, coords, x, y, xb, cb, width, s);
  set_error("pm_column_mass_tile: layout not built into the tile kernel "
            "(P1, 3-vector P1, CG1 x DG0, CG1 x DG1)");
  return PM_EINVAL;
}

// experiments: copy the PM_TILE_TRACE stamps out (host buffer of
// 8 * (stages + 2) * 256 * 4 uint64); returns the stage count, 0 when the
// library was built without tracing
extern "C" int pm_tile_trace(unsigned long long *out) {
#if PM_TILE_TRACE
  if (cudaMemcpyFromSymbol(out, pm::g_tile_trace, sizeof(pm::g_tile_trace)) !=
      cudaSuccess)
    return -1;
  cudaMemset(&pm::g_tile_trace, 0, 0);
  return pm::kTileStages;
#else
  (void)out;
  return 0;
#endif
}

#else // !PM_EXPERIMENTAL

extern "C" int pm_tile_smem_layout(const int32_t *, int32_t, int32_t,
                                   int32_t, int32_t *stages,
                                   int32_t *threads) {
  if (stages) *stages = 0;
  if (threads) *threads = 0;
  return -1;
}

extern "C" int pm_column_mass_tile(const int32_t *, int32_t, const double *,
                                   int64_t, const double *, const double *,
                                   const double *, double *, int64_t,
                                   const int32_t *, const int64_t *,
                                   const int32_t *, const int32_t *,
                                   const int32_t *, int32_t *, int32_t *,
                                   int32_t, int32_t, int32_t, int32_t,
                                   int32_t, int32_t, void *) {
  pm::clear_error();
  pm::set_error("the tile schedule is experimental: rebuild with "
                "PM_EXPERIMENTAL=1");
  return PM_EINVAL;
}

extern "C" int pm_tile_trace(unsigned long long *) { return PM_EINVAL; }

#endif // PM_EXPERIMENTAL
