// Microbenchmark of the data movement of a band-tile CG kernel (no element
// math): C5a-shaped P1 field (N0 x 65 doubles) + coordinates (N0 x 195),
// synthetic RCM bands (vertex id = diag * LD + pos), a tile = P positions of
// diagonal d and P + 1 of d + 1 (two contiguous vertex runs), loaded in two
// 33-level chunks.  Variants:
//   A: 2-D TMA boxes over "vertex pair" rows (row stride 2 columns, always a
//      multiple of 16 bytes), even / odd vertices in separate boxes
//   B: one 1-D bulk copy per vertex chunk (16-byte aligned superset)
//   C: 16-byte LDG + STS by the whole CTA
//   out: + per tile the f-shaped partial columns added back (A: 1-D bulk
//      reduce per vertex chunk, C: REDG per element)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ubench_tile.cu -o ubench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int LAY = 64, LV = LAY + 1, CLV = 3 * LV;
constexpr int LD = 2049;            // diagonal length
constexpr int CW = 32;              // layers per chunk
constexpr int FB = 34, CB = 100;    // box widths (doubles, 16-byte multiples)

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void expect(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t *b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\nW%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}\n" ::"r"(su(b)), "r"(ph) : "memory"); }
__device__ __forceinline__ void tma2d(void *dst, const CUtensorMap *m, int c0, int c1, uint64_t *b) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(su(dst)), "l"(m), "r"(c0), "r"(c1), "r"(su(b)) : "memory"); }
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t n, uint64_t *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su(dst)), "l"(src), "r"(n), "r"(su(b)) : "memory"); }
__device__ __forceinline__ void bulk_red(double *dst, const void *src, uint32_t n) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;"
               ::"l"(dst), "r"(su(src)), "r"(n) : "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

struct Tile { int a, na, b, nb; };

__device__ __forceinline__ Tile tile_of(int t, int P, int n_diag) {
  const int per = (LD + P - 1) / P;
  const int d = t / per, p = (t % per) * P;
  Tile T;
  T.a = d * LD + p; T.na = min(P, LD - p);
  T.b = (d + 1) * LD + p; T.nb = min(P + 1, LD - p);
  return T;
}

// ---- A: 2-D TMA pair-row boxes -------------------------------------------
template <bool OUT>
__global__ void __launch_bounds__(128) kA(const __grid_constant__ CUtensorMap mf,
                                         const __grid_constant__ CUtensorMap mc,
                                         int ntiles, int P, int *ctr, double *y,
                                         double *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int R = P / 2 + 2;                       // pair rows per run
  const int FS = (R * FB + 15) / 16 * 16, CS = (R * CB + 15) / 16 * 16; // 128 B aligned boxes
  double *fb = (double *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023); // [2 runs][2 par][FS]
  double *cb = fb + 4 * FS;                       // [2 runs][2 par][CS]
  uint64_t *bar = (uint64_t *)(cb + 4 * CS);
  __shared__ int tk;
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  uint32_t ph = 0;
  double acc = 0;
  const uint32_t bytes = 4 * R * (FB + CB) * 8;
  for (;;) {
    if (threadIdx.x == 0) tk = atomicAdd(ctr, 1);
    __syncthreads();
    const int t = tk;
    if (t >= ntiles) break;
    const Tile T = tile_of(t, P, 0);
    for (int ch = 0; ch < 2; ++ch) {
      const int l0 = ch * CW;
      if (threadIdx.x == 0) {
        expect(bar, bytes);
        const int r0[2] = {T.a >> 1, T.b >> 1};
        for (int r = 0; r < 2; ++r)
          for (int q = 0; q < 2; ++q) {
            // box starts must be 16-byte aligned: odd vertices start one
            // double early (LV, CLV odd)
            tma2d(fb + (r * 2 + q) * FS, &mf, q * (LV - 1) + l0, r0[r], bar);
            tma2d(cb + (r * 2 + q) * CS, &mc, q * (CLV - 1) + 3 * l0, r0[r], bar);
          }
      }
      mwait(bar, ph); ph ^= 1;
      // touch every loaded double once (stand-in for the strip walk)
      for (int i = threadIdx.x; i < 4 * R * (FB + CB); i += blockDim.x) acc += fb[i];
      __syncthreads();
      if (OUT) {
        // partial columns back: one 1-D bulk reduce per vertex chunk
        if (threadIdx.x < 32) {
          fence_async();
          for (int i = threadIdx.x; i < T.na + T.nb; i += 32) {
            const int v = i < T.na ? T.a + i : T.b + (i - T.na);
            const int r = i < T.na ? 0 : 1, base = r ? T.b : T.a;
            const int q = v & 1, row = (v >> 1) - (base >> 1);
            const double *src = fb + (r * 2 + q) * FS + row * FB;
            double *dst = y + (size_t)v * LV + l0;
            // 16-byte aligned destination span: shift by the parity
            const int sh = (int)(((uintptr_t)dst) >> 3) & 1;
            bulk_red(dst - sh, src, 8 * 32 + (sh ? 0 : 0));
          }
          bulk_commit();
          bulk_wait_read0();
        }
        __syncthreads();
      }
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

// ---- B: 1-D bulk per vertex chunk ------------------------------------------
__global__ void __launch_bounds__(128) kB(const double *f, const double *c,
                                         int ntiles, int P, int *ctr, double *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int NV = 2 * P + 1;
  double *fb = (double *)sm;               // [NV][36]
  double *cb = fb + NV * 36;               // [NV][102]
  uint64_t *bar = (uint64_t *)(cb + NV * 102);
  __shared__ int tk;
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  uint32_t ph = 0;
  double acc = 0;
  for (;;) {
    if (threadIdx.x == 0) tk = atomicAdd(ctr, 1);
    __syncthreads();
    const int t = tk;
    if (t >= ntiles) break;
    const Tile T = tile_of(t, P, 0);
    const int nv = T.na + T.nb;
    for (int ch = 0; ch < 2; ++ch) {
      const int l0 = ch * CW;
      if (threadIdx.x < 32) {
        // each lane: bytes of its copies, summed by the warp for expect_tx
        uint32_t my = 0;
        for (int i = threadIdx.x; i < nv; i += 32) {
          const int v = i < T.na ? T.a + i : T.b + (i - T.na);
          const double *fs = f + (size_t)v * LV + l0;
          const double *cs = c + (size_t)v * CLV + 3 * l0;
          const int fsh = (int)((uintptr_t)fs >> 3) & 1, csh = (int)((uintptr_t)cs >> 3) & 1;
          my += ((33 + fsh + 1) / 2) * 16 + ((99 + csh + 1) / 2) * 16;
        }
        for (int o = 16; o; o >>= 1) my += __shfl_xor_sync(~0u, my, o);
        if (threadIdx.x == 0) expect(bar, my);
        __syncwarp();
        for (int i = threadIdx.x; i < nv; i += 32) {
          const int v = i < T.na ? T.a + i : T.b + (i - T.na);
          const double *fs = f + (size_t)v * LV + l0;
          const double *cs = c + (size_t)v * CLV + 3 * l0;
          const int fsh = (int)((uintptr_t)fs >> 3) & 1, csh = (int)((uintptr_t)cs >> 3) & 1;
          bulk(fb + i * 36, fs - fsh, ((33 + fsh + 1) / 2) * 16, bar);
          bulk(cb + i * 102, cs - csh, ((99 + csh + 1) / 2) * 16, bar);
        }
      }
      mwait(bar, ph); ph ^= 1;
      for (int i = threadIdx.x; i < nv * 138; i += blockDim.x) acc += fb[i];
      __syncthreads();
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

// ---- C: LDG.128 + STS -------------------------------------------------------
template <bool OUT>
__global__ void __launch_bounds__(128) kC(const double *f, const double *c,
                                         int ntiles, int P, int *ctr, double *y, double *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int NV = 2 * P + 1;
  double *fb = (double *)sm;               // [NV][36]
  double *cb = fb + NV * 36;
  __shared__ int tk;
  double acc = 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) tk = atomicAdd(ctr, 1);
    __syncthreads();
    const int t = tk;
    if (t >= ntiles) break;
    const Tile T = tile_of(t, P, 0);
    const int nv = T.na + T.nb;
    for (int ch = 0; ch < 2; ++ch) {
      const int l0 = ch * CW;
      for (int i = w; i < nv; i += 4) {   // warp per vertex chunk
        const int v = i < T.na ? T.a + i : T.b + (i - T.na);
        const double *fs = f + (size_t)v * LV + l0;
        const double *cs = c + (size_t)v * CLV + 3 * l0;
        const int fsh = (int)((uintptr_t)fs >> 3) & 1, csh = (int)((uintptr_t)cs >> 3) & 1;
        if (lane < 17) {
          double2 d = reinterpret_cast<const double2 *>(fs - fsh)[lane];
          reinterpret_cast<double2 *>(fb + i * 36)[lane] = d;
        }
        for (int k = lane; k < 50; k += 32) {
          double2 d = reinterpret_cast<const double2 *>(cs - csh)[k];
          reinterpret_cast<double2 *>(cb + i * 102)[k] = d;
        }
      }
      __syncthreads();
      for (int i = threadIdx.x; i < nv * 138; i += blockDim.x) acc += fb[i];
      if (OUT) {
        for (int i = w; i < nv; i += 4) {
          const int v = i < T.na ? T.a + i : T.b + (i - T.na);
          atomicAdd(y + (size_t)v * LV + l0 + lane, fb[i * 36 + lane]);
          if (lane == 0) atomicAdd(y + (size_t)v * LV + l0 + 32, fb[i * 36 + 32]);
        }
      }
      __syncthreads();
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

// ---- D: full columns, one 1-D bulk copy per run and array -----------------
__global__ void __launch_bounds__(128) kD(const double *f, const double *c,
                                         int ntiles, int P, int *ctr, double *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int NV = 2 * P + 2;
  double *fb = (double *)(((uintptr_t)sm + 127) & ~(uintptr_t)127);
  double *cb = fb + NV * LV + 8;
  uint64_t *bar = (uint64_t *)(cb + NV * CLV + 8);
  __shared__ int tk;
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  uint32_t ph = 0;
  double acc = 0;
  for (;;) {
    if (threadIdx.x == 0) tk = atomicAdd(ctr, 1);
    __syncthreads();
    const int t = tk;
    if (t >= ntiles) break;
    const Tile T = tile_of(t, P, 0);
    if (threadIdx.x == 0) {
      uint32_t tot = 0;
      const int s[2] = {T.a, T.b}, n[2] = {T.na, T.nb};
      uint32_t fo = 0, co = 0, fbytes[2], cbytes[2], fsh[2], csh[2];
      for (int r = 0; r < 2; ++r) {
        const double *fs = f + (size_t)s[r] * LV, *cs = c + (size_t)s[r] * CLV;
        fsh[r] = ((uintptr_t)fs >> 3) & 1; csh[r] = ((uintptr_t)cs >> 3) & 1;
        fbytes[r] = ((n[r] * LV + fsh[r] + 1) / 2) * 16; cbytes[r] = ((n[r] * CLV + csh[r] + 1) / 2) * 16;
        tot += fbytes[r] + cbytes[r];
      }
      expect(bar, tot);
      for (int r = 0; r < 2; ++r) {
        const double *fs = f + (size_t)s[r] * LV, *cs = c + (size_t)s[r] * CLV;
        bulk(fb + fo, fs - fsh[r], fbytes[r], bar); fo += fbytes[r] / 8;
        bulk(cb + co, cs - csh[r], cbytes[r], bar); co += cbytes[r] / 8;
      }
    }
    mwait(bar, ph); ph ^= 1;
    for (int i = threadIdx.x; i < (T.na + T.nb) * LV; i += blockDim.x) acc += fb[i];
    __syncthreads();
  }
  if (acc == 12345.678) sink[0] = acc;
}

__global__ void kcopy(const double2 *a, double2 *b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
// L2-resident read bandwidth: every CTA re-reads a 32 MB window
__global__ void kl2(const double2 *a, size_t n, int reps, double *sink) {
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 d = __ldcg(a + i); s += d.x + d.y; }
  if (s == 1.2345) sink[0] = s;
}

int main(int argc, char **argv) {
  const int P = argc > 1 ? atoi(argv[1]) : 32;
  const int ndiag = 2049;
  const size_t N0 = (size_t)LD * ndiag;
  double *f, *c, *y, *sink; int *ctr;
  CK(cudaMalloc(&f, N0 * LV * 8)); CK(cudaMalloc(&c, N0 * CLV * 8));
  CK(cudaMalloc(&y, N0 * LV * 8)); CK(cudaMalloc(&sink, 64)); CK(cudaMalloc(&ctr, 4));
  CK(cudaMemset(f, 0, N0 * LV * 8)); CK(cudaMemset(c, 0, N0 * CLV * 8)); CK(cudaMemset(y, 0, N0 * LV * 8));
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
  auto mk = [&](void *base, uint64_t rowlen, uint32_t boxw, uint32_t boxr) {
    CUtensorMap m; cuuint64_t dims[2] = {rowlen, N0 / 2}; cuuint64_t str[1] = {rowlen * 8};
    cuuint32_t box[2] = {boxw, boxr}; cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
    return m; };
  const int R = P / 2 + 2;
  CUtensorMap mf = mk(f, 2 * LV, FB, R), mc = mk(c, 2 * CLV, CB, R);
  const int per = (LD + P - 1) / P;
  const int ntiles = per * (ndiag - 1);
  const double uniq = (double)N0 * (LV + CLV) * 8;
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto timeit = [&](const char *name, auto launch, double extra_bytes) {
    float best = 1e9;
    for (int it = 0; it < 4; ++it) {
      CK(cudaMemset(ctr, 0, 4));
      CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (it) best = ms < best ? ms : best;
    }
    printf("%-28s P=%d %8.3f ms  unique-input %7.1f GB/s  (+out %7.1f GB/s)\n", name, P, best,
           uniq / best / 1e6, (uniq + extra_bytes) / best / 1e6);
  };
  size_t smD = (2 * P + 2) * (LV + CLV) * 8 + 1024;
  CK(cudaFuncSetAttribute(kD, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smD));
  size_t smA = 4 * ((R * FB + 15) / 16 * 16 + (R * CB + 15) / 16 * 16) * 8 + 1024 + 64, smB = (2 * P + 1) * 138 * 8 + 64;
  CK(cudaFuncSetAttribute(kA<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA));
  CK(cudaFuncSetAttribute(kA<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA));
  CK(cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB));
  CK(cudaFuncSetAttribute(kC<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB));
  CK(cudaFuncSetAttribute(kC<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB));
  printf("tiles %d, smem A %zu B %zu\n", ntiles, smA, smB);
  for (int cps : {2, 3, 4, 6}) {
    int g = sms * cps;
    printf("-- %d CTAs/SM\n", cps);
    if (smA * cps < 225000) {
      timeit("A tma2d", [&] { kA<false><<<g, 128, smA>>>(mf, mc, ntiles, P, ctr, y, sink); }, 0);
      timeit("A tma2d + bulk-red out", [&] { kA<true><<<g, 128, smA>>>(mf, mc, ntiles, P, ctr, y, sink); }, (double)N0 * LV * 8);
    }
    if (smD * cps < 225000)
      timeit("D full-column bulk per run", [&] { kD<<<g, 128, smD>>>(f, c, ntiles, P, ctr, sink); }, 0);
    if (smB * cps < 220000) {
      timeit("B bulk per vertex", [&] { kB<<<g, 128, smB>>>(f, c, ntiles, P, ctr, sink); }, 0);
      timeit("C ldg128", [&] { kC<false><<<g, 128, smB>>>(f, c, ntiles, P, ctr, y, sink); }, 0);
      timeit("C ldg128 + redg out", [&] { kC<true><<<g, 128, smB>>>(f, c, ntiles, P, ctr, y, sink); }, (double)N0 * LV * 8);
    }
  }
  // references: copy bandwidth, L2 read bandwidth
  {
    size_t n = N0 * LV * 8 / 16;
    timeit("copy f->y (r+w)", [&] { kcopy<<<sms * 8, 256>>>((double2 *)f, (double2 *)y, n); }, 0);
    float best = 1e9;
    for (int it = 0; it < 4; ++it) {
      CK(cudaEventRecord(e0)); kl2<<<sms * 8, 256>>>((double2 *)f, (32u << 20) / 16, 20, sink);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      if (it) best = ms < best ? ms : best; }
    printf("L2 read 32MB x20: %.3f ms = %.1f GB/s\n", best, 20.0 * (32 << 20) / best / 1e6);
  }
  return 0;
}
