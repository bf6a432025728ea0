// User stencil kernels for iterate_columns (a
// StencilKernel is an arbitrary procedure over per-argument slot-value
// views).  The reference's consumers (Firedrake/PyOP2)
// generate C for each local kernel and compile it at run time; here the
// user's kernel is CUDA C++ compiled with NVRTC for sm_100a and inlined
// into a generated column loop (Alg. 3):
//
//   __device__ void pm_kernel(double *out, const double *const *in,
//                             long long cell, int layer);
//
// in[a][j]  = value of argument a at slot j of this cell-layer (gathered
//             through the bottom-layer map + layer * offset, Alg. 2);
// out[j]    = contribution to slot j of the output argument (starts at 0;
//             the loop adds it into the output field, the SPEC's +=).
//
// Two generated loops:
//   pm_stencil_atomic  -- thread per cell-layer, consecutive threads on
//                         consecutive layers of a column (coalesced column
//                         gathers), output by fp64 REDG;
//   pm_stencil_colored -- thread per cell of one colour (cells of a colour
//                         share no DoF), layers walked in order, plain +=:
//                         bitwise deterministic (SPEC.md:341 contract).
// NVRTC is loaded with dlopen and the driver API through
// cudaGetDriverEntryPoint, so the library still loads without either.
#include <cuda.h>
#include <dlfcn.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "pm_common.cuh"

namespace {

constexpr int kMaxArgs = 8;
constexpr int kMaxSlots = 64;

// ---- NVRTC (dlopen) -------------------------------------------------------
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram *nvrtcProgram_t;
struct Nvrtc {
  nvrtcResult_t (*create)(nvrtcProgram_t *, const char *, const char *, int,
                          const char *const *, const char *const *);
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char *const *);
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t *);
  nvrtcResult_t (*log)(nvrtcProgram_t, char *);
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t *);
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char *);
  nvrtcResult_t (*destroy)(nvrtcProgram_t *);
  const char *(*error_string)(nvrtcResult_t);
  bool ok = false;
};

const Nvrtc &nvrtc() {
  static Nvrtc n;
  static bool tried = false;
  if (tried) return n;
  tried = true;
  void *h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12",
                     RTLD_NOW | RTLD_LOCAL);
  if (!h) return n;
#define PM_SYM(f, name)                                                      \
  *reinterpret_cast<void **>(&n.f) = dlsym(h, name);                         \
  if (!n.f) return n;
  PM_SYM(create, "nvrtcCreateProgram")
  PM_SYM(compile, "nvrtcCompileProgram")
  PM_SYM(log_size, "nvrtcGetProgramLogSize")
  PM_SYM(log, "nvrtcGetProgramLog")
  PM_SYM(cubin_size, "nvrtcGetCUBINSize")
  PM_SYM(cubin, "nvrtcGetCUBIN")
  PM_SYM(destroy, "nvrtcDestroyProgram")
  PM_SYM(error_string, "nvrtcGetErrorString")
#undef PM_SYM
  n.ok = true;
  return n;
}

// ---- driver API (cudaGetDriverEntryPoint) ----------------------------------
struct Driver {
  CUresult (*load)(CUmodule *, const void *);
  CUresult (*unload)(CUmodule);
  CUresult (*get_function)(CUfunction *, CUmodule, const char *);
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned,
                     unsigned, unsigned, unsigned, CUstream, void **, void **);
  bool ok = false;
};

int driver(const Driver **out) {
  static Driver d;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char *names[4] = {"cuModuleLoadData", "cuModuleUnload",
                            "cuModuleGetFunction", "cuLaunchKernel"};
    void **slots[4] = {reinterpret_cast<void **>(&d.load),
                       reinterpret_cast<void **>(&d.unload),
                       reinterpret_cast<void **>(&d.get_function),
                       reinterpret_cast<void **>(&d.launch)};
    bool all = true;
    for (int i = 0; i < 4; ++i) {
      cudaDriverEntryPointQueryResult q;
      void *f = nullptr;
      if (cudaGetDriverEntryPoint(names[i], &f, cudaEnableDefault, &q) !=
              cudaSuccess ||
          q != cudaDriverEntryPointSuccess || !f) {
        all = false;
        break;
      }
      *slots[i] = f;
    }
    d.ok = all;
  }
  if (!d.ok) {
    pm::set_error("CUDA driver entry points (cuModuleLoadData, "
                  "cuLaunchKernel) not available");
    return PM_ECUDA;
  }
  *out = &d;
  return PM_OK;
}

// kernel parameter block (same layout in the generated source)
struct StencilArgs {
  const double *f[kMaxArgs];
  const int32_t *map[kMaxArgs];
  const int32_t *off[kMaxArgs];
  double *out;
  const int32_t *omap;
  const int32_t *ooff;
  const int32_t *cells;
  long long n;
  int layers;
};

struct Stencil {
  CUmodule mod = nullptr;
  CUfunction atomic = nullptr, colored = nullptr;
  int n_in = 0, k_out = 0;
  int k_in[kMaxArgs] = {};
};

std::string generated_source(const char *user, int n_in, const int32_t *k_in,
                             int k_out) {
  std::string s;
  char buf[256];
  int sum = 0;
  std::string ks = "{", offs = "{";
  for (int i = 0; i < n_in; ++i) {
    snprintf(buf, sizeof buf, "%s%d", i ? ", " : "", k_in[i]);
    ks += buf;
    snprintf(buf, sizeof buf, "%s%d", i ? ", " : "", sum);
    offs += buf;
    sum += k_in[i];
  }
  if (n_in == 0) {
    ks += "0";
    offs += "0";
  }
  ks += "}";
  offs += "}";
  snprintf(buf, sizeof buf,
           "#define PM_NIN %d\n#define PM_KOUT %d\n#define PM_KSUM %d\n",
           n_in, k_out, sum);
  s += buf;
  s += "__device__ constexpr int pm_kin[] = " + ks + ";\n";
  s += "__device__ constexpr int pm_koff[] = " + offs + ";\n";
  s += R"(struct pm_args {
  const double *f[8];
  const int *map[8];
  const int *off[8];
  double *out;
  const int *omap;
  const int *ooff;
  const int *cells;
  long long n;
  int layers;
};
#line 1 "user_kernel"
)";
  s += user;
  s += R"(
#line 1 "column_loop"
__device__ __forceinline__ void pm_gather(const pm_args &a, long long cell,
                                          int l, double *v,
                                          const double **in) {
#pragma unroll
  for (int i = 0; i < PM_NIN; ++i) {
    const int k = pm_kin[i];
    const int *m = a.map[i] + cell * k;
#pragma unroll
    for (int j = 0; j < k; ++j)
      v[pm_koff[i] + j] =
          a.f[i][(long long)m[j] + (long long)l * a.off[i][j]];
    in[i] = v + pm_koff[i];
  }
}

extern "C" __global__ void pm_stencil_atomic(const pm_args a) {
  const long long total = a.n * a.layers;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
       t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long c = t / a.layers;
    const int l = (int)(t - c * a.layers);
    const long long cell = a.cells ? a.cells[c] : c;
    double v[PM_KSUM > 0 ? PM_KSUM : 1];
    const double *in[PM_NIN > 0 ? PM_NIN : 1];
    pm_gather(a, cell, l, v, in);
    double o[PM_KOUT];
#pragma unroll
    for (int j = 0; j < PM_KOUT; ++j) o[j] = 0.0;
    pm_kernel(o, in, cell, l);
    const int *m = a.omap + cell * PM_KOUT;
#pragma unroll
    for (int j = 0; j < PM_KOUT; ++j)
      atomicAdd(a.out + (long long)m[j] + (long long)l * a.ooff[j], o[j]);
  }
}

extern "C" __global__ void pm_stencil_colored(const pm_args a) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
       c < a.n; c += (long long)gridDim.x * blockDim.x) {
    const long long cell = a.cells ? a.cells[c] : c;
    const int *m = a.omap + cell * PM_KOUT;
    for (int l = 0; l < a.layers; ++l) {
      double v[PM_KSUM > 0 ? PM_KSUM : 1];
      const double *in[PM_NIN > 0 ? PM_NIN : 1];
      pm_gather(a, cell, l, v, in);
      double o[PM_KOUT];
#pragma unroll
      for (int j = 0; j < PM_KOUT; ++j) o[j] = 0.0;
      pm_kernel(o, in, cell, l);
#pragma unroll
      for (int j = 0; j < PM_KOUT; ++j)
        a.out[(long long)m[j] + (long long)l * a.ooff[j]] += o[j];
    }
  }
}
)";
  return s;
}

// NVRTC: the generated column loop with the user's kernel -> sm_100a cubin
int compile_cubin(const char *source, int32_t n_in, const int32_t *k_in,
                  int32_t k_out, std::vector<char> *bin) {
  if (!source || n_in < 0 || n_in > kMaxArgs || (n_in > 0 && !k_in) ||
      k_out < 1 || k_out > kMaxSlots) {
    pm::set_error("stencil kernel: bad arguments (0 <= n_in <= %d, "
                  "1 <= k_out <= %d)", kMaxArgs, kMaxSlots);
    return PM_EINVAL;
  }
  for (int i = 0; i < n_in; ++i)
    if (k_in[i] < 1 || k_in[i] > kMaxSlots) {
      pm::set_error("stencil kernel: argument %d has %d slots", i, k_in[i]);
      return PM_EINVAL;
    }
  const Nvrtc &rt = nvrtc();
  if (!rt.ok) {
    pm::set_error("NVRTC (libnvrtc.so.12) not available");
    return PM_ECUDA;
  }
  const std::string src = generated_source(source, n_in, k_in, k_out);
  nvrtcProgram_t prog = nullptr;
  if (rt.create(&prog, src.c_str(), "pm_stencil.cu", 0, nullptr, nullptr)) {
    pm::set_error("nvrtcCreateProgram failed");
    return PM_ECUDA;
  }
  const char *opts[] = {"--gpu-architecture=sm_100a", "-std=c++17",
                        "-lineinfo", "-default-device"};
  const nvrtcResult_t cr = rt.compile(prog, 4, opts);
  if (cr) {
    size_t n = 0;
    rt.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) rt.log(prog, &log[0]);
    rt.destroy(&prog);
    pm::set_error("stencil kernel does not compile (%s):\n%s",
                  rt.error_string(cr), log.c_str());
    return PM_EINVAL;
  }
  size_t nbin = 0;
  rt.cubin_size(prog, &nbin);
  bin->resize(nbin);
  rt.cubin(prog, bin->data());
  rt.destroy(&prog);
  return PM_OK;
}

} // namespace

extern "C" int pm_stencil_check(const char *source, int32_t n_in,
                                const int32_t *k_in, int32_t k_out,
                                int64_t *cubin_bytes) {
  pm::clear_error();
  std::vector<char> bin;
  const int rc = compile_cubin(source, n_in, k_in, k_out, &bin);
  if (rc == PM_OK && cubin_bytes) *cubin_bytes = (int64_t)bin.size();
  return rc;
}

extern "C" int pm_stencil_compile(const char *source, int32_t n_in,
                                  const int32_t *k_in, int32_t k_out,
                                  void **handle) {
  pm::clear_error();
  if (!handle) {
    pm::set_error("pm_stencil_compile: NULL handle");
    return PM_EINVAL;
  }
  std::vector<char> bin;
  int rc = compile_cubin(source, n_in, k_in, k_out, &bin);
  if (rc) return rc;
  const Driver *drv = nullptr;
  rc = driver(&drv);
  if (rc) return rc;
  PM_CUDA_TRY(cudaFree(nullptr)); // the runtime's primary context is current
  Stencil *st = new Stencil;
  st->n_in = n_in;
  st->k_out = k_out;
  for (int i = 0; i < n_in; ++i) st->k_in[i] = k_in[i];
  CUresult e = drv->load(&st->mod, bin.data());
  if (e == CUDA_SUCCESS)
    e = drv->get_function(&st->atomic, st->mod, "pm_stencil_atomic");
  if (e == CUDA_SUCCESS)
    e = drv->get_function(&st->colored, st->mod, "pm_stencil_colored");
  if (e != CUDA_SUCCESS) {
    if (st->mod) drv->unload(st->mod);
    delete st;
    pm::set_error("loading the stencil module failed (CUresult %d)", (int)e);
    return PM_ECUDA;
  }
  *handle = st;
  return PM_OK;
}

extern "C" int pm_stencil_launch(void *handle, int32_t colored,
                                 int64_t n_cells, int32_t layers,
                                 const double *const *in_fields,
                                 const int32_t *const *in_maps,
                                 const int32_t *const *in_offsets,
                                 double *out, const int32_t *out_map,
                                 const int32_t *out_offsets,
                                 const int32_t *cells, void *stream) {
  pm::clear_error();
  Stencil *st = static_cast<Stencil *>(handle);
  if (!st || n_cells < 0 || layers < 0 || !out || !out_map ||
      !out_offsets || (st->n_in > 0 && (!in_fields || !in_maps ||
                                        !in_offsets))) {
    pm::set_error("pm_stencil_launch: bad arguments");
    return PM_EINVAL;
  }
  if (n_cells == 0 || layers == 0) return PM_OK;
  StencilArgs a = {};
  for (int i = 0; i < st->n_in; ++i) {
    if (!in_fields[i] || !in_maps[i] || !in_offsets[i]) {
      pm::set_error("pm_stencil_launch: NULL pointer for argument %d", i);
      return PM_EINVAL;
    }
    a.f[i] = in_fields[i];
    a.map[i] = in_maps[i];
    a.off[i] = in_offsets[i];
  }
  a.out = out;
  a.omap = out_map;
  a.ooff = out_offsets;
  a.cells = cells;
  a.n = n_cells;
  a.layers = layers;
  const Driver *drv = nullptr;
  int rc = driver(&drv);
  if (rc) return rc;
  const int T = 128;
  const int64_t work = colored ? n_cells : n_cells * layers;
  const unsigned grid = pm::grid_for(work, T, 8);
  void *params[] = {&a};
  const CUresult e =
      drv->launch(colored ? st->colored : st->atomic, grid, 1, 1, T, 1, 1, 0,
                  (CUstream)stream, params, nullptr);
  if (e != CUDA_SUCCESS) {
    pm::set_error("stencil launch failed (CUresult %d)", (int)e);
    return PM_ECUDA;
  }
  return PM_OK;
}

extern "C" int pm_stencil_free(void *handle) {
  pm::clear_error();
  Stencil *st = static_cast<Stencil *>(handle);
  if (!st) return PM_OK;
  const Driver *drv = nullptr;
  if (st->mod && driver(&drv) == PM_OK) drv->unload(st->mod);
  delete st;
  return PM_OK;
}
