// Device helpers and launch plumbing shared by the column-loop kernels.
#pragma once
#include <stdint.h>

#include "pm_common.cuh"

namespace pm {

constexpr int kMaxK = 18; // largest stencil built (P2 x P2, 3-vector P1)

template <int K> struct MassMat {
  double m[K * K]; // reference-prism mass matrix, row-major, slot order
};

// The same |det J| from per-vertex mid-layer positions and heights
// (xm_a, ym_a, dz_a), identical operation order.
__device__ __forceinline__ double
prism_abs_detj_mid(double xm0, double ym0, double dz0, double xm1, double ym1,
                   double dz1, double xm2, double ym2, double dz2) {
  const double a2 = (xm1 - xm0) * (ym2 - ym0) - (xm2 - xm0) * (ym1 - ym0);
  constexpr double kThird = 1.0 / 3.0;
  const double h = (dz0 + dz1 + dz2) * kThird;
  return fabs(a2 * h);
}

// The same with the constant factors left out (12 |det J| from per-vertex
// bottom+top sums of x, y and heights); callers fold 1/12 into their
// Kronecker factors (kron_fold12).
__device__ __forceinline__ double
prism_abs_detj_12(double xs0, double ys0, double dz0, double xs1, double ys1,
                  double dz1, double xs2, double ys2, double dz2) {
  const double a2 = (xs1 - xs0) * (ys2 - ys0) - (xs2 - xs0) * (ys1 - ys0);
  return fabs(a2 * (dz0 + dz1 + dz2));
}

// Reference-prism mass matrix as the tensor product of its triangle and
// interval factors: Mref[(c,h,v),(c,h',v')] = Mtri[h][h'] * Mline[v][v'].
struct KronMat {
  double t[36]; // Mtri, row-major (<= 6 x 6)
  double l[9];  // Mline, row-major (<= 3 x 3)
  // Mtri = ta I + tb J (3 x 3 with equal diagonal and equal off-diagonal
  // entries: P1 triangles under any symmetric rule), see kron_sym3
  double ta, tb;
  // 6 x 6 (vertices 0-2, edges 3-5, edge e opposite vertex e) invariant
  // under the vertex permutations: every 3 x 3 block is a I + b J,
  // p = {a1, a2 (vertex-vertex), c1, c2 (edge-edge), bm, b2 (vertex-edge)}
  double p[6];
};

// Does the 3 x 3 block at (r0, c0) of the nh x nh matrix t have the form
// a I + b J (to a relative 4 ulp of `big`)?
inline bool block_sym(const double *t, int nh, int r0, int c0, double big,
                      double *a, double *b) {
  double d = 0, o = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) (i == j ? d : o) += t[(r0 + i) * nh + c0 + j];
  d /= 3, o /= 6;
  const double tol = 4 * 2.220446049250313e-16 * big;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (fabs(t[(r0 + i) * nh + c0 + j] - (i == j ? d : o)) > tol)
        return false;
  *a = d - o;
  *b = o;
  return true;
}

// The 6 x 6 triangle factor of P2 in the block form of KronMat::p?
inline bool kron_sym6(KronMat &M) {
  double big = 0;
  for (int i = 0; i < 36; ++i) big = fmax(big, fabs(M.t[i]));
  double q[2];
  return block_sym(M.t, 6, 0, 0, big, &M.p[0], &M.p[1]) &&
         block_sym(M.t, 6, 3, 3, big, &M.p[2], &M.p[3]) &&
         block_sym(M.t, 6, 0, 3, big, &M.p[4], &M.p[5]) &&
         block_sym(M.t, 6, 3, 0, big, &q[0], &q[1]) &&
         fabs(q[0] - M.p[4]) <= 8 * 2.220446049250313e-16 * big &&
         fabs(q[1] - M.p[5]) <= 8 * 2.220446049250313e-16 * big;
}

// Scale the triangle-stage factors by 1/12 (the strip kernels accumulate
// with 12 |det J|, prism_abs_detj_12)
inline void kron_fold12(KronMat &M) {
  constexpr double k = 1.0 / 12.0;
  for (double &t : M.t) t *= k;
  M.ta *= k;
  M.tb *= k;
  for (double &q : M.p) q *= k;
}

// Does the 3 x 3 triangle factor have the form ta I + tb J (to a relative
// 4 ulp)?  Fills ta, tb from the averaged diagonal / off-diagonal.
inline bool kron_sym3(KronMat &M) {
  double d = 0, o = 0, big = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      (i == j ? d : o) += M.t[3 * i + j];
      big = fmax(big, fabs(M.t[3 * i + j]));
    }
  d /= 3, o /= 6;
  const double tol = 4 * 2.220446049250313e-16 * big;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (fabs(M.t[3 * i + j] - (i == j ? d : o)) > tol) return false;
  M.ta = d - o;
  M.tb = o;
  return true;
}

// |det J| of the affine map reference prism -> physical prism cell-layer.
// Vertex index v = 2a + b (a: triangle vertex, b: 0 bottom / 1 top level).
// Same operation order as the oracle (oracle/prismesh_oracle.c) except the
// mean height is a multiplication by 1/3 instead of a division (no DDIV
// sequence per cell-layer; differs from the oracle in the last bit only).
__device__ __forceinline__ double prism_abs_detj(const double *X,
                                                 const double *Y,
                                                 const double *Z) {
  const double xm0 = 0.5 * (X[0] + X[1]), ym0 = 0.5 * (Y[0] + Y[1]);
  const double xm1 = 0.5 * (X[2] + X[3]), ym1 = 0.5 * (Y[2] + Y[3]);
  const double xm2 = 0.5 * (X[4] + X[5]), ym2 = 0.5 * (Y[4] + Y[5]);
  const double a2 = (xm1 - xm0) * (ym2 - ym0) - (xm2 - xm0) * (ym1 - ym0);
  constexpr double kThird = 1.0 / 3.0;
  const double h = ((Z[1] - Z[0]) + (Z[3] - Z[2]) + (Z[5] - Z[4])) * kThird;
  return fabs(a2 * h);
}

// Everything a column-loop launch needs (host side).
struct LoopArgs {
  int k;
  int64_t n_cells; // cells in the launch (list length if `cells` != null)
  int layers;
  const int32_t *cells; // optional cell list (colour / order), device
  const int32_t *cmap, *coff, *xmap, *xoff;
  const double *coords, *mref, *x;
  const double *mtri, *mline; // Kronecker factors (host), may be NULL
  double *y;
  int accumulate;
  SlotTable st;
  bool dg_only;  // DoFs only on (2,1): contiguous (cell, layer, slot) field
  bool hshared;  // some DoF shared between columns
  cudaStream_t s;
  // fused halo (strip kernel): vertices v < ghost_end are owned by the
  // peer whose y (global-index window, peer memory) is y_peer
  double *y_peer = nullptr;
  int64_t ghost_end = 0;
  // store-first patch strips (pm_column_mass_patch_strips): the strips of
  // group p are item_ptr[p] .. item_ptr[p+1] (NULL: one strip per group);
  // store = flagged residencies store instead of adding
  const int32_t *item_ptr = nullptr;
  int store = 0;
  // strip kernels: the launch covers levels [lbeg, lend) of the columns in
  // chunks of its own width (mixed-width chunk plans, strip_red.cu)
  int lbeg = 0, lend = 0;
};

// y = det * (Mtri (x) Mline) x by sum factorisation over a layout's
// compile-time slot table T (NH x NV functions per component).
template <class LY>
__device__ __forceinline__ void kron_apply(const KronMat &M, const double *xv,
                                           double det, double *yv) {
  constexpr typename LY::Tab T = LY::make();
  constexpr int NH = LY::NH, NV = LY::NV, NC = LY::NC;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double z[NH][NV];
#pragma unroll
    for (int h = 0; h < NH; ++h)
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NV; ++w)
          s = fma(M.l[v * NV + w], xv[T.slot[c][h][w]], s);
        z[h][v] = s;
      }
#pragma unroll
    for (int h = 0; h < NH; ++h)
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double s = 0.0;
#pragma unroll
        for (int g = 0; g < NH; ++g) s = fma(M.t[h * NH + g], z[g][v], s);
        yv[T.slot[c][h][v]] = det * s;
      }
  }
}

// Kernel launchers (one translation unit each).
int launch_generic(const LoopArgs &a, bool atomic, int64_t cl_begin);
int launch_dg_stream(const LoopArgs &a, bool *handled, int64_t cl_begin = 0);
constexpr int kStreamT = 256; // cell-layers per DG stream unit (default)
int launch_column(const LoopArgs &a, const int32_t *delta6, bool colored);
int launch_cell_stream(const LoopArgs &a, const int32_t *delta6,
                       bool *handled);
bool column_supports(const int32_t *delta6);

} // namespace pm
