// Compile-time layout traits shared by the column and patch kernels.
#pragma once
#include "column_loop.cuh"

namespace pm {

// Compile-time restatement of the slot table (fspace.py:110-131) for a
// layout given as template arguments delta(d1,d2): the slot count, each
// slot's level kind, the bottom partner of each top copy and whether the
// DoF is shared with other columns are all constants, so the per-slot
// branches below vanish at compile time.
template <int D00, int D01, int D10, int D11, int D20, int D21>
struct Layout {
  struct Tab {
    int k;
    int8_t level[kMaxK];
    int8_t pair[kMaxK];
    int8_t hshare[kMaxK];
    int8_t offset[kMaxK]; // Alg. 2: delta(d,0) + delta(d,1)
    int8_t comp[kMaxK];   // vector component of the slot's basis function
    int8_t h[kMaxK];      // triangle basis function of the slot
    int8_t v[kMaxK];      // interval basis function of the slot
    int8_t slot[3][6][3]; // inverse map (comp, h, v) -> slot
    int8_t pos[kMaxK];    // entity position: vertex a -> a, edge e -> 3+e,
                          // cell -> 6
    int8_t ch[kMaxK];     // channel inside the entity's layer block
                          // (= the DoF's `within` minus level offset)
  };
  // The element of each built layout (quadrature.py element_for_layout):
  // triangle / interval basis sizes and the component count.
  struct Fam {
    int nh, nv, nc;
  };
  static constexpr Fam fam() {
    const bool v0 = !D10 && !D11 && !D20 && !D21;
    const bool c0 = !D00 && !D01 && !D10 && !D11;
    if (D00 == 1 && !D01 && v0) return {3, 2, 1};           // CG1 x CG1
    if (!D00 && D01 == 1 && v0) return {3, 1, 1};           // CG1 x DG0
    if (!D00 && D01 == 2 && v0) return {3, 2, 1};           // CG1 x DG1
    if (c0 && D20 == 1 && !D21) return {1, 2, 1};           // DG0 x CG1
    if (c0 && !D20 && D21 == 1) return {1, 1, 1};           // DG0 x DG0
    if (c0 && !D20 && D21 == 2) return {1, 2, 1};           // DG0 x DG1
    if (c0 && D20 == 3 && !D21) return {3, 2, 1};           // DG1 x CG1
    if (c0 && !D20 && D21 == 3) return {3, 1, 1};           // DG1 x DG0
    if (c0 && !D20 && D21 == 6) return {3, 2, 1};           // DG1 x DG1
    if (D00 == 1 && D01 == 1 && D10 == 1 && D11 == 1 && !D20 && !D21)
      return {6, 3, 1};                                     // P2 x P2
    if (D00 == 3 && !D01 && v0) return {3, 2, 3};           // 3-vector P1
    return {0, 0, 0};
  }
  static constexpr Tab make() {
    Tab t{};
    const int dl[3] = {D00, D10, D20}, dc[3] = {D01, D11, D21};
    const int n_local[3] = {3, 3, 1};
    int k = 0;
    for (int d = 0; d < 3; ++d) {
      if (!dl[d] && !dc[d]) continue;
      for (int loc = 0; loc < n_local[d]; ++loc) {
        const int first = k;
        const int8_t off = (int8_t)(dl[d] + dc[d]);
        const int8_t pos = (int8_t)(d == 0 ? loc : d == 1 ? 3 + loc : 6);
        for (int j = 0; j < dl[d]; ++j, ++k) {
          t.level[k] = 0, t.pair[k] = -1, t.hshare[k] = d != 2;
          t.offset[k] = off, t.pos[k] = pos, t.ch[k] = (int8_t)j;
        }
        for (int j = 0; j < dc[d]; ++j, ++k) {
          t.level[k] = 1, t.pair[k] = -1, t.hshare[k] = d != 2;
          t.offset[k] = off, t.pos[k] = pos, t.ch[k] = (int8_t)(dl[d] + j);
        }
        for (int j = 0; j < dl[d]; ++j, ++k) {
          t.level[k] = 2, t.pair[k] = (int8_t)(first + j);
          t.hshare[k] = d != 2;
          t.offset[k] = off, t.pos[k] = pos, t.ch[k] = (int8_t)j;
        }
      }
    }
    t.k = k;
    // slot -> (h, v, comp): the convention of DESIGN.md / quadrature.py
    // (oracle or_slot_basis restates it independently)
    const Fam f = fam();
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 6; ++b)
        for (int c = 0; c < 3; ++c) t.slot[a][b][c] = -1;
    for (int j = 0; j < k; ++j) {
      const int d = t.pos[j] < 3 ? 0 : t.pos[j] < 6 ? 1 : 2;
      const bool vcont = dl[d] > 0;
      const int lev = t.level[j];
      const int n_v = lev == 1 ? (vcont ? f.nv - 2 : f.nv) : 1;
      const int dof = lev == 1 ? t.ch[j] - dl[d] : t.ch[j];
      const int per = (n_v > 0 ? n_v : 1) * f.nc;
      const int hi = dof / per, rem = dof % per;
      const int vi = rem / f.nc, comp = rem % f.nc;
      t.h[j] = (int8_t)(d == 0 ? t.pos[j] : d == 1 ? t.pos[j] : hi);
      t.v[j] = (int8_t)(lev == 0 ? 0 : lev == 2 ? f.nv - 1
                                               : (vcont ? 1 : 0) + vi);
      t.comp[j] = (int8_t)comp;
      t.slot[comp][t.h[j]][t.v[j]] = (int8_t)j;
    }
    return t;
  }
  static constexpr int K = make().k;
  static constexpr int NH = fam().nh, NV = fam().nv, NC = fam().nc;
  // entity-level constants for the patch kernel
  static constexpr int CH0 = D00 + D01; // DoFs per layer block of a vertex
  static constexpr int CH1 = D10 + D11; // ... of an edge
  static constexpr int LV0 = D00, LV1 = D10; // level-copy DoFs
  static constexpr bool has_edges = (D10 + D11) > 0;
  static constexpr bool has_cells = (D20 + D21) > 0;
  static bool matches(const int32_t *d) {
    return d[0] == D00 && d[1] == D01 && d[2] == D10 && d[3] == D11 &&
           d[4] == D20 && d[5] == D21;
  }
};

// The layouts built into the column kernel: the nine CG1/DG0/DG1 tensor
// layouts (fspace.py:23-33), P2 x P2 and the 3-vector P1 (= COORDS).
#define PM_LAYOUTS(X)                                                        \
  X(1, 0, 0, 0, 0, 0) /* CG1 x CG1, 3-vector via (3,...) below */            \
  X(0, 1, 0, 0, 0, 0) /* CG1 x DG0 */                                        \
  X(0, 2, 0, 0, 0, 0) /* CG1 x DG1 */                                        \
  X(0, 0, 0, 0, 1, 0) /* DG0 x CG1 */                                        \
  X(0, 0, 0, 0, 0, 1) /* DG0 x DG0 */                                        \
  X(0, 0, 0, 0, 0, 2) /* DG0 x DG1 */                                        \
  X(0, 0, 0, 0, 3, 0) /* DG1 x CG1 */                                        \
  X(0, 0, 0, 0, 0, 3) /* DG1 x DG0 */                                        \
  X(0, 0, 0, 0, 0, 6) /* DG1 x DG1 */                                        \
  X(1, 1, 1, 1, 0, 0) /* P2 x P2 */                                          \
  X(3, 0, 0, 0, 0, 0) /* 3-vector P1 x P1 */


} // namespace pm
