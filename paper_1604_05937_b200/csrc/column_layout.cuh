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
    int8_t comp[kMaxK];   // vector component (3-vector P1 only, else 0)
    int8_t pos[kMaxK];    // entity position: vertex a -> a, edge e -> 3+e,
                          // cell -> 6
    int8_t ch[kMaxK];     // channel inside the entity's layer block
                          // (= the DoF's `within` minus level offset)
  };
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
    // the 3-DoF-per-vertex layout is the 3-vector P1 element: slot
    // 6a+3b+q carries component q, and Mref is block-diagonal in q
    const bool vec3 = D00 == 3 && !D01 && !D10 && !D11 && !D20 && !D21;
    for (int j = 0; j < k; ++j) t.comp[j] = vec3 ? (int8_t)(j % 3) : 0;
    return t;
  }
  static constexpr int K = make().k;
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
