// Host-side mesh setup: the Cuthill-McKee breadth-first search.
//
// Restates reference ordering.py:45-90 (numba `_cuthill_mckee`): components
// are taken in order of their smallest unvisited vertex; each is searched
// once to find its minimum-degree vertex (ties -> lowest index) and then
// traversed breadth-first from it, neighbours in the pre-sorted
// (degree, index) order.  The caller reverses the visit order.
#include <stdint.h>
#include <string.h>

#include <vector>

#include "prismesh_cuda.h"

namespace pm {
void set_error(const char *fmt, ...);
void clear_error();
} // namespace pm

extern "C" int pm_rcm_order(const int64_t *offsets, const int64_t *nb,
                            int64_t n, int64_t *order) {
  pm::clear_error();
  if (n < 0 || (n > 0 && (!offsets || !order))) {
    pm::set_error("pm_rcm_order: bad arguments");
    return PM_EINVAL;
  }
  std::vector<uint8_t> seen(n, 0);
  std::vector<int64_t> comp;
  comp.reserve(n);
  int64_t pos = 0, scan = 0;
  while (pos < n) {
    while (seen[scan]) ++scan;
    // pass 1: collect the component of `scan`, pick its min-degree vertex
    comp.clear();
    comp.push_back(scan);
    seen[scan] = 1;
    for (size_t h = 0; h < comp.size(); ++h) {
      const int64_t v = comp[h];
      for (int64_t e = offsets[v]; e < offsets[v + 1]; ++e) {
        const int64_t w = nb[e];
        if (w < 0 || w >= n) {
          pm::set_error("pm_rcm_order: neighbour %lld out of range",
                        (long long)w);
          return PM_EINVAL;
        }
        if (!seen[w]) {
          seen[w] = 1;
          comp.push_back(w);
        }
      }
    }
    int64_t start = comp[0];
    for (int64_t v : comp) {
      const int64_t dv = offsets[v + 1] - offsets[v];
      const int64_t ds = offsets[start + 1] - offsets[start];
      if (dv < ds || (dv == ds && v < start)) start = v;
    }
    for (int64_t v : comp) seen[v] = 0;
    // pass 2: breadth-first from `start`
    order[pos] = start;
    seen[start] = 1;
    int64_t tail = pos + 1;
    while (pos < tail) {
      const int64_t v = order[pos++];
      for (int64_t e = offsets[v]; e < offsets[v + 1]; ++e) {
        const int64_t w = nb[e];
        if (!seen[w]) {
          seen[w] = 1;
          order[tail++] = w;
        }
      }
    }
  }
  return PM_OK;
}

// Greedy colouring of base cells over the "shares a vertex" graph
// (SPEC.md:343-351): cells in index order, smallest colour not taken by an
// earlier cell sharing any vertex.  Deterministic.
extern "C" int pm_greedy_color_cells(const int32_t *cv, int64_t n_cells,
                                     const int64_t *vc_off,
                                     const int32_t *vc_cells, int32_t *color,
                                     int32_t *n_colors) {
  pm::clear_error();
  if (n_cells < 0 || (n_cells > 0 && (!cv || !vc_off || !vc_cells || !color))) {
    pm::set_error("pm_greedy_color_cells: bad arguments");
    return PM_EINVAL;
  }
  for (int64_t c = 0; c < n_cells; ++c) color[c] = -1;
  int32_t used_max = 0;
  std::vector<uint8_t> taken;
  for (int64_t c = 0; c < n_cells; ++c) {
    taken.assign((size_t)used_max + 1, 0);
    for (int a = 0; a < 3; ++a) {
      const int64_t v = cv[3 * c + a];
      for (int64_t e = vc_off[v]; e < vc_off[v + 1]; ++e) {
        const int32_t o = color[vc_cells[e]];
        if (o >= 0) taken[o] = 1;
      }
    }
    int32_t pick = 0;
    while (taken[pick]) ++pick;
    color[c] = pick;
    if (pick + 1 > used_max) used_max = pick + 1;
  }
  if (n_colors) *n_colors = used_max;
  return PM_OK;
}
