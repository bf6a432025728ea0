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

// ---------------------------------------------------------------------------
// Strip planner for the strip-patch column schedule (csrc/strip.cu).
//
// Per patch, the visited cells are walked as strips: consecutive cells share
// an edge, so each step brings exactly one new vertex into a 3-vertex window
// (the vertex opposite the shared edge leaves).  Greedy: start at the
// unvisited cell with the fewest unvisited edge-neighbours (ties: lowest
// visit index), always continue to the unvisited neighbour with the fewest
// unvisited neighbours; strips are cut at `max_len` cells.
//
// Output: one record per step.  A strip starts with three "fill" steps
// (window slots 0,1,2 <- the first cell's vertices); every following step
// replaces one slot.  flags bit0 = apply the cell kernel after this step.
// Each vertex residency (entry into a slot until it leaves / the strip ends)
// gets a Y slot if the vertex is owned by the patch (local id < n_owned),
// else -1; y slots are numbered per patch, and for every owned vertex the
// list of its y slots is returned (CSR over owned vertices, per patch).
// ---------------------------------------------------------------------------
#include <algorithm>

extern "C" int pm_build_strips(
    int64_t n_patches, const int32_t *cell_ptr, const int32_t *cells,
    const int32_t *cell_edges, const uint16_t *lents, const int32_t *owned,
    const int32_t *ent_ptr, int32_t max_len,
    // outputs (capacities: steps <= 3*n_visit, strips <= n_visit)
    int32_t *patch_strip_ptr, int32_t *strip_step_ptr, uint16_t *step_v,
    uint8_t *step_slot, uint8_t *step_flags, int32_t *step_y,
    int32_t *patch_y_count, int32_t *own_y_ptr, int32_t *own_y,
    int64_t *totals /* [n_strips, n_steps, n_own_y_entries] */) {
  pm::clear_error();
  if (n_patches < 0 || max_len < 1) {
    pm::set_error("pm_build_strips: bad arguments");
    return PM_EINVAL;
  }
  int64_t n_strips = 0, n_steps = 0, n_oy = 0, own_base = 0;
  strip_step_ptr[0] = 0;
  (void)ent_ptr;
  std::vector<int32_t> nb;      // neighbours (visit-local) of each cell, 3 each
  std::vector<int32_t> deg;
  std::vector<uint8_t> used;
  std::vector<std::vector<int32_t>> yl; // per owned vertex: its y slots
  for (int64_t p = 0; p < n_patches; ++p) {
    patch_strip_ptr[p] = (int32_t)n_strips;
    const int32_t c0 = cell_ptr[p], c1 = cell_ptr[p + 1], n = c1 - c0;
    // edge-adjacency inside the patch
    std::vector<std::pair<int32_t, int32_t>> ek; // (edge, local cell)
    ek.reserve(3 * n);
    for (int32_t i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k)
        ek.push_back({cell_edges[3 * (int64_t)cells[c0 + i] + k], i});
    std::sort(ek.begin(), ek.end());
    nb.assign(3 * (size_t)n, -1);
    for (size_t a = 0; a + 1 < ek.size(); ++a)
      if (ek[a].first == ek[a + 1].first) {
        const int32_t u = ek[a].second, w = ek[a + 1].second;
        for (int k = 0; k < 3; ++k)
          if (nb[3 * u + k] < 0) { nb[3 * u + k] = w; break; }
        for (int k = 0; k < 3; ++k)
          if (nb[3 * w + k] < 0) { nb[3 * w + k] = u; break; }
      }
    used.assign(n, 0);
    deg.assign(n, 0);
    for (int32_t i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) deg[i] += nb[3 * i + k] >= 0;
    const int32_t n_own = owned[p];
    yl.assign(n_own, {});
    int32_t ycount = 0;
    auto vid = [&](int32_t i, int k) { return (int32_t)lents[3 * (int64_t)(c0 + i) + k]; };
    auto take = [&](int32_t i) {
      used[i] = 1;
      for (int k = 0; k < 3; ++k) {
        const int32_t w = nb[3 * i + k];
        if (w >= 0) --deg[w];
      }
    };
    auto new_y = [&](int32_t v) -> int32_t {
      if (v >= n_own) return -1;
      yl[v].push_back(ycount);
      return ycount++;
    };
    // neighbour of visit-local cell i across the edge {u, w} (or -1)
    auto across = [&](int32_t i, int32_t u, int32_t w) -> int32_t {
      for (int k = 0; k < 3; ++k) {
        const int32_t j = nb[3 * i + k];
        if (j < 0) continue;
        int hit = 0;
        for (int q = 0; q < 3; ++q) hit += vid(j, q) == u || vid(j, q) == w;
        if (hit == 2) return j;
      }
      return -1;
    };
    auto third = [&](int32_t i, int32_t u, int32_t w) -> int32_t {
      for (int q = 0; q < 3; ++q)
        if (vid(i, q) != u && vid(i, q) != w) return vid(i, q);
      return -1;
    };
    auto push = [&](int32_t v, int slot, int flags) {
      step_v[n_steps] = (uint16_t)v;
      step_slot[n_steps] = (uint8_t)slot;
      step_flags[n_steps] = (uint8_t)flags;
      step_y[n_steps] = new_y(v);
      ++n_steps;
    };
    // Sequential strips: the window is kept in age order and the next cell
    // is always the one across the edge of the two youngest vertices, so
    // the replaced window slot cycles 0,1,2,0,... (compile-time in the
    // kernel after a 3-way unroll).
    int32_t remaining = n;
    while (remaining > 0) {
      int32_t cur = -1;
      for (int32_t i = 0; i < n; ++i)
        if (!used[i] && (cur < 0 || deg[i] < deg[cur])) cur = i;
      take(cur);
      --remaining;
      // choose the first step (and the zig-zag direction) greedily
      int32_t w0 = vid(cur, 0), w1 = vid(cur, 1), w2 = vid(cur, 2);
      int32_t best_next = -1, best_score = -1;
      int32_t bw[3] = {w0, w1, w2};
      for (int e = 0; e < 3; ++e) {
        const int32_t a0 = vid(cur, e), a1 = vid(cur, (e + 1) % 3),
                      a2 = vid(cur, (e + 2) % 3);
        const int32_t j = across(cur, a1, a2);
        if (j < 0 || used[j]) continue;
        for (int dir = 0; dir < 2; ++dir) {
          const int32_t u = dir ? a2 : a1, w = dir ? a1 : a2; // window a0,u,w
          const int32_t nv = third(j, u, w);
          const int32_t j2 = across(j, w, nv);
          const int32_t score = (j2 >= 0 && !used[j2] && j2 != cur ? 2 : 1) * 64 -
                                deg[j];
          if (score > best_score) {
            best_score = score;
            best_next = j;
            bw[0] = a0, bw[1] = u, bw[2] = w;
          }
        }
      }
      int32_t win[3] = {bw[0], bw[1], bw[2]};
      for (int k = 0; k < 3; ++k) push(win[k], k, k == 2 ? 1 : 0);
      int32_t len = 1, slot = 0; // next slot to replace (the oldest)
      int32_t next = best_next;
      while (next >= 0 && len < max_len) {
        const int32_t y1 = win[(slot + 1) % 3], y2 = win[(slot + 2) % 3];
        const int32_t nv = third(next, y1, y2);
        if (nv < 0) {
          pm::set_error("pm_build_strips: neighbours do not share an edge");
          return PM_EINVAL;
        }
        take(next);
        --remaining;
        win[slot] = nv;
        push(nv, slot, 1);
        cur = next;
        slot = (slot + 1) % 3;
        ++len;
        // the next cell lies across the edge of the two youngest vertices
        const int32_t j = across(cur, win[(slot + 1) % 3], win[(slot + 2) % 3]);
        next = (j >= 0 && !used[j]) ? j : -1;
      }
      ++n_strips;
      strip_step_ptr[n_strips] = (int32_t)n_steps;
    }
    // longest strips first (the kernel hands strips out dynamically)
    {
      const int64_t s_lo = patch_strip_ptr[p], s_hi = n_strips;
      const int64_t k_lo = strip_step_ptr[s_lo], k_hi = strip_step_ptr[s_hi];
      std::vector<int64_t> ord(s_hi - s_lo);
      for (int64_t i = 0; i < (int64_t)ord.size(); ++i) ord[i] = s_lo + i;
      std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
        return strip_step_ptr[a + 1] - strip_step_ptr[a] >
               strip_step_ptr[b + 1] - strip_step_ptr[b];
      });
      std::vector<uint16_t> tv(step_v + k_lo, step_v + k_hi);
      std::vector<uint8_t> ts(step_slot + k_lo, step_slot + k_hi);
      std::vector<uint8_t> tf(step_flags + k_lo, step_flags + k_hi);
      std::vector<int32_t> ty(step_y + k_lo, step_y + k_hi);
      std::vector<int32_t> tp(strip_step_ptr + s_lo, strip_step_ptr + s_hi + 1);
      int64_t k = k_lo;
      for (int64_t i = 0; i < (int64_t)ord.size(); ++i) {
        const int64_t a = tp[ord[i] - s_lo] - k_lo, b = tp[ord[i] - s_lo + 1] - k_lo;
        strip_step_ptr[s_lo + i] = (int32_t)k;
        for (int64_t q = a; q < b; ++q, ++k) {
          step_v[k] = tv[q];
          step_slot[k] = ts[q];
          step_flags[k] = tf[q];
          step_y[k] = ty[q];
        }
      }
      strip_step_ptr[s_hi] = (int32_t)k;
    }
    patch_y_count[p] = ycount;
    // owner lists: owned vertices are local ids 0..n_own-1; row of owned
    // vertex v of patch p is own_base + v (own_base = sum of earlier owned)
    for (int32_t v = 0; v < n_own; ++v) {
      own_y_ptr[own_base + v] = (int32_t)n_oy;
      for (int32_t y : yl[v]) own_y[n_oy++] = y;
    }
    own_base += n_own;
  }
  own_y_ptr[own_base] = (int32_t)n_oy;
  patch_strip_ptr[n_patches] = (int32_t)n_strips;
  totals[0] = n_strips;
  totals[1] = n_steps;
  totals[2] = n_oy;
  return PM_OK;
}

// ---------------------------------------------------------------------------
// Global sequential strips for the strip-REDG schedule (csrc/strip_red.cu):
// like pm_build_strips but over the whole mesh, starting each strip at the
// first unused cell in index order (RCM order keeps concurrent strips
// local), steps = global vertex ids (3 fills, then one per cell).
// ---------------------------------------------------------------------------
// `runs`: a strip's start orientation prefers the one whose even and odd
// vertices each continue by consecutive ids (v[k+2] == v[k] + 1): on a
// level-ordered (RCM) mesh the strip then follows the band between two BFS
// levels and its vertex columns are two contiguous slabs of the field, which
// the bulk-copy strip kernel (csrc/strip_tma.cu) fetches several columns
// per copy.
static int build_global_strips_impl(int64_t n_cells, int64_t n_edges,
                                    const int32_t *cell_vertices,
                                    const int32_t *cell_edges,
                                    const uint8_t *cell_mask,
                                    const int32_t *scan_order,
                                    int32_t max_len, int32_t *strip_ptr,
                                    int32_t *steps, int32_t *steps_e,
                                    int64_t *totals, bool runs) {
  pm::clear_error();
  if (n_cells < 0 || n_edges < 0 || max_len < 1) {
    pm::set_error("pm_build_global_strips: bad arguments");
    return PM_EINVAL;
  }
  std::vector<int32_t> ec(2 * (size_t)n_edges, -1);
  for (int64_t c = 0; c < n_cells; ++c)
    for (int k = 0; k < 3; ++k) {
      if (cell_mask && !cell_mask[c]) break;
      const int64_t e = cell_edges[3 * c + k];
      if (ec[2 * e] < 0)
        ec[2 * e] = (int32_t)c;
      else
        ec[2 * e + 1] = (int32_t)c;
    }
  // cells outside the mask count as used: strips stay inside the subset
  std::vector<uint8_t> used(n_cells, 0);
  if (cell_mask)
    for (int64_t c = 0; c < n_cells; ++c) used[c] = !cell_mask[c];
  auto vid = [&](int64_t c, int k) { return cell_vertices[3 * c + k]; };
  auto across = [&](int64_t c, int32_t u, int32_t w) -> int64_t {
    for (int k = 0; k < 3; ++k) {
      const int32_t a = vid(c, (k + 1) % 3), b = vid(c, (k + 2) % 3);
      if ((a == u && b == w) || (a == w && b == u)) {
        const int64_t e = cell_edges[3 * c + k];
        const int32_t o = ec[2 * e] == c ? ec[2 * e + 1] : ec[2 * e];
        return o;
      }
    }
    return -1;
  };
  auto third = [&](int64_t c, int32_t u, int32_t w) -> int32_t {
    for (int q = 0; q < 3; ++q)
      if (vid(c, q) != u && vid(c, q) != w) return vid(c, q);
    return -1;
  };
  // edge of cell c opposite its vertex v (joins the other two)
  auto opp = [&](int64_t c, int32_t v) -> int32_t {
    for (int q = 0; q < 3; ++q)
      if (vid(c, q) == v) return cell_edges[3 * c + q];
    return -1;
  };
  int64_t n_strips = 0, n_steps = 0, scan = 0;
  strip_ptr[0] = 0;
  // strips start at the first unused cell of the scan order (default: cell
  // index order, which follows the bands of an RCM-ordered mesh)
  auto at = [&](int64_t i) -> int64_t {
    return scan_order ? (int64_t)scan_order[i] : i;
  };
  // runs: a first pass starts strips only where both id runs continue (the
  // other cells wait, so a strip across the bands cannot cut every band at
  // its end); the second pass takes what is left by the plain rule
  for (int pass = runs ? 0 : 1; pass < 2; ++pass, scan = 0)
  while (true) {
    while (scan < n_cells && used[at(scan)]) ++scan;
    if (scan >= n_cells) break;
    int64_t cur = at(scan);
    used[cur] = 1;
    int32_t win[3] = {vid(cur, 0), vid(cur, 1), vid(cur, 2)};
    int64_t next = -1;
    int best = -1;
    for (int e = 0; e < 3; ++e) {
      const int32_t a0 = vid(cur, e), a1 = vid(cur, (e + 1) % 3),
                    a2 = vid(cur, (e + 2) % 3);
      const int64_t j = across(cur, a1, a2);
      if (j < 0 || used[j]) continue;
      for (int dir = 0; dir < 2; ++dir) {
        const int32_t u = dir ? a2 : a1, w = dir ? a1 : a2;
        const int32_t nv = third(j, u, w);
        const int64_t j2 = across(j, w, nv);
        // prefer a continuation; then the lower-index neighbour
        int score = (j2 >= 0 && !used[j2] && j2 != cur) ? 2 : 1;
        // (runs) the strip a0, u, w, nv, ... continues both id runs
        if (runs && w == a0 + 1 && nv == u + 1) score += 2;
        if (score > best) {
          best = score;
          next = j;
          win[0] = a0, win[1] = u, win[2] = w;
        }
      }
    }
    if (pass == 0 && best < 3) { // no run start here: second pass
      used[cur] = 0;
      ++scan;
      continue;
    }
    if (pass == 0) {
      // walk back along the band while both runs also continue downwards,
      // so the strip starts at the band's first free cell
      int64_t back = cur;
      for (int32_t n = 1; n < max_len; ++n) {
        const int64_t j = across(back, win[0], win[1]);
        if (j < 0 || used[j]) break;
        const int32_t pv = third(j, win[0], win[1]);
        if (pv != win[1] - 1) break;
        win[2] = win[1], win[1] = win[0], win[0] = pv;
        back = j;
      }
      if (back != cur) {
        used[cur] = 0;
        cur = back;
        used[cur] = 1;
        next = across(cur, win[1], win[2]);
      }
    }
    for (int k = 0; k < 3; ++k) {
      // fill: vertex slot k and the edge opposite it (edge slot k)
      if (steps_e) {
        steps_e[2 * n_steps] = opp(cur, win[k]);
        steps_e[2 * n_steps + 1] = -1;
      }
      steps[n_steps++] = win[k];
    }
    int32_t len = 1, slot = 0;
    while (next >= 0 && len < max_len) {
      const int32_t nv = third(next, win[(slot + 1) % 3], win[(slot + 2) % 3]);
      if (nv < 0) {
        pm::set_error("pm_build_global_strips: broken strip");
        return PM_EINVAL;
      }
      used[next] = 1;
      if (steps_e) {
        // new edge slots (slot+1)%3 and (slot+2)%3: opposite the kept
        // vertices in the new cell (edge slot `slot` keeps the shared edge)
        steps_e[2 * n_steps] = opp(next, win[(slot + 1) % 3]);
        steps_e[2 * n_steps + 1] = opp(next, win[(slot + 2) % 3]);
      }
      win[slot] = nv;
      steps[n_steps++] = nv;
      cur = next;
      slot = (slot + 1) % 3;
      ++len;
      const int64_t j = across(cur, win[(slot + 1) % 3], win[(slot + 2) % 3]);
      next = (j >= 0 && !used[j]) ? j : -1;
    }
    ++n_strips;
    strip_ptr[n_strips] = (int32_t)n_steps;
  }
  totals[0] = n_strips;
  totals[1] = n_steps;
  return PM_OK;
}

extern "C" int pm_build_global_strips(int64_t n_cells, int64_t n_edges,
                                      const int32_t *cell_vertices,
                                      const int32_t *cell_edges,
                                      const uint8_t *cell_mask,
                                      const int32_t *scan_order,
                                      int32_t max_len, int32_t *strip_ptr,
                                      int32_t *steps, int32_t *steps_e,
                                      int64_t *totals) {
  return build_global_strips_impl(n_cells, n_edges, cell_vertices, cell_edges,
                                  cell_mask, scan_order, max_len, strip_ptr,
                                  steps, steps_e, totals, false);
}

extern "C" int pm_build_run_strips(int64_t n_cells, int64_t n_edges,
                                   const int32_t *cell_vertices,
                                   const int32_t *cell_edges,
                                   const uint8_t *cell_mask,
                                   const int32_t *scan_order,
                                   int32_t max_len, int32_t *strip_ptr,
                                   int32_t *steps, int32_t *steps_e,
                                   int64_t *totals) {
  return build_global_strips_impl(n_cells, n_edges, cell_vertices, cell_edges,
                                  cell_mask, scan_order, max_len, strip_ptr,
                                  steps, steps_e, totals, true);
}

// ---------------------------------------------------------------------------
// Patch strips for the store-first strip schedule (csrc/strip_red.cu).
// Cells come grouped into compact patches (patch_cells[patch_ptr[p] ..
// patch_ptr[p+1]), e.g. runs of the Morton order of the centroids).  Inside
// a patch the cells are walked as sequential strips exactly like
// pm_build_global_strips (start at the patch's lowest unused cell, one new
// vertex per cell), but a strip never leaves its patch.  One warp segment
// walks all strips of a patch in order, so every partial column of an
// entity whose cells all lie in one patch comes from that segment: the
// first residency of such an entity in the patch's walk is flagged
// (PM_STEP_STORE, bit 30 of its step id) and the kernel STORES that partial
// column instead of adding it — the entity needs no zeroing and its output
// lines no L2 fill from HBM.  Entities touched by more than one patch are
// listed in zero_list (code v for vertex v, n_vertices + e for edge e); the
// kernel's zero pass clears them and every residency of theirs adds.
// item_ptr[p] .. item_ptr[p+1] = the strips of patch p.
// totals = {strips, steps, entities in zero_list}.
// ---------------------------------------------------------------------------
extern "C" int pm_build_patch_strips(
    int64_t n_cells, int64_t n_vertices, int64_t n_edges,
    const int32_t *cell_vertices, const int32_t *cell_edges,
    const int32_t *patch_cells, const int32_t *patch_ptr, int64_t n_patches,
    int32_t max_len, int32_t *item_ptr, int32_t *strip_ptr, int32_t *steps,
    int32_t *steps_e, int32_t *zero_list, int64_t *totals) {
  pm::clear_error();
  if (n_cells < 0 || n_vertices < 0 || n_edges < 0 || n_patches < 0 ||
      max_len < 1 || n_vertices + n_edges >= PM_STEP_NOCELL) {
    pm::set_error("pm_build_patch_strips: bad arguments (entity ids must "
                  "stay below 2^29)");
    return PM_EINVAL;
  }
  if (n_patches > 0 && patch_ptr[n_patches] != n_cells) {
    pm::set_error("pm_build_patch_strips: patches must cover every cell once");
    return PM_EINVAL;
  }
  std::vector<int32_t> patch_of(n_cells, -1);
  for (int64_t p = 0; p < n_patches; ++p)
    for (int32_t i = patch_ptr[p]; i < patch_ptr[p + 1]; ++i) {
      const int32_t c = patch_cells[i];
      if (c < 0 || c >= n_cells || patch_of[c] >= 0) {
        pm::set_error("pm_build_patch_strips: patch_cells is not a "
                      "permutation of the cells");
        return PM_EINVAL;
      }
      patch_of[c] = (int32_t)p;
    }
  // owner patch per entity, -2 = touched by several patches
  std::vector<int32_t> vown(n_vertices, -1), eown(steps_e ? n_edges : 0, -1);
  auto claim = [](std::vector<int32_t> &own, int64_t i, int32_t p) {
    if (own[i] == -1)
      own[i] = p;
    else if (own[i] != p)
      own[i] = -2;
  };
  for (int64_t c = 0; c < n_cells; ++c)
    for (int k = 0; k < 3; ++k) {
      claim(vown, cell_vertices[3 * c + k], patch_of[c]);
      if (steps_e) claim(eown, cell_edges[3 * c + k], patch_of[c]);
    }
  std::vector<int32_t> ec(2 * (size_t)n_edges, -1);
  for (int64_t c = 0; c < n_cells; ++c)
    for (int k = 0; k < 3; ++k) {
      const int64_t e = cell_edges[3 * c + k];
      if (ec[2 * e] < 0)
        ec[2 * e] = (int32_t)c;
      else
        ec[2 * e + 1] = (int32_t)c;
    }
  auto vid = [&](int64_t c, int k) { return cell_vertices[3 * c + k]; };
  auto across = [&](int64_t c, int32_t u, int32_t w) -> int64_t {
    for (int k = 0; k < 3; ++k) {
      const int32_t a = vid(c, (k + 1) % 3), b = vid(c, (k + 2) % 3);
      if ((a == u && b == w) || (a == w && b == u)) {
        const int64_t e = cell_edges[3 * c + k];
        return ec[2 * e] == c ? ec[2 * e + 1] : ec[2 * e];
      }
    }
    return -1;
  };
  auto third = [&](int64_t c, int32_t u, int32_t w) -> int32_t {
    for (int q = 0; q < 3; ++q)
      if (vid(c, q) != u && vid(c, q) != w) return vid(c, q);
    return -1;
  };
  auto opp = [&](int64_t c, int32_t v) -> int32_t {
    for (int q = 0; q < 3; ++q)
      if (vid(c, q) == v) return cell_edges[3 * c + q];
    return -1;
  };
  std::vector<uint8_t> used(n_cells, 0);
  std::vector<int32_t> vseen(n_vertices, -1), eseen(steps_e ? n_edges : 0, -1);
  std::vector<int32_t> order;
  int64_t n_strips = 0, n_steps = 0;
  strip_ptr[0] = 0;
  // a residency of entity i in patch p: flagged if it is the entity's first
  // in the patch and no other patch touches the entity
  auto flag = [&](std::vector<int32_t> &own, std::vector<int32_t> &seen,
                  int32_t i, int32_t p) -> int32_t {
    if (i < 0) return i;
    if (seen[i] == p) return i;
    seen[i] = p;
    return own[i] == p ? (i | PM_STEP_STORE) : i;
  };
  for (int64_t p = 0; p < n_patches; ++p) {
    item_ptr[p] = (int32_t)n_strips;
    order.assign(patch_cells + patch_ptr[p], patch_cells + patch_ptr[p + 1]);
    std::sort(order.begin(), order.end());
    const int32_t pp = (int32_t)p;
    auto ok = [&](int64_t j) { return j >= 0 && patch_of[j] == pp && !used[j]; };
    for (const int32_t start : order) {
      if (used[start]) continue;
      int64_t cur = start;
      used[cur] = 1;
      int32_t win[3] = {vid(cur, 0), vid(cur, 1), vid(cur, 2)};
      int64_t next = -1;
      int best = -1;
      for (int e = 0; e < 3; ++e) {
        const int32_t a0 = vid(cur, e), a1 = vid(cur, (e + 1) % 3),
                      a2 = vid(cur, (e + 2) % 3);
        const int64_t j = across(cur, a1, a2);
        if (!ok(j)) continue;
        for (int dir = 0; dir < 2; ++dir) {
          const int32_t u = dir ? a2 : a1, w = dir ? a1 : a2;
          const int32_t nv = third(j, u, w);
          const int64_t j2 = across(j, w, nv);
          const int score = (ok(j2) && j2 != cur) ? 2 : 1;
          if (score > best) {
            best = score;
            next = j;
            win[0] = a0, win[1] = u, win[2] = w;
          }
        }
      }
      // fill: one continuous stream per patch, every step in normal form
      // (slot s flushes / loads edge slots s+1, s+2): the first cell's
      // edges arrive as (-1, -1), (e01, -1), (e12, e02) so each lands in the
      // slot opposite its vertex and none is flushed before its cells ran
      const int32_t fe[3][2] = {{-1, -1},
                                {opp(cur, win[2]), -1},
                                {opp(cur, win[0]), opp(cur, win[1])}};
      for (int k = 0; k < 3; ++k) {
        if (steps_e) {
          steps_e[2 * n_steps] = flag(eown, eseen, fe[k][0], pp);
          steps_e[2 * n_steps + 1] = flag(eown, eseen, fe[k][1], pp);
        }
        steps[n_steps++] =
            flag(vown, vseen, win[k], pp) | (k < 2 ? PM_STEP_NOCELL : 0);
      }
      int32_t len = 1, slot = 0;
      while (next >= 0 && len < max_len) {
        const int32_t nv =
            third(next, win[(slot + 1) % 3], win[(slot + 2) % 3]);
        if (nv < 0) {
          pm::set_error("pm_build_patch_strips: broken strip");
          return PM_EINVAL;
        }
        used[next] = 1;
        if (steps_e) {
          steps_e[2 * n_steps] =
              flag(eown, eseen, opp(next, win[(slot + 1) % 3]), pp);
          steps_e[2 * n_steps + 1] =
              flag(eown, eseen, opp(next, win[(slot + 2) % 3]), pp);
        }
        win[slot] = nv;
        steps[n_steps++] = flag(vown, vseen, nv, pp);
        cur = next;
        slot = (slot + 1) % 3;
        ++len;
        const int64_t j = across(cur, win[(slot + 1) % 3], win[(slot + 2) % 3]);
        next = ok(j) ? j : -1;
      }
      ++n_strips;
      strip_ptr[n_strips] = (int32_t)n_steps;
    }
  }
  item_ptr[n_patches] = (int32_t)n_strips;
  int64_t nz = 0;
  for (int64_t v = 0; v < n_vertices; ++v)
    if (vown[v] < 0) zero_list[nz++] = (int32_t)v; // shared, or in no cell
  for (int64_t e = 0; e < (int64_t)eown.size(); ++e)
    if (eown[e] < 0) zero_list[nz++] = (int32_t)(n_vertices + e);
  totals[0] = n_strips;
  totals[1] = n_steps;
  totals[2] = nz;
  return PM_OK;
}

// ---------------------------------------------------------------------------
// The cell each strip step forms (for the DG strip kernel, whose field is
// per cell): step i >= 2 of a strip forms the cell of its window, the last
// three entered vertices {steps[i-2], steps[i-1], steps[i]}; the first two
// (fill) steps form none (-1).  Found through the vertex -> cell incidence
// of steps[i].
// ---------------------------------------------------------------------------
extern "C" int pm_strip_step_cells(int64_t n_cells, int64_t n_vertices,
                                   const int32_t *cell_vertices,
                                   const int32_t *strip_ptr, int64_t n_strips,
                                   const int32_t *steps, int32_t *step_cells) {
  pm::clear_error();
  if (n_cells < 0 || n_vertices < 0 || n_strips < 0 ||
      (n_strips > 0 && (!strip_ptr || !steps || !step_cells))) {
    pm::set_error("pm_strip_step_cells: bad arguments");
    return PM_EINVAL;
  }
  std::vector<int64_t> off(n_vertices + 1, 0);
  for (int64_t c = 0; c < 3 * n_cells; ++c) {
    const int32_t v = cell_vertices[c];
    if (v < 0 || v >= n_vertices) {
      pm::set_error("pm_strip_step_cells: vertex %d out of range", v);
      return PM_EINVAL;
    }
    ++off[v + 1];
  }
  for (int64_t v = 0; v < n_vertices; ++v) off[v + 1] += off[v];
  std::vector<int32_t> vc(3 * n_cells);
  std::vector<int64_t> fill(off.begin(), off.end() - 1);
  for (int64_t c = 0; c < n_cells; ++c)
    for (int k = 0; k < 3; ++k) vc[fill[cell_vertices[3 * c + k]]++] = (int32_t)c;
  for (int64_t s = 0; s < n_strips; ++s) {
    const int32_t a = strip_ptr[s], b = strip_ptr[s + 1];
    for (int32_t i = a; i < b; ++i) {
      step_cells[i] = -1;
      if (i < a + 2) continue;
      const int32_t u = steps[i - 2], w = steps[i - 1], v = steps[i];
      for (int64_t e = off[v]; e < off[v + 1]; ++e) {
        const int32_t c = vc[e];
        const int32_t *t = cell_vertices + 3 * (int64_t)c;
        const bool hu = t[0] == u || t[1] == u || t[2] == u;
        const bool hw = t[0] == w || t[1] == w || t[2] == w;
        if (hu && hw) {
          step_cells[i] = c;
          break;
        }
      }
      if (step_cells[i] < 0) {
        pm::set_error("pm_strip_step_cells: step %d of strip %lld forms no "
                      "cell", i - a, (long long)s);
        return PM_EINVAL;
      }
    }
  }
  return PM_OK;
}
