// Band-tile plan for the tile schedule of the vertex-column CG layouts
// (csrc/tile.cu, PM_VARIANT_TILE).
//
// The base cells are cut, in index order, into tiles of consecutive cells.
// On a mesh ordered like the reference's apply_ordering (cells sorted by
// their lowest new vertex, ordering.py:147-152) over an RCM vertex order
// (ordering.py:45-114), consecutive cells form bands between two adjacent
// BFS levels of the base graph, so a tile's vertices are two (rarely more)
// runs of consecutive vertex ids: under the reference numbering (Alg. 1,
// fspace.py:134-149) each run is ONE contiguous range of the field and one
// of the coordinate field, which the kernel stages into shared memory with
// one bulk copy each.  A tile is grown until its vertex columns would
// exceed the shared-memory budget.
//
// Per tile the plan holds
//   * the vertex runs (first vertex, count) and their shared-memory areas
//     (byte offsets, each run reserved round_up16(n * col) + 16 bytes: the
//     16-byte aligned superset of any placement of the run);
//   * the "first-touch" runs: vertices whose lowest-index tile is this one.
//     Tiles are claimed in index order at run time; a tile zeroes the
//     output columns it touches first, so y needs no memset and the zeroed
//     lines are still in L2 when the other tiles' partial columns arrive;
//   * the tiles whose zeroing it must wait for (the first-touch tiles of
//     its other vertices, always lower indices);
//   * its sequential strips (consecutive cells share the edge of the two
//     youngest window vertices, as pm_build_global_strips), as steps = the
//     tile-local slot (index in the sorted vertex list) of each step's new
//     vertex, long strips split so the tile has at least `min_strips`.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "pm_common.cuh"

namespace {

struct Tiles {
  std::vector<int32_t> cell_ptr, run_ptr, run_v0, run_n, run_fa, run_ca,
      zero_ptr, zero_v0, zero_n, dep_ptr, deps, strip_ptr, strip_step0,
      strip_len;
  std::vector<int16_t> steps;
  int64_t max_fa = 0, max_ca = 0;
  int32_t max_slots = 0, max_cells = 0, max_strips = 0;
};

inline int64_t up16(int64_t b) { return (b + 15) & ~(int64_t)15; }

} // namespace

extern "C" int pm_tiles_build(int64_t n_cells, int64_t n_vertices,
                              int64_t n_edges, const int32_t *cell_vertices,
                              const int32_t *cell_edges, int64_t col_f,
                              int64_t col_c, int64_t budget, int32_t max_cells,
                              int32_t min_strips, int32_t min_sub,
                              void **handle) {
  pm::clear_error();
  *handle = nullptr;
  if (n_cells < 0 || n_vertices <= 0 || n_edges < 0 || col_f <= 0 ||
      col_c <= 0 || max_cells < 1 || min_strips < 1 || min_sub < 1) {
    pm::set_error("pm_tiles_build: bad arguments");
    return PM_EINVAL;
  }
  if (3 * (col_f + col_c + 32) > budget) {
    pm::set_error("pm_tiles_build: one cell's vertex columns (%lld bytes) do "
                  "not fit the %lld-byte tile budget",
                  (long long)(3 * (col_f + col_c)), (long long)budget);
    return PM_EINVAL;
  }
  Tiles *T = new Tiles();
  std::vector<int32_t> vmark(n_vertices, -1), first(n_vertices, -1);
  std::vector<int32_t> emark(n_edges, -1), ecell(2 * n_edges, -1);
  std::vector<int32_t> verts, lcells, dep_tmp;
  std::vector<uint8_t> used;
  std::vector<std::vector<int32_t>> strips;
  T->cell_ptr.push_back(0);
  T->run_ptr.push_back(0);
  T->zero_ptr.push_back(0);
  T->dep_ptr.push_back(0);
  T->strip_ptr.push_back(0);
  const int64_t per_v = col_f + col_c + 32; // conservative growth bound
  int64_t c = 0;
  int32_t t = 0;
  while (c < n_cells) {
    // ---- grow the tile over consecutive cells
    verts.clear();
    const int64_t c0 = c;
    while (c < n_cells && c - c0 < max_cells) {
      int add = 0;
      for (int k = 0; k < 3; ++k) {
        const int32_t v = cell_vertices[3 * c + k];
        if (v < 0 || v >= n_vertices) {
          pm::set_error("pm_tiles_build: cell %lld has vertex %d out of range",
                        (long long)c, v);
          delete T;
          return PM_EINVAL;
        }
        add += vmark[v] != t;
      }
      if ((int64_t)(verts.size() + add) * per_v > budget) break;
      for (int k = 0; k < 3; ++k) {
        const int32_t v = cell_vertices[3 * c + k];
        if (vmark[v] != t) vmark[v] = t, verts.push_back(v);
      }
      ++c;
    }
    const int64_t c1 = c;
    // ---- vertex runs, shared-memory areas
    std::sort(verts.begin(), verts.end());
    const int nv = (int)verts.size();
    int64_t fa = 0, ca = 0;
    for (int i = 0; i < nv;) {
      int j = i + 1;
      while (j < nv && verts[j] == verts[j - 1] + 1) ++j;
      const int n = j - i;
      T->run_v0.push_back(verts[i]);
      T->run_n.push_back(n);
      T->run_fa.push_back((int32_t)fa);
      T->run_ca.push_back((int32_t)ca);
      fa += up16(n * col_f) + 16;
      ca += up16(n * col_c) + 16;
      i = j;
    }
    T->max_fa = std::max(T->max_fa, fa);
    T->max_ca = std::max(T->max_ca, ca);
    T->max_slots = std::max(T->max_slots, (int32_t)nv);
    T->max_cells = std::max(T->max_cells, (int32_t)(c1 - c0));
    // ---- first-touch zeroing, dependencies
    dep_tmp.clear();
    for (int i = 0; i < nv;) {
      if (first[verts[i]] >= 0) {
        dep_tmp.push_back(first[verts[i]]);
        ++i;
        continue;
      }
      int j = i;
      while (j < nv && first[verts[j]] < 0 &&
             (j == i || verts[j] == verts[j - 1] + 1))
        first[verts[j]] = t, ++j;
      T->zero_v0.push_back(verts[i]);
      T->zero_n.push_back(j - i);
      i = j;
    }
    std::sort(dep_tmp.begin(), dep_tmp.end());
    dep_tmp.erase(std::unique(dep_tmp.begin(), dep_tmp.end()), dep_tmp.end());
    for (int32_t d : dep_tmp) T->deps.push_back(d);
    // ---- strips over the tile's cells (edge adjacency through edge ids)
    const int nc = (int)(c1 - c0);
    for (int i = 0; i < nc; ++i)
      for (int k = 0; k < 3; ++k) {
        const int32_t e = cell_edges[3 * (c0 + i) + k];
        if (emark[e] != t) emark[e] = t, ecell[2 * e] = i, ecell[2 * e + 1] = -1;
        else ecell[2 * e + 1] = i;
      }
    used.assign(nc, 0);
    auto vid = [&](int i, int k) { return cell_vertices[3 * (c0 + i) + k]; };
    auto across = [&](int i, int32_t u, int32_t w) -> int {
      for (int k = 0; k < 3; ++k) {
        const int32_t a = vid(i, (k + 1) % 3), b = vid(i, (k + 2) % 3);
        if ((a == u && b == w) || (a == w && b == u)) {
          const int32_t e = cell_edges[3 * (c0 + i) + k];
          return ecell[2 * e] == i ? ecell[2 * e + 1] : ecell[2 * e];
        }
      }
      return -1;
    };
    auto third = [&](int i, int32_t u, int32_t w) -> int32_t {
      for (int q = 0; q < 3; ++q)
        if (vid(i, q) != u && vid(i, q) != w) return vid(i, q);
      return -1;
    };
    strips.clear();
    int scan = 0;
    while (true) {
      while (scan < nc && used[scan]) ++scan;
      if (scan >= nc) break;
      int cur = scan;
      used[cur] = 1;
      int32_t win[3] = {vid(cur, 0), vid(cur, 1), vid(cur, 2)};
      int next = -1, best = -1;
      for (int e = 0; e < 3; ++e) {
        const int32_t a0 = vid(cur, e), a1 = vid(cur, (e + 1) % 3),
                      a2 = vid(cur, (e + 2) % 3);
        const int j = across(cur, a1, a2);
        if (j < 0 || used[j]) continue;
        for (int dir = 0; dir < 2; ++dir) {
          const int32_t u = dir ? a2 : a1, w = dir ? a1 : a2;
          const int32_t nv2 = third(j, u, w);
          const int j2 = across(j, w, nv2);
          const int score = (j2 >= 0 && !used[j2] && j2 != cur) ? 2 : 1;
          if (score > best) {
            best = score;
            next = j;
            win[0] = a0, win[1] = u, win[2] = w;
          }
        }
      }
      std::vector<int32_t> s(win, win + 3);
      int slot = 0;
      while (next >= 0) {
        const int32_t nv2 = third(next, win[(slot + 1) % 3], win[(slot + 2) % 3]);
        used[next] = 1;
        win[slot] = nv2;
        s.push_back(nv2);
        cur = next;
        slot = (slot + 1) % 3;
        const int j = across(cur, win[(slot + 1) % 3], win[(slot + 2) % 3]);
        next = (j >= 0 && !used[j]) ? j : -1;
      }
      strips.push_back(std::move(s));
    }
    // split the longest strips until the tile has min_strips of them
    while ((int)strips.size() < min_strips) {
      size_t li = 0;
      for (size_t i = 1; i < strips.size(); ++i)
        if (strips[i].size() > strips[li].size()) li = i;
      const int cells = (int)strips[li].size() - 2;
      if (cells < 2 * min_sub) break;
      const int j = cells / 2; // second part: cells j .. cells-1
      std::vector<int32_t> b(strips[li].begin() + j, strips[li].end());
      strips[li].resize(j + 2);
      strips.push_back(std::move(b));
    }
    T->max_strips = std::max(T->max_strips, (int32_t)strips.size());
    for (auto &s : strips) {
      T->strip_step0.push_back((int32_t)T->steps.size());
      T->strip_len.push_back((int32_t)s.size());
      for (int32_t v : s) {
        const int slot = (int)(std::lower_bound(verts.begin(), verts.end(), v) -
                               verts.begin());
        T->steps.push_back((int16_t)slot);
      }
    }
    if (nv > 32767) {
      pm::set_error("pm_tiles_build: %d vertices in one tile", nv);
      delete T;
      return PM_EINVAL;
    }
    T->cell_ptr.push_back((int32_t)c1);
    T->run_ptr.push_back((int32_t)T->run_v0.size());
    T->zero_ptr.push_back((int32_t)T->zero_v0.size());
    T->dep_ptr.push_back((int32_t)T->deps.size());
    T->strip_ptr.push_back((int32_t)T->strip_step0.size());
    ++t;
  }
  // vertices no cell touches (unreferenced): zeroed by tile 0 as well
  if (t > 0) {
    std::vector<int32_t> zv, zn;
    for (int64_t v = 0; v < n_vertices;) {
      if (first[v] >= 0) {
        ++v;
        continue;
      }
      int64_t w = v;
      while (w < n_vertices && first[w] < 0) ++w;
      zv.push_back((int32_t)v);
      zn.push_back((int32_t)(w - v));
      v = w;
    }
    if (!zv.empty()) {
      T->zero_v0.insert(T->zero_v0.begin(), zv.begin(), zv.end());
      T->zero_n.insert(T->zero_n.begin(), zn.begin(), zn.end());
      for (size_t i = 1; i < T->zero_ptr.size(); ++i)
        T->zero_ptr[i] += (int32_t)zv.size();
    }
  }
  *handle = T;
  return PM_OK;
}

// info: {tiles, runs, zero runs, deps, strips, steps, max f area bytes,
//        max coordinate area bytes, max slots, max cells per tile,
//        max strips per tile}
extern "C" int pm_tiles_info(void *handle, int64_t *info) {
  const Tiles *T = static_cast<const Tiles *>(handle);
  if (!T) {
    pm::set_error("pm_tiles_info: null handle");
    return PM_EINVAL;
  }
  info[0] = (int64_t)T->cell_ptr.size() - 1;
  info[1] = (int64_t)T->run_v0.size();
  info[2] = (int64_t)T->zero_v0.size();
  info[3] = (int64_t)T->deps.size();
  info[4] = (int64_t)T->strip_step0.size();
  info[5] = (int64_t)T->steps.size();
  info[6] = T->max_fa;
  info[7] = T->max_ca;
  info[8] = T->max_slots;
  info[9] = T->max_cells;
  info[10] = T->max_strips;
  return PM_OK;
}

// Copies the plan out: int32 arrays in the order cell_ptr, run_ptr, run_v0,
// run_n, run_fa, run_ca, zero_ptr, zero_v0, zero_n, dep_ptr, deps,
// strip_ptr, strip_step0, strip_len (sizes from pm_tiles_info), then the
// int16 steps.
extern "C" int pm_tiles_export(void *handle, int32_t **arrays, int16_t *steps) {
  const Tiles *T = static_cast<const Tiles *>(handle);
  if (!T) {
    pm::set_error("pm_tiles_export: null handle");
    return PM_EINVAL;
  }
  const std::vector<int32_t> *src[14] = {
      &T->cell_ptr, &T->run_ptr, &T->run_v0,   &T->run_n,
      &T->run_fa,   &T->run_ca,  &T->zero_ptr, &T->zero_v0,
      &T->zero_n,   &T->dep_ptr, &T->deps,     &T->strip_ptr,
      &T->strip_step0, &T->strip_len};
  for (int i = 0; i < 14; ++i)
    if (arrays[i] && !src[i]->empty())
      std::memcpy(arrays[i], src[i]->data(), src[i]->size() * sizeof(int32_t));
  if (steps && !T->steps.empty())
    std::memcpy(steps, T->steps.data(), T->steps.size() * sizeof(int16_t));
  return PM_OK;
}

// One contiguous int32 record per tile, padded to 16 bytes (the kernel's
// producer warp fetches a tile's record with one bulk copy):
//   [0] n_runs [1] n_zero [2] n_deps [3] n_strips [4] n_steps [5] n_slots
//   [6] tile [7] 0, runs (v0, n, field area, coordinate area) x n_runs,
//   zero runs (v0, n) x n_zero, deps x n_deps,
//   strips (first step, steps) x n_strips, steps as int16 pairs.
// off[t] .. off[t+1] = tile t's words.  sizes: {total words, max words}.
extern "C" int pm_tiles_blob(void *handle, int32_t *blob, int64_t *off,
                             int64_t *sizes) {
  const Tiles *T = static_cast<const Tiles *>(handle);
  if (!T) {
    pm::set_error("pm_tiles_blob: null handle");
    return PM_EINVAL;
  }
  const int64_t nt = (int64_t)T->cell_ptr.size() - 1;
  int64_t w = 0, mx = 0;
  for (int64_t t = 0; t < nt; ++t) {
    const int32_t r0 = T->run_ptr[t], r1 = T->run_ptr[t + 1];
    const int32_t z0 = T->zero_ptr[t], z1 = T->zero_ptr[t + 1];
    const int32_t d0 = T->dep_ptr[t], d1 = T->dep_ptr[t + 1];
    const int32_t s0 = T->strip_ptr[t], s1 = T->strip_ptr[t + 1];
    const int32_t k0 = s1 > s0 ? T->strip_step0[s0] : 0;
    const int32_t k1 = s1 > s0 ? T->strip_step0[s1 - 1] + T->strip_len[s1 - 1]
                               : 0;
    int32_t nslots = 0;
    for (int32_t r = r0; r < r1; ++r) nslots += T->run_n[r];
    // 16-byte aligned records (the kernel fetches them by bulk copy)
    const int64_t words = (8 + 4 * (r1 - r0) + 2 * (z1 - z0) + (d1 - d0) +
                           2 * (s1 - s0) + (k1 - k0 + 1) / 2 + 3) & ~3;
    if (off) off[t] = w;
    if (blob) {
      int32_t *b = blob + w;
      b[0] = r1 - r0, b[1] = z1 - z0, b[2] = d1 - d0, b[3] = s1 - s0;
      b[4] = k1 - k0, b[5] = nslots, b[6] = (int32_t)t, b[7] = 0;
      int i = 8;
      for (int32_t r = r0; r < r1; ++r) {
        b[i++] = T->run_v0[r], b[i++] = T->run_n[r];
        b[i++] = T->run_fa[r], b[i++] = T->run_ca[r];
      }
      for (int32_t z = z0; z < z1; ++z) b[i++] = T->zero_v0[z], b[i++] = T->zero_n[z];
      for (int32_t d = d0; d < d1; ++d) b[i++] = T->deps[d];
      for (int32_t q = s0; q < s1; ++q)
        b[i++] = T->strip_step0[q] - k0, b[i++] = T->strip_len[q];
      int16_t *st = reinterpret_cast<int16_t *>(b + i);
      for (int32_t k = k0; k < k1; ++k) st[k - k0] = T->steps[k];
      for (int64_t k = k1 - k0; k < 2 * (words - i); ++k) st[k] = 0;
    }
    w += words;
    mx = std::max(mx, words);
  }
  if (off) off[nt] = w;
  sizes[0] = w;
  sizes[1] = mx;
  return PM_OK;
}

extern "C" void pm_tiles_free(void *handle) {
  delete static_cast<Tiles *>(handle);
}
