/*
 * oracle_mesh.c -- TEST INFRASTRUCTURE ONLY (the checker, never shipped).
 *
 * Plain-C restatement of the reference's base-mesh pipeline, so that the
 * CPU oracle (tests, the bench's CPU arm) can build every BASELINE mesh
 * without the product library:
 *   or_unit_square  pkg/src/prismesh/mesh.py:228-254 generate_unit_square_mesh
 *   or_derive_edges mesh.py:33-84 derive_edges (edges numbered by the sorted
 *                   vertex pair, cell_edges[c][k] = edge opposite vertex k)
 *   or_rcm_order    ordering.py:93-114 rcm_order over mesh.py:171-181
 *                   vertex_neighbours (rows by (degree, index)), the BFS of
 *                   ordering.py:45-90 _cuthill_mckee, reversed
 *   or_apply_ordering ordering.py:134-152 apply_ordering (cells by their
 *                   sorted new vertex triple, coordinates follow)
 * The seeded random order (ordering.py:123-131) and the jitter draws come
 * from numpy in oracle/__init__.py, exactly as the reference draws them.
 * Pinned by tests/golden (meshes and permutations of the reference itself).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* LSD radix sort of (key, payload) pairs by the low `bits` of the keys,
 * stable; tmp buffers of n each. */
static void radix_sort(uint64_t *key, int64_t *val, int64_t n, int bits,
                       uint64_t *tk, int64_t *tv) {
  const int D = 11, R = 1 << D;
  int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * R);
  for (int sh = 0; sh < bits; sh += D) {
    memset(cnt, 0, sizeof(int64_t) * R);
    for (int64_t i = 0; i < n; ++i) cnt[(key[i] >> sh) & (R - 1)]++;
    int64_t s = 0;
    for (int r = 0; r < R; ++r) {
      const int64_t c = cnt[r];
      cnt[r] = s;
      s += c;
    }
    for (int64_t i = 0; i < n; ++i) {
      const int64_t p = cnt[(key[i] >> sh) & (R - 1)]++;
      tk[p] = key[i];
      tv[p] = val[i];
    }
    memcpy(key, tk, sizeof(uint64_t) * n);
    memcpy(val, tv, sizeof(int64_t) * n);
  }
  free(cnt);
}

static int bits_for(uint64_t maxkey) {
  int b = 1;
  while (b < 64 && (maxkey >> b)) ++b;
  return b;
}

/* mesh.py:228-254 */
void or_unit_square(int32_t n, int32_t *cells, double *coords) {
  const int64_t k = n + 1;
  for (int64_t i = 0; i < k; ++i)
    for (int64_t j = 0; j < k; ++j) {
      coords[2 * (i * k + j)] = (double)i / (double)n;
      coords[2 * (i * k + j) + 1] = (double)j / (double)n;
    }
  const int64_t nsq = (int64_t)n * n;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const int64_t q = i * n + j;
      const int32_t v00 = (int32_t)(i * k + j), v10 = (int32_t)((i + 1) * k + j);
      const int32_t v01 = (int32_t)(i * k + j + 1);
      const int32_t v11 = (int32_t)((i + 1) * k + j + 1);
      int32_t *lo = cells + 3 * q, *up = cells + 3 * (nsq + q);
      lo[0] = v00, lo[1] = v10, lo[2] = v11; /* lower */
      up[0] = v00, up[1] = v11, up[2] = v01; /* upper */
    }
}

/* mesh.py:33-84; returns the edge count (edge_vertices sized 3 n_cells x 2
 * by the caller), -1 when an edge has more than two cells */
int64_t or_derive_edges(const int32_t *cells, int64_t n_cells,
                        int32_t *edge_vertices, int32_t *cell_edges) {
  const int64_t m = 3 * n_cells;
  uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * m);
  int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * m);
  uint64_t *tk = (uint64_t *)malloc(sizeof(uint64_t) * m);
  int64_t *tv = (int64_t *)malloc(sizeof(int64_t) * m);
  uint64_t mx = 0;
  for (int64_t c = 0; c < n_cells; ++c)
    for (int s = 0; s < 3; ++s) {
      /* side s joins the two vertices opposite local vertex s */
      uint64_t a = (uint32_t)cells[3 * c + (s + 1) % 3];
      uint64_t b = (uint32_t)cells[3 * c + (s + 2) % 3];
      if (a > b) {
        const uint64_t t = a;
        a = b, b = t;
      }
      const int64_t i = s * n_cells + c; /* row of the reference's concat */
      key[i] = (a << 32) | b;
      pos[i] = i;
      if (key[i] > mx) mx = key[i];
    }
  radix_sort(key, pos, m, bits_for(mx), tk, tv);
  int64_t ne = 0, run = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (i == 0 || key[i] != key[i - 1]) {
      edge_vertices[2 * ne] = (int32_t)(key[i] >> 32);
      edge_vertices[2 * ne + 1] = (int32_t)(key[i] & 0xffffffffu);
      ++ne;
      run = 0;
    }
    if (++run > 2) {
      ne = -1;
      break;
    }
    const int64_t r = pos[i];
    cell_edges[3 * (r % n_cells) + r / n_cells] = (int32_t)(ne - 1);
  }
  free(key), free(pos), free(tk), free(tv);
  return ne;
}

/* ordering.py:45-114 over mesh.py:171-181; forward[old] = new */
void or_rcm_order(const int32_t *edge_vertices, int64_t n_edges,
                  int64_t n_vertices, int64_t *forward) {
  const int64_t n = n_vertices, m = 2 * n_edges;
  int64_t *off = (int64_t *)calloc(n + 1, sizeof(int64_t));
  int64_t *nb = (int64_t *)malloc(sizeof(int64_t) * (m > 0 ? m : 1));
  for (int64_t e = 0; e < n_edges; ++e) {
    off[edge_vertices[2 * e] + 1]++;
    off[edge_vertices[2 * e + 1] + 1]++;
  }
  for (int64_t v = 0; v < n; ++v) off[v + 1] += off[v];
  /* rows by (degree(w), w): sort (row, degree, w) packed keys */
  uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * (m > 0 ? m : 1));
  int64_t *val = (int64_t *)malloc(sizeof(int64_t) * (m > 0 ? m : 1));
  uint64_t *tk = (uint64_t *)malloc(sizeof(uint64_t) * (m > 0 ? m : 1));
  int64_t *tv = (int64_t *)malloc(sizeof(int64_t) * (m > 0 ? m : 1));
  const int vb = bits_for((uint64_t)(n > 1 ? n - 1 : 1));
  int64_t maxdeg = 0;
  for (int64_t v = 0; v < n; ++v)
    if (off[v + 1] - off[v] > maxdeg) maxdeg = off[v + 1] - off[v];
  const int db = bits_for((uint64_t)(maxdeg > 0 ? maxdeg : 1));
  int64_t i = 0;
  for (int64_t e = 0; e < n_edges; ++e)
    for (int d = 0; d < 2; ++d) {
      const uint64_t src = (uint32_t)edge_vertices[2 * e + d];
      const uint64_t dst = (uint32_t)edge_vertices[2 * e + 1 - d];
      const uint64_t deg = (uint64_t)(off[dst + 1] - off[dst]);
      key[i] = (src << (db + vb)) | (deg << vb) | dst;
      val[i] = (int64_t)dst;
      ++i;
    }
  radix_sort(key, val, m, 2 * vb + db, tk, tv);
  memcpy(nb, val, sizeof(int64_t) * m);
  free(key), free(val), free(tk), free(tv);
  /* _cuthill_mckee */
  char *visited = (char *)calloc(n > 0 ? n : 1, 1);
  int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  int64_t *comp = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  int64_t pos = 0, scan = 0;
  while (pos < n) {
    while (visited[scan]) ++scan;
    comp[0] = scan;
    visited[scan] = 1;
    int64_t head = 0, tail = 1;
    while (head < tail) {
      const int64_t v = comp[head++];
      for (int64_t j = off[v]; j < off[v + 1]; ++j)
        if (!visited[nb[j]]) visited[nb[j]] = 1, comp[tail++] = nb[j];
    }
    int64_t start = comp[0];
    for (int64_t j = 0; j < tail; ++j) {
      const int64_t v = comp[j];
      const int64_t dv = off[v + 1] - off[v], ds = off[start + 1] - off[start];
      if (dv < ds || (dv == ds && v < start)) start = v;
    }
    for (int64_t j = 0; j < tail; ++j) visited[comp[j]] = 0;
    order[pos] = start;
    visited[start] = 1;
    tail = pos + 1;
    while (pos < tail) {
      const int64_t v = order[pos++];
      for (int64_t j = off[v]; j < off[v + 1]; ++j)
        if (!visited[nb[j]]) visited[nb[j]] = 1, order[tail++] = nb[j];
    }
  }
  for (int64_t j = 0; j < n; ++j) forward[order[n - 1 - j]] = j;
  free(visited), free(order), free(comp), free(off), free(nb);
}

/* ordering.py:134-152: new cells (in the new order) and coordinates */
void or_apply_ordering(const int32_t *cells, int64_t n_cells,
                       const double *coords, int64_t n_vertices,
                       const int64_t *forward, int32_t *new_cells,
                       double *new_coords) {
  const int64_t n = n_cells;
  uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * (n > 0 ? n : 1));
  int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  uint64_t *tk = (uint64_t *)malloc(sizeof(uint64_t) * (n > 0 ? n : 1));
  int64_t *tv = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  int32_t *srt = (int32_t *)malloc(sizeof(int32_t) * 3 * (n > 0 ? n : 1));
  for (int64_t c = 0; c < n; ++c) {
    int32_t a = (int32_t)forward[cells[3 * c]], b = (int32_t)forward[cells[3 * c + 1]],
            d = (int32_t)forward[cells[3 * c + 2]], t;
    if (a > b) t = a, a = b, b = t;
    if (b > d) t = b, b = d, d = t;
    if (a > b) t = a, a = b, b = t;
    srt[3 * c] = a, srt[3 * c + 1] = b, srt[3 * c + 2] = d;
  }
  /* np.lexsort((k2, k1, k0)): stable passes on k2, then k1, then k0 */
  for (int64_t c = 0; c < n; ++c) idx[c] = c;
  const int vb = bits_for((uint64_t)(n_vertices > 1 ? n_vertices - 1 : 1));
  for (int pass = 2; pass >= 0; --pass) {
    for (int64_t i = 0; i < n; ++i) key[i] = (uint64_t)srt[3 * idx[i] + pass];
    radix_sort(key, idx, n, vb, tk, tv);
  }
  for (int64_t i = 0; i < n; ++i)
    for (int q = 0; q < 3; ++q)
      new_cells[3 * i + q] = (int32_t)forward[cells[3 * idx[i] + q]];
  for (int64_t v = 0; v < n_vertices; ++v) {
    new_coords[2 * forward[v]] = coords[2 * v];
    new_coords[2 * forward[v] + 1] = coords[2 * v + 1];
  }
  free(key), free(idx), free(tk), free(tv), free(srt);
}
