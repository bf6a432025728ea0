/*
 * prismesh_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never shipped).
 *
 * A plain-C CPU restatement of the reference's extruded-mesh numbering and
 * of the SPEC's column par-loop + residual kernel.  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's CPU-baseline / reference
 * arm may load it.  The product (paper_1604_05937_b200/) never does.
 *
 * Restated reference behaviour (paths under /root/reference):
 *   or_slot_table      pkg/src/prismesh/fspace.py:110-131 (slot_table)
 *   or_build_cell_map  fspace.py:137-149 (closed-form Alg. 1 origins),
 *                      fspace.py:192-215 (build_cell_map, int32 store wraps),
 *                      fspace.py:218-229 (compute_offsets, Alg. 2)
 *   or_extrude         extrusion.py:66-85 (extrude_coordinates)
 *   or_assemble        SPEC.md:333-341 iterate_columns (Alg. 3,
 *                      PAPER.md:567-587) driving SPEC.md:412-420
 *                      assemble_residual with the literal quadrature sum
 *                      b_j += sum_q w_q |detJ| phi_j(q) sum_i f_i phi_i(q)
 *   or_assemble_colored SPEC.md:358-364 coloured-parallel schedule (OpenMP)
 *   or_greedy_color    SPEC.md:343-351 color_base_cells
 *   or_tri_rule / or_line_rule  SPEC.md:402-410 prism_quadrature
 *
 * Parity pins: tests/golden/ (generated from the reference itself by
 * tests/golden/make_golden.py) and the SPEC known-answer cases.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define OR_MAX_SLOTS 64
#define OR_MAX_Q 128

typedef struct {
  int k;
  int kind[OR_MAX_SLOTS], local[OR_MAX_SLOTS], level[OR_MAX_SLOTS];
  int dof[OR_MAX_SLOTS], within[OR_MAX_SLOTS], offset[OR_MAX_SLOTS];
} or_slots_t;

/* fspace.py:110-131 */
static int slots_of(const int32_t *delta, or_slots_t *t) {
  static const int n_local[3] = {3, 3, 1};
  int k = 0;
  for (int d = 0; d < 3; ++d) {
    int lo = delta[2 * d], conn = delta[2 * d + 1];
    if (!lo && !conn) continue;
    for (int loc = 0; loc < n_local[d]; ++loc) {
      int cnt[3] = {lo, conn, lo}, base[3] = {0, lo, lo + conn};
      for (int lev = 0; lev < 3; ++lev)
        for (int j = 0; j < cnt[lev]; ++j) {
          if (k >= OR_MAX_SLOTS) return -1;
          t->kind[k] = d;
          t->local[k] = loc;
          t->level[k] = lev;
          t->dof[k] = j;
          t->within[k] = base[lev] + j;
          t->offset[k] = lo + conn;
          ++k;
        }
    }
  }
  t->k = k;
  return k;
}

int or_slot_table(const int32_t *delta, int32_t *kind, int32_t *local,
                  int32_t *level, int32_t *dof) {
  or_slots_t t;
  int k = slots_of(delta, &t);
  for (int j = 0; j < k; ++j) {
    if (kind) kind[j] = t.kind[j];
    if (local) local[j] = t.local[j];
    if (level) level[j] = t.level[j];
    if (dof) dof[j] = t.dof[j];
  }
  return k;
}

/* fspace.py:137-149 + :192-229.  Returns total_dofs. */
int64_t or_build_cell_map(const int32_t *cv, const int32_t *ce,
                          int64_t n_cells, int64_t nv, int64_t ne,
                          const int32_t *delta, int32_t layers, int32_t *map,
                          int32_t *offsets) {
  or_slots_t t;
  int k = slots_of(delta, &t);
  if (k < 0) return -1;
  int64_t start[3], column[3], count[3] = {nv, ne, n_cells}, acc = 0;
  for (int d = 0; d < 3; ++d) {
    column[d] = (int64_t)layers * (delta[2 * d] + delta[2 * d + 1]) +
                delta[2 * d];
    start[d] = acc;
    acc += column[d] * count[d];
  }
  for (int64_t c = 0; c < n_cells && map; ++c)
    for (int j = 0; j < k; ++j) {
      int64_t ent = t.kind[j] == 0   ? cv[3 * c + t.local[j]]
                    : t.kind[j] == 1 ? ce[3 * c + t.local[j]]
                                     : c;
      int64_t v = start[t.kind[j]] + column[t.kind[j]] * ent + t.within[j];
      map[c * k + j] = (int32_t)(uint32_t)(uint64_t)v;
    }
  for (int j = 0; j < k && offsets; ++j) offsets[j] = t.offset[j];
  return acc;
}

/* extrusion.py:66-85 */
void or_extrude(const double *base, int64_t nv, int32_t layers, double h,
                double *out) {
  for (int64_t i = 0; i < nv; ++i)
    for (int l = 0; l <= layers; ++l) {
      double *p = out + 3 * (i * (layers + 1) + l);
      p[0] = base[2 * i];
      p[1] = base[2 * i + 1];
      p[2] = h * (double)l;
    }
}

/* ---------------- quadrature ------------------------- */
static int orbit_a(double w, double a, double *xy, double *wt, int n) {
  const double p[3][2] = {{a, a}, {1 - 2 * a, a}, {a, 1 - 2 * a}};
  for (int i = 0; i < 3; ++i) {
    xy[2 * n] = p[i][0];
    xy[2 * n + 1] = p[i][1];
    wt[n++] = w;
  }
  return n;
}

static int orbit_ab(double w, double a, double b, double *xy, double *wt,
                    int n) {
  double c = 1 - a - b;
  const double p[6][2] = {{a, b}, {b, a}, {a, c}, {c, a}, {b, c}, {c, b}};
  for (int i = 0; i < 6; ++i) {
    xy[2 * n] = p[i][0];
    xy[2 * n + 1] = p[i][1];
    wt[n++] = w;
  }
  return n;
}

/* Symmetric rules on the triangle (0,0),(1,0),(0,1); weights sum to 1/2.
 * Degree 4 / 6: Dunavant's 6- and 12-point orbits, degree 5: Radon's
 * 7-point rule (constants polished by tools/polish_triangle_rules.py). */
int or_tri_rule(int degree, double *xy, double *w) {
  int n = 0;
  if (degree < 0) return -1;
  if (degree <= 1) {
    xy[0] = xy[1] = 1.0 / 3.0;
    w[0] = 0.5;
    return 1;
  }
  if (degree == 2) return orbit_a(1.0 / 6.0, 1.0 / 6.0, xy, w, 0);
  if (degree <= 4) {
    n = orbit_a(0.11169079483900567, 0.4459484909159648, xy, w, 0);
    return orbit_a(0.054975871827661, 0.09157621350977078, xy, w, n);
  }
  if (degree == 5) {
    double r = sqrt(15.0);
    xy[0] = xy[1] = 1.0 / 3.0;
    w[0] = 9.0 / 80.0;
    n = orbit_a((155 - r) / 2400, (6 - r) / 21, xy, w, 1);
    return orbit_a((155 + r) / 2400, (6 + r) / 21, xy, w, n);
  }
  if (degree == 6) {
    n = orbit_a(0.05839313786319256, 0.24928674517090688, xy, w, 0);
    n = orbit_a(0.025422453185103333, 0.06308901449150202, xy, w, n);
    return orbit_ab(0.041425537809185384, 0.05314504984481456,
                    0.31035245103378556, xy, w, n);
  }
  return -1;
}

/* Gauss-Legendre on [0,1], degree//2+1 points, Newton on P_n. */
int or_line_rule(int degree, double *z, double *w) {
  if (degree < 0) return -1;
  int n = degree / 2 + 1;
  for (int i = 0; i < n; ++i) {
    double x = cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 1;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1, p1 = x;
      for (int m = 2; m <= n; ++m) {
        double p2 = ((2 * m - 1) * x * p1 - (m - 1) * p0) / m;
        p0 = p1;
        p1 = p2;
      }
      const double pn = p1, pm1 = p0; /* P_n(x), P_{n-1}(x) */
      dp = n * (x * pn - pm1) / (x * x - 1);
      double dx = pn / dp;
      x -= dx;
      if (fabs(dx) < 1e-17) break;
    }
    /* ascending order on [0,1] */
    z[n - 1 - i] = 0.5 * (x + 1);
    w[n - 1 - i] = 1.0 / ((1 - x * x) * dp * dp);
  }
  return n;
}

/* ---------------- basis functions -------------------------------------- */
static double tri_phi(int fam, int h, double xi, double eta) {
  double l[3] = {1.0 - xi - eta, xi, eta};
  if (fam == 0) return 1.0;
  if (fam == 1) return l[h];
  if (h < 3) return l[h] * (2 * l[h] - 1);
  /* edge e opposite vertex e joins (e+1, e+2) */
  int e = h - 3;
  return 4 * l[(e + 1) % 3] * l[(e + 2) % 3];
}

static double line_psi(int fam, int v, double z) {
  if (fam == 0) return 1.0;
  if (fam == 1) return v == 0 ? 1.0 - z : z;
  if (v == 0) return (1 - z) * (1 - 2 * z);
  if (v == 1) return 4 * z * (1 - z);
  return z * (2 * z - 1);
}

/* Slot -> (horizontal fn, vertical fn, component); the convention stated
 * in DESIGN.md ("slot <-> basis").  fam: 0 P0, 1 P1, 2 P2. */
int or_slot_basis(const int32_t *delta, int tri_fam, int line_fam, int ncomp,
                  int32_t *h_out, int32_t *v_out, int32_t *c_out) {
  static const int nh_of[3] = {1, 3, 6}, nv_of[3] = {1, 2, 3};
  or_slots_t t;
  int k = slots_of(delta, &t);
  if (k < 0) return -1;
  int nh = nh_of[tri_fam], nv = nv_of[line_fam];
  for (int j = 0; j < k; ++j) {
    int d = t.kind[j], vcont = delta[2 * d] > 0;
    int n_v = t.level[j] == 1 ? (vcont ? nv - 2 : nv) : 1;
    int n_h = d == 2 ? nh : 1;
    if (n_v < 1) return -2;
    int per = n_h * n_v * ncomp;
    int want = delta[2 * d + (t.level[j] == 1)];
    if (want != per) return -3;
    int hi = t.dof[j] / (n_v * ncomp), rem = t.dof[j] % (n_v * ncomp);
    int vi = rem / ncomp, comp = rem % ncomp;
    h_out[j] = d == 0 ? t.local[j] : d == 1 ? 3 + t.local[j] : hi;
    v_out[j] = t.level[j] == 0   ? 0
               : t.level[j] == 2 ? nv - 1
                                 : (vcont ? 1 : 0) + vi;
    c_out[j] = comp;
  }
  return k;
}

/* ---------------- the par-loop (Alg. 3) + residual kernel -------------- */
typedef struct {
  int k, nq, ncomp;
  double B[OR_MAX_SLOTS][OR_MAX_Q]; /* tabulated basis */
  double w[OR_MAX_Q];
  int comp[OR_MAX_SLOTS];
} or_kernel_t;

static int make_kernel(or_kernel_t *K, int k, int tri_fam, int line_fam,
                       int ncomp, const int32_t *sh, const int32_t *sv,
                       const int32_t *sc, int tri_deg, int line_deg) {
  double txy[2 * 32], tw[32], lz[16], lw[16];
  int nt = or_tri_rule(tri_deg, txy, tw), nl = or_line_rule(line_deg, lz, lw);
  if (nt < 0 || nl < 0 || nt * nl > OR_MAX_Q || k > OR_MAX_SLOTS) return -1;
  K->k = k;
  K->nq = nt * nl;
  K->ncomp = ncomp;
  for (int a = 0; a < nt; ++a)
    for (int b = 0; b < nl; ++b) {
      int q = a * nl + b; /* triangle index slowest */
      K->w[q] = tw[a] * lw[b];
      for (int j = 0; j < k; ++j)
        K->B[j][q] = tri_phi(tri_fam, sh[j], txy[2 * a], txy[2 * a + 1]) *
                     line_psi(line_fam, sv[j], lz[b]);
    }
  for (int j = 0; j < k; ++j) K->comp[j] = sc[j];
  return 0;
}

/* SPEC.md:415 |detJ| = vol(prism)/vol(ref prism), from the 6 vertices
 * (v = 2a+b); operation order matches csrc/column_loop.cuh. */
static double prism_abs_detj(const double *X, const double *Y,
                             const double *Z) {
  double xm0 = 0.5 * (X[0] + X[1]), ym0 = 0.5 * (Y[0] + Y[1]);
  double xm1 = 0.5 * (X[2] + X[3]), ym1 = 0.5 * (Y[2] + Y[3]);
  double xm2 = 0.5 * (X[4] + X[5]), ym2 = 0.5 * (Y[4] + Y[5]);
  double a2 = (xm1 - xm0) * (ym2 - ym0) - (xm2 - xm0) * (ym1 - ym0);
  double h = ((Z[1] - Z[0]) + (Z[3] - Z[2]) + (Z[5] - Z[4])) / 3.0;
  return fabs(a2 * h);
}

static void column(const or_kernel_t *K, int64_t c, int layers,
                   const int32_t *map, const int32_t *off,
                   const int32_t *xmap, const int32_t *xoff,
                   const double *coords, const double *f, double *out) {
  const int k = K->k;
  int64_t L[OR_MAX_SLOTS], LX[18];
  for (int j = 0; j < k; ++j) L[j] = map[c * k + j]; /* load once / column */
  for (int j = 0; j < 18; ++j) LX[j] = xmap[c * 18 + j];
  for (int l = 0; l < layers; ++l) {
    double X[6], Y[6], Z[6];
    for (int v = 0; v < 6; ++v) {
      X[v] = coords[LX[3 * v]];
      Y[v] = coords[LX[3 * v + 1]];
      Z[v] = coords[LX[3 * v + 2]];
    }
    const double det = prism_abs_detj(X, Y, Z);
    double loc[OR_MAX_SLOTS];
    for (int j = 0; j < k; ++j) loc[j] = 0.0;
    for (int q = 0; q < K->nq; ++q) {
      double fq[3] = {0, 0, 0};
      for (int i = 0; i < k; ++i) fq[K->comp[i]] += f[L[i]] * K->B[i][q];
      const double wd = K->w[q] * det;
      for (int j = 0; j < k; ++j) loc[j] += (wd * fq[K->comp[j]]) * K->B[j][q];
    }
    for (int j = 0; j < k; ++j) out[L[j]] += loc[j];
    /* direct vertical addressing: bump every slot by its offset */
    for (int j = 0; j < k; ++j) L[j] += off[j];
    for (int j = 0; j < 18; ++j) LX[j] += xoff[j];
  }
}

/* Sequential schedule over `order` (or 0..n_cells-1 when NULL). */
int or_assemble(int64_t n_cells, int32_t layers, int32_t k,
                const int32_t *map, const int32_t *off, const int32_t *xmap,
                const int32_t *xoff, const double *coords, int tri_fam,
                int line_fam, int ncomp, const int32_t *sh, const int32_t *sv,
                const int32_t *sc, int tri_deg, int line_deg, const double *f,
                double *out, const int32_t *order, int64_t n_order) {
  static or_kernel_t K;
  if (make_kernel(&K, k, tri_fam, line_fam, ncomp, sh, sv, sc, tri_deg,
                  line_deg))
    return -1;
  int64_t n = order ? n_order : n_cells;
  for (int64_t i = 0; i < n; ++i)
    column(&K, order ? order[i] : i, layers, map, off, xmap, xoff, coords, f,
           out);
  return 0;
}

/* Coloured-parallel schedule: colours in order, cells of one colour
 * concurrently on `threads` pthreads (cells sharing a vertex never share a
 * colour, so each DoF gets at most one contribution per colour and the
 * result is bitwise independent of the thread count). */
typedef struct {
  const or_kernel_t *K;
  const int32_t *cells;
  int64_t lo, hi;
  int32_t layers;
  const int32_t *map, *off, *xmap, *xoff;
  const double *coords, *f;
  double *out;
} or_task_t;

static void *run_task(void *p) {
  or_task_t *t = (or_task_t *)p;
  for (int64_t i = t->lo; i < t->hi; ++i)
    column(t->K, t->cells[i], t->layers, t->map, t->off, t->xmap, t->xoff,
           t->coords, t->f, t->out);
  return NULL;
}

int or_max_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

int or_assemble_colored(int64_t n_cells, int32_t layers, int32_t k,
                        const int32_t *map, const int32_t *off,
                        const int32_t *xmap, const int32_t *xoff,
                        const double *coords, int tri_fam, int line_fam,
                        int ncomp, const int32_t *sh, const int32_t *sv,
                        const int32_t *sc, int tri_deg, int line_deg,
                        const double *f, double *out,
                        const int32_t *cells_by_color, const int64_t *ptr,
                        int32_t n_colors, int32_t threads) {
  static or_kernel_t K;
  (void)n_cells;
  if (make_kernel(&K, k, tri_fam, line_fam, ncomp, sh, sv, sc, tri_deg,
                  line_deg))
    return -1;
  if (threads < 1) threads = or_max_threads();
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  or_task_t task[256];
  for (int col = 0; col < n_colors; ++col) {
    const int64_t lo = ptr[col], hi = ptr[col + 1], n = hi - lo;
    for (int t = 0; t < threads; ++t) {
      task[t] = (or_task_t){&K, cells_by_color, lo + n * t / threads,
                            lo + n * (t + 1) / threads, layers, map, off,
                            xmap, xoff, coords, f, out};
      if (t) pthread_create(&tid[t], NULL, run_task, &task[t]);
    }
    run_task(&task[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
  }
  return 0;
}

/* greedy over cells in index order. */
int32_t or_greedy_color(const int32_t *cv, int64_t n_cells,
                        const int64_t *vc_off, const int32_t *vc_cells,
                        int32_t *color) {
  int32_t ncol = 0;
  unsigned char taken[256];
  for (int64_t c = 0; c < n_cells; ++c) color[c] = -1;
  for (int64_t c = 0; c < n_cells; ++c) {
    memset(taken, 0, sizeof taken);
    for (int a = 0; a < 3; ++a) {
      int64_t v = cv[3 * c + a];
      for (int64_t e = vc_off[v]; e < vc_off[v + 1]; ++e) {
        int32_t o = color[vc_cells[e]];
        if (o >= 0 && o < 256) taken[o] = 1;
      }
    }
    int32_t p = 0;
    while (p < 255 && taken[p]) ++p;
    color[c] = p;
    if (p + 1 > ncol) ncol = p + 1;
  }
  return ncol;
}
