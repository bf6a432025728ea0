/*
 * cpu_fast.c -- TEST INFRASTRUCTURE ONLY: the CPU baseline of bench.py.
 *
 * The reference's column loop (SPEC.md:333-341 iterate_columns, Alg. 3 of
 * PAPER.md:567-587) in a race-free parallel schedule (SPEC.md:358-364's
 * colouring, or -- cache-friendlier -- contiguous cell blocks, even blocks
 * then odd ones, when no two blocks of a parity share an entity), as a
 * tuned CPU code would run it: the element matrix pre-integrated once
 * (the same M_ref the GPU uses, SPEC.md:412-420 b = |det J| M_ref f per
 * cell-layer), only its nonzeros applied, |det J| from the extruded
 * coordinate field read through the coordinate map (the same formula as
 * the oracle, prismesh_oracle.c prism_abs_detj), output zeroed by the
 * worker threads (first touch), all host cores, built -O3 -march=native
 * -ffast-math on the machine that runs it (PAPER.md:777-783 used GCC -O3
 * -march=native -ffast-math).  Checked against the literal oracle in
 * tests/test_cpu_baseline.py.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define CF_MAXK 64

typedef struct {
  int64_t n_cells;
  int32_t layers, k, nnz;
  const int32_t *map, *off, *xmap, *xoff;
  const double *coords, *x;
  double *y;
  int64_t n_dofs;
  const int32_t *order;
  const int64_t *tptr; /* [n_colors * threads + 1]: colour c, thread t */
  int32_t n_colors, threads;
  int32_t ri[CF_MAXK * CF_MAXK], ci[CF_MAXK * CF_MAXK];
  double mv[CF_MAXK * CF_MAXK];
  pthread_barrier_t bar;
} cf_job_t;

typedef struct {
  cf_job_t *job;
  int tid;
} cf_arg_t;

static inline __attribute__((unused)) double abs_detj(const double *X, const double *Y,
                              const double *Z) {
  const double xm0 = 0.5 * (X[0] + X[1]), ym0 = 0.5 * (Y[0] + Y[1]);
  const double xm1 = 0.5 * (X[2] + X[3]), ym1 = 0.5 * (Y[2] + Y[3]);
  const double xm2 = 0.5 * (X[4] + X[5]), ym2 = 0.5 * (Y[4] + Y[5]);
  const double a2 = (xm1 - xm0) * (ym2 - ym0) - (xm2 - xm0) * (ym1 - ym0);
  const double h = ((Z[1] - Z[0]) + (Z[3] - Z[2]) + (Z[5] - Z[4])) / 3.0;
  return fabs(a2 * h);
}

static void *cf_worker(void *p) {
  cf_arg_t *a = (cf_arg_t *)p;
  cf_job_t *J = a->job;
  const int T = J->threads, t = a->tid;
  /* first-touch zeroing of this thread's slice of y */
  const int64_t z0 = J->n_dofs * t / T, z1 = J->n_dofs * (t + 1) / T;
  memset(J->y + z0, 0, sizeof(double) * (size_t)(z1 - z0));
  pthread_barrier_wait(&J->bar);
  const int k = J->k, L = J->layers, nnz = J->nnz;
  /* locals (restrict): the compiler may keep maps, offsets and the matrix
   * in registers / L1 instead of reloading them after every store to y */
  const double *restrict x = J->x, *restrict coords = J->coords;
  double *restrict y = J->y;
  int64_t off[CF_MAXK], xoff[18];
  int32_t ri[CF_MAXK * CF_MAXK], ci[CF_MAXK * CF_MAXK];
  double mv[CF_MAXK * CF_MAXK];
  for (int j = 0; j < k; ++j) off[j] = J->off[j];
  for (int j = 0; j < 18; ++j) xoff[j] = J->xoff[j];
  for (int q = 0; q < nnz; ++q) ri[q] = J->ri[q], ci[q] = J->ci[q], mv[q] = J->mv[q];
  /* the layer loop innermost over whole column chunks (the structure the
   * paper's generated code has): gather a chunk of every slot's column,
   * |det J| for the chunk, the element matrix applied row by row over the
   * chunk (vectorised over layers), then the scatter */
  enum { LC = 64 };
  double xl[CF_MAXK][LC], yl[CF_MAXK][LC], cc[18][LC], det[LC];
  int64_t dof[CF_MAXK], xd[18];
  for (int col = 0; col < J->n_colors; ++col) {
    const int64_t c0 = J->tptr[col * T + t], c1 = J->tptr[col * T + t + 1];
    for (int64_t i = c0; i < c1; ++i) {
      const int64_t c = J->order[i];
      for (int j = 0; j < k; ++j) dof[j] = J->map[c * k + j];
      for (int j = 0; j < 18; ++j) xd[j] = J->xmap[c * 18 + j];
      for (int l0 = 0; l0 < L; l0 += LC) {
        const int nl = L - l0 < LC ? L - l0 : LC;
        for (int j = 0; j < k; ++j) {
          const double *restrict xp = x + dof[j] + l0 * off[j];
          const int64_t o = off[j];
          for (int l = 0; l < nl; ++l) xl[j][l] = xp[l * o];
        }
        for (int j = 0; j < 18; ++j) {
          const double *restrict cp = coords + xd[j] + l0 * xoff[j];
          const int64_t o = xoff[j];
          for (int l = 0; l < nl; ++l) cc[j][l] = cp[l * o];
        }
        /* coordinate slots 6a + 3b + comp (vertex a, level b) */
        for (int l = 0; l < nl; ++l) {
          const double xm0 = 0.5 * (cc[0][l] + cc[3][l]),
                       ym0 = 0.5 * (cc[1][l] + cc[4][l]);
          const double xm1 = 0.5 * (cc[6][l] + cc[9][l]),
                       ym1 = 0.5 * (cc[7][l] + cc[10][l]);
          const double xm2 = 0.5 * (cc[12][l] + cc[15][l]),
                       ym2 = 0.5 * (cc[13][l] + cc[16][l]);
          const double a2 =
              (xm1 - xm0) * (ym2 - ym0) - (xm2 - xm0) * (ym1 - ym0);
          const double h = ((cc[5][l] - cc[2][l]) + (cc[11][l] - cc[8][l]) +
                            (cc[17][l] - cc[14][l])) / 3.0;
          det[l] = fabs(a2 * h);
        }
        for (int j = 0; j < k; ++j)
          for (int l = 0; l < nl; ++l) yl[j][l] = 0.0;
        for (int q = 0; q < nnz; ++q) {
          const double m = mv[q];
          double *restrict yr = yl[ri[q]];
          const double *restrict xr = xl[ci[q]];
          for (int l = 0; l < nl; ++l) yr[l] += m * xr[l];
        }
        for (int j = 0; j < k; ++j) {
          double *yp = y + dof[j] + l0 * off[j];
          const int64_t o = off[j];
          for (int l = 0; l < nl; ++l) yp[l * o] += det[l] * yl[j][l];
        }
      }
    }
    pthread_barrier_wait(&J->bar);
  }
  return NULL;
}

int cf_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

/* y = M x over all cell-layers (y zeroed here); thread t of colour c walks
 * cells order[tptr[c T + t] .. tptr[c T + t + 1]), colours one after the
 * other (no two threads of a colour touch one DoF) */
int cf_mass(int64_t n_cells, int32_t layers, int32_t k, const int32_t *map,
            const int32_t *off, const int32_t *xmap, const int32_t *xoff,
            const double *coords, const double *mref, const double *x,
            double *y, int64_t n_dofs, const int32_t *order,
            const int64_t *tptr, int32_t n_colors, int32_t threads) {
  if (k < 1 || k > CF_MAXK || layers < 1 || n_cells < 0) return 1;
  cf_job_t *J = (cf_job_t *)calloc(1, sizeof(cf_job_t));
  J->n_cells = n_cells, J->layers = layers, J->k = k;
  J->map = map, J->off = off, J->xmap = xmap, J->xoff = xoff;
  J->coords = coords, J->x = x, J->y = y, J->n_dofs = n_dofs;
  J->order = order, J->tptr = tptr, J->n_colors = n_colors;
  J->threads = threads > 0 ? threads : cf_threads();
  for (int r = 0; r < k; ++r)
    for (int c = 0; c < k; ++c)
      if (mref[r * k + c] != 0.0) {
        J->ri[J->nnz] = r, J->ci[J->nnz] = c, J->mv[J->nnz] = mref[r * k + c];
        ++J->nnz;
      }
  pthread_barrier_init(&J->bar, NULL, (unsigned)J->threads);
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * J->threads);
  cf_arg_t *args = (cf_arg_t *)malloc(sizeof(cf_arg_t) * J->threads);
  for (int t = 0; t < J->threads; ++t) {
    args[t].job = J, args[t].tid = t;
    if (t) pthread_create(&th[t], NULL, cf_worker, &args[t]);
  }
  cf_worker(&args[0]);
  for (int t = 1; t < J->threads; ++t) pthread_join(th[t], NULL);
  pthread_barrier_destroy(&J->bar);
  free(th), free(args), free(J);
  return 0;
}
