/*
 * mgr_oracle.c -- CPU restatement of the reference hot path (TEST ORACLE).
 *
 * Test infrastructure only: see mgr_oracle.h.  Geometry/hierarchy part here;
 * the precision-generic engine is mgr_oracle_engine.inc, instantiated for
 * double and float below.  Build: oracle/Makefile (-O2 -ffp-contract=off).
 */
#include "mgr_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* status codes: keep in sync with include/mgrg.h (errors.hpp:27-37) */
enum {
  ST_OK = 0,
  ST_INVALID_GRID = 1,
  ST_INVALID_LEVEL = 2,
  ST_SHAPE_ERROR = 3,
  ST_INVALID_FUSION = 4,
  ST_SINGULAR_SYSTEM = 5,
  ST_MISSING_CLASS = 9,
  ST_UNSUPPORTED = 14,
  ST_INVALID_ARGUMENT = 15,
  ST_OUT_OF_MEMORY = 16
};

#define MAXD 4
#define MAXL 64

typedef struct {
  int nd;
  int L;
  uint64_t shape[MAXD];
  uint64_t ext[MAXL + 1][MAXD];
  double *h[MAXD][MAXL + 1]; /* ext-1 spacings (grid.cpp:60-65) */
  double *r[MAXD][MAXL + 1]; /* ext-2 ratios (grid.cpp:66-71) */
} hier_t;

static void hier_free(hier_t *H) {
  for (int d = 0; d < MAXD; ++d)
    for (int l = 0; l <= MAXL; ++l) {
      free(H->h[d][l]);
      free(H->r[d][l]);
      H->h[d][l] = H->r[d][l] = NULL;
    }
}

static uint64_t coarse_extent(uint64_t n) { return n / 2 + 1; } /* grid.hpp:77 */
static int is_coarse_pos(uint64_t p, uint64_t n) { /* grid.hpp:74-76 */
  return p % 2 == 0 || p == n - 1;
}
static uint64_t coarse_rank(uint64_t p) { /* grid.hpp:78-80 */
  return p % 2 == 0 ? p / 2 : p / 2 + 1;
}
static uint64_t fine_rank(uint64_t p) { return (p - 1) / 2; } /* grid.hpp:81 */
static uint64_t coarse_pos(uint64_t k, uint64_t n) {          /* grid.hpp:83 */
  return 2 * k < n - 1 ? 2 * k : n - 1;
}

/* validate_grid_geometry (grid.cpp:14-36) + build_hierarchy (grid.cpp:78-112)
 * + build_dim_levels (grid.cpp:40-74). */
static int hier_build(hier_t *H, int nd, const uint64_t *shape,
                      const double *coords, int levels_cap, int min_extent) {
  memset(H, 0, sizeof(*H));
  if (nd < 1 || nd > MAXD)
    return ST_INVALID_GRID;
  H->nd = nd;
  const double *cd[MAXD];
  double *own[MAXD] = {0};
  const double *cur = coords;
  for (int d = 0; d < nd; ++d) {
    uint64_t n = shape[d];
    H->shape[d] = n;
    if (n < (uint64_t)min_extent)
      return ST_INVALID_GRID;
    if (coords) {
      cd[d] = cur;
      cur += n;
    } else {
      own[d] = (double *)malloc(sizeof(double) * n);
      for (uint64_t i = 0; i < n; ++i)
        own[d][i] = n > 1 ? (double)i / (double)(n - 1) : 0.0;
      cd[d] = own[d];
    }
    for (uint64_t i = 0; i + 1 < n; ++i)
      if (!(cd[d][i] < cd[d][i + 1])) {
        for (int k = 0; k < nd; ++k)
          free(own[k]);
        return ST_INVALID_GRID;
      }
  }
  int levels = 0, any = 0;
  for (int d = 0; d < nd; ++d) {
    uint64_t e = shape[d];
    if (e < 3)
      continue;
    int depth = (int)floor(log2((double)(e - 1)));
    levels = any ? (depth < levels ? depth : levels) : depth;
    any = 1;
  }
  int st = ST_OK;
  if (!any)
    st = ST_INVALID_GRID;
  else if (levels_cap < 0)
    st = ST_INVALID_LEVEL;
  if (st == ST_OK && levels_cap > 0 && levels_cap < levels)
    levels = levels_cap;
  if (st == ST_OK && levels > MAXL)
    st = ST_UNSUPPORTED;
  if (st != ST_OK) {
    for (int k = 0; k < nd; ++k)
      free(own[k]);
    return st;
  }
  H->L = levels;
  for (int d = 0; d < nd; ++d) {
    uint64_t n = shape[d];
    /* index sets: idx[L] = 0..n-1, idx[l] = evens of idx[l+1] + last */
    uint64_t *idx[MAXL + 1];
    idx[levels] = (uint64_t *)malloc(sizeof(uint64_t) * n);
    for (uint64_t i = 0; i < n; ++i)
      idx[levels][i] = i;
    H->ext[levels][d] = n;
    for (int l = levels - 1; l >= 0; --l) {
      uint64_t fn = H->ext[l + 1][d];
      uint64_t *fine = idx[l + 1];
      uint64_t *c = (uint64_t *)malloc(sizeof(uint64_t) * (fn / 2 + 2));
      uint64_t m = 0;
      for (uint64_t p = 0; p < fn; p += 2)
        c[m++] = fine[p];
      if (c[m - 1] != fine[fn - 1])
        c[m++] = fine[fn - 1];
      idx[l] = c;
      H->ext[l][d] = m;
    }
    for (int l = 0; l <= levels; ++l) {
      uint64_t e = H->ext[l][d];
      double *h = (double *)malloc(sizeof(double) * (e > 1 ? e - 1 : 1));
      for (uint64_t i = 0; i + 1 < e; ++i)
        h[i] = cd[d][idx[l][i + 1]] - cd[d][idx[l][i]];
      double *r = (double *)malloc(sizeof(double) * (e > 2 ? e - 2 : 1));
      if (e >= 3)
        for (uint64_t i = 0; i + 2 < e; ++i)
          r[i] = h[i] / (h[i] + h[i + 1]);
      H->h[d][l] = h;
      H->r[d][l] = r;
    }
    for (int l = 0; l <= levels; ++l)
      free(idx[l]);
  }
  for (int k = 0; k < nd; ++k)
    free(own[k]);
  return ST_OK;
}

static uint64_t num_nodes(const hier_t *H, int l) {
  uint64_t n = 1;
  for (int d = 0; d < H->nd; ++d)
    n *= H->ext[l][d];
  return n;
}

/* make_class_layout (grid.cpp:140-165). */
typedef struct {
  uint64_t base[1 << MAXD];
  uint64_t ext[1 << MAXD][MAXD];
  uint64_t total;
} layout_t;

static void make_layout(const hier_t *H, int l, layout_t *c) {
  memset(c, 0, sizeof(*c));
  uint64_t off = 0;
  for (unsigned mask = 1; mask < (1u << H->nd); ++mask) {
    uint64_t count = 1;
    for (int d = 0; d < H->nd; ++d) {
      uint64_t n = H->ext[l][d];
      c->ext[mask][d] = ((mask >> d) & 1) ? n - coarse_extent(n) : coarse_extent(n);
      count *= c->ext[mask][d];
    }
    c->base[mask] = off;
    off += count;
  }
  c->total = off;
}

/* class_slot (grid.hpp:149-164). */
static uint64_t class_slot(const layout_t *c, int nd, const uint64_t *lshape,
                           const uint64_t *pos) {
  unsigned mask = 0;
  for (int d = 0; d < nd; ++d)
    if (!is_coarse_pos(pos[d], lshape[d]))
      mask |= 1u << d;
  uint64_t idx = 0, mult = 1;
  for (int d = 0; d < nd; ++d) {
    uint64_t w = ((mask >> d) & 1) ? fine_rank(pos[d]) : coarse_rank(pos[d]);
    idx += w * mult;
    mult *= c->ext[mask][d];
  }
  return c->base[mask] + idx;
}

/* ---- row-parallel loops (pthreads) ----------------------------------------
 * The engine's row loops (GPK rows, mass-transfer fibers, Thomas fibers,
 * pack / expand / scatter elements) are independent: every element is
 * computed by exactly the reference expression in the reference order, so
 * splitting a loop over threads never changes a value.  This only makes the
 * checker fast enough to run at the BASELINE sizes (1025^3) inside the GPU
 * test suite.  Small loops run on the calling thread. */
static int g_threads = 0; /* 0 = all online CPUs */

int mgro_set_threads(int n) {
  int old = g_threads;
  g_threads = n < 0 ? 0 : n;
  return old;
}

typedef void (*range_fn)(void *ctx, int64_t lo, int64_t hi);
typedef struct {
  range_fn fn;
  void *ctx;
  int64_t lo, hi;
} par_job;

static void *par_tramp(void *p) {
  par_job *j = (par_job *)p;
  j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}

/* fn over [0, n) split in contiguous ranges; `work` = elements touched, the
 * serial cutoff. */
static void par_for(int64_t n, uint64_t work, range_fn fn, void *ctx) {
  int T = g_threads;
  if (T <= 0) {
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    T = c > 0 ? (int)c : 1;
  }
  if (T > 64)
    T = 64;
  if ((int64_t)T > n)
    T = (int)n;
  if (T <= 1 || work < (1u << 18)) {
    if (n > 0)
      fn(ctx, 0, n);
    return;
  }
  pthread_t th[64];
  par_job job[64];
  int started[64] = {0};
  for (int t = 0; t < T; ++t) {
    job[t].fn = fn;
    job[t].ctx = ctx;
    job[t].lo = n * t / T;
    job[t].hi = n * (t + 1) / T;
    if (t > 0)
      started[t] = pthread_create(&th[t], NULL, par_tramp, &job[t]) == 0;
  }
  fn(ctx, job[0].lo, job[0].hi);
  for (int t = 1; t < T; ++t) {
    if (started[t])
      pthread_join(th[t], NULL);
    else
      fn(ctx, job[t].lo, job[t].hi); /* thread creation failed: run inline */
  }
}

int mgro_hierarchy(int ndims, const uint64_t *shape, const double *coords,
                   int levels_cap, int min_extent, int *levels_out,
                   uint64_t *level_extents) {
  hier_t H;
  int st = hier_build(&H, ndims, shape, coords, levels_cap, min_extent);
  if (st)
    return st;
  *levels_out = H.L;
  if (level_extents)
    for (int l = 0; l <= H.L; ++l)
      for (int d = 0; d < ndims; ++d)
        level_extents[l * ndims + d] = H.ext[l][d];
  hier_free(&H);
  return ST_OK;
}

int mgro_class_offsets(int ndims, const uint64_t *shape, int levels,
                       uint64_t *offsets) {
  hier_t H;
  int st = hier_build(&H, ndims, shape, NULL, levels, 2);
  if (st)
    return st;
  if (H.L != levels) {
    hier_free(&H);
    return ST_INVALID_LEVEL;
  }
  offsets[0] = 0;
  for (int l = 0; l <= H.L; ++l)
    offsets[l + 1] = num_nodes(&H, l);
  hier_free(&H);
  return ST_OK;
}

int mgro_class_layout(int ndims, const uint64_t *shape, int levels, int level,
                      uint64_t *type_base, uint64_t *type_extents) {
  hier_t H;
  int st = hier_build(&H, ndims, shape, NULL, levels, 2);
  if (st)
    return st;
  if (level < 1 || level > H.L) {
    hier_free(&H);
    return ST_INVALID_LEVEL;
  }
  layout_t c;
  make_layout(&H, level, &c);
  for (unsigned m = 0; m < (1u << ndims); ++m) {
    type_base[m] = c.base[m];
    for (int d = 0; d < ndims; ++d)
      type_extents[m * ndims + d] = c.ext[m][d];
  }
  hier_free(&H);
  return ST_OK;
}

/* make_layout_map + reorder (grid.cpp:167-221, grid.hpp:177-196). */
int mgro_reorder_f64(int ndims, const uint64_t *shape, const double *coords,
                     int levels_cap, int level, int direction,
                     const double *in, double *out) {
  hier_t H;
  int st = hier_build(&H, ndims, shape, coords, levels_cap, 3);
  if (st)
    return st;
  if (level < 1 || level > H.L) {
    hier_free(&H);
    return ST_INVALID_LEVEL;
  }
  const int nd = ndims;
  uint64_t lshape[MAXD], cshape[MAXD], str[MAXD];
  uint64_t acc = 1;
  for (int d = 0; d < nd; ++d) {
    lshape[d] = H.ext[level][d];
    cshape[d] = H.ext[level - 1][d];
    str[d] = acc;
    acc *= lshape[d];
  }
  const uint64_t total = acc;
  uint64_t *perm = (uint64_t *)malloc(sizeof(uint64_t) * total);
  uint64_t k = 0, pos[MAXD] = {0};
  const uint64_t ccount = num_nodes(&H, level - 1);
  for (uint64_t c = 0; c < ccount; ++c) {
    uint64_t off = 0;
    for (int d = 0; d < nd; ++d)
      off += coarse_pos(pos[d], lshape[d]) * str[d];
    perm[k++] = off;
    for (int d = 0; d < nd; ++d) {
      if (++pos[d] < cshape[d])
        break;
      pos[d] = 0;
    }
  }
  layout_t cl;
  make_layout(&H, level, &cl);
  for (unsigned mask = 1; mask < (1u << nd); ++mask) {
    uint64_t count = 1, w[MAXD] = {0};
    for (int d = 0; d < nd; ++d)
      count *= cl.ext[mask][d];
    for (uint64_t c = 0; c < count; ++c) {
      uint64_t off = 0;
      for (int d = 0; d < nd; ++d) {
        uint64_t p = ((mask >> d) & 1) ? 2 * w[d] + 1 : coarse_pos(w[d], lshape[d]);
        off += p * str[d];
      }
      perm[ccount + cl.base[mask] + c] = off;
      for (int d = 0; d < nd; ++d) {
        if (++w[d] < cl.ext[mask][d])
          break;
        w[d] = 0;
      }
    }
  }
  if (direction == 0)
    for (uint64_t i = 0; i < total; ++i)
      out[i] = in[perm[i]];
  else
    for (uint64_t i = 0; i < total; ++i)
      out[perm[i]] = in[i];
  free(perm);
  hier_free(&H);
  return ST_OK;
}

/* ---- precision-generic engine ---- */
#define REAL double
#define SFX(name) name##_f64
#include "mgr_oracle_engine.inc"
#undef REAL
#undef SFX

#define REAL float
#define SFX(name) name##_f32
#include "mgr_oracle_engine.inc"
#undef REAL
#undef SFX
