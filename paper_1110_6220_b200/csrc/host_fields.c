/*
 * Host-side speed fields and cell geometry for the Eikonal hot path.
 *
 * Speed fields are evaluated on the host with the same libm the reference
 * links (speed evaluation is a host std::function in the reference,
 * grid.hpp:64,71), and the device only ever sees the sampled arrays -- the
 * "F bit-identity rule" of SURVEY.md §8(d).  Compiled with
 * -ffp-contract=off so expression shapes round exactly like the reference's
 * Release build (no FMA).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "eikonal_b200.h"

static const double kPi = 3.14159265358979323846; /* speed_fields.cpp:10 */

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
static double clampd(double v, double lo, double hi) {
  /* std::clamp(v, lo, hi): v < lo ? lo : (hi < v ? hi : v) */
  return v < lo ? lo : (hi < v ? hi : v);
}

/* Sinusoid-sum term, separable form: sin(a+b) = sin a cos b + cos a sin b
 * with a = pi*p*x + phi, b = pi*q*y.  This separable expression *is* the
 * definition of the config-5 field, so grid sampling can tabulate the x and
 * y factors and still match on-demand evaluation bit for bit. */
static double sinsum_eval(const eik_field* f, double x, double y) {
  double s = 0.0;
  for (int k = 0; k < f->K; ++k) {
    double a = kPi * f->kp[k] * x + f->kphi[k];
    double b = kPi * f->kq[k] * y;
    s = s + (sin(a) * cos(b) + cos(a) * sin(b));
  }
  return 1.0 + 0.5 * (s / (double)f->K);
}

double eik_field_eval(const eik_field* f, double x, double y) {
  switch (f->kind) {
    case EIK_FIELD_CONSTANT:
      return f->value;
    case EIK_FIELD_SINUSOID:
      /* speed_fields.cpp:27-29 */
      return 1.0 + f->amp * sin(f->freq * kPi * x) * sin(f->freq * kPi * y);
    case EIK_FIELD_CHECKER: {
      /* speed_fields.cpp:12-14,23-26 */
      int a = clampi((int)floor(x * f->checkers), 0, f->checkers - 1);
      int b = clampi((int)floor(y * f->checkers), 0, f->checkers - 1);
      return ((a + b) % 2 == 0) ? f->slow : f->fast;
    }
    case EIK_FIELD_COMB: {
      /* speed_fields.cpp:30-41 */
      for (int b = 1; b <= f->n_barriers; ++b) {
        double xc = (double)b / (f->n_barriers + 1);
        if (x < xc - 0.5 * f->barrier_width || x > xc + 0.5 * f->barrier_width)
          continue;
        int gap_at_top = (b % 2 == 1);
        int in_barrier = gap_at_top ? (y <= 1.0 - f->gap_fraction)
                                    : (y >= f->gap_fraction);
        if (in_barrier) return f->barrier_speed;
      }
      return 1.0;
    }
    case EIK_FIELD_BLOCKS: {
      int bx = clampi((int)floor((x - f->bx0) * f->bscale), 0, f->nb - 1);
      int by = clampi((int)floor((y - f->by0) * f->bscale), 0, f->nb - 1);
      return f->block_speed[(int64_t)by * f->nb + bx];
    }
    case EIK_FIELD_NODEMASK: {
      const eik_grid* g = &f->mask_grid;
      int64_t i = (int64_t)llround((x - g->x0) / g->h);
      int64_t j = (int64_t)llround((y - g->y0) / g->h);
      if (i < 0) i = 0;
      if (i > g->m - 1) i = g->m - 1;
      if (j < 0) j = 0;
      if (j > g->n - 1) j = g->n - 1;
      return f->mask[j * g->m + i] ? f->slow : f->fast;
    }
    case EIK_FIELD_SINSUM:
      return sinsum_eval(f, x, y);
  }
  return NAN;
}

int eik_field_eval_points(const eik_field* f, const double* xy, int64_t count,
                          double* out) {
  if (!f || (!xy && count) || (!out && count) || count < 0) return EIK_ERR_DOMAIN;
  /* independent points: any thread count gives the same bits */
#pragma omp parallel for schedule(static) if (count > 65536)
  for (int64_t k = 0; k < count; ++k) out[k] = eik_field_eval(f, xy[2 * k], xy[2 * k + 1]);
  return EIK_OK;
}

/* Grid coordinates exactly as Grid::x / Grid::y (grid.hpp:51-52). */
static double gx(const eik_grid* g, int64_t i) { return g->x0 + (double)i * g->h; }
static double gy(const eik_grid* g, int64_t j) { return g->y0 + (double)j * g->h; }

int eik_field_sample(const eik_field* f, const eik_grid* g, double* out,
                     int32_t threads) {
  if (!g) return EIK_ERR_DOMAIN;
  return eik_field_sample_rows(f, g, 0, g->n, out, threads);
}

/* Rows [row0, row0 + nrows) of the grid's nodes (out[(j - row0) * m + i]),
 * with the GLOBAL coordinates y0 + j*h: a strip samples exactly the bits the
 * whole grid's sampling holds there (a local grid with a shifted y0 would
 * round differently). */
int eik_field_sample_rows(const eik_field* f, const eik_grid* g, int64_t row0, int64_t nrows,
                          double* out, int32_t threads) {
  if (!f || !g || !out || g->m < 1 || g->n < 1 || row0 < 0 || nrows < 0 || row0 + nrows > g->n)
    return EIK_ERR_DOMAIN;
  const int64_t m = g->m, n = nrows;
  if (f->kind == EIK_FIELD_SINSUM) {
    /* Tabulated separable evaluation; identical bits to sinsum_eval. */
    const int K = f->K;
    double* sa = (double*)malloc(sizeof(double) * (size_t)K * (size_t)m);
    double* ca = (double*)malloc(sizeof(double) * (size_t)K * (size_t)m);
    double* sb = (double*)malloc(sizeof(double) * (size_t)K * (size_t)(n + 1));
    double* cb = (double*)malloc(sizeof(double) * (size_t)K * (size_t)(n + 1));
    if (!sa || !ca || !sb || !cb) {
      free(sa); free(ca); free(sb); free(cb);
      return EIK_ERR_DOMAIN;
    }
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) schedule(static)
    for (int64_t i = 0; i < m; ++i) {
      double x = gx(g, i);
      for (int k = 0; k < K; ++k) {
        double a = kPi * f->kp[k] * x + f->kphi[k];
        sa[(size_t)i * K + k] = sin(a);
        ca[(size_t)i * K + k] = cos(a);
      }
    }
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) schedule(static)
    for (int64_t jj = 0; jj < n; ++jj) {
      double y = gy(g, row0 + jj);
      for (int k = 0; k < K; ++k) {
        double b = kPi * f->kq[k] * y;
        sb[(size_t)jj * K + k] = sin(b);
        cb[(size_t)jj * K + k] = cos(b);
      }
    }
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) schedule(static)
    for (int64_t j = row0; j < row0 + n; ++j) {
      const double* sbj = sb + (size_t)(j - row0) * K;
      const double* cbj = cb + (size_t)(j - row0) * K;
      for (int64_t i = 0; i < m; ++i) {
        const double* sai = sa + (size_t)i * K;
        const double* cai = ca + (size_t)i * K;
        double s = 0.0;
        for (int k = 0; k < K; ++k) s = s + (sai[k] * cbj[k] + cai[k] * sbj[k]);
        out[(j - row0) * m + i] = 1.0 + 0.5 * (s / (double)K);
      }
    }
    free(sa); free(ca); free(sb); free(cb);
    return EIK_OK;
  }
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) schedule(static)
  for (int64_t j = row0; j < row0 + n; ++j) {
    double y = gy(g, j);
    for (int64_t i = 0; i < m; ++i) out[(j - row0) * m + i] = eik_field_eval(f, gx(g, i), y);
  }
  return EIK_OK;
}

/* ---- cell geometry: build_cells (cells.cpp:7-47) ----------------------- */

static void split_axis(int64_t nodes, int32_t cells, int64_t* begin, int64_t* end) {
  const int64_t base = nodes / cells;
  int64_t at = 0;
  for (int32_t c = 0; c < cells; ++c) {
    begin[c] = at;
    at += base;
    if (c == cells - 1) at = nodes; /* remainder goes to the last cell */
    end[c] = at;
  }
}

static int cells_ok(const eik_grid* g, int32_t cx, int32_t cy) {
  return g && cx >= 1 && cy >= 1 && cx <= g->m && cy <= g->n;
}

int64_t eik_cell_probe_points(const eik_grid* g, int32_t cells_x,
                              int32_t cells_y, int32_t side, double* xy) {
  if (!cells_ok(g, cells_x, cells_y) || side < 0 || side > 3) return -1;
  const int64_t m = g->m, n = g->n;
  const int vertical = (side == 0 || side == 1);
  const int32_t ncell = vertical ? cells_x : cells_y;
  const int64_t len = vertical ? n : m;
  if (!xy) return (int64_t)ncell * len;
  int64_t* b = (int64_t*)malloc(sizeof(int64_t) * (size_t)ncell);
  int64_t* e = (int64_t*)malloc(sizeof(int64_t) * (size_t)ncell);
  if (!b || !e) { free(b); free(e); return -1; }
  split_axis(vertical ? m : n, ncell, b, e);
  /* hc along the side's axis: (m / cells_x) * h (cells.cpp:44-45) */
  const double hc = vertical ? (double)(m / cells_x) * g->h : (double)(n / cells_y) * g->h;
  const double step = 0.5 * (g->h + hc); /* heap_cell.cpp:199 */
  const double xmax = gx(g, m - 1), ymax = gy(g, n - 1);
#pragma omp parallel for schedule(static) if ((int64_t)ncell * len > 65536)
  for (int32_t c = 0; c < ncell; ++c) {
    for (int64_t t = 0; t < len; ++t) {
      int64_t i, j;
      int adi = 0, adj = 0;
      /* strip_for (heap_cell.cpp:29-40) */
      switch (side) {
        case 0: i = b[c]; j = t; adi = -1; break;
        case 1: i = e[c] - 1; j = t; adi = 1; break;
        case 2: i = t; j = b[c]; adj = -1; break;
        default: i = t; j = e[c] - 1; adj = 1; break;
      }
      double px = gx(g, i) + step * (double)adi;
      double py = gy(g, j) + step * (double)adj;
      px = clampd(px, g->x0, xmax);
      py = clampd(py, g->y0, ymax);
      int64_t k = (int64_t)c * len + t;
      xy[2 * k] = px;
      xy[2 * k + 1] = py;
    }
  }
  free(b);
  free(e);
  return (int64_t)ncell * len;
}

int64_t eik_cell_centers(const eik_grid* g, int32_t cells_x, int32_t cells_y,
                         double* xy) {
  if (!cells_ok(g, cells_x, cells_y)) return -1;
  const int64_t J = (int64_t)cells_x * cells_y;
  if (!xy) return J;
  int64_t* ib = (int64_t*)malloc(sizeof(int64_t) * (size_t)cells_x);
  int64_t* ie = (int64_t*)malloc(sizeof(int64_t) * (size_t)cells_x);
  int64_t* jb = (int64_t*)malloc(sizeof(int64_t) * (size_t)cells_y);
  int64_t* je = (int64_t*)malloc(sizeof(int64_t) * (size_t)cells_y);
  if (!ib || !ie || !jb || !je) { free(ib); free(ie); free(jb); free(je); return -1; }
  split_axis(g->m, cells_x, ib, ie);
  split_axis(g->n, cells_y, jb, je);
  for (int32_t cy = 0; cy < cells_y; ++cy)
    for (int32_t cx = 0; cx < cells_x; ++cx) {
      int64_t k = (int64_t)cy * cells_x + cx;
      /* CellDecomposition::center (cells.hpp:44-48) */
      xy[2 * k] = 0.5 * (gx(g, ib[cx]) + gx(g, ie[cx] - 1));
      xy[2 * k + 1] = 0.5 * (gy(g, jb[cy]) + gy(g, je[cy] - 1));
    }
  free(ib); free(ie); free(jb); free(je);
  return J;
}
