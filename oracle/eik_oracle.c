/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY (see eik_oracle.h).
 *
 * Sequential CPU restatement of the reference algorithms; every function
 * cites the reference lines it follows.  Compiled with -O2
 * -ffp-contract=off (no FMA), matching the reference's Release objects.
 */
#include "eik_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define INF (1.0 / 0.0)

enum { SW = 0, NW = 1, NE = 2, SE = 3 }; /* SweepDir, local_update.hpp:23 */
enum { WEST = 0, EAST = 1, SOUTH = 2, NORTH = 3 }; /* Side, cells.hpp:12 */

static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */
static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* ---- local update: local_update.hpp:30-64 ------------------------------ */

double orc_quadrant_update(double ua, double ub, double f, double h) {
  const double c = h / f;
  if (isfinite(ua) && isfinite(ub)) {
    const double diff = ua - ub;
    if (fabs(diff) <= c) return 0.5 * (ua + ub) + 0.5 * sqrt(2.0 * c * c - diff * diff);
  }
  return c + dmin(ua, ub);
}

double orc_node_update(const double nb[4], double f, double h) {
  return orc_quadrant_update(dmin(nb[0], nb[1]), dmin(nb[2], nb[3]), f, h);
}

double orc_directional_update(const double nb[4], int dir, double f, double h) {
  switch (dir) {
    case NE: return orc_quadrant_update(nb[0], nb[2], f, h);
    case NW: return orc_quadrant_update(nb[1], nb[2], f, h);
    case SE: return orc_quadrant_update(nb[0], nb[3], f, h);
    case SW: return orc_quadrant_update(nb[1], nb[3], f, h);
  }
  return INF;
}

/* gather_neighbors (local_update.hpp:67-74): {E, W, N, S}, off-grid +inf */
static void gather(const double* v, int64_t m, int64_t n, int64_t i, int64_t j, double nb[4]) {
  nb[0] = (i + 1 < m) ? v[j * m + i + 1] : INF;
  nb[1] = (i - 1 >= 0) ? v[j * m + i - 1] : INF;
  nb[2] = (j + 1 < n) ? v[(j + 1) * m + i] : INF;
  nb[3] = (j - 1 >= 0) ? v[(j - 1) * m + i] : INF;
}

static void init_values(const orc_problem* p, double* v, char* is_exit) {
  const int64_t M = p->m * p->n;
  for (int64_t k = 0; k < M; ++k) v[k] = INF;
  if (is_exit) memset(is_exit, 0, (size_t)M);
  for (int64_t k = 0; k < p->n_exit; ++k) {
    v[p->exit_nodes[k]] = p->exit_cost[k];
    if (is_exit) is_exit[p->exit_nodes[k]] = 1;
  }
}

/* ---- IndexedMinHeap (indexed_min_heap.hpp:11-106) ---------------------- */

typedef struct heap {
  double* key;
  int64_t* pos;
  int64_t* h;
  int64_t size;
} heap;

static int heap_init(heap* H, int64_t cap) {
  H->key = (double*)calloc((size_t)(cap > 0 ? cap : 1), sizeof(double));
  H->pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  H->h = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  H->size = 0;
  if (!H->key || !H->pos || !H->h) return 1;
  for (int64_t k = 0; k < cap; ++k) H->pos[k] = -1;
  return 0;
}
static void heap_free(heap* H) { free(H->key); free(H->pos); free(H->h); }
static int hless(int64_t a, double ka, int64_t b, double kb) {
  if (ka != kb) return ka < kb;
  return a < b; /* ties -> smaller id, indexed_min_heap.hpp:66-69 */
}
static void sift_up(heap* H, int64_t p) {
  int64_t id = H->h[p];
  while (p > 0) {
    int64_t parent = (p - 1) / 2;
    if (!hless(id, H->key[id], H->h[parent], H->key[H->h[parent]])) break;
    H->h[p] = H->h[parent];
    H->pos[H->h[p]] = p;
    p = parent;
  }
  H->h[p] = id;
  H->pos[id] = p;
}
static void sift_down(heap* H, int64_t p) {
  int64_t id = H->h[p];
  for (;;) {
    int64_t child = 2 * p + 1;
    if (child >= H->size) break;
    int64_t right = child + 1;
    if (right < H->size && hless(H->h[right], H->key[H->h[right]], H->h[child], H->key[H->h[child]]))
      child = right;
    if (!hless(H->h[child], H->key[H->h[child]], id, H->key[id])) break;
    H->h[p] = H->h[child];
    H->pos[H->h[p]] = p;
    p = child;
  }
  H->h[p] = id;
  H->pos[id] = p;
}
static int heap_contains(const heap* H, int64_t id) { return H->pos[id] != -1; }
static void heap_insert(heap* H, int64_t id, double key) {
  H->key[id] = key;
  H->pos[id] = H->size;
  H->h[H->size++] = id;
  sift_up(H, H->pos[id]);
}
static void heap_decrease(heap* H, int64_t id, double key) {
  H->key[id] = key;
  sift_up(H, H->pos[id]);
}
static int64_t heap_pop(heap* H) {
  int64_t top = H->h[0];
  int64_t last = H->h[--H->size];
  H->pos[top] = -1;
  if (H->size > 0) {
    H->h[0] = last;
    H->pos[last] = 0;
    sift_down(H, 0);
  }
  return top;
}

/* ---- FMM: classic_solvers.cpp:28-92 ------------------------------------ */

int orc_fmm(const orc_problem* p, double* v, orc_stats* st) {
  const int64_t m = p->m, n = p->n, M = m * n;
  memset(st, 0, sizeof *st);
  char* label = (char*)calloc((size_t)M, 1); /* 0 Far, 1 Considered, 2 Accepted */
  char* is_exit = (char*)malloc((size_t)M);
  heap H;
  if (!label || !is_exit || heap_init(&H, M)) { free(label); free(is_exit); return 1; }
  init_values(p, v, is_exit);
  for (int64_t k = 0; k < p->n_exit; ++k) label[p->exit_nodes[k]] = 2;
  static const int di[4] = {1, -1, 0, 0}, dj[4] = {0, 0, 1, -1};
  double nb[4];
  for (int64_t k = 0; k < p->n_exit; ++k) {
    int64_t idx = p->exit_nodes[k], i = idx % m, j = idx / m;
    for (int d = 0; d < 4; ++d) {
      int64_t ni = i + di[d], nj = j + dj[d];
      if (ni < 0 || ni >= m || nj < 0 || nj >= n) continue;
      int64_t nidx = nj * m + ni;
      if (label[nidx] != 0) continue;
      label[nidx] = 1;
      ++st->node_updates;
      gather(v, m, n, ni, nj, nb);
      double cand = orc_node_update(nb, p->F[nidx], p->h);
      if (cand < v[nidx]) v[nidx] = cand;
      heap_insert(&H, nidx, v[nidx]);
    }
  }
  while (H.size > 0) {
    int64_t idx = heap_pop(&H);
    ++st->heap_removals;
    label[idx] = 2;
    int64_t i = idx % m, j = idx / m;
    for (int d = 0; d < 4; ++d) {
      int64_t ni = i + di[d], nj = j + dj[d];
      if (ni < 0 || ni >= m || nj < 0 || nj >= n) continue;
      int64_t nidx = nj * m + ni;
      if (label[nidx] == 2 || is_exit[nidx]) continue;
      ++st->node_updates;
      gather(v, m, n, ni, nj, nb);
      double cand = orc_node_update(nb, p->F[nidx], p->h);
      if (label[nidx] == 0) {
        label[nidx] = 1;
        if (cand < v[nidx]) v[nidx] = cand;
        heap_insert(&H, nidx, v[nidx]);
      } else if (cand < v[nidx]) {
        v[nidx] = cand;
        heap_decrease(&H, nidx, cand);
      }
    }
  }
  heap_free(&H);
  free(label);
  free(is_exit);
  return 0;
}

/* ---- FSM: classic_solvers.cpp:94-158 ----------------------------------- */

typedef struct axis { int64_t begin, end, step; } axis;
static axis i_order(int d, int64_t lo, int64_t hi) { /* classic_solvers.cpp:116-119 */
  axis a = {lo, hi, 1}, b = {hi - 1, lo - 1, -1};
  return (d == SW || d == NW) ? a : b;
}
static axis j_order(int d, int64_t lo, int64_t hi) { /* classic_solvers.cpp:121-124 */
  axis a = {lo, hi, 1}, b = {hi - 1, lo - 1, -1};
  return (d == SW || d == SE) ? a : b;
}

int orc_fsm(const orc_problem* p, double* v, orc_stats* st) {
  const int64_t m = p->m, n = p->n;
  memset(st, 0, sizeof *st);
  char* is_exit = (char*)malloc((size_t)(m * n));
  if (!is_exit) return 1;
  init_values(p, v, is_exit);
  int64_t sweep = 0;
  int changed = 1;
  double nb[4];
  while (changed) {
    changed = 0;
    int dir = (int)(sweep % 4);
    axis io = i_order(dir, 0, m), jo = j_order(dir, 0, n);
    for (int64_t i = io.begin; i != io.end; i += io.step)
      for (int64_t j = jo.begin; j != jo.end; j += jo.step) {
        int64_t idx = j * m + i;
        if (is_exit[idx]) continue;
        ++st->node_updates;
        gather(v, m, n, i, j, nb);
        double cand = orc_node_update(nb, p->F[idx], p->h);
        if (cand < v[idx]) {
          v[idx] = cand;
          changed = 1;
        }
      }
    ++sweep;
  }
  st->sweeps = sweep;
  free(is_exit);
  return 0;
}

/* One sweep of the loop body above (classic_solvers.cpp:140-155) in direction
 * dir over v; nodes with frozen[idx] != 0 are skipped (exits, and the ghost
 * rows of a strip in the strip-Jacobi emulation).  Returns 1 if a value
 * decreased. */
int orc_fsm_sweep(int64_t m, int64_t n, double h, const double* F, const char* frozen, double* v,
                  int dir) {
  int changed = 0;
  double nb[4];
  axis io = i_order(dir & 3, 0, m), jo = j_order(dir & 3, 0, n);
  for (int64_t i = io.begin; i != io.end; i += io.step)
    for (int64_t j = jo.begin; j != jo.end; j += jo.step) {
      int64_t idx = j * m + i;
      if (frozen[idx]) continue;
      gather(v, m, n, i, j, nb);
      double cand = orc_node_update(nb, F[idx], h);
      if (cand < v[idx]) {
        v[idx] = cand;
        changed = 1;
      }
    }
  return changed;
}

/* ---- LSM: classic_solvers.cpp:160-212 ---------------------------------- */

int orc_lsm(const orc_problem* p, double* v, orc_stats* st) {
  const int64_t m = p->m, n = p->n, M = m * n;
  memset(st, 0, sizeof *st);
  char* is_exit = (char*)malloc((size_t)M);
  char* unlocked = (char*)calloc((size_t)M, 1);
  if (!is_exit || !unlocked) { free(is_exit); free(unlocked); return 1; }
  init_values(p, v, is_exit);
  static const int di[4] = {1, -1, 0, 0}, dj[4] = {0, 0, 1, -1};
  for (int64_t k = 0; k < p->n_exit; ++k) {
    int64_t idx = p->exit_nodes[k], i = idx % m, j = idx / m;
    for (int d = 0; d < 4; ++d) {
      int64_t ni = i + di[d], nj = j + dj[d];
      if (ni < 0 || ni >= m || nj < 0 || nj >= n) continue;
      if (!is_exit[nj * m + ni]) unlocked[nj * m + ni] = 1;
    }
  }
  int64_t sweep = 0;
  int changed = 1;
  double nb[4];
  while (changed) {
    changed = 0;
    int dir = (int)(sweep % 4);
    axis io = i_order(dir, 0, m), jo = j_order(dir, 0, n);
    for (int64_t i = io.begin; i != io.end; i += io.step)
      for (int64_t j = jo.begin; j != jo.end; j += jo.step) {
        int64_t idx = j * m + i;
        if (!unlocked[idx]) continue;
        unlocked[idx] = 0;
        ++st->node_updates;
        gather(v, m, n, i, j, nb);
        double cand = orc_node_update(nb, p->F[idx], p->h);
        if (cand < v[idx]) {
          v[idx] = cand;
          changed = 1;
          for (int d = 0; d < 4; ++d) {
            int64_t ni = i + di[d], nj = j + dj[d];
            if (ni < 0 || ni >= m || nj < 0 || nj >= n) continue;
            int64_t nidx = nj * m + ni;
            if (!is_exit[nidx] && v[nidx] > cand) unlocked[nidx] = 1;
          }
        }
      }
    ++sweep;
  }
  st->sweeps = sweep;
  free(is_exit);
  free(unlocked);
  return 0;
}

/* ---- cell decomposition: cells.cpp:7-47, cells.hpp:27-121 --------------- */

typedef struct cellgeo {
  int64_t cx, cy;
  int64_t *ib, *ie, *jb, *je;
  double hc_x, hc_y;
} cellgeo;

static void split_axis(int64_t nodes, int64_t cells, int64_t* b, int64_t* e) {
  const int64_t base = nodes / cells;
  int64_t at = 0;
  for (int64_t c = 0; c < cells; ++c) {
    b[c] = at;
    at += base;
    if (c == cells - 1) at = nodes;
    e[c] = at;
  }
}

static int geo_init(cellgeo* G, const orc_problem* p, const orc_cells* c) {
  if (c->cells_x < 1 || c->cells_y < 1 || c->cells_x > p->m || c->cells_y > p->n) return 1;
  G->cx = c->cells_x;
  G->cy = c->cells_y;
  G->ib = (int64_t*)malloc(sizeof(int64_t) * (size_t)G->cx);
  G->ie = (int64_t*)malloc(sizeof(int64_t) * (size_t)G->cx);
  G->jb = (int64_t*)malloc(sizeof(int64_t) * (size_t)G->cy);
  G->je = (int64_t*)malloc(sizeof(int64_t) * (size_t)G->cy);
  split_axis(p->m, G->cx, G->ib, G->ie);
  split_axis(p->n, G->cy, G->jb, G->je);
  G->hc_x = (double)(p->m / G->cx) * p->h;
  G->hc_y = (double)(p->n / G->cy) * p->h;
  return 0;
}
static void geo_free(cellgeo* G) { free(G->ib); free(G->ie); free(G->jb); free(G->je); }

static int64_t neighbor(const cellgeo* G, int64_t cell, int side) { /* cells.hpp:51-61 */
  int64_t cx = cell % G->cx, cy = cell / G->cx;
  switch (side) {
    case WEST: return cx > 0 ? cell - 1 : -1;
    case EAST: return cx + 1 < G->cx ? cell + 1 : -1;
    case SOUTH: return cy > 0 ? cell - G->cx : -1;
    default: return cy + 1 < G->cy ? cell + G->cx : -1;
  }
}

static int64_t cell_of_node(const cellgeo* G, int64_t i, int64_t j) { /* cells.cpp:23-30 */
  int64_t a = 0, b = 0;
  while (G->ie[a] <= i) ++a;
  while (G->je[b] <= j) ++b;
  return b * G->cx + a;
}

typedef struct rect { int64_t ib, ie, jb, je; } rect;
static rect cell_rect(const cellgeo* G, int64_t cell) {
  rect r = {G->ib[cell % G->cx], G->ie[cell % G->cx], G->jb[cell / G->cx], G->je[cell / G->cx]};
  return r;
}

/* ---- heap-cell methods: heap_cell.cpp ------------------------------------ */

static const int kFlagOrder[4] = {NE, NW, SE, SW}; /* heap_cell.cpp:13-14 */
static const int kRotation[4] = {SW, NW, NE, SE};   /* heap_cell.cpp:15-16 */

typedef struct strip { int64_t i0, j0, di, dj, len, adi, adj; } strip;
static strip strip_for(const cellgeo* G, int64_t cell, int side) { /* heap_cell.cpp:29-40 */
  rect r = cell_rect(G, cell);
  strip s;
  switch (side) {
    case WEST: s = (strip){r.ib, r.jb, 0, 1, r.je - r.jb, -1, 0}; break;
    case EAST: s = (strip){r.ie - 1, r.jb, 0, 1, r.je - r.jb, 1, 0}; break;
    case SOUTH: s = (strip){r.ib, r.jb, 1, 0, r.ie - r.ib, 0, -1}; break;
    default: s = (strip){r.ib, r.je - 1, 1, 0, r.ie - r.ib, 0, 1}; break;
  }
  return s;
}

typedef struct hcrun {
  const orc_problem* p;
  const orc_cells* c;
  cellgeo G;
  double* v;
  char* is_exit;
  char* unlocked;
  orc_stats* st;
} hcrun;

static void reset_locks(hcrun* R, int64_t cell) { /* heap_cell.cpp:65-94 */
  const int64_t m = R->p->m, n = R->p->n;
  rect r = cell_rect(&R->G, cell);
  for (int64_t j = r.jb; j < r.je; ++j)
    for (int64_t i = r.ib; i < r.ie; ++i) R->unlocked[j * m + i] = 0;
#define UNLOCK(ii, jj)                                    \
  do {                                                    \
    int64_t idx_ = (jj) * m + (ii);                       \
    if (!R->is_exit[idx_]) R->unlocked[idx_] = 1;         \
  } while (0)
  if (r.ib > 0)
    for (int64_t j = r.jb; j < r.je; ++j) UNLOCK(r.ib, j);
  if (r.ie < m)
    for (int64_t j = r.jb; j < r.je; ++j) UNLOCK(r.ie - 1, j);
  if (r.jb > 0)
    for (int64_t i = r.ib; i < r.ie; ++i) UNLOCK(i, r.jb);
  if (r.je < n)
    for (int64_t i = r.ib; i < r.ie; ++i) UNLOCK(i, r.je - 1);
  static const int di[4] = {1, -1, 0, 0}, dj[4] = {0, 0, 1, -1};
  for (int64_t j = r.jb; j < r.je; ++j)
    for (int64_t i = r.ib; i < r.ie; ++i) {
      if (!R->is_exit[j * m + i]) continue;
      for (int d = 0; d < 4; ++d) {
        int64_t ni = i + di[d], nj = j + dj[d];
        if (ni >= r.ib && ni < r.ie && nj >= r.jb && nj < r.je) UNLOCK(ni, nj);
      }
    }
#undef UNLOCK
}

static int locked_sweep(hcrun* R, int64_t cell, int dir) { /* heap_cell.cpp:98-126 */
  const int64_t m = R->p->m, n = R->p->n;
  rect r = cell_rect(&R->G, cell);
  axis io = i_order(dir, r.ib, r.ie), jo = j_order(dir, r.jb, r.je);
  static const int di[4] = {1, -1, 0, 0}, dj[4] = {0, 0, 1, -1};
  int changed = 0;
  double nb[4];
  for (int64_t i = io.begin; i != io.end; i += io.step)
    for (int64_t j = jo.begin; j != jo.end; j += jo.step) {
      int64_t idx = j * m + i;
      if (!R->unlocked[idx]) continue;
      R->unlocked[idx] = 0;
      ++R->st->node_updates;
      gather(R->v, m, n, i, j, nb);
      double cand = orc_node_update(nb, R->p->F[idx], R->p->h);
      if (cand < R->v[idx]) {
        R->v[idx] = cand;
        changed = 1;
        for (int d = 0; d < 4; ++d) {
          int64_t ni = i + di[d], nj = j + dj[d];
          if (!(ni >= r.ib && ni < r.ie && nj >= r.jb && nj < r.je)) continue;
          int64_t nidx = nj * m + ni;
          if (!R->is_exit[nidx] && R->v[nidx] > cand) R->unlocked[nidx] = 1;
        }
      }
    }
  return changed;
}

static int64_t process_to_convergence(hcrun* R, int64_t cell, unsigned flags) { /* :130-147 */
  int perm[4], at = 0;
  for (int k = 0; k < 4; ++k)
    if (flags & (1u << kFlagOrder[k])) perm[at++] = kFlagOrder[k];
  for (int k = 0; k < 4; ++k)
    if (!(flags & (1u << kRotation[k]))) perm[at++] = kRotation[k];
  reset_locks(R, cell);
  int64_t sweeps = 0;
  int changed = 1;
  while (changed) {
    int dir = sweeps < 4 ? perm[sweeps] : kRotation[sweeps % 4];
    changed = locked_sweep(R, cell, dir);
    ++sweeps;
  }
  return sweeps;
}

static int64_t process_flagged_once(hcrun* R, int64_t cell, unsigned flags) { /* :150-160 */
  reset_locks(R, cell);
  int64_t sweeps = 0;
  for (int k = 0; k < 4; ++k) {
    if (!(flags & (1u << kFlagOrder[k]))) continue;
    locked_sweep(R, cell, kFlagOrder[k]);
    ++sweeps;
  }
  return sweeps;
}

/* monotonicity_sides (cells.cpp:49-60): {dir when non-decreasing, when non-increasing} */
static void mono_sides(int from_side, int out[2]) {
  switch (from_side) {
    case WEST: out[0] = NW; out[1] = SW; break;
    case EAST: out[0] = NE; out[1] = SE; break;
    case SOUTH: out[0] = SW; out[1] = SE; break;
    default: out[0] = NW; out[1] = NE; break;
  }
}
static int opposite(int s) { return s ^ 1; } /* W<->E, S<->N */

typedef struct scanres {
  int should_add;
  unsigned flags;
  double cand;
  int mon_checked, mon_single;
} scanres;

/* scan_cell_boundary (heap_cell.cpp:173-239) */
static scanres scan_border(hcrun* R, int64_t cell, int side, const double* before,
                           int first_removal, int use_mono) {
  scanres res = {0, 0u, INF, 0, 0};
  const orc_problem* p = R->p;
  const int64_t m = p->m;
  strip s = strip_for(&R->G, cell, side);
  double vmax = -INF;
  int64_t argmax = 0;
  for (int64_t t = 0; t < s.len; ++t) {
    int64_t i = s.i0 + t * s.di, j = s.j0 + t * s.dj;
    int64_t idx = j * m + i;
    double vi = R->v[idx];
    if (vi > vmax) {
      vmax = vi;
      argmax = t;
    }
    int64_t aidx = (j + s.adj) * m + (i + s.adi);
    int vi_changed = vi < before[t];
    if (!R->is_exit[aidx] && vi < R->v[aidx] && (vi_changed || (first_removal && R->is_exit[idx])))
      res.should_add = 1;
  }
  if (isfinite(vmax)) {
    const int vertical = (side == WEST || side == EAST);
    const double hc = vertical ? R->G.hc_x : R->G.hc_y;
    int64_t i = s.i0 + argmax * s.di, j = s.j0 + argmax * s.dj;
    /* F at the clamped probe point, pre-sampled by the caller */
    int64_t col = vertical ? cell % R->G.cx : cell / R->G.cx;
    double fprobe;
    switch (side) {
      case WEST: fprobe = R->c->probe_w[col * p->n + j]; break;
      case EAST: fprobe = R->c->probe_e[col * p->n + j]; break;
      case SOUTH: fprobe = R->c->probe_s[col * p->m + i]; break;
      default: fprobe = R->c->probe_n[col * p->m + i]; break;
    }
    /* cell_value_candidate (cells.hpp:109-112) */
    res.cand = vmax + 0.5 * (p->h + hc) / fprobe;
  }
  if (res.should_add) {
    int both[2];
    mono_sides(opposite(side), both);
    if (use_mono) {
      const int vertical = (side == WEST || side == EAST);
      int nondec = 1, noninc = 1;
      double prev = 0.0;
      for (int64_t t = 0; t < s.len; ++t) {
        int64_t u = vertical ? s.len - 1 - t : t;
        double x = R->v[(s.j0 + u * s.dj) * m + (s.i0 + u * s.di)];
        if (t > 0) {
          if (x < prev) nondec = 0;
          if (x > prev) noninc = 0;
        }
        prev = x;
      }
      if (nondec && !noninc) res.flags = 1u << both[0];
      else if (noninc && !nondec) res.flags = 1u << both[1];
      else res.flags = (1u << both[0]) | (1u << both[1]);
      res.mon_checked = 1;
      res.mon_single = (nondec != noninc);
    } else {
      res.flags = (1u << both[0]) | (1u << both[1]);
    }
  }
  return res;
}

/* heap_cell_solve (heap_cell.cpp:243-324) */
static int heap_cell_solve(const orc_problem* p, const orc_cells* c, double* v, orc_stats* st,
                           int fast) {
  memset(st, 0, sizeof *st);
  hcrun R;
  R.p = p;
  R.c = c;
  R.v = v;
  R.st = st;
  if (geo_init(&R.G, p, c)) return 1;
  const int64_t M = p->m * p->n, J = R.G.cx * R.G.cy;
  R.is_exit = (char*)malloc((size_t)M);
  R.unlocked = (char*)calloc((size_t)M, 1);
  double* cell_value = (double*)malloc(sizeof(double) * (size_t)J);
  unsigned* flags = (unsigned*)calloc((size_t)J, sizeof(unsigned));
  char* first_done = (char*)calloc((size_t)J, 1);
  int64_t maxlen = (p->m > p->n ? p->m : p->n);
  double* before[4];
  for (int d = 0; d < 4; ++d) before[d] = (double*)malloc(sizeof(double) * (size_t)maxlen);
  heap H;
  heap_init(&H, J);
  init_values(p, v, R.is_exit);
  for (int64_t k = 0; k < J; ++k) cell_value[k] = INF;
  for (int64_t k = 0; k < p->n_exit; ++k) {
    int64_t idx = p->exit_nodes[k];
    int64_t cell = cell_of_node(&R.G, idx % p->m, idx / p->m);
    double q = p->exit_cost[k];
    cell_value[cell] = isfinite(cell_value[cell]) ? dmax(cell_value[cell], q) : q;
  }
  for (int64_t cell = 0; cell < J; ++cell) {
    if (!isfinite(cell_value[cell])) continue;
    heap_insert(&H, cell, cell_value[cell]);
    if (fast) flags[cell] = 0xF;
  }
  const int64_t budget = 100 * J + 16;
  int rc = 0;
  while (H.size > 0) {
    const int64_t cell = heap_pop(&H);
    ++st->heap_removals;
    if (st->heap_removals > budget) { rc = 3; break; }
    for (int d = 0; d < 4; ++d)
      if (neighbor(&R.G, cell, d) >= 0) {
        strip s = strip_for(&R.G, cell, d);
        for (int64_t t = 0; t < s.len; ++t)
          before[d][t] = v[(s.j0 + t * s.dj) * p->m + (s.i0 + t * s.di)];
      }
    const unsigned my_flags = flags[cell];
    flags[cell] = 0;
    st->sweeps += fast ? process_flagged_once(&R, cell, my_flags)
                       : process_to_convergence(&R, cell, my_flags);
    const int first_removal = !first_done[cell];
    first_done[cell] = 1;
    for (int d = 0; d < 4; ++d) {
      const int64_t nb = neighbor(&R.G, cell, d);
      if (nb < 0) continue;
      scanres sc = scan_border(&R, cell, d, before[d], first_removal, fast);
      if (sc.cand < cell_value[nb]) {
        cell_value[nb] = sc.cand;
        if (heap_contains(&H, nb)) heap_decrease(&H, nb, cell_value[nb]);
      }
      if (sc.should_add) {
        flags[nb] |= sc.flags;
        if (sc.mon_checked) {
          ++st->mon_checks;
          if (sc.mon_single) ++st->mon_single;
        }
        if (!heap_contains(&H, nb)) heap_insert(&H, nb, cell_value[nb]);
      }
    }
  }
  heap_free(&H);
  for (int d = 0; d < 4; ++d) free(before[d]);
  free(cell_value);
  free(flags);
  free(first_done);
  free(R.is_exit);
  free(R.unlocked);
  geo_free(&R.G);
  return rc;
}

int orc_hcm(const orc_problem* p, const orc_cells* c, double* v, orc_stats* st) {
  return heap_cell_solve(p, c, v, st, 0);
}
int orc_fhcm(const orc_problem* p, const orc_cells* c, double* v, orc_stats* st) {
  return heap_cell_solve(p, c, v, st, 1);
}

/* ---- FMSM: fmsm.cpp ------------------------------------------------------ */

/* fmsm_sweep_directions (fmsm.cpp:83-120): returns count, dirs in NE,NW,SE,SW order */
static int fmsm_dirs(int w, int e, int s, int nn, int out[4]) {
  int xs[2], nx = 0, ys[2], ny = 0;
  if (w && !e) xs[nx++] = 0;
  else if (e && !w) xs[nx++] = 1;
  else { xs[nx++] = 0; xs[nx++] = 1; }
  if (s && !nn) ys[ny++] = 0;
  else if (nn && !s) ys[ny++] = 1;
  else { ys[ny++] = 0; ys[ny++] = 1; }
  int present[4] = {0, 0, 0, 0};
  for (int a = 0; a < ny; ++a)
    for (int b = 0; b < nx; ++b) {
      int yn = ys[a], xe = xs[b];
      int d = (yn && xe) ? NE : (yn && !xe) ? NW : (!yn && xe) ? SE : SW;
      present[d] = 1;
    }
  int cnt = 0;
  static const int rank_order[4] = {NE, NW, SE, SW};
  for (int k = 0; k < 4; ++k)
    if (present[rank_order[k]]) out[cnt++] = rank_order[k];
  return cnt;
}

typedef struct keyed { int64_t key; int64_t id; } keyed;
static int keyed_cmp(const void* a, const void* b) {
  const keyed* x = (const keyed*)a;
  const keyed* y = (const keyed*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->id < y->id ? -1 : (x->id > y->id);
}

int orc_fmsm(const orc_problem* p, const orc_cells* c, double* v, orc_stats* st) {
  return orc_fmsm_ex(p, c, v, st, NULL);
}

/* orc_fmsm with the quantised cell order (fmsm.cpp:138-160) copied to
 * order_out (J entries) when non-NULL; v == NULL stops after Part I. */
int orc_fmsm_ex(const orc_problem* p, const orc_cells* c, double* v, orc_stats* st,
                int64_t* order_out) {
  memset(st, 0, sizeof *st);
  if (c->cells_x < 2 || c->cells_y < 2) return 1; /* fmsm.cpp:124-125 */
  cellgeo G;
  if (geo_init(&G, p, c)) return 1;
  const int64_t m = p->m, n = p->n, J = G.cx * G.cy;
  const double h = p->h;

  /* build_coarse_problem (fmsm.cpp:10-81).  centres: cells.hpp:44-48 */
  double* cxy = (double*)malloc(sizeof(double) * 2 * (size_t)J);
  for (int64_t cell = 0; cell < J; ++cell) {
    int64_t a = cell % G.cx, b = cell / G.cx;
    cxy[2 * cell] = 0.5 * ((p->x0 + (double)G.ib[a] * h) + (p->x0 + (double)(G.ie[a] - 1) * h));
    cxy[2 * cell + 1] = 0.5 * ((p->y0 + (double)G.jb[b] * h) + (p->y0 + (double)(G.je[b] - 1) * h));
  }
  double* best = (double*)malloc(sizeof(double) * (size_t)J);
  for (int64_t k = 0; k < J; ++k) best[k] = INF;
  if (p->n_exit_points > 0) {
    const int single = p->n_exit_points == 1;
    for (int64_t k = 0; k < p->n_exit_points; ++k) {
      double qx = p->exit_points_xy[2 * k], qy = p->exit_points_xy[2 * k + 1];
      double dm = INF;
      for (int64_t cell = 0; cell < J; ++cell)
        dm = dmin(dm, hypot(qx - cxy[2 * cell], qy - cxy[2 * cell + 1]));
      const double tie = 1e-12 * (h + dm);
      for (int64_t cell = 0; cell < J; ++cell) {
        double dist = hypot(qx - cxy[2 * cell], qy - cxy[2 * cell + 1]);
        if (dist > dm + tie) continue;
        double cost = single ? p->exit_point_cost[k]
                             : p->exit_point_cost[k] + dist / c->center_F[cell];
        best[cell] = dmin(best[cell], cost);
      }
    }
  } else {
    const int single = p->n_exit == 1;
    for (int64_t k = 0; k < p->n_exit; ++k) {
      int64_t idx = p->exit_nodes[k], i = idx % m, j = idx / m;
      int64_t cell = cell_of_node(&G, i, j);
      double dist = hypot((p->x0 + (double)i * h) - cxy[2 * cell], (p->y0 + (double)j * h) - cxy[2 * cell + 1]);
      double cost = single ? p->exit_cost[k] : p->exit_cost[k] + dist / c->center_F[cell];
      best[cell] = dmin(best[cell], cost);
    }
  }
  int64_t ncx = 0;
  for (int64_t k = 0; k < J; ++k) ncx += isfinite(best[k]) ? 1 : 0;
  int64_t* cex = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ncx > 0 ? ncx : 1));
  double* cec = (double*)malloc(sizeof(double) * (size_t)(ncx > 0 ? ncx : 1));
  char* cell_is_exit = (char*)calloc((size_t)J, 1);
  ncx = 0;
  for (int64_t k = 0; k < J; ++k)
    if (isfinite(best[k])) {
      cex[ncx] = k;
      cec[ncx] = best[k];
      cell_is_exit[k] = 1;
      ++ncx;
    }
  /* coarse grid: cells_x x cells_y, spacing hc_x, speed = F at actual centres */
  orc_problem cp = {G.cx, G.cy, G.hc_x, cxy[0], cxy[1], c->center_F, cex, cec, ncx, NULL, NULL, 0};
  double* cv = (double*)malloc(sizeof(double) * (size_t)J);
  orc_stats cst;
  int rc = 0;
  if (ncx == 0) rc = 1;
  else orc_fmm(&cp, cv, &cst);

  int64_t* rank = (int64_t*)malloc(sizeof(int64_t) * (size_t)J);
  keyed* order = (keyed*)malloc(sizeof(keyed) * (size_t)J);
  if (rc == 0) {
    /* quantised acceptance order (fmsm.cpp:138-160) */
    double vmax = G.hc_x;
    for (int64_t cell = 0; cell < J; ++cell)
      if (isfinite(cv[cell])) vmax = dmax(vmax, cv[cell]);
    const double quantum = 1e-9 * vmax;
    for (int64_t cell = 0; cell < J; ++cell) {
      order[cell].id = cell;
      order[cell].key = isfinite(cv[cell]) ? (int64_t)floor(cv[cell] / quantum) : INT64_MAX;
    }
    qsort(order, (size_t)J, sizeof(keyed), keyed_cmp);
    for (int64_t k = 0; k < J; ++k) rank[order[k].id] = k;
    if (order_out)
      for (int64_t k = 0; k < J; ++k) order_out[k] = order[k].id;
    st->heap_removals = cst.heap_removals;
    st->node_updates = cst.node_updates;
  }
  if (rc == 0 && v) {

    char* is_exit = (char*)malloc((size_t)(m * n));
    init_values(p, v, is_exit);
    st->heap_removals = cst.heap_removals;
    st->node_updates = cst.node_updates;
    double nb[4];
    for (int64_t pidx = 0; pidx < J; ++pidx) {
      const int64_t cell = order[pidx].id;
      rect r = cell_rect(&G, cell);
      int dirs[4], nd;
      int full = cell_is_exit[cell];
      if (!full) {
        int acc[4];
        for (int d = 0; d < 4; ++d) {
          int64_t nbc = neighbor(&G, cell, d);
          acc[d] = nbc >= 0 && rank[nbc] < pidx;
        }
        nd = fmsm_dirs(acc[0], acc[1], acc[2], acc[3], dirs);
      } else {
        nd = 0;
      }
      int64_t sweep = 0;
      int changed = 1;
      for (int k = 0; full ? changed : (k < nd); ++k) {
        int dir = full ? (int)(sweep % 4) : dirs[k];
        changed = 0;
        /* full_sweep lambda (fmsm.cpp:176-195) */
        axis io = i_order(dir, r.ib, r.ie), jo = j_order(dir, r.jb, r.je);
        for (int64_t i = io.begin; i != io.end; i += io.step)
          for (int64_t j = jo.begin; j != jo.end; j += jo.step) {
            int64_t idx = j * m + i;
            if (is_exit[idx]) continue;
            ++st->node_updates;
            gather(v, m, n, i, j, nb);
            double cand = full ? orc_node_update(nb, p->F[idx], h)
                               : orc_directional_update(nb, dir, p->F[idx], h);
            if (cand < v[idx]) {
              v[idx] = cand;
              changed = 1;
            }
          }
        ++sweep;
      }
      st->sweeps += full ? sweep : nd;
    }
    free(is_exit);
  }
  free(rank);
  free(order);
  free(cv);
  free(cex);
  free(cec);
  free(cell_is_exit);
  free(best);
  free(cxy);
  geo_free(&G);
  return rc;
}
