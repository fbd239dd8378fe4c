/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Never linked into the product.
 *
 * Plain-C restatement of the reference's CPU algorithms for the hot path
 * (/root/reference/proj/src/{classic_solvers,heap_cell,fmsm,cells}.cpp and
 * include/eikonal/{local_update,indexed_min_heap,cells}.hpp).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker.  Parity is pinned against the reference itself
 * (oracle/_ref, built from /root/reference by oracle/Makefile) and against
 * the known-answer values of the reference's own tests (tests/golden/).
 *
 * Inputs are sampled arrays (the same ones the product receives through the
 * C-ABI, include/eikonal_b200.h), so the oracle never evaluates a speed
 * function itself.
 */
#ifndef EIK_ORACLE_H
#define EIK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_problem {
  int64_t m, n;
  double h, x0, y0;
  const double* F;            /* m*n speed at nodes */
  const int64_t* exit_nodes;  /* ascending */
  const double* exit_cost;
  int64_t n_exit;
  const double* exit_points_xy; /* pre-snap sources (FMSM), may be NULL */
  const double* exit_point_cost;
  int64_t n_exit_points;
} orc_problem;

typedef struct orc_cells {
  int32_t cells_x, cells_y;
  const double* probe_w; const double* probe_e; /* cells_x*n, cx*n+j */
  const double* probe_s; const double* probe_n; /* cells_y*m, cy*m+i */
  const double* center_F;                         /* cells_x*cells_y */
} orc_cells;

typedef struct orc_stats {
  int64_t sweeps, node_updates, heap_removals;
  int64_t mon_checks, mon_single;
} orc_stats;

/* local_update.hpp:30-64 */
double orc_quadrant_update(double ua, double ub, double f, double h);
/* nb = {east, west, north, south} */
double orc_node_update(const double nb[4], double f, double h);
double orc_directional_update(const double nb[4], int dir, double f, double h);

/* Solvers; u is caller-allocated m*n.  Return 0, or 1 on a bad argument
 * (ConfigError), 3 when the heap-cell removal budget is exceeded. */
int orc_fmm(const orc_problem* p, double* u, orc_stats* st);
int orc_fsm(const orc_problem* p, double* u, orc_stats* st);
/* one FSM sweep in direction dir; frozen nodes are not updated; 1 if changed */
int orc_fsm_sweep(int64_t m, int64_t n, double h, const double* F, const char* frozen, double* u,
                  int dir);
int orc_lsm(const orc_problem* p, double* u, orc_stats* st);
int orc_hcm(const orc_problem* p, const orc_cells* c, double* u, orc_stats* st);
int orc_fhcm(const orc_problem* p, const orc_cells* c, double* u, orc_stats* st);
int orc_fmsm(const orc_problem* p, const orc_cells* c, double* u, orc_stats* st);
/* orc_fmsm plus the quantised cell order (order_out: J ids, may be NULL);
 * u == NULL runs Part I only (stats: the coarse Fast March's counters). */
int orc_fmsm_ex(const orc_problem* p, const orc_cells* c, double* u, orc_stats* st,
                int64_t* order_out);

#ifdef __cplusplus
}
#endif

#endif
