/*
 * eikonal_b200.h -- C-ABI of the B200-native Eikonal hot path.
 *
 * Drop-in boundary for the reference's solver interface
 * (/root/reference/proj/include/eikonal/*.hpp).  Each entry point replaces one
 * reference function; the reference-side binding a maintainer adds is shown
 * in INTEGRATION.md.  Plain C: no exceptions, no torch types, plain pointers
 * and sizes.  Errors come back as status codes plus a thread-local message
 * (eik_last_error), mapping the reference's exception types:
 *   EIK_ERR_CONFIG  <- eikonal::ConfigError          (grid.hpp:16-19)
 *   EIK_ERR_BUDGET  <- std::runtime_error "heap-cell removal budget exceeded"
 *                                                     (heap_cell.cpp:276-277)
 *   EIK_ERR_DOMAIN  <- std::domain_error / invalid_argument (grid.cpp:32-35)
 *
 * Layout conventions (grid.hpp:36-58): node (i,j) sits at (x0+i*h, y0+j*h),
 * linear index j*m+i (row-major, rows are constant j).  Values are fp64;
 * +inf marks unreached nodes.  Indices are 64-bit on this side of the ABI.
 */
#ifndef EIKONAL_B200_H
#define EIKONAL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EIK_ABI_VERSION 4

/* Solver selection; numbering mirrors eikonal::Method (experiment.hpp:11). */
enum eik_method {
  EIK_FMM = 0,  /* fmm_solve   classic_solvers.hpp:18 */
  EIK_FSM = 1,  /* fsm_solve   classic_solvers.hpp:33 */
  EIK_LSM = 2,  /* lsm_solve   classic_solvers.hpp:38 */
  EIK_HCM = 3,  /* hcm_solve   heap_cell.hpp:36 */
  EIK_FHCM = 4, /* fhcm_solve  heap_cell.hpp:41 */
  EIK_FMSM = 5, /* fmsm_solve  fmsm.hpp:36 */
  /* hcm_solve by the exact replay of its heap order: bit-identical field and
   * counters (EIK_HCM's default is the band scheduler, eik_set_hcm_mode) */
  EIK_HCM_EXACT = 6
};

enum eik_status {
  EIK_OK = 0,
  EIK_ERR_CONFIG = 1,   /* bad problem / decomposition (ConfigError) */
  EIK_ERR_CUDA = 2,     /* CUDA runtime failure or no usable device */
  EIK_ERR_BUDGET = 3,   /* iteration / removal budget exceeded */
  EIK_ERR_NOT_IMPL = 4, /* method not implemented on the device path */
  EIK_ERR_DOMAIN = 5    /* argument outside the domain (domain_error) */
};

/* Grid (grid.hpp:36-58). */
typedef struct eik_grid {
  int64_t m, n; /* node counts in x and y, >= 2 */
  double h;     /* spacing > 0 */
  double x0, y0;
} eik_grid;

/* Problem (grid.hpp:69-80) with the speed function sampled on the host:
 * speed[j*m+i] == problem.speed(x0+i*h, y0+j*h) bit for bit
 * (Problem::speed_at, grid.hpp:77-79). */
typedef struct eik_problem {
  eik_grid grid;
  const double* speed;        /* F > 0 at every node, m*n */
  int32_t speed_on_device;    /* 1: `speed` is a device pointer (cuda:0) */
  const int64_t* exit_nodes;  /* strictly ascending linear indices */
  const double* exit_cost;    /* parallel to exit_nodes, finite */
  int64_t n_exit;             /* >= 1 */
  /* Pre-snap point-source positions and costs (grid.hpp:76-77), only read by
   * FMSM's coarse discretisation (fmsm.cpp:40-61).  May be empty. */
  const double* exit_points_xy; /* 2*n_exit_points, interleaved x,y */
  const double* exit_point_cost;
  int64_t n_exit_points;
} eik_problem;

/* Cell decomposition (cells.hpp:27-75, built exactly like build_cells,
 * cells.cpp:32-47) plus the host-sampled speed tables the two-scale methods
 * evaluate off-grid.  Build the tables with eik_cell_probe_points /
 * eik_cell_centers and the problem's own speed function. */
typedef struct eik_cells {
  int32_t cells_x, cells_y;
  /* HCM/FHCM: F at the clamped border probe point of every border node
   * (heap_cell.cpp:195-205).  west/east: cells_x*n entries, index cx*n+j;
   * south/north: cells_y*m entries, index cy*m+i. */
  const double* probe_speed_w;
  const double* probe_speed_e;
  const double* probe_speed_s;
  const double* probe_speed_n;
  /* FMSM: F at the geometric centre of every cell (cells.hpp:44-48,
   * fmsm.cpp:18-30), cells_x*cells_y entries. */
  const double* center_speed;
} eik_cells;

/* SolverOutput + HybridStats (grid.hpp:132-149). */
typedef struct eik_output {
  double* u;            /* caller-allocated m*n */
  int32_t u_on_device;  /* 1: `u` is a device pointer (cuda:0) */
  int64_t sweeps;
  int64_t node_updates;
  int64_t heap_removals;
  int64_t cell_removals, cell_sweeps, mon_checks, mon_single;
  double avhr, avs, mon_pct;
  double device_ms;     /* CUDA-event time of the device solve proper */
  double host_ms;       /* host part of the solve (FMSM Part I), else 0 */
  int64_t kernel_launches; /* kernels this call launched (evidence) */
  /* HCM/FHCM speculative replay: pops whose worker result was valid at
   * commit, pops that waited on a worker, pops processed by the committer */
  int64_t spec_hits, spec_waits, spec_self;
  int64_t grid_ctas;    /* CTAs of the persistent solve kernel this run launched */
  int64_t rounds;       /* HCM band scheduler: rounds (heap_removals = its pops) */
} eik_output;

/* One solve.  `cells` may be NULL for FMM/FSM.  Thread-safe: each call owns
 * its device buffers and stream. */
int eik_solve(const eik_problem* p, const eik_cells* cells, int32_t method,
              eik_output* out);

/* Several GPUs of this process (SURVEY.md 8(b) "n_gpus plus device list"):
 * fsm_solve (EIK_FSM) or the FMM row (EIK_FMM) with the grid's rows split
 * into n_devices strips, one per device, strip-Jacobi rounds with the strips'
 * edge rows exchanged by peer copies over NVLink after every sweep (no
 * communicator: one process drives every device).  The field is the discrete
 * fixed point fsm_solve converges to (<= 1e-10; bit-identical with
 * n_devices = 1, which is eik_solve); `sweeps` (= `rounds`) counts the
 * rounds.  Each device holds only its strip.  Host speed and u buffers. */
int eik_solve_multi(const eik_problem* p, int32_t method, const int32_t* devices,
                    int32_t n_devices, eik_output* out);

/* Resident plan: uploads the problem once and keeps device work buffers, so
 * repeated solves (benchmarks) time the device path alone.  The plan copies
 * every input; the caller's arrays may be freed after eik_plan_create. */
typedef struct eik_plan eik_plan;
eik_plan* eik_plan_create(const eik_problem* p, const eik_cells* cells,
                          int32_t method);
/* Solve into out->u (host or device per out->u_on_device; NULL u keeps the
 * result resident in the plan).  */
int eik_plan_run(eik_plan* plan, eik_output* out);
/* Device pointer to the plan's resident value field: node (i,j) is at
 * values[j*pitch + i] with pitch = eik_plan_pitch(plan) (the device layout is
 * row-padded for the sweep kernels). */
const double* eik_plan_values(const eik_plan* plan);
int64_t eik_plan_pitch(const eik_plan* plan);
void eik_plan_destroy(eik_plan* plan);

/* ---- several solves sharing one GPU ------------------------------------
 * The device-side counterpart of the reference's experiment runner, which
 * runs the rows of its method matrix on a pool of --jobs threads
 * (experiment.cpp:284-310): every solve's persistent kernel gets a slice of
 * the device and the solves run concurrently, one stream and one host
 * thread each.  Results, counters and errors per solve are exactly those of
 * eik_plan_run / eik_solve.
 *
 * eik_plan_set_ctas   cap the CTAs of a plan's persistent kernel (0 = the
 *                     whole device, the default).  FSM/FMM grids are fixed
 *                     (one warp per 32-row strip) and ignore the cap.
 * eik_plan_capacity   CTAs of the plan's persistent kernel the whole device
 *                     holds, and the fixed grid size (FSM/FMM) or 0.
 * eik_plan_run_batch  run n distinct plans of one device as a list
 *                     schedule: each plan's persistent kernel gets a slice of
 *                     whole SMs (heap-cell replays 2 J^(1/4)/sqrt(warps per
 *                     CTA), FSM/FMM their fixed grid, FMSM 16 CTAs, a capped
 *                     plan its cap) and starts as soon as the slice is free.
 *                     *batch_ms = device time from the call until the last
 *                     solve ended.  Returns the first failing plan's code
 *                     (eik_last_error names it).
 * eik_solve_batch     n eik_solve calls run the same way (uploads, solves
 *                     and downloads overlap); cells[k] may be NULL for
 *                     FMM/FSM and `cells` itself NULL when no solve needs one. */
int eik_plan_set_ctas(eik_plan* plan, int32_t max_ctas);
/* HCM ordering (north_star item 3).  mode 0 (default): the band scheduler --
 * every round processes all queued cells within the acceptance band
 * [kmin, kmin + (h+h_c)/(2 F_max)] that are local minima among their in-band
 * queued neighbours (never two adjacent cells), in one persistent launch;
 * the field is hcm_solve's fixed point within rounding (<= 1e-10, measured
 * ~1e-15), pops / sweeps / node updates are this order's.  mode 1: the exact
 * replay of hcm_solve's heap order -- bit-identical field and counters.
 * eik_set_hcm_mode sets the default for plans created afterwards
 * (EIK_HCM_EXACT=1 in the environment sets it to 1); eik_plan_set_hcm_mode
 * one plan's. */
int eik_set_hcm_mode(int32_t mode);
int eik_plan_set_hcm_mode(eik_plan* plan, int32_t mode);
/* eik_plan_set_partitions  strip-Jacobi on one device for an EIK_FSM/EIK_FMM
 *                     plan: parts of part_rows rows (a multiple of 32; 0 =
 *                     one exact Gauss-Seidel wavefront, the default) sweep
 *                     side by side and read each other's edge rows as they
 *                     were at the end of the previous sweep -- the rounds of
 *                     the multi-GPU strip decomposition (SURVEY.md 8(e)
 *                     option A) inside one launch.  Same discrete fixed
 *                     point; the sweep count is the rounds', not fsm_solve's. */
int eik_plan_set_partitions(eik_plan* plan, int32_t part_rows);
int eik_plan_capacity(eik_plan* plan, int32_t* device_ctas, int32_t* fixed_ctas);
int eik_plan_run_batch(eik_plan* const* plans, int32_t n, eik_output* outs, double* batch_ms);
int eik_solve_batch(const eik_problem* const* problems, const eik_cells* const* cells,
                    const int32_t* methods, int32_t n, eik_output* outs, double* batch_ms);

/* Sweep-level control of an EIK_FSM / EIK_FMM plan -- the building blocks of
 * strip-Jacobi FSM across GPUs (SURVEY.md section 8(e)
 * option A).  They replace no single reference function: a rank owns a row
 * strip of fsm_solve's grid (classic_solvers.cpp:128-158) plus one frozen
 * ghost row on each side, given as exit nodes whose values are overwritten
 * after every exchange.
 *   eik_plan_prepare  u <- +inf, exits <- their cost, C <- h/F (the start of
 *                     fsm_solve, classic_solvers.cpp:130-137).
 *   eik_plan_sweep    exactly `count` Gauss-Seidel sweeps on the current
 *                     values, local sweep k in direction (first_sweep+k) mod 4
 *                     (sweep_direction, classic_solvers.cpp:94-96);
 *                     changed[k] = 1 iff sweep k lowered some value.
 *   eik_plan_get_rows / eik_plan_set_rows  copy rows [row0, row0+nrows) of
 *                     the value field out of / into the plan (dense m-wide
 *                     rows; host or device buffer). */
/* FmmOptions::record_acceptance_order (classic_solvers.hpp:10-13,
 * classic_solvers.cpp:64-71): after an EIK_FMM plan has run, write the
 * order fmm_solve accepts the non-exit nodes in -- M - n_exit linear indices
 * by non-decreasing value (equal values in index order) -- into `order`
 * (host or device buffer). */
int eik_plan_acceptance_order(eik_plan* plan, int32_t* order, int32_t on_device);

int eik_plan_prepare(eik_plan* plan);
int eik_plan_sweep(eik_plan* plan, int64_t first_sweep, int32_t count, int32_t* changed);
int eik_plan_get_rows(eik_plan* plan, int64_t row0, int64_t nrows, double* dst, int32_t on_device);
int eik_plan_set_rows(eik_plan* plan, int64_t row0, int64_t nrows, const double* src,
                      int32_t on_device);
/* Stream-ordered variants for a rank that drives its rounds without host
 * synchronisation (distributed.py): the sweeps and row copies are enqueued on
 * `stream` (a cudaStream_t of the calling framework; NULL = the plan's own),
 * the per-sweep change flags land in device memory (changed_dev[count]).
 * eik_plan_get_rows reports a watchdog failure of an earlier async sweep. */
int eik_plan_sweep_async(eik_plan* plan, int64_t first_sweep, int32_t count, int32_t* changed_dev,
                         void* stream);
int eik_plan_rows_async(eik_plan* plan, int64_t row0, int64_t nrows, double* dev_buf,
                        int32_t to_plan, void* stream);

/* ---- FMSM sharded by row strips of cells ------------------
 * fmsm_solve (fmsm.cpp:126-226) over several GPUs, driven by
 * paper_1110_6220_b200/distributed.py fmsm_solve_strips.  Part I is computed
 * by every rank identically; Part II runs by LEVELS of the cell DAG (a cell's
 * earlier-ranked neighbours lie in earlier levels, so the cells of one level
 * are pairwise non-adjacent and independent), with the strips' edge rows
 * exchanged after the levels that changed them.  Exact: every cell reads the
 * same inputs as in the reference's rank-order pass.
 *
 * eik_fmsm_schedule: order/rank (fmsm.cpp:138-160), per-cell sweep flags (bit
 *   d = SweepDir d, 16 = Q-cell; fmsm.cpp:83-120,196-222), per-cell level;
 *   counters2 = coarse heap removals, coarse node updates.  Any output may be
 *   NULL.  Host only.
 * eik_plan_create_fmsm_strip: a plan over one strip's own problem (its rows
 *   plus a ghost row on each interior side, ghost nodes as exits) holding
 *   cells_y rows of cells_x cells, rows of height base_y from local node row
 *   row0, the last ending at row_end (exclusive).
 * eik_plan_fmsm_levels: the strip's cells grouped by level (local ids, level L
 *   = cells[level_off[L] .. level_off[L+1])), their flags; prepares u and C.
 * eik_plan_fmsm_level_async: sweep the cells of one level, enqueued on
 *   `stream` (NULL: the plan's stream).
 * eik_plan_fmsm_counters: sweeps and node updates so far (synchronises). */
int eik_fmsm_schedule(const eik_problem* p, const eik_cells* c, int32_t* order, int32_t* rank,
                      uint8_t* flags, int32_t* level, int64_t* counters2);
eik_plan* eik_plan_create_fmsm_strip(const eik_problem* local, int32_t cells_x, int32_t cells_y,
                                     int64_t base_y, int64_t row0, int64_t row_end);
int eik_plan_fmsm_levels(eik_plan* plan, const int32_t* cells, const int32_t* level_off,
                         int32_t nlevels, const uint8_t* flags);
int eik_plan_fmsm_level_async(eik_plan* plan, int32_t level, void* stream);
int eik_plan_fmsm_counters(eik_plan* plan, int64_t* out2);

/* Thread-local description / status code of the last failure on this
 * thread (eik_plan_create returns NULL and sets both). */
const char* eik_last_error(void);
int eik_last_status(void);
int eik_abi_version(void);
/* Re-read the EIK_* tuning/debug environment knobs (read once at load
 * otherwise; none of them changes a result).  Test hook. */
void eik_debug_reload_knobs(void);
/* Number of visible CUDA devices (0 on a CPU-only host; never fails). */
int eik_device_count(void);
/* Error metrics of a method's field against a ground truth
 * (metrics.cpp:11-69, error_fields + error_ratios): e = |u_exact - u_truth|,
 * E = |u_method - u_truth|, X+ = non-exit nodes with e > 1e-14.  Fields are
 * dense m*n (host or device per on_device); exit_nodes is a host array.  Maxima and counts match the
 * reference exactly; l_1 and avg_error_ratio are deterministic block-ordered
 * sums (within a few ulps of the reference's sequential sums). */
typedef struct eik_metrics_out {
  double l_inf, l_1, max_error_ratio, avg_error_ratio, ratio_of_max;
  int64_t m_plus;
  int32_t x_plus_empty;
} eik_metrics_out;
int eik_metrics(const double* u_method, const double* u_exact, const double* u_truth, int64_t m,
                int64_t n, const int64_t* exit_nodes, int64_t n_exit, int32_t on_device,
                eik_metrics_out* out);

/* Select the device later eik_solve / eik_plan_create calls on this thread
 * use (the library carries its own CUDA runtime, so a host framework's
 * device selection does not reach it).  One process per GPU calls this with
 * its local rank. */
int eik_set_device(int32_t device);
/* Free the device buffers the library keeps cached for reuse by later plans
 * (released plans return their buffers to a per-device cache). */
void eik_release_cached(void);

/* ---- host-side geometry helpers (bit-exact restatements) ------------- */

/* Clamped probe points of heap_cell.cpp:195-205 for every border node of
 * every cell column/row; side 0=W,1=E,2=S,3=N.  `xy` receives 2*count
 * doubles (x,y interleaved) where count = cells_x*n (W/E) or cells_y*m
 * (S/N).  Returns count, or -1 on bad arguments. */
int64_t eik_cell_probe_points(const eik_grid* g, int32_t cells_x,
                              int32_t cells_y, int32_t side, double* xy);
/* Cell centres (cells.hpp:44-48), 2*cells_x*cells_y doubles. */
int64_t eik_cell_centers(const eik_grid* g, int32_t cells_x, int32_t cells_y,
                         double* xy);

/* ---- native speed fields (BASELINE synthetic inputs) ------------------ */

enum eik_field_kind {
  EIK_FIELD_CONSTANT = 0,  /* F = value */
  EIK_FIELD_SINUSOID = 1,  /* 1 + amp*sin(freq*pi*x)*sin(freq*pi*y), speed_fields.cpp:27-29 */
  EIK_FIELD_CHECKER = 2,   /* k x k unit-square checkerboard, speed_fields.cpp:23-26 */
  EIK_FIELD_COMB = 3,      /* comb maze, speed_fields.cpp:30-41 */
  EIK_FIELD_BLOCKS = 4,    /* nb x nb piecewise-constant blocks (config 3) */
  EIK_FIELD_NODEMASK = 5,  /* nearest-node wall mask (config 4 maze) */
  EIK_FIELD_SINSUM = 6     /* 1 + 0.5*S/K, K random-phase sinusoids (config 5) */
};

typedef struct eik_field {
  int32_t kind;
  double value;                           /* CONSTANT */
  double amp; int32_t freq;               /* SINUSOID */
  int32_t checkers; double slow, fast;    /* CHECKER (slow on even index sum) */
  int32_t n_barriers;                     /* COMB */
  double barrier_speed, barrier_width, gap_fraction;
  int32_t nb; double bx0, by0, bscale;    /* BLOCKS: b = clamp(floor((x-bx0)*bscale),0,nb-1) */
  const double* block_speed;              /*   nb*nb, index by*nb+bx */
  eik_grid mask_grid;                     /* NODEMASK: lattice of the mask */
  const uint8_t* mask;                    /*   1 = wall (speed `slow`), else `fast` */
  int32_t K;                              /* SINSUM terms */
  const double* kp; const double* kq; const double* kphi;
} eik_field;

double eik_field_eval(const eik_field* f, double x, double y);
/* out[j*m+i] = eik_field_eval(f, x0+i*h, y0+j*h) bit for bit. */
int eik_field_sample(const eik_field* f, const eik_grid* g, double* out,
                     int32_t threads);
int eik_field_eval_points(const eik_field* f, const double* xy, int64_t count,
                          double* out);
/* Rows [row0, row0+nrows) of eik_field_sample's array (global coordinates:
 * bit-identical to the whole grid's sampling), for a rank's row strip. */
int eik_field_sample_rows(const eik_field* f, const eik_grid* g, int64_t row0, int64_t nrows,
                          double* out, int32_t threads);

#ifdef __cplusplus
}
#endif

#endif /* EIKONAL_B200_H */
