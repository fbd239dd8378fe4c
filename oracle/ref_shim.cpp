// ORACLE -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points around the UNMODIFIED reference library, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/.  The
// reference runs exactly as shipped: its own Problem, its own solvers, and
// an on-demand SpeedFn (grid.hpp:64,71) that evaluates our native field
// definitions (paper_1110_6220_b200/csrc/host_fields.c) -- the same
// function the product samples, so F bits agree.  Used (1) to pin the C
// restatement in oracle/eik_oracle.c, (2) as the "reference" CPU baseline in
// bench.py, (3) to generate golden fixtures.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "eikonal/cells.hpp"
#include "eikonal/experiment.hpp"
#include "eikonal/field_io.hpp"
#include "eikonal/classic_solvers.hpp"
#include "eikonal/fmsm.hpp"
#include "eikonal/grid.hpp"
#include "eikonal/heap_cell.hpp"
#include "eikonal/local_update.hpp"
#include "eikonal/metrics.hpp"
#include "eikonal/speed_fields.hpp"
#include "eikonal_b200.h"

namespace {
thread_local std::string g_err;
}

extern "C" {

struct ref_stats {
  int64_t sweeps, node_updates, heap_removals;
  int64_t cell_removals, cell_sweeps, mon_checks, mon_single;
  double avhr, avs, mon_pct;
  double elapsed_ms;  // steady_clock around the solver call (experiment.cpp:204-213)
};

const char* ref_last_error() { return g_err.c_str(); }

double ref_quadrant_update(double a, double b, double f, double h) {
  return eikonal::quadrant_update(a, b, f, h);
}
double ref_node_update(const double nb[4], double f, double h) {
  return eikonal::node_update({nb[0], nb[1], nb[2], nb[3]}, f, h);
}
double ref_directional_update(const double nb[4], int dir, double f, double h) {
  return eikonal::directional_update({nb[0], nb[1], nb[2], nb[3]},
                                     static_cast<eikonal::SweepDir>(dir), f, h);
}

// The reference's own named speed fields (speed_fields.cpp:94-110), used to
// pin our native restatement of them bit for bit.
double ref_named_speed(const char* name, double x, double y) {
  return eikonal::named_problem(name).speed(x, y);
}

// snap_point_to_node (grid.cpp:22-41); returns 0 or 5 on domain_error
int ref_snap(const eik_grid* g, double x, double y, int64_t* i, int64_t* j) {
  try {
    eikonal::Grid grid(static_cast<int>(g->m), static_cast<int>(g->n), g->h, g->x0, g->y0);
    eikonal::NodeIndex nd = eikonal::snap_point_to_node(grid, {x, y});
    *i = nd.i;
    *j = nd.j;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

// method numbering = eik_method.  cells_* ignored for exact methods.
// threads: unused (every reference solve is single-threaded).
int ref_solve(int method, const eik_grid* g, const eik_field* field,
              const int64_t* exit_nodes, const double* exit_cost, int64_t n_exit,
              const double* exit_points_xy, const double* exit_point_cost,
              int64_t n_points, int cells_x, int cells_y, double* u,
              ref_stats* st) {
  try {
    using namespace eikonal;
    Problem p;
    p.grid = Grid(static_cast<int>(g->m), static_cast<int>(g->n), g->h, g->x0, g->y0);
    eik_field fcopy = *field;
    p.speed = [fcopy](double x, double y) { return eik_field_eval(&fcopy, x, y); };
    for (int64_t k = 0; k < n_exit; ++k) {
      p.exit_nodes.push_back(static_cast<int>(exit_nodes[k]));
      p.exit_cost.push_back(exit_cost[k]);
    }
    for (int64_t k = 0; k < n_points; ++k) {
      p.exit_points.push_back({exit_points_xy[2 * k], exit_points_xy[2 * k + 1]});
      p.exit_point_cost.push_back(exit_point_cost[k]);
    }
    SolverOutput out;
    auto t0 = std::chrono::steady_clock::now();
    switch (method) {
      case 0: out = fmm_solve(p); break;
      case 1: out = fsm_solve(p); break;
      case 2: out = lsm_solve(p); break;
      case 3: out = hcm_solve(p, build_cells(p.grid, cells_x, cells_y)); break;
      case 4: out = fhcm_solve(p, build_cells(p.grid, cells_x, cells_y)); break;
      case 5: out = fmsm_solve(p, build_cells(p.grid, cells_x, cells_y)); break;
      default: g_err = "bad method"; return 1;
    }
    auto t1 = std::chrono::steady_clock::now();
    std::memcpy(u, out.values.values.data(), sizeof(double) * out.values.values.size());
    st->sweeps = out.sweeps;
    st->node_updates = out.node_updates;
    st->heap_removals = out.heap_removals;
    st->cell_removals = out.hybrid.cell_removals;
    st->cell_sweeps = out.hybrid.cell_sweeps;
    st->mon_checks = out.hybrid.mon_checks;
    st->mon_single = out.hybrid.mon_single;
    st->avhr = out.hybrid.avhr;
    st->avs = out.hybrid.avs;
    st->mon_pct = out.hybrid.mon_pct;
    st->elapsed_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    return 0;
  } catch (const eikonal::ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

// bench.py --impl reference: BASELINE config 2 (or any sinusoid field) built
// entirely by the reference -- its own SpeedSpec (speed_fields.cpp:27-29) and
// build_problem (grid.cpp:43-90) on Grid(m, m, 2/(m-1), -1, -1) with a point
// source at the origin -- and solved by its own solver.  Returns the solver
// call's steady_clock time in *ms (the scope of run_row, experiment.cpp:204-213)
// and the field's checksum (sum of finite values) in *sum.
int ref_bench_sinusoid(int method, int m, double amp, int freq, int cells, double* ms,
                       double* sum) {
  try {
    using namespace eikonal;
    Grid g(m, m, 2.0 / (m - 1), -1.0, -1.0);
    ExitSpec ex;
    ex.kind = ExitKind::Point;
    ex.point = {0.0, 0.0};
    Problem p = build_problem(g, speed_sinusoid(amp, freq).fn(), ex);
    SolverOutput out;
    auto t0 = std::chrono::steady_clock::now();
    switch (method) {
      case 0: out = fmm_solve(p); break;
      case 1: out = fsm_solve(p); break;
      case 2: out = lsm_solve(p); break;
      case 3: out = hcm_solve(p, build_cells(p.grid, cells, cells)); break;
      case 4: out = fhcm_solve(p, build_cells(p.grid, cells, cells)); break;
      case 5: out = fmsm_solve(p, build_cells(p.grid, cells, cells)); break;
      default: g_err = "bad method"; return 1;
    }
    auto t1 = std::chrono::steady_clock::now();
    *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    double acc = 0.0;
    for (double v : out.values.values)
      if (v < kInf) acc += v;
    *sum = acc;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

// Config 5 at full size (32769^2): the same reference solvers with an
// ARRAY-BACKED SpeedFn.  On a grid node
// (x == x0 + i*h and y == y0 + j*h exactly, Grid::x/y of grid.hpp:52-53) it
// returns F[j*m+i], which holds the bits eik_field_eval gives at that node
// (eik_field_sample is the same function, tabulated); off-grid points (the
// FHCM/HCM border probes, heap_cell.cpp:195-205, and FMSM cell centres,
// fmsm.cpp:18-30) are evaluated in closed form.  So the result is bit for bit
// what the on-demand SpeedFn would give, hours faster.
//
// The result stays in the reference's own SolverOutput (no 8.6 GB copy):
// ref_solve_array returns a handle, ref_result_values points at its field
// and ref_result_free releases it.
void* ref_solve_array(int method, const eik_grid* g, const eik_field* field,
                      const double* F, const int64_t* exit_nodes, const double* exit_cost,
                      int64_t n_exit, int cells_x, int cells_y, ref_stats* st) {
  try {
    using namespace eikonal;
    Problem p;
    p.grid = Grid(static_cast<int>(g->m), static_cast<int>(g->n), g->h, g->x0, g->y0);
    eik_field fcopy = *field;
    const int64_t m = g->m, n = g->n;
    const double x0 = g->x0, y0 = g->y0, h = g->h;
    p.speed = [fcopy, F, m, n, x0, y0, h](double x, double y) {
      const long long i = std::llround((x - x0) / h), j = std::llround((y - y0) / h);
      if (i >= 0 && i < m && j >= 0 && j < n && x0 + static_cast<int>(i) * h == x &&
          y0 + static_cast<int>(j) * h == y)
        return F[j * m + i];
      return eik_field_eval(&fcopy, x, y);
    };
    for (int64_t k = 0; k < n_exit; ++k) {
      p.exit_nodes.push_back(static_cast<int>(exit_nodes[k]));
      p.exit_cost.push_back(exit_cost[k]);
    }
    auto* out = new SolverOutput;
    auto t0 = std::chrono::steady_clock::now();
    switch (method) {
      case 0: *out = fmm_solve(p); break;
      case 1: *out = fsm_solve(p); break;
      case 2: *out = lsm_solve(p); break;
      case 3: *out = hcm_solve(p, build_cells(p.grid, cells_x, cells_y)); break;
      case 4: *out = fhcm_solve(p, build_cells(p.grid, cells_x, cells_y)); break;
      case 5: *out = fmsm_solve(p, build_cells(p.grid, cells_x, cells_y)); break;
      default: delete out; g_err = "bad method"; return nullptr;
    }
    auto t1 = std::chrono::steady_clock::now();
    st->sweeps = out->sweeps;
    st->node_updates = out->node_updates;
    st->heap_removals = out->heap_removals;
    st->cell_removals = out->hybrid.cell_removals;
    st->cell_sweeps = out->hybrid.cell_sweeps;
    st->mon_checks = out->hybrid.mon_checks;
    st->mon_single = out->hybrid.mon_single;
    st->avhr = out->hybrid.avhr;
    st->avs = out->hybrid.avs;
    st->mon_pct = out->hybrid.mon_pct;
    st->elapsed_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    return out;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

const double* ref_result_values(void* r) {
  return static_cast<eikonal::SolverOutput*>(r)->values.values.data();
}

void ref_result_free(void* r) { delete static_cast<eikonal::SolverOutput*>(r); }

// ground_truth (metrics.cpp:77-99) + method_metrics (metrics.cpp:70-75):
// fills l_inf, l_1, R, rho, R-ratio of `u_method` against FMM-on-refined
// truth; `u_exact` is the exact-solver field (FMM).  Returns 0 on success.
int ref_metrics(const eik_grid* g, const eik_field* field, const int64_t* exit_nodes,
                const double* exit_cost, int64_t n_exit, int refine,
                const double* u_method, const double* u_exact, double* out5) {  // out5[7]
  try {
    using namespace eikonal;
    Problem p;
    p.grid = Grid(static_cast<int>(g->m), static_cast<int>(g->n), g->h, g->x0, g->y0);
    eik_field fcopy = *field;
    p.speed = [fcopy](double x, double y) { return eik_field_eval(&fcopy, x, y); };
    for (int64_t k = 0; k < n_exit; ++k) {
      p.exit_nodes.push_back(static_cast<int>(exit_nodes[k]));
      p.exit_cost.push_back(exit_cost[k]);
    }
    ValueField truth = ground_truth(p, refine);
    ValueField vm(p.grid.m, p.grid.n), ve(p.grid.m, p.grid.n);
    std::memcpy(vm.values.data(), u_method, sizeof(double) * vm.values.size());
    std::memcpy(ve.values.data(), u_exact, sizeof(double) * ve.values.size());
    MetricsReport r = method_metrics(vm, ve, truth, p.exit_nodes);
    out5[0] = r.l_inf;
    out5[1] = r.l_1;
    out5[2] = r.max_error_ratio;
    out5[3] = r.avg_error_ratio;
    out5[4] = r.ratio_of_max;
    out5[5] = static_cast<double>(r.m_plus);
    out5[6] = r.x_plus_empty ? 1.0 : 0.0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

// The reference's own writers, for byte-level comparisons (field_io.cpp,
// experiment.cpp:314-329).
int ref_dump_field(const double* u, int m, int n, double h, const char* path, int ascii) {
  try {
    using namespace eikonal;
    ValueField v(m, n);
    std::memcpy(v.values.data(), u, sizeof(double) * (size_t)m * n);
    dump_field(v, h, path, ascii ? DumpFormat::Ascii : DumpFormat::Raw);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

int ref_csv_line(const char* problem, int method, int grid_m, int cells_x, const double* d9,
                 const long long* c3, char* out, int cap) {
  using namespace eikonal;
  ExperimentRow r;
  r.problem = problem;
  r.method = static_cast<Method>(method);
  r.grid_m = grid_m;
  r.cells_x = cells_x;
  r.elapsed_ms = d9[0];
  r.l_inf = d9[1];
  r.l_1 = d9[2];
  r.max_ratio = d9[3];
  r.rho = d9[4];
  r.ratio_of_max = d9[5];
  r.avhr = d9[6];
  r.avs = d9[7];
  r.mon_pct = d9[8];
  r.sweeps = c3[0];
  r.node_updates = c3[1];
  r.heap_removals = c3[2];
  std::string line = csv_line(r);
  std::snprintf(out, (size_t)cap, "%s", line.c_str());
  return (int)line.size();
}

const char* ref_csv_header() {
  static std::string h = eikonal::csv_header();
  return h.c_str();
}

}  // extern "C"
