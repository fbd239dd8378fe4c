// Drop-in replacement for the reference's solver free functions
// (/root/reference/proj/include/eikonal/classic_solvers.hpp:18,33,38,
//  heap_cell.hpp:36,41, fmsm.hpp:36), implemented over the C-ABI of
// include/eikonal_b200.h.  This is the binding a maintainer of the reference
// adds: compile it against the reference's own headers and link it instead
// of classic_solvers.cpp / heap_cell.cpp / fmsm.cpp.  The speed function
// stays a host std::function: it is sampled here, exactly as
// Problem::speed_at does (grid.hpp:77-79), at every node, at the clamped
// border probe points (heap_cell.cpp:195-205) and at the cell centres
// (fmsm.cpp:18-30).  Status codes become the reference's exceptions.
//
// Every one of the six solvers runs on the device, including lsm_solve and
// fmm_solve's record_acceptance_order option.
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "eikonal/cells.hpp"
#include "eikonal/classic_solvers.hpp"
#include "eikonal/fmsm.hpp"
#include "eikonal/grid.hpp"
#include "eikonal/heap_cell.hpp"
#include "eikonal_b200.h"

namespace eikonal {

namespace {

[[noreturn]] void rethrow(int code) {
  const std::string msg = eik_last_error();
  switch (code) {
    case EIK_ERR_CONFIG: throw ConfigError(msg);
    case EIK_ERR_BUDGET: throw std::runtime_error(msg);
    case EIK_ERR_DOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error("eikonal_b200: " + msg);
  }
}

struct Sampled {
  eik_problem p{};
  std::vector<double> F;
  std::vector<int64_t> exits;
  std::vector<double> pts;
};

Sampled sample(const Problem& problem) {
  const Grid& g = problem.grid;
  Sampled s;
  s.F.resize((size_t)g.m * g.n);
  for (int j = 0; j < g.n; ++j)
    for (int i = 0; i < g.m; ++i) s.F[(size_t)j * g.m + i] = problem.speed_at(i, j);
  s.exits.assign(problem.exit_nodes.begin(), problem.exit_nodes.end());
  for (const Point& q : problem.exit_points) {
    s.pts.push_back(q.x);
    s.pts.push_back(q.y);
  }
  s.p.grid = {g.m, g.n, g.h, g.x0, g.y0};
  s.p.speed = s.F.data();
  s.p.exit_nodes = s.exits.data();
  s.p.exit_cost = problem.exit_cost.data();
  s.p.n_exit = (int64_t)s.exits.size();
  s.p.exit_points_xy = s.pts.empty() ? nullptr : s.pts.data();
  s.p.exit_point_cost = problem.exit_point_cost.empty() ? nullptr : problem.exit_point_cost.data();
  s.p.n_exit_points = (int64_t)problem.exit_point_cost.size();
  return s;
}

struct Tables {
  eik_cells c{};
  std::vector<double> probe[4], center;
};

Tables cell_tables(const Problem& problem, const CellDecomposition& cells) {
  Tables t;
  const eik_grid g{problem.grid.m, problem.grid.n, problem.grid.h, problem.grid.x0,
                   problem.grid.y0};
  for (int side = 0; side < 4; ++side) {
    const int64_t cnt = eik_cell_probe_points(&g, cells.cells_x, cells.cells_y, side, nullptr);
    if (cnt < 0) throw ConfigError("bad cell decomposition");
    std::vector<double> xy(2 * cnt);
    eik_cell_probe_points(&g, cells.cells_x, cells.cells_y, side, xy.data());
    t.probe[side].resize(cnt);
    for (int64_t k = 0; k < cnt; ++k) t.probe[side][k] = problem.speed(xy[2 * k], xy[2 * k + 1]);
  }
  t.center.resize(cells.cell_count());
  for (int c = 0; c < cells.cell_count(); ++c) {
    const Point q = cells.center(c);
    t.center[c] = problem.speed(q.x, q.y);
  }
  t.c.cells_x = cells.cells_x;
  t.c.cells_y = cells.cells_y;
  t.c.probe_speed_w = t.probe[0].data();
  t.c.probe_speed_e = t.probe[1].data();
  t.c.probe_speed_s = t.probe[2].data();
  t.c.probe_speed_n = t.probe[3].data();
  t.c.center_speed = t.center.data();
  return t;
}

SolverOutput run(const Problem& problem, const CellDecomposition* cells, int method,
                 bool acceptance_order = false) {
  Sampled s = sample(problem);
  Tables t;
  if (cells) t = cell_tables(problem, *cells);
  SolverOutput out;
  out.values = ValueField(problem.grid.m, problem.grid.n);
  eik_output o{};
  o.u = out.values.values.data();
  if (acceptance_order) {  // a resident plan: the order comes from its field
    eik_plan* plan = eik_plan_create(&s.p, nullptr, method);
    if (!plan) rethrow(eik_last_status());
    int rc = eik_plan_run(plan, &o);
    if (rc == EIK_OK) {
      out.acceptance_order.resize((size_t)(problem.grid.size() - s.p.n_exit));
      rc = eik_plan_acceptance_order(plan, out.acceptance_order.data(), 0);
    }
    eik_plan_destroy(plan);
    if (rc != EIK_OK) rethrow(rc);
  } else {
    const int rc = eik_solve(&s.p, cells ? &t.c : nullptr, method, &o);
    if (rc != EIK_OK) rethrow(rc);
  }
  out.sweeps = o.sweeps;
  out.node_updates = o.node_updates;
  out.heap_removals = o.heap_removals;
  out.hybrid.avhr = o.avhr;
  out.hybrid.avs = o.avs;
  out.hybrid.mon_pct = o.mon_pct;
  out.hybrid.cell_removals = o.cell_removals;
  out.hybrid.cell_sweeps = o.cell_sweeps;
  out.hybrid.mon_checks = o.mon_checks;
  out.hybrid.mon_single = o.mon_single;
  return out;
}

}  // namespace

SolverOutput fmm_solve(const Problem& problem, const FmmOptions& opts) {
  return run(problem, nullptr, EIK_FMM, opts.record_acceptance_order);
}
SolverOutput fsm_solve(const Problem& problem) { return run(problem, nullptr, EIK_FSM); }
SolverOutput lsm_solve(const Problem& problem) { return run(problem, nullptr, EIK_LSM); }
SolverOutput hcm_solve(const Problem& problem, const CellDecomposition& cells) {
  return run(problem, &cells, EIK_HCM);
}
SolverOutput fhcm_solve(const Problem& problem, const CellDecomposition& cells) {
  return run(problem, &cells, EIK_FHCM);
}
SolverOutput fmsm_solve(const Problem& problem, const CellDecomposition& cells) {
  if (cells.cells_x < 2 || cells.cells_y < 2)  // fmsm.cpp:124-125
    throw ConfigError("fmsm needs at least 2x2 cells");
  return run(problem, &cells, EIK_FMSM);
}

}  // namespace eikonal
