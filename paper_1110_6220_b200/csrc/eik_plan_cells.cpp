// Host runtime of the two-scale methods: cell geometry, FMSM Part I on the
// host (as in the reference), uploads, and the device dataflow launch.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <vector>

#include "eik_host.h"
#include "eik_plan.h"

namespace eikb200 {

namespace {

constexpr size_t kTileBudget = 96 * 1024;  // smem per CTA for warp tiles
constexpr size_t kTileMax = 200 * 1024;

int even_up(int x) { return (x + 1) & ~1; }

// fmsm_sweep_directions (fmsm.cpp:83-120) as a bit mask over SweepDir values.
uint8_t fmsm_dir_mask(bool w, bool e, bool s, bool n) {
  int xs[2], nx = 0, ys[2], ny = 0;
  if (w && !e) xs[nx++] = 0;
  else if (e && !w) xs[nx++] = 1;
  else { xs[nx++] = 0; xs[nx++] = 1; }
  if (s && !n) ys[ny++] = 0;
  else if (n && !s) ys[ny++] = 1;
  else { ys[ny++] = 0; ys[ny++] = 1; }
  uint8_t mask = 0;
  for (int a = 0; a < ny; ++a)
    for (int b = 0; b < nx; ++b) {
      const int yn = ys[a], xe = xs[b];
      const int d = (yn && xe) ? 2 /*NE*/ : (yn && !xe) ? 1 /*NW*/ : (!yn && xe) ? 3 /*SE*/ : 0;
      mask |= (uint8_t)(1u << d);
    }
  return mask;
}

}  // namespace

int plan_init_cells(eik_plan* P, const eik_problem* p, const eik_cells* c) {
  P->cells_x = c->cells_x;
  P->cells_y = c->cells_y;
  const int64_t J = (int64_t)c->cells_x * c->cells_y;
  P->exit_nodes.assign(p->exit_nodes, p->exit_nodes + p->n_exit);
  P->exit_cost.assign(p->exit_cost, p->exit_cost + p->n_exit);
  if (p->n_exit_points > 0) {
    P->exit_points_xy.assign(p->exit_points_xy, p->exit_points_xy + 2 * p->n_exit_points);
    P->exit_point_cost.assign(p->exit_point_cost, p->exit_point_cost + p->n_exit_points);
  }
  if (c->center_speed) P->center_speed.assign(c->center_speed, c->center_speed + J);
  const int64_t vlen = (int64_t)c->cells_x * P->g.n, hlen = (int64_t)c->cells_y * P->g.m;
  const double* tabs[4] = {c->probe_speed_w, c->probe_speed_e, c->probe_speed_s, c->probe_speed_n};
  for (int s = 0; s < 4; ++s)
    if (tabs[s]) P->probe[s].assign(tabs[s], tabs[s] + (s < 2 ? vlen : hlen));

  CellGeom& g = P->cg;
  g.m = P->g.m;
  g.n = P->g.n;
  g.P = P->pitch;
  g.pad = kPad;
  g.cells_x = c->cells_x;
  g.cells_y = c->cells_y;
  g.base_x = P->g.m / c->cells_x;
  g.base_y = P->g.n / c->cells_y;
  g.max_w = (int)(P->g.m - (c->cells_x - 1) * g.base_x);
  g.max_h = (int)(P->g.n - (c->cells_y - 1) * g.base_y);
  g.pu = even_up(g.max_w + 2);
  g.pc = even_up(g.max_w);
  g.tile_doubles = (int64_t)(g.max_h + 2) * g.pu + (int64_t)g.max_h * g.pc;
  const size_t tile_bytes = (size_t)g.tile_doubles * sizeof(double);
  if (tile_bytes > kTileMax)
    return fail(EIK_ERR_NOT_IMPL, "cell too large for the shared-memory tile (max ~150x150 nodes)");
  P->warps_per_cta = (int)std::max<size_t>(1, std::min<size_t>(8, kTileBudget / tile_bytes));

  int rc;
  if ((rc = dalloc(&P->dOrder, J))) return rc;
  P->allocs.push_back(P->dOrder);
  if ((rc = dalloc(&P->dRank, J))) return rc;
  P->allocs.push_back(P->dRank);
  if ((rc = dalloc(&P->dFlags, J))) return rc;
  P->allocs.push_back(P->dFlags);
  if ((rc = dalloc(&P->dCellDone, J))) return rc;
  P->allocs.push_back(P->dCellDone);
  if ((rc = dalloc(&P->dNext, 4))) return rc;
  P->allocs.push_back(P->dNext);
  if ((rc = dalloc(&P->dCounters, 8))) return rc;
  P->allocs.push_back(P->dCounters);
  return EIK_OK;
}

int plan_run_fmsm(eik_plan* P, eik_output* out) {
  using clk = std::chrono::steady_clock;
  const int64_t J = (int64_t)P->cells_x * P->cells_y;
  // ---- Part I on the host (the reference's own split, fmsm.cpp:130-162) --
  const auto t0 = clk::now();
  eik_problem hp{};
  hp.grid = P->g;
  hp.exit_nodes = P->exit_nodes.data();
  hp.exit_cost = P->exit_cost.data();
  hp.n_exit = (int64_t)P->exit_nodes.size();
  hp.exit_points_xy = P->exit_points_xy.empty() ? nullptr : P->exit_points_xy.data();
  hp.exit_point_cost = P->exit_point_cost.empty() ? nullptr : P->exit_point_cost.data();
  hp.n_exit_points = (int64_t)P->exit_point_cost.size();
  eik_cells hc{};
  hc.cells_x = P->cells_x;
  hc.cells_y = P->cells_y;
  hc.center_speed = P->center_speed.data();
  FmsmOrder ord;
  if (fmsm_part1(&hp, &hc, &ord)) return fail(EIK_ERR_CONFIG, "fmsm: empty coarse exit set");
  std::vector<uint8_t> flags(J);
  for (int64_t cell = 0; cell < J; ++cell) {
    if (ord.is_q[cell]) {
      flags[cell] = 16;
      continue;
    }
    const int64_t cx = cell % P->cells_x, cy = cell / P->cells_x;
    const int32_t r = ord.rank[cell];
    const bool w = cx > 0 && ord.rank[cell - 1] < r;
    const bool e = cx + 1 < P->cells_x && ord.rank[cell + 1] < r;
    const bool s = cy > 0 && ord.rank[cell - P->cells_x] < r;
    const bool n = cy + 1 < P->cells_y && ord.rank[cell + P->cells_x] < r;
    flags[cell] = fmsm_dir_mask(w, e, s, n);
  }
  const double host_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();

  // ---- Part II on the device -------------------------------------------
  int launches = 0;
  CK(cudaEventRecord(P->ev0, P->stream));
  CK(cudaMemcpyAsync(P->dOrder, ord.order.data(), sizeof(int32_t) * J, cudaMemcpyHostToDevice,
                     P->stream));
  CK(cudaMemcpyAsync(P->dRank, ord.rank.data(), sizeof(int32_t) * J, cudaMemcpyHostToDevice,
                     P->stream));
  CK(cudaMemcpyAsync(P->dFlags, flags.data(), J, cudaMemcpyHostToDevice, P->stream));
  CK(cudaMemsetAsync(P->dCellDone, 0, sizeof(int) * J, P->stream));
  CK(cudaMemsetAsync(P->dNext, 0, sizeof(int) * 4, P->stream));
  CK(cudaMemsetAsync(P->dCounters, 0, sizeof(unsigned long long) * 8, P->stream));
  CK(launch_prepare(P->dF, P->dC, P->dU, P->g.m, P->g.n, P->pitch, kPad, P->g.h, P->dExit,
                    P->dExitCost, P->n_exit, P->dStatus, P->stream, &launches));
  FmsmArgs a;
  a.g = P->cg;
  a.C = P->dC;
  a.u = P->dU;
  a.order = P->dOrder;
  a.rank = P->dRank;
  a.flags = P->dFlags;
  a.done = P->dCellDone;
  a.next = P->dNext;
  a.counters = P->dCounters;
  a.status = P->dStatus;
  a.J = (int)J;
  a.max_cell_sweeps = 1 << 20;
  CK(launch_fmsm(a, P->warps_per_cta, P->stream, &launches));
  CK(cudaEventRecord(P->ev1, P->stream));
  int st[8];
  unsigned long long cnt[2];
  CK(cudaMemcpyAsync(st, P->dStatus, sizeof(st), cudaMemcpyDeviceToHost, P->stream));
  CK(cudaMemcpyAsync(cnt, P->dCounters, sizeof(cnt), cudaMemcpyDeviceToHost, P->stream));
  CK(cudaStreamSynchronize(P->stream));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, P->ev0, P->ev1));
  if (st[0] == 1) return fail(EIK_ERR_DOMAIN, "speed must be positive and finite at every node");
  if (st[0] == 3) return fail(EIK_ERR_BUDGET, "fmsm: in-cell sweep budget exceeded");
  if (st[0] == 4) return fail(EIK_ERR_CUDA, "fmsm dataflow watchdog fired (scheduling bug)");
  // counters: sweeps are fine-pass cell sweeps; removals/updates include the
  // coarse Fast March's (fmsm.cpp:173-174)
  out->sweeps = (int64_t)cnt[0];
  out->node_updates = ord.coarse_updates + (int64_t)cnt[1];
  out->heap_removals = ord.coarse_pops;
  out->cell_sweeps = out->sweeps;
  out->avs = (double)out->sweeps / (double)J;
  out->device_ms = ms;
  out->host_ms = host_ms;
  out->kernel_launches = launches;
  return EIK_OK;
}

}  // namespace eikb200
