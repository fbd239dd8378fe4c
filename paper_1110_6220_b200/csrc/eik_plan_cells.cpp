// Host runtime of the two-scale methods: cell geometry, FMSM Part I on the
// host (as in the reference), uploads, and the device dataflow launch.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "eik_host.h"
#include "eik_plan.h"

namespace eikb200 {

namespace {

constexpr int kStatusWatchdogHost = 4;  // k_common.cuh kStatusWatchdog
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

thread_local const StripGeom* t_strip_geom = nullptr;

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
  // border-probe speed tables (HCM/FHCM): uploaded straight from the
  // caller's arrays -- by the first run when the plan defers its uploads
  // (eik_solve_batch), else now
  const double* tabs[4] = {c->probe_speed_w, c->probe_speed_e, c->probe_speed_s, c->probe_speed_n};
  for (int s = 0; s < 4; ++s) P->probe_len[s] = tabs[s] ? (s < 2 ? vlen : hlen) : 0;

  CellGeom& g = P->cg;
  g.m = P->g.m;
  g.n = P->g.n;
  g.P = P->pitch;
  g.pad = kPad;
  g.cells_x = c->cells_x;
  g.cells_y = c->cells_y;
  g.base_x = P->g.m / c->cells_x;
  g.base_y = P->g.n / c->cells_y;
  g.row0 = 0;
  g.row_end = P->g.n;
  if (const StripGeom* sg = t_strip_geom) {  // a sharded FMSM's strip
    g.base_y = sg->base_y;
    g.row0 = sg->row0;
    g.row_end = sg->row_end;
  }
  g.max_w = (int)(P->g.m - (c->cells_x - 1) * g.base_x);
  g.max_h = (int)std::max<int64_t>(g.base_y, g.row_end - (g.row0 + (c->cells_y - 1) * g.base_y));
  g.pu = even_up(g.max_w + 2);
  // heap-cell tiles put node x at column x+2 (16-byte aligned value pairs)
  if (P->method == EIK_HCM || P->method == EIK_FHCM) g.pu = even_up(g.max_w + 3);
  // FMSM tiles by TMA: boxes start on an even padded column, so node 0 sits
  // at tile column 1 or 2 -- two more columns than the halo needs
  if (P->method == EIK_FMSM) g.pu = even_up(g.max_w + 2) + 2;
  g.pc = even_up(g.max_w);
  // values + costs, both with halo; each half 128-byte aligned (TMA destinations)
  g.tile_doubles = 2 * (((int64_t)(g.max_h + 2) * g.pu + 15) & ~(int64_t)15);
  const size_t tile_bytes = (size_t)g.tile_doubles * sizeof(double);
  const bool hc = P->method == EIK_HCM || P->method == EIK_FHCM;
  P->max_len = std::max(g.max_w, g.max_h);
  // Cells whose tile does not fit shared memory (or taller than the 4 rows
  // per lane of the register engine) are swept in place in the padded field
  // by the band-splitting engine (k_cellsweep.cuh big_cell_sweep): FMSM by
  // the same dataflow kernel, HCM/FHCM by the exact serial heap loop
  // (heapcell_serial_kernel) -- any decomposition cells.cpp:32-47 accepts.
  P->cells_big = tile_bytes > kTileMax || (hc && heapcell_smem_bytes(g, P->max_len) > 227 * 1024);
  if (P->cells_big) g.tile_doubles = 0;
  P->warps_per_cta = P->cells_big
                         ? 8
                         : (int)std::max<size_t>(1, std::min<size_t>(8, kTileBudget / tile_bytes));

  int rc;
  if (hc && P->cells_big) {
    for (int s = 0; s < 4; ++s) {
      if ((rc = dalloc(&P->dProbe[s], (size_t)P->probe_len[s]))) return rc;
      P->allocs.push_back(P->dProbe[s]);
      if (P->deferred) {
        P->defer_probe[s] = tabs[s];
      } else {
        CK(cudaMemcpyAsync(P->dProbe[s], tabs[s], sizeof(double) * P->probe_len[s],
                           cudaMemcpyHostToDevice, P->stream));
      }
    }
    if ((rc = dalloc(&P->dCVal, J))) return rc;
    P->allocs.push_back(P->dCVal);
    if ((rc = dalloc(&P->dInitCells, J))) return rc;
    P->allocs.push_back(P->dInitCells);
    if ((rc = dalloc(&P->dInitValues, J))) return rc;
    P->allocs.push_back(P->dInitValues);
    if ((rc = dalloc(&P->dCounters, 48))) return rc;
    P->allocs.push_back(P->dCounters);
    if ((rc = dalloc(&P->dBInq, J))) return rc;
    P->allocs.push_back(P->dBInq);
    if ((rc = dalloc(&P->dBFlags, J))) return rc;
    P->allocs.push_back(P->dBFlags);
    if ((rc = dalloc(&P->dBFdone, J))) return rc;
    P->allocs.push_back(P->dBFdone);
    if ((rc = dalloc(&P->dBigLock, (size_t)g.max_w * g.max_h))) return rc;
    P->allocs.push_back(P->dBigLock);
    if ((rc = dalloc(&P->dBigScratch, 8 * (size_t)P->max_len))) return rc;
    P->allocs.push_back(P->dBigScratch);
    {  // row of a cell id by a multiply and shift, checked for every id
      const uint64_t d = (uint64_t)P->cells_x;
      uint64_t magic = ((1ull << 40) + d - 1) / d;
      for (int64_t c = 0; magic && c < J; ++c)
        if ((((uint64_t)c * magic) >> 40) != (uint64_t)c / d) magic = 0;
      P->hc_cx_magic = magic;
    }
    P->hc_warps_per_cta = 1;
    P->hc_min_smem = 0;
    P->hc_max_ctas = 1;
    return EIK_OK;
  }
  if (hc) {
    const size_t smem = heapcell_smem_bytes(g, P->max_len);
    for (int s = 0; s < 4; ++s) {
      if ((rc = dalloc(&P->dProbe[s], (size_t)P->probe_len[s]))) return rc;
      P->allocs.push_back(P->dProbe[s]);
      if (P->deferred) {
        P->defer_probe[s] = tabs[s];
      } else {
        CK(cudaMemcpyAsync(P->dProbe[s], tabs[s], sizeof(double) * P->probe_len[s],
                           cudaMemcpyHostToDevice, P->stream));
      }
    }
    if ((rc = dalloc(&P->dState, J))) return rc;
    P->allocs.push_back(P->dState);
    // committer queue bucket of cell (x, y): (x + 2y) mod 32 (k_heapcell.cu);
    // the global layout holds every cell of the fullest bucket
    int64_t capb_g = 1;
    {
      std::vector<int64_t> per(32, 0);
      for (int64_t y = 0; y < c->cells_y; ++y)
        for (int64_t x = 0; x < c->cells_x; ++x) ++per[(x + 2 * y) & 31];
      for (int64_t v : per) capb_g = std::max(capb_g, v);
    }
    P->hc_capb_global = (int)capb_g;
    if ((rc = dalloc(&P->dHKey, 32 * capb_g))) return rc;
    P->allocs.push_back(P->dHKey);
    if ((rc = dalloc(&P->dCKey, J))) return rc;
    P->allocs.push_back(P->dCKey);
    if ((rc = dalloc(&P->dCTag, J))) return rc;
    P->allocs.push_back(P->dCTag);
    if ((rc = dalloc(&P->dCVal, J))) return rc;
    P->allocs.push_back(P->dCVal);
    if ((rc = dalloc(&P->dHPos, J))) return rc;
    P->allocs.push_back(P->dHPos);
    if ((rc = dalloc(&P->dHArr, 32 * capb_g))) return rc;
    P->allocs.push_back(P->dHArr);
    if ((rc = dalloc(&P->dInitCells, J))) return rc;
    P->allocs.push_back(P->dInitCells);
    if ((rc = dalloc(&P->dInitValues, J))) return rc;
    P->allocs.push_back(P->dInitValues);
    if ((rc = dalloc(&P->dCounters, 48))) return rc;
    P->allocs.push_back(P->dCounters);
    const size_t cellsz = (size_t)even_up(g.max_w) * g.max_h;  // even slot pitch
    if ((rc = dalloc(&P->dSlots, 3 * (size_t)J * cellsz))) return rc;
    P->allocs.push_back(P->dSlots);
    if ((rc = dalloc(&P->dSpecVer, 2 * J))) return rc;
    P->allocs.push_back(P->dSpecVer);
    if ((rc = dalloc(&P->dBusy, 2 * J))) return rc;
    P->allocs.push_back(P->dBusy);
    if ((rc = dalloc(&P->dRec, 2 * J))) return rc;
    P->allocs.push_back(P->dRec);
    // [0] done flag (its own line), then the 32 published bucket counts, one
    // 128-byte line each (all workers poll them)
    if ((rc = dalloc(&P->dHcMisc, 32 + 2 * 32 * 32))) return rc;
    P->allocs.push_back(P->dHcMisc);
    if (P->method == EIK_HCM) {  // band scheduler state (hcm_band_kernel)
      if ((rc = dalloc(&P->dBInq, J))) return rc;
      P->allocs.push_back(P->dBInq);
      if ((rc = dalloc(&P->dBFlags, J))) return rc;
      P->allocs.push_back(P->dBFlags);
      if ((rc = dalloc(&P->dBFdone, J))) return rc;
      P->allocs.push_back(P->dBFdone);
      if ((rc = dalloc(&P->dBList, 2 * J))) return rc;
      P->allocs.push_back(P->dBList);
      if ((rc = dalloc(&P->dBWork, J))) return rc;
      P->allocs.push_back(P->dBWork);
      if ((rc = dalloc(&P->dBCtl, 8))) return rc;
      P->allocs.push_back(P->dBCtl);
      if ((rc = dalloc(&P->dBKmin, 2))) return rc;
      P->allocs.push_back(P->dBKmin);
      P->hcm_band = !P->hcm_exact_req && hcm_default_mode() == 0;
    }
    // per-warp tile: values + costs with halo, 4 border snapshots, lock bytes
    const size_t tile = ((smem + sizeof(double) - 1) / sizeof(double) + 1) & ~(size_t)1;
    P->cg.tile_doubles = (int64_t)tile;
    // One CTA per SM: up to 8 warps (their tiles within 216 KB) and a shared-
    // memory floor above half the SM, so no second CTA of this or another
    // smem-using kernel lands on the SM (8 warps x 250 registers also fill the
    // register file).  The committer (CTA 0) then has its SM to itself, and
    // plans sharing the GPU (eik_plan_run_batch) split it by whole SMs.
    // Solo times within 3 % of 2-warp CTAs packed 1-4 per SM.
    // EIK_HC_WARPS / EIK_HC_MIN_SMEM override.
    const int fit = (int)std::max<size_t>(1, std::min<size_t>(8, (216 * 1024) / (tile * 8)));
    P->hc_warps_per_cta = fit;
    const Knobs& kn = knobs();
    if (kn.hc_warps > 0) P->hc_warps_per_cta = std::max(1, std::min(fit, kn.hc_warps));
    P->hc_min_smem = 116 * 1024;
    {  // row of a cell id by a multiply and shift, checked for every id
      const uint64_t d = (uint64_t)P->cells_x;
      uint64_t magic = ((1ull << 40) + d - 1) / d;
      if (J > 1 && (uint64_t)(J - 1) > ~0ull / magic) magic = 0;
      for (int64_t c = 0; magic && c < J; ++c)
        if ((((uint64_t)c * magic) >> 40) != (uint64_t)c / d) magic = 0;
      P->hc_cx_magic = magic;
    }
    if (kn.hc_min_smem >= 0) P->hc_min_smem = kn.hc_min_smem;
    // the committer's heap + cell values go to its shared memory when they
    // fit next to its tile (uint16 heap indices)
    {
      // committer queue buckets in shared memory next to its tile; a bucket
      // that fills up raises a status and the run repeats with global buckets
      const size_t room = 220 * 1024 > tile * 8 ? 220 * 1024 - tile * 8 : 0;
      size_t capb = std::min<size_t>((size_t)capb_g, room / (32 * 12));
      while (capb > 0 && heapcell_committer_heap_bytes((int)capb) > room) --capb;
      P->hc_heap_cap = capb >= 8 ? (int)capb : 0;
    }
    if (kn.hc_global_heap) P->hc_heap_cap = 0;
    // EIK_HC_HEAP_CAP=n caps the shared-memory heap (exercises the overflow
    // fallback in tests)
    if (kn.hc_heap_cap > 0) P->hc_heap_cap = std::min(P->hc_heap_cap, kn.hc_heap_cap);
    // EIK_HC_CHAIN: 0 plain speculations only, 1 chain on the neighbour
    // expected next (default), 2 on every neighbour expected first
    P->hc_chain = kn.hc_chain;
    // EIK_HC_CTAS=1 runs the committer alone (serial exact replay)
    P->hc_max_ctas = 1 << 20;
    if (kn.hc_ctas > 0) P->hc_max_ctas = kn.hc_ctas;
    return EIK_OK;
  }
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

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// libcuda link dependency); null when the driver does not provide it
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// Tensor maps of the tile loads: the padded u and C from row -1, box = one
// tile (pu x (max_h + 2)).  False when a box dimension or the row stride is
// outside what the TMA unit takes (the warps then stage by loads), or
// EIK_TILE_TMA=0.  nmaps = 2: u then C (FMSM); 1: C alone (heap cells).
static bool tile_tensor_maps(eik_plan* P, int nmaps) {
  const EncodeTiledFn enc = encode_tiled();
  const CellGeom& g = P->cg;
  if (!enc || g.pu > 256 || g.max_h + 2 > 256 || (P->pitch * 8) % 16 != 0) return false;
  if (knobs().tile_tma == 0) return false;
  alignas(64) CUtensorMap maps[2];
  const cuuint64_t dims[2] = {(cuuint64_t)P->pitch, (cuuint64_t)(P->g.n + 2)};
  const cuuint64_t strides[1] = {(cuuint64_t)P->pitch * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)g.pu, (cuuint32_t)(g.max_h + 2)};
  const cuuint32_t estr[2] = {1, 1};
  for (int t = 0; t < nmaps; ++t) {
    double* base = (nmaps == 2 && t == 0 ? P->dU : P->dC) - P->pitch;  // row -1
    CUresult r = enc(&maps[t], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
  }
  // the maps live in device memory (64-byte aligned), copied before the launch
  if (!P->dTmaps) {
    if (pool_alloc(&P->dTmaps, sizeof(maps)) != cudaSuccess) return false;
    P->allocs.push_back(P->dTmaps);
  }
  if (cudaMemcpyAsync(P->dTmaps, maps, sizeof(maps), cudaMemcpyHostToDevice, P->stream) !=
      cudaSuccess)
    return false;
  return true;
}

bool fmsm_tensor_maps(eik_plan* P, FmsmArgs* a) {
  if (!tile_tensor_maps(P, 2)) return false;
  a->tmaps = static_cast<const CUtensorMap*>(P->dTmaps);
  return true;
}

int plan_prepare_host(eik_plan* P) {
  if (P->method != EIK_FMSM || P->fmsm_ready) return EIK_OK;
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
  std::vector<uint8_t>& flags = P->fmsm_flags;
  flags.resize(J);
  const int32_t* rank = ord.rank.data();
  for (int64_t cy = 0, cell = 0; cy < P->cells_y; ++cy)
    for (int64_t cx = 0; cx < P->cells_x; ++cx, ++cell) {
      if (ord.is_q[cell]) {
        flags[cell] = 16;
        continue;
      }
      const int32_t r = rank[cell];
      const bool w = cx > 0 && rank[cell - 1] < r;
      const bool e = cx + 1 < P->cells_x && rank[cell + 1] < r;
      const bool s = cy > 0 && rank[cell - P->cells_x] < r;
      const bool n = cy + 1 < P->cells_y && rank[cell + P->cells_x] < r;
      flags[cell] = fmsm_dir_mask(w, e, s, n);
    }
  P->fmsm_order = std::move(ord.order);
  P->fmsm_rank = std::move(ord.rank);
  P->fmsm_coarse_pops = ord.coarse_pops;
  P->fmsm_coarse_updates = ord.coarse_updates;
  P->fmsm_host_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
  P->fmsm_ready = true;
  return EIK_OK;
}

int plan_run_fmsm(eik_plan* P, eik_output* out) {
  const int64_t J = (int64_t)P->cells_x * P->cells_y;
  int rc0 = plan_prepare_host(P);
  if (rc0) return rc0;
  P->fmsm_ready = false;  // every run computes its own Part I
  const double host_ms = P->fmsm_host_ms;

  // ---- Part II on the device -------------------------------------------
  int launches = 0;
  CK(cudaEventRecord(P->ev0, P->stream));
  CK(cudaMemcpyAsync(P->dOrder, P->fmsm_order.data(), sizeof(int32_t) * J,
                     cudaMemcpyHostToDevice, P->stream));
  CK(cudaMemcpyAsync(P->dRank, P->fmsm_rank.data(), sizeof(int32_t) * J, cudaMemcpyHostToDevice,
                     P->stream));
  CK(cudaMemcpyAsync(P->dFlags, P->fmsm_flags.data(), J, cudaMemcpyHostToDevice, P->stream));
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
  a.big = P->cells_big ? 1 : 0;
  a.nowait = 0;
  a.use_tma = (!P->cells_big && fmsm_tensor_maps(P, &a)) ? 1 : 0;
  int grid = 0;
  CK(launch_fmsm(a, P->warps_per_cta, P->cap(), P->stream, &launches, &grid));
  out->grid_ctas = grid;
  CK(cudaEventRecord(P->ev1, P->stream));
  int st[8];
  unsigned long long cnt[2];
  CK(stream_wait(P->stream));  // no spinning core while the solve runs
  CK(cudaMemcpyAsync(st, P->dStatus, sizeof(st), cudaMemcpyDeviceToHost, P->stream));
  CK(cudaMemcpyAsync(cnt, P->dCounters, sizeof(cnt), cudaMemcpyDeviceToHost, P->stream));
  CK(stream_wait(P->stream));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, P->ev0, P->ev1));
  if (st[0] == 1) return fail(EIK_ERR_DOMAIN, "speed must be positive and finite, and h / F within [2^-480, 2^500], at every node");
  if (st[0] == 3) return fail(EIK_ERR_BUDGET, "fmsm: in-cell sweep budget exceeded");
  if (st[0] == 4) return fail(EIK_ERR_CUDA, "fmsm dataflow watchdog fired (scheduling bug)");
  // counters: sweeps are fine-pass cell sweeps; removals/updates include the
  // coarse Fast March's (fmsm.cpp:173-174)
  out->sweeps = (int64_t)cnt[0];
  out->node_updates = P->fmsm_coarse_updates + (int64_t)cnt[1];
  out->heap_removals = P->fmsm_coarse_pops;
  out->cell_sweeps = out->sweeps;
  out->avs = (double)out->sweeps / (double)J;
  out->device_ms = ms;
  out->host_ms = host_ms;
  out->kernel_launches = launches;
  return EIK_OK;
}

// Cells too large for a shared-memory tile: the exact serial heap loop.
int plan_run_heapcell_serial(eik_plan* P, eik_output* out, const std::vector<int>& icells,
                             const std::vector<double>& ivals) {
  const int64_t J = (int64_t)P->cells_x * P->cells_y;
  int launches = 0;
  CK(cudaEventRecord(P->ev0, P->stream));
  CK(cudaMemcpyAsync(P->dInitCells, icells.data(), sizeof(int) * icells.size(),
                     cudaMemcpyHostToDevice, P->stream));
  CK(cudaMemcpyAsync(P->dInitValues, ivals.data(), sizeof(double) * ivals.size(),
                     cudaMemcpyHostToDevice, P->stream));
  CK(cudaMemsetAsync(P->dCounters, 0, sizeof(unsigned long long) * 48, P->stream));
  CK(launch_prepare(P->dF, P->dC, P->dU, P->g.m, P->g.n, P->pitch, kPad, P->g.h, P->dExit,
                    P->dExitCost, P->n_exit, P->dStatus, P->stream, &launches));
  HcArgs a{};
  a.g = P->cg;
  a.C = P->dC;
  a.u = P->dU;
  for (int s = 0; s < 4; ++s) a.probe[s] = P->dProbe[s];
  a.h = P->g.h;
  a.hc_x = (double)(P->g.m / P->cells_x) * P->g.h;  // cells.cpp:44-45
  a.hc_y = (double)(P->g.n / P->cells_y) * P->g.h;
  a.cval = P->dCVal;
  a.init_cells = P->dInitCells;
  a.init_values = P->dInitValues;
  a.n_init = (int)icells.size();
  a.counters = P->dCounters;
  a.status = P->dStatus;
  a.J = (int)J;
  a.fast = P->method == EIK_FHCM ? 1 : 0;
  a.budget = 100LL * J + 16;
  a.max_len = P->max_len;
  a.cx_magic = P->hc_cx_magic;
  a.b_inq = P->dBInq;
  a.b_flags = P->dBFlags;
  a.b_fdone = P->dBFdone;
  a.big_lock = P->dBigLock;
  a.big_scratch = P->dBigScratch;
  CK(launch_heapcell_serial(a, P->stream, &launches));
  out->grid_ctas = 1;
  if (P->on_launched) {
    auto f = std::move(P->on_launched);
    P->on_launched = nullptr;
    f();
  }
  CK(cudaEventRecord(P->ev1, P->stream));
  int st[8];
  unsigned long long cnt[5];
  CK(stream_wait(P->stream));  // no spinning core while the solve runs
  CK(cudaMemcpyAsync(st, P->dStatus, sizeof(st), cudaMemcpyDeviceToHost, P->stream));
  CK(cudaMemcpyAsync(cnt, P->dCounters, sizeof(cnt), cudaMemcpyDeviceToHost, P->stream));
  CK(stream_wait(P->stream));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, P->ev0, P->ev1));
  if (st[0] == 1) return fail(EIK_ERR_DOMAIN, "speed must be positive and finite, and h / F within [2^-480, 2^500], at every node");
  if (st[0] == 3) return fail(EIK_ERR_BUDGET, "heap-cell removal budget exceeded");
  out->heap_removals = (int64_t)cnt[0];
  out->sweeps = (int64_t)cnt[1];
  out->node_updates = (int64_t)cnt[2];
  out->mon_checks = (int64_t)cnt[3];
  out->mon_single = (int64_t)cnt[4];
  out->cell_removals = out->heap_removals;
  out->cell_sweeps = out->sweeps;
  out->avhr = (double)out->heap_removals / (double)J;
  out->avs = (double)out->sweeps / (double)J;
  out->mon_pct = out->mon_checks == 0 ? 0.0 : 100.0 * out->mon_single / (double)out->mon_checks;
  out->device_ms = ms;
  out->kernel_launches = launches;
  return EIK_OK;
}

// HCM by rounds of the acceptance band (k_heapcell.cu hcm_band_kernel).
int plan_run_hcm_band(eik_plan* P, eik_output* out, const std::vector<int>& icells,
                      const std::vector<double>& ivals) {
  const int64_t J = (int64_t)P->cells_x * P->cells_y;
  const Knobs& kn = knobs();
  int launches = 0;
  CK(cudaEventRecord(P->ev0, P->stream));
  CK(cudaMemcpyAsync(P->dInitCells, icells.data(), sizeof(int) * icells.size(),
                     cudaMemcpyHostToDevice, P->stream));
  CK(cudaMemcpyAsync(P->dInitValues, ivals.data(), sizeof(double) * ivals.size(),
                     cudaMemcpyHostToDevice, P->stream));
  CK(cudaMemsetAsync(P->dCounters, 0, sizeof(unsigned long long) * 48, P->stream));
  CK(cudaMemsetAsync(P->dBCtl, 0, sizeof(int) * 8, P->stream));
  CK(cudaMemsetAsync(P->dBKmin, 0xFF, sizeof(unsigned long long) * 2, P->stream));
  CK(launch_prepare(P->dF, P->dC, P->dU, P->g.m, P->g.n, P->pitch, kPad, P->g.h, P->dExit,
                    P->dExitCost, P->n_exit, P->dStatus, P->stream, &launches));
  HcArgs a{};
  a.g = P->cg;
  a.C = P->dC;
  a.u = P->dU;
  for (int s = 0; s < 4; ++s) a.probe[s] = P->dProbe[s];
  a.h = P->g.h;
  a.hc_x = (double)(P->g.m / P->cells_x) * P->g.h;  // cells.cpp:44-45
  a.hc_y = (double)(P->g.n / P->cells_y) * P->g.h;
  a.cval = P->dCVal;
  a.init_cells = P->dInitCells;
  a.init_values = P->dInitValues;
  a.n_init = (int)icells.size();
  a.counters = P->dCounters;
  a.status = P->dStatus;
  a.J = (int)J;
  a.fast = 0;
  a.budget = 100LL * J + 16;
  a.max_len = P->max_len;
  a.tile_doubles = P->cg.tile_doubles;
  // value and cost tiles by TMA when every cell's box starts on a 16-byte
  // column (even cell width)
  if (!P->cells_big && P->cg.base_x % 2 == 0 && tile_tensor_maps(P, 2)) {
    a.use_tma = 1;
    a.tm_band = static_cast<const CUtensorMap*>(P->dTmaps);
  }
  a.min_smem = P->hc_min_smem;
  a.cx_magic = P->hc_cx_magic;
  a.skip_from = kn.hc_skip_from;
  a.b_inq = P->dBInq;
  a.b_flags = P->dBFlags;
  a.b_fdone = P->dBFdone;
  a.b_list = P->dBList;
  a.b_work = P->dBWork;
  a.b_ctl = P->dBCtl;
  a.b_kmin = P->dBKmin;
  a.band_scale = kn.hcm_band > 0.0 ? kn.hcm_band : 4.0;
  a.band_adapt = kn.hcm_band > 0.0 ? 0 : 1;  // an explicit EIK_HCM_BAND fixes the width
  a.band_shrink = kn.hcm_band_shrink;
  a.prof = kn.hc_profile ? 1 : 0;
  const int hc_ctas = P->cap() > 0 ? std::min(P->hc_max_ctas, P->cap()) : P->hc_max_ctas;
  int grid = 0;
  CK(launch_hcm_band(a, P->hc_warps_per_cta, hc_ctas, P->stream, &launches, &grid));
  out->grid_ctas = grid;
  if (P->on_launched) {
    auto f = std::move(P->on_launched);
    P->on_launched = nullptr;
    f();
  }
  CK(cudaEventRecord(P->ev1, P->stream));
  int st[8];
  int ctl[8];
  unsigned long long cnt[12];
  CK(stream_wait(P->stream));  // no spinning core while the solve runs
  CK(cudaMemcpyAsync(st, P->dStatus, sizeof(st), cudaMemcpyDeviceToHost, P->stream));
  CK(cudaMemcpyAsync(ctl, P->dBCtl, sizeof(ctl), cudaMemcpyDeviceToHost, P->stream));
  CK(cudaMemcpyAsync(cnt, P->dCounters, sizeof(cnt), cudaMemcpyDeviceToHost, P->stream));
  CK(stream_wait(P->stream));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, P->ev0, P->ev1));
  if (st[0] == 1) return fail(EIK_ERR_DOMAIN, "speed must be positive and finite, and h / F within [2^-480, 2^500], at every node");
  if (st[0] == 3) return fail(EIK_ERR_BUDGET, "heap-cell removal budget exceeded");
  if (st[0] == kStatusWatchdogHost)
    return fail(EIK_ERR_CUDA, "hcm band scheduler made no progress (scheduling bug)");
  if (kn.hc_profile && grid > 0)
    std::fprintf(stderr, "hcm band: %d rounds, per CTA per round (cycles): sync %.0f select %.0f "
                 "work %.0f kmin %.0f\n", ctl[4], (double)cnt[8] / grid / std::max(1, ctl[4]),
                 (double)cnt[9] / grid / std::max(1, ctl[4]), (double)cnt[10] / grid / std::max(1, ctl[4]),
                 (double)cnt[11] / grid / std::max(1, ctl[4]));
  out->heap_removals = (int64_t)cnt[0];
  out->sweeps = (int64_t)cnt[1];
  out->node_updates = (int64_t)cnt[2];
  out->mon_checks = out->mon_single = 0;
  out->cell_removals = out->heap_removals;
  out->cell_sweeps = out->sweeps;
  out->avhr = (double)out->heap_removals / (double)J;
  out->avs = (double)out->sweeps / (double)J;
  out->mon_pct = 0.0;
  out->rounds = ctl[4];
  out->device_ms = ms;
  out->kernel_launches = launches;
  return EIK_OK;
}

int plan_run_heapcell(eik_plan* P, eik_output* out) {
  const int64_t J = (int64_t)P->cells_x * P->cells_y;
  // Cells intersecting the exit set start on the list with value = max exit
  // cost inside the cell (heap_cell.cpp:255-268); O(|Q|) host work.
  std::vector<int64_t> ib, ie, jb, je;
  split_axis(P->g.m, P->cells_x, ib, ie);
  split_axis(P->g.n, P->cells_y, jb, je);
  std::vector<std::pair<int, double>> init;
  {
    std::vector<double> cv;
    std::vector<int> touched;
    std::vector<char> seen;
    const int64_t m = P->g.m;
    for (size_t k = 0; k < P->exit_nodes.size(); ++k) {
      const int64_t i = P->exit_nodes[k] % m, j = P->exit_nodes[k] / m;
      const int64_t a = std::upper_bound(ie.begin(), ie.end(), i) - ie.begin();
      const int64_t b = std::upper_bound(je.begin(), je.end(), j) - je.begin();
      const int cell = (int)(b * P->cells_x + a);
      const double q = P->exit_cost[k];
      bool found = false;
      for (auto& pr : init)
        if (pr.first == cell) {
          pr.second = std::max(pr.second, q);
          found = true;
          break;
        }
      if (!found) init.push_back({cell, q});
    }
    std::sort(init.begin(), init.end(),
              [](const std::pair<int, double>& x, const std::pair<int, double>& y) {
                return x.first < y.first;
              });
  }
  std::vector<int> icells(init.size());
  std::vector<double> ivals(init.size());
  for (size_t k = 0; k < init.size(); ++k) {
    icells[k] = init[k].first;
    ivals[k] = init[k].second;
  }
  int launches = 0;
  if (P->cells_big) return plan_run_heapcell_serial(P, out, icells, ivals);
  if (P->method == EIK_HCM && P->hcm_band) return plan_run_hcm_band(P, out, icells, ivals);
retry:  // after a committer heap overflow, with the heap in global memory
  CK(cudaEventRecord(P->ev0, P->stream));
  CK(cudaMemcpyAsync(P->dInitCells, icells.data(), sizeof(int) * icells.size(),
                     cudaMemcpyHostToDevice, P->stream));
  CK(cudaMemcpyAsync(P->dInitValues, ivals.data(), sizeof(double) * ivals.size(),
                     cudaMemcpyHostToDevice, P->stream));
  CK(cudaMemsetAsync(P->dCounters, 0, sizeof(unsigned long long) * 48, P->stream));
  CK(launch_prepare(P->dF, P->dC, P->dU, P->g.m, P->g.n, P->pitch, kPad, P->g.h, P->dExit,
                    P->dExitCost, P->n_exit, P->dStatus, P->stream, &launches));
  HcArgs a;
  a.g = P->cg;
  a.C = P->dC;
  a.u = P->dU;
  for (int s = 0; s < 4; ++s) a.probe[s] = P->dProbe[s];
  a.h = P->g.h;
  a.hc_x = (double)(P->g.m / P->cells_x) * P->g.h;  // cells.cpp:44-45
  a.hc_y = (double)(P->g.n / P->cells_y) * P->g.h;
  a.state = P->dState;
  a.heap_cap = P->hc_heap_cap;
  a.cval = P->dCVal;
  a.hkey = P->dHKey;
  a.hpos = P->dHPos;
  a.harr = P->dHArr;
  a.init_cells = P->dInitCells;
  a.init_values = P->dInitValues;
  a.n_init = (int)icells.size();
  a.counters = P->dCounters;
  a.status = P->dStatus;
  a.J = (int)J;
  a.fast = P->method == EIK_FHCM ? 1 : 0;
  a.budget = 100LL * J + 16;
  a.max_len = P->max_len;
  a.slots = P->dSlots;
  a.spw = even_up(P->cg.max_w);
  a.cellsz = (int64_t)a.spw * P->cg.max_h;
  a.spec_ver = P->dSpecVer;
  a.busy = P->dBusy;
  a.rec = P->dRec;
  a.ckey = P->dCKey;
  a.wdbg = nullptr;
  a.owner = nullptr;
  const Knobs& kn = knobs();
  if (kn.hc_debug) {  // per-plan debug buffers sized for this grid and device
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->device);
    const size_t nw = (size_t)4 * sms * 64;
    if (!P->dDbg) {
      int rc2;
      if ((rc2 = dalloc(&P->dDbg, nw))) return rc2;
      P->allocs.push_back(P->dDbg);
      if ((rc2 = dalloc(&P->dOwner, 2 * (size_t)J))) return rc2;
      P->allocs.push_back(P->dOwner);
    }
    CK(cudaMemsetAsync(P->dDbg, 0, sizeof(int) * nw, P->stream));
    CK(cudaMemsetAsync(P->dOwner, 0xFF, sizeof(int) * 2 * (size_t)J, P->stream));
    a.wdbg = P->dDbg;
    a.owner = P->dOwner;
  }
  a.ctag = P->dCTag;
  a.chain = P->hc_chain;
  a.bands = knobs().hc_bands;
  a.prof = kn.hc_profile ? 1 : 0;
  a.idle_ns = kn.hc_idle_ns;
  a.done_flag = P->dHcMisc;
  a.hsize_pub = P->dHcMisc + 32;
  a.pubmin = P->dHcMisc + 32 + 32 * 32;
  a.first_min = kn.hc_first_min;
  a.first_min_pool = kn.hc_first_min_pool;
  a.heap_capb_global = P->hc_capb_global;
  // cost tiles by TMA when every cell's box starts on a 16-byte column
  // (even cell width: node ib - 2 of an even ib); the maps travel with the
  // plan's stream ahead of the launch
  a.use_tma = 0;
  a.tmc = nullptr;
  if (!P->cells_big && P->cg.base_x % 2 == 0 && tile_tensor_maps(P, 1)) {
    a.use_tma = 1;
    a.tmc = static_cast<const CUtensorMap*>(P->dTmaps);
  }
  a.pub_capb = P->hc_heap_cap > 0 ? P->hc_heap_cap : P->hc_capb_global;
  a.tile_doubles = P->cg.tile_doubles;
  a.min_smem = P->hc_min_smem;
  a.cx_magic = P->hc_cx_magic;
  // HCM's first sweep runs mostly unlocked nodes: the branch-free engine wins
  // there, the vote-skip one on the convergence sweeps (measured 1-3 % at
  // every cell size; EIK_HC_SKIP_FROM overrides)
  a.skip_from = kn.hc_skip_from;
  CK(cudaMemsetAsync(P->dHcMisc, 0, sizeof(int) * (32 + 32 * 32), P->stream));
  CK(cudaMemsetAsync(a.pubmin, 0xFF, sizeof(int) * 32 * 32, P->stream));
  const int hc_ctas = P->cap() > 0 ? std::min(P->hc_max_ctas, P->cap()) : P->hc_max_ctas;
  int grid = 0;
  CK(launch_heapcell(a, P->hc_warps_per_cta, hc_ctas, P->stream, &launches, &grid));
  out->grid_ctas = grid;
  if (P->on_launched) {
    auto f = std::move(P->on_launched);
    P->on_launched = nullptr;
    f();
  }
  CK(cudaEventRecord(P->ev1, P->stream));
  int st[8];
  unsigned long long cnt[48];
  CK(stream_wait(P->stream));  // no spinning core while the solve runs
  CK(cudaMemcpyAsync(st, P->dStatus, sizeof(st), cudaMemcpyDeviceToHost, P->stream));
  CK(cudaMemcpyAsync(cnt, P->dCounters, sizeof(cnt), cudaMemcpyDeviceToHost, P->stream));
  CK(stream_wait(P->stream));
  if (st[0] == 6 && P->hc_heap_cap == 0)
    return fail(EIK_ERR_CUDA, "heap-cell queue bucket overflow in global memory (sizing bug)");
  if (st[0] == 6 && P->hc_heap_cap > 0) {
    P->hc_heap_cap = 0;
    CK(cudaMemsetAsync(P->dStatus, 0, sizeof(int) * 8, P->stream));
    goto retry;
  }
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, P->ev0, P->ev1));
  if (st[0] == 1) return fail(EIK_ERR_DOMAIN, "speed must be positive and finite, and h / F within [2^-480, 2^500], at every node");
  if (st[0] == 3) return fail(EIK_ERR_BUDGET, "heap-cell removal budget exceeded");
  if (st[0] == 4 || st[0] == 5) {
    std::fprintf(stderr,
                 "heapcell stuck: status %d cell %llu busy %llu/%llu state %llx spec %llx/%llx "
                 "after %llu pops; bad-slot state %llx | owner %llx phase %llu cell %llu kind %llu "
                 "age %llu kcycles worker %lld\n",
                 st[0], cnt[24], cnt[25], cnt[26], cnt[27], cnt[28], cnt[29], cnt[30], cnt[31],
                 (long long)cnt[32], cnt[33], cnt[34], cnt[35], cnt[36], (long long)cnt[37]);
    return fail(EIK_ERR_CUDA, st[0] == 4 ? "heap-cell committer watchdog fired"
                                         : "heap-cell slot index out of range");
  }
  if (kn.hc_profile)
    std::fprintf(stderr,
                 "heapcell committer cycles: pop %llu obtain %llu self %llu commit %llu | self: "
                 "stage %llu sweeps %llu scans %llu | hits %llu (chained %llu) self %llu | "
                 "heap max %llu cap %d | stage: %llu reset_locks %llu steps %llu | commit: record %llu | "
                 "obtain: rescan %llu first-rt %llu waits %llu (%llu cycles) | commit to end of "
                 "the neighbour block %llu\n",
                 cnt[8], cnt[9], cnt[10], cnt[11], cnt[12], cnt[13], cnt[14], cnt[6], cnt[15],
                 cnt[5], cnt[38], P->hc_heap_cap, cnt[39], cnt[40], cnt[41], cnt[42], cnt[43],
                 cnt[44], cnt[7], cnt[45], cnt[46]);
  if (kn.hc_profile)
    std::fprintf(stderr,
                 "heapcell misses: unchained %llu pending %llu stale %llu wrong-inst %llu "
                 "other-side %llu | last=self %llu prev-pop-adjacent %llu plain-stale-by-1 %llu\n",
                 cnt[16], cnt[17], cnt[18], cnt[19], cnt[20], cnt[21], cnt[22], cnt[23]);
  out->spec_self = (int64_t)cnt[5];
  out->spec_hits = (int64_t)cnt[6];
  out->spec_waits = (int64_t)cnt[7];
  // SolverOutput / HybridStats (heap_cell.cpp:314-322)
  out->heap_removals = (int64_t)cnt[0];
  out->sweeps = (int64_t)cnt[1];
  out->node_updates = (int64_t)cnt[2];
  out->mon_checks = (int64_t)cnt[3];
  out->mon_single = (int64_t)cnt[4];
  out->cell_removals = out->heap_removals;
  out->cell_sweeps = out->sweeps;
  out->avhr = (double)out->heap_removals / (double)J;
  out->avs = (double)out->sweeps / (double)J;
  out->mon_pct = out->mon_checks == 0 ? 0.0 : 100.0 * out->mon_single / (double)out->mon_checks;
  out->device_ms = ms;
  out->kernel_launches = launches;
  return EIK_OK;
}

// ---- a sharded FMSM's strip: levels of the cell DAG ----------------------
// (distributed.fmsm_solve_strips).  The cells of one level are pairwise
// non-adjacent and every earlier-ranked neighbour of each sits in an earlier
// level, so a level runs with no waiting: its inputs are final once the
// earlier levels and the ghost rows they changed are in place.
int plan_fmsm_levels(eik_plan* P, const int32_t* cells, const int32_t* off, int32_t nlevels,
                     const uint8_t* flags) {
  if (P->method != EIK_FMSM) return fail(EIK_ERR_CONFIG, "fmsm levels need an fmsm plan");
  if (nlevels < 0 || (nlevels > 0 && (!cells || !off))) return fail(EIK_ERR_DOMAIN, "bad levels");
  const int64_t J = (int64_t)P->cells_x * P->cells_y;
  const int64_t total = nlevels > 0 ? off[nlevels] : 0;
  if (total != J) return fail(EIK_ERR_DOMAIN, "the levels must list every cell of the strip once");
  for (int32_t L = 0; L < nlevels; ++L)
    if (off[L] > off[L + 1]) return fail(EIK_ERR_DOMAIN, "level offsets must not decrease");
  for (int64_t k = 0; k < total; ++k)
    if (cells[k] < 0 || cells[k] >= J) return fail(EIK_ERR_DOMAIN, "level cell id out of range");
  CK(cudaSetDevice(P->device));
  AllocStream alloc_on(P->stream);
  if (P->level_cap < std::max<int64_t>(1, nlevels)) {
    int rc;
    if ((rc = dalloc(&P->dLevelNext, std::max<int64_t>(1, nlevels)))) return rc;
    P->allocs.push_back(P->dLevelNext);
    P->level_cap = std::max<int64_t>(1, nlevels);
  }
  P->level_off.assign(off, off + nlevels + 1);
  CK(cudaMemcpyAsync(P->dOrder, cells, sizeof(int32_t) * J, cudaMemcpyHostToDevice, P->stream));
  CK(cudaMemcpyAsync(P->dFlags, flags, J, cudaMemcpyHostToDevice, P->stream));
  CK(cudaMemsetAsync(P->dLevelNext, 0, sizeof(int) * P->level_cap, P->stream));
  CK(cudaMemsetAsync(P->dCellDone, 0, sizeof(int) * J, P->stream));
  CK(cudaMemsetAsync(P->dCounters, 0, sizeof(unsigned long long) * 8, P->stream));
  CK(cudaMemsetAsync(P->dStatus, 0, sizeof(int) * 8, P->stream));
  int launches = 0;
  CK(launch_prepare(P->dF, P->dC, P->dU, P->g.m, P->g.n, P->pitch, kPad, P->g.h, P->dExit,
                    P->dExitCost, P->n_exit, P->dStatus, P->stream, &launches));
  CK(stream_wait(P->stream));
  return EIK_OK;
}

int plan_fmsm_level_async(eik_plan* P, int32_t L, cudaStream_t stream) {
  if (P->method != EIK_FMSM || L < 0 || L + 1 >= (int32_t)P->level_off.size())
    return fail(EIK_ERR_CONFIG, "no such fmsm level (eik_plan_fmsm_levels first)");
  const int32_t n = P->level_off[L + 1] - P->level_off[L];
  if (n == 0) return EIK_OK;
  CK(cudaSetDevice(P->device));
  const cudaStream_t s = stream ? stream : P->stream;
  FmsmArgs a;
  a.g = P->cg;
  a.C = P->dC;
  a.u = P->dU;
  a.order = P->dOrder + P->level_off[L];
  a.rank = P->dRank;
  a.flags = P->dFlags;
  a.done = P->dCellDone;
  a.next = P->dLevelNext + L;
  a.counters = P->dCounters;
  a.status = P->dStatus;
  a.J = n;
  a.max_cell_sweeps = 1 << 20;
  a.big = P->cells_big ? 1 : 0;
  a.nowait = 1;
  a.use_tma = 0;
  a.tmaps = nullptr;
  if (!P->cells_big) {
    // the tensor maps were copied on the plan's stream: order it before `s`
    if (!P->tma_tried) {
      P->tma_ok = fmsm_tensor_maps(P, &a);
      P->tma_tried = true;
      CK(stream_wait(P->stream));
    }
    if (P->tma_ok) {
      a.use_tma = 1;
      a.tmaps = static_cast<const CUtensorMap*>(P->dTmaps);
    }
  }
  int launches = 0;
  CK(launch_fmsm(a, P->warps_per_cta, P->cap(), s, &launches, nullptr));
  return EIK_OK;
}

int plan_fmsm_counters(eik_plan* P, int64_t out[2]) {
  CK(cudaSetDevice(P->device));
  CK(stream_wait(P->stream));
  CK(cudaDeviceSynchronize());
  int st[8];
  unsigned long long cnt[2];
  CK(cudaMemcpy(st, P->dStatus, sizeof(st), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cnt, P->dCounters, sizeof(cnt), cudaMemcpyDeviceToHost));
  if (st[0] == 1) return fail(EIK_ERR_DOMAIN, "speed must be positive and finite, and h / F within [2^-480, 2^500], at every node");
  if (st[0] == 3) return fail(EIK_ERR_BUDGET, "fmsm: in-cell sweep budget exceeded");
  out[0] = (int64_t)cnt[0];
  out[1] = (int64_t)cnt[1];
  return EIK_OK;
}

// The schedule every rank of a sharded FMSM computes identically: Part I's
// order and rank, each cell's sweep flags, and its DAG level.
int fmsm_schedule(const eik_problem* p, const eik_cells* c, int32_t* order, int32_t* rank,
                  uint8_t* flags, int32_t* level, int64_t* counters) {
  if (!p || !c || !c->center_speed) return fail(EIK_ERR_DOMAIN, "fmsm schedule: null argument");
  if (c->cells_x < 2 || c->cells_y < 2) return fail(EIK_ERR_CONFIG, "fmsm needs at least 2x2 cells");
  const int32_t cx = c->cells_x, cy = c->cells_y;
  const int64_t J = (int64_t)cx * cy;
  FmsmOrder ord;
  if (fmsm_part1(p, c, &ord)) return fail(EIK_ERR_CONFIG, "fmsm: empty coarse exit set");
  const int32_t* rk = ord.rank.data();
  for (int64_t y = 0, cell = 0; y < cy; ++y)
    for (int64_t x = 0; x < cx; ++x, ++cell) {
      uint8_t f = 16;
      if (!ord.is_q[cell]) {
        const int32_t r = rk[cell];
        f = fmsm_dir_mask(x > 0 && rk[cell - 1] < r, x + 1 < cx && rk[cell + 1] < r,
                          y > 0 && rk[cell - cx] < r, y + 1 < cy && rk[cell + cx] < r);
      }
      if (flags) flags[cell] = f;
    }
  if (level) {
    std::vector<int32_t> lv(J, 0);
    for (int64_t p2 = 0; p2 < J; ++p2) {  // rank order: predecessors first
      const int64_t cell = ord.order[p2], x = cell % cx, y = cell / cx;
      int32_t L = 0;
      const int32_t r = rk[cell];
      if (x > 0 && rk[cell - 1] < r) L = std::max(L, lv[cell - 1] + 1);
      if (x + 1 < cx && rk[cell + 1] < r) L = std::max(L, lv[cell + 1] + 1);
      if (y > 0 && rk[cell - cx] < r) L = std::max(L, lv[cell - cx] + 1);
      if (y + 1 < cy && rk[cell + cx] < r) L = std::max(L, lv[cell + cx] + 1);
      lv[cell] = L;
    }
    std::memcpy(level, lv.data(), sizeof(int32_t) * J);
  }
  if (order) std::memcpy(order, ord.order.data(), sizeof(int32_t) * J);
  if (rank) std::memcpy(rank, ord.rank.data(), sizeof(int32_t) * J);
  if (counters) {
    counters[0] = ord.coarse_pops;
    counters[1] = ord.coarse_updates;
  }
  return EIK_OK;
}

}  // namespace eikb200
