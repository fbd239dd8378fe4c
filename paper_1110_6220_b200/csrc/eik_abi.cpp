#include <chrono>
// Host runtime behind the C-ABI (include/eikonal_b200.h): argument checks
// with the reference's error semantics, device buffers, streams, dispatch to
// the sm_100a kernels, and SolverOutput packing.  No CPU solver lives here:
// every method either runs on the device or fails with EIK_ERR_NOT_IMPL /
// EIK_ERR_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "eik_internal.h"
#include "eik_plan.h"
#include "eikonal_b200.h"

namespace eikb200 {

namespace {
constexpr double kInfHost = __builtin_huge_val();
// Concurrent plans (eik_plan_run_batch) run best with one hardware work queue
// per stream (CUDA_DEVICE_MAX_CONNECTIONS=32): with the driver's default of 8,
// streams share queues and a solve can wait behind another stream's
// persistent kernel.  The library does not touch the process environment;
// the caller exports it before CUDA initialises (bench.py does).
}  // namespace

namespace {
Knobs read_knobs() {
  Knobs k;
  auto gi = [](const char* n, int d) {
    const char* v = std::getenv(n);
    return v ? std::atoi(v) : d;
  };
  auto gd = [](const char* n, double d) {
    const char* v = std::getenv(n);
    return v ? std::atof(v) : d;
  };
  auto gb = [](const char* n) { return std::getenv(n) != nullptr; };
  k.fsm_noskip = gb("EIK_FSM_NOSKIP");
  static std::string trace_path;  // owned copy (the environment may change)
  trace_path = std::getenv("EIK_TRACE_FSM") ? std::getenv("EIK_TRACE_FSM") : "";
  k.fsm_trace = trace_path.empty() ? nullptr : trace_path.c_str();
  k.fsm_wpc = gi("EIK_FSM_WPC", 0);
  k.fsm_sb = gi("EIK_FSM_SB", 1);
  k.fsm_cont = gi("EIK_FSM_CONT", 1);
  k.fsm_sb_wait_div = gi("EIK_FSM_SB_WAIT_DIV", 1);
  k.fsm_start_ahead = std::max(0, gi("EIK_FSM_START_AHEAD", 12));
  k.hc_warps = gi("EIK_HC_WARPS", 0);
  k.hc_min_smem = std::getenv("EIK_HC_MIN_SMEM") ? std::atol(std::getenv("EIK_HC_MIN_SMEM")) : -1;
  k.hc_global_heap = gb("EIK_HC_GLOBAL_HEAP");
  k.hc_heap_cap = gi("EIK_HC_HEAP_CAP", 0);
  k.hc_chain = gi("EIK_HC_CHAIN", 1);
  k.hc_bands = gi("EIK_HC_BANDS", 1);
  k.tile_tma = gi("EIK_TILE_TMA", gi("EIK_FMSM_TMA", 1));
  k.hc_ctas = gi("EIK_HC_CTAS", 0);
  k.hc_debug = gb("EIK_HC_DEBUG");
  k.hc_profile = gb("EIK_HC_PROFILE");
  k.hc_idle_ns = gi("EIK_HC_IDLE_NS", 200);
  k.hc_first_min = gi("EIK_HC_FIRST_MIN", 2);
  k.hc_first_min_pool = gi("EIK_HC_FIRST_MIN_POOL", 256);
  k.hc_skip_from = gi("EIK_HC_SKIP_FROM", 1);
  k.batch_sms_scale = gd("EIK_BATCH_SMS_SCALE", 0.0);
  k.batch_fmsm_ctas = std::max(1, gi("EIK_BATCH_FMSM_CTAS", 16));
  k.batch_fmsm_prio = gd("EIK_BATCH_FMSM_PRIO", 0.5);
  k.batch_fixed_per_sm = gi("EIK_BATCH_FIXED_PER_SM", 0);
  k.batch_trace = gb("EIK_BATCH_TRACE");
  k.batch_timing = gb("EIK_BATCH_TIMING");
  k.batch_workers = gi("EIK_BATCH_WORKERS", 0);
  k.hcm_exact = gi("EIK_HCM_EXACT", 0);
  k.hcm_band = gd("EIK_HCM_BAND", 0.0);
  k.hcm_band_shrink = gi("EIK_HCM_BAND_SHRINK", 128);
  return k;
}
std::mutex g_knobs_mu;
Knobs g_knobs = read_knobs();
}  // namespace

const Knobs& knobs() { return g_knobs; }

namespace {
std::atomic<int> g_hcm_mode{-1};  // -1: not set by eik_set_hcm_mode, use the knob
}  // namespace
int hcm_default_mode() {
  const int m = g_hcm_mode.load();
  return m >= 0 ? m : (knobs().hcm_exact ? 1 : 0);
}
void reload_knobs() {
  std::lock_guard<std::mutex> lk(g_knobs_mu);
  g_knobs = read_knobs();
}

thread_local SlowCall t_slow;
double now_ms_host() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

cudaError_t stream_wait(cudaStream_t s) {
  for (int i = 0;; ++i) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e != cudaErrorNotReady) return e;
    if (i < 32) std::this_thread::yield();
    else std::this_thread::sleep_for(std::chrono::microseconds(i < 256 ? 5 : 20));
  }
}

thread_local std::string g_last_error;
thread_local int g_last_code = EIK_OK;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  g_last_code = code;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(EIK_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

namespace {

int check_problem(const eik_problem* p) {
  if (!p) return fail(EIK_ERR_DOMAIN, "null problem");
  const eik_grid& g = p->grid;
  // Grid::Grid (grid.cpp:8-12)
  if (g.m < 2 || g.n < 2) return fail(EIK_ERR_CONFIG, "grid needs at least 2 nodes per axis");
  if (!(g.h > 0.0)) return fail(EIK_ERR_CONFIG, "grid spacing must be positive");
  if (!p->speed) return fail(EIK_ERR_DOMAIN, "null speed array");
  // build_problem (grid.cpp:77)
  if (p->n_exit < 1 || !p->exit_nodes || !p->exit_cost)
    return fail(EIK_ERR_CONFIG, "exit set is empty");
  const int64_t M = g.m * g.n;
  for (int64_t k = 0; k < p->n_exit; ++k) {
    if (p->exit_nodes[k] < 0 || p->exit_nodes[k] >= M)
      return fail(EIK_ERR_CONFIG, "exit node outside grid");
    if (k > 0 && p->exit_nodes[k] <= p->exit_nodes[k - 1])
      return fail(EIK_ERR_DOMAIN, "exit nodes must be strictly ascending");
    if (!std::isfinite(p->exit_cost[k])) return fail(EIK_ERR_CONFIG, "exit cost must be finite");
    // The reference accepts any finite cost (grid.cpp:70); the device path
    // orders values by their bit patterns (heap-cell queues) and carries the
    // FSM strip hand-off's change flag in the sign bit, both of which need
    // values >= 0, so negative costs are refused instead of solved wrongly.
    if (p->exit_cost[k] < 0.0)
      return fail(EIK_ERR_DOMAIN, "negative exit costs are not supported on the device path");
  }
  if (p->n_exit_points < 0 || (p->n_exit_points > 0 && (!p->exit_points_xy || !p->exit_point_cost)))
    return fail(EIK_ERR_DOMAIN, "bad exit point list");
  return EIK_OK;
}

int check_cells(const eik_problem* p, const eik_cells* c, int method) {
  const bool hybrid = method == EIK_HCM || method == EIK_FHCM || method == EIK_FMSM ||
                      method == EIK_HCM_EXACT;
  if (!hybrid) return EIK_OK;
  if (!c) return fail(EIK_ERR_CONFIG, "two-scale methods need a cell decomposition");
  // build_cells (cells.cpp:33-36)
  if (c->cells_x < 1 || c->cells_y < 1) return fail(EIK_ERR_CONFIG, "cell counts must be positive");
  if (c->cells_x > p->grid.m || c->cells_y > p->grid.n)
    return fail(EIK_ERR_CONFIG, "more cells than grid nodes along an axis");
  if (method == EIK_FMSM) {
    if (c->cells_x < 2 || c->cells_y < 2) return fail(EIK_ERR_CONFIG, "fmsm needs at least 2x2 cells");
    if (!c->center_speed) return fail(EIK_ERR_DOMAIN, "fmsm needs center_speed");
  } else {
    if (!c->probe_speed_w || !c->probe_speed_e || !c->probe_speed_s || !c->probe_speed_n)
      return fail(EIK_ERR_DOMAIN, "hcm/fhcm need the four probe_speed tables");
  }
  return EIK_OK;
}

}  // namespace

// ---- device buffer cache ------------------------------------------------
namespace {
std::mutex g_pool_mu;
std::atomic<long long> g_malloc_calls{0}, g_malloc_us{0}, g_free_calls{0};
std::map<std::pair<int, size_t>, std::vector<void*>> g_pool_free;  // (device, bytes)
std::map<void*, std::pair<int, size_t>> g_pool_live;
size_t g_pool_cached = 0;
// cached bytes kept at most: 40 % of the device (72 GB on a B200), at least
// 32 GB -- enough that a benchmark's resident plans return to the cache
// without driver frees
size_t pool_cap() {
  static size_t cap = [] {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
      cudaGetLastError();
      tot = 0;
    }
    return std::max<size_t>(size_t(32) << 30, tot / 10 * 4);
  }();
  return cap;
}
// Cache misses allocate from a per-device stream-ordered memory pool
// (cudaMallocFromPoolAsync on the allocating plan's stream, release threshold
// unlimited): cudaMalloc can block until kernels running on OTHER streams end,
// which stalled eik_solve_batch's plan creation behind the persistent solves
// of earlier jobs (measured: 438 cudaMalloc calls, 22 s blocked, over a
// 20-step batch).
cudaMemPool_t device_pool(int dev) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lk(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
    cudaGetLastError();
    pool = nullptr;
  } else {
    unsigned long long thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  pools[dev] = pool;
  return pool;
}
thread_local cudaStream_t t_alloc_stream = nullptr;
}  // namespace

AllocStream::AllocStream(cudaStream_t s) : prev_(t_alloc_stream) { t_alloc_stream = s; }
AllocStream::~AllocStream() { t_alloc_stream = prev_; }

cudaError_t pool_alloc(void** p, size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_pool_free.find({dev, bytes});
    if (it != g_pool_free.end() && !it->second.empty()) {
      *p = it->second.back();
      it->second.pop_back();
      g_pool_cached -= bytes;
      g_pool_live[*p] = {dev, bytes};
      return cudaSuccess;
    }
  }
  const auto tm0 = std::chrono::steady_clock::now();
  cudaMemPool_t pool = t_alloc_stream ? device_pool(dev) : nullptr;
  e = pool ? cudaMallocFromPoolAsync(p, bytes, pool, t_alloc_stream) : cudaMalloc(p, bytes);
  g_malloc_calls.fetch_add(1);
  g_malloc_us.fetch_add((long long)std::chrono::duration<double, std::micro>(
                            std::chrono::steady_clock::now() - tm0).count());
  if (e == cudaErrorMemoryAllocation) {  // give the cache back and retry once
    eik_release_cached();
    cudaGetLastError();
    e = pool ? cudaMallocFromPoolAsync(p, bytes, pool, t_alloc_stream) : cudaMalloc(p, bytes);
  }
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_pool_live[*p] = {dev, bytes};
  return cudaSuccess;
}

void pool_release(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  auto it = g_pool_live.find(p);
  if (it == g_pool_live.end()) return;
  const auto key = it->second;
  g_pool_live.erase(it);
  if (g_pool_cached + key.second > pool_cap()) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(key.first);
    cudaFree(p);
    g_free_calls.fetch_add(1);
    cudaSetDevice(cur);
    return;
  }
  g_pool_free[key].push_back(p);
  g_pool_cached += key.second;
}

cudaError_t ensure_dynamic_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> set;  // (device, kernel) -> limit
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = set[{dev, kernel}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

// fmm_solve's counters (classic_solvers.cpp:40-43,64-90): every non-exit
// node adjacent to an exit is evaluated once at initialisation, and every
// edge between two non-exit nodes once, when its first end is accepted; no
// sweeps.  Independent of the acceptance order.
int64_t fmm_node_updates(const eik_grid& g, const int64_t* ex, int64_t ne) {
  const int64_t m = g.m, n = g.n;
  auto is_exit = [&](int64_t idx) { return std::binary_search(ex, ex + ne, idx); };
  int64_t exit_edges = 0, exit_exit = 0;
  std::vector<int64_t> adj;
  adj.reserve((size_t)ne * 4);
  for (int64_t k = 0; k < ne; ++k) {
    const int64_t i = ex[k] % m, j = ex[k] / m;
    const int64_t nb[4] = {i + 1 < m ? ex[k] + 1 : -1, i > 0 ? ex[k] - 1 : -1,
                           j + 1 < n ? ex[k] + m : -1, j > 0 ? ex[k] - m : -1};
    for (int d = 0; d < 4; ++d) {
      if (nb[d] < 0) continue;
      ++exit_edges;
      if (is_exit(nb[d])) ++exit_exit;  // counted from both ends
      else adj.push_back(nb[d]);
    }
  }
  std::sort(adj.begin(), adj.end());
  const int64_t n_adj = std::unique(adj.begin(), adj.end()) - adj.begin();
  const int64_t edges = (m - 1) * n + m * (n - 1);
  return edges - (exit_edges - exit_exit / 2) + n_adj;
}

int solve_multi(const eik_problem* p, int32_t method, const int32_t* devices, int32_t n_dev,
                eik_output* out);

int plan_capacity(eik_plan* P, int* device, int* fixed) {
  CK(cudaSetDevice(P->device));
  *fixed = 0;
  switch (P->method) {
    case EIK_FSM:
    case EIK_FMM:
    case EIK_LSM:
      CK(fsm_capacity(P->nstrips, fixed, device, P->method == EIK_LSM));
      break;
    case EIK_FMSM:
      CK(fmsm_capacity(P->cg.tile_doubles, P->warps_per_cta, device));
      break;
    case EIK_HCM:
    case EIK_FHCM:
      if (P->cells_big) {  // one warp: the serial heap loop
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->device));
        *device = sms;
        break;
      }
      if (P->method == EIK_HCM && P->hcm_band) {
        CK(hcm_band_capacity(P->cg.tile_doubles, P->hc_warps_per_cta, (size_t)P->hc_min_smem,
                             device));
        break;
      }
      [[fallthrough]];
    default:
      CK(heapcell_capacity(P->cg.tile_doubles, P->hc_heap_cap, P->hc_warps_per_cta,
                           (size_t)P->hc_min_smem, device));
  }
  return EIK_OK;
}

void plan_free(eik_plan* P) {
  if (!P) return;
  if (P->stream) cudaStreamSynchronize(P->stream);  // nothing in flight on reused blocks
  for (void* ptr : P->allocs) pool_release(ptr);
  if (P->own_events) {
    if (P->ev0) cudaEventDestroy(P->ev0);
    if (P->ev1) cudaEventDestroy(P->ev1);
  }
  if (P->stream && P->own_stream) cudaStreamDestroy(P->stream);
  delete P;
}

int plan_init(eik_plan* P, const eik_problem* p, const eik_cells* c, int method,
              bool defer_upload = false, cudaStream_t ext_stream = nullptr,
              const cudaEvent_t* ext_events = nullptr) {
  P->hcm_exact_req = method == EIK_HCM_EXACT;
  if (method == EIK_HCM_EXACT) method = EIK_HCM;
  P->method = method;
  P->g = p->grid;
  P->M = p->grid.m * p->grid.n;
  P->n_exit = p->n_exit;
  CK(cudaGetDevice(&P->device));
  if (ext_stream) {
    P->stream = ext_stream;
    P->own_stream = false;
  } else {
    CK(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking));
  }
  AllocStream alloc_on(P->stream);  // cache misses: stream-ordered pool
  if (ext_events) {  // borrowed: event create/destroy can block behind running kernels
    P->ev0 = ext_events[0];
    P->ev1 = ext_events[1];
    P->own_events = false;
  } else {
    CK(cudaEventCreate(&P->ev0));
    CK(cudaEventCreate(&P->ev1));
  }
  auto track = [&](void* q) { P->allocs.push_back(q); };
  int rc;
  if ((rc = dalloc(&P->dF, P->M))) return rc;
  track(P->dF);
  // even pitch: 16-byte row strides (the FMSM tile loads' tensor maps need it)
  P->pitch = P->g.m + 2 * kPad + (P->g.m & 1);
  // rows -1 .. n (both dummies): dC / dU point at row 0
  const size_t padded = (size_t)(P->g.n + 2) * P->pitch;
  double* base = nullptr;
  if ((rc = dalloc(&base, padded))) return rc;
  track(base);
  P->dC = base + P->pitch;
  if ((rc = dalloc(&base, padded))) return rc;
  track(base);
  P->dU = base + P->pitch;
  if ((rc = dalloc(&P->dExit, P->n_exit))) return rc;
  track(P->dExit);
  if ((rc = dalloc(&P->dExitCost, P->n_exit))) return rc;
  track(P->dExitCost);
  if ((rc = dalloc(&P->dStatus, 8))) return rc;
  track(P->dStatus);
  P->deferred = defer_upload;
  if (defer_upload) {
    P->defer_F = p->speed;
    P->defer_F_dev = p->speed_on_device != 0;
  } else {
    CK(cudaMemcpyAsync(P->dF, p->speed, sizeof(double) * P->M,
                       p->speed_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       P->stream));
  }
  CK(cudaMemcpyAsync(P->dExit, p->exit_nodes, sizeof(int64_t) * P->n_exit,
                     cudaMemcpyHostToDevice, P->stream));
  CK(cudaMemcpyAsync(P->dExitCost, p->exit_cost, sizeof(double) * P->n_exit,
                     cudaMemcpyHostToDevice, P->stream));
  P->h2d_bytes = (p->speed_on_device ? 0 : 8 * P->M) + 16 * P->n_exit;
  if (method == EIK_FSM || method == EIK_FMM || method == EIK_LSM) {
    P->nstrips = (int)((P->g.n + 31) / 32);
    P->max_sweeps = 1 << 16;
    {  // every strip's warp must be resident (cooperative launch)
      int need = 0, ctas = 0;
      CK(fsm_capacity(P->nstrips, &need, &ctas, method == EIK_LSM));
      if (need > ctas)
        return fail(EIK_ERR_NOT_IMPL,
                    "grid has " + std::to_string(P->g.n) + " rows: one device's FSM wavefront "
                    "holds " + std::to_string(ctas) + " CTAs (" + std::to_string(need) +
                    " needed); shard the rows across devices (distributed.fsm_solve_strips)");
    }
    if (method == EIK_FMM) P->fmm_updates = fmm_node_updates(P->g, p->exit_nodes, p->n_exit);
    if (method == EIK_LSM) {
      if ((rc = dalloc(&P->dLsmCnt, P->max_sweeps))) return rc;
      track(P->dLsmCnt);
      CK(cudaMemsetAsync(P->dLsmCnt, 0, sizeof(unsigned long long) * P->max_sweeps, P->stream));
    }
    if ((rc = dalloc(&P->dProg, P->nstrips))) return rc;
    track(P->dProg);
    if ((rc = dalloc(&P->dMbox, (size_t)2 * P->nstrips * P->pitch))) return rc;
    track(P->dMbox);
    if ((rc = dalloc(&P->dChanged, P->max_sweeps))) return rc;
    track(P->dChanged);
    if ((rc = dalloc(&P->dDone, P->max_sweeps))) return rc;
    track(P->dDone);
    // change bits: zeroed once; every sweep rewrites every word of a real row
    // and nothing ever writes a nonzero bit into the pad rows/words
    P->chg_cw = (P->g.m + 31) / 32 + kChgWordPad;
    const size_t nchg = (size_t)2 * (P->g.n + 3) * P->chg_cw;
    if ((rc = dalloc(&P->dChg, nchg))) return rc;
    track(P->dChg);
    CK(cudaMemsetAsync(P->dChg, 0, sizeof(unsigned) * nchg, P->stream));
    P->nsb = fsm_nsb(P->g.m);
    if ((rc = dalloc(&P->dSb, (size_t)4 * P->nstrips * P->nsb + P->nstrips))) return rc;
    track(P->dSb);
  } else {
    if ((rc = plan_init_cells(P, p, c))) return rc;
  }
  const auto ts0 = std::chrono::steady_clock::now();
  CK(stream_wait(P->stream));
  P->init_sync_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ts0).count();
  return EIK_OK;
}

int plan_run_fsm(eik_plan* P, eik_output* out) {
  FsmArgs a;
  a.C = P->dC;
  a.u = P->dU;
  a.m = P->g.m;
  a.n = P->g.n;
  a.P = P->pitch;
  a.pad = kPad;
  a.nstrips = P->nstrips;
  a.prog = P->dProg;
  a.mbox = P->dMbox;
  a.changed = P->dChanged;
  a.done = P->dDone;
  a.max_sweeps = P->max_sweeps;
  a.lookahead = 3;
  a.first_sweep = 0;
  a.fixed = 0;
  a.status = P->dStatus;
  a.trace = nullptr;
  a.chg = P->dChg;
  a.cw = P->chg_cw;
  a.noskip = knobs().fsm_noskip ? 1 : 0;
  a.part_strips = 0;
  a.snap = nullptr;
  a.lsm_cnt = P->method == EIK_LSM ? P->dLsmCnt : nullptr;
  a.sb = (knobs().fsm_sb && P->nsb <= kFsmSbMaxPerRow) ? P->dSb : nullptr;
  a.nsb = P->nsb;
  a.sb_wait_div = knobs().fsm_sb_wait_div;
  a.start_ahead = knobs().fsm_start_ahead;
  a.cont = 0;
  a.par0 = 0;
  P->chg_valid = false;  // a later sweep-level launch starts from scratch
  if (P->part_strips > 0 && P->part_strips < P->nstrips) {
    const int nb = (P->nstrips - 1) / P->part_strips;
    const int64_t need = (int64_t)2 * nb * 2 * P->pitch;
    if (need > P->snap_count) {
      if (P->dSnap) {
        pool_release(P->dSnap);
        P->allocs.erase(std::find(P->allocs.begin(), P->allocs.end(), (void*)P->dSnap));
        P->dSnap = nullptr;
      }
      int rc = dalloc(&P->dSnap, (size_t)need);
      if (rc) return rc;
      P->allocs.push_back(P->dSnap);
      P->snap_count = need;
    }
    a.part_strips = P->part_strips;
    a.snap = P->dSnap;
    a.sb = nullptr;  // part edges exchange snapshot rows every block
  }
  if (knobs().fsm_trace) {
    if (!P->dTrace) {
      int rc = dalloc(&P->dTrace, (size_t)kTraceSweeps * P->nstrips * kTraceWords);
      if (rc) return rc;
      P->allocs.push_back(P->dTrace);
    }
    CK(cudaMemsetAsync(P->dTrace, 0, sizeof(unsigned long long) * kTraceSweeps * P->nstrips * kTraceWords,
                       P->stream));
    a.trace = P->dTrace;
  }
  int launches = 0;
  CK(cudaEventRecord(P->ev0, P->stream));
  CK(cudaMemsetAsync(P->dProg, 0, sizeof(unsigned long long) * P->nstrips, P->stream));
  CK(cudaMemsetAsync(P->dMbox, 0xFF, sizeof(double) * 2 * P->nstrips * P->pitch, P->stream));
  if (a.sb) CK(cudaMemsetAsync(P->dSb, 0, sizeof(unsigned) * 4 * P->nstrips * P->nsb, P->stream));
  // only the sweeps that can run need clearing; bound by the previous run
  size_t clear = (size_t)std::min<int64_t>(P->max_sweeps, P->last_sweeps_bound);
  CK(cudaMemsetAsync(P->dChanged, 0, sizeof(int) * clear, P->stream));
  CK(cudaMemsetAsync(P->dDone, 0, sizeof(int) * clear, P->stream));
  if (a.lsm_cnt)
    CK(cudaMemsetAsync(P->dLsmCnt, 0, sizeof(unsigned long long) * clear, P->stream));
  CK(launch_prepare(P->dF, P->dC, P->dU, P->g.m, P->g.n, P->pitch, kPad, P->g.h, P->dExit,
                    P->dExitCost, P->n_exit, P->dStatus, P->stream, &launches));
  if (a.part_strips > 0)  // part edges read +inf before the first exchange
    CK(launch_fill(a.snap, P->snap_count, kInfHost, P->stream, &launches));
  int grid = 0;
  CK(launch_fsm(a, P->stream, &launches, &grid));
  out->grid_ctas = grid;
  CK(cudaEventRecord(P->ev1, P->stream));
  int st[8];
  CK(stream_wait(P->stream));  // no spinning core while the solve runs
  CK(cudaMemcpyAsync(st, P->dStatus, sizeof(st), cudaMemcpyDeviceToHost, P->stream));
  CK(stream_wait(P->stream));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, P->ev0, P->ev1));
  if (st[0] != 0) P->last_sweeps_bound = P->max_sweeps;  // flags of a failed run: clear all
  if (st[0] == 1) return fail(EIK_ERR_DOMAIN, "speed must be positive and finite, and h / F within [2^-480, 2^500], at every node");
  if (st[0] == 3) return fail(EIK_ERR_BUDGET, "fsm exceeded the device sweep budget");
  if (st[0] == 4) return fail(EIK_ERR_CUDA, "fsm wavefront watchdog fired (scheduling bug)");
  P->last_sweeps_bound = std::min<int64_t>(P->max_sweeps, (int64_t)st[1] + 8);
  out->sweeps = st[1];
  out->node_updates = (int64_t)st[1] * (P->M - P->n_exit);
  out->heap_removals = 0;
  if (P->method == EIK_FMM) {
    // The FMM row is served by the exact fixed-point solver (SURVEY.md §8f
    // row 1) and reports fmm_solve's own counters: accepted nodes M - |Q|
    // (classic_solvers.cpp:67-69), candidate evaluations (plan_init), no sweeps.
    out->heap_removals = P->M - P->n_exit;
    out->node_updates = P->fmm_updates;
    out->sweeps = 0;
  } else if (P->method == EIK_LSM) {
    // lsm_solve's node_updates: nodes processed unlocked, summed over the
    // reference's sweeps (the pipelined wavefront may run a few more)
    std::vector<unsigned long long> cnt((size_t)st[1]);
    CK(cudaMemcpyAsync(cnt.data(), P->dLsmCnt, sizeof(unsigned long long) * cnt.size(),
                       cudaMemcpyDeviceToHost, P->stream));
    CK(stream_wait(P->stream));
    int64_t tot = 0;
    for (unsigned long long c : cnt) tot += (int64_t)c;
    out->node_updates = tot;
  }
  out->device_ms = ms;
  out->kernel_launches = launches;
  if (a.trace) {
    std::vector<unsigned long long> tr((size_t)kTraceSweeps * P->nstrips * kTraceWords);
    CK(cudaMemcpy(tr.data(), a.trace, sizeof(unsigned long long) * tr.size(),
                  cudaMemcpyDeviceToHost));
    const char* path = knobs().fsm_trace;
    if (FILE* f = std::fopen(path, "w")) {
      for (int k = 0; k < kTraceSweeps; ++k)
        for (int b = 0; b < P->nstrips; ++b) {
          const unsigned long long* t = &tr[((size_t)k * P->nstrips + b) * kTraceWords];
          if (t[0])
            std::fprintf(f, "%d %d %llu %llu %llu %llu %llu %llu %llu %llu\n", k, b, t[0], t[1], t[2],
                         t[3], t[4], t[5], t[6], t[7]);
        }
      std::fclose(f);
    }
  }
  return EIK_OK;
}

int plan_run(eik_plan* P, eik_output* out) {
  if (!out) return fail(EIK_ERR_DOMAIN, "null output");
  CK(cudaSetDevice(P->device));
  out->sweeps = out->node_updates = out->heap_removals = 0;
  out->cell_removals = out->cell_sweeps = out->mon_checks = out->mon_single = 0;
  out->avhr = out->avs = out->mon_pct = 0.0;
  out->host_ms = 0.0;
  out->spec_hits = out->spec_waits = out->spec_self = 0;
  out->grid_ctas = 0;
  out->rounds = 0;
  CK(cudaMemsetAsync(P->dStatus, 0, sizeof(int) * 8, P->stream));
  if (P->defer_F) {  // created by eik_solve_batch: the field goes up now
    CK(cudaMemcpyAsync(P->dF, P->defer_F, sizeof(double) * P->M,
                       P->defer_F_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       P->stream));
    P->defer_F = nullptr;
  }
  for (int s = 0; s < 4; ++s)
    if (P->defer_probe[s]) {
      CK(cudaMemcpyAsync(P->dProbe[s], P->defer_probe[s], sizeof(double) * P->probe_len[s],
                         cudaMemcpyHostToDevice, P->stream));
      P->defer_probe[s] = nullptr;
    }
  int rc;
  switch (P->method) {
    case EIK_FSM:
    case EIK_FMM:
    case EIK_LSM:
      rc = plan_run_fsm(P, out);
      break;
    case EIK_FMSM:
      rc = plan_run_fmsm(P, out);
      break;
    case EIK_HCM:
    case EIK_FHCM:
      rc = plan_run_heapcell(P, out);
      break;
    default:
      return fail(EIK_ERR_NOT_IMPL, "method not implemented on the device path");
  }
  if (rc) return rc;
  P->last_ms = out->device_ms + out->host_ms;
  P->ran = true;
  if (out->u) {
    // padded device layout -> caller's dense row-major m*n field
    CK(cudaMemcpy2DAsync(out->u, sizeof(double) * P->g.m, P->dU + kPad,
                         sizeof(double) * P->pitch, sizeof(double) * P->g.m, P->g.n,
                         out->u_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                         P->stream));
    CK(stream_wait(P->stream));
  }
  return EIK_OK;
}

// ---- sweep-level control of FSM plans (strip-Jacobi FSM across GPUs) ----
int plan_prepare(eik_plan* P) {
  if (P->method != EIK_FSM && P->method != EIK_FMM)
    return fail(EIK_ERR_CONFIG, "sweep-level control needs an fsm/fmm plan");
  CK(cudaSetDevice(P->device));
  CK(cudaMemsetAsync(P->dStatus, 0, sizeof(int) * 8, P->stream));
  P->chg_valid = false;  // fresh values: the next sweep launch evaluates every node
  int launches = 0;
  CK(launch_prepare(P->dF, P->dC, P->dU, P->g.m, P->g.n, P->pitch, kPad, P->g.h, P->dExit,
                    P->dExitCost, P->n_exit, P->dStatus, P->stream, &launches));
  int st[8];
  CK(stream_wait(P->stream));  // no spinning core while the solve runs
  CK(cudaMemcpyAsync(st, P->dStatus, sizeof(st), cudaMemcpyDeviceToHost, P->stream));
  CK(stream_wait(P->stream));
  if (st[0] == 1) return fail(EIK_ERR_DOMAIN, "speed must be positive and finite, and h / F within [2^-480, 2^500], at every node");
  return EIK_OK;
}

// sync: read the flags back (changed) and check the watchdog; async: leave
// them in device memory (changed_dev) on `stream`, the caller reads them later
int plan_sweep_impl(eik_plan* P, int64_t first_sweep, int count, int* changed, int* changed_dev,
                    cudaStream_t stream) {
  if (P->method != EIK_FSM && P->method != EIK_FMM)
    return fail(EIK_ERR_CONFIG, "sweep-level control needs an fsm/fmm plan");
  if (count < 1 || count > P->max_sweeps || first_sweep < 0)
    return fail(EIK_ERR_CONFIG, "sweep count out of range");
  CK(cudaSetDevice(P->device));
  FsmArgs a;
  a.C = P->dC;
  a.u = P->dU;
  a.m = P->g.m;
  a.n = P->g.n;
  a.P = P->pitch;
  a.pad = kPad;
  a.nstrips = P->nstrips;
  a.prog = P->dProg;
  a.mbox = P->dMbox;
  a.changed = P->dChanged;
  a.done = P->dDone;
  a.max_sweeps = count;
  a.lookahead = 3;
  a.first_sweep = (int)(first_sweep & 3);
  a.fixed = 1;
  a.status = P->dStatus;
  a.trace = nullptr;
  a.chg = P->dChg;
  a.cw = P->chg_cw;
  a.noskip = knobs().fsm_noskip ? 1 : 0;
  a.part_strips = 0;  // sweep-level control is one Gauss-Seidel wavefront
  a.snap = nullptr;
  a.lsm_cnt = nullptr;
  a.sb = (knobs().fsm_sb && P->nsb <= kFsmSbMaxPerRow) ? P->dSb : nullptr;
  a.nsb = P->nsb;
  a.sb_wait_div = knobs().fsm_sb_wait_div;
  a.start_ahead = knobs().fsm_start_ahead;
  // A launch that follows another sweep launch on the same values continues
  // from its change bits (rows written in between were marked, plan_rows):
  // only the first launch after eik_plan_prepare evaluates every node.
  a.cont = (P->chg_valid && knobs().fsm_cont) ? 1 : 0;
  a.par0 = a.cont ? ((P->chg_last_par + 1) & 1) : 0;
  P->chg_last_par = (count - 1 + a.par0) & 1;
  P->chg_valid = true;
  // the flags this call leaves in [0, count) must be cleared by a later run
  P->last_sweeps_bound = std::min<int64_t>(P->max_sweeps,
                                           std::max<int64_t>(P->last_sweeps_bound, count + 8));
  int launches = 0;
  const cudaStream_t s = stream ? stream : P->stream;
  if (!changed_dev) CK(cudaMemsetAsync(P->dStatus, 0, sizeof(int) * 8, s));
  CK(cudaMemsetAsync(P->dProg, 0, sizeof(unsigned long long) * P->nstrips, s));
  CK(cudaMemsetAsync(P->dMbox, 0xFF, sizeof(double) * 2 * P->nstrips * P->pitch, s));
  if (a.sb) {  // edge tokens always; the summaries only when nothing carries over
    const size_t half = (size_t)2 * P->nstrips * P->nsb;
    if (a.cont) CK(cudaMemsetAsync(P->dSb + half, 0, sizeof(unsigned) * half, s));
    else CK(cudaMemsetAsync(P->dSb, 0, sizeof(unsigned) * (2 * half + P->nstrips), s));
  }
  CK(cudaMemsetAsync(P->dChanged, 0, sizeof(int) * count, s));
  CK(cudaMemsetAsync(P->dDone, 0, sizeof(int) * count, s));
  CK(launch_fsm(a, s, &launches));
  if (changed_dev) {  // stream-ordered: no host synchronisation
    CK(cudaMemcpyAsync(changed_dev, P->dChanged, sizeof(int) * count, cudaMemcpyDeviceToDevice, s));
    return EIK_OK;
  }
  int st[8];
  std::vector<int> ch((size_t)count);
  CK(stream_wait(P->stream));  // no spinning core while the solve runs
  CK(cudaMemcpyAsync(st, P->dStatus, sizeof(st), cudaMemcpyDeviceToHost, P->stream));
  CK(cudaMemcpyAsync(ch.data(), P->dChanged, sizeof(int) * count, cudaMemcpyDeviceToHost,
                     P->stream));
  CK(stream_wait(P->stream));
  if (st[0] == 4) return fail(EIK_ERR_CUDA, "fsm wavefront watchdog fired (scheduling bug)");
  if (changed)
    for (int k = 0; k < count; ++k) changed[k] = ch[k] != 0;
  return EIK_OK;
}

int plan_sweep(eik_plan* P, int64_t first_sweep, int count, int* changed) {
  return plan_sweep_impl(P, first_sweep, count, changed, nullptr, nullptr);
}

int plan_rows(eik_plan* P, int64_t row0, int64_t nrows, double* host_or_dev, int on_device,
              bool to_plan) {
  if (row0 < 0 || nrows < 0 || row0 + nrows > P->g.n)
    return fail(EIK_ERR_CONFIG, "row range outside the grid");
  if (nrows == 0) return EIK_OK;
  if (!host_or_dev) return fail(EIK_ERR_DOMAIN, "null row buffer");
  CK(cudaSetDevice(P->device));
  double* dev = P->dU + row0 * P->pitch + kPad;
  const size_t w = sizeof(double) * P->g.m, dp = sizeof(double) * P->pitch;
  if (to_plan && P->chg_valid && P->dChg) {
    // between sweep launches: mark what the new rows change (k_fsm.cu)
    double* stage = nullptr;
    const double* src = host_or_dev;
    cudaError_t e = cudaSuccess;
    if (!on_device) {
      CK(pool_alloc((void**)&stage, w * nrows));
      e = cudaMemcpyAsync(stage, host_or_dev, w * nrows, cudaMemcpyHostToDevice, P->stream);
      src = stage;
    }
    if (e == cudaSuccess)
      e = launch_set_rows_marked(P->dU, src, row0, nrows, P->g.m, P->pitch, kPad,
                                 P->dChg + (int64_t)P->chg_last_par * (P->g.n + 3) * P->chg_cw,
                                 P->chg_cw,
                                 P->dSb + (int64_t)P->chg_last_par * P->nstrips * P->nsb, P->nsb,
                                 P->stream);
    if (stage) {  // the staging buffer goes back whatever happened
      const cudaError_t es = cudaStreamSynchronize(P->stream);
      pool_release(stage);
      if (e == cudaSuccess) e = es;
    }
    CK(e);
  } else if (to_plan)
    CK(cudaMemcpy2DAsync(dev, dp, host_or_dev, w, w, nrows,
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, P->stream));
  else
    CK(cudaMemcpy2DAsync(host_or_dev, w, dev, dp, w, nrows,
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, P->stream));
  int st = 0;
  CK(stream_wait(P->stream));
  CK(cudaMemcpyAsync(&st, P->dStatus, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
  CK(stream_wait(P->stream));
  if (st == 4) return fail(EIK_ERR_CUDA, "fsm wavefront watchdog fired (scheduling bug)");
  return EIK_OK;
}

// stream-ordered row copies between the plan and a device buffer (dense
// m-wide rows), no host synchronisation
int plan_rows_async(eik_plan* P, int64_t row0, int64_t nrows, double* dev_buf, bool to_plan,
                    cudaStream_t stream) {
  if (row0 < 0 || nrows < 0 || row0 + nrows > P->g.n)
    return fail(EIK_ERR_CONFIG, "row range outside the grid");
  if (nrows == 0) return EIK_OK;
  if (!dev_buf) return fail(EIK_ERR_DOMAIN, "null row buffer");
  CK(cudaSetDevice(P->device));
  double* dev = P->dU + row0 * P->pitch + kPad;
  const size_t w = sizeof(double) * P->g.m, dp = sizeof(double) * P->pitch;
  const cudaStream_t s = stream ? stream : P->stream;
  if (to_plan && P->chg_valid && P->dChg)
    CK(launch_set_rows_marked(P->dU, dev_buf, row0, nrows, P->g.m, P->pitch, kPad,
                              P->dChg + (int64_t)P->chg_last_par * (P->g.n + 3) * P->chg_cw,
                              P->chg_cw,
                              P->dSb + (int64_t)P->chg_last_par * P->nstrips * P->nsb, P->nsb, s));
  else if (to_plan) CK(cudaMemcpy2DAsync(dev, dp, dev_buf, w, w, nrows, cudaMemcpyDeviceToDevice, s));
  else CK(cudaMemcpy2DAsync(dev_buf, w, dev, dp, w, nrows, cudaMemcpyDeviceToDevice, s));
  return EIK_OK;
}

// Device slices for plans sharing one GPU (eik_plan_run_batch), in SMs.
// Every persistent grid holds whole SMs: the heap-cell CTAs and the FSM
// strips (12 warps x 168 registers) fill an SM's register file, FMSM CTAs
// its shared memory.  A heap-cell replay is bound by its committer's serial
// chain once it has enough workers; more cells (more pops in flight) or
// fewer warps per SM (large cells) need more SMs to get there, and past that
// point SMs buy little (measured on C2: HCM/8 at 8/13/20/30 SMs
// 428/300/288/284 ms, HCM/64 313/265/234/212 ms, HCM/32 162/150/144/142 ms),
// so it asks for 2 J^(1/4) / sqrt(warps per CTA) SMs (EIK_BATCH_SMS_SCALE
// overrides the 2): the slice where SM-time per solve is near its minimum,
// which is what a schedule of many solves needs (C2, 3 steps: 2 -> 134 ms
// per step, 4 -> 190 ms; one step alone 332 vs 295 ms).  Admission order:
// heap-cell replays by that weight (larger first, HCM before FHCM), then the
// fixed grids, then FMSM -- measured better than ordering by the last run's
// time (170 ms per step).  FMSM dataflows (a few ms alone on the GPU) get 16
// CTAs: admitted last, they finish the schedule, and a short tail beats a
// small slice (2 CTAs: ~100 ms at 64-node cells, the step 6-8 % slower and
// twice as variable); fixed grids get what they need, capped plans their cap.
struct BatchSlot {
  int sms = 0;        // SMs the plan's grid holds while it runs
  double prio = 0.0;  // admission order
  bool hc = false;
};

int batch_slot(eik_plan* P, int sms, int budget, BatchSlot& b, double scale = 2.0) {
  const Knobs& kn = knobs();
  int dev = 0, fixed = 0;
  int rc = plan_capacity(P, &dev, &fixed);
  if (rc) return rc;
  if (dev < 1) return fail(EIK_ERR_CUDA, "batch: a kernel does not fit on the device");
  const int per_sm = std::max(1, dev / sms);
  b = BatchSlot{};
  P->run_cap = 0;
  if (fixed > 0) {
    const int pf = kn.batch_fixed_per_sm > 0 ? std::min(kn.batch_fixed_per_sm, per_sm) : per_sm;
    b.sms = (fixed + pf - 1) / pf;
    b.prio = 1.0;
  } else if (P->ctas_cap > 0) {
    b.sms = (std::min(P->ctas_cap, dev) + per_sm - 1) / per_sm;
    b.prio = 1.5;
    b.hc = P->method == EIK_HCM || P->method == EIK_FHCM;
  } else if (P->method == EIK_FMSM) {
    P->run_cap = kn.batch_fmsm_ctas;
    b.sms = kn.batch_fmsm_ctas;
    b.prio = kn.batch_fmsm_prio;
  } else {
    const double J = (double)P->cells_x * P->cells_y;
    const double w = std::pow(J, 0.25) / std::sqrt((double)std::max(1, P->hc_warps_per_cta));
    b.sms = std::max(2, (int)std::lround(scale * w));
    b.prio = 2.0 + w + (P->method == EIK_HCM ? 0.01 : 0.0);
    b.hc = true;
  }
  b.sms = std::min(b.sms, budget);
  if (P->run_cap == 0 && fixed == 0 && P->ctas_cap == 0) P->run_cap = b.sms * per_sm;
  return EIK_OK;
}

// Heap-cell slice scale for a batch: 2 J^(1/4)/sqrt(w) SMs per replay keeps
// the schedule's tail short when the batch is about one wave of the device;
// a batch of many waves is bound by total SM-time instead, which is lower on
// smaller slices (C2 matrix, 20 steps = 280 solves: scale 2 -> 891, 1 -> 1022
// M points/s; 3 steps: 2 -> 550, 1 -> 440).  `waves` = the batch's slices at
// scale 2 over the SM budget.  EIK_BATCH_SMS_SCALE > 0 overrides.
double batch_scale_for(double waves) {
  const double k = knobs().batch_sms_scale;
  if (k > 0.0) return k;
  return waves >= 8.0 ? 1.0 : 2.0;
}

int batch_slots(eik_plan* const* plans, int n, int budget, std::vector<BatchSlot>& slot) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, plans[0]->device));
  slot.assign(n, BatchSlot{});
  double total = 0.0;
  for (int k = 0; k < n; ++k) {
    int rc = batch_slot(plans[k], sms, budget, slot[k]);
    if (rc) return rc;
    total += slot[k].sms;
  }
  const double scale = batch_scale_for(total / budget);
  if (scale != 2.0)
    for (int k = 0; k < n; ++k) {
      int rc = batch_slot(plans[k], sms, budget, slot[k], scale);
      if (rc) return rc;
    }
  return EIK_OK;
}

// The same waves estimate before any plan exists (eik_solve_batch): slices
// from the problem shapes alone, heap-cell warps per CTA as plan_init_cells
// sizes them (k_heapcell.cu heapcell_smem_bytes).
double batch_waves_estimate(const eik_problem* const* problems, const eik_cells* const* cells,
                            const int32_t* methods, int n, int budget) {
  const Knobs& kn = knobs();
  double total = 0.0;
  for (int k = 0; k < n; ++k) {
    const int32_t m = methods[k];
    const eik_grid& g = problems[k]->grid;
    if (m == EIK_FMSM) {
      total += kn.batch_fmsm_ctas;
    } else if ((m == EIK_HCM || m == EIK_FHCM || m == EIK_HCM_EXACT) && cells && cells[k]) {
      const int64_t cx = cells[k]->cells_x, cy = cells[k]->cells_y;
      const int64_t bw = g.m / cx, bh = g.n / cy;
      const int64_t mw = g.m - (cx - 1) * bw, mh = g.n - (cy - 1) * bh;
      const int64_t pu = (mw + 4) & ~(int64_t)1, ml = std::max(mw, mh);
      const double bytes = 8.0 * (2.0 * (mh + 2) * pu + 8.0 * ml) + (double)mw * mh + 128.0;
      const double w = std::max(1.0, std::min(8.0, std::floor(216.0 * 1024 / bytes)));
      total += std::max(2.0, std::round(2.0 * std::pow((double)cx * cy, 0.25) / std::sqrt(w)));
    } else {
      total += std::max<int64_t>(1, (g.n + 32 * 12 - 1) / (32 * 12));  // FSM strips, 12 per SM
    }
  }
  return total / std::max(1, budget);
}

// Runs the plans as a list schedule: in order of priority, each plan starts
// (on its own host thread and stream) as soon as its SMs are free, later
// plans filling in behind one that does not fit yet; a plan ending returns
// its SMs.  Admitted heap-cell grids are submitted before the other
// admitted plans start, so their SM-exclusive CTAs find whole free SMs.
int plan_run_batch(eik_plan* const* plans, int n, eik_output* outs, double* batch_ms) {
  for (int k = 0; k < n; ++k) {
    if (!plans[k]) return fail(EIK_ERR_DOMAIN, "batch: null plan");
    for (int j = 0; j < k; ++j)
      if (plans[j] == plans[k]) return fail(EIK_ERR_DOMAIN, "batch: a plan appears twice");
    if (plans[k]->device != plans[0]->device)
      return fail(EIK_ERR_CONFIG, "batch: plans on different devices");
  }
  const int device = plans[0]->device;
  CK(cudaSetDevice(device));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const int budget = std::max(1, (int)std::floor(0.98 * sms));
  std::vector<BatchSlot> slot;
  int rc = batch_slots(plans, n, budget, slot);
  if (rc) return rc;
  std::vector<int> order(n);
  for (int k = 0; k < n; ++k) order[k] = k;
  std::stable_sort(order.begin(), order.end(),
                   [&](int x, int y) { return slot[x].prio > slot[y].prio; });
  CK(cudaDeviceSynchronize());
  cudaEvent_t ref;
  CK(cudaEventCreate(&ref));
  CK(cudaEventRecord(ref, plans[0]->stream));
  CK(cudaEventSynchronize(ref));
  std::vector<int> codes(n, EIK_OK);
  std::vector<std::string> msgs(n);
  {
    std::mutex mu;
    std::condition_variable cv;
    int free_sms = budget;
    int hc_launching = 0;               // admitted heap-cell plans not yet submitted
    std::vector<char> admitted(n, 0);
    auto admit = [&]() {                // under mu
      for (int k : order) {
        if (admitted[k] || slot[k].sms > free_sms) continue;
        admitted[k] = 1;
        free_sms -= slot[k].sms;
        if (slot[k].hc) ++hc_launching;
      }
      cv.notify_all();
    };
    {
      std::lock_guard<std::mutex> lk(mu);
      admit();
    }
    std::vector<std::thread> th;
    th.reserve(n);
    for (int k = 0; k < n; ++k) {
      eik_plan* P = plans[k];
      th.emplace_back([&, k, P]() {
        cudaSetDevice(device);
        const bool hc = slot[k].hc;
        // FMSM Part I runs before the plan waits for its SMs (a failure is
        // reported by plan_run, which calls it again)
        if (plan_prepare_host(P)) P->fmsm_ready = false;
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&]() { return admitted[k] && (hc || hc_launching == 0); });
        }
        bool signalled = !hc;
        auto launched = [&]() {
          std::lock_guard<std::mutex> lk(mu);
          if (--hc_launching == 0) cv.notify_all();
        };
        if (hc) P->on_launched = [&]() {
          signalled = true;
          launched();
        };
        codes[k] = plan_run(P, &outs[k]);
        if (codes[k]) msgs[k] = g_last_error;  // thread-local: carry it back
        P->on_launched = nullptr;
        if (!signalled) launched();            // failed before its launch
        std::lock_guard<std::mutex> lk(mu);
        free_sms += slot[k].sms;
        admit();
      });
    }
    for (auto& t : th) t.join();
  }
  for (int k = 0; k < n; ++k) plans[k]->run_cap = 0;
  double t_end = 0.0;
  cudaError_t e = cudaSuccess;
  const bool trace = knobs().batch_trace;
  for (int k = 0; k < n && e == cudaSuccess; ++k) {
    float ms = 0.f, ms0 = 0.f;
    if (codes[k] == EIK_OK) e = cudaEventElapsedTime(&ms, ref, plans[k]->ev1);
    if (trace && codes[k] == EIK_OK && cudaEventElapsedTime(&ms0, ref, plans[k]->ev0) == cudaSuccess)
      std::fprintf(stderr, "batch plan %d method %d ctas %lld sms %d: %.1f -> %.1f ms\n", k,
                   plans[k]->method, (long long)outs[k].grid_ctas, slot[k].sms, ms0, ms);
    t_end = std::max(t_end, (double)ms);
  }
  cudaEventDestroy(ref);
  for (int k = 0; k < n; ++k)
    if (codes[k]) return fail(codes[k], "batch plan " + std::to_string(k) + ": " + msgs[k]);
  if (e != cudaSuccess) return cuda_fail(e, "batch timing");
  if (batch_ms) *batch_ms = t_end;
  return EIK_OK;
}

eik_plan* plan_create(const eik_problem* p, const eik_cells* c, int32_t method, bool defer_upload,
                      cudaStream_t stream = nullptr, const cudaEvent_t* events = nullptr) {
  g_last_code = EIK_OK;
  g_last_error.clear();
  if (check_problem(p) || check_cells(p, c, method)) return nullptr;
  if (method < EIK_FMM || method > EIK_HCM_EXACT) {
    fail(EIK_ERR_CONFIG, "unknown method");
    return nullptr;
  }
  if (eik_device_count() < 1) {
    fail(EIK_ERR_CUDA, "no CUDA device visible: the Eikonal hot path has no CPU fallback");
    return nullptr;
  }
  eik_plan* P = new eik_plan();
  if (plan_init(P, p, c, method, defer_upload, stream, events)) {
    std::string keep = g_last_error;
    int keep_code = g_last_code;
    plan_free(P);
    g_last_error = keep;
    g_last_code = keep_code;
    return nullptr;
  }
  return P;
}

// eik_solve_batch: the same list schedule as plan_run_batch, but each
// solve's plan exists only while it is needed.  A fixed pool of worker
// threads (one stream each) takes the jobs in order; a worker creates the
// job's plan (device buffers from the pool cache, inputs uploaded from the
// caller's host arrays), waits until the schedule admits it (priority order
// among the created jobs, SMs free), runs it, downloads u, and returns the
// buffers before taking the next job.  Device memory and host threads are
// bounded by the pool size, not by the number of solves, and no buffer is
// allocated from the driver in steady state (the exact-size cache serves
// every plan after the first of its shape).
// Worker streams and events for eik_solve_batch, created once per process and
// reused by every call: creating or destroying an event while other kernels
// run blocks the calling thread until they end (measured: 0.1-1.6 s per
// cudaEventCreate inside a 20-step batch), so none is created on that path.
struct WorkerRes {
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
};
std::mutex g_wres_mu;
std::map<int, std::vector<WorkerRes>> g_wres_free;  // device -> idle resources

int take_worker_res(int device, int count, std::vector<WorkerRes>& out) {
  std::lock_guard<std::mutex> lk(g_wres_mu);
  auto& fl = g_wres_free[device];
  while ((int)out.size() < count) {
    if (!fl.empty()) {
      out.push_back(fl.back());
      fl.pop_back();
      continue;
    }
    WorkerRes r;
    CK(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&r.ev[0]));
    CK(cudaEventCreate(&r.ev[1]));
    out.push_back(r);
  }
  return EIK_OK;
}

void give_worker_res(int device, std::vector<WorkerRes>& res) {
  std::lock_guard<std::mutex> lk(g_wres_mu);
  for (auto& r : res) g_wres_free[device].push_back(r);
  res.clear();
}

int solve_batch_pipelined(const eik_problem* const* problems, const eik_cells* const* cells,
                          const int32_t* methods, int n, eik_output* outs, double* batch_ms) {
  int device = 0, sms = 0;
  CK(cudaGetDevice(&device));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const int budget = std::max(1, (int)std::floor(0.98 * sms));
  const Knobs& kn = knobs();
  const int workers = std::max(1, std::min(n, kn.batch_workers > 0 ? kn.batch_workers : 64));
  const double scale = batch_scale_for(batch_waves_estimate(problems, cells, methods, n, budget));
  struct Waiting {
    int k;
    BatchSlot b;
  };
  std::mutex mu;
  std::condition_variable cv;
  int next_job = 0, free_sms = budget, hc_launching = 0;
  // Plan creation (the uploads) in job order, kCreateWindow at a time: the
  // first jobs' inputs reach the device first instead of sharing the link with 64
  // workers' uploads (measured: the first heap-cell replays of a 20-step
  // batch admitted only after 50-170 ms).  create_prefix = jobs [0, prefix)
  // are created.
  constexpr int kCreateWindow = 8;
  int create_prefix = 0;
  std::vector<char> created(n, 0);  // by position in `order`
  // Jobs are taken in the schedule's admission order (batch_slot's
  // priorities, estimated from the shapes: heap-cell replays by weight, then
  // the fixed grids, then FMSM), so the long replays of every step upload and
  // start first, as in plan_run_batch where all plans exist up front.
  std::vector<int> order(n);
  {
    std::vector<double> prio(n, 1.0);
    for (int k = 0; k < n; ++k) {
      const int32_t m = methods[k];
      if (m == EIK_FMSM) {
        prio[k] = kn.batch_fmsm_prio;
      } else if ((m == EIK_HCM || m == EIK_FHCM || m == EIK_HCM_EXACT) && cells && cells[k]) {
        const double J = (double)cells[k]->cells_x * cells[k]->cells_y;
        prio[k] = 2.0 + std::pow(J, 0.25) + (m == EIK_FHCM ? 0.0 : 0.01);
      }
    }
    for (int k = 0; k < n; ++k) order[k] = k;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return prio[x] > prio[y]; });
  }
  bool abort = false;
  std::vector<Waiting> waiting;
  std::vector<char> admitted(n, 0);
  std::vector<int> codes(n, EIK_OK);
  std::vector<std::string> msgs(n);
  double t_end = 0.0;
  auto admit = [&]() {  // under mu: highest priority first, later ones fill in
    std::stable_sort(waiting.begin(), waiting.end(),
                     [](const Waiting& x, const Waiting& y) { return x.b.prio > y.b.prio; });
    for (size_t i = 0; i < waiting.size();) {
      if (waiting[i].b.sms <= free_sms) {
        admitted[waiting[i].k] = 1;
        free_sms -= waiting[i].b.sms;
        if (waiting[i].b.hc) ++hc_launching;
        waiting.erase(waiting.begin() + i);
      } else {
        ++i;
      }
    }
    cv.notify_all();
  };
  std::vector<WorkerRes> wres;
  {
    const int rc = take_worker_res(device, workers + 1, wres);  // +1: the reference event
    if (rc) {
      give_worker_res(device, wres);
      return rc;
    }
  }
  cudaEvent_t ref = wres[workers].ev[0];
  CK(cudaEventRecord(ref, wres[workers].stream));
  CK(cudaEventSynchronize(ref));
  std::atomic<int> next_worker{0};
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  auto now_ms = [&]() { return std::chrono::duration<double, std::milli>(clk::now() - t0).count(); };
  auto worker = [&]() {
    cudaSetDevice(device);
    const WorkerRes& wr = wres[next_worker.fetch_add(1)];
    cudaStream_t st = wr.stream;
    const cudaEvent_t* evs = wr.ev;
    for (;;) {
      int k, pos;
      {
        std::lock_guard<std::mutex> lk(mu);
        if (abort || next_job >= n) break;
        pos = next_job++;
        k = order[pos];
      }
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&]() { return abort || create_prefix >= pos - kCreateWindow + 1; });
        if (abort) break;
      }
      const double tc0 = now_ms();
      t_slow = SlowCall{};
      eik_plan* P = plan_create(problems[k], cells ? cells[k] : nullptr, methods[k], false, st, evs);
      const double tc1 = now_ms();
      {
        std::lock_guard<std::mutex> lk(mu);
        created[pos] = 1;
        while (create_prefix < n && created[create_prefix]) ++create_prefix;
        cv.notify_all();
      }
      const SlowCall slow_create = t_slow;
      t_slow = SlowCall{};
      BatchSlot b;
      int rc = P ? batch_slot(P, sms, budget, b, scale)
                 : (g_last_code != EIK_OK ? g_last_code : EIK_ERR_CUDA);
      if (!rc) rc = plan_prepare_host(P);  // FMSM Part I before the SMs are held
      if (rc) {
        codes[k] = rc;
        msgs[k] = g_last_error;
        plan_free(P);
        std::lock_guard<std::mutex> lk(mu);
        abort = true;
        cv.notify_all();
        break;
      }
      {
        std::unique_lock<std::mutex> lk(mu);
        waiting.push_back({k, b});
        admit();
        cv.wait(lk, [&]() { return abort || (admitted[k] && (b.hc || hc_launching == 0)); });
        if (!admitted[k]) {  // aborted while waiting
          waiting.erase(std::remove_if(waiting.begin(), waiting.end(),
                                       [&](const Waiting& w) { return w.k == k; }),
                        waiting.end());
          plan_free(P);
          break;
        }
      }
      const double ta = now_ms();
      bool signalled = !b.hc;
      auto launched = [&]() {
        std::lock_guard<std::mutex> lk(mu);
        if (--hc_launching == 0) cv.notify_all();
      };
      if (b.hc) P->on_launched = [&]() {
        signalled = true;
        launched();
      };
      codes[k] = plan_run(P, &outs[k]);
      const double tr = now_ms();
      const double init_sync = P->init_sync_ms;
      P->on_launched = nullptr;
      if (!signalled) launched();
      if (codes[k]) msgs[k] = g_last_error;
      float ms = 0.f;
      const bool timed = codes[k] == EIK_OK && cudaEventElapsedTime(&ms, ref, P->ev1) == cudaSuccess;
      const SlowCall slow_run = t_slow;
      const double tf0 = now_ms();
      double tsync = 0, tpool = 0, tev = 0, x;
      {  // plan_free, timed piecewise
        x = now_ms();
        stream_wait(P->stream);
        tsync = now_ms() - x;
        x = now_ms();
        for (void* ptr : P->allocs) pool_release(ptr);
        P->allocs.clear();
        tpool = now_ms() - x;
        x = now_ms();
        plan_free(P);
        tev = now_ms() - x;
      }
      if (kn.batch_trace)
        std::fprintf(stderr, "solve_batch job %d method %d sms %d: create %.1f-%.1f (sync %.1f; "
                     "slowest %s %.1f) admit %.1f run+download -%.1f (slowest %s %.1f) free %.1f "
                     "(sync %.1f pool %.1f rest %.1f) (device end %.1f) mallocs %lld\n", k,
                     methods[k], b.sms, tc0, tc1, init_sync, slow_create.what ? slow_create.what : "-",
                     slow_create.ms, ta, tr, slow_run.what ? slow_run.what : "-", slow_run.ms,
                     now_ms() - tf0, tsync, tpool, tev, ms, g_malloc_calls.load());
      else
        (void)tf0;
      std::lock_guard<std::mutex> lk(mu);
      if (timed) t_end = std::max(t_end, (double)ms);
      if (codes[k]) abort = true;
      free_sms += b.sms;
      admit();
    }
    stream_wait(st);
  };
  std::vector<std::thread> th;
  th.reserve(workers);
  for (int w = 0; w < workers; ++w) th.emplace_back(worker);
  for (auto& t : th) t.join();
  give_worker_res(device, wres);
  for (int k = 0; k < n; ++k)
    if (codes[k]) return fail(codes[k], "batch problem " + std::to_string(k) + ": " + msgs[k]);
  if (abort) return fail(EIK_ERR_CUDA, "batch: a worker could not start");
  if (batch_ms) *batch_ms = t_end;
  return EIK_OK;
}

}  // namespace eikb200

using namespace eikb200;

extern "C" {

int eik_abi_version(void) { return EIK_ABI_VERSION; }

void eik_debug_reload_knobs(void) { reload_knobs(); }

const char* eik_last_error(void) { return g_last_error.c_str(); }

int eik_last_status(void) { return g_last_code; }

int eik_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int eik_metrics(const double* u_method, const double* u_exact, const double* u_truth, int64_t m,
                int64_t n, const int64_t* exit_nodes, int64_t n_exit, int32_t on_device,
                eik_metrics_out* out) {
  g_last_code = EIK_OK;
  g_last_error.clear();
  if (!out || !u_method || !u_exact || !u_truth || m < 1 || n < 1 || n_exit < 0 ||
      (n_exit > 0 && !exit_nodes))
    return fail(EIK_ERR_DOMAIN, "eik_metrics: bad arguments");
  if (eik_device_count() < 1)
    return fail(EIK_ERR_CUDA, "no CUDA device visible: the Eikonal hot path has no CPU fallback");
  const int64_t M = m * n;
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  std::vector<void*> tmp;
  AllocStream alloc_on(s);
  auto cleanup = [&]() {
    cudaStreamSynchronize(s);
    for (void* q : tmp) pool_release(q);
    cudaStreamDestroy(s);
  };
  auto dev_copy = [&](const void* src, size_t bytes, void** dst) -> cudaError_t {
    cudaError_t e = pool_alloc(dst, bytes);
    if (e != cudaSuccess) return e;
    tmp.push_back(*dst);
    return cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, s);
  };
  const double *vm = u_method, *ve = u_exact, *vt = u_truth;
  cudaError_t e = cudaSuccess;
  if (!on_device) {
    void *a = nullptr, *b = nullptr, *c = nullptr;
    if ((e = dev_copy(u_method, 8 * M, &a)) == cudaSuccess &&
        (e = dev_copy(u_exact, 8 * M, &b)) == cudaSuccess &&
        (e = dev_copy(u_truth, 8 * M, &c)) == cudaSuccess) {
      vm = static_cast<const double*>(a);
      ve = static_cast<const double*>(b);
      vt = static_cast<const double*>(c);
    }
  }
  void* dex = nullptr;
  void* mask = nullptr;
  if (e == cudaSuccess && n_exit > 0) e = dev_copy(exit_nodes, 8 * n_exit, &dex);
  if (e == cudaSuccess && (e = pool_alloc(&mask, (size_t)M)) == cudaSuccess) tmp.push_back(mask);
  double res[5];
  long long cnt[2];
  if (e == cudaSuccess)
    e = device_metrics(vm, ve, vt, M, static_cast<const int64_t*>(dex), n_exit,
                       static_cast<uint8_t*>(mask), s, res, cnt);
  cleanup();
  if (e != cudaSuccess) return cuda_fail(e, "eik_metrics");
  out->l_inf = res[0];
  out->l_1 = res[1];
  out->max_error_ratio = res[2];
  out->avg_error_ratio = res[3];
  out->ratio_of_max = res[4];
  out->m_plus = cnt[0];
  out->x_plus_empty = (int32_t)cnt[1];
  return EIK_OK;
}

void eik_release_cached(void) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& kv : g_pool_free) {
    cudaSetDevice(kv.first.first);
    for (void* q : kv.second) cudaFree(q);
  }
  for (auto& kv : g_pool_free) {
    cudaMemPool_t pool = device_pool(kv.first.first);
    if (pool) cudaMemPoolTrimTo(pool, 0);
  }
  cudaSetDevice(cur);
  g_pool_free.clear();
  g_pool_cached = 0;
}

int eik_set_device(int32_t device) {
  int n = eik_device_count();
  if (device < 0 || device >= n) return fail(EIK_ERR_CONFIG, "no such CUDA device");
  CK(cudaSetDevice(device));
  return EIK_OK;
}


eik_plan* eik_plan_create(const eik_problem* p, const eik_cells* c, int32_t method) {
  return plan_create(p, c, method, false);
}

int eik_plan_run(eik_plan* P, eik_output* out) {
  if (!P) return fail(EIK_ERR_DOMAIN, "null plan");
  return plan_run(P, out);
}

const double* eik_plan_values(const eik_plan* P) { return P ? P->dU + kPad : nullptr; }

int64_t eik_plan_pitch(const eik_plan* P) { return P ? P->pitch : 0; }

void eik_plan_destroy(eik_plan* P) { plan_free(P); }

int eik_plan_acceptance_order(eik_plan* P, int32_t* order, int32_t on_device) {
  if (!P || !order) return fail(EIK_ERR_DOMAIN, "null argument");
  if (P->method != EIK_FMM) return fail(EIK_ERR_CONFIG, "acceptance order needs an fmm plan");
  if (!P->ran) return fail(EIK_ERR_CONFIG, "acceptance order: run the plan first");
  if (P->M > INT32_MAX) return fail(EIK_ERR_NOT_IMPL, "acceptance order: grid exceeds int32 indices");
  CK(cudaSetDevice(P->device));
  int32_t* dst = order;
  void* tmp = nullptr;
  if (!on_device) {
    CK(pool_alloc(&tmp, sizeof(int32_t) * P->M));
    dst = static_cast<int32_t*>(tmp);
  }
  cudaError_t e = device_acceptance_order(P->dU, P->dC, P->g.m, P->g.n, P->pitch, kPad, dst,
                                          P->stream);
  if (e == cudaSuccess && !on_device)
    e = cudaMemcpy(order, dst, sizeof(int32_t) * (P->M - P->n_exit), cudaMemcpyDeviceToHost);
  if (tmp) pool_release(tmp);
  if (e != cudaSuccess) return cuda_fail(e, "eik_plan_acceptance_order");
  return EIK_OK;
}

eik_plan* eik_plan_create_fmsm_strip(const eik_problem* local, int32_t cells_x, int32_t cells_y,
                                     int64_t base_y, int64_t row0, int64_t row_end) {
  g_last_code = EIK_OK;
  g_last_error.clear();
  if (check_problem(local)) return nullptr;
  const eik_grid& g = local->grid;
  if (cells_x < 1 || cells_y < 1 || cells_x > g.m || base_y < 1 || row0 < 0 ||
      row0 + (int64_t)(cells_y - 1) * base_y >= row_end || row_end > g.n) {
    fail(EIK_ERR_CONFIG, "fmsm strip: cell rows outside the strip's grid");
    return nullptr;
  }
  if (eik_device_count() < 1) {
    fail(EIK_ERR_CUDA, "no CUDA device visible: the Eikonal hot path has no CPU fallback");
    return nullptr;
  }
  eik_cells c{};
  c.cells_x = cells_x;
  c.cells_y = cells_y;
  const StripGeom sg{base_y, row0, row_end};
  t_strip_geom = &sg;
  eik_plan* P = new eik_plan();
  const int rc = plan_init(P, local, &c, EIK_FMSM);
  t_strip_geom = nullptr;
  if (rc) {
    std::string keep = g_last_error;
    int keep_code = g_last_code;
    plan_free(P);
    g_last_error = keep;
    g_last_code = keep_code;
    return nullptr;
  }
  return P;
}

int eik_plan_fmsm_levels(eik_plan* P, const int32_t* cells, const int32_t* level_off,
                         int32_t nlevels, const uint8_t* flags) {
  if (!P || !flags) return fail(EIK_ERR_DOMAIN, "null argument");
  return plan_fmsm_levels(P, cells, level_off, nlevels, flags);
}

int eik_plan_fmsm_level_async(eik_plan* P, int32_t level, void* stream) {
  if (!P) return fail(EIK_ERR_DOMAIN, "null plan");
  return plan_fmsm_level_async(P, level, static_cast<cudaStream_t>(stream));
}

int eik_plan_fmsm_counters(eik_plan* P, int64_t* out2) {
  if (!P || !out2) return fail(EIK_ERR_DOMAIN, "null argument");
  return plan_fmsm_counters(P, out2);
}

int eik_fmsm_schedule(const eik_problem* p, const eik_cells* c, int32_t* order, int32_t* rank,
                      uint8_t* flags, int32_t* level, int64_t* counters2) {
  g_last_code = EIK_OK;
  g_last_error.clear();
  if (check_problem(p)) return g_last_code;
  return fmsm_schedule(p, c, order, rank, flags, level, counters2);
}

int eik_plan_prepare(eik_plan* P) {
  if (!P) return fail(EIK_ERR_DOMAIN, "null plan");
  return plan_prepare(P);
}

int eik_plan_sweep(eik_plan* P, int64_t first_sweep, int32_t count, int32_t* changed) {
  if (!P) return fail(EIK_ERR_DOMAIN, "null plan");
  return plan_sweep(P, first_sweep, count, changed);
}

int eik_plan_sweep_async(eik_plan* P, int64_t first_sweep, int32_t count, int32_t* changed_dev,
                         void* stream) {
  if (!P || !changed_dev) return fail(EIK_ERR_DOMAIN, "null argument");
  return plan_sweep_impl(P, first_sweep, count, nullptr, changed_dev,
                         static_cast<cudaStream_t>(stream));
}

int eik_plan_rows_async(eik_plan* P, int64_t row0, int64_t nrows, double* dev_buf, int32_t to_plan,
                        void* stream) {
  if (!P) return fail(EIK_ERR_DOMAIN, "null plan");
  return plan_rows_async(P, row0, nrows, dev_buf, to_plan != 0, static_cast<cudaStream_t>(stream));
}

int eik_plan_get_rows(eik_plan* P, int64_t row0, int64_t nrows, double* dst, int32_t on_device) {
  if (!P) return fail(EIK_ERR_DOMAIN, "null plan");
  return plan_rows(P, row0, nrows, dst, on_device, false);
}

int eik_plan_set_rows(eik_plan* P, int64_t row0, int64_t nrows, const double* src,
                      int32_t on_device) {
  if (!P) return fail(EIK_ERR_DOMAIN, "null plan");
  return plan_rows(P, row0, nrows, const_cast<double*>(src), on_device, true);
}

int eik_set_hcm_mode(int32_t mode) {
  if (mode != 0 && mode != 1) return fail(EIK_ERR_CONFIG, "hcm mode is 0 (band) or 1 (exact)");
  g_hcm_mode.store(mode);
  return EIK_OK;
}

int eik_plan_set_hcm_mode(eik_plan* P, int32_t mode) {
  if (!P) return fail(EIK_ERR_DOMAIN, "null plan");
  if (mode != 0 && mode != 1) return fail(EIK_ERR_CONFIG, "hcm mode is 0 (band) or 1 (exact)");
  if (P->method != EIK_HCM) return fail(EIK_ERR_CONFIG, "hcm mode applies to hcm plans");
  P->hcm_band = mode == 0;
  return EIK_OK;
}

int eik_plan_set_ctas(eik_plan* P, int32_t max_ctas) {
  if (!P) return fail(EIK_ERR_DOMAIN, "null plan");
  if (max_ctas < 0) return fail(EIK_ERR_CONFIG, "max_ctas must be >= 0");
  P->ctas_cap = max_ctas;
  return EIK_OK;
}

int eik_plan_set_partitions(eik_plan* P, int32_t part_rows) {
  if (!P) return fail(EIK_ERR_DOMAIN, "null plan");
  if (P->method != EIK_FSM && P->method != EIK_FMM)
    return fail(EIK_ERR_CONFIG, "partitions apply to fsm/fmm plans");
  if (part_rows < 0 || part_rows % 32 != 0)
    return fail(EIK_ERR_CONFIG, "part_rows must be a non-negative multiple of 32");
  P->part_strips = part_rows / 32;
  P->last_sweeps_bound = P->max_sweeps;  // the next run may need more sweeps
  return EIK_OK;
}

int eik_plan_capacity(eik_plan* P, int32_t* device_ctas, int32_t* fixed_ctas) {
  if (!P || !device_ctas || !fixed_ctas) return fail(EIK_ERR_DOMAIN, "null argument");
  int d = 0, f = 0;
  int rc = plan_capacity(P, &d, &f);
  if (rc) return rc;
  *device_ctas = d;
  *fixed_ctas = f;
  return EIK_OK;
}

int eik_plan_run_batch(eik_plan* const* plans, int32_t n, eik_output* outs, double* batch_ms) {
  g_last_code = EIK_OK;
  g_last_error.clear();
  if (n < 0 || (n > 0 && (!plans || !outs))) return fail(EIK_ERR_DOMAIN, "batch: bad arguments");
  if (n == 0) {
    if (batch_ms) *batch_ms = 0.0;
    return EIK_OK;
  }
  return plan_run_batch(plans, n, outs, batch_ms);
}

int eik_solve_batch(const eik_problem* const* problems, const eik_cells* const* cells,
                    const int32_t* methods, int32_t n, eik_output* outs, double* batch_ms) {
  g_last_code = EIK_OK;
  g_last_error.clear();
  if (n < 0 || (n > 0 && (!problems || !methods || !outs)))
    return fail(EIK_ERR_DOMAIN, "batch: bad arguments");
  for (int k = 0; k < n; ++k)
    if (!outs[k].u) return fail(EIK_ERR_DOMAIN, "output needs a u buffer");
  if (n == 0) {
    if (batch_ms) *batch_ms = 0.0;
    return EIK_OK;
  }
  if (eik_device_count() < 1)
    return fail(EIK_ERR_CUDA, "no CUDA device visible: the Eikonal hot path has no CPU fallback");
  return solve_batch_pipelined(problems, cells, methods, n, outs, batch_ms);
}

int eik_solve_multi(const eik_problem* p, int32_t method, const int32_t* devices,
                    int32_t n_devices, eik_output* out) {
  g_last_code = EIK_OK;
  g_last_error.clear();
  if (!out || !out->u) return fail(EIK_ERR_DOMAIN, "output needs a u buffer");
  if (n_devices < 1 || !devices) return fail(EIK_ERR_DOMAIN, "need at least one device");
  const int nd = eik_device_count();
  for (int d = 0; d < n_devices; ++d)
    if (devices[d] < 0 || devices[d] >= nd) return fail(EIK_ERR_CONFIG, "no such CUDA device");
  if (n_devices == 1) {
    CK(cudaSetDevice(devices[0]));
    return eik_solve(p, nullptr, method, out);
  }
  if (method != EIK_FSM && method != EIK_FMM)
    return fail(EIK_ERR_NOT_IMPL, "eik_solve_multi shards fsm / fmm (row strips)");
  if (check_problem(p)) return g_last_code;
  out->sweeps = out->node_updates = out->heap_removals = 0;
  out->cell_removals = out->cell_sweeps = out->mon_checks = out->mon_single = 0;
  out->avhr = out->avs = out->mon_pct = 0.0;
  out->host_ms = 0.0;
  out->spec_hits = out->spec_waits = out->spec_self = 0;
  out->kernel_launches = 0;
  return solve_multi(p, method, devices, n_devices, out);
}

int eik_solve(const eik_problem* p, const eik_cells* c, int32_t method, eik_output* out) {
  if (!out || !out->u) return fail(EIK_ERR_DOMAIN, "output needs a u buffer");
  eik_plan* P = eik_plan_create(p, c, method);
  if (!P) return g_last_code != EIK_OK ? g_last_code : EIK_ERR_CUDA;
  int rc = plan_run(P, out);
  plan_free(P);
  return rc;
}

}  // extern "C"
