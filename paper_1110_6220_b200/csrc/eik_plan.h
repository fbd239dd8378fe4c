// Resident solve plan: device buffers, host copies of the inputs and the
// stream owned by one eik_plan, plus the host runtime's shared helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "eik_internal.h"
#include "eikonal_b200.h"

struct eik_plan {
  int method = 0;
  eik_grid g{};
  int64_t M = 0;
  int64_t n_exit = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;   // false: borrowed from eik_solve_batch's worker
  bool own_events = true;   // ev0/ev1 likewise
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<void*> allocs;
  double* dF = nullptr;   // speed (resident input)
  double* dC = nullptr;   // padded h/F, -1 at exits and padding
  double* dU = nullptr;   // padded value field
  int64_t* dExit = nullptr;
  double* dExitCost = nullptr;
  int* dStatus = nullptr;
  int64_t h2d_bytes = 0;
  // eik_solve_batch: the speed field is uploaded by the plan's first run, on
  // its stream, instead of at creation (later plans' uploads overlap earlier
  // plans' solves)
  const double* defer_F = nullptr;
  bool defer_F_dev = false;
  bool deferred = false;                      // created with deferred uploads
  const double* defer_probe[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t probe_len[4] = {0, 0, 0, 0};
  int64_t pitch = 0;       // padded row pitch of dC / dU (m + 2*kPad)
  // FSM wavefront state
  int nstrips = 0;
  int max_sweeps = 0;
  int64_t last_sweeps_bound = 1 << 16;
  unsigned long long* dProg = nullptr;
  double* dMbox = nullptr;
  unsigned long long* dTrace = nullptr;
  int* dChanged = nullptr;
  unsigned* dChg = nullptr;   // [2][n+3][chg_cw] change bits (k_fsm.cu)
  int64_t chg_cw = 0;
  unsigned* dSb = nullptr;    // [4][nstrips][nsb] super-block summaries + edge tokens (k_fsm.cu)
  int nsb = 0;
  bool chg_valid = false;     // the change bits describe every change since the last sweep launch
  int chg_last_par = 0;       // parity the last sweep of that launch wrote
  int part_strips = 0;        // strip-Jacobi parts (eik_plan_set_partitions), 0 = exact GS
  double* dSnap = nullptr;    // [2][boundaries][2] padded rows
  int64_t snap_count = 0;
  int* dDone = nullptr;
  unsigned long long* dLsmCnt = nullptr;  // [max_sweeps] LSM unlocked nodes per sweep
  int64_t fmm_updates = 0;    // fmm_solve's node_updates (order independent)
  // two-scale methods: host copies of the inputs (the plan owns them)
  int32_t cells_x = 0, cells_y = 0;
  std::vector<int64_t> exit_nodes;
  std::vector<double> exit_cost, exit_points_xy, exit_point_cost;
  std::vector<double> center_speed;
  eikb200::CellGeom cg{};
  int warps_per_cta = 0;
  int32_t* dOrder = nullptr;
  int32_t* dRank = nullptr;
  uint8_t* dFlags = nullptr;
  int* dCellDone = nullptr;
  int* dNext = nullptr;
  unsigned long long* dCounters = nullptr;
  // heap-cell state
  double* dProbe[4] = {nullptr, nullptr, nullptr, nullptr};
  unsigned long long* dState = nullptr;   // packed per-cell state words
  double* dCKey = nullptr;                // published heap keys
  unsigned* dCTag = nullptr;              // last committed instance per cell
  int hc_chain = 1;
  int hc_heap_cap = 0;                    // committer queue bucket capacity in smem (0 = global)
  int hc_capb_global = 0;                 // bucket capacity in global memory
  double* dCVal = nullptr;                // cell values
  double* dHKey = nullptr;
  int* dHPos = nullptr;
  int* dHArr = nullptr;
  int* dInitCells = nullptr;
  double* dInitValues = nullptr;
  int max_len = 0;
  double* dSlots = nullptr;
  unsigned* dSpecVer = nullptr;
  int* dBusy = nullptr;
  eikb200::PRec* dRec = nullptr;
  int* dHcMisc = nullptr;
  // HCM band scheduler (k_heapcell.cu hcm_band_kernel)
  bool hcm_band = false;    // HCM plan runs the band scheduler (else the exact replay)
  bool hcm_exact_req = false;  // created as EIK_HCM_EXACT
  int* dBInq = nullptr;
  unsigned* dBFlags = nullptr;
  unsigned char* dBFdone = nullptr;
  int* dBList = nullptr;
  int* dBWork = nullptr;
  int* dBCtl = nullptr;
  unsigned long long* dBKmin = nullptr;
  bool cells_big = false;   // cell tiles exceed shared memory: swept in place in u
  uint8_t* dBigLock = nullptr;
  double* dBigScratch = nullptr;
  int* dDbg = nullptr;      // EIK_HC_DEBUG: per-worker phase trace
  int* dOwner = nullptr;    // EIK_HC_DEBUG: last claiming worker per speculation   // [0] done flag, [1] published heap size
  int hc_warps_per_cta = 1;
  int64_t hc_min_smem = 0;  // dynamic smem floor per CTA (one CTA per SM)
  uint64_t hc_cx_magic = 0; // cell id -> row by multiply-shift (0: division)
  int hc_max_ctas = 1;
  // CTA cap of the persistent kernel (0 = the whole device): ctas_cap set by
  // eik_plan_set_ctas, run_cap by eik_plan_run_batch's device split for one run
  int ctas_cap = 0;
  int run_cap = 0;

  int cap() const { return run_cap > 0 ? run_cap : ctas_cap; }
  double last_ms = 0.0;
  bool ran = false;
  double init_sync_ms = 0.0;  // creation: wait for the uploads (diagnostics)      // a run completed (the resident field is a solution)  // device + host ms of the last run (batch admission order)
  // batch runs: called (then cleared) once the heap-cell grid is submitted
  std::function<void()> on_launched;
  // FMSM Part I computed ahead of the run (plan_prepare_host, called by the
  // batch paths before a plan waits for its SMs); consumed by the next run
  void* dTmaps = nullptr;   // FMSM tile-load tensor maps (device copy, 2 x 128 B)
  bool tma_tried = false, tma_ok = false;  // a strip plan's maps (levels)
  int* dLevelNext = nullptr;               // a sharded FMSM's strip: claim counter per level
  int64_t level_cap = 0;
  std::vector<int32_t> level_off;
  bool fmsm_ready = false;
  std::vector<int32_t> fmsm_order, fmsm_rank;
  std::vector<uint8_t> fmsm_flags;
  int64_t fmsm_coarse_pops = 0, fmsm_coarse_updates = 0;
  double fmsm_host_ms = 0.0;
};

namespace eikb200 {

// Tuning and debug knobs, read from the environment ONCE per process
// (eik_debug_reload_knobs re-reads them; tests use it).  None changes a
// result: every variant is tested bit-exact.  Defaults are the measured
// optima.
struct Knobs {
  // FSM wavefront
  bool fsm_noskip = false;         // EIK_FSM_NOSKIP: evaluate every node
  const char* fsm_trace = nullptr; // EIK_TRACE_FSM=path: per-strip timing trace (copied)
  int fsm_wpc = 0;                 // EIK_FSM_WPC: strips per CTA (0 = auto)
  int fsm_sb = 1;                  // EIK_FSM_SB=0: no super-block skipping
  int fsm_cont = 1;                // EIK_FSM_CONT=0: every sweep-level launch evaluates every node
  int fsm_start_ahead = 12;        // EIK_FSM_START_AHEAD (FsmArgs::start_ahead)
  int fsm_sb_wait_div = 1;         // EIK_FSM_SB_WAIT_DIV: token-wait threshold (FsmArgs::sb_wait_div)
  // heap-cell replay
  int hc_warps = 0;                // EIK_HC_WARPS (0 = fit)
  long hc_min_smem = -1;           // EIK_HC_MIN_SMEM (-1 = 116 KB)
  bool hc_global_heap = false;     // EIK_HC_GLOBAL_HEAP
  int hc_heap_cap = 0;             // EIK_HC_HEAP_CAP (0 = fit)
  int hc_chain = 1;                // EIK_HC_CHAIN
  int hc_bands = 1;                // EIK_HC_BANDS=0: tall cells with several rows per lane
  int tile_tma = 1;                // EIK_TILE_TMA=0: stage cell tiles by loads, not TMA
  int hc_ctas = 0;                 // EIK_HC_CTAS (0 = device)
  bool hc_debug = false;           // EIK_HC_DEBUG: per-worker phase trace
  bool hc_profile = false;         // EIK_HC_PROFILE: instrumented kernel
  int hc_idle_ns = 200;            // EIK_HC_IDLE_NS
  int hc_first_min = 2;            // EIK_HC_FIRST_MIN: worker rows of 32 that chase bucket minima
  int hc_first_min_pool = 256;     // EIK_HC_FIRST_MIN_POOL: ... in pools up to this size
  int hc_skip_from = 1;            // EIK_HC_SKIP_FROM
  // batches
  double batch_sms_scale = 0.0;    // EIK_BATCH_SMS_SCALE (0 = by the batch size)
  int batch_fmsm_ctas = 16;        // EIK_BATCH_FMSM_CTAS
  double batch_fmsm_prio = 0.5;    // EIK_BATCH_FMSM_PRIO
  int batch_fixed_per_sm = 0;      // EIK_BATCH_FIXED_PER_SM
  bool batch_trace = false;        // EIK_BATCH_TRACE
  bool batch_timing = false;       // EIK_BATCH_TIMING
  int batch_workers = 0;           // EIK_BATCH_WORKERS (0 = auto)
  // HCM band scheduler
  int hcm_exact = 0;               // EIK_HCM_EXACT=1: HCM by the exact replay
  double hcm_band = 0.0;           // EIK_HCM_BAND: band width scale (0 = default)
  int hcm_band_shrink = 128;       // EIK_HCM_BAND_SHRINK: narrow after rounds of more cells
};
const Knobs& knobs();
void reload_knobs();
// HCM ordering for new plans: 0 = band scheduler, 1 = exact replay
// (eik_set_hcm_mode; EIK_HCM_EXACT=1 sets the default to 1)
int hcm_default_mode();

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

// slowest CUDA call of this thread since the last reset (diagnostics for
// EIK_BATCH_TRACE): which API call blocks a batch worker
struct SlowCall {
  const char* what = nullptr;
  double ms = 0.0;
};
extern thread_local SlowCall t_slow;
double now_ms_host();
// Waits for the stream's work without spinning a core: the batch paths run
// dozens of host threads that each wait on a solve, and the runtime's default
// schedule (one context) spins in every blocking call -- starving the threads
// that create the next plans and run FMSM Part I.  Polls, then sleeps.
cudaError_t stream_wait(cudaStream_t s);

#define CK(expr)                                                  \
  do {                                                            \
    const double t0_ = now_ms_host();                             \
    cudaError_t e_ = (expr);                                      \
    const double dt_ = now_ms_host() - t0_;                       \
    if (dt_ > t_slow.ms) t_slow = SlowCall{#expr, dt_};           \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr);           \
  } while (0)

// Device buffers come from a per-device cache of released blocks (exact-size
// reuse): plans of one problem shape are created and destroyed repeatedly
// through eik_solve, and cudaMalloc/cudaFree (which synchronises the device)
// would otherwise sit on that path.  Released blocks stay cached up to a cap
// (eik_release_cached frees them).
cudaError_t pool_alloc(void** p, size_t bytes);
void pool_release(void* p);
// While alive, cache misses of this thread's pool_alloc are served
// stream-ordered on `s` (the plan's stream) instead of by cudaMalloc.
struct AllocStream {
  explicit AllocStream(cudaStream_t s);
  ~AllocStream();
  AllocStream(const AllocStream&) = delete;
  AllocStream& operator=(const AllocStream&) = delete;

 private:
  cudaStream_t prev_;
};

template <class T>
int dalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = pool_alloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  return EIK_OK;
}

int plan_init_cells(eik_plan* P, const eik_problem* p, const eik_cells* c);
// CTAs of the plan's persistent kernel the whole device holds (*device) and,
// for kernels whose grid size is fixed (FSM/FMM strips), that size (*fixed,
// else 0).
int plan_capacity(eik_plan* P, int* device, int* fixed);
int plan_run_fmsm(eik_plan* P, eik_output* out);
int plan_run_heapcell(eik_plan* P, eik_output* out);
// Host-side work of the next run that needs no device (FMSM Part I): the
// batch paths call it before a plan waits for SMs, so no SM is held idle
// while the host computes.  A no-op for the other methods.
int plan_prepare_host(eik_plan* P);
// A sharded FMSM's strip (distributed.fmsm_solve_strips): cell rows of height
// base_y from local node row row0, the last ending at row_end.
struct StripGeom {
  int64_t base_y, row0, row_end;
};
extern thread_local const StripGeom* t_strip_geom;  // read by plan_init_cells
int plan_fmsm_levels(eik_plan* P, const int32_t* cells, const int32_t* off, int32_t nlevels,
                     const uint8_t* flags);
int plan_fmsm_level_async(eik_plan* P, int32_t L, cudaStream_t stream);
int plan_fmsm_counters(eik_plan* P, int64_t out[2]);
int fmsm_schedule(const eik_problem* p, const eik_cells* c, int32_t* order, int32_t* rank,
                  uint8_t* flags, int32_t* level, int64_t* counters);

}  // namespace eikb200
