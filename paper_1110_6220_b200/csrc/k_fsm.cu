// Kernel (1): exact Gauss-Seidel Fast Sweeping on the whole grid as a
// pipelined anti-diagonal wavefront (replaces fsm_solve's loop,
// /root/reference/proj/src/classic_solvers.cpp:128-158).
//
// Why it is exact.  In sweep direction d the reference visits (i,j) after its
// two upwind neighbours (new values) and before its two downwind neighbours
// (old values) (classic_solvers.cpp:137-155).  Any schedule that respects
// exactly those read-after-write / write-after-read edges reproduces the
// sequential result bit for bit.  The wavefront below is such a schedule:
//
//   * the grid is cut into strips of 32 rows; one warp owns a strip; lane t
//     owns one row and walks the columns in sweep order, lagging lane t-1 by
//     one step (skewed pipeline): the upwind-row neighbour arrives from lane
//     t-1 through __shfl_up_sync, the downwind-row neighbour (old) from lane
//     t+1's prefetched register through __shfl_down_sync, the upwind-column
//     neighbour is the lane's own previous result, the downwind-column one its
//     own prefetched old value;
//   * strips hand their edge row to the next strip through global memory and a
//     per-strip progress counter (release/acquire at gpu scope);
//   * sweeps are pipelined: a strip starts sweep k once its own sweep k-1 is
//     done and the strip downwind of it in sweep k has finished sweep k-1.
//     Extra sweeps after convergence change nothing (a fixed point stays
//     fixed), so the stop decision for sweep k is taken from the global change
//     flag of sweep k-D, identically by every strip.
//
// Counters match the reference: sweeps = first unchanged sweep + 1
// (classic_solvers.cpp:146-157), node_updates = sweeps * (M - |Q|).
#include "eik_internal.h"
#include "k_common.cuh"

namespace eikb200 {

namespace {

constexpr int kU = 8;          // columns per register block (prefetch unit)
constexpr int kWarpsPerCta = 4;
// Mailbox slots hold a strip's edge-row value for its downwind neighbour; an
// all-ones NaN marks "empty" (values are never NaN).  The datum is its own
// flag, so the per-column hand-off needs no fence at all.
constexpr unsigned long long kSent = ~0ull;

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const void* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool is_sent(double v) {
  return (unsigned long long)__double_as_longlong(v) == kSent;
}
__device__ __noinline__ double poll_slot(const double* p, int* status) {
  long long spins = 0;
  unsigned long long v;
  while ((v = ld_relaxed_u64(p)) == kSent) {
    if (++spins > kSpinCap) {
      atomicExch(status, kStatusWatchdog);
      return kInf;
    }
    if ((spins & 1023) == 0 && *(volatile int*)status == kStatusWatchdog) return kInf;
  }
  return __longlong_as_double((long long)v);
}
// Measured (profiles/README.md): handing edges between the warps of one CTA
// through shared-memory rings with per-column spinning is 2-5x slower than
// these global mailboxes -- the spinning LDS traffic competes with the
// shuffles for the MIO pipe -- so every strip boundary uses a mailbox.
struct Chan {
  double* gin;            // global mailbox row of the upwind strip (or the dummy row)
  double* gout;           // global mailbox row to the downwind strip (or dummy)
  const double* dnh;      // downwind edge row (old values) in u (or dummy)
  bool in_glob, out_glob; // lane 0 / lane 31 use the mailboxes
};

// One sweep of one warp-strip.  IASC selects the column direction at compile
// time so every access in the unrolled block is an immediate offset from a
// per-block pointer; the padded layout (kPad columns of +inf / -1 on both
// sides, a dummy row for lanes past the last grid row) removes every bounds
// check from the step.
template <bool IASC>
__device__ __forceinline__ bool sweep_strip(const FsmArgs& a, int lane, int64_t rowp,
                                            const Chan& ch) {
  constexpr int S = IASC ? 1 : -1;
  const int64_t m = a.m, P = a.P;
  const int64_t q0off = IASC ? 0 : m - 1;  // element q of a row sits at base + S*q
  double* pu = a.u + rowp * P + a.pad + q0off - S * lane;
  const double* pc = a.C + rowp * P + a.pad + q0off - S * lane;
  const bool in_lane = (lane == 0) && ch.in_glob;
  const bool dn_lane = (lane == 31);
  const bool halo_lane = in_lane || dn_lane;
  double* ph = (lane == 0 ? ch.gin : const_cast<double*>(ch.dnh)) + a.pad + q0off - S * lane;
  double* po = ch.gout + a.pad + q0off - S * lane;
  const bool out_glob = dn_lane && ch.out_glob;
  const int nblocks = (int)((m + 31 + kU - 1) / kU);

  double cu[kU + 1], cc[kU], hv[kU];
  double nu[kU + 1], nc[kU], nh[kU];
#pragma unroll
  for (int t = 0; t <= kU; ++t) cu[t] = pu[S * t];
#pragma unroll
  for (int t = 0; t < kU; ++t) {
    cc[t] = __ldg(pc + S * t);
    hv[t] = halo_lane ? __ldcg(ph + S * t) : kInf;
  }
  double res_prev = kInf;
  bool changed = false;
  int q0 = -lane;
  const double sent = __longlong_as_double((long long)kSent);

  for (int blk = 0; blk < nblocks; ++blk) {
#pragma unroll
    for (int t = 1; t <= kU; ++t) nu[t] = pu[S * (kU + t)];
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      nc[t] = __ldg(pc + S * (kU + t));
      nh[t] = halo_lane ? __ldcg(ph + S * (kU + t)) : kInf;
    }
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      const int q = q0 + t;
      double sv = __shfl_up_sync(kFull, res_prev, 1);
      double nv = __shfl_down_sync(kFull, cu[t + 1], 1);
      double h = hv[t];
      if (in_lane && q < m) {
        if (is_sent(h)) h = poll_slot(ph + S * t, a.status);
        ph[S * t] = sent;  // re-arm the slot for the next sweep
      }
      if (lane == 0) sv = h;
      if (lane == 31) nv = h;
      const double cur = cu[t];
      const double c = cc[t];
      const double cand = node_update4(cu[t + 1], res_prev, nv, sv, c);
      const bool upd = (c > 0.0) && (cand < cur);  // exits / padding carry c = -1
      const double res = upd ? cand : cur;
      if (upd) pu[S * t] = cand;
      changed |= upd;
      if (out_glob) __stcg(po + S * t, res);  // straight to L2: the next strip polls it
      res_prev = res;
    }
    pu += S * kU;
    pc += S * kU;
    ph += S * kU;
    po += S * kU;
    q0 += kU;
    cu[0] = cu[kU];
#pragma unroll
    for (int t = 1; t <= kU; ++t) cu[t] = nu[t];
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      cc[t] = nc[t];
      hv[t] = nh[t];
    }
  }
  return changed;
}

__global__ void __launch_bounds__(32 * kWarpsPerCta)
fsm_wavefront_kernel(FsmArgs a) {
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int b = blockIdx.x * kWarpsPerCta + w;
  if (b >= a.nstrips) return;  // warps past the last grid row do not exist
  const int64_t n = a.n, P = a.P;

  for (int k = 0;; ++k) {
    // ---- stop decision: identical in every strip --------------------------
    if (!a.fixed && k >= a.lookahead) {
      const int kk = k - a.lookahead;
      int chg = 1, ok = 1;
      if (lane == 0) {
        ok = wait_ge_s32(&a.done[kk], a.nstrips, a.status);
        chg = ld_acquire_s32(&a.changed[kk]);
      }
      if (!__shfl_sync(kFull, ok, 0)) return;
      chg = __shfl_sync(kFull, chg, 0);
      if (!chg) {
        if (b == 0 && lane == 0) a.status[1] = kk + 1;  // reference sweep count
        break;
      }
    }
    if (k >= a.max_sweeps) {
      if (a.fixed) {
        if (b == 0 && lane == 0) a.status[1] = k;
      } else if (lane == 0) {
        atomicExch(&a.status[0], 3);
      }
      break;
    }
    const int dir = (a.first_sweep + k) & 3;  // sweep_direction (classic_solvers.cpp:94-96)
    const bool iasc = (dir == 0 || dir == 1);
    const bool jasc = (dir == 0 || dir == 3);
    const int64_t base = (int64_t)b * 32;
    const int64_t row = jasc ? base + lane : base + 31 - lane;
    const int64_t rowp = row < n ? row : n;             // dummy row n: +inf / -1
    const int64_t uprow = jasc ? base - 1 : base + 32;  // upwind edge row (new)
    const int64_t dnrow = jasc ? base + 32 : base - 1;  // downwind edge row (old)
    const bool has_up = uprow >= 0 && uprow < n;
    const bool has_dn = dnrow >= 0 && dnrow < n;
    const int flow = jasc ? 0 : 1;
    unsigned long long* tr =
        (a.trace && k < kTraceSweeps) ? a.trace + ((int64_t)k * a.nstrips + b) * 3 : nullptr;
    if (tr && lane == 0) tr[0] = globaltimer();

    // The strip downwind of us in sweep k must have finished sweep k-1: its
    // edge row is our "old" neighbour row, and the hand-off slots it emptied
    // must be visible before we refill them.  Once per sweep.
    {
      int ok = 1;
      if (k > 0 && has_dn && lane == 0)
        ok = wait_ge_u64(&a.prog[jasc ? b + 1 : b - 1], (unsigned long long)k, a.status);
      if (!__shfl_sync(kFull, ok, 0)) return;
    }
    double* dummy = a.u + n * P;  // all +inf
    Chan ch;
    ch.in_glob = has_up;
    ch.out_glob = has_dn;
    ch.gin = ch.in_glob ? a.mbox + ((int64_t)flow * a.nstrips + (jasc ? b - 1 : b + 1)) * P : dummy;
    ch.gout = ch.out_glob ? a.mbox + ((int64_t)flow * a.nstrips + b) * P : dummy;
    ch.dnh = has_dn ? a.u + dnrow * P : dummy;

    if (tr && lane == 0) tr[1] = globaltimer();
    const bool changed = iasc ? sweep_strip<true>(a, lane, rowp, ch)
                              : sweep_strip<false>(a, lane, rowp, ch);

    // sweep complete for this strip: make every lane's writes visible, then
    // publish completion and the change flag (once per sweep).
    __threadfence();
    __syncwarp();
    const bool any = __any_sync(kFull, changed);
    if (tr && lane == 0) tr[2] = globaltimer();
    if (lane == 31) st_release_u64(&a.prog[b], (unsigned long long)(k + 1));
    if (lane == 0) {
      if (any) atomicOr(&a.changed[k], 1);
      __threadfence();
      atomicAdd(&a.done[k], 1);
    }
  }
}

// Padded layout: row r (0..n, row n is a dummy) holds element i at
// r*P + pad + i; padding columns and the dummy row carry u = +inf, C = -1.
__global__ void prepare_padded_kernel(const double* __restrict__ F, double* __restrict__ C,
                                      double* __restrict__ u, int64_t m, int64_t n, int64_t P,
                                      int64_t pad, double h, int* __restrict__ status) {
  const int64_t total = (n + 1) * P;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / P, i = idx - r * P - pad;
    double c = -1.0;
    if (r < n && i >= 0 && i < m) {
      const double f = F[r * m + i];
      if (!(f > 0.0) || !(f < kInf)) atomicExch(&status[0], 1);
      c = h / f;  // same IEEE division as local_update.hpp:33
    }
    C[idx] = c;
    u[idx] = kInf;
  }
}

__global__ void mark_exits_kernel(const int64_t* __restrict__ exits,
                                  const double* __restrict__ cost, int64_t n_exit, int64_t m,
                                  int64_t P, int64_t pad, double* __restrict__ C,
                                  double* __restrict__ u) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_exit;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = exits[k], r = e / m, i = e - r * m;
    C[r * P + pad + i] = -1.0;
    u[r * P + pad + i] = cost[k];
  }
}

}  // namespace

cudaError_t launch_prepare(const double* F, double* C, double* u, int64_t m, int64_t n,
                           int64_t P, int64_t pad, double h, const int64_t* exits,
                           const double* cost, int64_t n_exit, int* status, cudaStream_t s,
                           int* launches) {
  const int threads = 256;
  int64_t blocks = ((n + 1) * P + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  prepare_padded_kernel<<<(unsigned)blocks, threads, 0, s>>>(F, C, u, m, n, P, pad, h, status);
  int64_t eb = (n_exit + threads - 1) / threads;
  if (eb > 1024) eb = 1024;
  if (eb < 1) eb = 1;
  mark_exits_kernel<<<(unsigned)eb, threads, 0, s>>>(exits, cost, n_exit, m, P, pad, C, u);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t fsm_capacity(int nstrips, int* need, int* ctas) {
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, fsm_wavefront_kernel, 32 * kWarpsPerCta, 0);
  if (e != cudaSuccess) return e;
  *need = (nstrips + kWarpsPerCta - 1) / kWarpsPerCta;
  *ctas = per_sm * sms;
  return cudaSuccess;
}

cudaError_t launch_fsm(const FsmArgs& args, cudaStream_t s, int* launches, int* grid) {
  const int ctas = (args.nstrips + kWarpsPerCta - 1) / kWarpsPerCta;
  if (grid) *grid = ctas;
  FsmArgs a = args;
  void* params[] = {&a};
  // Strips spin on each other's progress, so every CTA must be co-resident:
  // a cooperative launch guarantees it (or fails loudly).
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)fsm_wavefront_kernel, dim3(ctas),
                                              dim3(32 * kWarpsPerCta), params, 0, s);
  *launches += 1;
  return e;
}

}  // namespace eikb200
