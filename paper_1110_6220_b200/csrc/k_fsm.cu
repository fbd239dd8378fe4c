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

__global__ void __launch_bounds__(32 * kWarpsPerCta)
fsm_wavefront_kernel(FsmArgs a) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (b >= a.nstrips) return;
  const int64_t m = a.m, n = a.n;
  const unsigned long long M1 = (unsigned long long)m + 1;
  const int nblocks = (int)((m + 31 + kU - 1) / kU);

  for (int k = 0;; ++k) {
    // ---- stop decision: identical in every strip --------------------------
    if (k >= a.lookahead) {
      const int kk = k - a.lookahead;
      int ch = 1;
      if (lane == 0) {
        while (ld_acquire_s32(&a.done[kk]) < a.nstrips) __nanosleep(64);
        ch = ld_acquire_s32(&a.changed[kk]);
      }
      ch = __shfl_sync(kFull, ch, 0);
      if (!ch) {
        if (b == 0 && lane == 0) a.status[1] = kk + 1;  // reference sweep count
        break;
      }
    }
    if (k >= a.max_sweeps) {
      if (lane == 0) atomicExch(&a.status[0], 3);
      break;
    }
    const int dir = k & 3;  // sweep_direction (classic_solvers.cpp:94-96)
    const bool iasc = (dir == 0 || dir == 1);
    const bool jasc = (dir == 0 || dir == 3);
    const int64_t base = (int64_t)b * 32;
    const int64_t row = jasc ? base + lane : base + 31 - lane;
    const bool rvalid = row < n;
    const int64_t uprow = jasc ? base - 1 : base + 32;  // upwind halo (new)
    const int64_t dnrow = jasc ? base + 32 : base - 1;  // downwind halo (old)
    const bool has_up = uprow >= 0 && uprow < n;
    const bool has_dn = dnrow >= 0 && dnrow < n;
    const int up = jasc ? b - 1 : b + 1;
    const int dn = jasc ? b + 1 : b - 1;
    const unsigned long long kbase = (unsigned long long)k * M1;

    // The strip downwind of us in sweep k must have finished sweep k-1 before
    // we overwrite the row it reads as "new" / it reads as "old".
    if (k > 0 && has_dn && lane == 0) {
      const unsigned long long need = kbase - M1 + (unsigned long long)m;
      while (ld_acquire_u64(&a.prog[dn]) < need) __nanosleep(32);
    }
    __syncwarp();

    const double* urow = a.u + (rvalid ? row * m : 0);
    const double* crow = a.C + (rvalid ? row * m : 0);
    // lane 0 reads the upwind halo row, lane 31 the downwind halo row
    const bool halo_lane = (lane == 0 && has_up) || (lane == 31 && has_dn);
    const double* hrow = a.u + (lane == 0 ? uprow : dnrow) * m;

    auto gi = [&](int64_t q) { return iasc ? q : m - 1 - q; };
    auto ld_u = [&](int64_t q) -> double {
      return (rvalid && q >= 0 && q < m) ? urow[gi(q)] : kInf;
    };
    auto ld_c = [&](int64_t q) -> double {
      return (rvalid && q >= 0 && q < m) ? __ldg(crow + gi(q)) : -1.0;
    };
    auto ld_h = [&](int64_t q) -> double {
      return (halo_lane && q >= 0 && q < m) ? ld_cg(hrow + gi(q)) : kInf;
    };
    auto wait_up = [&](int64_t cols) {  // upwind lane 31 has done `cols` columns
      if (lane == 0 && has_up) {
        const unsigned long long need = kbase + (unsigned long long)(cols < m ? cols : m);
        while (ld_acquire_u64(&a.prog[up]) < need) __nanosleep(16);
      }
      __syncwarp();
    };

    double cu[kU + 1], cc[kU], hv[kU];
    double nu[kU + 1], nc[kU], nh[kU];
    int64_t q0 = -(int64_t)lane;  // this lane's column at block start
    wait_up(kU);
#pragma unroll
    for (int t = 0; t <= kU; ++t) cu[t] = ld_u(q0 + t);
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      cc[t] = ld_c(q0 + t);
      hv[t] = ld_h(q0 + t);
    }
    double res_prev = kInf;
    bool changed = false;
    unsigned long long published = 0;

    for (int blk = 0; blk < nblocks; ++blk) {
      // prefetch the next block (halo needs the upwind strip one block ahead)
      wait_up(q0 + 2 * kU);
      nu[0] = 0.0;
#pragma unroll
      for (int t = 1; t <= kU; ++t) nu[t] = ld_u(q0 + kU + t);
#pragma unroll
      for (int t = 0; t < kU; ++t) {
        nc[t] = ld_c(q0 + kU + t);
        nh[t] = ld_h(q0 + kU + t);
      }
#pragma unroll
      for (int t = 0; t < kU; ++t) {
        const int64_t q = q0 + t;
        double sv = __shfl_up_sync(kFull, res_prev, 1);
        double nv = __shfl_down_sync(kFull, cu[t + 1], 1);
        if (lane == 0) sv = hv[t];
        if (lane == 31) nv = hv[t];
        const double cur = cu[t];
        double res = cur;
        const double c = cc[t];
        if (c > 0.0) {  // in range, not an exit (exits carry c = -1)
          const double cand = node_update4(cu[t + 1], res_prev, nv, sv, c);
          if (cand < cur) {
            res = cand;
            changed = true;
            a.u[row * m + gi(q)] = cand;
          }
        }
        res_prev = res;
      }
      // publish the last row's progress (lane 31 is the most lagging lane)
      if (lane == 31) {
        int64_t done_cols = q0 + kU;
        if (done_cols > m) done_cols = m;
        if (done_cols > 0 && (unsigned long long)done_cols > published) {
          published = (unsigned long long)done_cols;
          st_release_u64(&a.prog[b], kbase + published);
        }
      }
      q0 += kU;
      nu[0] = cu[kU];
#pragma unroll
      for (int t = 0; t <= kU; ++t) cu[t] = nu[t];
#pragma unroll
      for (int t = 0; t < kU; ++t) {
        cc[t] = nc[t];
        hv[t] = nh[t];
      }
    }
    // sweep complete for this strip: make every lane's writes visible, then
    // publish completion and the change flag.
    __threadfence();
    __syncwarp();
    const bool any = __any_sync(kFull, changed);
    if (lane == 31) st_release_u64(&a.prog[b], kbase + (unsigned long long)m);
    if (lane == 0) {
      if (any) atomicOr(&a.changed[k], 1);
      __threadfence();
      atomicAdd(&a.done[k], 1);
    }
  }
}

__global__ void fsm_prepare_kernel(const double* __restrict__ F, double* __restrict__ C,
                                   double* __restrict__ u, int64_t M, double h,
                                   int* __restrict__ status) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < M;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const double f = F[idx];
    if (!(f > 0.0) || !(f < kInf)) atomicExch(&status[0], 1);
    C[idx] = h / f;  // same IEEE division as local_update.hpp:33
    u[idx] = kInf;
  }
}

__global__ void mark_exits_kernel(const int64_t* __restrict__ exits,
                                  const double* __restrict__ cost, int64_t n_exit,
                                  double* __restrict__ C, double* __restrict__ u) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_exit;
       k += (int64_t)gridDim.x * blockDim.x) {
    C[exits[k]] = -1.0;
    u[exits[k]] = cost[k];
  }
}

}  // namespace

cudaError_t launch_prepare(const double* F, double* C, double* u, int64_t M, double h,
                           const int64_t* exits, const double* cost, int64_t n_exit,
                           int* status, cudaStream_t s, int* launches) {
  const int threads = 256;
  int64_t blocks = (M + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  fsm_prepare_kernel<<<(unsigned)blocks, threads, 0, s>>>(F, C, u, M, h, status);
  int64_t eb = (n_exit + threads - 1) / threads;
  if (eb > 1024) eb = 1024;
  if (eb < 1) eb = 1;
  mark_exits_kernel<<<(unsigned)eb, threads, 0, s>>>(exits, cost, n_exit, C, u);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_fsm(const FsmArgs& args, cudaStream_t s, int* launches) {
  const int ctas = (args.nstrips + kWarpsPerCta - 1) / kWarpsPerCta;
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
