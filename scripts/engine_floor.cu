// The in-cell wavefront's latency floor: cycles per step of a one-warp
// skewed pipeline that does only what every engine must (the upwind shuffle,
// the node update, the compare/select), against the production locking
// engine (k_cellsweep.cuh) on the same cell.  Development aid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 \
//        -I paper_1110_6220_b200/csrc -I include scripts/engine_floor.cu -o /tmp/ef
#include <cstdio>
#include <cstdlib>

#include "k_cellsweep.cuh"

using namespace eikb200;

namespace eikb200 {
template <bool SKIP, int NS, int DIR>
__device__ __forceinline__ bool cell_sweep_lock_d(const CellTile& T, int lane,
                                                long long& updates_out) {
  constexpr bool iasc = (DIR == kSW || DIR == kNW);
  constexpr bool jasc = (DIR == kSW || DIR == kSE);
  const int w = T.w, h = T.h, pu = T.pu, ox = T.ox;
  constexpr int dx = iasc ? 1 : -1;
  const int dyp = jasc ? pu : -pu;
  const int dyl = jasc ? w : -w;
  const int x0 = iasc ? 0 : w - 1;
  const bool up_in = jasc ? T.in_lo : T.in_hi;  // upwind / downwind halo row in the cell
  const bool dn_in = jasc ? T.in_hi : T.in_lo;
  double* __restrict__ U = T.U;
  const double* __restrict__ C = T.Ct;
  uint8_t* __restrict__ L = T.lock;
  int vb[NS], lb[NS];
  bool rv[NS], unW[NS];
  double wv[NS], cw[NS];
  unsigned nm[NS];
#pragma unroll
  for (int r = 0; r < NS; ++r) {
    const int b = lane + 32 * r;
    rv[r] = b < h;
    const int y = jasc ? b : h - 1 - b;
    vb[r] = rv[r] ? (y + 1) * pu + (x0 + ox) : pu + ox;  // value offset of a = 0
    lb[r] = rv[r] ? y * w + x0 : 0;                      // lock offset of a = 0
    wv[r] = rv[r] ? U[vb[r] - dx] : kInf;  // W: frozen halo column, then own new values
    cw[r] = -1.0;                          // W cost (< 0: halo or exit, never unlocked)
    unW[r] = false;                        // the W neighbour unlocked this node
    nm[r] = 0u;                            // last step's ballot of "unlock my N"
  }
  int updates = 0;
  bool changed = false;
  double q_cur[NS], q_cc[NS], q_e[NS], q_ce[NS], q_n[NS], q_cn[NS], q_cs[NS], q_hs[NS];
  int q_lk[NS];
  auto load = [&](int s) {
#pragma unroll
    for (int r = 0; r < NS; ++r) {
      const int a = s - lane - 32 * r;
      const bool act = rv[r] && a >= 0 && a < w;
      // (0,0) when inactive: every neighbour read stays in the tile
      const int o = act ? vb[r] + dx * a : pu + ox;
      q_cur[r] = U[o];
      q_cc[r] = C[o];
      q_e[r] = U[o + dx];
      q_ce[r] = C[o + dx];
      q_n[r] = U[o + dyp];
      q_cn[r] = C[o + dyp];
      q_cs[r] = C[o - dyp];
      q_hs[r] = U[o - dyp];
      q_lk[r] = L[act ? lb[r] + dx * a : 0];
    }
  };
  load(0);
  const int last = (h - 1) + (w - 1);
  // Unrolled by 2: no register moves for the prefetched operands, 3-11 %
  // faster per solve alone.  Concurrent solves contend for instruction cache:
  // with two engine call sites per kernel the unroll cost the batch 5 %; with
  // one (process_cell) it trades 2.4 % of the resident batch value for 1.8 %
  // of the end-to-end batch (9 runs each), and is kept.
#pragma unroll 2
  for (int s = 0; s <= last; ++s) {
    double cur[NS], cc[NS], e[NS], ce[NS], n[NS], cn[NS], cs[NS], hs[NS];
    int lk[NS];
#pragma unroll
    for (int r = 0; r < NS; ++r) {
      cur[r] = q_cur[r];
      cc[r] = q_cc[r];
      e[r] = q_e[r];
      ce[r] = q_ce[r];
      n[r] = q_n[r];
      cn[r] = q_cn[r];
      cs[r] = q_cs[r];
      hs[r] = q_hs[r];
      lk[r] = q_lk[r];
    }
    // phase 1, every slot: the upwind row's new value and unlock bit, and
    // whether the slot processes a node.  The slots' fp64 chains are
    // independent, so they are computed together (phase 2) and overlap;
    // the stores and ballots follow (phase 3).
    double sv[NS], cand[NS];
    bool act[NS], proc[NS];
    bool any = false;
#pragma unroll
    for (int r = 0; r < NS; ++r) {
      const int b = lane + 32 * r;
      const int a = s - b;
      act[r] = rv[r] && a >= 0 && a < w;
      // previous-step values: slot r's lane 0 takes slot r-1's lane 31
      const double send = (lane == 31 && r > 0) ? wv[r > 0 ? r - 1 : 0] : wv[r];
      sv[r] = __shfl_sync(kFull, send, (lane + 31) & 31);
      unsigned sbit = lane == 0 ? (r > 0 ? (nm[r > 0 ? r - 1 : 0] >> 31) & 1u : 0u)
                                : (nm[r] >> (lane - 1)) & 1u;
      if (b == 0) {
        sv[r] = hs[r];
        sbit = 0u;
      }
      proc[r] = act[r] && cc[r] >= 0.0 && (lk[r] != 0 || unW[r] || sbit != 0u);
      any = any || proc[r];
    }
    // the next step's operands: issued after the shuffles, so the critical
    // shuffle does not queue behind nine shared loads in the MIO pipe
    asm volatile("" ::: "memory");
    load(s + 1);  // prefetch while this step computes (past the end: harmless)
    if (SKIP && !__any_sync(kFull, any)) {
#pragma unroll
      for (int r = 0; r < NS; ++r) {
        unW[r] = false;
        nm[r] = 0u;
        if (act[r]) wv[r] = cur[r];
        cw[r] = act[r] ? cc[r] : -1.0;
      }
      continue;
    }
#pragma unroll
    for (int r = 0; r < NS; ++r) cand[r] = node_update4(e[r], wv[r], n[r], sv[r], cc[r]);
#pragma unroll
    for (int r = 0; r < NS; ++r) {
      const int b = lane + 32 * r;
      const int a = s - b;
      const int o = act[r] ? vb[r] + dx * a : pu + ox;
      const int lo = act[r] ? lb[r] + dx * a : 0;
      const bool dec = proc[r] && cand[r] < cur[r];
      const double res = dec ? cand[r] : cur[r];
      if (dec) {
        changed = true;
        U[o] = cand[r];
        // already-processed W and S neighbours: unlocked for the next sweep
        if (a > 0 && cw[r] >= 0.0 && wv[r] > cand[r]) L[lo - dx] = 1;
        if ((b > 0 || up_in) && cs[r] >= 0.0 && sv[r] > cand[r]) L[lo - dyl] = 1;
        // the next band's first row: unlocked in memory for this sweep
        if (b + 1 == h && dn_in && cn[r] >= 0.0 && n[r] > cand[r]) L[lo + dyl] = 1;
      }
      const bool un_n = dec && (b + 1 < h) && cn[r] >= 0.0 && n[r] > cand[r];
      unW[r] = dec && (a + 1 < w) && ce[r] >= 0.0 && e[r] > cand[r];
      if (proc[r]) {  // relock on processing (heap_cell.cpp:110-111)
        L[lo] = 0;
        ++updates;
      }
      nm[r] = __ballot_sync(kFull, un_n);
      if (act[r]) wv[r] = res;
      cw[r] = act[r] ? cc[r] : -1.0;
    }
  }
  __syncwarp();  // the next sweep / the scans read this sweep's stores
  updates_out += updates;
  return __any_sync(kFull, changed);
}


}  // namespace eikb200

// VAR 0: shuffle + node_update4 + select (IEEE sqrt); 1: the same with the
// sqrt replaced by a multiply; 2: shuffle + select only
template <int VAR>
__global__ void floor_kernel(int steps, int reps, long long* out, double* sink) {
  const int lane = threadIdx.x;
  double wv = 1.0 + lane * 1e-3, e = 2.0, n = 2.5, c = 0.01 + lane * 1e-5, cur = 3.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r)
    for (int s = 0; s < steps; ++s) {
      double sv = __shfl_sync(kFull, wv, (lane + 31) & 31);
      double cand;
      if (VAR == 0) {
        cand = node_update4(e, wv, n, sv, c);
      } else if (VAR == 3) {  // the FSM wavefront's update (straight-line sqrt)
        cand = node_update4_fast(e, wv, n, sv, c);
      } else if (VAR == 1) {
        const double ua = dmin(e, wv), ub = dmin(n, sv);
        const double diff = ua - ub;
        const bool two = (ua < kInf) && (ub < kInf) && (fabs(diff) <= c);
        const double arg = two ? (2.0 * c * c - diff * diff) : 1.0;
        const double ts = 0.5 * (ua + ub) + 0.5 * (arg * 1.0000001);
        cand = two ? ts : c + dmin(ua, ub);
      } else {
        cand = sv + c;
      }
      const bool dec = cand < cur;
      wv = dec ? cand : wv * 0.999;
      e = e * 1.0000001;
    }
  long long t1 = clock64();
  if (lane == 0) {
    out[0] = t1 - t0;
    *sink = wv;
  }
}

template <bool TEMPL>
__global__ void lock_kernel(int w, int h, int reps, long long* out, double* sink) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x;
  const int pu = (w + 3) & ~1;
  CellTile T;
  T.pu = pu;
  T.ox = 1;
  T.U = sm;
  T.Ct = sm + (h + 2) * pu;
  T.lock = reinterpret_cast<uint8_t*>(T.Ct + (h + 2) * pu);
  T.w = w;
  T.h = h;
  for (int k = lane; k < (h + 2) * pu; k += 32) {
    T.U[k] = 1e300;
    T.Ct[k] = 0.01 + 0.001 * (k % 7);
  }
  for (int k = lane; k < w * h; k += 32) T.lock[k] = 1;
  __syncwarp();
  if (lane == 0) T.U[pu + 1] = 0.0;
  __syncwarp();
  long long upd = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (!TEMPL) {
      cell_sweep_lock<false, 1>(T, r & 3, lane, upd);
    } else {
      switch (r & 3) {
        case 0: cell_sweep_lock_d<false, 1, 0>(T, lane, upd); break;
        case 1: cell_sweep_lock_d<false, 1, 1>(T, lane, upd); break;
        case 2: cell_sweep_lock_d<false, 1, 2>(T, lane, upd); break;
        default: cell_sweep_lock_d<false, 1, 3>(T, lane, upd); break;
      }
    }
    for (int k = lane; k < w * h; k += 32) T.lock[k] = 1;
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) {
    out[0] = t1 - t0;
    *sink = T.U[pu * 3 + 3] + (double)upd;
  }
}

int main(int argc, char** argv) {
  long long* d;
  double* s;
  cudaMalloc(&d, 8);
  cudaMalloc(&s, 8);
  long long c[3];
  const int steps = 64, reps = argc > 1 ? atoi(argv[1]) : 200;
  floor_kernel<0><<<1, 32>>>(steps, reps, d, s);
  cudaMemcpy(&c[0], d, 8, cudaMemcpyDeviceToHost);
  floor_kernel<1><<<1, 32>>>(steps, reps, d, s);
  cudaMemcpy(&c[1], d, 8, cudaMemcpyDeviceToHost);
  floor_kernel<2><<<1, 32>>>(steps, reps, d, s);
  cudaMemcpy(&c[2], d, 8, cudaMemcpyDeviceToHost);
  long long c3 = 0;
  floor_kernel<3><<<1, 32>>>(steps, reps, d, s);
  cudaMemcpy(&c3, d, 8, cudaMemcpyDeviceToHost);
  printf("floor cycles/step: shfl+update+select %.0f (straight-line sqrt: %.0f), without sqrt %.0f, "
         "shfl+select %.0f\n",
         c[0] / (double)(steps * reps), c3 / (double)(steps * reps), c[1] / (double)(steps * reps),
         c[2] / (double)(steps * reps));
  for (int w : {8, 16, 32}) {
    const int h = w, pu = (w + 3) & ~1;
    const size_t smem = 2 * (h + 2) * pu * 8 + w * h + 16;
    cudaFuncSetAttribute(lock_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(lock_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    lock_kernel<false><<<1, 32, smem>>>(w, h, reps, d, s);
    long long cy, cy2;
    double s1, s2;
    cudaMemcpy(&cy, d, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&s1, s, 8, cudaMemcpyDeviceToHost);
    lock_kernel<true><<<1, 32, smem>>>(w, h, reps, d, s);
    cudaMemcpy(&cy2, d, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&s2, s, 8, cudaMemcpyDeviceToHost);
    printf("locking engine %dx%d: %.0f cycles/step, direction-templated %.0f (same result %d) (%s)\n", w, h,
           cy / (double)(reps * (w + h - 1)), cy2 / (double)(reps * (w + h - 1)), s1 == s2,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
