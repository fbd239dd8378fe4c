// Kernel (2): in-cell sweeps for the two-scale methods, and the FMSM fine
// pass as a device-side dataflow schedule.
//
// In-cell sweep (replaces the `full_sweep` lambda, /root/reference/proj/src/
// fmsm.cpp:176-195): a warp stages one cell plus its one-node cross halo and
// its costs C = h/F in shared memory and sweeps it with the register-pipeline
// wavefront of k_cellsweep.cuh, bit-identical to the reference's row loop.
//
// FMSM Part II (fmsm.cpp:164-226): cells are claimed in the coarse order
// (host Part I, eik_coarse.cpp); a claimed cell waits only for its
// earlier-ranked neighbour cells.  Cells that run at the same time are never
// adjacent and a cell reads nothing but its own nodes and its cross halo, so
// any schedule respecting those edges reproduces the sequential pass bit for
// bit -- with far less waiting than level-synchronous batches.
#include "eik_internal.h"
#include "k_cellsweep.cuh"
#include "k_common.cuh"

namespace eikb200 {

namespace {

__device__ __forceinline__ void cell_rect(const CellGeom& g, int cell, int64_t& ib, int64_t& ie,
                                          int64_t& jb, int64_t& je) {
  const int cx = cell % g.cells_x, cy = cell / g.cells_x;
  ib = (int64_t)cx * g.base_x;
  ie = (cx == g.cells_x - 1) ? g.m : ib + g.base_x;  // remainder to the last cell
  jb = g.row0 + (int64_t)cy * g.base_y;
  je = (cy == g.cells_y - 1) ? g.row_end : jb + g.base_y;
}

__device__ __forceinline__ int cell_neighbor(const CellGeom& g, int cell, int side) {
  const int cx = cell % g.cells_x, cy = cell / g.cells_x;
  switch (side) {  // cells.hpp:51-61 (W, E, S, N)
    case 0: return cx > 0 ? cell - 1 : -1;
    case 1: return cx + 1 < g.cells_x ? cell + 1 : -1;
    case 2: return cy > 0 ? cell - g.cells_x : -1;
    default: return cy + 1 < g.cells_y ? cell + g.cells_x : -1;
  }
}

// Stage a cell, its cross halo (no corners) and the costs of both into the
// warp's tile; returns the number of exit nodes in the cell.
__device__ int stage_in(const CellGeom& g, const double* __restrict__ C, const double* u,
                        int64_t ib, int64_t jb, CellTile& T, int lane) {
  const int W2 = T.w + 2;
  const int tot = (T.h + 2) * W2;
  int exits = 0;
  for (int k = lane; k < tot; k += 32) {
    const int y = k / W2 - 1, x = k % W2 - 1;
    const bool corner = (x < 0 || x >= T.w) && (y < 0 || y >= T.h);
    if (corner) continue;
    const int64_t gj = jb + y;
    double v = kInf, c = -1.0;
    if (gj >= 0 && gj < g.n) {
      const int64_t o = gj * g.P + g.pad + ib + x;  // padding columns: +inf / -1
      v = __ldcg(u + o);
      c = __ldg(C + o);
    }
    T.U[(y + 1) * T.pu + (x + 1)] = v;
    T.Ct[(y + 1) * T.pu + (x + 1)] = c;
    if (x >= 0 && x < T.w && y >= 0 && y < T.h) exits += (c < 0.0);
  }
  __syncwarp();
  for (int o = 16; o > 0; o >>= 1) exits += __shfl_xor_sync(kFull, exits, o);
  return exits;
}

// ---- TMA tile loads (cp.async.bulk.tensor) ---------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one lane: expect `bytes`, then the two tile loads complete the phase
__device__ __forceinline__ void tma_tiles(const FmsmArgs& a, double* dU, double* dC, int x, int y,
                                          uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dU)), "l"(a.tmaps), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dC)), "l"(a.tmaps + 1), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  unsigned ok = 0;
  while (!ok)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase) : "memory");
}

// Stage by TMA: the value and cost tiles of the box whose top-left is node
// (ib - 1, jb - 1), or one column further west when that column is not on a
// 16-byte boundary (the TMA unit needs aligned box starts) -- the cell, its
// halo, the corners and a few nodes beyond, which no sweep reads.  Rows -1 and n
// are the padded layout's dummy rows; rows past them are zero-filled by the
// TMA unit and lie outside every cell's halo.  Returns the cell's exit count.
__device__ int stage_in_tma(const FmsmArgs& a, int64_t ib, int64_t jb, CellTile& T, uint64_t* bar,
                            unsigned& phase, int lane) {
  if (lane == 0) {
    // generic-proxy accesses of this tile (the last cell's sweeps) and the
    // neighbours' published values (acquired) before the async-proxy loads
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
    const unsigned bytes = 2u * (unsigned)a.g.pu * (unsigned)(a.g.max_h + 2) * 8u;
    tma_tiles(a, T.U, T.Ct, (int)((a.g.pad + ib - 1) & ~(int64_t)1), (int)jb, bar, bytes);
  }
  // a box starts on a 16-byte boundary (an even padded column): node 0 of
  // the cell sits at tile column 1 or 2 (pu leaves room for either)
  T.ox = 1 + (int)((a.g.pad + ib - 1) & 1);
  mbar_wait(bar, phase);
  phase ^= 1u;
  int exits = 0;
  for (int y = 0; y < T.h; ++y)
    for (int x = lane; x < T.w; x += 32) exits += T.Ct[(y + 1) * T.pu + (x + T.ox)] < 0.0;
  for (int o = 16; o > 0; o >>= 1) exits += __shfl_xor_sync(kFull, exits, o);
  return exits;
}

__device__ void stage_out(const CellGeom& g, double* u, int64_t ib, int64_t jb, const CellTile& T,
                          int lane) {
  if (T.w <= 32) {
    const int rows = 32 / T.w, x = lane % T.w, y0 = lane / T.w;  // rows per pass
    if (y0 < rows)
      for (int y = y0; y < T.h; y += rows)
        u[(jb + y) * g.P + g.pad + ib + x] = T.U[(y + 1) * T.pu + (x + T.ox)];
    return;
  }
  for (int y = 0; y < T.h; ++y)
    for (int x = lane; x < T.w; x += 32)
      u[(jb + y) * g.P + g.pad + ib + x] = T.U[(y + 1) * T.pu + (x + T.ox)];
}

__global__ void fmsm_dataflow_kernel(FmsmArgs a) {
  extern __shared__ __align__(128) double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  CellTile T;
  T.pu = a.g.pu;
  T.ox = 1;
  T.U = smem + (size_t)wib * a.g.tile_doubles;
  T.Ct = T.U + (size_t)a.g.tile_doubles / 2;
  T.lock = nullptr;
  long long my_sweeps = 0, my_updates = 0;
  // one mbarrier per warp, after the tiles
  uint64_t* bar =
      reinterpret_cast<uint64_t*>(smem + (size_t)(blockDim.x >> 5) * a.g.tile_doubles) + wib;
  unsigned phase = 0;
  if (a.use_tma && lane == 0) mbar_init(bar);
  __syncwarp();

  for (;;) {
    int p = 0;
    if (lane == 0) p = atomicAdd(a.next, 1);
    p = __shfl_sync(kFull, p, 0);
    if (p >= a.J) break;
    const int cell = a.order[p];
    int64_t ib, ie, jb, je;
    cell_rect(a.g, cell, ib, ie, jb, je);
    T.w = (int)(ie - ib);
    T.h = (int)(je - jb);
    // wait for the earlier-ranked neighbour cells (one lane per side)
    int ok = 1;
    if (lane < 4 && !a.nowait) {
      const int nb = cell_neighbor(a.g, cell, lane);
      if (nb >= 0 && a.rank[nb] < p) ok = wait_ge_s32(a.done + nb, 1, a.status);
    }
    if (__any_sync(kFull, !ok)) return;
    int exits = 0;
    if (a.big) {
      // a cell too large for the tile: swept in place, its cross halo being
      // the neighbours' nodes (adjacent cells never run at the same time)
      T.pu = (int)a.g.P;
      T.ox = 1;
      T.U = a.u + (jb - 1) * a.g.P + a.g.pad + ib - 1;
      T.Ct = const_cast<double*>(a.C) + (jb - 1) * a.g.P + a.g.pad + ib - 1;
      for (int k = lane; k < T.w * T.h; k += 32)
        exits += __ldg(a.C + (jb + k / T.w) * a.g.P + a.g.pad + ib + k % T.w) < 0.0;
      for (int o = 16; o > 0; o >>= 1) exits += __shfl_xor_sync(kFull, exits, o);
    } else if (a.use_tma) {
      exits = stage_in_tma(a, ib, jb, T, bar, phase, lane);
    } else {
      T.ox = 1;
      exits = stage_in(a.g, a.C, a.u, ib, jb, T, lane);
    }
    const int flags = a.flags[cell];
    int nsw = 0;
    long long unused = 0;
    if (flags & 16) {
      // Q-cell: FSM to convergence with the halo frozen (fmsm.cpp:200-210)
      bool changed = true;
      while (changed) {
        changed = big_cell_sweep<0>(T, nsw & 3, lane, unused);
        ++nsw;
        if (nsw > a.max_cell_sweeps) {
          if (lane == 0) atomicExch(a.status, 3);
          return;
        }
      }
    } else {
      // one directional sweep per chosen direction, in NE, NW, SE, SW order
      const int order[4] = {kNE, kNW, kSE, kSW};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (flags & (1 << order[k])) {
          big_cell_sweep<1>(T, order[k], lane, unused);
          ++nsw;
        }
    }
    if (!a.big) stage_out(a.g, a.u, ib, jb, T, lane);
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release_s32(a.done + cell, 1);
    my_sweeps += nsw;
    my_updates += (long long)nsw * (T.w * T.h - exits);
  }
  if (lane == 0) {
    atomicAdd(a.counters + 0, (unsigned long long)my_sweeps);
    atomicAdd(a.counters + 1, (unsigned long long)my_updates);
  }
}

}  // namespace

// dynamic shared memory: the warps' tiles, then one mbarrier per warp
static size_t fmsm_smem(int64_t tile_doubles, int warps_per_cta) {
  return (size_t)warps_per_cta * tile_doubles * sizeof(double) + 8 * (size_t)warps_per_cta;
}

cudaError_t fmsm_capacity(int64_t tile_doubles, int warps_per_cta, int* ctas) {
  const size_t smem = fmsm_smem(tile_doubles, warps_per_cta);
  cudaError_t e = ensure_dynamic_smem((const void*)fmsm_dataflow_kernel, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fmsm_dataflow_kernel,
                                                    32 * warps_per_cta, smem);
  if (e != cudaSuccess) return e;
  *ctas = per_sm * sms;
  return cudaSuccess;
}

cudaError_t launch_fmsm(const FmsmArgs& args, int warps_per_cta, int max_ctas, cudaStream_t s,
                        int* launches, int* grid) {
  const size_t smem = fmsm_smem(args.g.tile_doubles, warps_per_cta);
  int ctas = 0;
  cudaError_t e = fmsm_capacity(args.g.tile_doubles, warps_per_cta, &ctas);
  if (e != cudaSuccess) return e;
  if (ctas < 1) return cudaErrorInvalidConfiguration;
  const int need = (args.J + warps_per_cta - 1) / warps_per_cta;
  if (ctas > need) ctas = need;
  if (max_ctas > 0 && ctas > max_ctas) ctas = max_ctas;
  if (grid) *grid = ctas;
  FmsmArgs a = args;
  void* params[] = {&a};
  // workers spin on each other's cells: all CTAs must be co-resident
  e = cudaLaunchCooperativeKernel((const void*)fmsm_dataflow_kernel, dim3(ctas),
                                  dim3(32 * warps_per_cta), params, smem, s);
  *launches += 1;
  return e;
}

}  // namespace eikb200
