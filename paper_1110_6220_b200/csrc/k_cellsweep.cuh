// In-cell sweep engine shared by FMSM (k_cells.cu) and HCM/FHCM
// (k_heapcell.cu): one warp sweeps one cell held in shared memory.
//
// Register pipeline.  Lane t owns sweep rows t, t+32, ... ("slots") and at
// step s processes column s-t-32r of slot r -- every node of one
// anti-diagonal at once, each after its two upwind neighbours, exactly the
// dependency order of the reference's row loop, so values and counters are
// bit-identical.  On the critical path sit only a shuffle (the new value of
// the upwind row) and the fp64 update; the old values, costs and lock bytes of
// the next step are prefetched from shared memory while the current step
// computes.  Lock propagation (heap_cell.cpp:113-122) into the next row goes
// through a ballot, into the lane's own next column through a register, and
// into already-processed neighbours (next sweep) through the lock bytes.
#pragma once

#include "k_common.cuh"

namespace eikb200 {

enum { kSW = 0, kNW = 1, kNE = 2, kSE = 3 };  // SweepDir (local_update.hpp:23)
constexpr int kMaxSlots = 4;                   // cells up to 128 rows

struct CellTile {
  double* U;        // (h+2) x pu values with cross halo, node (x,y) at (y+1)*pu + x+ox
  double* Ct;       // (h+2) x pu costs with halo; < 0 marks exits (and off-grid halo)
  uint8_t* lock;    // h x w lock bytes (1 = unlocked), locked sweeps only
  int pu, w, h;
  int ox;           // column of node x = 0 in a tile row (the west halo is ox-1)
  // A band of rows of a taller cell (big_cell_sweep): the halo row below
  // (y = -1) / above (y = h) is a row of the same cell, so the locking sweep
  // unlocks it like any in-cell neighbour (heap_cell.cpp:113-122).
  bool in_lo = false, in_hi = false;
};

// MODE 0: node_update over all non-exit nodes (FSM inside a cell,
//         fmsm.cpp:200-210); MODE 1: directional_update with the two upwind
//         neighbours (fmsm.cpp:211-221); MODE 2: locking sweep
//         (heap_cell.cpp:98-126).
// Returns the warp-wide "some value decreased" flag and adds this lane's
// processed nodes to `updates` (MODE 2 counts unlocked nodes only).
template <int MODE, int NS>
__device__ bool cell_sweep_ns(const CellTile& T, int dir, int lane, long long& updates_out) {
  int updates = 0;
  const bool iasc = (dir == kSW || dir == kNW);
  const bool jasc = (dir == kSW || dir == kSE);
  const int dx = iasc ? 1 : -1;           // next column in sweep order
  const int dyp = jasc ? T.pu : -T.pu;    // next row in sweep order (value pitch)
  const int dyl = jasc ? T.w : -T.w;      // next row in sweep order (lock pitch)
  const int w = T.w, h = T.h;
  const int x0 = iasc ? 0 : w - 1;        // column of sweep step a = 0
  const bool up_in = jasc ? T.in_lo : T.in_hi;  // upwind / downwind halo row in the cell
  const bool dn_in = jasc ? T.in_hi : T.in_lo;

  int vbase[NS];             // value offset of (a = 0) for this lane's row
  int lbase[NS];             // lock offset of (a = 0)
  bool rvalid[NS];
  double res_prev[NS];       // own new value at the previous column (W)
  double c_prev[NS];         // own cost at the previous column
  bool unW[NS];              // W neighbour unlocked us for this sweep
  unsigned nmask[NS];        // ballot of "unlock my N neighbour" at the last step
  double cur[NS], eo[NS], no[NS], cc[NS], hs[NS], ce[NS], cn[NS], cs[NS];
  uint8_t lk[NS];

#pragma unroll
  for (int r = 0; r < NS; ++r) {
    const int b = lane + 32 * r;
    rvalid[r] = b < h;
    const int y = jasc ? b : h - 1 - b;
    vbase[r] = rvalid[r] ? (y + 1) * T.pu + (x0 + T.ox) : 0;
    lbase[r] = rvalid[r] ? y * w + x0 : 0;
    res_prev[r] = rvalid[r] ? T.U[vbase[r] - dx] : kInf;  // frozen halo column
    c_prev[r] = -1.0;
    unW[r] = false;
    nmask[r] = 0u;
  }

  auto load_step = [&](int s) {
#pragma unroll
    for (int r = 0; r < NS; ++r) {
      const int a = s - lane - 32 * r;
      const bool act = rvalid[r] && a >= 0 && a < w;
      const int o = act ? vbase[r] + dx * a : T.pu + T.ox;  // a safe in-tile offset
      cur[r] = act ? T.U[o] : kInf;
      eo[r] = act ? T.U[o + dx] : kInf;   // old E (halo at the last column)
      no[r] = act ? T.U[o + dyp] : kInf;  // old N (halo on the last row)
      hs[r] = act ? T.U[o - dyp] : kInf;  // S -- only used when it is the halo
      cc[r] = act ? T.Ct[o] : -1.0;
      if (MODE == 2) {
        ce[r] = (act && a + 1 < w) ? T.Ct[o + dx] : -1.0;
        cn[r] = act ? T.Ct[o + dyp] : -1.0;
        cs[r] = act ? T.Ct[o - dyp] : -1.0;
        lk[r] = act ? T.lock[lbase[r] + dx * a] : (uint8_t)0;
      }
    }
  };

  bool changed = false;
  const int last = (h - 1) + (w - 1);
  load_step(0);
  for (int s = 0; s <= last; ++s) {
    double c_cur[NS], c_e[NS], c_n[NS], c_cc[NS], c_hs[NS], c_ce[NS], c_cn[NS], c_cs[NS];
    uint8_t c_lk[NS];
#pragma unroll
    for (int r = 0; r < NS; ++r) {
      c_cur[r] = cur[r];
      c_e[r] = eo[r];
      c_n[r] = no[r];
      c_cc[r] = cc[r];
      c_hs[r] = hs[r];
      c_ce[r] = ce[r];
      c_cn[r] = cn[r];
      c_cs[r] = cs[r];
      c_lk[r] = lk[r];
    }
    // previous-step results of every slot: slot r's lane 0 reads slot r-1's
    // lane 31, which this step's iteration r-1 is about to overwrite
    double rp_old[NS];
    unsigned nm_old[NS];
#pragma unroll
    for (int r = 0; r < NS; ++r) {
      rp_old[r] = res_prev[r];
      nm_old[r] = nmask[r];
    }
    // new value of the upwind row: lane-1 of this slot, lane 31 of the
    // previous slot for lane 0 (the frozen halo for sweep row 0, below)
    double svs[NS];
#pragma unroll
    for (int r = 0; r < NS; ++r) {
      const double send = (lane == 31 && r > 0) ? rp_old[r > 0 ? r - 1 : 0] : rp_old[r];
      svs[r] = __shfl_sync(kFull, send, (lane + 31) & 31);
    }
    // the next step's operands after the shuffles: loads queued ahead of a
    // shuffle in the MIO pipe would delay it
    asm volatile("" ::: "memory");
    if (s < last) load_step(s + 1);  // prefetch while this step computes
#pragma unroll
    for (int r = 0; r < NS; ++r) {
      const int b = lane + 32 * r;
      const int a = s - b;
      const bool act = rvalid[r] && a >= 0 && a < w;
      double sv = svs[r];
      unsigned sbit = 0u;
      if (MODE == 2) {
        if (lane == 0) sbit = (r > 0) ? (nm_old[r > 0 ? r - 1 : 0] >> 31) & 1u : 0u;
        else sbit = (nm_old[r] >> (lane - 1)) & 1u;
      }
      if (b == 0) {
        sv = c_hs[r];
        sbit = 0u;
      }
      const double wv = res_prev[r];
      double res = c_cur[r];
      bool un_n = false, proc = false;
      // Branchy on purpose: a slot/step whose lanes are all inactive or locked
      // skips the fp64 chain (measured faster than predicating it away).
      if (act && c_cc[r] >= 0.0) {
        proc = (MODE != 2) || c_lk[r] || unW[r] || sbit;
        if (proc) {
          const double cand = (MODE == 1) ? quad_update(wv, sv, c_cc[r])
                                          : node_update4(c_e[r], wv, c_n[r], sv, c_cc[r]);
          ++updates;
          if (cand < res) {
            res = cand;
            changed = true;
            T.U[vbase[r] + dx * a] = res;
            if (MODE == 2) {
              uint8_t* lp = T.lock + lbase[r] + dx * a;
              // already-processed W and S neighbours: unlocked for the next sweep
              if (a > 0 && c_prev[r] >= 0.0 && wv > cand) lp[-dx] = 1;
              if ((b > 0 || up_in) && c_cs[r] >= 0.0 && sv > cand) lp[-dyl] = 1;
              un_n = (b + 1 < h) && c_cn[r] >= 0.0 && c_n[r] > cand;
              // the next band's first row: unlocked in memory for this sweep
              if (b + 1 == h && dn_in && c_cn[r] >= 0.0 && c_n[r] > cand) lp[dyl] = 1;
            }
          }
          // relock on processing (heap_cell.cpp:110-111)
          if (MODE == 2) T.lock[lbase[r] + dx * a] = 0;
        }
      }
      if (MODE == 2) {
        const bool dec = proc && res < c_cur[r];
        unW[r] = dec && (a + 1 < w) && c_ce[r] >= 0.0 && c_e[r] > res;
        nmask[r] = __ballot_sync(kFull, un_n);
      }
      c_prev[r] = act ? c_cc[r] : -1.0;
      if (act) res_prev[r] = res;
    }
    __syncwarp();
  }
  updates_out += updates;
  return __any_sync(kFull, changed);
}

// Locking sweep (MODE 2), NS rows per lane (row lane + 32r in slot r): the
// dataflow of cell_sweep_ns<2, NS> restated with branch-free operand loads
// (clamped in-tile addresses) and predicated stores.  SKIP jumps over the
// fp64 chain when no lane holds an unlocked node (a vote on the critical
// path, worth it for mostly-locked sweeps); otherwise only value -> shuffle
// -> update -> select lies between consecutive steps.  Within a sweep no lane
// reads shared memory another lane wrote at an earlier step (operands come
// from later diagonals; unlocks target already-processed nodes for the next
// sweep), and the full-mask shuffles/ballots keep the lanes converged, so
// there is no per-step barrier.
template <bool SKIP, int NS>
__device__ __forceinline__ bool cell_sweep_lock(const CellTile& T, int dir, int lane,
                                                long long& updates_out) {
  const bool iasc = (dir == kSW || dir == kNW);
  const bool jasc = (dir == kSW || dir == kSE);
  const int w = T.w, h = T.h, pu = T.pu, ox = T.ox;
  const int dx = iasc ? 1 : -1;
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
      if (SKIP) {
        // HCM's convergence sweeps (few updates per step): flat predicated
        // stores, no branch between the unrolled steps (band HCM 4-6 % faster;
        // the same form costs FHCM's banded cells 7 %, so it keeps the branch)
        changed = changed | dec;
        if (dec) U[o] = cand[r];
        const bool unl_w = dec & (a > 0) & (cw[r] >= 0.0) & (wv[r] > cand[r]);
        const bool unl_s = dec & ((b > 0) | up_in) & (cs[r] >= 0.0) & (sv[r] > cand[r]);
        const bool unl_nb = dec & (b + 1 == h) & dn_in & (cn[r] >= 0.0) & (n[r] > cand[r]);
        if (unl_w) L[lo - dx] = 1;
        if (unl_s) L[lo - dyl] = 1;
        if (unl_nb) L[lo + dyl] = 1;
      } else if (dec) {
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

// skip (MODE 2): jump over steps in which no node is unlocked -- worth it for
// sweeps that are mostly locked (HCM's convergence sweeps).
template <int MODE>
__device__ bool cell_sweep(const CellTile& T, int dir, int lane, long long& updates,
                           bool skip = false) {
  if (MODE == 2) {
    if (T.h <= 32)
      return skip ? cell_sweep_lock<true, 1>(T, dir, lane, updates)
                  : cell_sweep_lock<false, 1>(T, dir, lane, updates);
    if (T.h <= 64)
      return skip ? cell_sweep_lock<true, 2>(T, dir, lane, updates)
                  : cell_sweep_lock<false, 2>(T, dir, lane, updates);
    if (T.h <= 96)
      return skip ? cell_sweep_lock<true, 3>(T, dir, lane, updates)
                  : cell_sweep_lock<false, 3>(T, dir, lane, updates);
  }
  if (T.h <= 32) return cell_sweep_ns<MODE, 1>(T, dir, lane, updates);
  if (T.h <= 64) return cell_sweep_ns<MODE, 2>(T, dir, lane, updates);
  if (T.h <= 96) return cell_sweep_ns<MODE, 3>(T, dir, lane, updates);
  return cell_sweep_ns<MODE, 4>(T, dir, lane, updates);
}

// Locking sweep of a cell of up to 128 rows as bands of 32 rows, one row per
// lane: with several rows per lane the slots' update chains run one after
// the other (each sqrt carries its own slow-path branch), so a step of two
// slots costs 2.3 steps of one (625-691 against 287-303 cycles alone, 919
// against 385 inside the heap-cell kernel) while two bands of a 64 x 64 cell
// take only 190 steps against 127.  Same band rule as big_cell_sweep below
// (the reference's row loop: a band's upwind halo row holds the previous
// band's new values, unlocks across a band edge go through the lock bytes).
__device__ __forceinline__ bool cell_sweep_lock_bands(const CellTile& T, int dir, int lane,
                                                      long long& updates, bool skip) {
  if (T.h <= 32)
    return skip ? cell_sweep_lock<true, 1>(T, dir, lane, updates)
                : cell_sweep_lock<false, 1>(T, dir, lane, updates);
  const bool jasc = (dir == kSW || dir == kSE);
  bool changed = false;
  const int nb = (T.h + 31) / 32;
  for (int k = 0; k < nb; ++k) {
    const int band = jasc ? k : nb - 1 - k;
    const int y0 = band * 32;
    CellTile S = T;
    S.U = T.U + y0 * T.pu;
    S.Ct = T.Ct + y0 * T.pu;
    S.lock = T.lock + y0 * T.w;
    S.h = min(32, T.h - y0);
    S.in_lo = y0 > 0 || T.in_lo;
    S.in_hi = y0 + S.h < T.h || T.in_hi;
    const bool c = skip ? cell_sweep_lock<true, 1>(S, dir, lane, updates)
                        : cell_sweep_lock<false, 1>(S, dir, lane, updates);
    changed = c || changed;
    __syncwarp();
  }
  return changed;
}

// A cell of any height: bands of at most 128 rows swept one after another in
// the sweep's row order.  A band's upwind halo row is the previous band's
// last row (new values) and its downwind halo row the next band's first row
// (old values), which is exactly the reference's row-loop order, so values
// and counters are the single sweep's.  Lock bytes of the whole cell are
// contiguous (row pitch w), so a band unlocks its neighbours' rows in place.
template <int MODE>
__device__ bool big_cell_sweep(const CellTile& T, int dir, int lane, long long& updates,
                               bool skip = false) {
  if (T.h <= 128) return cell_sweep<MODE>(T, dir, lane, updates, skip);
  const bool jasc = (dir == kSW || dir == kSE);
  bool changed = false;
  const int nb = (T.h + 127) / 128;
  for (int k = 0; k < nb; ++k) {
    const int band = jasc ? k : nb - 1 - k;
    const int y0 = band * 128;
    const int hb = min(128, T.h - y0);
    CellTile S = T;
    S.U = T.U + (size_t)y0 * T.pu;
    S.Ct = T.Ct + (size_t)y0 * T.pu;
    if (T.lock) S.lock = T.lock + (size_t)y0 * T.w;
    S.h = hb;
    S.in_lo = y0 > 0 || T.in_lo;
    S.in_hi = y0 + hb < T.h || T.in_hi;
    changed = cell_sweep<MODE>(S, dir, lane, updates, skip) || changed;
    __syncwarp();
  }
  return changed;
}

}  // namespace eikb200
