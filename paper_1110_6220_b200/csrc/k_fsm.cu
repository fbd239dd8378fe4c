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
#include <type_traits>
#include <cstdlib>
#include <algorithm>

#include "eik_internal.h"
#include "eik_plan.h"
#include "k_common.cuh"

namespace eikb200 {

namespace {

constexpr int kU = 8;          // columns per register block (prefetch unit)
constexpr int kWarpsPerCta = 4;  // strips per CTA up to 4 * SMs strips
constexpr int kMaxWarpsPerCta = 8;
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
__device__ __forceinline__ double poll_slot(const double* p, int* status) {
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

__device__ __forceinline__ unsigned ld_relaxed_u32(const void* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Super-block skipping.  A strip's sweep is cut into super-blocks of kSB
// blocks (kSbCols steps).  In sparse late sweeps most of them are clean: no
// node of the strip's rows (or of the two adjoining edge rows) changed in the
// previous sweep around their columns, no update is in flight inside the
// strip, and the upwind strip's edge row does not change over them in this
// sweep.  Every one of their 8-step blocks would then only forward old values
// (the block-level rule below), so the strip passes over the whole
// super-block without streaming u, C or the change bits: it copies its own
// edge row into the downwind mailbox, re-arms the upwind slots, zeroes its
// change bits and publishes
//   * a summary word per (sweep parity, strip, super-block): bit 0 = some node
//     updated, bit 1 / 2 = the strip's lowest / highest row updated -- read by
//     the next sweep's decision of this strip and its two neighbours;
//   * an edge token per (row direction, strip, super-block) = sweep stamp << 2
//     | state (2: edge row unchanged over the super-block, 3: changed), written
//     after the mailbox values it covers -- read by the downwind strip.
// Lane 0 of the downwind strip visits column q one step after... 31 steps
// before the upwind strip's lane 31 finishes the super-block holding q, so a
// strip needs the upwind tokens g and g+1 to skip its super-block g.  The
// decision only selects between two schedules with the same result.
constexpr int kSB = kFsmSbBlocks;
constexpr int kSbCols = kSB * kU;
constexpr int kSbShift = kSbCols == 16 ? 4 : (kSbCols == 32 ? 5 : (kSbCols == 64 ? 6 : (kSbCols == 128 ? 7 : 8)));
static_assert((1 << kSbShift) == kSbCols && kSbCols >= 16, "super-block: 16..256 steps, power of two");
// the upwind super-block whose lane 31 visits the column lane 0 visits first in super-block g is g + kTokOff
constexpr int kTokOff = 31 >> kSbShift;

struct SbCtx {
  bool pub;                // summaries and tokens are kept (a.sb != null)
  bool skip;               // this sweep may skip (not a forced sweep)
  bool block;              // wait for the upwind tokens (sparse regime) or only look
  bool has_lo, has_hi;     // strips b-1 / b+1 exist
  bool prev_iasc;          // column direction of the previous sweep
  bool lo_is_lane0;        // lane 0 owns the strip's lowest row (jasc)
  int k, flow, b;          // sweep, row direction (mailbox / token set), strip
  int par;                 // parity this sweep writes (change bits and summaries)
};
// [2][nstrips][nsb] summaries by sweep parity, then [2][nstrips][nsb] tokens by row direction
__device__ __forceinline__ unsigned* sb_sum(const FsmArgs& a, int par, int b) {
  return a.sb + ((int64_t)par * a.nstrips + b) * a.nsb;
}
__device__ __forceinline__ unsigned* sb_tok(const FsmArgs& a, int flow, int b) {
  return a.sb + ((int64_t)(2 + flow) * a.nstrips + b) * a.nsb;
}

struct Chan {
  double* gin;            // global mailbox row of the upwind strip (or the dummy row)
  double* gout;           // global mailbox row to the downwind strip (or dummy)
  const double* dnh;      // downwind edge row (old values) in u (or dummy)
  bool in_glob, out_glob; // lane 0 / lane 31 use the mailboxes
  bool in_snap;           // lane 0 reads the upwind part's snapshot row (gin)
  double* sw0;            // lane 0 / lane 31 write their row's snapshot (part
  double* sw31;           // edges of a strip-Jacobi run), or null
};

// Change bits around one block: the four-neighbour change mask of the kU
// columns a block visits, from the previous sweep's bits of rows r-1, r, r+1
// (loaded two blocks ahead; L2 loads, since neighbouring strips on other SMs
// wrote them).
struct ChgWin {
  unsigned u0, u1, c0, c1, d0, d1;
  int sh;
};
__device__ __forceinline__ ChgWin ld_chgwin(const unsigned* rows, int64_t cw, int64_t a) {
  // bit j of the window = absolute column a + j (a >= -64: floor by shift)
  const unsigned* p = rows + (a >> 5) + kChgWordOff;
  ChgWin w;
  w.u0 = __ldcg(p);
  w.u1 = __ldcg(p + 1);
  w.c0 = __ldcg(p + cw);
  w.c1 = __ldcg(p + cw + 1);
  w.d0 = __ldcg(p + 2 * cw);
  w.d1 = __ldcg(p + 2 * cw + 1);
  w.sh = (int)(a & 31);
  return w;
}
// Node at column c is dirty iff a 4-neighbour changed: W/E from the own row
// (columns c-1, c+1), S/N from rows r-1, r+1 (column c).  The window starts
// at column lo-1, so own-row bits j and j+2 and the other rows' bit j+1 are
// the neighbours of column lo+j.
template <bool IASC>
__device__ __forceinline__ unsigned chg_mask(const ChgWin& w) {
  const unsigned long long xu = (((unsigned long long)w.u1 << 32) | w.u0) >> w.sh;
  const unsigned long long xc = (((unsigned long long)w.c1 << 32) | w.c0) >> w.sh;
  const unsigned long long xd = (((unsigned long long)w.d1 << 32) | w.d0) >> w.sh;
  const unsigned d = (unsigned)(xc | (xc >> 2) | (xu >> 1) | (xd >> 1)) & 0xFFu;
  // bit t of the result = the block's step t (column lo+t ascending, lo+7-t descending)
  return IASC ? d : (__brev(d) >> 24);
}

// LSM (lsm_solve, classic_solvers.cpp:160-212) processes exactly the nodes
// that are unlocked when their turn comes; every other node would recompute
// a candidate >= its value, so LSM's values and sweep count are FSM's (the
// reference's lsm_solve and fsm_solve return the same field; checked on every
// golden) and only node_updates differs.  A node is unlocked at its visit in
// sweep k iff a 4-neighbour lowered its value after the node's visit in sweep
// k-1 to below the node's value (classic_solvers.cpp:198-204; a neighbour's
// decreases are monotone, so its current value decides).  "After the visit in
// sweep k-1" = the neighbours downwind in sweep k-1's direction that changed
// in sweep k-1 (previous-sweep change bits) or the neighbours upwind in sweep
// k that changed in sweep k (in-sweep flags).  Sweep 0: a node is unlocked iff
// it neighbours an exit (classic_solvers.cpp:172-182) or an upwind neighbour
// changed -- both iff a neighbour is finite when it is visited.
// lsm_masks: per step t, bit t = the previous sweep changed the node's column
// neighbour (mc) / row neighbour (mr) on sweep k-1's downwind side.
template <bool IASC>
__device__ __forceinline__ void lsm_masks(const ChgWin& w, bool iasc_prev, bool jasc_prev,
                                          unsigned& mc, unsigned& mr) {
  const unsigned long long xu = (((unsigned long long)w.u1 << 32) | w.u0) >> w.sh;
  const unsigned long long xc = (((unsigned long long)w.c1 << 32) | w.c0) >> w.sh;
  const unsigned long long xd = (((unsigned long long)w.d1 << 32) | w.d0) >> w.sh;
  // absolute order: bit j = column lo+j; W = xc bit j, E = bit j+2, S/N = rows
  // r-1 / r+1 at bit j+1
  const unsigned c = (unsigned)(iasc_prev ? (xc >> 2) : xc) & 0xFFu;
  const unsigned r = (unsigned)((jasc_prev ? xd : xu) >> 1) & 0xFFu;
  mc = IASC ? c : (__brev(c) >> 24);
  mr = IASC ? r : (__brev(r) >> 24);
}

// Dirty map of a strip's super-blocks for one sweep, built once at the
// sweep's start (after both neighbouring strips finished the previous sweep)
// into the warp's shared-memory words: bit g = something changed in the
// previous sweep around super-block g (the strip's rows and the adjoining edge
// rows, one column wider on each side), i.e. the super-block is not locally
// clean.  prevw: scratch for the previous sweep's bits in its own order.
constexpr int kMapWords = kFsmSbMaxPerRow / 32;  // (host: longer rows keep sb off)
template <bool IASC>
__device__ __forceinline__ void sb_build_map(const FsmArgs& a, const SbCtx& sb, int lane,
                                             unsigned* prevw, unsigned* curw) {
  const int nsb = a.nsb, nw = (nsb + 31) >> 5;
  const unsigned* s0 = sb_sum(a, sb.par ^ 1, sb.b);
  const unsigned* slo = s0 - nsb;  // strip b-1: its highest row (bit 2)
  const unsigned* shi = s0 + nsb;  // strip b+1: its lowest row (bit 1)
  for (int j = 0; j < nw; ++j) {
    const int g = 32 * j + lane;
    unsigned v = 0;
    if (g < nsb) {
      v = __ldcg(s0 + g) & 1u;
      if (sb.has_lo) v |= __ldcg(slo + g) & 4u;
      if (sb.has_hi) v |= __ldcg(shi + g) & 2u;
    }
    const unsigned w = __ballot_sync(kFull, v != 0u);
    if (lane == 0) prevw[j] = w;
  }
  if (lane == 0) prevw[nw] = 0u;
  __syncwarp();
  const int64_t m = a.m;
  for (int j = 0; j < nw; ++j) {
    const int g = 32 * j + lane;
    int64_t lo = (int64_t)g * kSbCols - 32, hi = (int64_t)g * kSbCols + kSbCols;
    if (sb.prev_iasc != IASC) {
      const int64_t t = m - 1 - hi;
      hi = m - 1 - lo;
      lo = t;
    }
    // the previous sweep's super-block g' holds its sweep-order columns
    // [kSbCols g' - 31, kSbCols g' + kSbCols - 1]: at most 4 of them overlap
    int64_t g0 = lo >> kSbShift, g1 = (hi + 31) >> kSbShift;
    if (g0 < 0) g0 = 0;
    if (g1 > nsb - 1) g1 = nsb - 1;
    bool d = false;
    if (g < nsb && g1 >= g0) {
      const int wi = (int)(g0 >> 5);
      const unsigned long long x =
          ((((unsigned long long)prevw[wi + 1]) << 32) | prevw[wi]) >> (g0 & 31);
      d = (x & ((1ull << (g1 - g0 + 1)) - 1ull)) != 0ull;
    }
    const unsigned w = __ballot_sync(kFull, d);
    if (lane == 0) curw[j] = w;
  }
  __syncwarp();
}

// One sweep of one warp-strip.  IASC selects the column direction at compile
// time so every access in the unrolled block is an immediate offset from a
// per-block pointer; the padded layout (kPad columns of +inf / -1 on both
// sides, a dummy row for lanes past the last grid row) removes every bounds
// check from the step.
//
// Clean-step skipping (LSM's idea, classic_solvers.cpp:160-212, applied to
// the exact sweep): a node whose four neighbours did not change since its
// last evaluation recomputes exactly its old candidate, which cannot be below
// its value, so skipping it changes nothing.  A node is dirty when a
// neighbour changed in the previous sweep (change bits), or in this sweep its
// upwind column (the lane's previous step) or upwind row (lane t-1's previous
// step, or the upwind strip's edge value, sent with its sign bit set when it
// changed).  The decision is taken per 8-step block by one vote: a block in
// which no lane has a dirty node at any step, with no update at the step
// before it, only forwards its old values; any other block computes all 8
// steps (a per-step vote would sit on the fp64 chain).  While lane 0 waits
// for mailbox slots (SLOW), the per-step form with its vote is used.
template <bool IASC, bool LSM>
__device__ __forceinline__ bool sweep_strip(const FsmArgs& a, int lane, int64_t rowp,
                                            const Chan& ch, const unsigned* crd, unsigned* cwr,
                                            unsigned force, unsigned long long* tr, int dprev,
                                            bool jasc, unsigned long long& lcnt, const SbCtx& sb,
                                            const unsigned* sbmap, unsigned& ncomp_out) {
  constexpr int S = IASC ? 1 : -1;
  const int64_t m = a.m, cw = a.cw;
  const int64_t P = a.P;
  const int64_t q0off = IASC ? 0 : m - 1;  // element q of a row sits at base + S*q
  double* pu = a.u + rowp * P + a.pad + q0off - S * lane;
  const double* pc = a.C + rowp * P + a.pad + q0off - S * lane;
  const bool in_g = (lane == 0) && ch.in_glob;  // lane 0 reads the upwind mailbox
  const bool dn_lane = (lane == 31);
  const bool halo_lane = in_g || dn_lane || ((lane == 0) && ch.in_snap);
  double* psw = lane == 0 ? ch.sw0 : (lane == 31 ? ch.sw31 : nullptr);
  if (psw) psw += a.pad + q0off - S * lane;
  double* ph = (lane == 0 ? ch.gin : const_cast<double*>(ch.dnh)) + a.pad + q0off - S * lane;
  double* po = ch.gout + a.pad + q0off - S * lane;
  const bool out_g = dn_lane && ch.out_glob;
  const int nblocks = (int)((m + 31 + kU - 1) / kU);
  const unsigned* crow = crd + rowp * cw;                 // rows rowp-1 .. rowp+1
  unsigned* wrow = cwr + (rowp + 1) * cw + kChgWordOff;   // own row, word 0

  // lo(b) = lowest absolute column block b visits; the window starts at lo-1
  auto lo_of = [&](int b) -> int64_t {
    const int64_t q = (int64_t)b * kU - lane;
    return IASC ? q : m - 1 - q - (kU - 1);
  };
  // LSM: previous-sweep direction (dprev < 0: sweep 0 of the solve)
  const bool iasc_prev = dprev == 0 || dprev == 1, jasc_prev = dprev == 0 || dprev == 3;
  unsigned pm = 0, lmc = 0, lmr = 0;
  ChgWin wa, wb;
  double cu[kU + 1], cc[kU], hv[kU];
  double nu[kU + 1], nc[kU], nh[kU];
  double res_prev = kInf;
  bool upd_prev = false, changed = false;
  int q0 = -lane;
  const double sent = __longlong_as_double((long long)kSent);
  // change bits of the word holding the next column to visit
  int64_t wcur = (IASC ? (int64_t)-lane : m - 1 + lane) >> 5;
  unsigned acc = 0;
  unsigned npoll = 0, ncomp = 0, nskip = 0;

  // (re)start the register pipeline at block blk: at the sweep's start and
  // after skipped super-blocks (the lane's previous column is old there)
  auto prime = [&](int blk) {
    const ChgWin w0 = ld_chgwin(crow, cw, lo_of(blk) - 1);
    pm = force ? force : chg_mask<IASC>(w0);
    if (LSM && dprev >= 0) lsm_masks<IASC>(w0, iasc_prev, jasc_prev, lmc, lmr);
    wa = ld_chgwin(crow, cw, lo_of(blk + 1) - 1);
    wb = ld_chgwin(crow, cw, lo_of(blk + 2) - 1);
#pragma unroll
    for (int t = 0; t <= kU; ++t) cu[t] = pu[S * t];
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      cc[t] = __ldg(pc + S * t);
      hv[t] = halo_lane ? __ldcg(ph + S * t) : kInf;
    }
    res_prev = pu[-S];  // padding (+inf) ahead of the row's first column
    upd_prev = false;
  };

  // this block's change bits into the row's words (absolute columns lo..lo+7)
  auto put_bits = [&](int blk, unsigned um) {
    const int64_t lo = lo_of(blk);
    const unsigned ub = IASC ? um : (__brev(um) >> 24);
    const int64_t wl = lo >> 5;
    const unsigned long long x = (unsigned long long)ub << (lo & 31);
    const unsigned lowp = (unsigned)x, highp = (unsigned)(x >> 32);
    const int64_t wn = (IASC ? lo + kU : lo - 1) >> 5;  // word of the next column
    if (IASC) {
      acc |= lowp;
      if (wn != wl) {
        __stcg(wrow + wl, acc);
        acc = highp;
      }
    } else if (wcur != wl) {  // straddles: word wl+1 first, then wl
      __stcg(wrow + wcur, acc | highp);
      acc = lowp;
    } else {
      acc |= lowp;
      if (wn != wl) {
        __stcg(wrow + wl, acc);
        acc = 0;
      }
    }
    wcur = wn;
  };

  // ---- super-block skipping (see SbCtx) ----------------------------------
  const unsigned stamp = (unsigned)(sb.k + 1) << 2;
  const int nsb = a.nsb;
  auto dirty_at = [&](int g) -> bool { return (sbmap[g >> 5] >> (g & 31)) & 1u; };
  // first locally dirty super-block >= g (nsb if none): lane L looks at word L
  // and L + 32
  auto next_dirty = [&](int g) -> int {
    int best = nsb;
    const int nw = (nsb + 31) >> 5;
#pragma unroll
    for (int h = 0; h < kMapWords / 32; ++h) {
      const int wi = 32 * h + lane;
      unsigned w = wi < nw ? sbmap[wi] : 0u;
      if (wi == (g >> 5)) w &= ~0u << (g & 31);
      if (wi < (g >> 5)) w = 0u;
      const unsigned bal = __ballot_sync(kFull, w != 0u);
      if (bal && best == nsb) {
        const int src = __ffs(bal) - 1;
        const unsigned ww = __shfl_sync(kFull, w, src);
        best = 32 * (32 * h + src) + __ffs(ww) - 1;
      }
    }
    return best < nsb ? best : nsb;
  };
  // Pass over a run of locally clean super-blocks starting at block blk, as
  // far as the upwind tokens already allow (at most 30 at a time); returns the
  // number of super-blocks passed (0: the upwind edge row changes, or its
  // tokens are not there yet and the strip does not wait for them).
  auto try_skip = [&](int blk) -> int {
    const int g = blk / kSB;
    int rmax = next_dirty(g) - g;
    if (rmax > 30) rmax = 30;
    int r = rmax;
    if (ch.in_glob) {
      // lane 0's columns of super-blocks g .. g+r-1 are visited by the upwind
      // lane 31 in its super-blocks g + kTokOff .. g + kTokOff + r
      const unsigned* tp = sb_tok(a, sb.flow, sb.flow ? sb.b + 1 : sb.b - 1) + g + kTokOff + lane;
      const bool mine = lane <= rmax && g + kTokOff + lane < nsb;
      unsigned tk = mine ? ld_relaxed_u32(tp) : (stamp | 2u);
      if (sb.block && lane < 2 && mine) {
        long long spins = 0;
        while ((tk >> 2) != (stamp >> 2)) {
          if (++spins > kSpinCap) {
            atomicExch(a.status, kStatusWatchdog);
            break;
          }
          if ((spins & 1023) == 0 && *(volatile int*)a.status == kStatusWatchdog) break;
          __nanosleep(40);
          tk = ld_relaxed_u32(tp);
        }
      }
      const unsigned bad = __ballot_sync(kFull, tk != (stamp | 2u));
      const int lead = bad ? __ffs(bad) - 1 : 32;
      if (lead - 1 < r) r = lead - 1;
      if (r <= 0) return 0;
    }
    int nb = kSB * r;
    if (nb > nblocks - blk) nb = nblocks - blk;
    const int ncol = kSbCols * r;  // steps (columns per lane) of the run
    if (ch.in_glob) {
      // re-arm the upwind slots of lane 0's columns (their values have landed:
      // the tokens are written after them)
      double* gin_q0 = (double*)__shfl_sync(kFull, (unsigned long long)ph, 0);
      const int64_t q0_0 = (int64_t)q0 + lane;
      for (int j = lane; j < ncol; j += 32) {
        const int64_t q = (int64_t)g * kSbCols + j;
        if (q < m) __stcg(gin_q0 + S * (q - q0_0), sent);
      }
    }
    if (ch.out_glob) {
      // the strip's edge row (lane 31's) over the run into the downwind mailbox
      const int64_t q0_31 = (int64_t)q0 + lane - 31;
      const double* edge_q0 = (const double*)__shfl_sync(kFull, (unsigned long long)pu, 31);
      double* gout_q0 = (double*)__shfl_sync(kFull, (unsigned long long)po, 31);
      const int64_t qe0 = (int64_t)g * kSbCols - 31;
      for (int j0 = lane; j0 < ncol; j0 += 8 * 32) {
        double ev[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int jj = j0 + 32 * j;
          const int64_t q = qe0 + jj;
          ev[j] = (jj < ncol && q >= 0 && q < m) ? __ldcg(edge_q0 + S * (q - q0_31)) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int jj = j0 + 32 * j;
          const int64_t q = qe0 + jj;
          if (jj < ncol && q >= 0 && q < m) __stcg(gout_q0 + S * (q - q0_31), ev[j]);
        }
      }
      __threadfence();  // the values before the tokens
      __syncwarp();
      if (lane < r) __stcg(sb_tok(a, sb.flow, sb.b) + g + lane, stamp | 2u);
    }
    if (lane < r) __stcg(sb_sum(a, sb.par, sb.b) + g + lane, 0u);
    // zero change bits over the lane's ncol columns: the open word (acc) and
    // the whole words the run passes; the word of the next column to visit
    // stays open
    {
      const int64_t lo = lo_of(blk);
      const int64_t wn = (IASC ? lo + ncol : lo + kU - 1 - ncol) >> 5;
      if (wn != wcur) {
        __stcg(wrow + wcur, acc);
        acc = 0u;
        if (IASC) for (int64_t w = wcur + 1; w < wn; ++w) __stcg(wrow + w, 0u);
        else for (int64_t w = wcur - 1; w > wn; --w) __stcg(wrow + w, 0u);
        wcur = wn;
      }
    }
    pu += S * kU * nb;
    pc += S * kU * nb;
    ph += S * kU * nb;
    po += S * kU * nb;
    q0 += kU * nb;
    nskip += (unsigned)r;
    return r;
  };

  unsigned sb_um = 0;
  int blk = 0;
  unsigned long long t_norm = 0;  // trace: time and blocks in the computed runs
  unsigned n_norm = 0;
  // Outer loop: a run of skipped super-blocks, then a run of computed blocks
  // with the register pipeline primed once (the pipeline is dead across the
  // skip phase, so the skip code shares its registers).
  bool local_clean = sb.skip && !dirty_at(0);
  for (;;) {
    if (local_clean) {
      for (;;) {
        const int r = try_skip(blk);
        blk += kSB * r;
        if (r == 0 || blk >= nblocks || dirty_at(blk / kSB)) break;
      }
      if (blk >= nblocks) break;
    }
    const unsigned long long tn0 = tr ? globaltimer() : 0ull;
    const int blk_n0 = blk;
    if (a.start_ahead > 0 && in_g) {
      // start a computed run only once the upwind strip is start_ahead
      // columns ahead: the block prefetches then find their slots filled and
      // the run never drops to the per-step polling path
      // (lane 0 past the row's end has consumed and re-armed every slot)
      int64_t q = (int64_t)q0 + a.start_ahead;
      if (q > m - 1) q = m - 1;
      if (q0 < m) (void)poll_slot(ph + S * (q - q0), a.status);
    }
    __syncwarp();
    prime(blk);
    for (;;) {
    {
      // land the previous prefetch before issuing the next one: the steps
      // below then never wait on a scoreboard shared with fresh loads
      unsigned x = 0;
#pragma unroll
      for (int t = 0; t < kU; ++t)
        x |= (unsigned)__double2hiint(cu[t + 1]) ^ (unsigned)__double2hiint(cc[t]) ^
             (unsigned)__double2hiint(hv[t]);
      if (x == 0x7ff7dea1u) atomicAdd(a.status + 7, 1);  // never true
    }
#pragma unroll
    for (int t = 1; t <= kU; ++t) nu[t] = pu[S * (kU + t)];
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      nc[t] = __ldg(pc + S * (kU + t));
      nh[t] = halo_lane ? __ldcg(ph + S * (kU + t)) : kInf;
    }
    const unsigned pm_next = force ? force : chg_mask<IASC>(wa);
    unsigned lmc_next = 0, lmr_next = 0;
    if (LSM && dprev >= 0) lsm_masks<IASC>(wa, iasc_prev, jasc_prev, lmc_next, lmr_next);
    wa = wb;
    wb = ld_chgwin(crow, cw, lo_of(blk + 3) - 1);
    unsigned um = 0;
    // The block's steps.  SLOW: lane 0 found an empty mailbox slot among the
    // block's prefetched values and polls per step; otherwise the mailbox
    // costs the steps nothing (no divergent branch on lane 0) and the slots
    // are re-armed after the block.
    auto steps = [&](auto slow_tag, auto all_tag) {
      constexpr bool SLOW = decltype(slow_tag)::value;
      constexpr bool ALL = decltype(all_tag)::value;  // compute every step (no per-step vote)
#pragma unroll
      for (int t = 0; t < kU; ++t) {
        const int q = q0 + t;
        double h = hv[t];
        if (SLOW && in_g && q < m) {
          if (is_sent(h)) {
            h = poll_slot(ph + S * t, a.status);
            ++npoll;
            // the upwind strip is close ahead: every later slot loaded so far
            // predates its write too; reload them once instead of polling
            // each one a round trip apart
#pragma unroll
            for (int t2 = t + 1; t2 < kU; ++t2) hv[t2] = __ldcg(ph + S * t2);
#pragma unroll
            for (int t2 = 0; t2 < kU; ++t2) nh[t2] = __ldcg(ph + S * (kU + t2));
          }
          ph[S * t] = sent;  // re-arm the slot for the next sweep
        }
        // the upwind strip's edge value carries "changed in this sweep" in its sign
        const bool h_chg = (lane == 0) && q < m && (__double_as_longlong(h) < 0);
        const bool dirty = ((pm >> t) & 1u) || upd_prev || h_chg;
        const double cur = cu[t];
        double res = cur;
        bool upd = false;
        if (ALL || __any_sync(kFull, dirty)) {
          ++ncomp;
          double sv = __shfl_up_sync(kFull, res_prev, 1);
          double nv = __shfl_down_sync(kFull, cu[t + 1], 1);
          const double hval = fabs(h);
          if (lane == 0) sv = hval;
          if (lane == 31) nv = hval;
          const double c = cc[t];
          const double cand = node_update4_fast(cu[t + 1], res_prev, nv, sv, c);
          upd = (c > 0.0) && (cand < cur);  // exits / padding carry c = -1
          if (LSM) {
            // lane t-1's step at this column (its previous step) lowered it
            const unsigned bal = __ballot_sync(kFull, upd_prev);
            const bool row_up_upd = lane == 0 ? h_chg : ((bal >> (lane - 1)) & 1u);
            // (both rules evaluated and selected: a branch here would split
            // the block's eight steps into separate scheduling regions)
            const bool unl0 = (cu[t + 1] < kInf) | (res_prev < kInf) | (nv < kInf) | (sv < kInf);
            // the changed neighbour's current value: the column one is
            // downwind now iff the column direction did not turn (old value
            // cu[t+1]) else upwind (new value res_prev); rows alike (nv / sv)
            const double vpc = (iasc_prev == IASC) ? cu[t + 1] : res_prev;
            const double vpr = (jasc_prev == jasc) ? nv : sv;
            const bool unl1 = ((((lmc >> t) & 1u) != 0u) & (vpc < cur)) |
                              ((((lmr >> t) & 1u) != 0u) & (vpr < cur)) |
                              (upd_prev & (res_prev < cur)) | (row_up_upd & (sv < cur));
            const bool unl = dprev < 0 ? unl0 : unl1;
            lcnt += (unl && c > 0.0) ? 1ull : 0ull;
          }
          if (upd) {
            res = cand;
            pu[S * t] = cand;
          }
        }
        changed |= upd;
        um |= (unsigned)upd << t;
        const double ov = upd ? -res : res;
        if (out_g) __stcg(po + S * t, ov);  // straight to L2: the next strip polls it
        if (psw) __stcg(psw + S * t, res);  // part edge row for the next sweep
        res_prev = res;
        upd_prev = upd;
      }
      if (!SLOW && in_g) {
#pragma unroll
        for (int t = 0; t < kU; ++t)
          if (q0 + t < m) ph[S * t] = sent;  // re-arm the block's slots
      }
    };
    bool need_poll = false;
    if (in_g) {
#pragma unroll
      for (int t = 0; t < kU; ++t) need_poll |= (q0 + t < m) && is_sent(hv[t]);
    }
    if (__any_sync(kFull, need_poll)) {
      steps(std::true_type{}, std::false_type{});
    } else {
      // Block-level decision (one vote per 8 steps): no lane dirty at any
      // step -> the block only forwards its old values; otherwise every step
      // computes (a per-step vote would sit on the fp64 chain: measured
      // slower, C2 44.3 vs 41.9 ms)
      bool bd = (pm != 0u) || upd_prev;
      if (in_g) {
#pragma unroll
        for (int t = 0; t < kU; ++t)
          bd = bd || ((q0 + t < m) && (__double_as_longlong(hv[t]) < 0));
      }
      if (__any_sync(kFull, bd)) {
        steps(std::false_type{}, std::true_type{});
      } else {
#pragma unroll
        for (int t = 0; t < kU; ++t) {
          const double cur = cu[t];
          if (out_g) __stcg(po + S * t, cur);
          if (psw) __stcg(psw + S * t, cur);
        }
        if (in_g) {
#pragma unroll
          for (int t = 0; t < kU; ++t)
            if (q0 + t < m) ph[S * t] = sent;  // re-arm the block's slots
        }
        res_prev = cu[kU - 1];
        upd_prev = false;
      }
    }
    put_bits(blk, um);
    if (sb.pub) {
      // end of a super-block: its summary for the next sweep's decisions and
      // the edge token for the downwind strip
      sb_um |= um;
      if (((blk + 1) & (kSB - 1)) == 0 || blk + 1 == nblocks) {
        const unsigned bal = __ballot_sync(kFull, sb_um != 0u);
        const bool e0 = bal & 1u, e31 = (bal >> 31) & 1u;
        const int g = blk / kSB;
        if (lane == 0)
          __stcg(sb_sum(a, sb.par, sb.b) + g, (bal ? 1u : 0u) | ((sb.lo_is_lane0 ? e0 : e31) ? 2u : 0u) |
                                   ((sb.lo_is_lane0 ? e31 : e0) ? 4u : 0u));
        if (out_g) {  // lane 31 wrote the mailbox values itself
          if (!e31) __threadfence();
          __stcg(sb_tok(a, sb.flow, sb.b) + g, stamp | (e31 ? 3u : 2u));
        }
        sb_um = 0;
      }
    }
    pm = pm_next;
    if (LSM) {
      lmc = lmc_next;
      lmr = lmr_next;
    }
    pu += S * kU;
    pc += S * kU;
    ph += S * kU;
    po += S * kU;
    if (psw) psw += S * kU;
    q0 += kU;
    cu[0] = cu[kU];
#pragma unroll
    for (int t = 1; t <= kU; ++t) cu[t] = nu[t];
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      cc[t] = nc[t];
      hv[t] = nh[t];
    }
    ++blk;
    if (blk >= nblocks) break;
    // at a super-block boundary with no update in flight and nothing changed
    // around the next super-block: leave the pipeline for the skip phase
    if (sb.skip && (blk & (kSB - 1)) == 0 && !dirty_at(blk / kSB) &&
        !__any_sync(kFull, upd_prev)) {
      local_clean = true;
      break;
    }
    }
    if (tr) {
      t_norm += globaltimer() - tn0;
      n_norm += (unsigned)(blk - blk_n0);
    }
    if (blk >= nblocks) break;
  }
  __stcg(wrow + wcur, acc);
  if (tr && lane == 0) {
    tr[3] = npoll;
    tr[4] = ncomp;
    tr[5] = nskip;
    tr[6] = t_norm;
    tr[7] = n_norm;
  }
  ncomp_out = ncomp;
  return changed;
}

template <bool LSM>
__global__ void __launch_bounds__(32 * kMaxWarpsPerCta)
fsm_wavefront_kernel(FsmArgs a) {
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int b = blockIdx.x * (blockDim.x >> 5) + w;
  if (b >= a.nstrips) return;  // warps past the last grid row do not exist
  const int64_t n = a.n, P = a.P;
  __shared__ unsigned s_sbmap[kMaxWarpsPerCta][2][kMapWords + 2];
  unsigned* const sbprev = s_sbmap[w][0];
  unsigned* const sbmap = s_sbmap[w][1];
  // steps this strip computed in its previous sweep (a continuing launch
  // reads what its predecessor left)
  unsigned prev_comp = (a.cont && a.sb) ? a.sb[(int64_t)4 * a.nstrips * a.nsb + b] : ~0u;

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
    unsigned long long* tr = (a.trace && k < kTraceSweeps)
                                 ? a.trace + ((int64_t)k * a.nstrips + b) * kTraceWords
                                 : nullptr;
    if (tr && lane == 0) tr[0] = globaltimer();

    // The strip downwind of us in sweep k must have finished sweep k-1: its
    // edge row is our "old" neighbour row, and the hand-off slots it emptied
    // must be visible before we refill them.  The strip upwind of us must
    // have finished sweep k-1 too: its edge row's change bits of sweep k-1
    // make our first row dirty (when the direction turns it finishes k-1
    // after us, but before it sends us any value of sweep k).  Once per sweep.
    {
      int ok = 1;
      if (k > 0 && has_dn && lane == 0)
        ok = wait_ge_u64(&a.prog[jasc ? b + 1 : b - 1], (unsigned long long)k, a.status);
      if (k > 0 && has_up && lane == 0 && ok)
        ok = wait_ge_u64(&a.prog[jasc ? b - 1 : b + 1], (unsigned long long)k, a.status);
      if (!__shfl_sync(kFull, ok, 0)) return;
    }
    double* dummy = a.u + n * P;  // all +inf
    // strip-Jacobi partitions: a strip at a part edge reads the neighbouring
    // part's edge row from the previous sweep's snapshot and writes its own
    const int ps = a.part_strips;
    const bool first_of_part = ps > 0 && b > 0 && (b % ps) == 0;
    const bool last_of_part = ps > 0 && b + 1 < a.nstrips && ((b + 1) % ps) == 0;
    const bool up_jac = has_up && (jasc ? first_of_part : last_of_part);
    const bool dn_jac = has_dn && (jasc ? last_of_part : first_of_part);
    const int nbnd = ps > 0 ? (a.nstrips - 1) / ps : 0;
    auto snap_row = [&](int par, int bnd, int side) -> double* {
      return a.snap + ((((int64_t)par * nbnd + bnd) * 2 + side) * P);
    };
    const int blo = ps > 0 ? b / ps - 1 : 0, bhi = ps > 0 ? b / ps : 0;  // boundaries below / above
    const int rd = (k + 1) & 1, wr = k & 1;
    Chan ch;
    ch.in_glob = has_up && !up_jac;
    ch.out_glob = has_dn && !dn_jac;
    ch.in_snap = up_jac;
    ch.gin = ch.in_glob ? a.mbox + ((int64_t)flow * a.nstrips + (jasc ? b - 1 : b + 1)) * P
                        : (up_jac ? (jasc ? snap_row(rd, blo, 0) : snap_row(rd, bhi, 1)) : dummy);
    ch.gout = ch.out_glob ? a.mbox + ((int64_t)flow * a.nstrips + b) * P : dummy;
    ch.dnh = dn_jac ? (jasc ? snap_row(rd, bhi, 1) : snap_row(rd, blo, 0))
                    : (has_dn ? a.u + dnrow * P : dummy);
    ch.sw0 = up_jac ? (jasc ? snap_row(wr, blo, 1) : snap_row(wr, bhi, 0)) : nullptr;
    ch.sw31 = dn_jac ? (jasc ? snap_row(wr, bhi, 0) : snap_row(wr, blo, 1)) : nullptr;

    if (tr && lane == 0) tr[1] = globaltimer();
    // change bits: read sweep k-1's parity, write sweep k's; the first sweep
    // of a launch evaluates every node (the bits of an earlier launch do not
    // describe changes made since, e.g. ghost rows set by the host)
    const int64_t cpar = (n + 3) * a.cw;
    // a continuing launch (a.cont: sweep-level control, one launch after
    // another on the same values) starts from the bits its predecessor left:
    // par0 lines the parities up, and rows written in between were marked by
    // mark_rows_kernel
    const int par = (k + a.par0) & 1;
    const unsigned* crd = a.chg + (int64_t)(par ^ 1) * cpar;
    unsigned* cwr = a.chg + (int64_t)par * cpar;
    const unsigned force = ((k == 0 && !a.cont) || a.noskip) ? 0xFFu : 0u;
    const int dprev = (k == 0 && !a.cont) ? -1 : ((a.first_sweep + k + 3) & 3);
    unsigned long long lcnt = 0;
    SbCtx sb;
    sb.pub = a.sb != nullptr;
#ifdef SB_NOSKIP
    sb.skip = false;
#else
    sb.skip = sb.pub && !force;
#endif
#ifdef SB_NOPUB
    sb.pub = false;
#endif
    // sparse regime (fewer than (m + 31) / sb_wait_div steps computed last
    // sweep): wait for the upwind tokens; otherwise only use them if present
    sb.block = a.sb_wait_div > 0 && prev_comp < (unsigned)((a.m + 31) / a.sb_wait_div);
    sb.prev_iasc = dprev == 0 || dprev == 1;
    sb.lo_is_lane0 = jasc;
    sb.has_lo = b > 0;
    sb.has_hi = b + 1 < a.nstrips;
    sb.k = k;
    sb.par = par;
    sb.flow = flow;
    sb.b = b;
    if (sb.skip) {
      if (iasc) sb_build_map<true>(a, sb, lane, sbprev, sbmap);
      else sb_build_map<false>(a, sb, lane, sbprev, sbmap);
    }
    unsigned ncomp = 0;
    const bool changed =
        iasc ? sweep_strip<true, LSM>(a, lane, rowp, ch, crd, cwr, force, tr, dprev, jasc, lcnt, sb,
                                      sbmap, ncomp)
             : sweep_strip<false, LSM>(a, lane, rowp, ch, crd, cwr, force, tr, dprev, jasc, lcnt, sb,
                                       sbmap, ncomp);
    prev_comp = __shfl_sync(kFull, ncomp, 0);
    if (a.sb && lane == 0) a.sb[(int64_t)4 * a.nstrips * a.nsb + b] = prev_comp;
    if (*(volatile int*)a.status == kStatusWatchdog) return;
    if (LSM) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lcnt += __shfl_xor_sync(kFull, lcnt, o);
      if (lane == 0 && lcnt) atomicAdd(&a.lsm_cnt[k], lcnt);
    }

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

// Padded layout: row r (-1..n; rows -1 and n are dummies) holds element i at
// r*P + pad + i; padding columns and the dummy rows carry u = +inf, C = -1.
__global__ void prepare_padded_kernel(const double* __restrict__ F, double* __restrict__ C,
                                      double* __restrict__ u, int64_t m, int64_t n, int64_t P,
                                      int64_t pad, double h, int* __restrict__ status) {
  const int64_t total = (n + 2) * P;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / P - 1, i = idx - (r + 1) * P - pad;
    double c = -1.0;
    if (r >= 0 && r < n && i >= 0 && i < m) {
      const double f = F[r * m + i];
      if (!(f > 0.0) || !(f < kInf)) atomicExch(&status[0], 1);
      c = h / f;  // same IEEE division as local_update.hpp:33
      // the update's square root runs without sqrt()'s out-of-range path
      // (k_common.cuh sqrt_rn_normal): 2 c^2 must stay in [2^-970, 2^1024)
      if (!(c >= 0x1p-480) || !(c <= 0x1p500)) atomicExch(&status[0], 1);
    }
    C[idx - P] = c;
    u[idx - P] = kInf;
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

__global__ void fill_kernel(double* __restrict__ p, int64_t count, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}


// Rows written between two launches of a sweep-by-sweep solve (ghost rows of
// a sharded run, eik_plan_set_rows): copy them in and mark what changed as
// "changed in the previous sweep" -- change bits of the parity the next
// launch reads, and the summary words of the row's strip (every super-block:
// the skewed indexing of the sweep to come is not known here) -- so that a
// continuing launch need not evaluate every node.
__global__ void set_rows_marked_kernel(double* __restrict__ u, const double* __restrict__ src,
                                       int64_t row0, int64_t nrows, int64_t m, int64_t P,
                                       int64_t pad, unsigned* __restrict__ chg_par, int64_t cw,
                                       unsigned* __restrict__ sum_par, int nsb) {
  const int lane = threadIdx.x & 31;
  const int64_t words = (m + 31) / 32;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = warp; it < nrows * words; it += nwarps) {
    const int64_t r = it / words, w = it - r * words, row = row0 + r, i = 32 * w + lane;
    bool ch = false;
    if (i < m) {
      const double v = src[r * m + i];
      double* p = u + row * P + pad + i;
      ch = __double_as_longlong(v) != __double_as_longlong(*p);
      *p = v;
    }
    const unsigned mask = __ballot_sync(kFull, ch);
    if (mask && lane == 0) {
      atomicOr(chg_par + (row + 1) * cw + kChgWordOff + w, mask);
      const unsigned bits = 1u | ((row & 31) == 0 ? 2u : 0u) | ((row & 31) == 31 ? 4u : 0u);
      unsigned* sp = sum_par + (row >> 5) * (int64_t)nsb;
      if ((atomicOr(sp, bits) & bits) != bits)  // first marker of this strip fills the rest
        for (int g = 1; g < nsb; ++g) atomicOr(sp + g, bits);
    }
  }
}

}  // namespace

cudaError_t launch_fill(double* p, int64_t count, double v, cudaStream_t s, int* launches) {
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  fill_kernel<<<(unsigned)blocks, 256, 0, s>>>(p, count, v);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_set_rows_marked(double* u, const double* src, int64_t row0, int64_t nrows,
                                   int64_t m, int64_t P, int64_t pad, unsigned* chg_par, int64_t cw,
                                   unsigned* sum_par, int nsb, cudaStream_t s) {
  int64_t warps = nrows * ((m + 31) / 32);
  int64_t blocks = (warps + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  set_rows_marked_kernel<<<(unsigned)blocks, 256, 0, s>>>(u, src, row0, nrows, m, P, pad, chg_par,
                                                         cw, sum_par, nsb);
  return cudaGetLastError();
}

cudaError_t launch_prepare(const double* F, double* C, double* u, int64_t m, int64_t n,
                           int64_t P, int64_t pad, double h, const int64_t* exits,
                           const double* cost, int64_t n_exit, int* status, cudaStream_t s,
                           int* launches) {
  const int threads = 256;
  int64_t blocks = ((n + 2) * P + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  prepare_padded_kernel<<<(unsigned)blocks, threads, 0, s>>>(F, C, u, m, n, P, pad, h, status);
  int64_t eb = (n_exit + threads - 1) / threads;
  if (eb > 1024) eb = 1024;
  if (eb < 1) eb = 1;
  mark_exits_kernel<<<(unsigned)eb, threads, 0, s>>>(exits, cost, n_exit, m, P, pad, C, u);
  *launches += 2;
  return cudaGetLastError();
}

// Strips per CTA: 4, or the same number on every SM when the grid has more
// strips than 4 per SM (config 5: 1025 strips -> 7 per CTA, one CTA per SM,
// instead of 1-2 CTAs of 4 per SM whose 8-warp SMs would pace the pipeline).
static int fsm_wpc(int nstrips) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (knobs().fsm_wpc > 0) return std::min(kMaxWarpsPerCta, knobs().fsm_wpc);
  if (nstrips <= kWarpsPerCta * sms) return kWarpsPerCta;
  return std::min(kMaxWarpsPerCta, (nstrips + sms - 1) / sms);
}

static const void* fsm_kernel_fn(bool lsm = false) {
  return lsm ? (const void*)fsm_wavefront_kernel<true> : (const void*)fsm_wavefront_kernel<false>;
}

cudaError_t fsm_capacity(int nstrips, int* need, int* ctas, bool lsm) {
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int wpc = fsm_wpc(nstrips);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fsm_kernel_fn(lsm),
                                                                32 * wpc, 0);
  if (e != cudaSuccess) return e;
  *need = (nstrips + wpc - 1) / wpc;
  *ctas = per_sm * sms;
  return cudaSuccess;
}

cudaError_t launch_fsm(const FsmArgs& args, cudaStream_t s, int* launches, int* grid) {
  const int wpc = fsm_wpc(args.nstrips);
  const int ctas = (args.nstrips + wpc - 1) / wpc;
  if (grid) *grid = ctas;
  FsmArgs a = args;
  void* params[] = {&a};
  // Strips spin on each other's progress, so every CTA must be co-resident:
  // a cooperative launch guarantees it (or fails loudly).
  cudaError_t e = cudaLaunchCooperativeKernel(fsm_kernel_fn(a.lsm_cnt != nullptr), dim3(ctas),
                                              dim3(32 * wpc), params, 0, s);
  *launches += 1;
  return e;
}

}  // namespace eikb200
