// Kernel (3): the heap-cell methods HCM / FHCM (/root/reference/proj/src/
// heap_cell.cpp:13-336) as a device-resident speculative exact replay.
//
// The reference pops cells from a (value, id) min-heap one at a time; FHCM's
// output depends on that exact order (SURVEY.md finding 6), so the order is
// replayed exactly.  A cell's processing (border snapshot, reset_locks,
// locking sweeps, the four border scans) reads only its own nodes, the cross
// halo from its 4 neighbour cells, its flags and its first-removal bit.  All
// of that changes only when the cell itself or a neighbour is committed, so
// version[c] = number of commits in {c} u N(c) identifies the inputs:
//
//   * worker warps process cells near the top of the heap into a spare value
//     slot and tag the result record with the version they read (a "plain"
//     speculation);
//   * a worker may also process a cell x on top of the pending, not yet
//     committed results of a set A of neighbours expected to be committed
//     before x (a "chained" speculation).  Every result carries a unique
//     instance number and the committer records the last committed instance
//     of each cell; the chained result is valid iff x's version advanced by
//     exactly |A| and each y in A last committed the very instance x read.
//     Neighbours of x are not adjacent to each other, so their commits
//     commute and the test is exact;
//   * the committer (CTA 0, warp 0) pops cells in the reference's order and
//     commits a valid result -- a slot flip plus the precomputed scans -- and
//     otherwise processes the cell itself.
//
// Each cell has three value slots: the committed one and one per speculation
// kind.  The slot of kind K changes role only when a result of kind K is
// committed, so a writer whose result went stale only ever writes into a slot
// no valid result lives in.  The committer's heap and cell values live in its
// shared memory when they fit (uint16 indices), else in global.  Every value
// and counter equals the reference's (tests/test_gpu_cells.py).
#include <algorithm>

#include <cooperative_groups.h>

#include "eik_internal.h"
#include "k_cellsweep.cuh"
#include "k_common.cuh"

namespace eikb200 {

namespace {

enum { SW = 0, NW = 1, NE = 2, SE = 3 };
enum { WEST = 0, EAST = 1, SOUTH = 2, NORTH = 3 };
__device__ const int kFlagOrder[4] = {NE, NW, SE, SW};  // heap_cell.cpp:13-14
__device__ const int kRotation[4] = {SW, NW, NE, SE};   // heap_cell.cpp:15-16

using u64 = unsigned long long;

// ---- per-cell state word -----------------------------------------------------
// low 32 bits: 0-3 raised sweep flags, 4 first removal done, 5-6 committed
//   slot, 8-31 version (commits in {c} u N(c), mod 2^24)
// high 32 bits: 0-1 slot of the plain speculation (the chained one uses the
//   third), 2-9 the committed slot of the neighbour on side d at bits 2+2d
//   (kept current by the committer, which rewrites this word whenever that
//   neighbour commits; the halo is then located without reading its state)
__device__ __forceinline__ unsigned st_flags(u64 s) { return (unsigned)s & 15u; }
__device__ __forceinline__ bool st_first_done(u64 s) { return (s >> 4) & 1u; }
__device__ __forceinline__ int st_cur(u64 s) { return (int)((s >> 5) & 3u); }
__device__ __forceinline__ unsigned st_ver(u64 s) { return (unsigned)s >> 8; }
__device__ __forceinline__ int st_pslot(u64 s) { return (int)((s >> 32) & 3u); }
__device__ __forceinline__ int st_nbcur(u64 s, int d) { return (int)((s >> (34 + 2 * d)) & 3u); }
__device__ __forceinline__ int kind_slot(u64 s, int kind) {
  return kind == 0 ? st_pslot(s) : 3 - st_cur(s) - st_pslot(s);
}
constexpr unsigned kVerOne = 1u << 8;
constexpr unsigned kSpecNone = 0xFFFFFFFFu;
constexpr unsigned kTagMask = 0xFFFFFFu;

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// same loads without the compiler memory barrier, so independent loads are
// issued together (still volatile: never hoisted out of a polling loop)
__device__ __forceinline__ unsigned ld_relaxed_u32_nb(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ u64 ld_relaxed_u64(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 ld_relaxed_u64_nb(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ u64 ld_acquire_u64(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u32(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_s32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// predicated stores (generic addresses: the queue lives in shared or global
// memory), so lanes taking different cases stay in one instruction stream
__device__ __forceinline__ void st_pred_f64(double* p, double v, bool c) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.f64 [%0], %1; }"
               ::"l"(p), "d"(v), "r"((unsigned)c) : "memory");
}
__device__ __forceinline__ void st_pred_s32(int* p, int v, bool c) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.s32 [%0], %1; }"
               ::"l"(p), "r"(v), "r"((unsigned)c) : "memory");
}
__device__ __forceinline__ void st_pred_relaxed_u64(unsigned long long* p, unsigned long long v,
                                                    bool c) {
  asm volatile(
      "{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.relaxed.gpu.global.u64 [%0], %1; }"
      ::"l"(p), "l"(v), "r"((unsigned)c) : "memory");
}
// release fence at gpu scope (a fence.acq_rel followed by a relaxed store
// is a release pattern); lighter than __threadfence's sequentially
// consistent MEMBAR.SC
__device__ __forceinline__ void fence_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ bool tag_is(unsigned sv, unsigned v) {
  return sv != kSpecNone && (sv & kTagMask) == v;
}
// Instance numbers: workers' writes (nseq << 1 | kind) below bit 23, the
// committer's own processings kSelfInst | removal count -- unique per cell,
// so a chained speculation built on a worker's result never matches a
// processing the committer did itself.
constexpr unsigned kInstMask = 0x7FFFFFu;
constexpr unsigned kSelfInst = 0x800000u;
// 128-bit single-copy-atomic accesses to the record words (PRec)
__device__ __forceinline__ uint4 mk4(unsigned long long a, unsigned long long b) {
  return make_uint4((unsigned)a, (unsigned)(a >> 32), (unsigned)b, (unsigned)(b >> 32));
}
__device__ __forceinline__ uint4 ld_w128(const uint4* p) {
  unsigned long long a, b;
  asm volatile("{ .reg .b128 t; ld.relaxed.gpu.global.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
               : "=l"(a), "=l"(b) : "l"(p) : "memory");
  return mk4(a, b);
}
// without the compiler memory barrier: independent loads issue together
__device__ __forceinline__ uint4 ld_w128_nb(const uint4* p) {
  unsigned long long a, b;
  asm volatile("{ .reg .b128 t; ld.relaxed.gpu.global.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
               : "=l"(a), "=l"(b) : "l"(p));
  return mk4(a, b);
}
__device__ __forceinline__ uint4 ld_acquire_w128(const uint4* p) {
  unsigned long long a, b;
  asm volatile("{ .reg .b128 t; ld.acquire.gpu.global.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
               : "=l"(a), "=l"(b) : "l"(p) : "memory");
  return mk4(a, b);
}
__device__ __forceinline__ void st_w128(uint4* p, uint4 v) {
  const unsigned long long a = ((unsigned long long)v.y << 32) | v.x;
  const unsigned long long b = ((unsigned long long)v.w << 32) | v.z;
  asm volatile("{ .reg .b128 t; mov.b128 t, {%1, %2}; st.relaxed.gpu.global.b128 [%0], t; }"
               ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ double w_cand(uint4 w) {
  return __hiloint2double((int)w.y, (int)w.x);
}
// named barriers between the committer (warp 0) and its queue helper (warp 1)
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
constexpr int kBarQueueDone = 1;  // helper -> committer: the popped bucket is renewed
constexpr int kBarQueuePop = 2;   // committer -> helper: a pop to remove (or -1: stop)

// ---- the committer's priority queue over cells keyed by (cell value, id) ---
// The reference pops the minimum (value, id) of an indexed binary heap
// (indexed_min_heap.hpp:11-106, ties to the smaller id); the pop order depends
// only on the keys, not on the heap's shape, so any exact min-structure
// replays it.  Here: 32 buckets of unordered entries with each bucket's
// minimum cached; cell (x, y) goes to bucket (x + 2y) mod 32, so the W/E/S/N
// neighbours of any cell sit in four distinct buckets (b-1, b+1, b-2, b+2)
// and a commit updates them from four lanes at once.  pop = one warp argmin over the 32 cached
// minima + a warp rescan of the winning bucket; insert and decrease-key are
// O(1).  Entries live in the committer's shared memory (or global memory
// when a bucket could overflow it); every cell's position is mirrored to
// global memory (pos[], needed only for the popped cell's 4 neighbours,
// prefetched with the rest of the commit and tracked through moves).  The
// bucket arrays and counts are mirrored to global memory for the workers.
// Cell id -> (column, row) without an integer division: q = (id * magic)
// >> 40, exact for every id < J (the host checks all of them and passes 0
// when it is not, which falls back to the division).
__device__ __forceinline__ void cell_xy(int cell, int cells_x, u64 magic, int& cx, int& cy) {
  cy = magic ? (int)(((u64)(unsigned)cell * magic) >> 40) : cell / cells_x;
  cx = cell - cy * cells_x;
}

struct BucketPQ {
  double* bk;     // [32][capb] keys
  int* bi;        // [32][capb] ids
  int* cnt;       // [32] entries per bucket
  double* mk;     // [32] cached bucket minima (+inf when empty)
  int* mi;        //      their ids (INT_MAX when empty)
  int* msl;       //      their slots
  int capb;
  int* pos;       // global [J]: bucket << 24 | slot, -1 = not queued
  int* pub;       // global [32][capb] id mirror (null: bi is global already)
  int* pubcnt;    // global count mirror, bucket l at pubcnt[32 * l] (one line each)
  int* pubmin;    // global mirror of each bucket's minimum id (-1: empty), [32 * l]
  int size;       // entries (instrumented build only)
  __device__ static bool less(double ka, int ia, double kb, int ib) {
    return ka < kb || (ka == kb && ia < ib);
  }
  __device__ void set(int l, int s, double k, int id) {  // lane 0
    bk[l * capb + s] = k;
    bi[l * capb + s] = id;
    pos[id] = (l << 24) | s;
    if (pub) pub[l * capb + s] = id;
  }
  // bucket of cell (x, y); its W/E/S/N neighbours sit in b-1, b+1, b-2, b+2
  __device__ static int bucket_xy(int x, int y) { return (x + 2 * y) & 31; }
  // one lane per bucket at a time; false when bucket l is full
  __device__ bool insert(int id, double k, int l) {
    const int s = cnt[l];
    if (s >= capb) return false;
    set(l, s, k, id);
    cnt[l] = s + 1;
    pubcnt[32 * l] = s + 1;
    if (less(k, id, mk[l], mi[l])) {
      mk[l] = k;
      mi[l] = id;
      msl[l] = s;
      pubmin[32 * l] = id;
    }
    return true;
  }
  __device__ void decrease(int enc, double k) {  // one lane per bucket; keys only decrease
    const int l = enc >> 24, s = enc & 0xFFFFFF;
    const int id = bi[l * capb + s];
    bk[l * capb + s] = k;
    if (less(k, id, mk[l], mi[l])) {
      mk[l] = k;
      mi[l] = id;
      msl[l] = s;
      pubmin[32 * l] = id;
    }
  }
  // all lanes: the minimum's id (or -1 when empty) and its bucket in w_out;
  // remove(w) takes it out, rescan(w) renews the bucket's cached minimum --
  // the committer overlaps both with the loads the popped cell needs
  __device__ int argmin(int lane, int& w_out) const {
    // Keys are cell values: >= 0 or +inf, so their bit patterns (with -0
    // folded into +0) order like the values; (key, id) is then a 96-bit
    // unsigned key and three warp min-reductions find the minimum, ties to
    // the smaller id as the reference heap pops them.
    const double kl = mk[lane];
    const int il = mi[lane];
    const unsigned long long kb =
        kl == 0.0 ? 0ull : (unsigned long long)__double_as_longlong(kl);
    const unsigned hi = (unsigned)(kb >> 32), lo = (unsigned)kb;
    const unsigned mhi = __reduce_min_sync(kFull, hi);
    const unsigned mlo = __reduce_min_sync(kFull, hi == mhi ? lo : 0xFFFFFFFFu);
    const bool kmin = hi == mhi && lo == mlo;
    const unsigned mid = __reduce_min_sync(kFull, kmin ? (unsigned)il : 0xFFFFFFFFu);
    const unsigned won = __ballot_sync(kFull, kmin && (unsigned)il == mid);
    w_out = __ffs(won) - 1;
    const bool empty = mhi == 0x7FF00000u && mlo == 0u && mid == 0x7fffffffu;
    return empty ? -1 : (int)mid;  // every bucket empty: -1
  }
  __device__ void remove(int lane, int w, int top) {
    if (lane == 0) {
      const int s = msl[w], last = cnt[w] - 1;
      if (s != last) set(w, s, bk[w * capb + last], bi[w * capb + last]);
      cnt[w] = last;
      pubcnt[32 * w] = last;
      pos[top] = -1;
    }
    __syncwarp();
  }
  // all lanes: recompute bucket w's cached minimum
  __device__ void rescan(int lane, int w) {
    const int n = cnt[w];
    double kb = kInf;
    int ib = 0x7fffffff, sb = 0;
    for (int s = lane; s < n; s += 32) {
      const double k = bk[w * capb + s];
      const int id = bi[w * capb + s];
      if (less(k, id, kb, ib)) {
        kb = k;
        ib = id;
        sb = s;
      }
    }
    // warp minimum of (key, id) by three min-reductions (see argmin)
    const unsigned long long kbits =
        kb == 0.0 ? 0ull : (unsigned long long)__double_as_longlong(kb);
    const unsigned hi = (unsigned)(kbits >> 32), lo = (unsigned)kbits;
    const unsigned mhi = __reduce_min_sync(kFull, hi);
    const unsigned mlo = __reduce_min_sync(kFull, hi == mhi ? lo : 0xFFFFFFFFu);
    const bool kmin = hi == mhi && lo == mlo;
    const unsigned mid = __reduce_min_sync(kFull, kmin ? (unsigned)ib : 0xFFFFFFFFu);
    const unsigned won = __ballot_sync(kFull, kmin && (unsigned)ib == mid);
    const int src = __ffs(won) - 1;
    const double kw = __shfl_sync(kFull, kb, src);
    const int sw = __shfl_sync(kFull, sb, src);
    if (lane == 0) {
      mk[w] = kw;
      mi[w] = (int)mid;
      msl[w] = sw;
      pubmin[32 * w] = n > 0 ? (int)mid : -1;
    }
    __syncwarp();
  }
};

// Node (x, y) of the cell sits at row y+1, column x+2 of the tile, so even
// columns of the interior are 16-byte aligned (async 16-byte copies of value
// pairs); the west halo is column 1.
// value / cost halves of a warp's tile: (max_h + 2) rows of pu doubles,
// each rounded to 128 bytes (the cost tile is a TMA destination)
__host__ __device__ __forceinline__ int64_t hc_half(const CellGeom& g) {
  return ((int64_t)(g.max_h + 2) * g.pu + 15) & ~(int64_t)15;
}

struct HTile {
  double* U;      // (h+2) x pu values with cross halo
  double* Ct;     // (h+2) x pu costs with halo (-1 = exit / off-grid)
  uint8_t* lock;  // h x w, 1 = unlocked
  uint64_t* bar;  // the warp's mbarrier (TMA cost-tile loads)
  int pu, w, h;
  __device__ int ci(int x, int y) const { return (y + 1) * pu + (x + 2); }
  __device__ double& u(int x, int y) const { return U[ci(x, y)]; }
  __device__ double c(int x, int y) const { return Ct[ci(x, y)]; }
};

__device__ __forceinline__ void cp_async16_cg(void* sdst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8_ca(void* sdst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// The cost tile by TMA (one lane): the box of pu x (max_h + 2) costs whose
// top-left is node (ib - 2, jb - 1) of the padded C -- 16-byte aligned when
// the cell's first column is even -- completing on the warp's mbarrier;
// returns the arrival's state token for the wait.
__device__ __forceinline__ unsigned long long tma_cost_tile(const HcArgs& a, const HTile& T,
                                                            int64_t ib, int64_t jb) {
  const unsigned bar = (unsigned)__cvta_generic_to_shared(T.bar);
  const unsigned dst = (unsigned)__cvta_generic_to_shared(T.Ct);
  const unsigned bytes = (unsigned)a.g.pu * (unsigned)(a.g.max_h + 2) * 8u;
  unsigned long long tok;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
               : "=l"(tok) : "r"(bar), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(a.tmc), "r"((int)(a.g.pad + ib - 2)), "r"((int)jb), "r"(bar) : "memory");
  return tok;
}
// Band rounds (cells swept in place in u): the value and cost tiles of the
// same box from the padded u and C, after the neighbours' values stored
// before the last grid barrier (generic proxy) are ordered before the
// async-proxy reads.
__device__ __forceinline__ unsigned long long tma_band_tiles(const HcArgs& a, const HTile& T,
                                                             int64_t ib, int64_t jb) {
  const unsigned bar = (unsigned)__cvta_generic_to_shared(T.bar);
  const unsigned bytes = 2u * (unsigned)a.g.pu * (unsigned)(a.g.max_h + 2) * 8u;
  const int x = (int)(a.g.pad + ib - 2), y = (int)jb;
  unsigned long long tok;
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
               : "=l"(tok) : "r"(bar), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];"
      ::"r"((unsigned)__cvta_generic_to_shared(T.U)), "l"(a.tm_band), "r"(x), "r"(y), "r"(bar)
      : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];"
      ::"r"((unsigned)__cvta_generic_to_shared(T.Ct)), "l"(a.tm_band + 1), "r"(x), "r"(y),
        "r"(bar)
      : "memory");
  return tok;
}
__device__ __forceinline__ void tma_wait(const HTile& T, unsigned long long tok) {
  const unsigned bar = (unsigned)__cvta_generic_to_shared(T.bar);
  unsigned ok = 0;
  while (!ok)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok) : "r"(bar), "l"(tok) : "memory");
}

// reset_locks (heap_cell.cpp:65-94).  Lanes take (row offset, column) pairs
// with one division per call, and every node's five cost loads are issued
// together (the neighbour reads stay inside the tile: halo rows/columns).
__device__ void reset_locks(const HTile& T, bool west_in, bool east_in, bool south_in,
                            bool north_in, int lane) {
  const int w = T.w, h = T.h, pu = T.pu;
  const int rows = w <= 32 ? 32 / w : 1;  // rows per pass
  const int x0 = w <= 32 ? lane % w : lane, y0 = w <= 32 ? lane / w : 0;
  const int xstep = w <= 32 ? w : 32;
  if (y0 < rows) {
    for (int x = x0; x < w; x += xstep) {
      const bool bw = west_in && x == 0, be = east_in && x == w - 1;
      const bool inE = x + 1 < w, inW = x > 0;
#pragma unroll 4
      for (int y = y0; y < h; y += rows) {
        const double* c = &T.Ct[T.ci(x, y)];
        const double cc = c[0], ce = c[1], cw = c[-1], cn = c[pu], cs = c[-pu];
        const bool edge = bw || be || (south_in && y == 0) || (north_in && y == h - 1);
        const bool exit_nb = (inE && ce < 0.0) | (inW && cw < 0.0) | (y + 1 < h && cn < 0.0) |
                             (y > 0 && cs < 0.0);
        T.lock[y * w + x] = (cc >= 0.0 && (edge || exit_nb)) ? 1 : 0;
      }
    }
  }
  __syncwarp();
}

__device__ void mono_sides(int from_side, int out[2]) {  // cells.cpp:49-60
  switch (from_side) {
    case WEST: out[0] = NW; out[1] = SW; break;
    case EAST: out[0] = NE; out[1] = SE; break;
    case SOUTH: out[0] = SW; out[1] = SE; break;
    default: out[0] = NW; out[1] = NE; break;
  }
}

// scan_cell_boundary (heap_cell.cpp:173-239) for the four sides at once:
// lanes 8s..8s+7 scan side s, so the
// reductions (first strict maximum, should_add, monotonicity) stay inside an
// 8-lane group and the four candidate divisions run in parallel; lane 8s
// writes side s of the record.
__device__ void scan_all(const HcArgs& a, const HTile& T, const double* before,
                         const double* pstrip, bool first_removal, unsigned nbmask, SpecRec* rec,
                         int lane) {
  const int side = lane >> 3, q = lane & 7;
  const bool vertical = side == WEST || side == EAST;
  const int len = vertical ? T.h : T.w;
  const double* bf = before + side * a.max_len;
  const bool has = (nbmask >> side) & 1u;
  double vmax = -kInf;
  int arg = 0x7fffffff;
  bool add = false, inc_viol = false, dec_viol = false;
  if (has) {
    // the strip's node t and the node across the border, as offsets from the
    // strip's first node (one instruction stream for the four 8-lane groups:
    // their sides differ only in these constants)
    const int x0 = side == EAST ? T.w - 1 : 0, y0 = side == NORTH ? T.h - 1 : 0;
    const int step = vertical ? T.pu : 1;           // along the strip
    const int across = side == WEST ? -1 : side == EAST ? 1 : side == SOUTH ? -T.pu : T.pu;
    const int o0 = T.ci(x0, y0);
    for (int t = q; t < len; t += 8) {
      const int o = o0 + t * step;
      const double vi = T.U[o];
      if (vi > vmax) {  // first strict maximum along the strip
        vmax = vi;
        arg = t;
      }
      const bool across_exit = T.Ct[o + across] < 0.0;
      const bool changed = vi < bf[t];
      add = add || (!across_exit && vi < T.U[o + across] &&
                    (changed || (first_removal && T.Ct[o] < 0.0)));
      if (t > 0) {
        const double prev = T.U[o - step];
        inc_viol = inc_viol || vi < prev;
        dec_viol = dec_viol || vi > prev;
      }
    }
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(kFull, vmax, o);
    const int oa = __shfl_xor_sync(kFull, arg, o);
    if (ov > vmax || (ov == vmax && oa < arg)) {
      vmax = ov;
      arg = oa;
    }
  }
  const unsigned gm = 0xFFu << (8 * side);
  add = (__ballot_sync(kFull, add) & gm) != 0u;
  inc_viol = (__ballot_sync(kFull, inc_viol) & gm) != 0u;
  dec_viol = (__ballot_sync(kFull, dec_viol) & gm) != 0u;
  if (q != 0) return;
  double cand = kInf;
  unsigned fl = 0;
  bool mon_checked = false, mon_single = false;
  if (has) {
    if (vmax < kInf) {  // isfinite(vmax): vmax > -inf always holds here
      const double fprobe = pstrip[side * a.max_len + arg];
      const double hc = vertical ? a.hc_x : a.hc_y;
      cand = vmax + 0.5 * (a.h + hc) / fprobe;  // cell_value_candidate (cells.hpp:109-112)
    }
    if (add) {
      int both[2];
      mono_sides(side ^ 1, both);  // the neighbour is entered through the opposite side
      if (a.fast) {
        // sequences run north-to-south (vertical borders reversed) or west-to-east
        const bool nondec = vertical ? !dec_viol : !inc_viol;
        const bool noninc = vertical ? !inc_viol : !dec_viol;
        if (nondec && !noninc) fl = 1u << both[0];
        else if (noninc && !nondec) fl = 1u << both[1];
        else fl = (1u << both[0]) | (1u << both[1]);
        mon_checked = true;
        mon_single = (nondec != noninc);
      } else {
        fl = (1u << both[0]) | (1u << both[1]);
      }
    }
  } else {
    add = false;
  }
  rec->cand[side] = cand;
  rec->side[side] = (add ? 1u : 0u) | (fl << 8) | (mon_checked ? 1u << 16 : 0u) |
                    (mon_single ? 1u << 24 : 0u);
}

__device__ __forceinline__ void hc_cell_rect(const CellGeom& g, u64 magic, int cell, int64_t& ib,
                                             int64_t& ie, int64_t& jb, int64_t& je) {
  int cx, cy;
  cell_xy(cell, g.cells_x, magic, cx, cy);
  ib = (int64_t)cx * g.base_x;
  ie = (cx == g.cells_x - 1) ? g.m : ib + g.base_x;
  jb = (int64_t)cy * g.base_y;
  je = (cy == g.cells_y - 1) ? g.n : jb + g.base_y;
}

__device__ __forceinline__ double* slot_ptr(const HcArgs& a, int s, int cell) {
  return a.slots + ((size_t)s * a.J + cell) * a.cellsz;
}
__device__ __forceinline__ PRec* rec_ptr(const HcArgs& a, int kind, int cell) {
  return a.rec + (size_t)kind * a.J + cell;
}

// Process `cell` against the state word `st` into the slot of speculation
// `kind`: stage own values from the committed slot and the halo from the
// neighbours' committed slots -- except the sides in `omask`, whose values
// come from slot oslot[side] (the pending results a chained speculation
// builds on, whose scans add `cflags` to the cell's flags) -- then sweep,
// scan and write the record (all fields but the instance number and tags).
__device__ __forceinline__ void process_cell(const HcArgs& a, HTile& T, double* before, SpecRec* stg,
                             int cell, int kind, u64 st, unsigned omask, const int oslot[4],
                             unsigned cflags, int lane, long long* prof = nullptr) {
  const long long p0 = prof ? clock64() : 0;
  const CellGeom& g = a.g;
  int64_t ib, ie, jb, je;
  hc_cell_rect(g, a.cx_magic, cell, ib, ie, jb, je);
  T.w = (int)(ie - ib);
  T.h = (int)(je - jb);
  int cx, cy;
  cell_xy(cell, g.cells_x, a.cx_magic, cx, cy);
  const int mw = a.spw;  // slot row pitch (even)
  const bool has_nb[4] = {cx > 0, cx + 1 < g.cells_x, cy > 0, cy + 1 < g.cells_y};
  const int nbs[4] = {cell - 1, cell + 1, cell - g.cells_x, cell + g.cells_x};
  // Staging with every load in flight at once: the cell's own values as
  // 16-byte async copies that bypass L1 (other SMs write the slots), its costs
  // with the cost halo as 8-byte async copies (read-only data), and -- once
  // the neighbours' state words locate their committed slots -- the value
  // halo and the probe strips through registers.
  const double* own = slot_ptr(a, st_cur(st), cell);
  double* pstrip = before + 4 * a.max_len;
  unsigned long long tma_tok = 0;
  {
    const int pr = (T.w + 1) >> 1;  // value pairs per row (an odd width copies
                                    // one pad value into the east halo column,
                                    // overwritten below after the wait)
    if (pr <= 32) {
      const int rstep = 32 / pr, px = lane % pr, ry = lane / pr;
      if (ry < rstep)
        for (int y = ry; y < T.h; y += rstep)
          cp_async16_cg(&T.U[T.ci(2 * px, y)], own + y * mw + 2 * px);
    } else {
      for (int p2 = lane; p2 < pr; p2 += 32)
        for (int y = 0; y < T.h; ++y) cp_async16_cg(&T.U[T.ci(2 * p2, y)], own + y * mw + 2 * p2);
    }
    if (a.use_tma) {
      if (lane == 0) tma_tok = tma_cost_tile(a, T, ib, jb);
    } else {
      for (int xb = 0; xb < T.w + 2; xb += 32) {
        const int x = xb + lane - 1;  // tile column -1 .. w
        if (x > T.w) continue;
        const bool xin = x >= 0 && x < T.w;
        const double* cb = a.C + (jb - 1) * g.P + g.pad + ib + x;  // row y = -1
        for (int y = xin ? -1 : 0; y <= (xin ? T.h : T.h - 1); ++y) {
          const int64_t gj = jb + y;
          double* dst = &T.Ct[T.ci(x, y)];
          if (gj >= 0 && gj < g.n) cp_async8_ca(dst, cb + (int64_t)(y + 1) * g.P);
          else *dst = -1.0;
        }
      }
    }
  }
  {
    int ncur[4];
#pragma unroll
    for (int d = 0; d < 4; ++d)
      ncur[d] = !has_nb[d] ? 0 : (omask >> d) & 1u ? oslot[d] : st_nbcur(st, d);
    const double* sw = slot_ptr(a, ncur[0], nbs[0]) + (int)(g.base_x - 1);
    const double* se = slot_ptr(a, ncur[1], nbs[1]);
    const double* ss = slot_ptr(a, ncur[2], nbs[2]) + (int)(g.base_y - 1) * mw;
    const double* sn = slot_ptr(a, ncur[3], nbs[3]);
    // cross halo values from the neighbours' slots (+inf off-grid) and the
    // four border probe strips (F at the clamped probe points,
    // heap_cell.cpp:195-205), used by the scans after the sweeps
    bool first = true;
    for (int t = lane; t < a.max_len; t += 32) {
      const bool tv = t < T.h, th = t < T.w;
      const double hw = has_nb[0] && tv ? __ldcg(sw + t * mw) : kInf;
      const double he = has_nb[1] && tv ? __ldcg(se + t * mw) : kInf;
      const double hs = has_nb[2] && th ? __ldcg(ss + t) : kInf;
      const double hn = has_nb[3] && th ? __ldcg(sn + t) : kInf;
      const double p0v = has_nb[0] && tv ? __ldg(a.probe[0] + (int64_t)cx * g.n + jb + t) : 1.0;
      const double p1v = has_nb[1] && tv ? __ldg(a.probe[1] + (int64_t)cx * g.n + jb + t) : 1.0;
      const double p2v = has_nb[2] && th ? __ldg(a.probe[2] + (int64_t)cy * g.m + ib + t) : 1.0;
      const double p3v = has_nb[3] && th ? __ldg(a.probe[3] + (int64_t)cy * g.m + ib + t) : 1.0;
      if (first) {
        cp_async_wait_all();  // the east halo column may hold a copied pad value
        first = false;
      }
      if (tv) {
        T.u(-1, t) = hw;
        T.u(T.w, t) = he;
        pstrip[0 * a.max_len + t] = p0v;
        pstrip[1 * a.max_len + t] = p1v;
      }
      if (th) {
        T.u(t, -1) = hs;
        T.u(t, T.h) = hn;
        pstrip[2 * a.max_len + t] = p2v;
        pstrip[3 * a.max_len + t] = p3v;
      }
    }
    if (first) cp_async_wait_all();
    if (a.use_tma) tma_wait(T, __shfl_sync(kFull, tma_tok, 0));
    if (prof) prof[3] += clock64() - p0;
  }
  __syncwarp();
  // border snapshots (heap_cell.cpp:279-282)
  for (int t = lane; t < T.h; t += 32) {
    before[0 * a.max_len + t] = T.u(0, t);
    before[1 * a.max_len + t] = T.u(T.w - 1, t);
  }
  for (int t = lane; t < T.w; t += 32) {
    before[2 * a.max_len + t] = T.u(t, 0);
    before[3 * a.max_len + t] = T.u(t, T.h - 1);
  }
  const long long p1 = prof ? clock64() : 0;
  const unsigned my_flags = st_flags(st) | cflags;
  const bool first_removal = !st_first_done(st);
  reset_locks(T, ib > 0, ie < g.m, jb > 0, je < g.n, lane);
  const long long p1b = prof ? clock64() : 0;
  const CellTile ct{T.U, T.Ct, T.lock, T.pu, T.w, T.h, 2};
  long long nsw = 0, upd = 0;
  {
    // FHCM, process_flagged_once (heap_cell.cpp:150-160): one sweep per raised
    // flag, NE, NW, SE, SW.  HCM, process_to_convergence (:130-147): the
    // flagged directions first, then the unflagged ones in rotation order,
    // then the rotation, until a sweep changes nothing.  One call site, so
    // the kernel holds one copy of each engine variant.
    int perm[4], nflag = 0;
    for (int k = 0; k < 4; ++k)
      if (my_flags & (1u << kFlagOrder[k])) perm[nflag++] = kFlagOrder[k];
    int at = nflag;
    for (int k = 0; k < 4; ++k)
      if (!(my_flags & (1u << kRotation[k]))) perm[at++] = kRotation[k];
    bool changed = true;
    for (;;) {
      if (a.fast ? nsw >= nflag : !changed) break;
      const int dir = nsw < 4 ? perm[nsw] : kRotation[nsw % 4];
      // cells taller than 32 rows as 32-row bands (a.bands, EIK_HC_BANDS=0:
      // several rows per lane).  The multi-slot variants stay compiled in on
      // purpose: without them ptxas allocates 139 registers instead of 255
      // and the 8-32-node cells get 6-9 % slower (FHCM/8 165 -> 176 ms).
      const bool skip = !a.fast && nsw >= a.skip_from;
      changed = (ct.h <= 32 || !a.bands) ? cell_sweep<2>(ct, dir, lane, upd, skip)
                                         : cell_sweep_lock_bands(ct, dir, lane, upd, skip);
      ++nsw;
    }
  }
  for (int o = 16; o > 0; o >>= 1) upd += __shfl_xor_sync(kFull, upd, o);
  const long long p2 = prof ? clock64() : 0;
  // processed values into the slot of this speculation kind
  double* spare = slot_ptr(a, kind_slot(st, kind), cell);
  for (int k = lane; k < T.w * T.h; k += 32) {
    const int y = k / T.w, x = k % T.w;
    spare[y * mw + x] = T.u(x, y);
  }
  scan_all(a, T, before, pstrip, first_removal,
           (has_nb[0] ? 1u : 0u) | (has_nb[1] ? 2u : 0u) | (has_nb[2] ? 4u : 0u) |
               (has_nb[3] ? 8u : 0u),
           stg, lane);
  if (lane == 0) {
    stg->sweeps = (int)nsw;
    stg->updates = (int)upd;
  }
  if (prof) {
    prof[4] += p1b - p1;                        // reset_locks
    prof[5] += nsw * (long long)(T.w + T.h - 1);  // wavefront steps
    const long long p3 = clock64();
    prof[0] += p1 - p0;  // staging
    prof[1] += p2 - p1;  // locks + sweeps
    prof[2] += p3 - p2;  // spare slot + scans + record
  }
}

// Publish the result process_cell just wrote (all lanes call; lane 0 writes):
// the record words from the staging copy, each stamped with a fresh instance
// number, then the speculation tag, then free the cell.  A chained result
// assuming |A| commits is valid at version (read version + |A|).
__device__ void publish(const HcArgs& a, int cell, int kind, u64 st, unsigned dmask,
                        const unsigned dinst[4], const SpecRec* stg, int lane) {
  PRec* rec = rec_ptr(a, kind, cell);
  const unsigned tag = (st_ver(st) + (unsigned)__popc(dmask)) & kTagMask;
  fence_rel_gpu();  // the slot values (every lane's stores) before the record
  __syncwarp();
  if (lane == 0) {
    const unsigned n = ld_w128(&rec->w[6]).z + 1u;  // writes so far (busy holder only)
    const unsigned inst = ((n << 1) | (unsigned)kind) & kInstMask;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const unsigned long long cb = (unsigned long long)__double_as_longlong(stg->cand[d]);
      st_w128(&rec->w[d], make_uint4((unsigned)cb, (unsigned)(cb >> 32), stg->side[d], inst));
    }
    st_w128(&rec->w[4], make_uint4((unsigned)stg->sweeps, (unsigned)stg->updates, tag, inst));
    st_w128(&rec->w[5], make_uint4(dmask, dinst[0], dinst[1], inst));
    st_w128(&rec->w[6], make_uint4(dinst[2], dinst[3], n, inst));
    st_release_u32(a.spec_ver + (size_t)kind * a.J + cell, tag);
    if (a.wdbg) a.owner[(size_t)kind * a.J + cell] = 0x60000 | kind;
    st_release_s32(a.busy + (size_t)kind * a.J + cell, 0);
  }
}

// ---- the committer: the reference's heap loop in exact order ----------------
// PROF: the cycle / miss-class instrumentation (EIK_HC_PROFILE); compiled out
// of the production instantiation, where those ~25 live counters would cost
// registers the hot path needs.
template <bool PROF>
__device__ void committer(const HcArgs& a, BucketPQ& H, HTile& T, double* before, SpecRec* stg,
                          int lane) {
  const CellGeom& g = a.g;
  bool ovf = false;  // a bucket filled up (per lane; voted once per pop)
  if (lane == 0) {
    for (int k = 0; k < a.n_init; ++k) {  // heap_cell.cpp:255-268
      const int cell = a.init_cells[k];
      a.cval[cell] = a.init_values[k];
      int ix, iy;
      cell_xy(cell, g.cells_x, a.cx_magic, ix, iy);
      if (H.insert(cell, a.init_values[k], BucketPQ::bucket_xy(ix, iy))) ++H.size;
      else ovf = true;
      a.ckey[cell] = a.init_values[k];
      if (a.fast) st_relaxed_u64(a.state + cell, (1ull << 32) | 0xFull);  // Q-cells: all flags
    }
  }
  __syncwarp();
  long long removals = 0, sweeps = 0, updates = 0, mon_checks = 0, mon_single = 0;
  long long self_processed = 0, fast_hits = 0, waits = 0, chain_hits = 0;
  long long cyc_pop = 0, cyc_obtain = 0, cyc_self = 0, cyc_commit = 0, cyc_rec = 0;
  long long cyc_rescan = 0, cyc_rt1 = 0, cyc_wait = 0, cyc_nbb = 0;
  long long prof[6] = {0, 0, 0, 0, 0, 0};
  long long miss_cls[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int max_size = H.size;
  int prev_cell = -1;
  const unsigned* spec_p = a.spec_ver;
  const unsigned* spec_c = a.spec_ver + a.J;
  bool over = false;
  // With a second warp in the CTA, the popped cell's bucket removal and the
  // bucket's new minimum are its job (queue_helper), off this warp's path:
  // the commit touches only the neighbours' buckets, never the popped one.
  const bool helper = blockDim.x >= 64;
  int* mbox = H.cnt + 32;  // [0] popped cell (-1: stop), [1] its bucket
  bool pending = false;    // the helper is renewing the last pop's bucket
  for (;;) {
    long long t0 = PROF ? clock64() : 0;
    if (pending) {
      named_bar_sync(kBarQueueDone, 64);
      pending = false;
    }
    // a full bucket dropped an entry: stop, the host reruns with global buckets
    if (__any_sync(kFull, ovf)) {
      over = true;
      break;
    }
    int wpop = 0;
    const int cell = H.argmin(lane, wpop);
    long long t1 = PROF ? clock64() : 0;
    if (PROF) cyc_pop += t1 - t0;
    if (cell < 0) break;
    ++removals;
    if (removals > a.budget) {  // heap_cell.cpp:276-277
      if (lane == 0) atomicExch(a.status, 3);
      break;
    }
    int cxi, cyi;
    cell_xy(cell, g.cells_x, a.cx_magic, cxi, cyi);
    const int nbs[4] = {cxi > 0 ? cell - 1 : -1, cxi + 1 < g.cells_x ? cell + 1 : -1,
                        cyi > 0 ? cell - g.cells_x : -1, cyi + 1 < g.cells_y ? cell + g.cells_x : -1};
    // obtain a valid result: the plain speculation if its tag is the current
    // version, else the chained one if its tag is the current version and
    // every neighbour it assumed last committed the instance it read, else
    // process the cell here.  The records are read word by word (128-bit
    // single-copy-atomic loads, one batch): lanes 0-4 the plain record's
    // words 0-4, lanes 8-14 the chained one's words 0-6; a record is whole
    // iff its words carry one instance number, so the tags, the scans and
    // the counters arrive in ONE round trip.  Polls are relaxed (an acquire
    // would flush this SM's L1).
    int mode = 0, kind = 0;  // mode 0: valid speculation, 1: process here
    u64 st = 0;
    // lanes 0-3 load side `lane`: the neighbour's state, cell value, queue
    // position and committed instance (only this warp writes those words)
    u64 my_nst = 0ull;
    double my_cv = kInf;
    int my_pos = -1;
    unsigned my_ctag = kSpecNone;
    if (lane < 4 && nbs[lane < 4 ? lane : 0] >= 0) {
      const int nb = nbs[lane];
      my_nst = ld_relaxed_u64_nb(a.state + nb);
      my_cv = __ldcg(a.cval + nb);
      my_pos = __ldcg(a.hpos + nb);
      my_ctag = __ldcg(a.ctag + nb);
    }
    st = ld_relaxed_u64_nb(a.state + cell);  // every lane: one warp-wide load each
    const int wkind = lane >> 3, wi = lane & 7;  // record word this lane reads
    const bool wlane = (wkind == 0 && wi < 5) || (wkind == 1 && wi < 7);
    const uint4* wptr = &rec_ptr(a, wkind & 1, cell)->w[wi < 7 ? wi : 0];
    uint4 rw = make_uint4(0u, 0u, 0u, kSpecNone);
    if (wlane) rw = ld_w128_nb(wptr);
    // hand the pop to the helper only now: the barrier waits for this warp's
    // earlier memory operations, and the loads above are then already in flight
    if (helper) {
      if (lane == 0) {
        mbox[0] = cell;
        mbox[1] = wpop;
      }
      named_bar_arrive(kBarQueuePop, 64);  // orders the mailbox stores (BAR drains STS)
      pending = true;
    }
    // take the cell out of its bucket and renew that bucket's minimum while
    // those loads are in flight (the neighbours sit in other buckets, so
    // neither moves their prefetched positions)
    if (!helper) {
      H.remove(lane, wpop, cell);
      if (lane == 0) a.ckey[cell] = kInf;
      H.rescan(lane, wpop);
    }
    const long long t1a = PROF ? clock64() : 0;
    if (PROF) cyc_rescan += t1a - t1;
    // every lane validates from the shuffled words; lane 0 alone claims
    {
      const unsigned v = st_ver(st);
      long long spins = 0;
      bool waited = false;
      long long tw0 = 0;
      if (PROF) {
        tw0 = clock64();
        cyc_rt1 += (v == 0xFFFFFFFFu ? 1 : 0) + tw0 - t1a;
      }
      for (;;) {
        // plain: words 0-4 on lanes 0-4 (the common hit: checked first, alone)
        const unsigned ip = __shfl_sync(kFull, rw.w, 4), tp = __shfl_sync(kFull, rw.z, 4);
        if (__ballot_sync(kFull, lane < 5 && rw.w != ip) == 0u && ip != kSpecNone &&
            tag_is(tp, v)) {
          kind = 0;
          break;
        }
        // chained: words 0-6 on lanes 8-14; lane d (0-3) checks the instance
        // the record assumed for side d against the neighbour's committed one
        const unsigned ic = __shfl_sync(kFull, rw.w, 12), tc = __shfl_sync(kFull, rw.z, 12);
        if (__ballot_sync(kFull, wkind == 1 && wlane && rw.w != ic) == 0u && ic != kSpecNone &&
            tag_is(tc, v)) {
          // dinst[0], [3] sit in .y of lanes 13 / 14, dinst[1], [2] in .z of
          // 13 / .x of 14; the mask in .x of 13
          const unsigned r2 = lane == 13 ? rw.z : rw.x;
          const unsigned dm = __shfl_sync(kFull, rw.x, 13);
          const int src = lane < 2 ? 13 : 14;
          const unsigned s1 = __shfl_sync(kFull, rw.y, src), s2 = __shfl_sync(kFull, r2, src);
          const unsigned mine = (lane == 0 || lane == 3) ? s1 : s2;
          const bool bad_side = lane < 4 && ((dm >> lane) & 1u) && mine != my_ctag;
          if (__ballot_sync(kFull, bad_side) == 0u) {
            kind = 1;
            ++chain_hits;
            break;
          }
        }
        int got = 0;
        if (lane == 0) got = atomicCAS(a.busy + cell, 0, 1) == 0 ? 1 : 0;
        if (__shfl_sync(kFull, got, 0)) {
          if (lane == 0 && a.wdbg) a.owner[cell] = 0x30000;
          // The cell is ours to process.  A worker may have published a
          // valid result between the loads above and the claim; processing
          // it here anyway is exact (the plain slot is ours now, and the
          // commit's new version and committer instance invalidate that
          // result and every speculation built on it) and saves the round
          // trip of a re-read on every miss.
          {
            mode = 1;
            if (lane == 0 && a.wdbg) a.owner[cell] = 0x50000;
            // classify the miss (profiling counters 16..23)
            if (PROF && lane == 0) {
            const unsigned svc2 = ld_relaxed_u32(spec_c + cell);
            int cls;
            if (svc2 == kSpecNone) {
              cls = 0;  // never chained
            } else {
              const unsigned diff = ((svc2 & kTagMask) - v) & kTagMask;
              if (diff >= 1 && diff <= 4) cls = 1;  // assumed commits not all done
              else if (diff != 0) cls = 2;          // stale: more commits than assumed
              else cls = 3;                         // a commit it did not assume
            }
            ++miss_cls[cls];
            if (prev_cell >= 0 && (prev_cell == nbs[0] || prev_cell == nbs[1] ||
                                   prev_cell == nbs[2] || prev_cell == nbs[3]))
              ++miss_cls[6];  // the previous pop was a neighbour
            if (((ld_relaxed_u32(spec_p + cell) & kTagMask) + 1u) == v) ++miss_cls[7];
            }
          }
          break;
        }
        waited = true;
        if (++spins > kSpinCap) {
          if (lane == 0) {
          atomicExch(a.status, kStatusWatchdog);
          // diagnostics for the host (EIK_HC_PROFILE)
          a.counters[24] = (unsigned long long)cell;
          a.counters[25] = (unsigned long long)(unsigned)ld_relaxed_s32(a.busy + cell);
          a.counters[26] = (unsigned long long)(unsigned)ld_relaxed_s32(a.busy + a.J + cell);
          a.counters[27] = ld_relaxed_u64(a.state + cell);
          a.counters[28] = ld_relaxed_u32(spec_p + cell);
          a.counters[29] = ld_relaxed_u32(spec_c + cell);
          a.counters[30] = (unsigned long long)removals;
          if (a.wdbg) {
            const int ow0 = a.owner[cell];
            a.counters[32] = (unsigned long long)ow0;
            int ow = -1;
            for (int w = 0; w < 148 * 16; ++w)
              if (a.wdbg[4 * w + 1] == cell && a.wdbg[4 * w + 0] >= 10) ow = w;
            a.counters[37] = (unsigned long long)(long long)ow;
            if (ow >= 0) {
              a.counters[33] = (unsigned)a.wdbg[4 * ow + 0];
              a.counters[34] = (unsigned)a.wdbg[4 * ow + 1];
              a.counters[35] = (unsigned)a.wdbg[4 * ow + 2];
              a.counters[36] = (unsigned long long)((clock64() >> 10) - a.wdbg[4 * ow + 3]);
            }
          }
          }
          mode = 2;
          break;
        }
        if (wlane) rw = ld_w128(wptr);  // poll both records again
      }
      if (mode == 0) ++fast_hits;
      if (waited) ++waits;
      if (PROF && waited) cyc_wait += clock64() - tw0;
    }
    long long t2 = PROF ? clock64() : 0;
    if (PROF) cyc_obtain += t2 - t1;
    if (mode == 2) break;
    // the result to commit: side d's scan on lane d, counters on lane 0
    double rcand = kInf;
    unsigned rside = 0u, rinst = 0u;
    int rsweeps = 0, rupdates = 0;
    if (mode == 1) {
      // processed here: the scans stay in the staging record (shared
      // memory), the values go to the plain slot, made visible before the
      // commit's state words; no record is published and the instance is
      // the committer's own (kSelfInst | removal count)
      const int none[4] = {0, 0, 0, 0};
      process_cell(a, T, before, stg, cell, 0, st, 0u, none, 0u, lane, PROF ? prof : nullptr);
      fence_rel_gpu();
      __syncwarp();
      if (lane < 4) {
        rcand = stg->cand[lane];
        rside = stg->side[lane];
      }
      rsweeps = stg->sweeps;
      rupdates = stg->updates;
      rinst = kSelfInst | ((unsigned)removals & kInstMask);
      if (lane == 0) {  // every lane's fence above ordered its slot stores first
        if (a.wdbg) a.owner[cell] = 0x60000;
        st_relaxed_u32(reinterpret_cast<unsigned*>(a.busy + cell), 0u);
      }
      kind = 0;
      ++self_processed;
    } else {
      const int src = kind ? lane + 8 : lane;  // word `lane` of the chosen record
      const unsigned x = __shfl_sync(kFull, rw.x, src & 31), y = __shfl_sync(kFull, rw.y, src & 31);
      const unsigned z = __shfl_sync(kFull, rw.z, src & 31);
      const int s4 = kind ? 12 : 4;
      rsweeps = (int)__shfl_sync(kFull, rw.x, s4);
      rupdates = (int)__shfl_sync(kFull, rw.y, s4);
      rinst = __shfl_sync(kFull, rw.w, s4);
      if (lane < 4) {
        rcand = __hiloint2double((int)y, (int)x);
        rside = z;
      }
    }
    long long t3 = PROF ? clock64() : 0;
    if (PROF) cyc_self += t3 - t2;
    // commit: the popped cell on lane 0, its four neighbours on lanes 0-3 at
    // once (their queue buckets differ); every load before the first update
    {
      const int cur = st_cur(st), ps = st_pslot(st), qs = 3 - cur - ps;
      const int ncur = kind ? qs : ps, nps = kind ? ps : cur;
      int ins = 0;
      if (lane < 4) {
        const int d = lane, nb = nbs[d];
        const double cand = rcand;
        const unsigned sw = rside;
        const unsigned add = sw & 1u, fl = (sw >> 8) & 0xFFu;
        const unsigned mc = (sw >> 16) & 1u, ms = sw >> 24;
        if (d == 0) {
          sweeps += rsweeps;
          updates += rupdates;
          if (PROF) cyc_rec += clock64() - t3;
          // popped cell: flags cleared, first removal done, the committed
          // kind's slot becomes current and the old current slot takes its
          // role, +1 version
          const unsigned lo =
              (((unsigned)st & ~(15u | (3u << 5))) | 16u | ((unsigned)ncur << 5)) + kVerOne;
          st_relaxed_u64(a.state + cell, (u64)lo | (st & (0xFFull << 34)) | ((u64)nps << 32));
          a.ctag[cell] = rinst;
        }
        // heap_cell.cpp:288-311, branch-free: the four lanes run one
        // instruction stream (their cases -- lower the key, queue the cell,
        // neither -- differ), every store predicated on its case
        const bool has = nb >= 0;
        const int nbq = has ? nb : cell;  // an in-range id for the addresses
        // the neighbour's bucket: its queue entry's, or the one it would be
        // inserted into (side d of bucket wpop: -1, +1, -2, +2); its count and
        // cached minimum are loaded ahead of the stores
        const int lq = my_pos >= 0 ? (my_pos >> 24)
                                   : ((wpop + (d < 2 ? 2 * d - 1 : 2 * (2 * d - 5))) & 31);
        const int cnt_l = H.cnt[lq];
        const double mk_l = H.mk[lq];
        const int mi_l = H.mi[lq];
        const bool lower = has && cand < my_cv;
        const double cvd = lower ? cand : my_cv;
        const bool addq = has && add != 0u;
        const bool dec = lower && my_pos >= 0;
        const bool try_ins = addq && my_pos < 0;
        const bool do_ins = try_ins && cnt_l < H.capb;
        ovf = ovf || (try_ins && !do_ins);
        const int sl = dec ? (my_pos & 0xFFFFFF) : cnt_l;
        const int ix = lq * H.capb + sl;
        const bool newmin = (dec || do_ins) && BucketPQ::less(cvd, nbq, mk_l, mi_l);
        st_pred_f64(H.bk + ix, cvd, dec || do_ins);
        st_pred_s32(H.bi + ix, nbq, do_ins);
        st_pred_s32(H.pos + nbq, (lq << 24) | sl, do_ins);
        if (H.pub) st_pred_s32(H.pub + ix, nbq, do_ins);
        st_pred_s32(H.cnt + lq, sl + 1, do_ins);
        st_pred_s32(H.pubcnt + 32 * lq, sl + 1, do_ins);
        st_pred_f64(H.mk + lq, cvd, newmin);
        st_pred_s32(H.mi + lq, nbq, newmin);
        st_pred_s32(H.msl + lq, sl, newmin);
        st_pred_s32(H.pubmin + 32 * lq, nbq, newmin);
        st_pred_f64(a.cval + nbq, cand, lower);
        st_pred_f64(a.ckey + nbq, cvd, dec || try_ins);
        ins += do_ins ? 1 : 0;
        if (addq && mc) {
          ++mon_checks;
          if (ms) ++mon_single;
        }
        const unsigned lo = ((unsigned)my_nst + kVerOne) | (addq ? fl : 0u);
        // the popped cell sits on side (d ^ 1) of its neighbour, which
        // learns its new slot
        const int sh = 34 + 2 * (d ^ 1);
        st_pred_relaxed_u64(a.state + nbq,
                            (u64)lo | (my_nst & ~((3ull << sh) | 0xFFFFFFFFull)) |
                                ((u64)ncur << sh),
                            has);
      }
      if (PROF) {
        __syncwarp();
        if (lane == 0) cyc_nbb += clock64() - t3;
        ins += __shfl_xor_sync(kFull, ins, 1);
        ins += __shfl_xor_sync(kFull, ins, 2);
        if (lane == 0) {
          H.size += ins - 1;
          if (H.size > max_size) max_size = H.size;
        }
      }
    }
    __syncwarp();
    if (PROF) {
      cyc_commit += clock64() - t3;
      prev_cell = cell;
    }
  }
  if (helper) {  // stop the helper
    if (pending) named_bar_sync(kBarQueueDone, 64);
    if (lane == 0) mbox[0] = -1;
    named_bar_arrive(kBarQueuePop, 64);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mon_checks += __shfl_xor_sync(kFull, mon_checks, o);
    mon_single += __shfl_xor_sync(kFull, mon_single, o);
  }
  if (lane == 0) {
    a.counters[0] = removals;
    a.counters[1] = sweeps;
    a.counters[2] = updates;
    a.counters[3] = mon_checks;
    a.counters[4] = mon_single;
    a.counters[5] = self_processed;
    a.counters[6] = fast_hits;
    a.counters[7] = waits;
    a.counters[15] = chain_hits;
  }
  if (PROF && lane == 0) {
    a.counters[8] = cyc_pop;
    a.counters[9] = cyc_obtain;
    a.counters[10] = cyc_self;
    a.counters[11] = cyc_commit;
    a.counters[12] = prof[0];
    a.counters[13] = prof[1];
    a.counters[14] = prof[2];
    a.counters[39] = prof[3];
    a.counters[40] = prof[4];
    a.counters[41] = prof[5];
    a.counters[42] = cyc_rec;
    a.counters[43] = cyc_rescan;
    a.counters[44] = cyc_rt1;
    a.counters[45] = cyc_wait;
    a.counters[46] = cyc_nbb;
    for (int k = 0; k < 8; ++k) a.counters[16 + k] = miss_cls[k];
    a.counters[38] = (unsigned long long)max_size;
  }
  if (lane == 0) {
    if (over) atomicExch(a.status, 6);
    __threadfence();
    st_release_s32(a.done_flag, 1);
  }
}

// Warp 1 of the committer's CTA: for every pop, take the cell out of its
// bucket and renew the bucket's cached minimum while the committer validates
// and commits (which touches only the neighbours' buckets).
__device__ void queue_helper(const HcArgs& a, BucketPQ& H, int lane) {
  const int* mbox = H.cnt + 32;
  for (;;) {
    named_bar_sync(kBarQueuePop, 64);
    const int cell = mbox[0], w = mbox[1];
    if (cell < 0) return;
    H.remove(lane, w, cell);
    if (lane == 0) a.ckey[cell] = kInf;
    H.rescan(lane, w);
    named_bar_arrive(kBarQueueDone, 64);  // the bucket's new minimum is in shared memory
  }
}

__device__ __forceinline__ void cell_nbs(const HcArgs& a, int cell, int nbs[4]) {
  const CellGeom& g = a.g;
  int cx, cy;
  cell_xy(cell, g.cells_x, a.cx_magic, cx, cy);
  nbs[0] = cx > 0 ? cell - 1 : -1;
  nbs[1] = cx + 1 < g.cells_x ? cell + 1 : -1;
  nbs[2] = cy > 0 ? cell - g.cells_x : -1;
  nbs[3] = cy + 1 < g.cells_y ? cell + g.cells_x : -1;
}

// A chained speculation of x assuming the set A (|A| = n) is dead -- it can
// never become valid -- once more than n commits happened in {x} u N(x) since
// it was read, or a commit that is not one of A's.  k commits happened; c of
// them are A's (their last committed instance is the one assumed).  Reading
// x's version before the ctags keeps the test conservative, and both
// conditions only get more true as commits happen.  Exact when the caller
// holds x's chained busy flag (the record is then stable).
__device__ bool chain_dead(const HcArgs& a, int x, unsigned svc, u64 st, const int nbx[4]) {
  if (svc == kSpecNone) return true;
  const PRec* r = rec_ptr(a, 1, x);
  const uint4 w5 = ld_w128(&r->w[5]), w6 = ld_w128(&r->w[6]);
  if (w5.w != w6.w) return false;  // being rewritten (only without x's busy flag)
  const unsigned dm = w5.x;
  const unsigned di[4] = {w5.y, w5.z, w6.x, w6.y};
  const unsigned n = (unsigned)__popc(dm);
  const unsigned k = (st_ver(st) - (((svc & kTagMask) - n) & kTagMask)) & kTagMask;
  if (k > n) return true;
  unsigned c = 0;
#pragma unroll
  for (int d = 0; d < 4; ++d)
    if ((dm >> d) & 1u) c += __ldcg(a.ctag + nbx[d]) == di[d] ? 1u : 0u;
  return k > c;
}

// The result of y a neighbour's chained speculation builds on: y's chained
// result while it is not dead (valid, or waiting for commits of y's own
// neighbours expected first), else y's plain result if valid; -1 if none.
__device__ int pick_kind(const HcArgs& a, int y, u64 sty) {
  int nby[4];
  cell_nbs(a, y, nby);
  const unsigned svc = ld_relaxed_u32(a.spec_ver + a.J + y);
  if (svc != kSpecNone && !chain_dead(a, y, svc, sty, nby)) return 1;
  if (tag_is(ld_relaxed_u32(a.spec_ver + y), st_ver(sty))) return 0;
  return -1;
}

struct Job {
  int cell, kind;
  u64 st;
  unsigned omask, cflags;
  int oslot[4];
  unsigned dinst[4];
};

// Claim a chained speculation of x on the current results of its neighbours
// on the sides in amask.  For each y: the instance number of y's result is
// read first (acquire), y's state and the record's tag after it.  A tag at
// most 4 ahead of y's version means that instance was not committed when y's
// state was read -- after x's state was read -- so its values are still in
// y's slot of that kind.  A result replaced meanwhile can never be committed,
// so neither can this speculation.
__device__ bool claim_chain(const HcArgs& a, int x, const int nbx[4], unsigned amask, Job& j) {
  if (atomicCAS(a.busy + (size_t)a.J + x, 0, 1) != 0) return false;
  const u64 st = ld_acquire_u64(a.state + x);
  bool ok = chain_dead(a, x, ld_relaxed_u32(a.spec_ver + a.J + x), st, nbx);
  j.cflags = 0;
  for (int d = 0; d < 4 && ok; ++d) {
    j.oslot[d] = 0;
    j.dinst[d] = 0;
    if (!((amask >> d) & 1u)) continue;
    const int y = nbx[d];
    const int yk = pick_kind(a, y, ld_relaxed_u64(a.state + y));
    if (yk < 0) {
      ok = false;
      break;
    }
    const PRec* ry = rec_ptr(a, yk, y);
    const uint4 w4 = ld_acquire_w128(&ry->w[4]);  // instance and tag of one write
    const unsigned inst = w4.w;
    const u64 sty = ld_relaxed_u64(a.state + y);
    const unsigned ahead = (w4.z - st_ver(sty)) & kTagMask;
    const int xside_of_y = d ^ 1;
    const uint4 wsd = ld_w128(&ry->w[xside_of_y]);
    if (inst == kSpecNone || ahead > 4 || wsd.w != inst) {
      ok = false;
      break;
    }
    const unsigned sw = wsd.z;
    if (sw & 1u) j.cflags |= (sw >> 8) & 0xFFu;
    j.oslot[d] = kind_slot(sty, yk);
    j.dinst[d] = inst;
  }
  if (!ok) {
    st_release_s32(a.busy + (size_t)a.J + x, 0);
    return false;
  }
  j.cell = x;
  j.kind = 1;
  j.st = st;
  j.omask = amask;
  return true;
}

__device__ __forceinline__ bool key_before(double ka, int a_id, double kb, int b_id) {
  return ka < kb || (ka == kb && a_id < b_id);
}

// Worker lane 0: choose and claim a job around heap position pidx.  For the
// queued cell c there:
//   1. a chained speculation of c on its neighbours queued above it (they
//      will be committed first unless keys change), if its chained result is
//      dead; else a plain speculation if the plain result is stale;
//   2. chained speculations of c's neighbours that c's commit will queue or
//      move up (the front's next cells), on c and on their other neighbours
//      queued above them.
__device__ bool pick_job_cell(const HcArgs& a, int cell, Job& j, int wid);
__device__ bool pick_job(const HcArgs& a, int pidx, Job& j, int wid) {
  const int cell = ld_relaxed_s32(a.harr + pidx);
  if (cell < 0 || cell >= a.J) return false;
  return pick_job_cell(a, cell, j, wid);
}
__device__ bool pick_job_cell(const HcArgs& a, int cell, Job& j, int wid) {
  int nbs[4];
  cell_nbs(a, cell, nbs);
  u64 st = ld_relaxed_u64_nb(a.state + cell);
  const unsigned svp = ld_relaxed_u32_nb(a.spec_ver + cell);
  const unsigned svc = ld_relaxed_u32_nb(a.spec_ver + a.J + cell);
  double kc = kInf, knb[4] = {kInf, kInf, kInf, kInf};
  unsigned amask = 0;
  if (a.chain) {
    kc = __ldcg(a.ckey + cell);
#pragma unroll
    for (int d = 0; d < 4; ++d) knb[d] = nbs[d] >= 0 ? __ldcg(a.ckey + nbs[d]) : kInf;
    double kb = kc;
    int yb = cell;
#pragma unroll
    for (int d = 0; d < 4; ++d)
      if (nbs[d] >= 0 && knb[d] < kInf && key_before(knb[d], nbs[d], kc, cell)) {
        amask |= 1u << d;
        if (key_before(knb[d], nbs[d], kb, yb)) {
          kb = knb[d];
          yb = nbs[d];
        }
      }
    // chain mode 1: only the neighbour expected next; 2: all expected first
    if (a.chain == 1 && amask)
      for (int d = 0; d < 4; ++d)
        if (nbs[d] == yb) amask = 1u << d;
  }
  // 1. the queued cell itself
  if (amask && chain_dead(a, cell, svc, st, nbs) && claim_chain(a, cell, nbs, amask, j))
    return true;
  if (!tag_is(svp, st_ver(st)) && atomicCAS(a.busy + cell, 0, 1) == 0) {
    if (a.wdbg) {
      a.owner[cell] = 0x10000;
      a.wdbg[4 * wid + 0] = 10;
      a.wdbg[4 * wid + 1] = cell;
      a.wdbg[4 * wid + 3] = (int)(clock64() >> 10);
    }
    st = ld_acquire_u64(a.state + cell);
    if (a.wdbg) a.wdbg[4 * wid + 0] = 11;
    if (!tag_is(ld_relaxed_u32(a.spec_ver + cell), st_ver(st))) {
      j.cell = cell;
      j.kind = 0;
      j.st = st;
      j.omask = 0;
      j.cflags = 0;
      for (int d = 0; d < 4; ++d) j.oslot[d] = 0, j.dinst[d] = 0;
      if (a.wdbg) a.wdbg[4 * wid + 0] = 12;
      return true;
    }
    if (a.wdbg) a.owner[cell] = 0x20000;
    st_release_s32(a.busy + cell, 0);
  }
  if (!a.chain) return false;
  // 2. neighbours that the commit of this cell's result queues or moves up
  const int ck = pick_kind(a, cell, st);
  if (ck < 0) return false;
  const PRec* rc = rec_ptr(a, ck, cell);
  for (int d = 0; d < 4; ++d) {
    const int x = nbs[d];
    if (x < 0) continue;
    const uint4 wd = ld_w128(&rc->w[d]);
    const double cand = w_cand(wd);
    if (!(wd.z & 1u) && !(cand < knb[d])) continue;
    const double kx = cand < knb[d] ? cand : knb[d];  // x's key after this commit
    int nbx[4];
    cell_nbs(a, x, nbx);
    unsigned am = 0;
    for (int e = 0; e < 4; ++e) {
      const int y = nbx[e];
      if (y < 0) continue;
      if (y == cell) {
        am |= 1u << e;
        continue;
      }
      const double ky = a.chain == 2 ? __ldcg(a.ckey + y) : kInf;
      if (ky < kInf && key_before(ky, y, kx, x)) am |= 1u << e;
    }
    if (!chain_dead(a, x, ld_relaxed_u32(a.spec_ver + a.J + x), ld_relaxed_u64(a.state + x), nbx))
      continue;
    if (claim_chain(a, x, nbx, am, j)) return true;
  }
  return false;
}

template <bool PROF>
__global__ void heapcell_spec_kernel(HcArgs a) {
  extern __shared__ __align__(128) double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const CellGeom& g = a.g;
  HTile T;
  T.pu = g.pu;
  T.U = smem + (size_t)wib * a.tile_doubles;
  T.Ct = T.U + hc_half(g);
  double* before = T.Ct + hc_half(g);  // [4][max_len]
  // [4] snapshots + [4] probes, then the staging record (128 bytes), then locks
  SpecRec* stg = reinterpret_cast<SpecRec*>(before + 8 * a.max_len);
  T.lock = reinterpret_cast<uint8_t*>(before + 8 * a.max_len + 16);
  T.bar = reinterpret_cast<uint64_t*>(T.lock + (((size_t)g.max_w * g.max_h + 7) & ~(size_t)7));
  // (only the warps that process cells own a tile: in CTA 0 the committer's
  // queue lies past warp 0's tile)
  if (a.use_tma && lane == 0 && (blockIdx.x != 0 || wib == 0)) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;"
                 ::"r"((unsigned)__cvta_generic_to_shared(T.bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // The committer runs alone in CTA 0: every gpu-scope acquire issued on an
  // SM invalidates that SM's L1 (CCTL.IVALL).  Workers poll with relaxed
  // loads and acquire once per speculation.
  if (blockIdx.x == 0) {
    if (wib > 1) return;  // warp 0 commits, warp 1 (if any) keeps the queue
    BucketPQ H;
    // [tile][keys: 32 capb doubles][ids: 32 capb ints] in smem when heap_cap
    // > 0, else in global memory; [minima: 32 doubles][ids][slots][counts]
    double* qbase = smem + a.tile_doubles;
    if (a.heap_cap > 0) {
      H.capb = a.heap_cap;
      H.bk = qbase;
      H.bi = reinterpret_cast<int*>(H.bk + 32 * H.capb);
      H.pub = a.harr;
      qbase = reinterpret_cast<double*>(H.bi + 32 * H.capb);
    } else {
      H.capb = a.heap_capb_global;
      H.bk = a.hkey;
      H.bi = a.harr;
      H.pub = nullptr;
    }
    H.mk = qbase;
    H.mi = reinterpret_cast<int*>(H.mk + 32);
    H.msl = H.mi + 32;
    H.cnt = H.msl + 32;
    H.pos = a.hpos;
    H.pubcnt = a.hsize_pub;  // bucket counts, one 128-byte line each
    H.pubmin = a.pubmin;
    H.size = 0;
    if (wib == 1) {
      queue_helper(a, H, lane);
      return;
    }
    H.mk[lane] = kInf;
    H.mi[lane] = 0x7fffffff;
    H.msl[lane] = 0;
    H.cnt[lane] = 0;
    H.pubcnt[32 * lane] = 0;
    __syncwarp();
    committer<PROF>(a, H, T, before, stg, lane);
    return;
  }

  // ---- worker: speculate cells near the top of the heap ----------------------
  const int wpc = blockDim.x >> 5;
  const int wid = (blockIdx.x - 1) * wpc + wib;
  const int nworkers = (gridDim.x - 1) * wpc;
  // small pools (the batch's slices) leave the cells about to be popped
  // unspeculated while the workers walk the buckets: some of them chase the
  // buckets' minima (FHCM/8 on 6 CTAs 345 -> 233 ms); in the full-device pool
  // every queued cell is covered anyway and chasing only re-speculates
  // (148 CTAs: 169 -> 174 ms)
  const bool first_min = nworkers <= a.first_min_pool && (wid >> 5) < a.first_min;
  unsigned polls = 0;
  for (;;) {
    int done = 0;
    if (lane == 0 && (++polls & 7) == 0) done = ld_relaxed_s32(a.done_flag);  // 1 poll in 8
    if (__shfl_sync(kFull, done, 0)) return;
    // Lane 0 alone chooses the job and broadcasts it (lanes reading the
    // shared words independently could see different values, run different
    // trip counts and meet at mismatched warp collectives: a deadlock).  A small pool of workers first tries
    // its bucket's current minimum -- a cell about to be popped -- then, as
    // every pool does, the queued cells: bucket b's entries [b*pub_capb,
    // b*pub_capb + count_b) of the mirror, workers spread over the buckets,
    // then over their slots.
    Job j;
    int got = 0;
    if (lane == 0) {
      const bool wide = nworkers >= 32;
      if (first_min) {
        const int c = ld_relaxed_s32(a.pubmin + 32 * (wid & 31));
        if (c >= 0 && c < a.J) got = pick_job_cell(a, c, j, wid) ? 1 : 0;
      }
      for (int bkt = wide ? (wid & 31) : wid; bkt < 32 && !got; bkt += wide ? 32 : nworkers) {
        const int nb = ld_relaxed_s32(a.hsize_pub + 32 * bkt);
        const int sstep = wide ? (nworkers >> 5) : 1;
        for (int sl = wide ? (wid >> 5) : 0; sl < nb && !got; sl += sstep)
          got = pick_job(a, bkt * a.pub_capb + sl, j, wid) ? 1 : 0;
      }
    }
    if (lane == 0 && a.wdbg) a.wdbg[4 * wid + 2] = 100 + got;
    if (!__shfl_sync(kFull, got, 0)) {
      __nanosleep(a.idle_ns);
      continue;
    }
    if (lane == 0 && a.wdbg) {
      a.wdbg[4 * wid + 0] = 1;
      a.wdbg[4 * wid + 1] = j.cell;
      a.wdbg[4 * wid + 2] = j.kind;
      a.wdbg[4 * wid + 3] = (int)(clock64() >> 10);
      a.owner[(size_t)j.kind * a.J + j.cell] = 0x70000 | wid;
    }
    j.cell = __shfl_sync(kFull, j.cell, 0);
    j.kind = __shfl_sync(kFull, j.kind, 0);
    j.st = __shfl_sync(kFull, j.st, 0);
    j.omask = __shfl_sync(kFull, j.omask, 0);
    j.cflags = __shfl_sync(kFull, j.cflags, 0);
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      j.oslot[d] = __shfl_sync(kFull, j.oslot[d], 0);
      j.dinst[d] = __shfl_sync(kFull, j.dinst[d], 0);
    }
    if (lane == 0 && a.wdbg) a.wdbg[4 * wid + 0] = 13;
    process_cell(a, T, before, stg, j.cell, j.kind, j.st, j.omask, j.oslot, j.cflags, lane);
    if (lane == 0 && a.wdbg) a.wdbg[4 * wid + 0] = 2;
    publish(a, j.cell, j.kind, j.st, j.omask, j.dinst, stg, lane);
    if (lane == 0 && a.wdbg) a.wdbg[4 * wid + 0] = 3;
  }
}

__global__ void heapcell_init_kernel(HcArgs a) {
  const int64_t cellsz = a.cellsz;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < (int64_t)a.J * cellsz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int cell = (int)(k / cellsz);
    const int r = (int)(k - (int64_t)cell * cellsz);
    const int y = r / a.spw, x = r % a.spw;
    int64_t ib, ie, jb, je;
    hc_cell_rect(a.g, a.cx_magic, cell, ib, ie, jb, je);
    double v = kInf;
    if (x < ie - ib && y < je - jb) v = a.u[(jb + y) * a.g.P + a.g.pad + ib + x];
    a.slots[k] = v;  // slot 0 <- the prepared field
    if (r == 0) {
      a.state[cell] = 1ull << 32;  // committed slot 0, plain slot 1, chained slot 2
      for (int kind = 0; kind < 2; ++kind) {
        a.spec_ver[(size_t)kind * a.J + cell] = kSpecNone;
        a.busy[(size_t)kind * a.J + cell] = 0;
        PRec* rec = rec_ptr(a, kind, cell);
        const uint4 none = make_uint4(0u, 0u, 0u, kSpecNone);
        for (int w = 0; w < 8; ++w) rec->w[w] = none;
        rec->w[4].z = kSpecNone;  // tag
      }
      a.ckey[cell] = kInf;
      a.ctag[cell] = kSpecNone;
      a.cval[cell] = kInf;
      a.hpos[cell] = -1;
    }
  }
}

__global__ void heapcell_gather_kernel(HcArgs a) {
  const int64_t cellsz = a.cellsz;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < (int64_t)a.J * cellsz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int cell = (int)(k / cellsz);
    const int r = (int)(k - (int64_t)cell * cellsz);
    const int y = r / a.spw, x = r % a.spw;
    int64_t ib, ie, jb, je;
    hc_cell_rect(a.g, a.cx_magic, cell, ib, ie, jb, je);
    if (x < ie - ib && y < je - jb)
      a.u[(jb + y) * a.g.P + a.g.pad + ib + x] = slot_ptr(a, st_cur(a.state[cell]), cell)[r];
  }
}

// ---- HCM band scheduler ------------------------------------------------------
// north_star (3): instead of popping one cell at a time, every round processes
// all queued cells whose value lies in the acceptance band [kmin, kmin+delta]
// and that are a (value, id) local minimum among the in-band queued cells
// next to them -- so no two cells of a round are adjacent: each reads only
// its own nodes and the cross halo of its four neighbours, none of which
// changes during the round, and the round equals the same pops made one
// after another in any order.  Every pop is the reference's HCM processing
// (heap_cell.cpp:273-312: snapshot, process_to_convergence, the four border
// scans with cell_value min-update, flag OR and insertion), so the algorithm
// is HCM with a different pop order: it ends, like the reference, when no
// cell is queued, i.e. at the discrete fixed point -- within rounding of the
// reference's field (tests: <= 1e-10; measured ~1e-15).  delta =
// (h + h_c) / (2 F_max) is the smallest increment a border scan can add to a
// neighbour's value (cell_value_candidate, cells.hpp:109-112): no cell in the
// band can receive a smaller key from another in-band cell's processing
// (SURVEY finding 5: 854 rounds instead of 22k pops on C2 at 16-node cells).
// Pops, sweeps and node updates are this order's, reported beside the
// reference's; EIK_HCM_EXACT=1 / eik_plan_set_hcm_mode select the exact
// replay (bit-identical, the reference's counters).
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long key_bits(double k) {
  return k == 0.0 ? 0ull : (unsigned long long)__double_as_longlong(k);  // k >= 0
}
__device__ __forceinline__ bool key_less(double ka, int ia, double kb, int ib) {
  return ka < kb || (ka == kb && ia < ib);
}
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(kFull, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// One pop of HCM, in place in u: stage the cell and its cross halo, sweep to
// convergence, write the values back, scan the borders and apply the scans to
// the neighbours (atomics: neighbours of a round's cells may be shared).
__device__ void band_process(const HcArgs& a, HTile& T, double* before, SpecRec* rec, int cell,
                             int lane, long long& sweeps, long long& updates, int* nxt,
                             int* nxt_cnt) {
  const CellGeom& g = a.g;
  int64_t ib, ie, jb, je;
  hc_cell_rect(g, a.cx_magic, cell, ib, ie, jb, je);
  T.w = (int)(ie - ib);
  T.h = (int)(je - jb);
  int cx, cy;
  cell_xy(cell, g.cells_x, a.cx_magic, cx, cy);
  const bool has_nb[4] = {cx > 0, cx + 1 < g.cells_x, cy > 0, cy + 1 < g.cells_y};
  const int nbs[4] = {cell - 1, cell + 1, cell - g.cells_x, cell + g.cells_x};
  double* pstrip = before + 4 * a.max_len;
  // values and costs with the cross halo: by TMA (the box of the padded u
  // and C, +inf / -1 beside the grid and on the dummy rows), or row by row
  unsigned long long tma_tok = 0;
  if (a.use_tma) {
    if (lane == 0) tma_tok = tma_band_tiles(a, T, ib, jb);
  }
  const int tw = a.use_tma ? 0 : T.w + 2;
  for (int y = -1; y <= T.h && !a.use_tma; ++y) {
    const int64_t gj = jb + y;
    const bool rin = gj >= 0 && gj < g.n;
    const double* ur = a.u + gj * g.P + g.pad + ib;
    const double* cr = a.C + gj * g.P + g.pad + ib;
    for (int t = lane; t < tw; t += 32) {
      const int x = t - 1;
      const bool corner = (y < 0 || y >= T.h) && (x < 0 || x >= T.w);
      if (corner) continue;
      T.u(x, y) = rin ? __ldcg(ur + x) : kInf;
      T.Ct[T.ci(x, y)] = rin ? __ldg(cr + x) : -1.0;
    }
  }
  for (int t = lane; t < a.max_len; t += 32) {  // F at the border probe points
    if (t < T.h) {
      pstrip[0 * a.max_len + t] = has_nb[0] ? __ldg(a.probe[0] + (int64_t)cx * g.n + jb + t) : 1.0;
      pstrip[1 * a.max_len + t] = has_nb[1] ? __ldg(a.probe[1] + (int64_t)cx * g.n + jb + t) : 1.0;
    }
    if (t < T.w) {
      pstrip[2 * a.max_len + t] = has_nb[2] ? __ldg(a.probe[2] + (int64_t)cy * g.m + ib + t) : 1.0;
      pstrip[3 * a.max_len + t] = has_nb[3] ? __ldg(a.probe[3] + (int64_t)cy * g.m + ib + t) : 1.0;
    }
  }
  if (a.use_tma) tma_wait(T, __shfl_sync(kFull, tma_tok, 0));
  __syncwarp();
  for (int t = lane; t < T.h; t += 32) {  // border snapshots (heap_cell.cpp:279-282)
    before[0 * a.max_len + t] = T.u(0, t);
    before[1 * a.max_len + t] = T.u(T.w - 1, t);
  }
  for (int t = lane; t < T.w; t += 32) {
    before[2 * a.max_len + t] = T.u(t, 0);
    before[3 * a.max_len + t] = T.u(t, T.h - 1);
  }
  // flags and first removal: only this cell's neighbours write them, and
  // none of them is processed in this round
  unsigned my_flags = 0;
  bool first_removal = false;
  if (lane == 0) {
    my_flags = __ldcg(a.b_flags + cell);
    a.b_flags[cell] = 0;
    first_removal = !__ldcg(a.b_fdone + cell);
    a.b_fdone[cell] = 1;
  }
  my_flags = __shfl_sync(kFull, my_flags, 0);
  first_removal = __shfl_sync(kFull, first_removal, 0);
  reset_locks(T, ib > 0, ie < g.m, jb > 0, je < g.n, lane);
  const CellTile ct{T.U, T.Ct, T.lock, T.pu, T.w, T.h, 2};
  long long nsw = 0, upd = 0;
  {  // process_to_convergence (heap_cell.cpp:130-147)
    int perm[4], nflag = 0;
    for (int k = 0; k < 4; ++k)
      if (my_flags & (1u << kFlagOrder[k])) perm[nflag++] = kFlagOrder[k];
    int at = nflag;
    for (int k = 0; k < 4; ++k)
      if (!(my_flags & (1u << kRotation[k]))) perm[at++] = kRotation[k];
    bool changed = true;
    while (changed) {
      const int dir = nsw < 4 ? perm[nsw] : kRotation[nsw % 4];
      changed = cell_sweep_lock_bands(ct, dir, lane, upd, /*skip=*/nsw >= a.skip_from);
      ++nsw;
    }
  }
  for (int o = 16; o > 0; o >>= 1) upd += __shfl_xor_sync(kFull, upd, o);
  sweeps += nsw;
  updates += upd;
  // values back into the field
  for (int k = lane; k < T.w * T.h; k += 32) {
    const int y = k / T.w, x = k % T.w;
    __stcg(a.u + (jb + y) * g.P + g.pad + ib + x, T.u(x, y));
  }
  scan_all(a, T, before, pstrip, first_removal,
           (has_nb[0] ? 1u : 0u) | (has_nb[1] ? 2u : 0u) | (has_nb[2] ? 4u : 0u) |
               (has_nb[3] ? 8u : 0u),
           rec, lane);
  __syncwarp();
  if (lane < 4 && has_nb[lane]) {  // the scans' effects on the four neighbours
    const int nb = nbs[lane];
    const double cand = rec->cand[lane];
    const unsigned sd = rec->side[lane];
    if (cand < kInf)  // cell_value[nb] = min(cell_value[nb], cand); keys >= 0
      atomicMin(reinterpret_cast<unsigned long long*>(a.cval + nb), key_bits(cand));
    if (sd & 1u) {
      atomicOr(a.b_flags + nb, (sd >> 8) & 0xFFu);
      if (atomicExch(a.b_inq + nb, 1) == 0) nxt[atomicAdd(nxt_cnt, 1)] = nb;
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(256, 1) hcm_band_kernel(HcArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) double smem[];
  __shared__ SpecRec srec[8];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int wpc = blockDim.x >> 5;
  const CellGeom& g = a.g;
  HTile T;
  T.pu = g.pu;
  T.U = smem + (size_t)wib * a.tile_doubles;
  T.Ct = T.U + hc_half(g);
  double* before = T.Ct + hc_half(g);
  T.lock = reinterpret_cast<uint8_t*>(before + 8 * a.max_len);
  T.bar = reinterpret_cast<uint64_t*>(T.lock + (((size_t)g.max_w * g.max_h + 7) & ~(size_t)7));
  if (a.use_tma && (threadIdx.x & 31) == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;"
                 ::"r"((unsigned)__cvta_generic_to_shared(T.bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nthreads = gridDim.x * blockDim.x;
  const int J = a.J;

  // ---- init: cell state, F_max (the band width), the Q-cells -----------------
  unsigned long long cmin = ~0ull;
  for (int c = tid; c < J; c += nthreads) {
    a.cval[c] = kInf;
    a.b_inq[c] = 0;
    a.b_flags[c] = 0;
    a.b_fdone[c] = 0;
  }
  for (int64_t k = tid; k < g.n * g.P; k += nthreads) {  // min C = h / F_max over nodes
    const double c = a.C[k];
    if (c > 0.0) cmin = min(cmin, (unsigned long long)__double_as_longlong(c));
  }
  cmin = warp_min_u64(cmin);
  if (lane == 0 && cmin != ~0ull) atomicMin(a.b_kmin + 1, cmin);
  grid.sync();
  if (tid == 0) {
    for (int k = 0; k < a.n_init; ++k) {  // heap_cell.cpp:255-268
      const int c = a.init_cells[k];
      a.cval[c] = a.init_values[k];
      a.b_inq[c] = 1;
      a.b_list[k] = c;
    }
    a.b_ctl[0] = a.n_init;
    a.b_ctl[1] = 0;
  }
  grid.sync();
  // no node with C > 0 (every node an exit): width 0 -- the minimum cell is
  // still selected every round, so every round makes progress
  const unsigned long long cmin_bits = *(volatile unsigned long long*)(a.b_kmin + 1);
  double delta = 0.0;
  if (cmin_bits != ~0ull)
    delta = a.band_scale * 0.5 * (a.h + fmin(a.hc_x, a.hc_y)) *
            (__longlong_as_double((long long)cmin_bits) / a.h);
  if (!(delta >= 0.0 && delta < kInf)) delta = 0.0;

  long long removals = 0, sweeps = 0, updates = 0;
  long long cyc_sync = 0, cyc_sel = 0, cyc_work = 0, cyc_kmin = 0;  // EIK_HC_PROFILE
  const bool prof = a.prof && threadIdx.x == 0;
  long long tp = prof ? clock64() : 0;
  auto lap = [&](long long& acc) {
    if (prof) {
      const long long t = clock64();
      acc += t - tp;
      tp = t;
    }
  };
  // Adaptive width: a front a few cells wide (the maze, C4) leaves the
  // device idle at the base width, and there a wider band costs no extra
  // pops -- the walls' h/F is 100x the base's (C4 HCM/16: x4 2.44 s, 303 k
  // pops; x64 0.40 s, 282 k; x128 41 ms, 255 k; x256 31 ms, 233 k) -- while a
  // wide front re-queues cells under a wide band (C2 HCM/16 x16: 2.1x the
  // pops).  The multiplier doubles after a round of fewer than 32 cells and
  // halves after one of more than band_shrink (128; x1..x64 of the base): a
  // function of the values alone, so a solve stays bit-reproducible on any
  // grid size.  (Narrowing later -- 256, 512, 1024 -- buys C4 HCM/16 90, 38,
  // 33 ms but costs the C2 matrix 5-10 % in re-queued pops: 1169 -> 1111,
  // 1083, 1053 M points/s at 20 steps.)
  double mult = 1.0;
  int round = 0;
  for (;; ++round) {
    const int par = round & 1;
    int* cur = a.b_list + (size_t)par * J;
    int* nxt = a.b_list + (size_t)(par ^ 1) * J;
    const int ncur = *(volatile int*)(a.b_ctl + par);
    if (ncur == 0) break;
    // phase 1: the band's base, the minimum key of the queued cells
    unsigned long long mk = ~0ull;
    for (int i = tid; i < ncur; i += nthreads) mk = min(mk, key_bits(__ldcg(a.cval + __ldcg(cur + i))));
    mk = warp_min_u64(mk);
    if (lane == 0 && mk != ~0ull) atomicMin(a.b_kmin, mk);
    if (tid == 0) {
      a.b_ctl[par ^ 1] = 0;
      a.b_ctl[2] = 0;
      a.b_ctl[3] = 0;
    }
    lap(cyc_kmin);
    grid.sync();
    lap(cyc_sync);
    // phase 2: select the in-band local minima; the rest stay queued
    const double kmin = __longlong_as_double((long long)*(volatile unsigned long long*)a.b_kmin);
    const double band = kmin + delta * mult;
    for (int i = tid; i < ncur; i += nthreads) {
      const int c = __ldcg(cur + i);
      const double k = __ldcg(a.cval + c);
      bool sel = k <= band;
      if (sel) {
        int cx, cy;
        cell_xy(c, g.cells_x, a.cx_magic, cx, cy);
        const int nbs[4] = {cx > 0 ? c - 1 : -1, cx + 1 < g.cells_x ? c + 1 : -1,
                            cy > 0 ? c - g.cells_x : -1, cy + 1 < g.cells_y ? c + g.cells_x : -1};
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          const int nb = nbs[d];
          if (nb >= 0 && __ldcg(a.b_inq + nb)) {
            const double kn = __ldcg(a.cval + nb);
            if (kn <= band && key_less(kn, nb, k, c)) sel = false;
          }
        }
      }
      if (sel) a.b_work[atomicAdd(a.b_ctl + 2, 1)] = c;
      else nxt[atomicAdd(a.b_ctl + (par ^ 1), 1)] = c;
    }
    lap(cyc_sel);
    grid.sync();
    lap(cyc_sync);
    // phase 3: the selected cells, one warp each
    if (tid == 0) a.b_kmin[0] = ~0ull;
    const int nwork = *(volatile int*)(a.b_ctl + 2);
    if (a.band_adapt) {
      if (nwork < 32 && mult < 64.0) mult *= 2.0;
      else if (nwork > a.band_shrink && mult > 1.0) mult *= 0.5;
    }
    if (tid == 0) {
      removals += nwork;
      if (removals > a.budget) atomicExch(a.status, 3);  // read by all after the sync
      // every round selects at least the minimum cell; an empty one is a bug
      if (nwork == 0 || round > a.budget) atomicExch(a.status, kStatusWatchdog);
    }
    for (;;) {
      int i = 0;
      if (lane == 0) i = atomicAdd(a.b_ctl + 3, 1);
      i = __shfl_sync(kFull, i, 0);
      if (i >= nwork) break;
      const int c = __ldcg(a.b_work + i);
      if (lane == 0) a.b_inq[c] = 0;  // popped
      band_process(a, T, before, &srec[wib], c, lane, sweeps, updates, nxt, a.b_ctl + (par ^ 1));
    }
    lap(cyc_work);
    grid.sync();
    lap(cyc_sync);
    const int stv = *(volatile int*)a.status;  // set before the sync: all threads agree
    if (stv == 3 || stv == kStatusWatchdog) break;
  }
  if (lane == 0) {
    atomicAdd(a.counters + 1, (unsigned long long)sweeps);
    atomicAdd(a.counters + 2, (unsigned long long)updates);
  }
  if (tid == 0) {
    atomicAdd(a.counters + 0, (unsigned long long)removals);
    a.b_ctl[4] = round;
  }
  if (prof) {  // per-CTA sums (thread 0): where a round's time goes
    atomicAdd(a.counters + 8, (unsigned long long)cyc_sync);
    atomicAdd(a.counters + 9, (unsigned long long)cyc_sel);
    atomicAdd(a.counters + 10, (unsigned long long)cyc_work);
    atomicAdd(a.counters + 11, (unsigned long long)cyc_kmin);
  }
}

// ---- cells too large for a shared-memory tile ------------------------------
// heap_cell_solve (heap_cell.cpp:243-324) exactly as the reference runs it:
// one warp pops the minimum (value, id) cell (a warp argmin over the J cells;
// big cells mean small J), processes it in place in u -- the tile aliases the
// padded global field, so the cross halo is the neighbours' nodes -- with the
// band-splitting engine (big_cell_sweep), scans its borders and updates the
// neighbours.  The order is the reference's, so values and every counter are.
__global__ void __launch_bounds__(32) heapcell_serial_kernel(HcArgs a) {
  __shared__ SpecRec rec;
  const int lane = threadIdx.x;
  const CellGeom& g = a.g;
  const int J = a.J;
  for (int c = lane; c < J; c += 32) {
    a.cval[c] = kInf;
    a.b_inq[c] = 0;
    a.b_flags[c] = 0;
    a.b_fdone[c] = 0;
  }
  __syncwarp();
  if (lane == 0)
    for (int k = 0; k < a.n_init; ++k) {  // heap_cell.cpp:255-268
      const int c = a.init_cells[k];
      a.cval[c] = a.init_values[k];
      a.b_inq[c] = 1;
      if (a.fast) a.b_flags[c] = 0xFu;
    }
  __syncwarp();
  double* before = a.big_scratch;
  double* pstrip = before + 4 * a.max_len;
  long long removals = 0, sweeps = 0, updates = 0, mon_checks = 0, mon_single = 0;
  for (;;) {
    // pop: minimum (value, id) over the queued cells (ties to the smaller id)
    double kb = kInf;
    int ib_ = 0x7fffffff;
    for (int c = lane; c < J; c += 32)
      if (a.b_inq[c] && key_less(a.cval[c], c, kb, ib_)) {
        kb = a.cval[c];
        ib_ = c;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ok = __shfl_xor_sync(kFull, kb, o);
      const int oi = __shfl_xor_sync(kFull, ib_, o);
      if (key_less(ok, oi, kb, ib_)) {
        kb = ok;
        ib_ = oi;
      }
    }
    if (ib_ == 0x7fffffff) break;
    const int cell = ib_;
    if (++removals > a.budget) {
      if (lane == 0) atomicExch(a.status, 3);
      return;
    }
    int64_t ib, ie, jb, je;
    hc_cell_rect(g, a.cx_magic, cell, ib, ie, jb, je);
    HTile T;
    T.pu = (int)g.P;
    T.w = (int)(ie - ib);
    T.h = (int)(je - jb);
    T.U = a.u + (jb - 1) * g.P + g.pad + ib - 2;  // node (x, y) at (y+1)*P + x+2
    T.Ct = const_cast<double*>(a.C) + (jb - 1) * g.P + g.pad + ib - 2;
    T.lock = a.big_lock;
    int cx, cy;
    cell_xy(cell, g.cells_x, a.cx_magic, cx, cy);
    const bool has_nb[4] = {cx > 0, cx + 1 < g.cells_x, cy > 0, cy + 1 < g.cells_y};
    const int nbs[4] = {cell - 1, cell + 1, cell - g.cells_x, cell + g.cells_x};
    for (int t = lane; t < a.max_len; t += 32) {
      if (t < T.h) {
        before[0 * a.max_len + t] = T.u(0, t);
        before[1 * a.max_len + t] = T.u(T.w - 1, t);
        pstrip[0 * a.max_len + t] = has_nb[0] ? __ldg(a.probe[0] + (int64_t)cx * g.n + jb + t) : 1.0;
        pstrip[1 * a.max_len + t] = has_nb[1] ? __ldg(a.probe[1] + (int64_t)cx * g.n + jb + t) : 1.0;
      }
      if (t < T.w) {
        before[2 * a.max_len + t] = T.u(t, 0);
        before[3 * a.max_len + t] = T.u(t, T.h - 1);
        pstrip[2 * a.max_len + t] = has_nb[2] ? __ldg(a.probe[2] + (int64_t)cy * g.m + ib + t) : 1.0;
        pstrip[3 * a.max_len + t] = has_nb[3] ? __ldg(a.probe[3] + (int64_t)cy * g.m + ib + t) : 1.0;
      }
    }
    const unsigned my_flags = a.b_flags[cell];
    const bool first_removal = !a.b_fdone[cell];
    __syncwarp();
    if (lane == 0) {
      a.b_inq[cell] = 0;
      a.b_flags[cell] = 0;
      a.b_fdone[cell] = 1;
    }
    reset_locks(T, ib > 0, ie < g.m, jb > 0, je < g.n, lane);
    const CellTile ct{T.U, T.Ct, T.lock, T.pu, T.w, T.h, 2};
    long long nsw = 0, upd = 0;
    {  // process_flagged_once / process_to_convergence (heap_cell.cpp:130-160)
      int perm[4], nflag = 0;
      for (int k = 0; k < 4; ++k)
        if (my_flags & (1u << kFlagOrder[k])) perm[nflag++] = kFlagOrder[k];
      int at = nflag;
      for (int k = 0; k < 4; ++k)
        if (!(my_flags & (1u << kRotation[k]))) perm[at++] = kRotation[k];
      bool changed = true;
      for (;;) {
        if (a.fast ? nsw >= nflag : !changed) break;
        const int dir = nsw < 4 ? perm[nsw] : kRotation[nsw % 4];
        changed = big_cell_sweep<2>(ct, dir, lane, upd);
        ++nsw;
      }
    }
    for (int o = 16; o > 0; o >>= 1) upd += __shfl_xor_sync(kFull, upd, o);
    sweeps += nsw;
    updates += upd;
    __syncwarp();
    scan_all(a, T, before, pstrip, first_removal,
             (has_nb[0] ? 1u : 0u) | (has_nb[1] ? 2u : 0u) | (has_nb[2] ? 4u : 0u) |
                 (has_nb[3] ? 8u : 0u),
             &rec, lane);
    __syncwarp();
    if (lane == 0) {
      for (int d = 0; d < 4; ++d) {  // W, E, S, N in the reference's order
        if (!has_nb[d]) continue;
        const int nb = nbs[d];
        const unsigned sd = rec.side[d];
        if (rec.cand[d] < a.cval[nb]) a.cval[nb] = rec.cand[d];
        if (sd & 1u) {
          a.b_flags[nb] |= (sd >> 8) & 0xFFu;
          if (sd & (1u << 16)) {
            ++mon_checks;
            if (sd & (1u << 24)) ++mon_single;
          }
          a.b_inq[nb] = 1;
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    a.counters[0] = (unsigned long long)removals;
    a.counters[1] = (unsigned long long)sweeps;
    a.counters[2] = (unsigned long long)updates;
    a.counters[3] = (unsigned long long)mon_checks;
    a.counters[4] = (unsigned long long)mon_single;
  }
}

}  // namespace

size_t heapcell_smem_bytes(const CellGeom& g, int max_len) {
  // values, costs, 4 snapshots + 4 probe strips, the staging record, the lock
  // bytes, the warp's mbarrier; a multiple of 128 bytes (aligned tiles)
  const size_t b = sizeof(double) * (2 * (size_t)hc_half(g) + 8 * (size_t)max_len + 16) +
                   (((size_t)g.max_w * g.max_h + 7) & ~(size_t)7) + 8;
  return (b + 127) & ~(size_t)127;
}

size_t heapcell_committer_heap_bytes(int capb) {
  // 32 buckets of capb (key, id) entries + per-bucket minimum, id, slot,
  // count + the committer -> helper mailbox
  return (size_t)32 * capb * (sizeof(double) + 4) + 32 * (sizeof(double) + 12) + 16;
}

namespace {
size_t heapcell_launch_smem(int64_t tile_doubles, int heap_cap, int warps_per_cta,
                            size_t min_smem) {
  size_t smem = (size_t)warps_per_cta * tile_doubles * sizeof(double);
  smem = std::max(smem, tile_doubles * sizeof(double) +
                            heapcell_committer_heap_bytes(heap_cap > 0 ? heap_cap : 0));
  return std::max(smem, min_smem);
}
}  // namespace

cudaError_t heapcell_capacity(int64_t tile_doubles, int heap_cap, int warps_per_cta,
                              size_t min_smem, int* ctas) {
  const size_t smem = heapcell_launch_smem(tile_doubles, heap_cap, warps_per_cta, min_smem);
  const void* kern = (const void*)heapcell_spec_kernel<false>;
  cudaError_t e = ensure_dynamic_smem(kern, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * warps_per_cta, smem);
  if (e != cudaSuccess) return e;
  *ctas = per_sm * sms;
  return cudaSuccess;
}

cudaError_t launch_heapcell(const HcArgs& args, int warps_per_cta, int max_ctas, cudaStream_t s,
                            int* launches, int* grid) {
  const int64_t total = (int64_t)args.J * args.cellsz;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  heapcell_init_kernel<<<blocks, 256, 0, s>>>(args);
  const size_t smem =
      heapcell_launch_smem(args.tile_doubles, args.heap_cap, warps_per_cta, (size_t)args.min_smem);
  // the instrumented instantiation only when EIK_HC_PROFILE asked for it
  const void* kern = args.prof ? (const void*)heapcell_spec_kernel<true>
                               : (const void*)heapcell_spec_kernel<false>;
  cudaError_t e = ensure_dynamic_smem(kern, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern,
                                                    32 * warps_per_cta, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int ctas = std::min(per_sm * sms, max_ctas);
  if (ctas < 1) ctas = 1;
  if (grid) *grid = ctas;
  HcArgs a = args;
  void* params[] = {&a};
  e = cudaLaunchCooperativeKernel(kern, dim3(ctas),
                                  dim3(32 * warps_per_cta), params, smem, s);
  if (e != cudaSuccess) return e;
  heapcell_gather_kernel<<<blocks, 256, 0, s>>>(args);
  *launches += 3;
  return cudaGetLastError();
}

cudaError_t hcm_band_capacity(int64_t tile_doubles, int warps_per_cta, size_t min_smem,
                              int* ctas) {
  const size_t smem = std::max((size_t)warps_per_cta * tile_doubles * sizeof(double), min_smem);
  const void* kern = (const void*)hcm_band_kernel;
  cudaError_t e = ensure_dynamic_smem(kern, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * warps_per_cta, smem);
  if (e != cudaSuccess) return e;
  *ctas = per_sm * sms;
  return cudaSuccess;
}

cudaError_t launch_hcm_band(const HcArgs& args, int warps_per_cta, int max_ctas, cudaStream_t s,
                            int* launches, int* grid) {
  const size_t smem =
      std::max((size_t)warps_per_cta * args.tile_doubles * sizeof(double), (size_t)args.min_smem);
  const void* kern = (const void*)hcm_band_kernel;
  cudaError_t e = ensure_dynamic_smem(kern, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * warps_per_cta, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int ctas = std::min(per_sm * sms, max_ctas);
  if (ctas < 1) ctas = 1;
  if (grid) *grid = ctas;
  HcArgs a = args;
  void* params[] = {&a};
  e = cudaLaunchCooperativeKernel(kern, dim3(ctas), dim3(32 * warps_per_cta), params, smem, s);
  *launches += 1;
  return e;
}

cudaError_t launch_heapcell_serial(const HcArgs& a, cudaStream_t s, int* launches) {
  heapcell_serial_kernel<<<1, 32, 0, s>>>(a);
  *launches += 1;
  return cudaGetLastError();
}

}  // namespace eikb200
