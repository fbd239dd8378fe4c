// FMSM Part I on the host: the coarse problem, its Fast March, and the
// quantised one-pass cell order (/root/reference/proj/src/fmsm.cpp:10-162).
// The reference runs this part on the host too; the fine pass (Part II) is
// the device kernel in k_cells.cu.  Everything here is O(J log J) in the
// number of cells J and must reproduce the reference's order bit for bit,
// so it follows the reference's arithmetic exactly (no FMA: this file is
// compiled with -ffp-contract=off through nvcc's host compiler flags).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

#include "eik_host.h"

namespace eikb200 {

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

// local_update.hpp:30-43 with c = h / f precomputed (the same IEEE division)
inline double quadrant_c(double ua, double ub, double c) {
  if (std::isfinite(ua) && std::isfinite(ub)) {
    const double diff = ua - ub;
    if (std::abs(diff) <= c) return 0.5 * (ua + ub) + 0.5 * std::sqrt(2.0 * c * c - diff * diff);
  }
  return c + std::min(ua, ub);
}

// 4-ary min-heap of (value, id) entries with lazy deletion: a decrease-key
// pushes a new entry and the superseded one is skipped when it surfaces.
// The live entries are exactly an indexed heap's -- a node's current (value,
// id) -- and a stale entry of a node carries a larger value than its live
// one, so pops come out in the reference's order: minimum value, ties to the
// smaller id (indexed_min_heap.hpp:36-48,66-69).  Values are >= 0 (exit
// costs are refused when negative, candidates only add to them), so an
// entry packs into one 128-bit word -- value bits above the id -- whose
// unsigned order is the (value, id) order; -0.0 is folded into +0.0.
class Heap {
 public:
  using Ent = unsigned __int128;
  Heap() { h_.reserve(1024); }
  bool empty() const { return h_.empty(); }
  static Ent pack(int32_t id, double k) {
    uint64_t b;
    std::memcpy(&b, &k, 8);
    if (k == 0.0) b = 0;
    return ((Ent)b << 32) | (uint32_t)id;
  }
  static double key_of(Ent e) {
    const uint64_t b = (uint64_t)(e >> 32);
    double k;
    std::memcpy(&k, &b, 8);
    return k;
  }
  bool push(int32_t id, double k) {
    const Ent e = pack(id, k);
    h_.push_back(e);
    int32_t p = (int32_t)h_.size() - 1;
    while (p > 0) {
      const int32_t par = (p - 1) >> 2;
      if (!(e < h_[par])) break;
      h_[p] = h_[par];
      p = par;
    }
    h_[p] = e;
    return true;
  }
  // the minimum entry (value, id); removes it
  void pop(double& k, int32_t& id) {
    const Ent top = h_[0];
    k = key_of(top);
    id = (int32_t)(uint32_t)top;
    const Ent last = h_.back();
    h_.pop_back();
    const int32_t n = (int32_t)h_.size();
    if (n == 0) return;
    int32_t p = 0;
    Ent* h = h_.data();
    for (;;) {
      const int32_t c0 = 4 * p + 1;
      if (c0 >= n) break;
      int32_t c = c0;
      Ent mc = h[c0];
      if (c0 + 3 < n) {  // branch-free minimum of four children
        const Ent a1 = h[c0 + 1], a2 = h[c0 + 2], a3 = h[c0 + 3];
        const int32_t i01 = a1 < mc ? c0 + 1 : c0;
        const Ent m01 = a1 < mc ? a1 : mc;
        const int32_t i23 = a3 < a2 ? c0 + 3 : c0 + 2;
        const Ent m23 = a3 < a2 ? a3 : a2;
        c = m23 < m01 ? i23 : i01;
        mc = m23 < m01 ? m23 : m01;
      } else {
        for (int32_t q = c0 + 1; q < n; ++q)
          if (h[q] < mc) {
            mc = h[q];
            c = q;
          }
      }
      if (!(mc < last)) break;
      h[p] = mc;
      p = c;
    }
    h[p] = last;
  }

 private:
  std::vector<Ent> h_;
};

// Exact (value, id) priority queue for the coarse Fast March, bucketed by
// value: bucket b holds the entries with floor((value - base) / delta) == b,
// kept in a ring of nb buckets past the current one.  A Fast March's keys
// only move forward by at most max(h_c / F) per acceptance (a candidate is at
// most the accepted value plus its own h_c / F, local_update.hpp:30-43), so
// every live entry lies within the ring; the current bucket is sorted once
// when it becomes current and popped from its end, and an entry landing at
// or below the current bucket (ulp-level non-monotone candidates) is
// inserted into it in order.  Buckets partition the value axis monotonically,
// so pops come out in exactly the (value, id) order of Heap (and of the
// reference's indexed heap).  push() returns false when an entry would fall
// past the ring (the caller then restarts with Heap).
class BucketQueue {
 public:
  using Ent = Heap::Ent;
  BucketQueue(double base, double delta, int nb) : base_(base), inv_(1.0 / delta), mask_(nb - 1),
                                                    ring_(nb) {}
  bool empty() const { return count_ == 0; }
  bool push(int32_t id, double k) {
    const Ent e = Heap::pack(id, k);
    const double f = std::floor((k - base_) * inv_);
    if (!(f < 9.0e15)) return false;  // inf / NaN / beyond any ring
    const int64_t b = (int64_t)f;
    if (b <= cur_) {  // into the current (sorted, descending) bucket
      auto it = std::upper_bound(curv_.begin(), curv_.end(), e, [](const Ent& x, const Ent& y) {
        return x > y;
      });
      curv_.insert(it, e);
    } else {
      if (b - cur_ > mask_) return false;
      ring_[b & mask_].push_back(e);
    }
    ++count_;
    return true;
  }
  void pop(double& k, int32_t& id) {
    while (curv_.empty()) {  // the next non-empty bucket becomes current
      ++cur_;
      std::vector<Ent>& r = ring_[cur_ & mask_];
      if (r.empty()) continue;
      curv_.swap(r);
      std::sort(curv_.begin(), curv_.end(), [](const Ent& x, const Ent& y) { return x > y; });
    }
    const Ent e = curv_.back();
    curv_.pop_back();
    --count_;
    k = Heap::key_of(e);
    id = (int32_t)(uint32_t)e;
  }

 private:
  double base_, inv_;
  int64_t mask_;
  int64_t cur_ = -1;
  int64_t count_ = 0;
  std::vector<std::vector<Ent>> ring_;
  std::vector<Ent> curv_;
};

// Stable LSD radix sort of 64-bit keys, 11-bit digits (cache-sized count
// tables), skipping digits that are equal in every key.
void radix_sort_u64(std::vector<uint64_t>& a) {
  constexpr int kBits = 11;
  constexpr uint64_t kMask = (1u << kBits) - 1;
  std::vector<uint64_t> tmp(a.size());
  uint64_t all_or = 0, all_and = ~0ull;
  for (uint64_t v : a) {
    all_or |= v;
    all_and &= v;
  }
  std::vector<uint32_t> cnt(1u << kBits);
  for (int shift = 0; shift < 64; shift += kBits) {
    if ((((all_or ^ all_and) >> shift) & kMask) == 0) continue;  // constant digit
    std::fill(cnt.begin(), cnt.end(), 0u);
    for (uint64_t v : a) ++cnt[(v >> shift) & kMask];
    uint32_t sum = 0;
    for (auto& c : cnt) {
      const uint32_t t = c;
      c = sum;
      sum += t;
    }
    for (uint64_t v : a) tmp[cnt[(v >> shift) & kMask]++] = v;
    a.swap(tmp);
  }
}

}  // namespace

void split_axis(int64_t nodes, int32_t cells, std::vector<int64_t>& b, std::vector<int64_t>& e) {
  const int64_t base = nodes / cells;  // cells.cpp:7-19
  b.resize(cells);
  e.resize(cells);
  int64_t at = 0;
  for (int32_t c = 0; c < cells; ++c) {
    b[c] = at;
    at += base;
    if (c == cells - 1) at = nodes;
    e[c] = at;
  }
}

int fmsm_part1(const eik_problem* p, const eik_cells* cells, FmsmOrder* out) {
  const eik_grid& g = p->grid;
  const int32_t cx = cells->cells_x, cy = cells->cells_y;
  const int64_t J = (int64_t)cx * cy;
  std::vector<int64_t> ib, ie, jb, je;
  split_axis(g.m, cx, ib, ie);
  split_axis(g.n, cy, jb, je);
  const double hc_x = (double)(g.m / cx) * g.h;  // cells.cpp:44
  auto gx = [&](int64_t i) { return g.x0 + (double)i * g.h; };
  auto gy = [&](int64_t j) { return g.y0 + (double)j * g.h; };
  // cell centres (cells.hpp:44-48), one per column and per row
  std::vector<double> ccx(cx), ccy(cy);
  for (int32_t a = 0; a < cx; ++a) ccx[a] = 0.5 * (gx(ib[a]) + gx(ie[a] - 1));
  for (int32_t b = 0; b < cy; ++b) ccy[b] = 0.5 * (gy(jb[b]) + gy(je[b] - 1));
  const double* Fc = cells->center_speed;

  // coarse exits (fmsm.cpp:37-81)
  std::vector<double> best(J, kInf);
  if (p->n_exit_points > 0) {
    const bool single = p->n_exit_points == 1;
    std::vector<int64_t> cand;
    for (int64_t k = 0; k < p->n_exit_points; ++k) {
      const double qx = p->exit_points_xy[2 * k], qy = p->exit_points_xy[2 * k + 1];
      // The reference takes dmin = min hypot over every cell, then every cell
      // with hypot <= dmin + 1e-12 (h + dmin).  Squared distances prune first:
      // a cell with dx^2 + dy^2 > R^2, R = sqrt(smin)(1 + 1e-6) + 1e-9 h, has
      // hypot > dmin + tie by a margin far above rounding, so hypot is
      // evaluated only on the few cells that can be nearest or tie.
      double smin = kInf;
      for (int32_t b = 0; b < cy; ++b) {
        const double dy = qy - ccy[b], dy2 = dy * dy;
        for (int32_t a = 0; a < cx; ++a) {
          const double dx = qx - ccx[a];
          smin = std::min(smin, dx * dx + dy2);
        }
      }
      const double R = std::sqrt(smin) * (1.0 + 1e-6) + 1e-9 * g.h, R2 = R * R;
      cand.clear();
      for (int32_t b = 0; b < cy; ++b) {
        const double dy = qy - ccy[b], dy2 = dy * dy;
        if (dy2 > R2) continue;
        for (int32_t a = 0; a < cx; ++a) {
          const double dx = qx - ccx[a];
          if (dx * dx + dy2 <= R2) cand.push_back((int64_t)b * cx + a);
        }
      }
      double dmin = kInf;
      for (int64_t c : cand) dmin = std::min(dmin, std::hypot(qx - ccx[c % cx], qy - ccy[c / cx]));
      const double tie = 1e-12 * (g.h + dmin);
      for (int64_t c : cand) {
        const double dist = std::hypot(qx - ccx[c % cx], qy - ccy[c / cx]);
        if (dist > dmin + tie) continue;
        const double cost = single ? p->exit_point_cost[k] : p->exit_point_cost[k] + dist / Fc[c];
        best[c] = std::min(best[c], cost);
      }
    }
  } else {
    const bool single = p->n_exit == 1;
    for (int64_t k = 0; k < p->n_exit; ++k) {
      const int64_t idx = p->exit_nodes[k], i = idx % g.m, j = idx / g.m;
      // cell_of_node (cells.cpp:23-30): the last cell with begin <= node
      const int64_t a = std::upper_bound(ib.begin(), ib.end(), i) - ib.begin() - 1;
      const int64_t b = std::upper_bound(jb.begin(), jb.end(), j) - jb.begin() - 1;
      const int64_t c = b * cx + a;
      const double dist = std::hypot(gx(i) - ccx[a], gy(j) - ccy[b]);
      const double cost = single ? p->exit_cost[k] : p->exit_cost[k] + dist / Fc[c];
      best[c] = std::min(best[c], cost);
    }
  }

  // coarse Fast March (classic_solvers.cpp:28-92) on the cx x cy lattice,
  // spacing hc_x, speed = F at the actual cell centres.  The lattice is
  // padded by one ring (value +inf, label accepted), so a neighbour outside
  // the lattice reads +inf and is never updated: no bounds checks, no
  // divisions.  Padded index p = (b + 1) * W + a + 1 orders like the cell id.
  const int64_t W = (int64_t)cx + 2;
  const int64_t NP = W * ((int64_t)cy + 2);
  std::vector<double> v(NP, kInf), cc(NP, 0.0);
  std::vector<uint8_t> label(NP, 2);  // 0 far, 1 considered, 2 accepted / exit / pad
  out->is_q.assign(J, 0);
  std::vector<int32_t> seq;  // acceptance sequence (cell ids): exits, then pops
  seq.reserve(J);
  for (int32_t b = 0; b < cy; ++b)
    for (int32_t a = 0; a < cx; ++a) {
      const int64_t c = (int64_t)b * cx + a, q = (b + 1) * W + a + 1;
      cc[q] = hc_x / Fc[c];  // h_c / F, as quadrant_update computes it
      if (std::isfinite(best[c])) {
        out->is_q[c] = 1;
        v[q] = best[c];
        seq.push_back((int32_t)c);
      } else {
        label[q] = 0;
      }
    }
  const int64_t nq = (int64_t)seq.size();
  if (nq == 0) return 1;

  int64_t updates = 0, pops = 0;
  const int64_t off[4] = {1, -1, W, -W};  // E, W, N, S (di/dj of classic_solvers.cpp:38-39)
  auto update = [&](int64_t q) {
    ++updates;
    return quadrant_c(std::min(v[q + 1], v[q - 1]), std::min(v[q + W], v[q - W]), cc[q]);
  };
  // Returns false when the bucketed queue overflows its ring (the run then
  // restarts from the initial state with the heap).
  auto march = [&](auto& H) -> bool {
    for (int64_t k = 0; k < nq; ++k) {
      const int64_t c = seq[k], q = (c / cx + 1) * W + c % cx + 1;
      for (int d = 0; d < 4; ++d) {
        const int64_t nqd = q + off[d];
        if (label[nqd] != 0) continue;
        label[nqd] = 1;
        const double cand = update(nqd);
        if (cand < v[nqd]) v[nqd] = cand;
        if (!H.push((int32_t)nqd, v[nqd])) return false;
      }
    }
    while (!H.empty()) {
      double key;
      int32_t top;
      H.pop(key, top);
      const int64_t q = top;
      if (label[q] == 2 || key != v[q]) continue;  // superseded entry
      ++pops;
      label[q] = 2;
      seq.push_back((int32_t)(q - W - 1 - 2 * (q / W - 1)));
      for (int d = 0; d < 4; ++d) {
        const int64_t nqd = q + off[d];
        if (label[nqd] == 2) continue;
        const double cand = update(nqd);
        if (label[nqd] == 0) {
          label[nqd] = 1;
          if (cand < v[nqd]) v[nqd] = cand;
          if (!H.push((int32_t)nqd, v[nqd])) return false;
        } else if (cand < v[nqd]) {
          v[nqd] = cand;
          if (!H.push((int32_t)nqd, cand)) return false;
        }
      }
    }
    return true;
  };
  // bucket width: an eighth of the smallest h_c / F; ring: the largest h_c / F
  // (the reach of one acceptance) plus the spread of the exits' costs
  double cmin = kInf, cmax = 0.0, qmin = kInf, qmax = -kInf;
  for (int64_t q = 0; q < NP; ++q)
    if (cc[q] > 0.0) {
      cmin = std::min(cmin, cc[q]);
      cmax = std::max(cmax, cc[q]);
    }
  for (int64_t k = 0; k < nq; ++k) {
    const int64_t c = seq[k];
    qmin = std::min(qmin, best[c]);
    qmax = std::max(qmax, best[c]);
  }
  bool done = false;
  const double delta = cmin / 8.0;
  const double span = (qmax - qmin) + 2.0 * cmax;
  if (delta > 0.0 && std::isfinite(span) && span / delta < (double)(1 << 20)) {
    int nb = 64;
    while ((double)nb < span / delta + 4.0) nb <<= 1;
    BucketQueue B(qmin, delta, nb);
    done = march(B);
    if (!done) {  // a key past the ring: start over with the heap
      for (int32_t b = 0; b < cy; ++b)
        for (int32_t a = 0; a < cx; ++a) {
          const int64_t c = (int64_t)b * cx + a, q = (b + 1) * W + a + 1;
          v[q] = std::isfinite(best[c]) ? best[c] : kInf;
          label[q] = std::isfinite(best[c]) ? 2 : 0;
        }
      seq.resize(nq);
      updates = pops = 0;
    }
  }
  if (!done) {
    Heap H;
    march(H);
  }
  out->coarse_updates = updates;
  out->coarse_pops = pops;
  const int64_t nreached = (int64_t)seq.size();
  for (int64_t c = 0; c < J && nreached < J; ++c)  // never reached: +inf, by id
    if (label[(c / cx + 1) * W + c % cx + 1] == 0) seq.push_back((int32_t)c);

  // quantised acceptance order (fmsm.cpp:138-160): sort by (floor(v /
  // 1e-9 vmax), id).  (key, id) packed into one word: keys are <= 1e9 < 2^31
  // (an unreached cell sorts last), ids < 2^31.  The acceptance sequence is
  // already sorted up to near-ties and the exits' place, so an insertion
  // sort with a move budget finishes it in O(J); past the budget, a radix
  // sort.  Either way the result is the reference's stable sort.
  std::vector<double> vc(J);  // values by cell id
  double vmax = hc_x;
  for (int32_t b = 0; b < cy; ++b)
    for (int32_t a = 0; a < cx; ++a) {
      const double x = v[(b + 1) * W + a + 1];
      vc[(int64_t)b * cx + a] = x;
      if (std::isfinite(x)) vmax = std::max(vmax, x);
    }
  const double quantum = 1e-9 * vmax;
  std::vector<uint64_t> kw(J);
  for (int64_t r = 0; r < J; ++r) {
    const int64_t c = seq[r];
    const double x = vc[c];
    const uint64_t key = std::isfinite(x) ? (uint64_t)std::floor(x / quantum) : 0xFFFFFFFFull;
    kw[r] = (key << 32) | (uint64_t)c;
  }
  {
    int64_t budget = 8 * J + 64;
    bool ok = true;
    for (int64_t r = 1; r < J && ok; ++r) {
      const uint64_t x = kw[r];
      int64_t s = r;
      while (s > 0 && kw[s - 1] > x) {
        kw[s] = kw[s - 1];
        --s;
        if (--budget < 0) {
          ok = false;
          break;
        }
      }
      kw[s] = x;
    }
    if (!ok) radix_sort_u64(kw);
  }
  out->order.resize(J);
  for (int64_t r = 0; r < J; ++r) out->order[r] = (int32_t)(kw[r] & 0xFFFFFFFFull);
  out->rank.resize(J);
  for (int64_t r = 0; r < J; ++r) out->rank[out->order[r]] = (int32_t)r;
  return 0;
}

}  // namespace eikb200
