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
// smaller id (indexed_min_heap.hpp:36-48,66-69).  No position index: every
// sift touches only the contiguous heap array.
class Heap {
 public:
  Heap() { h_.reserve(1024); }
  bool empty() const { return h_.empty(); }
  void push(int32_t id, double k) {
    h_.push_back({k, id});
    int32_t p = (int32_t)h_.size() - 1;
    const Ent e = h_[p];
    while (p > 0) {
      const int32_t par = (p - 1) >> 2;
      if (!less(e, h_[par])) break;
      h_[p] = h_[par];
      p = par;
    }
    h_[p] = e;
  }
  // the minimum entry (value, id); removes it
  void pop(double& k, int32_t& id) {
    k = h_[0].k;
    id = h_[0].id;
    const Ent last = h_.back();
    h_.pop_back();
    const int32_t n = (int32_t)h_.size();
    if (n == 0) return;
    int32_t p = 0;
    for (;;) {
      const int32_t c0 = 4 * p + 1;
      if (c0 >= n) break;
      int32_t c = c0;
      const int32_t ce = std::min(c0 + 4, n);
      for (int32_t q = c0 + 1; q < ce; ++q)
        if (less(h_[q], h_[c])) c = q;
      if (!less(h_[c], last)) break;
      h_[p] = h_[c];
      p = c;
    }
    h_[p] = last;
  }

 private:
  struct Ent {
    double k;
    int32_t id;
  };
  static bool less(const Ent& a, const Ent& b) { return a.k < b.k || (a.k == b.k && a.id < b.id); }
  std::vector<Ent> h_;
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
  // cell centres (cells.hpp:44-48)
  std::vector<double> ccx(J), ccy(J);
  for (int64_t c = 0; c < J; ++c) {
    const int64_t a = c % cx, b = c / cx;
    ccx[c] = 0.5 * (gx(ib[a]) + gx(ie[a] - 1));
    ccy[c] = 0.5 * (gy(jb[b]) + gy(je[b] - 1));
  }
  const double* Fc = cells->center_speed;

  // coarse exits (fmsm.cpp:37-81)
  std::vector<double> best(J, kInf);
  if (p->n_exit_points > 0) {
    const bool single = p->n_exit_points == 1;
    for (int64_t k = 0; k < p->n_exit_points; ++k) {
      const double qx = p->exit_points_xy[2 * k], qy = p->exit_points_xy[2 * k + 1];
      double dmin = kInf;
      for (int64_t c = 0; c < J; ++c) dmin = std::min(dmin, std::hypot(qx - ccx[c], qy - ccy[c]));
      const double tie = 1e-12 * (g.h + dmin);
      for (int64_t c = 0; c < J; ++c) {
        const double dist = std::hypot(qx - ccx[c], qy - ccy[c]);
        if (dist > dmin + tie) continue;
        const double cost = single ? p->exit_point_cost[k] : p->exit_point_cost[k] + dist / Fc[c];
        best[c] = std::min(best[c], cost);
      }
    }
  } else {
    const bool single = p->n_exit == 1;
    for (int64_t k = 0; k < p->n_exit; ++k) {
      const int64_t idx = p->exit_nodes[k], i = idx % g.m, j = idx / g.m;
      int64_t a = 0, b = 0;  // cell_of_node (cells.cpp:23-30)
      while (ie[a] <= i) ++a;
      while (je[b] <= j) ++b;
      const int64_t c = b * cx + a;
      const double dist = std::hypot(gx(i) - ccx[c], gy(j) - ccy[c]);
      const double cost = single ? p->exit_cost[k] : p->exit_cost[k] + dist / Fc[c];
      best[c] = std::min(best[c], cost);
    }
  }
  out->is_q.assign(J, 0);
  std::vector<double> v(J, kInf);
  std::vector<uint8_t> label(J, 0);  // 0 far, 1 considered, 2 accepted
  std::vector<uint8_t> isx(J, 0);
  int64_t nq = 0;
  for (int64_t c = 0; c < J; ++c)
    if (std::isfinite(best[c])) {
      out->is_q[c] = 1;
      isx[c] = 1;
      v[c] = best[c];
      label[c] = 2;
      ++nq;
    }
  if (nq == 0) return 1;

  // coarse Fast March (classic_solvers.cpp:28-92) on the cx x cy lattice,
  // spacing hc_x, speed = F at the actual cell centres
  out->coarse_updates = 0;
  out->coarse_pops = 0;
  Heap H;
  const int di[4] = {1, -1, 0, 0}, dj[4] = {0, 0, 1, -1};
  std::vector<double> cc(J);  // h_c / F per cell, as quadrant_update computes it
  for (int64_t c = 0; c < J; ++c) cc[c] = hc_x / Fc[c];
  auto update = [&](int64_t a, int64_t b) {
    ++out->coarse_updates;
    const double E = a + 1 < cx ? v[b * cx + a + 1] : kInf;
    const double W = a - 1 >= 0 ? v[b * cx + a - 1] : kInf;
    const double N = b + 1 < cy ? v[(b + 1) * cx + a] : kInf;
    const double S = b - 1 >= 0 ? v[(b - 1) * cx + a] : kInf;
    return quadrant_c(std::min(E, W), std::min(N, S), cc[b * cx + a]);
  };
  for (int64_t c = 0; c < J; ++c) {
    if (!isx[c]) continue;
    const int64_t a = c % cx, b = c / cx;
    for (int d = 0; d < 4; ++d) {
      const int64_t na = a + di[d], nb = b + dj[d];
      if (na < 0 || na >= cx || nb < 0 || nb >= cy) continue;
      const int64_t nc = nb * cx + na;
      if (label[nc] != 0) continue;
      label[nc] = 1;
      const double cand = update(na, nb);
      if (cand < v[nc]) v[nc] = cand;
      H.push((int32_t)nc, v[nc]);
    }
  }
  while (!H.empty()) {
    double key;
    int32_t top;
    H.pop(key, top);
    const int64_t c = top;
    if (label[c] == 2 || key != v[c]) continue;  // superseded entry
    ++out->coarse_pops;
    label[c] = 2;
    const int64_t a = c % cx, b = c / cx;
    for (int d = 0; d < 4; ++d) {
      const int64_t na = a + di[d], nb = b + dj[d];
      if (na < 0 || na >= cx || nb < 0 || nb >= cy) continue;
      const int64_t nc = nb * cx + na;
      if (label[nc] == 2 || isx[nc]) continue;
      const double cand = update(na, nb);
      if (label[nc] == 0) {
        label[nc] = 1;
        if (cand < v[nc]) v[nc] = cand;
        H.push((int32_t)nc, v[nc]);
      } else if (cand < v[nc]) {
        v[nc] = cand;
        H.push((int32_t)nc, cand);
      }
    }
  }

  // quantised acceptance order (fmsm.cpp:138-160)
  double vmax = hc_x;
  for (int64_t c = 0; c < J; ++c)
    if (std::isfinite(v[c])) vmax = std::max(vmax, v[c]);
  const double quantum = 1e-9 * vmax;
  // (key, id) packed into one word: keys are floor(v / (1e-9 vmax)) <= 1e9 <
  // 2^31 (an unreached cell sorts last), ids < 2^31 -- a radix sort of the
  // words is the reference's stable sort by key then id
  std::vector<uint64_t> kw(J);
  for (int64_t c = 0; c < J; ++c) {
    const uint64_t key = std::isfinite(v[c]) ? (uint64_t)std::floor(v[c] / quantum) : 0xFFFFFFFFull;
    kw[c] = (key << 32) | (uint64_t)c;
  }
  radix_sort_u64(kw);
  out->order.resize(J);
  for (int64_t r = 0; r < J; ++r) out->order[r] = (int32_t)(kw[r] & 0xFFFFFFFFull);
  out->rank.resize(J);
  for (int64_t r = 0; r < J; ++r) out->rank[out->order[r]] = (int32_t)r;
  return 0;
}

}  // namespace eikb200
