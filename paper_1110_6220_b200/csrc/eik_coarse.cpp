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

double quadrant(double ua, double ub, double f, double h) {  // local_update.hpp:30-43
  const double c = h / f;
  if (std::isfinite(ua) && std::isfinite(ub)) {
    const double diff = ua - ub;
    if (std::abs(diff) <= c) return 0.5 * (ua + ub) + 0.5 * std::sqrt(2.0 * c * c - diff * diff);
  }
  return c + std::min(ua, ub);
}

// Binary min-heap keyed by (value, id) with decrease-key, ties to the
// smaller id (indexed_min_heap.hpp:66-69).
class Heap {
 public:
  explicit Heap(int64_t cap) : key_(cap), pos_(cap, -1) { h_.reserve(cap); }
  bool empty() const { return h_.empty(); }
  bool contains(int64_t id) const { return pos_[id] >= 0; }
  void insert(int64_t id, double k) {
    key_[id] = k;
    pos_[id] = (int64_t)h_.size();
    h_.push_back(id);
    up(pos_[id]);
  }
  void decrease(int64_t id, double k) {
    key_[id] = k;
    up(pos_[id]);
  }
  int64_t pop() {
    int64_t top = h_[0], last = h_.back();
    h_.pop_back();
    pos_[top] = -1;
    if (!h_.empty()) {
      h_[0] = last;
      pos_[last] = 0;
      down(0);
    }
    return top;
  }

 private:
  bool less(int64_t a, int64_t b) const {
    if (key_[a] != key_[b]) return key_[a] < key_[b];
    return a < b;
  }
  void up(int64_t p) {
    int64_t id = h_[p];
    while (p > 0) {
      int64_t par = (p - 1) / 2;
      if (!less(id, h_[par])) break;
      h_[p] = h_[par];
      pos_[h_[p]] = p;
      p = par;
    }
    h_[p] = id;
    pos_[id] = p;
  }
  void down(int64_t p) {
    int64_t id = h_[p];
    const int64_t n = (int64_t)h_.size();
    for (;;) {
      int64_t c = 2 * p + 1;
      if (c >= n) break;
      if (c + 1 < n && less(h_[c + 1], h_[c])) ++c;
      if (!less(h_[c], id)) break;
      h_[p] = h_[c];
      pos_[h_[p]] = p;
      p = c;
    }
    h_[p] = id;
    pos_[id] = p;
  }
  std::vector<double> key_;
  std::vector<int64_t> pos_;
  std::vector<int64_t> h_;
};

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
  Heap H(J);
  const int di[4] = {1, -1, 0, 0}, dj[4] = {0, 0, 1, -1};
  auto update = [&](int64_t a, int64_t b) {
    ++out->coarse_updates;
    const double E = a + 1 < cx ? v[b * cx + a + 1] : kInf;
    const double W = a - 1 >= 0 ? v[b * cx + a - 1] : kInf;
    const double N = b + 1 < cy ? v[(b + 1) * cx + a] : kInf;
    const double S = b - 1 >= 0 ? v[(b - 1) * cx + a] : kInf;
    return quadrant(std::min(E, W), std::min(N, S), Fc[b * cx + a], hc_x);
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
      H.insert(nc, v[nc]);
    }
  }
  while (!H.empty()) {
    const int64_t c = H.pop();
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
        H.insert(nc, v[nc]);
      } else if (cand < v[nc]) {
        v[nc] = cand;
        H.decrease(nc, cand);
      }
    }
  }

  // quantised acceptance order (fmsm.cpp:138-160)
  double vmax = hc_x;
  for (int64_t c = 0; c < J; ++c)
    if (std::isfinite(v[c])) vmax = std::max(vmax, v[c]);
  const double quantum = 1e-9 * vmax;
  std::vector<long long> key(J);
  for (int64_t c = 0; c < J; ++c)
    key[c] = std::isfinite(v[c]) ? (long long)std::floor(v[c] / quantum)
                                 : std::numeric_limits<long long>::max();
  out->order.resize(J);
  for (int64_t c = 0; c < J; ++c) out->order[c] = (int32_t)c;
  std::sort(out->order.begin(), out->order.end(), [&](int32_t a, int32_t b) {
    if (key[a] != key[b]) return key[a] < key[b];
    return a < b;
  });
  out->rank.resize(J);
  for (int64_t r = 0; r < J; ++r) out->rank[out->order[r]] = (int32_t)r;
  return 0;
}

}  // namespace eikb200
