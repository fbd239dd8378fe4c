// Host-side pieces of the two-scale methods that the reference also runs on
// the host (FMSM Part I).
#pragma once

#include <cstdint>
#include <vector>

#include "eikonal_b200.h"

namespace eikb200 {

struct FmsmOrder {
  std::vector<int32_t> order;   // cells by quantised coarse value, then id
  std::vector<int32_t> rank;    // inverse of order
  std::vector<uint8_t> is_q;    // coarse exit cells (swept to convergence)
  int64_t coarse_pops = 0;      // coarse FMM heap removals
  int64_t coarse_updates = 0;   // coarse FMM node updates
};

void split_axis(int64_t nodes, int32_t cells, std::vector<int64_t>& b, std::vector<int64_t>& e);

// build_coarse_problem + fmm_solve(coarse) + quantised sort
// (fmsm.cpp:10-162).  Returns 0, or 1 if the coarse exit set is empty.
int fmsm_part1(const eik_problem* p, const eik_cells* cells, FmsmOrder* out);

}  // namespace eikb200
