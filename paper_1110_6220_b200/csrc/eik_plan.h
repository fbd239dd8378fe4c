// Resident solve plan: device buffers and stream owned by one eik_plan.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "eikonal_b200.h"

struct eik_plan {
  int method = 0;
  eik_grid g{};
  int64_t M = 0;
  int64_t n_exit = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<void*> allocs;
  double* dF = nullptr;   // speed (resident input)
  double* dC = nullptr;   // h/F, -1 at exits
  double* dU = nullptr;   // value field
  int64_t* dExit = nullptr;
  double* dExitCost = nullptr;
  int* dStatus = nullptr;
  int64_t h2d_bytes = 0;
  int64_t pitch = 0;       // padded row pitch of dC / dU (m + 2*kPad)
  // FSM wavefront state
  int nstrips = 0;
  int max_sweeps = 0;
  int64_t last_sweeps_bound = 1 << 16;
  unsigned long long* dProg = nullptr;
  double* dMbox = nullptr;
  unsigned long long* dTrace = nullptr;
  int* dChanged = nullptr;
  int* dDone = nullptr;
};
