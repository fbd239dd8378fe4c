// Internal interface between the host runtime (eik_abi.cpp) and the kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace eikb200 {

struct FsmArgs {
  const double* C;          // h/F per node, -1 for exits
  double* u;                // value field
  int64_t m, n;
  int nstrips;              // ceil(n / 32)
  unsigned long long* prog; // [nstrips] progress of each strip's last row
  int* changed;             // [max_sweeps] change flag per sweep
  int* done;                // [max_sweeps] strips finished per sweep
  int max_sweeps;
  int lookahead;            // D: stop decision for sweep k uses sweep k-D
  int* status;              // [0] error, [1] sweeps
};

cudaError_t launch_prepare(const double* F, double* C, double* u, int64_t M, double h,
                           const int64_t* exits, const double* cost, int64_t n_exit,
                           int* status, cudaStream_t s, int* launches);
cudaError_t launch_fsm(const FsmArgs& a, cudaStream_t s, int* launches);

}  // namespace eikb200
