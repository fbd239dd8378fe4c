// FMM acceptance order on the device (FmmOptions::record_acceptance_order,
// classic_solvers.hpp:10-13, classic_solvers.cpp:64-71).
//
// fmm_solve accepts the non-exit nodes in non-decreasing value order (the
// property its tests pin: test_classic_solvers.cpp:99-111,
// test_fmsm.cpp:117-128).  The FMM row here is the exact fixed point
// (kernel 1), so the order is recovered from the converged field: non-exit
// nodes sorted by (value, index).  Values are >= 0 (negative exit costs are
// refused at the ABI), so a double's bit pattern orders like the value and a
// stable radix sort of the 64-bit patterns keeps equal values in index order.
// Not on the timed hot path; CUB's radix sort is the library primitive.
#include <cub/device/device_radix_sort.cuh>

#include "eik_internal.h"

namespace eikb200 {

namespace {

__global__ void order_keys_kernel(const double* __restrict__ u, int64_t m, int64_t n, int64_t P,
                                  int64_t pad, const double* __restrict__ C,
                                  unsigned long long* __restrict__ keys,
                                  int32_t* __restrict__ idx) {
  const int64_t M = m * n;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < M;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = k / m, i = k - j * m;
    const int64_t p = j * P + pad + i;
    // exits (C = -1) sort last, behind every value (+inf is 0x7ff0...)
    keys[k] = C[p] < 0.0 ? ~0ull : (unsigned long long)__double_as_longlong(u[p]);
    idx[k] = (int32_t)k;
  }
}

}  // namespace

cudaError_t device_acceptance_order(const double* u, const double* C, int64_t m, int64_t n,
                                    int64_t P, int64_t pad, int32_t* order_dev,
                                    cudaStream_t s) {
  const int64_t M = m * n;
  if (M > INT32_MAX) return cudaErrorInvalidValue;
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  int32_t* i0 = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, k1, i0, order_dev,
                                                  (int)M, 0, 64, s);
  if (e != cudaSuccess) return e;
  if ((e = pool_alloc((void**)&k0, sizeof(*k0) * M)) != cudaSuccess) return e;
  if ((e = pool_alloc((void**)&k1, sizeof(*k1) * M)) == cudaSuccess &&
      (e = pool_alloc((void**)&i0, sizeof(*i0) * M)) == cudaSuccess &&
      (e = pool_alloc(&tmp, tmp_bytes)) == cudaSuccess) {
    int64_t blocks = (M + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    order_keys_kernel<<<(unsigned)blocks, 256, 0, s>>>(u, m, n, P, pad, C, k0, i0);
    e = cudaGetLastError();
    if (e == cudaSuccess)
      e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, i0, order_dev, (int)M, 0, 64,
                                          s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  pool_release(k0);
  pool_release(k1);
  pool_release(i0);
  pool_release(tmp);
  return e;
}

}  // namespace eikb200
