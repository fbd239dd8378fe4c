// Error metrics against a ground truth on the device (SURVEY.md section 8(f)
// row 2): error_fields + error_ratios of /root/reference/proj/src/metrics.cpp
// (:11-69) as one reduction pass.
//
//   e = |v_exact - v_truth|, E = |v_method - v_truth|          (metrics.cpp:27-28)
//   X+ = { non-exit nodes with e > 1e-14 }                     (:29)
//   l_inf = max E, l_1 = mean E over non-exit nodes             (:44-45, :60-61)
//   max / mean of E/e over X+, ratio_of_max = max E|X+ / max e|X+ (:46-66)
//
// Maxima and counts are order-independent, so they equal the reference's
// bit for bit given the same fields; the two sums (l_1, the mean ratio) are
// accumulated per thread, reduced per block in a fixed tree and the block
// partials summed in block order on the host: deterministic, and within a few
// ulps of the reference's sequential sums.
#include <algorithm>
#include <vector>

#include "eik_internal.h"
#include "k_common.cuh"

namespace eikb200 {

namespace {

constexpr int kThreads = 256;

struct Partial {
  double max_E, sum_E, max_ratio, sum_ratio, max_E_plus, max_e_plus;
  unsigned long long non_exit, m_plus;
};

__device__ __forceinline__ double dmax(double a, double b) { return b > a ? b : a; }

__global__ void metrics_kernel(const double* __restrict__ vm, const double* __restrict__ ve,
                               const double* __restrict__ vt, const uint8_t* __restrict__ is_exit,
                               int64_t M, Partial* __restrict__ out) {
  Partial p{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0ull, 0ull};
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < M;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (is_exit[k]) continue;
    const double e = fabs(ve[k] - vt[k]);
    const double E = fabs(vm[k] - vt[k]);
    ++p.non_exit;
    p.max_E = dmax(p.max_E, E);
    p.sum_E += E;
    if (!(e > 1e-14)) continue;
    ++p.m_plus;
    const double ratio = E / e;
    p.max_ratio = dmax(p.max_ratio, ratio);
    p.sum_ratio += ratio;
    p.max_E_plus = dmax(p.max_E_plus, E);
    p.max_e_plus = dmax(p.max_e_plus, e);
  }
  __shared__ Partial sh[kThreads];
  sh[threadIdx.x] = p;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      Partial& a = sh[threadIdx.x];
      const Partial& b = sh[threadIdx.x + s];
      a.max_E = dmax(a.max_E, b.max_E);
      a.sum_E += b.sum_E;
      a.max_ratio = dmax(a.max_ratio, b.max_ratio);
      a.sum_ratio += b.sum_ratio;
      a.max_E_plus = dmax(a.max_E_plus, b.max_E_plus);
      a.max_e_plus = dmax(a.max_e_plus, b.max_e_plus);
      a.non_exit += b.non_exit;
      a.m_plus += b.m_plus;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = sh[0];
}

__global__ void mark_kernel(uint8_t* is_exit, const int64_t* exits, int64_t n, int64_t M) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    if (exits[k] >= 0 && exits[k] < M) is_exit[exits[k]] = 1;
}

}  // namespace

// u_* are device pointers (m*n, dense); exits a device pointer.  Fills
// res[0..4] = l_inf, l_1, max_error_ratio, avg_error_ratio, ratio_of_max and
// counts[0..1] = m_plus, x_plus_empty.
cudaError_t device_metrics(const double* vm, const double* ve, const double* vt, int64_t M,
                           const int64_t* exits, int64_t n_exit, uint8_t* mask, cudaStream_t s,
                           double res[5], long long counts[2]) {
  cudaError_t e = cudaMemsetAsync(mask, 0, (size_t)M, s);
  if (e != cudaSuccess) return e;
  if (n_exit > 0) mark_kernel<<<(int)std::min<int64_t>((n_exit + 255) / 256, 1024), 256, 0, s>>>(
      mask, exits, n_exit, M);
  const int blocks = (int)std::min<int64_t>((M + kThreads - 1) / kThreads, 148 * 8);
  Partial* dpart = nullptr;
  e = cudaMallocAsync(reinterpret_cast<void**>(&dpart), sizeof(Partial) * blocks, s);
  if (e != cudaSuccess) return e;
  metrics_kernel<<<blocks, kThreads, 0, s>>>(vm, ve, vt, mask, M, dpart);
  std::vector<Partial> hp((size_t)blocks);
  e = cudaMemcpyAsync(hp.data(), dpart, sizeof(Partial) * blocks, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(dpart, s);
  if (e != cudaSuccess) return e;
  Partial t{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0ull, 0ull};
  for (const Partial& b : hp) {  // block order: deterministic
    t.max_E = std::max(t.max_E, b.max_E);
    t.sum_E += b.sum_E;
    t.max_ratio = std::max(t.max_ratio, b.max_ratio);
    t.sum_ratio += b.sum_ratio;
    t.max_E_plus = std::max(t.max_E_plus, b.max_E_plus);
    t.max_e_plus = std::max(t.max_e_plus, b.max_e_plus);
    t.non_exit += b.non_exit;
    t.m_plus += b.m_plus;
  }
  res[0] = t.max_E;                                              // metrics.cpp:60
  res[1] = t.non_exit > 0 ? t.sum_E / (double)t.non_exit : 0.0;  // :61
  if (t.m_plus == 0) {                                           // :62-64
    res[2] = res[3] = res[4] = 1.0;
  } else {
    res[2] = t.max_ratio;
    res[3] = t.sum_ratio / (double)t.m_plus;
    res[4] = t.max_E_plus / t.max_e_plus;
  }
  counts[0] = (long long)t.m_plus;
  counts[1] = t.m_plus == 0 ? 1 : 0;
  return cudaSuccess;
}

}  // namespace eikb200
