// Microbenchmark of the committer queue's warp argmin (k_heapcell.cu
// BucketPQ::rescan / pop_min): cycles per (key, id) argmin over 32 lanes for
// the shuffle tree and for a redux.sync formulation.  Development aid:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/pq_bench.cu -o build/pq_bench
#include <cstdio>
#include <cstdint>

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ bool less(double ka, int ia, double kb, int ib) {
  return ka < kb || (ka == kb && ia < ib);
}

// shuffle tree (as BucketPQ)
__device__ __forceinline__ int argmin_shfl(double k, int id, int lane, double& kout) {
  int wl = lane;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ko = __shfl_xor_sync(kFull, k, o);
    const int io = __shfl_xor_sync(kFull, id, o);
    const int wo = __shfl_xor_sync(kFull, wl, o);
    if (less(ko, io, k, id)) {
      k = ko;
      id = io;
      wl = wo;
    }
  }
  kout = k;
  return wl;
}

// redux.sync on the key's bit pattern (non-negative doubles order like their
// bits), ties broken by id
__device__ __forceinline__ int argmin_redux(double k, int id, int lane, double& kout) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(k);
  const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
  const unsigned mhi = __reduce_min_sync(kFull, hi);
  const unsigned m1 = __ballot_sync(kFull, hi == mhi);
  unsigned mlo = 0xffffffffu;
  if (hi == mhi) mlo = __reduce_min_sync(m1, lo);
  mlo = __shfl_sync(kFull, mlo, __ffs(m1) - 1);
  const unsigned m2 = __ballot_sync(kFull, hi == mhi && lo == mlo);
  int w = __ffs(m2) - 1;
  if (__popc(m2) > 1) {
    unsigned mid = 0xffffffffu;
    if ((m2 >> lane) & 1u) mid = __reduce_min_sync(m2, (unsigned)id);
    mid = __shfl_sync(kFull, mid, w);
    w = __ffs(__ballot_sync(kFull, ((m2 >> lane) & 1u) && (unsigned)id == mid)) - 1;
  }
  kout = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
  return w;
}

template <int V>
__global__ void bench(const double* keys, const int* ids, int reps, long long* out, int* sink) {
  const int lane = threadIdx.x;
  double k = keys[lane];
  int id = ids[lane];
  int acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double ko;
    const int w = V == 0 ? argmin_shfl(k, id, lane, ko) : argmin_redux(k, id, lane, ko);
    acc += w;
    // dependent next round: perturb the winner's key
    if (lane == w) k = k + 1.0;
  }
  long long t1 = clock64();
  if (lane == 0) {
    out[V] = t1 - t0;
    sink[V] = acc;
  }
}

int main() {
  double hk[32];
  int hi[32];
  for (int i = 0; i < 32; ++i) {
    hk[i] = 100.0 + ((i * 37) % 32) * 0.25 + (i % 5 == 0 ? 0.0 : 0.001 * i);
    hi[i] = 1000 + (i * 13) % 32;
  }
  hk[7] = hk[9];  // a tie
  double* dk;
  int *di, *ds;
  long long* dout;
  cudaMalloc(&dk, sizeof(hk));
  cudaMalloc(&di, sizeof(hi));
  cudaMalloc(&ds, 16);
  cudaMalloc(&dout, 16);
  cudaMemcpy(dk, hk, sizeof(hk), cudaMemcpyHostToDevice);
  cudaMemcpy(di, hi, sizeof(hi), cudaMemcpyHostToDevice);
  const int reps = 10000;
  bench<0><<<1, 32>>>(dk, di, reps, dout, ds);
  bench<1><<<1, 32>>>(dk, di, reps, dout, ds);
  long long c[2];
  int s[2];
  cudaMemcpy(c, dout, 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(s, ds, 8, cudaMemcpyDeviceToHost);
  printf("argmin cycles: shuffle tree %.1f, redux %.1f (checksums %d %d, %s)\n",
         (double)c[0] / reps, (double)c[1] / reps, s[0], s[1],
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
