// Dependent-chain latencies of the primitives on the in-cell critical path
// (B200 sm_100a).  Development aid: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -fmad=false scripts/latency_bench.cu -o /tmp/lb
#include <cstdio>

__global__ void lat(double seed, int n, long long* out, double* sink) {
  double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0, t1;
  // DADD
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  t1 = clock64();
  out[0] = t1 - t0;
  // DMUL
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  t1 = clock64();
  out[1] = t1 - t0;
  // DFMA
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-300);
  t1 = clock64();
  out[2] = t1 - t0;
  // sqrt (correctly rounded)
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 1.0;
  t1 = clock64();
  out[3] = t1 - t0;
  // shuffle of a double
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 31) & 31) + 1.0;
  t1 = clock64();
  out[4] = t1 - t0;
  // compare+select (min)
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = (y < x) ? y * 0.999 : x + 1.0;
  t1 = clock64();
  out[5] = t1 - t0;
  if (threadIdx.x == 0) *sink = x;
}

int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 64);
  cudaMalloc(&s, 8);
  const int n = 4096;
  lat<<<1, 32>>>(2.0, n, d, s);
  long long h[6];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[6] = {"DADD", "DMUL", "DFMA", "sqrt+DADD", "SHFL(f64)+DADD", "DSETP/FSEL+op"};
  for (int k = 0; k < 6; ++k) printf("%-16s %.1f cycles per dependent op\n", nm[k], (double)h[k] / n);
  return 0;
}
