// Dependent-load latency seen by one warp (the heap-cell committer's access
// pattern): pointer chasing through a 128 KB index array with ld.relaxed.gpu
// and ld.global.cg, alone and while the other CTAs stream a large buffer
// through L2 (the slot traffic of the workers) or poll a hot word.
// Development aid:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/mem_latency.cu -o /tmp/ml
#include <cstdio>

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void probe(const unsigned* chain, int n, int mode, double* big, size_t big_n,
                      volatile int* stop, unsigned* hot, long long* out, unsigned* sink,
                      int nst) {
  if (blockIdx.x == 0) {
    if (threadIdx.x != 0) return;
    unsigned idx = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) idx = ld_relaxed(chain + idx);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) idx = __ldcg(chain + idx);
    long long t2 = clock64();
    // nst relaxed stores to scattered words before every dependent load
    for (int i = 0; i < n; ++i) {
      for (int k = 0; k < nst; ++k) st_relaxed(sink + ((idx * 97u + k * 4099u) & 32767u), k);
      idx = ld_relaxed(chain + idx);
    }
    long long t3 = clock64();
    // the same with weak stores
    for (int i = 0; i < n; ++i) {
      for (int k = 0; k < nst; ++k) sink[(idx * 97u + k * 4099u) & 32767u] = k;
      idx = ld_relaxed(chain + idx);
    }
    long long t4 = clock64();
    // weak stores, weak loads
    for (int i = 0; i < n; ++i) {
      for (int k = 0; k < nst; ++k) sink[(idx * 97u + k * 4099u) & 32767u] = k;
      idx = __ldcg(chain + idx);
    }
    long long t5 = clock64();
    out[0] = (t1 - t0) / n;
    out[1] = (t2 - t1) / n;
    out[3] = (t3 - t2) / n;
    out[4] = (t4 - t3) / n;
    out[5] = (t5 - t4) / n;
    out[2] = idx;
    *stop = 1;
    return;
  }
  // background traffic until the probe is done
  size_t i = (size_t)(blockIdx.x - 1) * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)(gridDim.x - 1) * blockDim.x;
  double acc = 0.0;
  while (!*stop) {
    if (mode == 1) {  // stream reads + writes through L2
      for (int r = 0; r < 64; ++r) {
        big[i] = acc + 1.0;
        acc += __ldcg(big + ((i + big_n / 2) % big_n));
        i += stride;
        if (i >= big_n) i -= big_n;
      }
    } else if (mode == 2) {  // poll a hot word
      acc += ld_relaxed(hot + (threadIdx.x & 7));
      __nanosleep(200);
    } else {
      __nanosleep(1000);
    }
  }
  if (acc == -1.0) big[0] = acc;
}

int main2();
int main() {
  main2();
  const int n = 32768;  // 128 KB of indices
  unsigned* h = new unsigned[n];
  // random cyclic permutation (Sattolo)
  for (int i = 0; i < n; ++i) h[i] = i;
  unsigned s = 12345;
  for (int i = n - 1; i > 0; --i) {
    s = s * 1103515245u + 12345u;
    int j = s % i;
    unsigned t = h[i];
    h[i] = h[j];
    h[j] = t;
  }
  unsigned *chain, *hot;
  double* big;
  int* stop;
  long long* out;
  const size_t big_n = (size_t)256 << 20 >> 3;  // 256 MB
  cudaMalloc(&chain, n * 4);
  cudaMalloc(&hot, 64);
  cudaMalloc(&big, big_n * 8);
  cudaMalloc(&stop, 4);
  cudaMalloc(&out, 64);
  unsigned* sink;
  cudaMalloc(&sink, 32768 * 4);
  cudaMemcpy(chain, h, n * 4, cudaMemcpyHostToDevice);
  cudaMemset(big, 0, big_n * 8);
  const char* names[] = {"idle", "streaming 256MB", "polling a hot word"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(stop, 0, 4);
      probe<<<148, 256>>>(chain, 4096, mode, big, big_n, stop, hot, out, sink, 8);
      long long r[6];
      cudaMemcpy(r, out, 48, cudaMemcpyDeviceToHost);
      printf("%-20s relaxed.gpu %lld  ld.cg %lld | after 8 stores: relaxed st+ld %lld, weak st + "
             "relaxed ld %lld, weak st + ld.cg %lld cyc (%s)\n",
             names[mode], r[0], r[1], r[3], r[4], r[5], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

// Staging-shaped access: one warp loads, per "cell", 10 rows of 18 doubles
// from a pitched array (row stride 17 KB) and 10 rows of 16 doubles from a
// slot array, cells chosen at random in large (cold) arrays; cycles per cell.
__global__ void staging(const double* C, size_t Cn, const double* S, size_t Sn, int cells,
                        long long* out, double* sink) {
  const int lane = threadIdx.x;
  double acc = 0.0;
  unsigned s = 777;
  long long t0 = clock64();
  for (int c = 0; c < cells; ++c) {
    s = s * 1103515245u + 12345u;
    const size_t cbase = ((size_t)s * 4099u) % (Cn - 20 * 2177);
    const size_t sbase = (((size_t)s >> 3) * 8191u) % (Sn - 4096);
    double v[20];
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      v[i] = lane < 18 ? __ldg(C + cbase + (size_t)i * 2177 + lane) : 0.0;
      v[10 + i] = lane < 16 ? __ldcg(S + sbase + (size_t)i * 16 + lane) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 20; ++i) acc += v[i];
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0) / cells;
  if (acc == -1.0) sink[0] = acc;
}

int main2() {
  const size_t Cn = (size_t)34 << 20 >> 3 << 3, Sn = (size_t)100 << 20 >> 3 << 3;  // doubles
  double *C, *S, *sink;
  long long* out;
  cudaMalloc(&C, Cn * 8);
  cudaMalloc(&S, Sn * 8);
  cudaMalloc(&sink, 8);
  cudaMalloc(&out, 8);
  cudaMemset(C, 0, Cn * 8);
  cudaMemset(S, 0, Sn * 8);
  for (int rep = 0; rep < 3; ++rep) {
    staging<<<1, 32>>>(C, Cn, S, Sn, 2000, out, sink);
    long long r;
    cudaMemcpy(&r, out, 8, cudaMemcpyDeviceToHost);
    printf("staging-shaped group of 20 row loads: %lld cycles per cell (rep %d, %s)\n", r, rep,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
