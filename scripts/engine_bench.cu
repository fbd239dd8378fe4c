// Microbenchmark of the in-cell sweep engine (k_cellsweep.cuh): cycles per
// wavefront step for each mode on a synthetic cell.  Development aid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 \
//        -I paper_1110_6220_b200/csrc -I include scripts/engine_bench.cu -o build/engine_bench
#include <cstdio>
#include <vector>

#include "k_cellsweep.cuh"

using namespace eikb200;

template <int MODE>
__global__ void bench(int w, int h, int reps, long long* out, double* sink) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x;
  const int pu = (w + 3) & ~1;
  CellTile T;
  T.pu = pu;
  T.ox = 1;
  T.U = sm;
  T.Ct = sm + (h + 2) * pu;
  T.lock = reinterpret_cast<uint8_t*>(T.Ct + (h + 2) * pu);
  T.w = w;
  T.h = h;
  for (int k = lane; k < (h + 2) * pu; k += 32) {
    T.U[k] = 1e300;
    T.Ct[k] = 0.01 + 0.001 * (k % 7);
  }
  for (int k = lane; k < w * h; k += 32) T.lock[k] = 1;
  __syncwarp();
  if (lane == 0) T.U[pu + 1] = 0.0;
  __syncwarp();
  long long upd = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (MODE == 3) cell_sweep_ns<2, 1>(T, r & 3, lane, upd);  // the generic locked engine
    else if (MODE == 4) cell_sweep_lock<true, 1>(T, r & 3, lane, upd);  // with the vote skip
    else cell_sweep<MODE>(T, r & 3, lane, upd);
    if (MODE >= 2)
      for (int k = lane; k < w * h; k += 32) T.lock[k] = 1;
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) {
    out[0] = t1 - t0;
    *sink = T.U[pu * 3 + 3] + (double)upd;
  }
}

int main() {
  long long* d_out;
  double* d_sink;
  cudaMalloc(&d_out, 8);
  cudaMalloc(&d_sink, 8);
  const int sizes[][2] = {{16, 16}, {8, 8}, {32, 32}, {33, 33}, {64, 64}};
  for (auto& sz : sizes) {
    const int w = sz[0], h = sz[1], reps = 200;
    const int pu = (w + 3) & ~1;
    const size_t smem = 2 * (h + 2) * pu * 8 + w * h + 16;
    long long cyc[5];
    cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(bench<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(bench<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bench<0><<<1, 32, smem>>>(w, h, reps, d_out, d_sink);
    cudaMemcpy(&cyc[0], d_out, 8, cudaMemcpyDeviceToHost);
    bench<1><<<1, 32, smem>>>(w, h, reps, d_out, d_sink);
    cudaMemcpy(&cyc[1], d_out, 8, cudaMemcpyDeviceToHost);
    bench<2><<<1, 32, smem>>>(w, h, reps, d_out, d_sink);
    cudaMemcpy(&cyc[2], d_out, 8, cudaMemcpyDeviceToHost);
    bench<3><<<1, 32, smem>>>(w, h, reps, d_out, d_sink);
    cudaMemcpy(&cyc[3], d_out, 8, cudaMemcpyDeviceToHost);
    bench<4><<<1, 32, smem>>>(w, h, reps, d_out, d_sink);
    cudaMemcpy(&cyc[4], d_out, 8, cudaMemcpyDeviceToHost);
    const double steps = (double)reps * (w + h - 1);
    printf("cell %dx%d: cycles/step full %.0f directional %.0f locked %.0f (vote-skip %.0f, generic "
           "%.0f)  (%s)\n",
           w, h, cyc[0] / steps, cyc[1] / steps, cyc[2] / steps, cyc[4] / steps, cyc[3] / steps,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
