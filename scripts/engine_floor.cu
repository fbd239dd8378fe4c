// The in-cell wavefront's latency floor: cycles per step of a one-warp
// skewed pipeline that does only what every engine must (the upwind shuffle,
// the node update, the compare/select), against the production locking
// engine (k_cellsweep.cuh) on the same cell.  Development aid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 \
//        -I paper_1110_6220_b200/csrc -I include scripts/engine_floor.cu -o /tmp/ef
#include <cstdio>

#include "k_cellsweep.cuh"

using namespace eikb200;

// VAR 0: shuffle + node_update4 + select (IEEE sqrt); 1: the same with the
// sqrt replaced by a multiply; 2: shuffle + select only
template <int VAR>
__global__ void floor_kernel(int steps, int reps, long long* out, double* sink) {
  const int lane = threadIdx.x;
  double wv = 1.0 + lane * 1e-3, e = 2.0, n = 2.5, c = 0.01 + lane * 1e-5, cur = 3.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r)
    for (int s = 0; s < steps; ++s) {
      double sv = __shfl_sync(kFull, wv, (lane + 31) & 31);
      double cand;
      if (VAR == 0) {
        cand = node_update4(e, wv, n, sv, c);
      } else if (VAR == 1) {
        const double ua = dmin(e, wv), ub = dmin(n, sv);
        const double diff = ua - ub;
        const bool two = (ua < kInf) && (ub < kInf) && (fabs(diff) <= c);
        const double arg = two ? (2.0 * c * c - diff * diff) : 1.0;
        const double ts = 0.5 * (ua + ub) + 0.5 * (arg * 1.0000001);
        cand = two ? ts : c + dmin(ua, ub);
      } else {
        cand = sv + c;
      }
      const bool dec = cand < cur;
      wv = dec ? cand : wv * 0.999;
      e = e * 1.0000001;
    }
  long long t1 = clock64();
  if (lane == 0) {
    out[0] = t1 - t0;
    *sink = wv;
  }
}

__global__ void lock_kernel(int w, int h, int reps, long long* out, double* sink) {
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
    cell_sweep_lock<false, 1>(T, r & 3, lane, upd);
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
  long long* d;
  double* s;
  cudaMalloc(&d, 8);
  cudaMalloc(&s, 8);
  long long c[3];
  const int steps = 64, reps = 200;
  floor_kernel<0><<<1, 32>>>(steps, reps, d, s);
  cudaMemcpy(&c[0], d, 8, cudaMemcpyDeviceToHost);
  floor_kernel<1><<<1, 32>>>(steps, reps, d, s);
  cudaMemcpy(&c[1], d, 8, cudaMemcpyDeviceToHost);
  floor_kernel<2><<<1, 32>>>(steps, reps, d, s);
  cudaMemcpy(&c[2], d, 8, cudaMemcpyDeviceToHost);
  printf("floor cycles/step: shfl+update+select %.0f, without sqrt %.0f, shfl+select %.0f\n",
         c[0] / (double)(steps * reps), c[1] / (double)(steps * reps),
         c[2] / (double)(steps * reps));
  for (int w : {8, 16, 32}) {
    const int h = w, pu = (w + 3) & ~1;
    const size_t smem = 2 * (h + 2) * pu * 8 + w * h + 16;
    cudaFuncSetAttribute(lock_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    lock_kernel<<<1, 32, smem>>>(w, h, reps, d, s);
    long long cy;
    cudaMemcpy(&cy, d, 8, cudaMemcpyDeviceToHost);
    printf("locking engine %dx%d: %.0f cycles/step (%s)\n", w, h, cy / (double)(reps * (w + h - 1)),
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
