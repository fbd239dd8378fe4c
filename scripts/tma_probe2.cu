// TMA probe 2: the FMSM kernel's pattern -- several warps per CTA, each with
// its own tile and mbarrier, lane 0 issuing two 2-D loads per cell in a loop,
// cooperative launch over many CTAs.  Development aid.
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
struct Args { const CUtensorMap* tm; double* out; int tile; int iters; int cols; int variant; int two; };
__global__ void k(Args a) {
  extern __shared__ __align__(128) double sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* U = sm + (size_t)wib * a.tile;
  double* Cc = U + a.tile / 2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)(blockDim.x >> 5) * a.tile) + wib;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned phase = 0;
  double acc = 0;
  for (int it = 0; it < a.iters; ++it) {
    const int cell = (blockIdx.x * (blockDim.x >> 5) + wib) * a.iters + it;
    const int x = (a.variant & 4 ? 64 : 63) + (cell % 200) * 8, y = (cell / 200) % 250 * 8;
    if (lane == 0) {
      if (a.variant & 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (a.variant & 2) asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"((a.two ? 2 : 1) * 12 * 11 * 8) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su(U)), "l"(a.tm), "r"(x), "r"(y), "r"(su(bar)) : "memory");
      if (a.two)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su(Cc)), "l"(a.tm + 1), "r"(x), "r"(y), "r"(su(bar)) : "memory");
    }
    unsigned ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(su(bar)), "r"(phase) : "memory");
    phase ^= 1u;
    acc += U[lane] + Cc[lane];
    U[lane] = 0;  // generic writes into the tile before the next load
    __syncwarp();
  }
  if (lane == 0) a.out[blockIdx.x * (blockDim.x >> 5) + wib] = acc;
}
int main(int argc, char** argv) {
  const int variant = argc > 1 ? atoi(argv[1]) : 0;
  const int iters = argc > 2 ? atoi(argv[2]) : 50, warps = argc > 3 ? atoi(argv[3]) : 8;
  const int grid = argc > 4 ? atoi(argv[4]) : 100, two = argc > 5 ? atoi(argv[5]) : 1;
  const int P = 2178, R = 2051;
  double* g; cudaMalloc(&g, sizeof(double) * P * R * 2);
  cudaMemset(g, 0, sizeof(double) * P * R * 2);
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeTiledFn enc = (EncodeTiledFn)fp;
  alignas(64) CUtensorMap tm[2];
  cuuint64_t dims[2] = {(cuuint64_t)P, (cuuint64_t)R}, str[1] = {(cuuint64_t)P * 8};
  cuuint32_t box[2] = {12, 11}, es[2] = {1, 1};
  for (int t = 0; t < 2; ++t)
    enc(&tm[t], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g + (size_t)t * P * R, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap* dtm; cudaMalloc(&dtm, sizeof(tm)); cudaMemcpy(dtm, tm, sizeof(tm), cudaMemcpyHostToDevice);
  Args a; a.tm = dtm; cudaMalloc(&a.out, 8 * 4096); a.tile = 2 * 144; a.iters = iters; a.two = two; a.cols = P; a.variant = variant;
  size_t smem = (size_t)warps * a.tile * 8 + 8 * warps;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  void* args[] = {&a};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(32 * warps), args, smem, 0);
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("variant %d iters %d warps %d grid %d two %d: launch %s sync %s\n", variant, iters, warps, grid, two, cudaGetErrorString(e), cudaGetErrorString(e2));
  return 0;
}
