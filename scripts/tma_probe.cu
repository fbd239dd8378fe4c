// Minimal TMA (cp.async.bulk.tensor 2-D, fp64) probe: normal vs cooperative
// launch, tensor map in global memory vs __grid_constant__.  Development aid.
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

template <int VARIANT>
__global__ void k(const CUtensorMap* tm, const __grid_constant__ CUtensorMap tmp, double* out, int x, int y) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 1024);
  const CUtensorMap* t = VARIANT & 1 ? &tmp : tm;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (VARIANT & 2) asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(12 * 11 * 8) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su(sm)), "l"(t), "r"(x), "r"(y), "r"(su(bar)) : "memory");
  }
  unsigned ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(su(bar)), "r"(0u) : "memory");
  if (threadIdx.x < 132) out[threadIdx.x] = sm[threadIdx.x];
}

int main(int argc, char** argv) {
  const int sel = argc > 1 ? atoi(argv[1]) : 0;
  const int P = 2178, R = 2051;
  double* g; cudaMalloc(&g, sizeof(double) * P * R);
  double* h = new double[(size_t)P * R];
  for (size_t i = 0; i < (size_t)P * R; ++i) h[i] = (double)i;
  cudaMemcpy(g, h, sizeof(double) * P * R, cudaMemcpyHostToDevice);
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeTiledFn enc = (EncodeTiledFn)fp;
  alignas(64) CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)P, (cuuint64_t)R}, str[1] = {(cuuint64_t)P * 8};
  cuuint32_t box[2] = {12, 11}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d fp %p q %d\n", (int)r, fp, (int)q);
  CUtensorMap* dtm; cudaMalloc(&dtm, sizeof(tm)); cudaMemcpy(dtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
  double* out; cudaMalloc(&out, 8 * 256);
  int x = 100, y = 7;
  auto run = [&](auto kern, const char* name, bool coop) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    cudaError_t e;
    if (coop) {
      void* args[] = {&dtm, &tm, &out, &x, &y};
      e = cudaLaunchCooperativeKernel((const void*)kern, dim3(1), dim3(128), args, 16384, 0);
    } else {
      kern<<<1, 128, 16384>>>(dtm, tm, out, x, y);
      e = cudaGetLastError();
    }
    cudaError_t e2 = cudaDeviceSynchronize();
    double o[2] = {0, 0};
    cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
    printf("%-28s coop %d launch %s sync %s out0 %.0f (want %d)\n", name, coop, cudaGetErrorString(e), cudaGetErrorString(e2), o[0], y * P + x);
  };
  switch (sel) {
    case 0: run(k<0>, "global map", false); break;
    case 1: run(k<1>, "grid_constant map", false); break;
    case 2: run(k<2>, "global map + proxy fence", false); break;
    case 3: run(k<0>, "global map", true); break;
    default: run(k<2>, "global map + proxy fence", true); break;
  }
  return 0;
}
