// Micro-test: 2D TMA tiled loads with the relocation kernel's box shapes.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../../paper_2003_02200_b200/csrc/sks_ptx.cuh"
using namespace sks;
__device__ __forceinline__ void tma_load_2d(float* dst, const CUtensorMap* tm, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}
__global__ void k2(const __grid_constant__ CUtensorMap a, const __grid_constant__ CUtensorMap b, int which, int x, int y, float* out) {
  __shared__ __align__(128) float buf[2048];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_expect_tx(&bar, 8192); tma_load_2d(buf, which ? &b : &a, x, y, &bar); }
  __syncthreads();
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) out[i] = buf[i];
}
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  int rows = 200, cols = 160;
  float* d; cudaMalloc(&d, rows * cols * 4);
  float* h = new float[rows * cols]; for (int i = 0; i < rows * cols; ++i) h[i] = i;
  cudaMemcpy(d, h, rows * cols * 4, cudaMemcpyHostToDevice);
  float* o; cudaMalloc(&o, 8192);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiled fn = (EncodeTiled)p;
  CUtensorMap A, B;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, str[1] = {(cuuint64_t)cols * 4};
  cuuint32_t ba[2] = {64, 32}, bb[2] = {32, 64}, e[2] = {1, 1};
  printf("encA %d\n", fn(&A, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, ba, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  printf("encB %d\n", fn(&B, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, bb, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  int t[3] = {atoi(argv[1]), atoi(argv[2]), atoi(argv[3])};
  k2<<<1, 128>>>(A, B, t[0], t[1], t[2], o);
  cudaError_t err = cudaDeviceSynchronize();
  float r[4]; cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
  printf("which %d x %d y %d -> %s  first %g %g\n", t[0], t[1], t[2], cudaGetErrorString(err), r[0], r[1]);
  return 0;
}
