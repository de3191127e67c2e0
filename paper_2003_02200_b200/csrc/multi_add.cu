// Peer-add reduction kernel of the multi-GPU path (multi.cpp): ranks that
// share a device cannot form an NCCL communicator, so their partial maps are
// summed into the root's map with this kernel (rank order, FP64 adds).
#include <cuda_runtime.h>

namespace {

// map[i] += part[i]
__global__ void add_map_kernel(double* __restrict__ map, const double* __restrict__ part, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    map[i] = __dadd_rn(map[i], part[i]);
  }
}

}  // namespace

extern "C" cudaError_t sks_launch_add_map(double* map, const double* part, long long n, cudaStream_t stream) {
  add_map_kernel<<<1184, 256, 0, stream>>>(map, part, n);  // 8 CTAs of 256 per SM on 148 SMs
  return cudaGetLastError();
}
