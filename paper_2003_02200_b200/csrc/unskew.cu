// Unskew + ordered accumulation into the device-resident total-viewshed map.
//
// Replaces unskew_accumulate (reference skew.cpp:204-263) and the engine's
// ascending-k reduction (engine.cpp:85-92, 182-205). One thread per DEM cell
// (si, sj) — coalesced read-modify-write of the FP64 map — walks the batch's
// sectors in ascending k and, for each, maps the cell into pre_ops space,
// reconstructs the two covered() flags in FP64 exactly as the reference does
// (skew.cpp:233-240), gathers skwVS = cv * (1 + tan^2) at rows p and p-1 and
// adds the interpolated value. All FP64 operations are explicit _rn
// intrinsics in the reference's order, so the per-cell sum is bit-identical
// to total_viewshed_raw when sectors are accumulated on one GPU.
// HBM roofline: per sector ~4-8 B of cv gathered + 16 B of map RMW per cell
// (the map RMW is amortised over the whole batch: 16 B per cell per batch).
#include <cuda_runtime.h>

#include "sks_device.cuh"

namespace sks {

namespace {

constexpr double kTolD = static_cast<double>(1e-6f);  // skew.hpp:70, promoted

__device__ __forceinline__ bool full_d(double w) {
  return w > __dsub_rn(1.0, kTolD) && w < __dadd_rn(1.0, kTolD);
}

template <bool kFromCv>
__global__ void __launch_bounds__(256) unskew_kernel(BatchDev b, const double* __restrict__ vs,
                                                     double* __restrict__ map, int dimy,
                                                     int dimx) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long n = static_cast<long long>(dimy) * dimx;
  if (idx >= n) return;
  const int si = static_cast<int>(idx / dimx);
  const int sj = static_cast<int>(idx - static_cast<long long>(si) * dimx);
  double acc = map[idx];
  for (int s = 0; s < b.n_sectors; ++s) {
    const SectorDev& sd = b.sectors[s];
    const int i = sd.inv[0] * si + sd.inv[1] * sj + sd.inv[2];
    const int j = sd.inv[3] * si + sd.inv[4] * sj + sd.inv[5];
    const int dest = __ldg(b.dest + sd.col_off + j);
    const double r = __ldg(b.fracd + sd.col_off + j);
    const int p = sd.base + i - dest;
    const double omr = __dsub_rn(1.0, r);
    // covered(p, j): source rows i (main) and i+1 (carry)
    const double w_p = (i + 1 < sd.rows) ? __dadd_rn(omr, r) : omr;
    // covered(p-1, j): source rows i-1 (main) and i (carry)
    const double w_m = (i >= 1) ? __dadd_rn(omr, r) : r;
    const bool a = full_d(w_p);
    const bool c = full_d(w_m);
    const long long cell = sd.sdem_off + static_cast<long long>(p) * sd.pitch + j;
    double va = 0.0, vb = 0.0;
    if (kFromCv) {
      if (a) va = __dmul_rn(static_cast<double>(__ldg(b.cv + cell)), sd.correction);
      if (!a || c) vb = __dmul_rn(static_cast<double>(__ldg(b.cv + cell - sd.pitch)), sd.correction);
    } else {
      if (a) va = vs[cell];
      if (!a || c) vb = vs[cell - sd.pitch];
    }
    double v;
    if (a && c) {
      v = __dadd_rn(__dmul_rn(omr, va), __dmul_rn(r, vb));
    } else if (a) {
      v = va;
    } else {
      v = vb;
    }
    acc = __dadd_rn(acc, v);
  }
  map[idx] = acc;
}

__global__ void scale_kernel(double* map, long long n, double factor) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) map[i] = __dmul_rn(map[i], factor);
}

__global__ void cv_to_vs_kernel(const int* cvf, const int* cvb, double* out, long long n,
                                double correction) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    // reference: cv = fwd + bwd (exact integers in double), out = cv * corr
    const double cv = __dadd_rn(static_cast<double>(cvf[i]), static_cast<double>(cvb ? cvb[i] : 0));
    out[i] = __dmul_rn(cv, correction);
  }
}

}  // namespace

int launch_unskew(const BatchDev& b, const float*, double* map, int dimy, int dimx,
                  void* stream) {
  const long long n = static_cast<long long>(dimy) * dimx;
  const int threads = 256;
  const unsigned grid = static_cast<unsigned>((n + threads - 1) / threads);
  unskew_kernel<true><<<grid, threads, 0, static_cast<cudaStream_t>(stream)>>>(b, nullptr, map,
                                                                               dimy, dimx);
  return static_cast<int>(cudaGetLastError());
}

int launch_unskew_from_vs(const BatchDev& b, const double* skw_vs, double* map, int dimy,
                          int dimx, void* stream) {
  const long long n = static_cast<long long>(dimy) * dimx;
  const int threads = 256;
  const unsigned grid = static_cast<unsigned>((n + threads - 1) / threads);
  unskew_kernel<false><<<grid, threads, 0, static_cast<cudaStream_t>(stream)>>>(b, skw_vs, map,
                                                                                dimy, dimx);
  return static_cast<int>(cudaGetLastError());
}

int launch_scale(double* map, long long n, double factor, void* stream) {
  const int threads = 256;
  const unsigned grid = static_cast<unsigned>((n + threads - 1) / threads);
  scale_kernel<<<grid, threads, 0, static_cast<cudaStream_t>(stream)>>>(map, n, factor);
  return static_cast<int>(cudaGetLastError());
}

int launch_cv_to_vs(const int* cvf, const int* cvb, double* out, long long n, double correction,
                    void* stream) {
  const int threads = 256;
  const unsigned grid = static_cast<unsigned>((n + threads - 1) / threads);
  cv_to_vs_kernel<<<grid, threads, 0, static_cast<cudaStream_t>(stream)>>>(cvf, cvb, out, n,
                                                                            correction);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace sks
