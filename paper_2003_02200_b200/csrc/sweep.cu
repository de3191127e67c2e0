// GPU rotational-sweep viewshed: the reference's independent oracle
// (oracle.cpp:74-194 — linear_scan, singular_viewshed, multi_viewshed,
// total_viewshed_reference) re-laid for B200.
//
// sweep_dirs_kernel: one thread per (observer, azimuth). The block's 128
// threads are 128 consecutive observers of the same azimuth, so at every
// step the warp reads one table entry (a broadcast) and 32 neighbouring
// cells of one DEM row segment (coalesced). The recurrence is the
// reference's FP64 one verbatim (oracle.cpp:84-98, the build's --fmad=false
// keeps dist*dist - open*open unfused like the reference's
// -ffp-contract=off), so each per-azimuth ring sum is bit-identical.
// sweep_sum_kernel then adds the ns per-azimuth sums of each observer in the
// reference's order (forward, backward, k ascending; oracle.cpp:122-126) and
// applies (pi/ns)*cellsize^2 (oracle.cpp:128).
//
// Roofline: issue bound — FP32 filter per ray cell, an IEEE double divide
// only for the cells it cannot certify; DEM reads hit L1/L2 (the rays of a
// warp share rows).
#include <cuda_runtime.h>

#include <cmath>

#include "sks_device.cuh"

namespace sks {

namespace {

constexpr int kSweepThreads = 128;
constexpr float kBand = 5.9604644775390625e-07f;  // 10 * 2^-24, as in the scan kernels

// kFilter: an FP32 filter certifies the hidden targets —
// t = fl(fl(fl(e - hf) - hl) * fl32(1/dist)) below lo = Mf - 10u|Mf|, with
// Mf = fl32(M) of the exact running max M, cannot beat M (t is within ~4.5u
// of the exact slope); every other target (records, the band) takes the
// reference's FP64 divide and compare, so every decision is the reference's. Preconditions as in the scan: h splits
// exactly into hf + hl and every elevation magnitude is 0 or in
// [2^-40, 2^40] (checked on the device first; else the kernel runs without
// the filter).
template <bool kFilter>
__global__ void __launch_bounds__(kSweepThreads)
sweep_dirs_kernel(const float* __restrict__ dem, int rows, int cols, const SweepStepDev* __restrict__ tab,
                  const int* __restrict__ len, int stride, int ndir, const int2* __restrict__ povs,
                  long long pov0, int npov, double h0, double* __restrict__ buf) {
  const int t = blockIdx.x * kSweepThreads + threadIdx.x;
  if (t >= npov) return;
  int i0, j0;
  if (povs != nullptr) {
    const int2 p = povs[t];
    i0 = p.x;
    j0 = p.y;
  } else {
    const long long p = pov0 + t;
    i0 = static_cast<int>(p / cols);
    j0 = static_cast<int>(p % cols);
  }
  // pov_h = dem(i0, j0) + h0 (oracle.cpp:116)
  const double h = static_cast<double>(dem[static_cast<long long>(i0) * cols + j0]) + h0;
  const float hf = __double2float_rn(h);
  const double hld = h - static_cast<double>(hf);
  const float hl = __double2float_rn(hld);
  const bool filt = kFilter && static_cast<double>(hl) == hld && fabsf(hf) < 1e30f;
  for (int d = blockIdx.y; d < ndir; d += gridDim.y) {
    const SweepStepDev* s = tab + static_cast<long long>(d) * stride;
    const int L = len[d];
    double cv = 0.0, max_theta = -INFINITY, open_d = 0.0, last_d = 0.0;
    float lo = -INFINITY;  // fl32(M) - 10u|fl32(M)|
    bool visible = false;
    for (int n = 0; n < L; ++n) {
      const SweepStepDev st = s[n];
      const int i = i0 + st.di, j = j0 + st.dj;
      if (static_cast<unsigned>(i) >= static_cast<unsigned>(rows) ||
          static_cast<unsigned>(j) >= static_cast<unsigned>(cols)) {
        break;  // the ray left the grid (oracle.cpp:40,52)
      }
      const float e = __ldg(dem + static_cast<long long>(i) * cols + j);
      bool above;
      if (filt) {
        const float tf = __fmul_rn(__fadd_rn(__fadd_rn(e, -hf), -hl), st.inv);
        if (tf < lo) {
          above = false;  // certainly below the running max
        } else {
          const double theta = (static_cast<double>(e) - h) / st.dist;
          above = theta > max_theta;
          if (above) {
            max_theta = theta;
            const float mf = __double2float_rn(theta);
            lo = __fmaf_rn(fabsf(mf), -kBand, mf);
          }
        }
      } else {
        const double theta = (static_cast<double>(e) - h) / st.dist;  // oracle.cpp:86
        above = theta > max_theta;
        if (above) max_theta = theta;
      }
      if (above && !visible) {
        open_d = st.dist;
      } else if (!above && visible) {
        cv += st.dist * st.dist - open_d * open_d;
      }
      visible = above;
      last_d = st.dist;
    }
    if (visible) {  // close at the last cell + 1 (oracle.cpp:101-105)
      const double close_d = last_d + 1.0;
      cv += close_d * close_d - open_d * open_d;
    }
    buf[static_cast<long long>(d) * npov + t] = cv;
  }
}

__global__ void sweep_sum_kernel(const double* __restrict__ buf, int ndir, int npov, double pi_over_ns,
                                 double cellsize, double unit_factor, double* __restrict__ out,
                                 long long out_stride_off) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= npov) return;
  double cv = 0.0;
  for (int d = 0; d < ndir; ++d) cv += buf[static_cast<long long>(d) * npov + t];
  double area = cv * pi_over_ns * cellsize * cellsize;  // oracle.cpp:128
  if (unit_factor != 1.0) area = area * unit_factor;  // convert_units (dem.cpp:24-34)
  out[out_stride_off + t] = area;
}

// linear_scan (oracle.cpp:74-106) of one ray with its ring sectors: the
// reference's FP64 recurrence verbatim, one thread (a debug / API entry).
__global__ void linear_scan_kernel(const float* __restrict__ dem, int rows, int cols, int i0, int j0, double pov_h,
                                   const SweepStepDev* __restrict__ tab, int len, double* out_cv,
                                   double* rings, int cap, int* nrings) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double cv = 0.0, max_theta = -INFINITY, open_d = 0.0, last_d = 0.0;
  bool visible = false;
  int nr = 0;
  for (int n = 0; n < len; ++n) {
    const SweepStepDev st = tab[n];
    const int i = i0 + st.di, j = j0 + st.dj;
    if (static_cast<unsigned>(i) >= static_cast<unsigned>(rows) ||
        static_cast<unsigned>(j) >= static_cast<unsigned>(cols)) {
      break;
    }
    const double theta = (static_cast<double>(dem[static_cast<long long>(i) * cols + j]) - pov_h) / st.dist;
    const bool above = theta > max_theta;
    if (above && !visible) {
      open_d = st.dist;
    } else if (!above && visible) {
      cv += st.dist * st.dist - open_d * open_d;
      if (nr < cap) {
        rings[2 * nr] = open_d;
        rings[2 * nr + 1] = st.dist;
      }
      ++nr;
    }
    visible = above;
    if (above) max_theta = theta;
    last_d = st.dist;
  }
  if (visible) {
    const double close_d = last_d + 1.0;
    cv += close_d * close_d - open_d * open_d;
    if (nr < cap) {
      rings[2 * nr] = open_d;
      rings[2 * nr + 1] = close_d;
    }
    ++nr;
  }
  *out_cv = cv;
  *nrings = nr;
}

}  // namespace

int launch_sweep(const float* dem, int rows, int cols, const SweepStepDev* tab, const int* len, int stride,
                 int ndir, const int2* povs, long long pov0, int npov, double h0, double* buf, bool filter,
                 void* stream) {
  if (npov <= 0) return 0;
  const dim3 grid((npov + kSweepThreads - 1) / kSweepThreads, ndir < 65535 ? ndir : 65535);
  if (filter) {
    sweep_dirs_kernel<true><<<grid, kSweepThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        dem, rows, cols, tab, len, stride, ndir, povs, pov0, npov, h0, buf);
  } else {
    sweep_dirs_kernel<false><<<grid, kSweepThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        dem, rows, cols, tab, len, stride, ndir, povs, pov0, npov, h0, buf);
  }
  return static_cast<int>(cudaGetLastError());
}

int launch_linear_scan(const float* dem, int rows, int cols, int i0, int j0, double pov_h, const SweepStepDev* tab,
                       int len, double* out_cv, double* rings, int cap, int* nrings, void* stream) {
  linear_scan_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(dem, rows, cols, i0, j0, pov_h, tab, len, out_cv,
                                                                      rings, cap, nrings);
  return static_cast<int>(cudaGetLastError());
}

int launch_sweep_sum(const double* buf, int ndir, int npov, double pi_over_ns, double cellsize,
                     double unit_factor, double* out, long long out_off, void* stream) {
  if (npov <= 0) return 0;
  sweep_sum_kernel<<<(npov + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      buf, ndir, npov, pi_over_ns, cellsize, unit_factor, out, out_off);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace sks
