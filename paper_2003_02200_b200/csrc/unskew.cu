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
// HBM roofline: per sector ~8 B of cv gathered per cell (the cv block a tile
// needs, staged by unskew_tiled_kernel) + 16 B of map RMW per cell per batch.
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

// Tiled form of unskew_kernel<true> (same per-cell arithmetic, same
// ascending-k order). A CTA owns a 32x32 tile of DEM cells (each thread 4
// cells of one column); per sector it stages the block of cv rows the tile
// gathers from (<= 66 rows x 32 columns, loaded along j, i.e. coalesced for
// transposed sectors too) plus the tile's dest/frac columns in shared
// memory, then every cell reads its two values from there.
constexpr int kUT = 32;           // tile edge (cells)
constexpr int kUR = 2 * kUT + 2;  // cv rows a tile can touch (shear <= 45 deg)

__global__ void __launch_bounds__(256) unskew_tiled_kernel(BatchDev b, double* __restrict__ map,
                                                           int dimy, int dimx) {
  __shared__ int scv[kUR][kUT + 1];
  __shared__ int sdest[kUT];
  __shared__ double sfrac[kUT];
  const int tx = threadIdx.x & 31;
  const int ty = threadIdx.x >> 5;  // 0..7
  const int y0 = blockIdx.y * kUT, x0 = blockIdx.x * kUT;
  const int ye = min(dimy, y0 + kUT) - 1, xe = min(dimx, x0 + kUT) - 1;  // last cell of the tile
  const int sj = x0 + tx;
  double acc[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int si = y0 + ty + 8 * u;
    acc[u] = (si < dimy && sj < dimx) ? map[static_cast<long long>(si) * dimx + sj] : 0.0;
  }
  for (int s = 0; s < b.n_sectors; ++s) {
    const SectorDev& sd = b.sectors[s];
    const int* iv = sd.inv;
    // pre_ops ranges of the tile: the affine maps are axis permutations/flips,
    // so the extremes are at the corners
    const int ia = iv[0] * y0 + iv[1] * x0 + iv[2], ib = iv[0] * ye + iv[1] * xe + iv[2];
    const int ja = iv[3] * y0 + iv[4] * x0 + iv[5], jb = iv[3] * ye + iv[4] * xe + iv[5];
    const int i_lo = min(ia, ib), i_hi = max(ia, ib);
    const int j_lo = min(ja, jb), j_hi = max(ja, jb);
    const int nj = j_hi - j_lo + 1;
    const int* dest = b.dest + sd.col_off;
    const int d_lo = __ldg(dest + j_lo), d_hi = __ldg(dest + j_hi);
    const int p_lo = sd.base + i_lo - d_hi - 1;  // includes the p-1 rows
    const int np = sd.base + i_hi - d_lo - p_lo + 1;
    // row-block sharding: rows outside [q_lo, q_hi) belong to another run
    // (their cv contributes 0 here; the runs' maps sum to the total)
    const int q_lo = sd.q_lo, q_hi = sd.q_hi;
    if (max(p_lo, q_lo) >= min(p_lo + np, q_hi)) continue;  // nothing owned here (uniform across the CTA)
    const bool whole = q_lo <= p_lo && q_hi >= p_lo + np;   // always so on one GPU
    __syncthreads();  // previous sector's smem reads are done
    if (threadIdx.x < nj) {
      sdest[threadIdx.x] = __ldg(dest + j_lo + threadIdx.x);
      sfrac[threadIdx.x] = __ldg(b.fracd + sd.col_off + j_lo + threadIdx.x);
    }
    const int* cvb = b.cv + sd.sdem_off + static_cast<long long>(p_lo) * sd.pitch + j_lo;
    if (whole) {
      for (int r = ty; r < np; r += 8) {
        if (tx < nj) scv[r][tx] = __ldg(cvb + static_cast<long long>(r) * sd.pitch + tx);
      }
    } else {
      for (int r = ty; r < np; r += 8) {
        const int p = p_lo + r;
        if (tx < nj) scv[r][tx] = (p >= q_lo && p < q_hi) ? __ldg(cvb + static_cast<long long>(r) * sd.pitch + tx) : 0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int si = y0 + ty + 8 * u;
      if (si >= dimy || sj >= dimx) continue;
      const int i = iv[0] * si + iv[1] * sj + iv[2];
      const int j = iv[3] * si + iv[4] * sj + iv[5];
      const int jl = j - j_lo;
      const int p = sd.base + i - sdest[jl];
      const double r = sfrac[jl];
      const double omr = __dsub_rn(1.0, r);
      const double w_p = (i + 1 < sd.rows) ? __dadd_rn(omr, r) : omr;
      const double w_m = (i >= 1) ? __dadd_rn(omr, r) : r;
      const bool a = full_d(w_p);
      const bool c = full_d(w_m);
      double va = 0.0, vb = 0.0;
      if (a) va = __dmul_rn(static_cast<double>(scv[p - p_lo][jl]), sd.correction);
      if (!a || c) vb = __dmul_rn(static_cast<double>(scv[p - 1 - p_lo][jl]), sd.correction);
      if (!a && !c && b.dem != nullptr) {
        // the only read that may fall outside the row ranges (skwVS is 0
        // there, scan.cpp:66); with fused relocation nothing zeroed it
        const int2 rg = (p >= 1 && p - 1 < sd.skw_rows) ? __ldg(b.ranges + sd.row_off + p - 1) : make_int2(0, 0);
        if (j < rg.x || j >= rg.y) vb = 0.0;
      }
      double v;
      if (a && c) {
        v = __dadd_rn(__dmul_rn(omr, va), __dmul_rn(r, vb));
      } else if (a) {
        v = va;
      } else {
        v = vb;
      }
      acc[u] = __dadd_rn(acc[u], v);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int si = y0 + ty + 8 * u;
    if (si < dimy && sj < dimx) map[static_cast<long long>(si) * dimx + sj] = acc[u];
  }
}

// Input scan of the DEM on device (total_host): res[0] = first non-finite
// cell index (row-major, as validate(Dem) reports it, dem.cpp:36-60), res[1]
// != 0 if a nonzero |e| lies outside the FP32 filter's proven range
// [2^-40, 2^40]. res = {ULLONG_MAX, 0} before launch.
__global__ void dem_check_kernel(const float* __restrict__ dem, long long n,
                                 unsigned long long* res) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  bool oor = false;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = __ldg(dem + i);
    if (!isfinite(v)) atomicMin(res, static_cast<unsigned long long>(i));
    const float a = fabsf(v);
    if (a != 0.f && (a < 0x1p-40f || a > 0x1p40f)) oor = true;
  }
  if (__any_sync(0xffffffffu, oor) && (threadIdx.x & 31) == 0) res[1] = 1ull;
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
  dim3 grid((dimx + kUT - 1) / kUT, (dimy + kUT - 1) / kUT);
  unskew_tiled_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(b, map, dimy, dimx);
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

int launch_dem_check(const float* dem, long long n, unsigned long long* res, void* stream) {
  const int threads = 256;
  long long blocks = (n + threads * 8 - 1) / (threads * 8);
  if (blocks < 1) blocks = 1;
  if (blocks > 4096) blocks = 4096;
  dem_check_kernel<<<static_cast<unsigned>(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(dem, n, res);
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
