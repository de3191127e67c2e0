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
// needs, staged by unskew_pipe_kernel) + 16 B of map RMW per cell per batch.
#include <cuda_runtime.h>

#include <cstdlib>

#include "sks_device.cuh"

namespace sks {

namespace {

constexpr double kTolD = static_cast<double>(1e-6f);  // skew.hpp:70, promoted

__device__ __forceinline__ bool full_d(double w) {
  return w > __dsub_rn(1.0, kTolD) && w < __dadd_rn(1.0, kTolD);
}

// Untiled form over a caller's skwVS (sks_unskew_accumulate, the per-phase
// debug entry): one thread per DEM cell.
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
    if (a) va = vs[cell];
    if (!a || c) vb = vs[cell - sd.pitch];
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

constexpr int kUT = 32;           // tile edge (cells)

// Tiled unskew (same per-cell arithmetic as unskew_kernel, same
// ascending-k order). A CTA owns a 32x32 tile of DEM cells (each thread 4
// cells of one column) and walks the batch's sectors; the cv block is staged
// by SOURCE row: T[ir][jl] =
// cv(p = base + i - dest[j], j) for i = i_lo - 1 + ir, so a cell (i, j)
// reads rows p and p-1 as T[i - i_lo + 1][jl] and T[i - i_lo][jl]: a warp
// reads one T row (non-transposed sectors) or one T column (transposed;
// stride 33) and never hits a bank twice, where indexing the staged block
// by skewed row p serialises up to 32-way at 45 degrees. 33 x 32 staged
// values per sector instead of up to 66 x 32; dest[j] is recomputed with
// the reference's double ops (shear_params, skew.cpp:97-101), so the
// staging addresses need no dependent load. Sector s+1 is copied with
// cp.async into the second buffer while sector s is computed.
constexpr int kTR = kUT + 1;  // staged source rows (the tile's rows + the row above)

#ifndef SKS_UNSKEW_MINB
#define SKS_UNSKEW_MINB 5  // CTAs per SM (48 registers)
#endif

template <bool kBlocks>  // row-block sharding: some tiles own no row of a sector
__global__ void __launch_bounds__(256, SKS_UNSKEW_MINB) unskew_pipe_kernel(BatchDev b, double* __restrict__ map, int dimy,
                                                              int dimx) {
  __shared__ int scv[2][kTR][kUT + 1];
  __shared__ int sown[2];  // sector staged in the buffer has owned rows in the tile
  __shared__ int sdest[2][kUT];
  __shared__ double sfrac[2][kUT];
  const int tx = threadIdx.x & 31;
  const int ty = threadIdx.x >> 5;  // 0..7
  const int y0 = blockIdx.y * kUT, x0 = blockIdx.x * kUT;
  const int ye = min(dimy, y0 + kUT) - 1, xe = min(dimx, x0 + kUT) - 1;
  const int sj = x0 + tx;
  const unsigned scv_u32 = static_cast<unsigned>(__cvta_generic_to_shared(&scv[0][0][0]));
  const unsigned sdest_u32 = static_cast<unsigned>(__cvta_generic_to_shared(&sdest[0][0]));
  const unsigned sfrac_u32 = static_cast<unsigned>(__cvta_generic_to_shared(&sfrac[0][0]));
  double acc[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int si = y0 + ty + 8 * u;
    acc[u] = (si < dimy && sj < dimx) ? map[static_cast<long long>(si) * dimx + sj] : 0.0;
  }
  // the tile's pre_ops box of a sector (axis permutations/flips: corners)
  auto box = [&](const int* iv, int* i_lo, int* j_lo) {
    const int ia = iv[0] * y0 + iv[1] * x0 + iv[2], ib = iv[0] * ye + iv[1] * xe + iv[2];
    const int ja = iv[3] * y0 + iv[4] * x0 + iv[5], jb = iv[3] * ye + iv[4] * xe + iv[5];
    *i_lo = min(ia, ib);
    *j_lo = min(ja, jb);
    return max(ja, jb) - *j_lo + 1;  // nj
  };
  auto stage = [&](int s, int bf) {
    const SectorDev* sdp = b.sectors + s;
    int iv[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) iv[k] = __ldg(sdp->inv + k);
    const int base = __ldg(&sdp->base), q_lo = __ldg(&sdp->q_lo), q_hi = __ldg(&sdp->q_hi);
    const int skw_rows = __ldg(&sdp->skw_rows), pitch = __ldg(&sdp->pitch), col_off = __ldg(&sdp->col_off);
    const long long sdem_off = __ldg(&sdp->sdem_off);
    const double tan = __ldg(&sdp->shear_tan);
    int i_lo, j_lo;
    const int nj = box(iv, &i_lo, &j_lo);
    bool own = true;
    if (kBlocks && !(q_lo <= 0 && q_hi >= skw_rows)) {
      // none of the skewed rows the tile reads may belong to this run
      const int d_lo = __double2int_rz(__dmul_rn(tan, static_cast<double>(j_lo)));
      const int d_hi = __double2int_rz(__dmul_rn(tan, static_cast<double>(j_lo + nj - 1)));
      const int p_min = base + i_lo - 1 - d_hi, p_max = base + i_lo + kUT - 1 - d_lo;
      own = max(p_min, q_lo) <= min(p_max, q_hi - 1);
    }
    if (kBlocks && threadIdx.x == 0) sown[bf] = own ? 1 : 0;
    if (!own) return;
    if (threadIdx.x < nj) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sdest_u32 + 4u * (bf * kUT + threadIdx.x)),
                   "l"(b.dest + col_off + j_lo + threadIdx.x));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sfrac_u32 + 8u * (bf * kUT + threadIdx.x)),
                   "l"(b.fracd + col_off + j_lo + threadIdx.x));
    }
    if (tx < nj) {
      const int j = j_lo + tx;
      const int dj = __double2int_rz(__dmul_rn(tan, static_cast<double>(j)));
      const int* col = b.cv + sdem_off + j;
      const int p0 = base + i_lo - 1 - dj;  // skewed row of T row 0
      for (int ir = ty; ir < kTR; ir += 8) {
        const int p = p0 + ir;
        const unsigned dst = scv_u32 + 4u * ((bf * kTR + ir) * (kUT + 1) + tx);
        if (p >= q_lo && p < q_hi && p >= 0 && p < skw_rows) {
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(col + static_cast<long long>(p) * pitch));
        } else {
          scv[bf][ir][tx] = 0;  // outside the sector or another run's row
        }
      }
    }
  };
  stage(0, 0);
  asm volatile("cp.async.commit_group;\n" ::);
  for (int s = 0; s < b.n_sectors; ++s) {
    const int bf = s & 1;
    if (s + 1 < b.n_sectors) {
      stage(s + 1, bf ^ 1);
      asm volatile("cp.async.commit_group;\n" ::);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();  // sector s's buffer complete for every thread
    if (kBlocks && sown[bf] == 0) {
      __syncthreads();
      continue;
    }
    const SectorDev* sdp = b.sectors + s;
    int iv[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) iv[k] = __ldg(sdp->inv + k);
    const int rows = __ldg(&sdp->rows);
    const double corr = __ldg(&sdp->correction);
    int i_lo, j_lo;
    box(iv, &i_lo, &j_lo);
    // cell u of this thread: si = y0 + ty + 8u, sj fixed; (i, j) step by 8 * (iv[0], iv[3])
    const int i0 = iv[0] * (y0 + ty) + iv[1] * sj + iv[2];
    const int j0 = iv[3] * (y0 + ty) + iv[4] * sj + iv[5];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int si = y0 + ty + 8 * u;
      if (si >= dimy || sj >= dimx) continue;
      const int i = i0 + 8 * u * iv[0];
      const int j = j0 + 8 * u * iv[3];
      const int jl = j - j_lo;
      const int ir = i - i_lo + 1;  // T row of p; p - 1 is T row ir - 1
      const double r = sfrac[bf][jl];
      const double omr = __dsub_rn(1.0, r);
      const double w_p = (i + 1 < rows) ? __dadd_rn(omr, r) : omr;
      const double w_m = (i >= 1) ? __dadd_rn(omr, r) : r;
      const bool a = full_d(w_p);
      const bool c = full_d(w_m);
      double va = 0.0, vb = 0.0;
      if (a) va = __dmul_rn(static_cast<double>(scv[bf][ir][jl]), corr);
      if (!a || c) vb = __dmul_rn(static_cast<double>(scv[bf][ir - 1][jl]), corr);
      if (!a && !c && b.dem != nullptr) {
        const SectorDev& sd = b.sectors[s];
        const int p = sd.base + i - sdest[bf][jl];
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
    __syncthreads();  // buffer bf free before sector s+2 is staged into it
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
  if (b.row_blocks) {
    unskew_pipe_kernel<true><<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(b, map, dimy, dimx);
  } else {
    unskew_pipe_kernel<false><<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(b, map, dimy, dimx);
  }
  return static_cast<int>(cudaGetLastError());
}

int launch_unskew_from_vs(const BatchDev& b, const double* skw_vs, double* map, int dimy,
                          int dimx, void* stream) {
  const long long n = static_cast<long long>(dimy) * dimx;
  const int threads = 256;
  const unsigned grid = static_cast<unsigned>((n + threads - 1) / threads);
  unskew_kernel<<<grid, threads, 0, static_cast<cudaStream_t>(stream)>>>(b, skw_vs, map,
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
