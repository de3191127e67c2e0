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

#ifndef SKS_UNSKEW_CPT
#define SKS_UNSKEW_CPT 8  // cells per thread (8: 128 threads per tile; measured 0.79 ms vs 0.91 with 4, config 2)
#endif
constexpr int kCPT = SKS_UNSKEW_CPT;
constexpr int kNW = kUT / kCPT;                 // warps per CTA (cell rows of kCPT)
constexpr int kNV = (kTR + kNW - 1) / kNW;     // staged T rows per thread
#ifndef SKS_UNSKEW_MINB
#define SKS_UNSKEW_MINB (kCPT == 4 ? 5 : 8)  // CTAs per SM (4: 48 registers, 8: 64)
#endif

// Per-sector constants of a staged buffer (written by thread 0 with the
// staging, read as shared broadcasts).
struct USect {
  int iv[6];
  int rows, i_lo, j_lo;
  int fast;  // every cell of the tile is interior in pre_ops space (1 <= i <= rows-2)
  double corr;
};

template <bool kBlocks>  // row-block sharding: some tiles own no row of a sector
__global__ void __launch_bounds__(32 * kNW, SKS_UNSKEW_MINB) unskew_pipe_kernel(BatchDev b, double* __restrict__ map, int dimy,
                                                              int dimx, int tile_row0) {
  __shared__ int scv[2][kTR][kUT + 1];
  __shared__ int sown[2];  // sector staged in the buffer has owned rows in the tile
  __shared__ int sdest[2][kUT];
  __shared__ double sfrac[2][kUT];
  __shared__ USect ssec[2];
  // ring of the next sectors' descriptors (SectorDev copied word by word):
  // sector s sits in slot s % 3 from iteration s - 2 on
  constexpr int kSecWords = static_cast<int>(sizeof(SectorDev) / 4);
  static_assert(sizeof(SectorDev) % 8 == 0, "SectorDev copied as whole words");
  __shared__ SectorDev sring[3];
  // Row-block runs (kBlocks): the sectors with a skewed row of this run in
  // the tile, compacted in ascending order at the start, so the loop below
  // (one barrier per sector) walks only those (8 ranks: ~1/8 of them).
  constexpr int kMaxList = 2048;
  __shared__ short slist[kBlocks ? kMaxList : 1];
  __shared__ int nlist_s;
  auto load_sec = [&](int idx) {
    const int s = (kBlocks && nlist_s >= 0) ? slist[idx] : idx;
    if (threadIdx.x < kSecWords) {
      reinterpret_cast<int*>(sring + idx % 3)[threadIdx.x] =
          __ldg(reinterpret_cast<const int*>(b.sectors + s) + threadIdx.x);
    }
  };
  const int tx = threadIdx.x & 31;
  const int ty = threadIdx.x >> 5;  // 0 .. kNW-1
  const int y0 = (tile_row0 + blockIdx.y) * kUT, x0 = blockIdx.x * kUT;
  const int ye = min(dimy, y0 + kUT) - 1, xe = min(dimx, x0 + kUT) - 1;
  const bool full_tile = ye == y0 + kUT - 1 && xe == x0 + kUT - 1;
  const int sj = x0 + tx;
  const int sy = y0 + kCPT * ty;  // this thread's cells: (sy + u, sj), u < kCPT
  double acc[kCPT];
#pragma unroll
  for (int u = 0; u < kCPT; ++u) {
    const int si = sy + u;
    acc[u] = (si < dimy && sj < dimx) ? map[static_cast<long long>(si) * dimx + sj] : 0.0;
  }
  // the tile's pre_ops box of a sector (axis permutations/flips: corners)
  auto box = [&](const int* iv, int* i_lo, int* j_lo, int* ni) {
    const int ia = iv[0] * y0 + iv[1] * x0 + iv[2], ib = iv[0] * ye + iv[1] * xe + iv[2];
    const int ja = iv[3] * y0 + iv[4] * x0 + iv[5], jb = iv[3] * ye + iv[4] * xe + iv[5];
    *i_lo = min(ia, ib);
    *j_lo = min(ja, jb);
    *ni = max(ia, ib) - *i_lo + 1;
    return max(ja, jb) - *j_lo + 1;  // nj
  };
  // Staging is software-pipelined through registers: the loads of sector s+1
  // are issued before sector s is computed and stored to shared memory after
  // it, so one barrier per sector separates the stores from the reads.
  // Thread (tx, ty) stages column tx, T rows ty + kNW*k (< kTR).
  // The sector constants, dest and frac of sector s go straight to buffer
  // s & 1, last read while sector s-2 was computed, before the barrier that
  // precedes this fetch; only the cv values wait in registers.
  struct Pre {
    int v[kNV];
    int own;
  };
  auto fetch = [&](int s, Pre& P) {
    const int bf = s & 1;
    const SectorDev& sdp = sring[s % 3];
    int iv[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) iv[k] = sdp.inv[k];
    const int base = sdp.base, q_lo = sdp.q_lo, q_hi = sdp.q_hi;
    const int skw_rows = sdp.skw_rows, pitch = sdp.pitch, col_off = sdp.col_off;
    const long long sdem_off = sdp.sdem_off;
    const double tan = sdp.shear_tan;
    int i_lo, j_lo, ni;
    const int nj = box(iv, &i_lo, &j_lo, &ni);
    if (threadIdx.x == 0) {
      USect& c = ssec[bf];
#pragma unroll
      for (int k = 0; k < 6; ++k) c.iv[k] = iv[k];
      const int rows = sdp.rows;
      c.rows = rows;
      c.i_lo = i_lo;
      c.j_lo = j_lo;
      c.fast = full_tile && i_lo >= 1 && i_lo + ni - 1 <= rows - 2;
      c.corr = sdp.correction;
    }
    bool own = true;
    if (kBlocks && !(q_lo <= 0 && q_hi >= skw_rows)) {
      // none of the skewed rows the tile reads may belong to this run
      const int d_lo = __double2int_rz(__dmul_rn(tan, static_cast<double>(j_lo)));
      const int d_hi = __double2int_rz(__dmul_rn(tan, static_cast<double>(j_lo + nj - 1)));
      const int p_min = base + i_lo - 1 - d_hi, p_max = base + i_lo + kUT - 1 - d_lo;
      own = max(p_min, q_lo) <= min(p_max, q_hi - 1);
    }
    P.own = own;
    if (kBlocks && threadIdx.x == 0) sown[bf] = own ? 1 : 0;
    if (threadIdx.x < nj && own) {
      sdest[bf][threadIdx.x] = __ldg(b.dest + col_off + j_lo + threadIdx.x);
      sfrac[bf][threadIdx.x] = __ldg(b.fracd + col_off + j_lo + threadIdx.x);
    }
#pragma unroll
    for (int k = 0; k < kNV; ++k) P.v[k] = 0;
    if (tx < nj && own) {
      const int j = j_lo + tx;
      const int dj = __double2int_rz(__dmul_rn(tan, static_cast<double>(j)));
      const int p0 = base + i_lo - 1 - dj + ty;  // skewed row of T row ty
      const int plo = max(q_lo, 0), phi = min(q_hi, skw_rows);  // staged rows [plo, phi)
      // one 64-bit base per column (T row ty), 32-bit byte offsets from it
      const char* col = reinterpret_cast<const char*>(b.cv + sdem_off + j + static_cast<long long>(p0) * pitch);
      unsigned off = 0;
      const unsigned step = static_cast<unsigned>(kNW * pitch) * 4u;
#pragma unroll
      for (int k = 0; k < kNV; ++k) {
        const int p = p0 + kNW * k;
        if (ty + kNW * k < kTR && static_cast<unsigned>(p - plo) < static_cast<unsigned>(phi - plo)) {
          P.v[k] = __ldg(reinterpret_cast<const int*>(col + off));
        }
        off += step;
      }
    }
  };
  auto commit = [&](const Pre& P, int bf) {
    if (!P.own) return;
#pragma unroll
    for (int k = 0; k < kNV; ++k) {
      if (ty + kNW * k < kTR) scv[bf][ty + kNW * k][tx] = P.v[k];
    }
  };
  int nsec = b.n_sectors;
  if (kBlocks) {
    if (threadIdx.x == 0) nlist_s = b.n_sectors <= kMaxList ? 0 : -1;
    __syncthreads();
    if (nlist_s >= 0) {
      // same test as fetch's: some skewed row the tile reads is this run's
      for (int c0 = 0; c0 < b.n_sectors; c0 += blockDim.x) {
        const int s = c0 + threadIdx.x;
        bool own = false;
        if (s < b.n_sectors) {
          const SectorDev& sd = b.sectors[s];
          int iv[6];
#pragma unroll
          for (int k = 0; k < 6; ++k) iv[k] = sd.inv[k];
          int i_lo, j_lo, ni;
          const int nj = box(iv, &i_lo, &j_lo, &ni);
          own = true;
          if (!(sd.q_lo <= 0 && sd.q_hi >= sd.skw_rows)) {
            const double tan = sd.shear_tan;
            const int d_lo = __double2int_rz(__dmul_rn(tan, static_cast<double>(j_lo)));
            const int d_hi = __double2int_rz(__dmul_rn(tan, static_cast<double>(j_lo + nj - 1)));
            const int p_min = sd.base + i_lo - 1 - d_hi, p_max = sd.base + i_lo + kUT - 1 - d_lo;
            own = max(p_min, sd.q_lo) <= min(p_max, sd.q_hi - 1);
          }
        }
        // ordered compaction: warp ballots, then the warps in turn
        const unsigned m = __ballot_sync(0xffffffffu, own);
        for (int w = 0; w < kNW; ++w) {
          if (ty == w && own) slist[nlist_s + __popc(m & ((1u << tx) - 1u))] = static_cast<short>(s);
          __syncthreads();
          if (ty == w && tx == 0) nlist_s += __popc(m);
          __syncthreads();
        }
      }
      nsec = nlist_s;
    }
  }
  Pre P;
  if (nsec > 0) load_sec(0);
  if (nsec > 1) load_sec(1);
  __syncthreads();
  if (nsec > 0) fetch(0, P);
  for (int s = 0; s < nsec; ++s) {
    const int bf = s & 1;
    commit(P, bf);
    __syncthreads();  // sector s staged; sector s-1's buffer (bf ^ 1) no longer read
    // slot (s+2) % 3 held sector s-1, last read by fetch(s-1) before this barrier
    if (s + 2 < nsec) load_sec(s + 2);
    if (s + 1 < nsec) fetch(s + 1, P);
    if (kBlocks && sown[bf] == 0) continue;
    const USect& c = ssec[bf];
    const int iv0 = c.iv[0], iv1 = c.iv[1], iv2 = c.iv[2], iv3 = c.iv[3], iv4 = c.iv[4], iv5 = c.iv[5];
    const int i_lo = c.i_lo, j_lo = c.j_lo;
    const double corr = c.corr;
    const int i0 = iv0 * sy + iv1 * sj + iv2;  // pre_ops cell of (sy, sj); (sy + u, sj) adds u * (iv0, iv3)
    const int j0 = iv3 * sy + iv4 * sj + iv5;
    if (c.fast) {
      // Interior cells: both covered() weights are fl(fl(1-r)+r), within
      // 2^-52 of 1, so both flags hold (skew.cpp:233-240) and every cell
      // interpolates v = fl(fl(omr*fl(cv_p*corr)) + fl(r*fl(cv_{p-1}*corr))).
      if (iv0 != 0) {
        // pre_ops row i = iv0*si + ..: the cells are consecutive rows of one
        // column j; each group of 4 reads 5 consecutive staged rows
        const int jl = j0 - j_lo;
        const double r = sfrac[bf][jl];
        const double omr = __dsub_rn(1.0, r);
        const int ir0 = i0 - i_lo + 1;        // T row of cell 0's p
#pragma unroll
        for (int h = 0; h < kCPT / 4; ++h) {
          const int rb = min(ir0 + 4 * h * iv0, ir0 + (4 * h + 3) * iv0) - 1;  // first of the 5 T rows
          double va[5];
#pragma unroll
          for (int k = 0; k < 5; ++k) va[k] = __dmul_rn(static_cast<double>(scv[bf][rb + k][jl]), corr);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            // T row of cell 4h+u's p relative to rb (1..4)
            const int ka = iv0 > 0 ? u + 1 : 4 - u;
            acc[4 * h + u] = __dadd_rn(acc[4 * h + u], __dadd_rn(__dmul_rn(omr, va[ka]), __dmul_rn(r, va[ka - 1])));
          }
        }
      } else {
        // transposed: the cells are consecutive columns of one row i
        const int ir = i0 - i_lo + 1;
#pragma unroll
        for (int u = 0; u < kCPT; ++u) {
          const int jl = j0 + u * iv3 - j_lo;
          const double r = sfrac[bf][jl];
          const double omr = __dsub_rn(1.0, r);
          const double va = __dmul_rn(static_cast<double>(scv[bf][ir][jl]), corr);
          const double vb = __dmul_rn(static_cast<double>(scv[bf][ir - 1][jl]), corr);
          acc[u] = __dadd_rn(acc[u], __dadd_rn(__dmul_rn(omr, va), __dmul_rn(r, vb)));
        }
      }
    } else {
      const int rows = c.rows;
#pragma unroll
      for (int u = 0; u < kCPT; ++u) {
        const int si = sy + u;
        if (si >= dimy || sj >= dimx) continue;
        const int i = i0 + u * iv0;
        const int j = j0 + u * iv3;
        const int jl = j - j_lo;
        const int ir = i - i_lo + 1;  // T row of p; p - 1 is T row ir - 1
        const double r = sfrac[bf][jl];
        const double omr = __dsub_rn(1.0, r);
        const double w_p = (i + 1 < rows) ? __dadd_rn(omr, r) : omr;
        const double w_m = (i >= 1) ? __dadd_rn(omr, r) : r;
        const bool a = full_d(w_p);
        const bool cc = full_d(w_m);
        double va = 0.0, vb = 0.0;
        if (a) va = __dmul_rn(static_cast<double>(scv[bf][ir][jl]), corr);
        if (!a || cc) vb = __dmul_rn(static_cast<double>(scv[bf][ir - 1][jl]), corr);
        if (!a && !cc && b.dem != nullptr) {
          const SectorDev& sd = b.sectors[(kBlocks && nlist_s >= 0) ? slist[s] : s];
          const int p = sd.base + i - sdest[bf][jl];
          const int2 rg = (p >= 1 && p - 1 < sd.skw_rows) ? __ldg(b.ranges + sd.row_off + p - 1) : make_int2(0, 0);
          if (j < rg.x || j >= rg.y) vb = 0.0;
        }
        double v;
        if (a && cc) {
          v = __dadd_rn(__dmul_rn(omr, va), __dmul_rn(r, vb));
        } else if (a) {
          v = va;
        } else {
          v = vb;
        }
        acc[u] = __dadd_rn(acc[u], v);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kCPT; ++u) {
    const int si = sy + u;
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
                  void* stream, int tile_row0, int tile_rows) {
  const int all_rows = (dimy + kUT - 1) / kUT;
  if (tile_rows < 0) tile_rows = all_rows - tile_row0;
  if (tile_rows <= 0) return 0;
  dim3 grid((dimx + kUT - 1) / kUT, tile_rows);
  if (b.row_blocks) {
    unskew_pipe_kernel<true><<<grid, 32 * kNW, 0, static_cast<cudaStream_t>(stream)>>>(b, map, dimy, dimx, tile_row0);
  } else {
    unskew_pipe_kernel<false><<<grid, 32 * kNW, 0, static_cast<cudaStream_t>(stream)>>>(b, map, dimy, dimx, tile_row0);
  }
  return static_cast<int>(cudaGetLastError());
}

int unskew_tile_rows() { return kUT; }

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
