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

#include <cstddef>
#include <cstdlib>

#include <cuda.h>

#include <mutex>

#include "sks_device.cuh"
#include "sks_ptx.cuh"

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

// TMA-staged unskew (same per-cell arithmetic and ascending-k order as the
// kernels above, bit-identical maps). The copy engine brings each sector's cv
// parallelogram in as ONE 2-D box — 32 skewed-row columns [j_lo, j_lo + 32)
// x unskew_box_rows(tan) rows from p_min = base + i_lo - 1 - d(j_hi) — into a
// ring of kStages shared-memory stages (full/empty mbarriers), so the four
// consumer warps issue no staging loads, stores or CTA barriers. A fifth
// (producer) warp publishes each stage as soon as the consumers release it:
// the sector descriptor (prefetched a sector ahead, one word per lane), the
// tile's column table (r, 1 - r, box offsets, recomputed with the
// reference's double ops) and constants, then the TMA. Measured at config 2
// (0.80 ms register-staged): producer in warp 0 0.50 ms, rotating over the
// consumer warps 0.49, dedicated warp 0.45 (4 stages, 5 CTAs per SM).
// Box rows are 128 bytes, so the bank of a read is its box column: a warp's
// 32 lanes must read 32 different pre-op columns j. Plain sectors map DEM
// columns to j and transposed ones DEM rows, so each thread owns a diagonal
// of the tile — lane l, warp w: DEM column l, rows (l + 8w + u) mod 32,
// u < 8 — whose 32 lanes hold distinct DEM rows AND columns at every u:
// conflict-free in both orientations (the register-staged kernel stages by
// source row to get the same, at a load + store + barrier per value).
#ifndef SKS_UNSKEW_STAGES
#define SKS_UNSKEW_STAGES 4  // config 2: 2 stages 0.518 ms, 3 0.499 (producer in warp 0), 4 0.453 (producer warp), 5 0.523
#endif
#ifndef SKS_UNSKEW_TMA_MINB
#define SKS_UNSKEW_TMA_MINB 5  // CTAs per SM: 4 stages of 9.4 KB each
#endif
constexpr int kStages = SKS_UNSKEW_STAGES;
constexpr int kUThreads = 160;  // 4 consumer warps + the producer warp
constexpr int kBoxRowsMax = 66;  // unskew_box_rows(1.0)
static_assert(sizeof(SectorDev) == 128, "a sector descriptor is one word per lane");

struct __align__(128) UStage {
  int cv[kBoxRowsMax * kUT];  // box rows p_min .., 32 columns each
  double2 ro[kUT];            // (r, 1 - r) of box column jl (shear_params, skew.cpp:97-101)
  int offb[kUT];              // byte offset of (box row d_hi - d_j, column jl): row p of pre-op row i
                              // (il = i - i_lo + 1) at il * 128 + offb[jl]
  int iv[6];
  int i_lo, j_lo, rows, fast;
  int end;                    // no more sectors: the consumers leave
  double corr;
};

// Row-block runs (b.row_blocks): a sector's map covers only its owned rows
// [q_lo, q_hi) (the TMA zero-fills the rest, as the reference reads no cv
// there), and the producer publishes only the sectors with an owned skewed
// row in the tile's box (8 ranks: ~1/8 of them), in ascending k, then an
// end marker.
__global__ void __launch_bounds__(kUThreads, SKS_UNSKEW_TMA_MINB) unskew_tma_kernel(BatchDev b, double* __restrict__ map,
                                                                                   int dimy, int dimx, int tile_row0) {
  __shared__ UStage st[kStages];
  __shared__ uint64_t full[kStages], empty[kStages];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int y0 = (tile_row0 + blockIdx.y) * kUT, x0 = blockIdx.x * kUT;
  const int ye = min(dimy, y0 + kUT) - 1, xe = min(dimx, x0 + kUT) - 1;
  const bool full_tile = ye == y0 + kUT - 1 && xe == x0 + kUT - 1;
  const int nsec = b.n_sectors;
  if (threadIdx.x == 0) {
    for (int k = 0; k < kStages; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], 4);
    }
  }
  __syncthreads();
  if (w == 4) {
    // producer: stage n (the n-th published sector) in slot n % kStages
    int n = 0;
    auto acquire = [&](int slot) -> UStage& {
      if (n >= kStages) mbar_wait(&empty[slot], ((n / kStages) - 1) & 1);
      return st[slot];
    };
    int dw = nsec > 0 ? __ldg(reinterpret_cast<const int*>(b.sectors) + lane) : 0;
    for (int t = 0; t < nsec; ++t) {
      // sector t's descriptor words arrived while sector t - 1 was handled
      const int cur = dw;
      if (t + 1 < nsec) dw = __ldg(reinterpret_cast<const int*>(b.sectors + t + 1) + lane);
      int iv[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) iv[k] = __shfl_sync(0xffffffffu, cur, offsetof(SectorDev, inv) / 4 + k);
      const int ia = iv[0] * y0 + iv[1] * x0 + iv[2], ib = iv[0] * ye + iv[1] * xe + iv[2];
      const int ja = iv[3] * y0 + iv[4] * x0 + iv[5], jb = iv[3] * ye + iv[4] * xe + iv[5];
      const int i_lo = min(ia, ib), j_lo = min(ja, jb), i_hi = max(ia, ib), j_hi = max(ja, jb);
      auto word = [&](size_t off) { return __shfl_sync(0xffffffffu, cur, static_cast<int>(off / 4)); };
      const double tan = __hiloint2double(word(offsetof(SectorDev, shear_tan) + 4), word(offsetof(SectorDev, shear_tan)));
      const int base = word(offsetof(SectorDev, base));
      const int q_lo = word(offsetof(SectorDev, q_lo)), q_hi = word(offsetof(SectorDev, q_hi));
      const int rows = word(offsetof(SectorDev, rows));
      const double corr =
          __hiloint2double(word(offsetof(SectorDev, correction) + 4), word(offsetof(SectorDev, correction)));
      const int d_hi = __double2int_rz(__dmul_rn(tan, static_cast<double>(j_hi)));
      const int p_min = base + i_lo - 1 - d_hi;
      if (b.row_blocks) {
        // none of the skewed rows the tile reads may belong to this run
        const int d_lo = __double2int_rz(__dmul_rn(tan, static_cast<double>(j_lo)));
        const int p_max = base + i_hi - d_lo;
        if (max(p_min, q_lo) > min(p_max, q_hi - 1)) continue;
      }
      // the box must hold every row the tile reads: rows p - 1 .. p of pre-op
      // rows i_lo .. i_hi over columns j_lo .. j_hi (unskew_box_rows' bound);
      // a violation would read a neighbour's rows, so it stops the kernel
      if (i_hi - i_lo + 2 + d_hi - __double2int_rz(__dmul_rn(tan, static_cast<double>(j_lo))) >
          unskew_box_rows(tan)) {
        __trap();
      }
      const int slot = n % kStages;
      UStage& S = acquire(slot);
      {
        const int j = j_lo + lane;  // box column lane (columns past j_hi are never read)
        const double y = __dmul_rn(tan, static_cast<double>(j));
        const int d = __double2int_rz(y);
        const double r = __dsub_rn(y, static_cast<double>(d));
        S.ro[lane] = make_double2(r, __dsub_rn(1.0, r));
        S.offb[lane] = (d_hi - d) * 128 + lane * 4;
      }
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 6; ++k) S.iv[k] = iv[k];
        S.i_lo = i_lo;
        S.j_lo = j_lo;
        S.rows = rows;
        S.fast = full_tile && i_lo >= 1 && i_hi <= rows - 2;
        S.end = 0;
        S.corr = corr;
      }
      __syncwarp();
      if (lane == 0) {
        mbar_expect_tx(&full[slot], static_cast<unsigned>(unskew_box_rows(tan) * kUT * 4));
        tma_tile_2d(S.cv, static_cast<const char*>(b.umaps) + 128 * static_cast<size_t>(t), j_lo, p_min - q_lo,
                    &full[slot]);
      }
      ++n;
    }
    const int slot = n % kStages;
    UStage& S = acquire(slot);
    if (lane == 0) {
      S.end = 1;
      mbar_arrive(&full[slot]);
    }
    return;
  }
  const int sj = x0 + lane;
  const int rb = lane + 8 * w;  // this thread's rows: (rb + u) & 31
  double acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int si = y0 + ((rb + u) & 31);
    acc[u] = (si < dimy && sj < dimx) ? map[static_cast<long long>(si) * dimx + sj] : 0.0;
  }
  for (int n = 0;; ++n) {
    const int slot = n % kStages;
    mbar_wait(&full[slot], (n / kStages) & 1);
    const UStage& S = st[slot];
    if (S.end) break;
    const char* cvb = reinterpret_cast<const char*>(S.cv);
    const int iv0 = S.iv[0], iv1 = S.iv[1], iv2 = S.iv[2], iv3 = S.iv[3], iv4 = S.iv[4], iv5 = S.iv[5];
    const int i_lo = S.i_lo, j_lo = S.j_lo;
    const double corr = S.corr;
    if (S.fast) {
      // Interior tile: both covered() weights are fl(fl(1-r)+r), within
      // 2^-52 of 1, so both flags hold (skew.cpp:233-240) and every cell
      // interpolates v = fl(fl(omr*fl(cv_p*corr)) + fl(r*fl(cv_{p-1}*corr))).
      if (iv0 != 0) {
        // plain: the thread's column j is fixed, row i = iv0 * si + iv2
        const int jl = iv4 * sj + iv5 - j_lo;
        const double2 ro = S.ro[jl];
        const char* a0 = cvb + (S.offb[jl] + (iv0 * y0 + iv2 - i_lo + 1) * 128);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const char* a = a0 + iv0 * ((rb + u) & 31) * 128;
          const double va = __dmul_rn(static_cast<double>(*reinterpret_cast<const int*>(a)), corr);
          const double vb = __dmul_rn(static_cast<double>(*reinterpret_cast<const int*>(a - 128)), corr);
          acc[u] = __dadd_rn(acc[u], __dadd_rn(__dmul_rn(ro.y, va), __dmul_rn(ro.x, vb)));
        }
      } else {
        // transposed: the thread's row i is fixed, column j = iv3 * si + iv5
        const char* a0 = cvb + (iv1 * sj + iv2 - i_lo + 1) * 128;
        const int jb = iv3 * y0 + iv5 - j_lo;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int jl = jb + iv3 * ((rb + u) & 31);
          const double2 ro = S.ro[jl];
          const char* a = a0 + S.offb[jl];
          const double va = __dmul_rn(static_cast<double>(*reinterpret_cast<const int*>(a)), corr);
          const double vb = __dmul_rn(static_cast<double>(*reinterpret_cast<const int*>(a - 128)), corr);
          acc[u] = __dadd_rn(acc[u], __dadd_rn(__dmul_rn(ro.y, va), __dmul_rn(ro.x, vb)));
        }
      }
    } else {
      const int rows = S.rows;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int si = y0 + ((rb + u) & 31);
        if (si >= dimy || sj >= dimx) continue;
        const int i = iv0 * si + iv1 * sj + iv2;
        const int jl = iv3 * si + iv4 * sj + iv5 - j_lo;
        const double2 ro = S.ro[jl];
        const double r = ro.x, omr = ro.y;
        const char* a = cvb + ((i - i_lo + 1) * 128 + S.offb[jl]);
        const double w_p = (i + 1 < rows) ? __dadd_rn(omr, r) : omr;
        const double w_m = (i >= 1) ? __dadd_rn(omr, r) : r;
        const bool fa = full_d(w_p);
        const bool fc = full_d(w_m);
        double va = 0.0, vb = 0.0;
        if (fa) va = __dmul_rn(static_cast<double>(*reinterpret_cast<const int*>(a)), corr);
        if (!fa || fc) vb = __dmul_rn(static_cast<double>(*reinterpret_cast<const int*>(a - 128)), corr);
        double v;
        if (fa && fc) {
          v = __dadd_rn(__dmul_rn(omr, va), __dmul_rn(r, vb));
        } else if (fa) {
          v = va;
        } else {
          v = vb;
        }
        acc[u] = __dadd_rn(acc[u], v);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  // recompute the store addresses (an opaque copy of rb): holding the eight
  // load addresses across the sector loop costs 16 registers
  int rb2 = rb;
  asm volatile("" : "+r"(rb2));
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int si = y0 + ((rb2 + u) & 31);
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
  if (b.umaps != nullptr && b.dem == nullptr) {
    unskew_tma_kernel<<<grid, kUThreads, 0, static_cast<cudaStream_t>(stream)>>>(b, map, dimy, dimx, tile_row0);
  } else if (b.row_blocks) {
    unskew_pipe_kernel<true><<<grid, 32 * kNW, 0, static_cast<cudaStream_t>(stream)>>>(b, map, dimy, dimx, tile_row0);
  } else {
    unskew_pipe_kernel<false><<<grid, 32 * kNW, 0, static_cast<cudaStream_t>(stream)>>>(b, map, dimy, dimx, tile_row0);
  }
  return static_cast<int>(cudaGetLastError());
}

int unskew_tile_rows() { return kUT; }

namespace {
using EncodeTiledU = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledU encode_fn_u() {
  static EncodeTiledU fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<EncodeTiledU>(p);
    }
  });
  return fn;
}
}  // namespace

bool unskew_make_map(void* tm, const int* base, int pitch, int rows, int box_rows) {
  static_assert(sizeof(CUtensorMap) == 128, "tensor maps are 128 bytes");
  EncodeTiledU fn = encode_fn_u();
  if (fn == nullptr || rows < 1 || box_rows > kBoxRowsMax || pitch % 32 != 0 ||
      (reinterpret_cast<uintptr_t>(base) & 15u) != 0) {
    return false;
  }
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(pitch), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch) * sizeof(int)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kUT), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  return fn(static_cast<CUtensorMap*>(tm), CU_TENSOR_MAP_DATA_TYPE_INT32, 2, const_cast<int*>(base), dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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
