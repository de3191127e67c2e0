// Relocation kernel: DEM -> skewed DEM (sDEM) for every sector of a batch.
//
// Replaces apply_pre_ops + build_skw (reference skew.cpp:103-196). The
// reference scatters each source cell into rows p = base+i-dest[j] and p-1;
// here every output cell GATHERS its two sources
//     v(q, j) = (+0 + (1-f)*src[q-base+dest[j]]) + f*src[q-base+dest[j]+1]
// (each term only if its source row exists), which is the same sequence of
// IEEE float operations in the same order (main share first, skew.cpp:172-
// 183), so the sDEM is bit-identical. __fmul_rn/__fadd_rn forbid FMA
// contraction; starting from +0 reproduces the reference's signed zeros.
//
// A CTA owns an output tile of kTQ sDEM rows x kTJ columns. The pre_ops
// (transpose / flips, skew.cpp:103-142) are axis permutations, so the
// parallelogram of pre_ops-space source cells the tile needs lies in one DEM
// rectangle: it is fetched by TMA (cp.async.bulk.tensor.2d, one thread, an
// mbarrier) as up to 5 boxes of ~9 KB stacked along the long side, with the
// out-of-range parts zero-filled by the copy engine. No thread issues a
// global load for the source (the previous gather loop was 62 % of the
// kernel's instructions and 80 % of its stall samples, profiles/r02_*).
//   * sectors without transposition: boxes of 32 DEM rows x 68 columns; a
//     lane owns one output column and walks 16 output rows (17 shared loads:
//     the carry source of row q is the main source of row q+1). Lanes read
//     32 consecutive DEM columns: conflict-free whatever the shear.
//   * transposed sectors: boxes of 64 DEM rows x 36 columns; a lane owns one
//     output ROW and walks 16 columns (consecutive lanes read consecutive DEM
//     columns of one DEM row: conflict-free), results go through a padded
//     shared tile and leave as coalesced rows.
// Every output row leaves as coalesced 128-byte warp stores (streaming: the
// 2.9 GB of sDEM + cv must not push the DEM, which every tile reads, out of
// L2), and the cv pool cells of the tile are zeroed with it (this replaces a
// memset of the whole pool). HBM roofline: 4 B read + 4 B written per
// covered cell, plus 4 B of cv zeroing.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>

#include "sks_device.cuh"
#include "sks_ptx.cuh"

namespace sks {

namespace {

#ifndef SKS_RELOC_TQ
#define SKS_RELOC_TQ 64  // measured (config 2 / 4): 32 rows 0.98 / 4.40 ms (3 stages 1.01 / 4.90), 64 rows 0.77 / 3.76, 128 rows 0.78 / 3.67
#endif
constexpr int kTQ = SKS_RELOC_TQ;  // output rows per tile (64 or 32)
static_assert(kTQ == 32 || kTQ == 64 || kTQ == 128, "8 consumer warps: 4, 8 or 16 rows each");
constexpr int kRW = kTQ / 8;       // rows per consumer warp (plain tiles, stores)
constexpr int kTJ = 32;  // output columns per tile (narrow: the parallelogram overhang grows with the width)
constexpr int kConsumers = 256;  // 8 consumer warps (+ 1 producer warp)
constexpr int kBoxLong = 32;  // source cells per box along the parallelogram's long side
// The copy engine needs the innermost (DEM column) box coordinate at a 16-byte
// boundary (measured: an unaligned one is an illegal instruction), so the
// column start is rounded down to a multiple of 4 and every box carries 4
// more columns. One box shape serves both orientations: 36 DEM columns x 32
// DEM rows, stacked along the DEM rows (sectors without transposition: the
// tile's 32 columns + 4) or along the DEM columns (transposed sectors: box k
// serves source columns 32k .. 32k + 31 of the aligned start).
constexpr int kBW = kBoxLong + 4;           // box columns
constexpr int kBoxFloats = kBW * kBoxLong;  // 4.5 KB (a multiple of 128 B)
constexpr int kMaxBoxes = (kTQ + kTJ + 4 + kBoxLong - 1) / kBoxLong;  // n_src <= kTQ + kTJ + 1 (+3 of alignment)
#ifndef SKS_RELOC_STAGES
#define SKS_RELOC_STAGES 2  // measured (config 2): 2 stages 0.95 ms, 3 1.01, 4 1.18, 6 1.92 (CTAs per SM matter more than depth)
#endif
constexpr int kStages = SKS_RELOC_STAGES;   // tiles in flight per CTA (kStages - 1 prefetched)
constexpr int kOutLd = kTJ + 1;             // padded output tile (transposed sectors)
#ifndef SKS_RELOC_VZERO
#define SKS_RELOC_VZERO 1  // cv zeroing (and transposed-tile rows) as 16-byte stores: a quarter of the store instructions
#endif

// cv zeroing of warp w's 8 tile rows (q0 + 8w ..): 8 lanes x 16 B per
// 128-byte row, two rows per lane; rows past the sector's skewed rows are
// left alone (the last sector's rows end the pool). j0 + 32 <= pitch always
// (j0 is a multiple of 32 below cols <= pitch, a multiple of 32).
template <bool kInterior>
__device__ __forceinline__ void zero_cv_rows(int* cv, size_t row0_off, int pitch, int q_first, int skw_rows,
                                             int lane) {
#pragma unroll
  for (int k = 0; k < kRW / 4; ++k) {
    const int rr = 4 * k + (lane >> 3);
    if (kInterior || q_first + rr < skw_rows) {
      __stcs(reinterpret_cast<int4*>(cv + row0_off + static_cast<size_t>(rr) * pitch + 4 * (lane & 7)),
             make_int4(0, 0, 0, 0));
    }
  }
}

// Geometry of one output tile (t = sector * tiles_total + tile); s < 0: end.
struct Tile {
  int s, q0, j0, jn, nbox, S0, J0;  // J0: the boxes' first DEM column (16-byte aligned)
  int transposed;
  int interior;  // full tile whose every source row exists: no per-cell range tests
};

struct RelocSmem {
  float box[kStages][kMaxBoxes * kBoxFloats];  // 128-byte aligned TMA destinations
  float out[kTQ * kOutLd];                     // transposed sectors: the tile before its coalesced store
  Tile tile[kStages];
  uint64_t full[kStages];   // tile published + boxes landed (producer arrive + copy bytes)
  uint64_t empty[kStages];  // stage released by the 8 consumer warps
};

__device__ __forceinline__ void tma_load_2d(float* dst, const CUtensorMap* tm, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ bool tile_geom(const BatchDev& b, int tiles_x, int tiles_total, int t, Tile& g) {
  g.s = t / tiles_total;
  const int tile = t - g.s * tiles_total;
  const SectorDev& sd = b.sectors[g.s];
  const int q_lo = sd.q_lo, q_hi = sd.q_hi, skw_rows = sd.skw_rows, cols = sd.cols;
  // tile rows are counted from the first tile row holding an owned row
  const int tq = tile / tiles_x + q_lo / kTQ;
  const int tj = tile - (tile / tiles_x) * tiles_x;
  g.q0 = tq * kTQ;
  g.j0 = tj * kTJ;
  if (g.q0 >= skw_rows || g.j0 >= cols) return false;
  if (g.q0 + kTQ <= q_lo || g.q0 >= q_hi) return false;  // no row of this run's block (row sharding)
  g.jn = min(kTJ, cols - g.j0);
  const int* dest = b.dest + sd.col_off;
  // source rows touched by the tile: main rows start at q0-base+dest_lo,
  // carry rows end at (q0+kTQ-1)-base+dest_hi+1
  int i_lo = g.q0 - sd.base + __ldg(dest + g.j0);
  int i_hi = g.q0 + kTQ - 1 - sd.base + __ldg(dest + g.j0 + g.jn - 1) + 1;
  if (i_hi < 0 || i_lo > sd.rows - 1) return false;  // tile has no source cell
  g.interior = i_lo >= 0 && i_hi <= sd.rows - 1 && g.jn == kTJ && g.q0 + kTQ <= skw_rows;
  i_lo = max(i_lo, 0);
  i_hi = min(i_hi, sd.rows - 1);
  const int* m = sd.map;
  g.transposed = m[1] != 0;
  // DEM rectangle of the parallelogram: (S0, J) = its smallest DEM (row, column)
  int J;
  if (!g.transposed) {  // si = m0*i + m2, sj = m4*j + m5
    g.S0 = m[0] > 0 ? m[0] * i_lo + m[2] : m[0] * i_hi + m[2];
    J = m[4] > 0 ? m[4] * g.j0 + m[5] : m[4] * (g.j0 + kTJ - 1) + m[5];
    g.nbox = (i_hi - i_lo + kBoxLong) / kBoxLong;
  } else {  // si = m1*j + m2, sj = m3*i + m5
    g.S0 = m[1] > 0 ? m[1] * g.j0 + m[2] : m[1] * (g.j0 + kTJ - 1) + m[2];
    J = m[3] > 0 ? m[3] * i_lo + m[5] : m[3] * i_hi + m[5];
    g.nbox = (((J & 3) + i_hi - i_lo) >> 5) + 1;
  }
  g.J0 = J - (J & 3);
  return true;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync() {  // the kConsumers threads only
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

// Sector without transposition: lane = output column c, rows r0 .. r0+7 of
// the tile (the carry source of row q is the main source of row q+1: 9 shared
// loads for 8 outputs); smem index of pre (i, j) is
// (m0*i + m2 - S0)*kBW + (m4*j + m5 - J0) (boxes stacked along the DEM rows).
template <bool kInterior>
__device__ __forceinline__ void plain_tile(const Tile& g, const SectorDev& sd, const BatchDev& b,
                                           const float* box, int lane, int warp) {
  const int base = sd.base, rows = sd.rows, pitch = sd.pitch, skw_rows = sd.skw_rows;
  const int m0 = sd.map[0], m2 = sd.map[2], m4 = sd.map[4], m5 = sd.map[5];
  const int c = lane;
  const int r0 = kRW * warp;
  const bool colok = kInterior || c < g.jn;
  const float f = colok ? __ldg(b.fracf + sd.col_off + g.j0 + c) : 0.f;
  const float a = __fsub_rn(1.0f, f);
  const int im0 = g.q0 + r0 - base + (colok ? __ldg(b.dest + sd.col_off + g.j0 + c) : 0);  // main row of r0
  const int col = m4 * (g.j0 + c) + m5 - g.J0;
  const int rstep = kBW * m0;
  int idx = (m0 * im0 + m2 - g.S0) * kBW + col;
  float sv[kRW + 1];
#pragma unroll
  for (int u = 0; u < kRW + 1; ++u) {
    const int im = im0 + u;
    sv[u] = (kInterior || (colok && im >= 0 && im < rows)) ? box[idx] : 0.f;
    idx += rstep;
  }
  float* po = b.sdem + sd.sdem_off + static_cast<size_t>(g.q0 + r0) * pitch + g.j0 + c;
  int* pc = b.cv + sd.sdem_off + static_cast<size_t>(g.q0 + r0) * pitch + g.j0 + c;
  const bool store_col = kInterior || g.j0 + c < pitch;
#pragma unroll
  for (int u = 0; u < kRW; ++u) {
    const int im = im0 + u;
    float acc = 0.0f;
    if (kInterior) {
      acc = __fadd_rn(__fadd_rn(acc, __fmul_rn(a, sv[u])), __fmul_rn(f, sv[u + 1]));
    } else if (colok) {
      if (im >= 0 && im < rows) acc = __fadd_rn(acc, __fmul_rn(a, sv[u]));
      if (im + 1 >= 0 && im + 1 < rows) acc = __fadd_rn(acc, __fmul_rn(f, sv[u + 1]));
    }
    if (kInterior || (store_col && g.q0 + r0 + u < skw_rows)) {
      __stcs(po, acc);
#if !SKS_RELOC_VZERO
      __stcs(pc, 0);
#endif
    }
    po += pitch;
    pc += pitch;
  }
#if SKS_RELOC_VZERO
  (void)pc;
  zero_cv_rows<kInterior>(b.cv + sd.sdem_off, static_cast<size_t>(g.q0 + r0) * pitch + g.j0, pitch, g.q0 + r0,
                          skw_rows, lane);
#endif
}

// Transposed sector: lane = output row r = 32*(warp&1) + lane, columns
// c0 .. c0+7 into the padded output tile; smem index of pre (i, j) is box
// (sj-J0)/32, row si-S0, column (sj-J0)%32 of that box (boxes stacked along
// the DEM columns).
template <bool kInterior>
__device__ __forceinline__ void transposed_tile(const Tile& g, const SectorDev& sd, const BatchDev& b,
                                                const float* box, float* outs, int lane, int warp) {
  const int* dest = b.dest + sd.col_off + g.j0;
  const float* fracf = b.fracf + sd.col_off + g.j0;
  const int base = sd.base, rows = sd.rows;
  const int m1 = sd.map[1], m2 = sd.map[2], m3 = sd.map[3], m5 = sd.map[5];
  // lane = one of 32 output rows of a row group (kTQ / 32 groups), the
  // group's 8 / groups warps split the 32 columns (64-row tiles: 8 each)
  constexpr int kGroups = kTQ / 32, kCW = 4 * kGroups;
  const int r = 32 * (warp % kGroups) + lane;
  const int c0 = kCW * (warp / kGroups);
#pragma unroll 4
  for (int cc = 0; cc < kCW; ++cc) {
    const int c = c0 + cc;
    float acc = 0.0f;
    if (kInterior || c < g.jn) {
      const float f = __ldg(fracf + c);
      const float a = __fsub_rn(1.0f, f);
      const int im = g.q0 + r - base + __ldg(dest + c);
      const int srow = (m1 * (g.j0 + c) + m2 - g.S0) * kBW;
      const int sc = m3 * im + m5 - g.J0;
      const int sc1 = sc + m3;
      if (kInterior || (im >= 0 && im < rows)) {
        acc = __fadd_rn(acc, __fmul_rn(a, box[(sc >> 5) * kBoxFloats + srow + (sc & 31)]));
      }
      if (kInterior || (im + 1 >= 0 && im + 1 < rows)) {
        acc = __fadd_rn(acc, __fmul_rn(f, box[(sc1 >> 5) * kBoxFloats + srow + (sc1 & 31)]));
      }
    }
    outs[r * kOutLd + c] = acc;
  }
}

// Persistent and warp-specialised: a CTA walks tiles blockIdx.x, +gridDim.x,
// ... through a ring of kStages shared-memory stages. One producer warp finds
// the next tile with work (empty tiles skipped), publishes its geometry and
// requests its boxes from the copy engine (full[st]); eight consumer warps
// wait on full[st], compute and store the tile, and release the stage
// (empty[st]), so the producer's geometry walk and the copies overlap the
// consumers' work.
#ifndef SKS_RELOC_MINB
#define SKS_RELOC_MINB 5
#endif
__global__ void __launch_bounds__(kConsumers + 32, SKS_RELOC_MINB) relocate_kernel(const __grid_constant__ CUtensorMap tm,
                                                                   BatchDev b, int tiles_x, int tiles_total) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  RelocSmem& sm = *reinterpret_cast<RelocSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int k = 0; k < kStages; ++k) {
      mbar_init(&sm.full[k], 1);
      mbar_init(&sm.empty[k], kConsumers / 32);
    }
  }
  __syncthreads();
  if (warp == kConsumers / 32) {
    // producer
    if (lane != 0) return;
    const int n_all = b.n_sectors * tiles_total;
    int t = blockIdx.x;
    // the next tile's geometry (its descriptor and dest loads) is found
    // before waiting for a free stage, so that latency overlaps the wait
    Tile g;
    auto next_tile = [&]() {
      for (; t < n_all; t += gridDim.x) {
        if (tile_geom(b, tiles_x, tiles_total, t, g)) return;
      }
    };
    next_tile();
    for (int n = 0;; ++n) {
      const int st = n % kStages;
      mbar_wait(&sm.empty[st], (static_cast<unsigned>(n / kStages) & 1u) ^ 1u);
      if (t >= n_all) {
        sm.tile[st].s = -1;
        mbar_arrive(&sm.full[st]);
        return;
      }
      sm.tile[st] = g;
      // the stage was last read through the generic proxy
      fence_proxy_async();
      mbar_expect_tx(&sm.full[st], static_cast<unsigned>(g.nbox * kBoxFloats * 4));
      for (int k = 0; k < g.nbox; ++k) {
        float* dst = sm.box[st] + k * kBoxFloats;
        if (!g.transposed) {
          tma_load_2d(dst, &tm, g.J0, g.S0 + k * kBoxLong, &sm.full[st]);
        } else {
          tma_load_2d(dst, &tm, g.J0 + k * kBoxLong, g.S0, &sm.full[st]);
        }
      }
      t += gridDim.x;
      next_tile();
    }
  }
  for (int n = 0;; ++n) {
    const int st = n % kStages;
    mbar_wait(&sm.full[st], static_cast<unsigned>(n / kStages) & 1u);
    const Tile g = sm.tile[st];
    if (g.s < 0) break;
    const SectorDev& sd = b.sectors[g.s];
    const float* box = sm.box[st];
    if (!g.transposed) {
      if (g.interior) {
        plain_tile<true>(g, sd, b, box, lane, warp);
      } else {
        plain_tile<false>(g, sd, b, box, lane, warp);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[st]);
    } else {
      if (g.interior) {
        transposed_tile<true>(g, sd, b, box, sm.out, lane, warp);
      } else {
        transposed_tile<false>(g, sd, b, box, sm.out, lane, warp);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[st]);
      consumer_sync();  // output tile complete
      // warp w stores rows 8w .. 8w+7 (128 bytes each)
      const int pitch = sd.pitch, skw_rows = sd.skw_rows;
      float* out = b.sdem + sd.sdem_off;
      int* cvz = b.cv + sd.sdem_off;
#if SKS_RELOC_VZERO
      // rows as 16-byte stores: lane -> row 8w + 4k + lane/8, columns 4*(lane%8) ..
      const size_t o0 = static_cast<size_t>(g.q0 + kRW * warp) * pitch + g.j0;
#pragma unroll
      for (int k = 0; k < kRW / 4; ++k) {
        const int rr = 4 * k + (lane >> 3), c4 = 4 * (lane & 7);
        const int rt = kRW * warp + rr;
        if (g.interior || g.q0 + rt < skw_rows) {
          const float* src = sm.out + rt * kOutLd + c4;
          __stcs(reinterpret_cast<float4*>(out + o0 + static_cast<size_t>(rr) * pitch + c4),
                 make_float4(src[0], src[1], src[2], src[3]));
        }
      }
      zero_cv_rows<false>(cvz, o0, pitch, g.q0 + kRW * warp, skw_rows, lane);
#else
      const size_t o0 = static_cast<size_t>(g.q0 + kRW * warp) * pitch + g.j0 + lane;
#pragma unroll
      for (int rr = 0; rr < kRW; ++rr) {
        const int rt = kRW * warp + rr;
        if (g.interior || (g.q0 + rt < skw_rows && g.j0 + lane < pitch)) {
          const size_t o = o0 + static_cast<size_t>(rr) * pitch;
          __stcs(out + o, sm.out[rt * kOutLd + lane]);
          __stcs(cvz + o, 0);
        }
      }
#endif
      consumer_sync();  // output tile free
    }
  }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<EncodeTiled>(p);
    }
  });
  return fn;
}

bool make_map(CUtensorMap* tm, const float* dem, int rows, int cols, long long pitch, int box_w, int box_h) {
  EncodeTiled fn = encode_fn();
  if (fn == nullptr) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch) * sizeof(float)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_h)};
  const cuuint32_t estr[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(dem), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int relocate_dem_align() { return 4; }  // DEM row pitch (floats) and base alignment the TMA maps need

int launch_relocate_grid(const float* dem, int dem_rows, int dem_cols, long long dem_pitch, const BatchDev& b,
                         int tiles_x, int tiles_total, void* stream) {
  if ((reinterpret_cast<uintptr_t>(dem) & 15u) != 0 || dem_pitch % 4 != 0 || dem_pitch < dem_cols) {
    return static_cast<int>(cudaErrorMisalignedAddress);
  }
  CUtensorMap tm;
  if (!make_map(&tm, dem, dem_rows, dem_cols, dem_pitch, kBW, kBoxLong)) return static_cast<int>(cudaErrorInvalidValue);
  const int smem = static_cast<int>(sizeof(RelocSmem));
  cudaError_t e = cudaFuncSetAttribute(relocate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return static_cast<int>(e);
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, relocate_kernel, kConsumers + 32, smem);
  const long long n = static_cast<long long>(tiles_total) * b.n_sectors;
  const int grid = static_cast<int>(std::min<long long>(n, static_cast<long long>(sms) * std::max(per_sm, 1)));
  if (grid < 1) return 0;
  relocate_kernel<<<grid, kConsumers + 32, smem, static_cast<cudaStream_t>(stream)>>>(tm, b, tiles_x, tiles_total);
  return static_cast<int>(cudaGetLastError());
}

int relocate_tile_rows() { return kTQ; }
int relocate_tile_cols() { return kTJ; }

}  // namespace sks
