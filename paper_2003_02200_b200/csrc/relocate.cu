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
// The pre_ops (transpose / column flip) are fused into the tile loader: a CTA
// owns an output tile of kTQ sDEM rows x kTJ columns, loads the parallelogram
// of pre_ops-space source rows it needs into shared memory with loads that
// are coalesced in DEM space (thread.x walks DEM columns whichever pre_ops
// axis they map to), then writes the tile with 16-byte vector stores.
// HBM roofline: 4 B read + 4 B written per covered cell.
#include <cuda_runtime.h>

#include "sks_device.cuh"

namespace sks {

namespace {

constexpr int kTQ = 64;                 // output rows per tile
constexpr int kTJ = 64;                 // output columns per tile
constexpr int kSrcRows = kTQ + kTJ + 2;  // parallelogram height bound
constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
relocate_kernel(const float* __restrict__ dem, BatchDev b, int tiles_x) {
  __shared__ float src[kSrcRows][kTJ + 1];
  __shared__ int s_dest[kTJ];
  __shared__ float s_frac[kTJ];

  const SectorDev sd = b.sectors[blockIdx.y];
  const int tile = blockIdx.x;
  // tile rows are counted from the first tile row holding an owned row
  const int tq = tile / tiles_x + sd.q_lo / kTQ;
  const int tj = tile - (tile / tiles_x) * tiles_x;
  const int q0 = tq * kTQ;
  const int j0 = tj * kTJ;
  if (q0 >= sd.skw_rows || j0 >= sd.cols) return;
  if (q0 + kTQ <= sd.q_lo || q0 >= sd.q_hi) return;  // no row of this run's block (row sharding)
  const int jn = min(kTJ, sd.cols - j0);
  const int* dest = b.dest + sd.col_off;
  const float* fracf = b.fracf + sd.col_off;

  const int dest_lo = __ldg(dest + j0);
  const int dest_hi = __ldg(dest + j0 + jn - 1);
  // source rows touched by the tile: main rows start at q0-base+dest_lo,
  // carry rows end at (q0+kTQ-1)-base+dest_hi+1
  int i_lo = q0 - sd.base + dest_lo;
  int i_hi = q0 + kTQ - 1 - sd.base + dest_hi + 1;
  if (i_hi < 0 || i_lo > sd.rows - 1) return;  // tile has no source cell
  i_lo = max(i_lo, 0);
  i_hi = min(i_hi, sd.rows - 1);
  const int n_src = i_hi - i_lo + 1;

  for (int t = threadIdx.x; t < jn; t += kThreads) {
    s_dest[t] = __ldg(dest + j0 + t);
    s_frac[t] = __ldg(fracf + j0 + t);
  }
  // Load src[i - i_lo][j - j0] = pre(i, j) = dem(to_source(i, j)).
  const int* m = sd.map;
  if (m[1] == 0) {
    // DEM column depends on j only: thread.x over j is coalesced.
    for (int t = threadIdx.x; t < n_src * kTJ; t += kThreads) {
      int r = t / kTJ, c = t - r * kTJ;
      if (c < jn) {
        int i = i_lo + r, j = j0 + c;
        int si = m[0] * i + m[2];
        int sj = m[4] * j + m[5];
        src[r][c] = __ldg(dem + static_cast<size_t>(si) * sd.src_cols + sj);
      }
    }
  } else {
    // Transposed sectors: DEM column depends on i only; walk i fastest.
    for (int t = threadIdx.x; t < n_src * kTJ; t += kThreads) {
      int c = t / n_src, r = t - c * n_src;
      if (c < jn) {
        int i = i_lo + r, j = j0 + c;
        int si = m[1] * j + m[2];
        int sj = m[3] * i + m[5];
        src[r][c] = __ldg(dem + static_cast<size_t>(si) * sd.src_cols + sj);
      }
    }
  }
  __syncthreads();

  // Output: a thread owns 4 consecutive columns x 4 consecutive rows. Along
  // a column the carry source of row q is the main source of row q+1, so
  // each column needs 5 source values for its 4 outputs (register carry).
  // Each output row leaves as one 16-byte store; the cv pool cells of the
  // same tile are zeroed with it (this replaces a memset of the whole pool).
  float* out = b.sdem + sd.sdem_off;
  int* cvz = b.cv + sd.sdem_off;
  const int cx = (threadIdx.x & 15) * 4;
  const int r0 = (threadIdx.x >> 4) * 4;
  float v[4][4];  // [row][col]
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int jj = cx + c;
    const bool colok = jj < jn;
    const float f = colok ? s_frac[jj] : 0.f;
    const float a = __fsub_rn(1.0f, f);
    const int im0 = q0 + r0 - sd.base + (colok ? s_dest[jj] : 0);  // main source row of the first output
    float sv[5];
#pragma unroll
    for (int u = 0; u < 5; ++u) {
      const int im = im0 + u;
      sv[u] = (colok && im >= 0 && im < sd.rows) ? src[im - i_lo][jj] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int im = im0 + u;
      float acc = 0.0f;
      if (colok) {
        if (im >= 0 && im < sd.rows) acc = __fadd_rn(acc, __fmul_rn(a, sv[u]));
        if (im + 1 >= 0 && im + 1 < sd.rows) acc = __fadd_rn(acc, __fmul_rn(f, sv[u + 1]));
      }
      v[u][c] = acc;
    }
  }
  if (j0 + cx < sd.pitch) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = q0 + r0 + u;
      if (q < sd.skw_rows) {
        const size_t o = static_cast<size_t>(q) * sd.pitch + j0 + cx;
        // streaming (evict-first) stores: 2.9 GB of sDEM + cv must not push
        // the 16 MB DEM, which every tile gathers from, out of L2
        __stcs(reinterpret_cast<float4*>(out + o), make_float4(v[u][0], v[u][1], v[u][2], v[u][3]));
        __stcs(reinterpret_cast<int4*>(cvz + o), make_int4(0, 0, 0, 0));
      }
    }
  }
}

}  // namespace

int launch_relocate_grid(const float* dem, const BatchDev& b, int tiles_x,
                         int tiles_total, void* stream) {
  dim3 grid(tiles_total, b.n_sectors);
  relocate_kernel<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      dem, b, tiles_x);
  return static_cast<int>(cudaGetLastError());
}

int relocate_tile_rows() { return kTQ; }
int relocate_tile_cols() { return kTJ; }

}  // namespace sks
