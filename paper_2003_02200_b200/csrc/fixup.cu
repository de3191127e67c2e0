// Exact resolution of flagged POV groups (sm_100a).
//
// The scan kernels certify every decision they can with the FP32 filter
// and queue a POV group whenever a target fell inside the
// uncertainty band (or h does not split into two floats). This kernel
// re-runs those POVs with the reference's semantics (scan.cpp:8-62):
// the same FP32 filter certifies what it can, and every band target is
// decided with the reference's own IEEE FP64 operations
// theta = ((double)row[k] - h) / dd (scan.cpp:24-25) against the exact
// running maximum, recomputed from the last record r as
// ((double)row[r] - h) / r when needed. POVs whose h does not split exactly
// run the FP64 recurrence on every target. Every decision that reaches cv is
// therefore the reference's.
//
// Mapping. The queue is segmented per skewed row (one exact-bound segment
// per scan item, filled by the scan kernels), so a warp takes up to 4
// consecutive rows at a time (longest rows first, global counter), stages
// those with queued POVs in its own shared-memory buffers with coalesced
// loads, and spreads all their queued POVs over its lanes (about 10 per row
// on fractal terrain, so one row alone would leave most lanes idle).
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <cstdlib>

#include "sks_device.cuh"

namespace sks {

namespace {

constexpr float kBand = 5.9604644775390625e-07f;  // 10 * 2^-24, as in the scan kernels
constexpr int kWarps = 8;

// Exact state of one POV scan (the reference recurrence under the filter).
struct ExactState {
  float hf, hl;
  double h;
  float hi, lo;
  int r;          // last record (0: none yet, max = -inf)
  double M;       // exact max theta when Mvalid
  bool Mvalid;
  int cv;
};

// One target, every case handled (filter + exact FP64 inside the band).
__device__ __forceinline__ bool exact_step(ExactState& S, const float* row, int x, int sg, int dd,
                                           float e, float inv) {
  const float t = __fmul_rn(__fadd_rn(__fsub_rn(e, S.hf), -S.hl), inv);
  bool above;
  if (t > S.hi) {
    above = true;
    S.Mvalid = false;
  } else if (t >= S.lo) {
    const double th = __ddiv_rn(__dsub_rn(static_cast<double>(e), S.h), static_cast<double>(dd));
    if (!S.Mvalid) {
      S.M = __ddiv_rn(__dsub_rn(static_cast<double>(row[x + sg * S.r]), S.h), static_cast<double>(S.r));
      S.Mvalid = true;
    }
    above = th > S.M;
    if (above) S.M = th;
  } else {
    above = false;
  }
  if (above) {
    const float at = fabsf(t);
    S.hi = __fmaf_rn(at, kBand, t);
    S.lo = __fmaf_rn(at, -kBand, t);
    S.r = dd;
    S.cv += 2 * dd + 1;
  }
  return above;
}

// One POV: row in shared memory (row coordinates), observer at x, direction
// sg (+1 forward, -1 backward), D targets, ivt[d] = fl(1/d). Returns
// cv = sum (2dd+1) over the visible targets; writes per-target decisions to
// vis when non-null. Groups of 4 targets run a branch-free certified fast
// path (predicated updates only); a group containing a band target is rolled
// back and re-run target by target with the exact resolution.
__device__ int exact_pov(const float* row, const float* wm, int L, const float* ivt, int x, int sg,
                         int D, double h, bool force_exact, uint8_t* vis) {
  ExactState S;
  S.h = h;
  S.hf = __double2float_rn(h);
  const double hld = __dsub_rn(h, static_cast<double>(S.hf));
  S.hl = __double2float_rn(hld);
  S.hi = -INFINITY;
  S.lo = -FLT_MAX;
  S.r = 0;
  S.M = -INFINITY;
  S.Mvalid = true;
  S.cv = 0;
  const bool exact_all = force_exact || static_cast<double>(S.hl) != hld || !(fabsf(S.hf) < 1e30f);
  if (exact_all) {
    double M = -INFINITY;
    int cv = 0;
    for (int dd = 1; dd <= D; ++dd) {
      const float e = row[x + sg * dd];
      const double th = __ddiv_rn(__dsub_rn(static_cast<double>(e), h), static_cast<double>(dd));
      const bool above = th > M;
      if (above) {
        M = th;
        cv += 2 * dd + 1;
      }
      if (vis) vis[dd - 1] = above ? 1 : 0;
    }
    return cv;
  }
  int dd = 1;
  if (vis == nullptr) {
    for (; dd + 3 <= D; dd += 4) {
      // Hidden-window skip (per lane), as in the scan kernels: every target
      // of dd .. dd+15 has t <= max(fl(N*fl(1/dd)), fl(N*fl(1/de))) with
      // N = fl(fl(em - hf) - hl), em the maximum elevation of those targets
      // (two 16-position window maxima cover them); below lo nothing in the
      // window is a record or a band target.
      if ((dd & 15) == 1) {
        const int de = min(dd + 15, D);
        const int pa = sg > 0 ? x + dd : x - de;  // lowest position of the window
        const int pb = sg > 0 ? x + de : x - dd;  // highest
        const float em = fmaxf(wm[pa >> 4], wm[pb >> 4]);
        const float N = __fadd_rn(__fsub_rn(em, S.hf), -S.hl);
        if (__fmul_rn(N, ivt[dd]) < S.lo && __fmul_rn(N, ivt[de]) < S.lo) {
          dd += 12;  // + 4 by the loop: the next window
          continue;
        }
      }
      float t[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float e = row[x + sg * (dd + i)];
        t[i] = __fmul_rn(__fadd_rn(__fsub_rn(e, S.hf), -S.hl), ivt[dd + i]);
      }
      const float hi0 = S.hi, lo0 = S.lo;
      const int cv0 = S.cv, r0 = S.r;
      bool band = false, rec = false;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool pa = t[i] > S.hi;
        const bool pg = t[i] >= S.lo;
        band |= pg & !pa;
        rec |= pa;
        if (pa) {
          const float at = fabsf(t[i]);
          S.hi = __fmaf_rn(at, kBand, t[i]);
          S.lo = __fmaf_rn(at, -kBand, t[i]);
          S.cv += 2 * (dd + i) + 1;
          S.r = dd + i;
        }
      }
      if (band) {
        S.hi = hi0;
        S.lo = lo0;
        S.cv = cv0;
        S.r = r0;
#pragma unroll 1
        for (int i = 0; i < 4; ++i) {
          exact_step(S, row, x, sg, dd + i, row[x + sg * (dd + i)], ivt[dd + i]);
        }
      } else if (rec) {
        S.Mvalid = false;
      }
    }
  }
  for (; dd <= D; ++dd) {
    const bool above = exact_step(S, row, x, sg, dd, row[x + sg * dd], ivt[dd]);
    if (vis) vis[dd - 1] = above ? 1 : 0;
  }
  return S.cv;
}

constexpr int kMaxRows = 4;  // rows staged per warp (their queued POVs share the lanes)

__global__ void __launch_bounds__(kWarps * 32) fixup_kernel(ScanArgs a, int row_floats, int rpw) {
  extern __shared__ __align__(16) float fsm[];
  const int lane = threadIdx.x & 31;
  float* ivt = fsm;  // fl(1/d), d = 0 .. row_floats - 1
  // per warp: rpw rows, then rpw window-max tables of row_floats / 16
  float* rows = fsm + row_floats * (1 + rpw * (threadIdx.x >> 5)) + (row_floats / 16) * rpw * (threadIdx.x >> 5);
  float* wms = rows + rpw * row_floats;
  for (int d = threadIdx.x; d < row_floats; d += blockDim.x) {
    ivt[d] = __frcp_rn(static_cast<float>(d));
  }
  __syncthreads();
  const unsigned grp = static_cast<unsigned>(a.fix_group);
  for (;;) {
    // claim rpw consecutive rows; lane j < rpw inspects row it0 + j
    int it0 = 0;
    if (lane == 0) it0 = static_cast<int>(atomicAdd(a.fix_item_counter, static_cast<unsigned>(rpw)));
    it0 = __shfl_sync(0xffffffffu, it0, 0);
    if (it0 >= a.n_items) break;
    unsigned mycnt = 0;
    if (lane < rpw && it0 + lane < a.n_items) mycnt = a.fix_cnt[it0 + lane] * grp;  // POVs of row j
    // inclusive prefix over the rpw rows
    unsigned incl = mycnt;
#pragma unroll
    for (int o = 1; o < kMaxRows; o <<= 1) {
      const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    const unsigned total = __shfl_sync(0xffffffffu, incl, rpw - 1);
    if (total == 0) continue;
    unsigned ends[kMaxRows];
#pragma unroll
    for (int j = 0; j < kMaxRows; ++j) ends[j] = __shfl_sync(0xffffffffu, incl, j);
    // stage the rows that have queued POVs
    for (int j = 0; j < rpw; ++j) {
      const unsigned cj = ends[j] - (j ? ends[j - 1] : 0u);
      if (cj == 0) continue;
      const ScanItem item = a.items[it0 + j];
      const SectorDev& sd = a.b.sectors[item.s];
      const int2 rg = a.b.ranges[sd.row_off + item.q];
      const float* src = a.b.sdem + sd.sdem_off + static_cast<long long>(item.q) * sd.pitch + rg.x;
      float* row = rows + j * row_floats;
      const int L = rg.y - rg.x;
#pragma unroll 4
      for (int x = lane; x < L; x += 32) row[x] = __ldg(src + x);
      __syncwarp();
      float* wm = wms + j * (row_floats / 16);
      for (int w = lane; w * 16 < L; w += 32) {
        float m = -INFINITY;
        const int e = min(L, 16 * w + 16);
        for (int u = 16 * w; u < e; ++u) m = fmaxf(m, row[u]);
        wm[w] = m;
      }
    }
    __syncwarp();
    for (unsigned base = 0; base < total; base += 32) {
      const unsigned w = base + lane;
      if (w < total) {
        int j = 0;
#pragma unroll
        for (int u = 0; u < kMaxRows - 1; ++u) j += (u < rpw - 1 && w >= ends[u]) ? 1 : 0;
        const unsigned wj = w - (j ? ends[j - 1] : 0u);
        const int it = it0 + j;
        const ScanItem item = a.items[it];
        const SectorDev& sd = a.b.sectors[item.s];
        const int2 rg = a.b.ranges[sd.row_off + item.q];
        const int first = rg.x;
        const int L = rg.y - rg.x;
        const float* row = rows + j * row_floats;
        const unsigned ent = a.fix_queue[a.fix_off[it] + wj / grp];
        const int dir = static_cast<int>(ent >> 31);
        const int y = static_cast<int>((ent & 0x7fffffffu) * grp + wj % grp);
        if (y < L) {
          const int x = dir ? (L - 1 - y) : y;
          const int D = min(sd.max_dd, dir ? x : (L - 1 - x));
          const bool dbg = a.dbg_j0 >= 0 && item.s == 0 && item.q == 0 && first + x == a.dbg_j0;
          const double h = dbg ? a.dbg_h : __dadd_rn(static_cast<double>(row[x]), a.h0);
          uint8_t* vis = dbg ? (dir ? a.dbg_vis_bwd : a.dbg_vis_fwd) : nullptr;
          const int cv = exact_pov(row, wms + j * (row_floats / 16), L, ivt, x, dir ? -1 : 1, D, h,
                                   a.force_exact != 0, vis);
          if (cv != 0) {
            int* dst = ((dir && a.b.cv_bwd) ? a.b.cv_bwd : a.b.cv) + sd.sdem_off +
                       static_cast<long long>(item.q) * sd.pitch + first;
            atomicAdd(dst + x, cv);
          }
        }
      }
    }
    __syncwarp();  // the row buffers are reused for the next rows
  }
}

}  // namespace

int launch_fixup(const ScanArgs& a, void* stream) {
  if (a.n_items == 0) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int row_floats = ((a.lmax + 31) / 32) * 32;
  const size_t cap = 200 * 1024;
  // rows per warp (up to 4) and warps per CTA (up to 8) under the budget;
  // one more row-sized buffer holds the fl(1/d) table
  const size_t rowb = row_floats * sizeof(float) + (row_floats / 16) * sizeof(float);  // row + window maxima
  const size_t slots = (cap - row_floats * sizeof(float)) / rowb;  // rows that fit next to the 1/d table
  if (slots < 1) return static_cast<int>(cudaErrorInvalidValue);  // rows beyond ~24000 cells
  static const int rpw_env = [] {
    const char* s = std::getenv("SKS_FIXUP_RPW");
    return s != nullptr ? std::atoi(s) : 1;
  }();
  const int rpw = static_cast<int>(min(static_cast<size_t>(max(1, min(rpw_env, kMaxRows))), slots));
  const int warps = static_cast<int>(min(static_cast<size_t>(kWarps), slots / rpw));
  const size_t smem = row_floats * sizeof(float) + static_cast<size_t>(warps) * rpw * rowb;
  cudaError_t e = cudaFuncSetAttribute(fixup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return static_cast<int>(e);
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fixup_kernel, warps * 32, smem);
  if (e != cudaSuccess) return static_cast<int>(e);
  fixup_kernel<<<sms * (per_sm > 0 ? per_sm : 1), warps * 32, smem, static_cast<cudaStream_t>(stream)>>>(
      a, row_floats, rpw);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace sks
