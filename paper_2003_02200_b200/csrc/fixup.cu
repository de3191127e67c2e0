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
// per scan item, filled by the scan kernels). A one-CTA prefix over the
// per-row counts turns the segments into one flat list of queued POVs (in
// row order, longest rows first) and every thread takes POVs from it: work
// is spread over all lanes however the flags cluster (whole runs or the
// row blocks of one GPU of several). Rows are read through L1/L2 and each
// POV skips hidden 16-position blocks with the row's window maxima (written
// by the scan's row loader).
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdlib>
#include <string>
#include <algorithm>
#include <cstdint>

#include "sks_device.cuh"

namespace sks {

namespace {

constexpr float kBand = 5.9604644775390625e-07f;  // 10 * 2^-24, as in the scan kernels
#ifndef SKS_FIX_WARPS
#define SKS_FIX_WARPS 8
#endif
constexpr int kWarps = SKS_FIX_WARPS;
#ifndef SKS_FIX_FULL16
#define SKS_FIX_FULL16 1  // candidate blocks through eval16 (eval_block only for band blocks)
#endif
#ifndef SKS_FIX_COARSE
#define SKS_FIX_COARSE 1  // one bound test per batch of kWm windows before the per-window tests
#endif

// Exact state of one POV scan (the reference recurrence under the filter).
struct ExactState {
  float hf, hl;
  double h;
  float hi, lo;
  int r;          // last record (0: none yet, max = -inf)
  double M;       // exact max theta when Mvalid
  bool Mvalid;
  int cv;
#ifdef SKS_EXP_BANDHIST
  int first_band;  // dd of the first band target (-1: none)
  int gap;         // its distance to the last record
  int blk_before, blk_after;
#endif
};

#ifdef SKS_EXP_BANDHIST
// experiment build (tools/bandhist.py): where the first band target of each
// re-run POV falls and how the evaluated blocks split around it
__device__ unsigned long long g_bandhist[64];
#endif

// One target, every case handled (filter + exact FP64 inside the band).
__device__ __forceinline__ bool exact_step(ExactState& S, const float* row, int x, int sg, int dd,
                                           float e, float inv) {
  const float t = __fmul_rn(__fadd_rn(__fsub_rn(e, S.hf), -S.hl), inv);
  bool above;
  if (t > S.hi) {
    above = true;
    S.Mvalid = false;
  } else if (t >= S.lo) {
#ifdef SKS_EXP_BANDHIST
    if (S.first_band < 0) {
      S.first_band = dd;
      S.gap = dd - S.r;
    }
#endif
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

// Targets dd = da .. db of one POV, in order: branch-free certified fast
// path in groups of 4 (predicated updates only); a group containing a band
// target is rolled back and re-run target by target with the exact
// resolution, as is the remainder (< 4).
// Block form: the block's (up to 16) elevations are loaded together first
// (ev[i] = row[x + sg*(da+i)]), so a lane waits for one L2 round trip per
// block instead of one per group of 4.
__device__ __forceinline__ void eval_block(ExactState& S, const float* row, const float* ivt, int x,
                                           int sg, int da, int db) {
  float ev[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) ev[i] = da + i <= db ? __ldg(row + x + sg * (da + i)) : 0.f;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int dd = da + 4 * g;
    if (dd + 3 > db) {
      // remainder (< 4 targets): one by one
#pragma unroll
      // (elevations re-read through L1: ev stays in registers, statically indexed)
#pragma unroll 1
      for (int i = 0; i < 4; ++i) {
        if (dd + i <= db) exact_step(S, row, x, sg, dd + i, __ldg(row + x + sg * (dd + i)), ivt[dd + i]);
      }
      break;
    }
    float t[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) t[i] = __fmul_rn(__fadd_rn(__fsub_rn(ev[4 * g + i], S.hf), -S.hl), ivt[dd + i]);
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
      for (int i = 0; i < 4; ++i) exact_step(S, row, x, sg, dd + i, __ldg(row + x + sg * (dd + i)), ivt[dd + i]);
    } else if (rec) {
      S.Mvalid = false;
    }
  }
}

__device__ __forceinline__ void eval_range(ExactState& S, const float* row, const float* ivt, int x,
                                           int sg, int da, int db) {
  int dd = da;
  for (; dd + 3 <= db; dd += 4) {
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
      for (int i = 0; i < 4; ++i) exact_step(S, row, x, sg, dd + i, row[x + sg * (dd + i)], ivt[dd + i]);
    } else if (rec) {
      S.Mvalid = false;
    }
  }
  for (; dd <= db; ++dd) exact_step(S, row, x, sg, dd, row[x + sg * dd], ivt[dd]);
}

// The targets of block w (positions 16w .. 16w+15) with dd in [da, db], in
// scan order: target i of the block has dd = d0 + i (d0 = 16w - x forward,
// x - 16w - 15 backward) and elevation e[i] (e[15 - i] backward); targets
// outside [da, db] get a NaN 1/d and are no-ops. Branch-free certified pass
// (predicated updates, ring sums as one packed accumulator, a near-hit count);
// returns false with S untouched when a target fell in the band (the caller
// re-runs the block with eval_block). The row is read at positions up to
// 16 ceil(L / 16) - 1 (the sdem pool has slack for the last row).
__device__ __forceinline__ bool eval16(ExactState& S, const float* row, const float* ivt, int w, int sg, int d0,
                                       int da, int db) {
  float e[16], q[16];
  const float* pb = row + 16 * w;
#pragma unroll
  for (int i = 0; i < 16; ++i) e[i] = __ldg(pb + i);
  if (db - da == 15) {
    const float* iv = ivt + da;
#pragma unroll
    for (int i = 0; i < 16; ++i) q[i] = iv[i];
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int dd = d0 + i;
      const int idx = min(max(dd, da), db);
      const float v = ivt[idx];
      q[i] = dd == idx ? v : __int_as_float(0x7fc00000);
    }
  }
  int A = 0, rr = 0;
  float G = 0.f;
  float hi = S.hi, lo = S.lo;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float ev = sg > 0 ? e[i] : e[15 - i];
    const float t = __fmul_rn(__fadd_rn(__fsub_rn(ev, S.hf), -S.hl), q[i]);
    const int kb = (1 << 22) + i;
    asm("{\n\t.reg .pred pa, pg;\n\t.reg .f32 at;\n\t"
        "setp.gt.f32 pa, %5, %0;\n\t"
        "setp.ge.f32 pg, %5, %1;\n\t"
        "abs.f32 at, %5;\n\t"
        "@pa fma.rn.f32 %0, at, %8, %5;\n\t"
        "@pa fma.rn.f32 %1, at, %9, %5;\n\t"
        "@pa add.s32 %2, %2, %6;\n\t"
        "@pa mov.b32 %3, %7;\n\t"
        "@pg add.rn.f32 %4, %4, 0f3F800000;\n\t}"
        : "+f"(hi), "+f"(lo), "+r"(A), "+r"(rr), "+f"(G)
        : "f"(t), "r"(kb), "r"(i), "f"(kBand), "f"(-kBand));
  }
  const int n = A >> 22;
  if (__float2int_rn(G) != n) return false;
  if (n != 0) {
    S.hi = hi;
    S.lo = lo;
    S.cv += 2 * (n * d0 + (A & ((1 << 22) - 1))) + n;
    S.r = d0 + rr;
    S.Mvalid = false;
  }
  return true;
}

// One POV: row (row coordinates), observer at x, direction sg (+1 forward,
// -1 backward), D targets, ivt[d] = fl(1/d), wm[w] = max(row[16w .. 16w+15])
// (or nullptr). Returns cv = sum (2dd+1) over the visible targets; writes
// per-target decisions to vis when non-null (no skipping then).
//
// Hidden-window skip (per POV), as in the scan kernels: the targets of one
// 16-position block w have dd in [da, db] and t <= max(fl(N*fl(1/da)),
// fl(N*fl(1/db))) with N = fl(fl(wm[w] - hf) - hl) (monotone rounding); if
// that is below lo no target of the block is a record or a band target.
__device__ int exact_pov(const float* row, const float* wm, const float* ivt, int x, int sg, int D,
                         double h, bool force_exact, uint8_t* vis) {
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
#ifdef SKS_EXP_BANDHIST
  S.first_band = -1;
  S.gap = 0;
  S.blk_before = S.blk_after = 0;
#endif
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
  if (vis != nullptr || wm == nullptr) {
    for (int dd = 1; dd <= D; ++dd) {
      const bool above = exact_step(S, row, x, sg, dd, row[x + sg * dd], ivt[dd]);
      if (vis) vis[dd - 1] = above ? 1 : 0;
    }
    return S.cv;
  }
  if (D < 1) return 0;
  // position blocks in scan order, the window maxima of kWm blocks loaded
  // together (one L2 round trip per kWm blocks); candidates are re-tested
  // against lo as raised by the blocks evaluated since (it only rises)
  const int pfirst = x + sg, plast = x + sg * D;
  const int w0 = pfirst >> 4, w1 = plast >> 4;
  const int nblk = (w1 - w0) * sg + 1;
#ifndef SKS_FIX_WM
#define SKS_FIX_WM 8
#endif
  constexpr int kWm = SKS_FIX_WM;
  // block b (scan order) is w = w0 + sg*b and its first target has
  // dd = c0 + 16b (partial at the ends: da = max(1, .), db = min(D, .))
  const int c0 = sg > 0 ? 16 * w0 - x : x - 16 * w0 - 15;
  for (int b0 = 0; b0 < nblk; b0 += kWm) {
    const int df = c0 + 16 * b0;
    float wv[kWm];
#pragma unroll
    for (int u = 0; u < kWm; ++u) wv[u] = b0 + u < nblk ? __ldg(wm + w0 + sg * (b0 + u)) : -INFINITY;
#if SKS_FIX_COARSE
    {
      // the kWm blocks at once: the same bound over their whole dd span
      // with the maximum of their maxima (monotone rounding, both signs of N)
      float m = wv[0];
#pragma unroll
      for (int u = 1; u < kWm; ++u) m = fmaxf(m, wv[u]);
      const int da = max(1, df), db = min(D, df + 16 * kWm - 1);
      const float N = __fadd_rn(__fsub_rn(m, S.hf), -S.hl);
      if (__fmul_rn(N, ivt[da]) < S.lo && __fmul_rn(N, ivt[db]) < S.lo) continue;
    }
#endif
    unsigned cand = 0;
#pragma unroll
    for (int u = 0; u < kWm; ++u) {
      const int d0 = df + 16 * u;
      const int da = max(1, d0), db = min(D, d0 + 15);
      const float N = __fadd_rn(__fsub_rn(wv[u], S.hf), -S.hl);
      if (d0 <= D && !(__fmul_rn(N, ivt[da]) < S.lo && __fmul_rn(N, ivt[db]) < S.lo)) cand |= 1u << u;
    }
    while (cand != 0) {
      const int u = __ffs(cand) - 1;
      cand &= cand - 1;
      const int w = w0 + sg * (b0 + u);
      const int d0 = df + 16 * u;
      const int da = max(1, d0), db = min(D, d0 + 15);
      const float N = __fadd_rn(__fsub_rn(__ldg(wm + w), S.hf), -S.hl);  // L1 hit
      if (!(__fmul_rn(N, ivt[da]) < S.lo && __fmul_rn(N, ivt[db]) < S.lo)) {
#ifdef SKS_EXP_BANDHIST
        if (S.first_band < 0) ++S.blk_before; else ++S.blk_after;
#endif
#if SKS_FIX_FULL16
        if (!eval16(S, row, ivt, w, sg, d0, da, db)) eval_block(S, row, ivt, x, sg, da, db);
#else
        eval_block(S, row, ivt, x, sg, da, db);
#endif
      }
    }
  }
#ifdef SKS_EXP_BANDHIST
  {
    auto lg = [](int v) { int b = 0; while (v > 1 && b < 15) { v >>= 1; ++b; } return b; };
    atomicAdd(&g_bandhist[44], 1ull);
    if (S.first_band < 0) {
      atomicAdd(&g_bandhist[45], 1ull);
    } else {
      atomicAdd(&g_bandhist[min(9, static_cast<int>(10.0 * S.first_band / (D + 1)))], 1ull);
      atomicAdd(&g_bandhist[10 + lg(S.first_band)], 1ull);
      atomicAdd(&g_bandhist[26 + lg(S.gap + 1)], 1ull);
    }
    atomicAdd(&g_bandhist[42], static_cast<unsigned long long>(S.blk_before));
    atomicAdd(&g_bandhist[43], static_cast<unsigned long long>(S.blk_after));
  }
#endif
  return S.cv;
}

// Exclusive prefix of the queued POVs per scan item: off[it] = sum over
// items < it of fix_cnt * group, off[n_items] = total. Two fully parallel
// passes over contiguous item chunks (coalesced): block sums, then each
// block rescans its chunk from the sum of the blocks before it.
constexpr int kPrefixThreads = 1024;

__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned* warp_tot, unsigned* total) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  unsigned incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) warp_tot[wp] = incl;
  __syncthreads();
  if (wp == 0) {
    const unsigned ws = lane < (blockDim.x >> 5) ? warp_tot[lane] : 0u;
    unsigned wi = ws;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += u;
    }
    warp_tot[lane] = wi - ws;
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  const unsigned r = warp_tot[wp] + incl - v;
  __syncthreads();  // warp_tot / total reusable
  return r;
}

__global__ void __launch_bounds__(kPrefixThreads) fixup_prefix_sums_kernel(ScanArgs a, int chunk, unsigned* bsum) {
  __shared__ unsigned wt[32];
  __shared__ unsigned tot;
  const int b0 = blockIdx.x * chunk, b1 = min(a.n_items, b0 + chunk);
  unsigned local = 0;
  for (int i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const unsigned c = __ldg(a.fix_cnt + i);  // forward | backward << 16
    local += (c & 0xffffu) + (c >> 16);
  }
  block_excl_scan(local, wt, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot * static_cast<unsigned>(a.fix_group);
}

__global__ void __launch_bounds__(kPrefixThreads) fixup_prefix_write_kernel(ScanArgs a, int chunk, const unsigned* bsum,
                                                                           unsigned* off) {
  __shared__ unsigned wt[32];
  __shared__ unsigned tot;
  __shared__ unsigned base_s;
  if (threadIdx.x < 32) {
    unsigned b = 0;
    for (int k = threadIdx.x; k < static_cast<int>(blockIdx.x); k += 32) b += bsum[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) b += __shfl_down_sync(0xffffffffu, b, o);
    if (threadIdx.x == 0) base_s = b;
  }
  __syncthreads();
  unsigned base = base_s;
  const unsigned grp = static_cast<unsigned>(a.fix_group);
  const int b0 = blockIdx.x * chunk, b1 = min(a.n_items, b0 + chunk);
  for (int t0 = b0; t0 < b1; t0 += blockDim.x) {
    const int i = t0 + threadIdx.x;
    const unsigned c = i < b1 ? __ldg(a.fix_cnt + i) : 0u;
    const unsigned v = ((c & 0xffffu) + (c >> 16)) * grp;
    const unsigned ex = block_excl_scan(v, wt, &tot);
    if (i < b1) off[i] = base + ex;
    base += tot;
    __syncthreads();
  }
  if (b1 == a.n_items && b0 < b1 && threadIdx.x == 0) off[a.n_items] = base;
}

// One thread per queued POV (flat list over all rows, in row order, so
// neighbouring threads share rows): the POV's row is found by a binary search
// of the prefix, then the POV is re-run exactly (exact_pov). Rows are read
// through L1/L2; the fl(1/d) table sits in shared memory (kSmemTab), or in
// global memory for batches with rows too long for it (long rows).
#ifndef SKS_FIX_MINB
#define SKS_FIX_MINB 3  // 24 warps per SM (80 registers): the kernel is latency-bound
#endif
template <bool kSmemTab>
__global__ void __launch_bounds__(kWarps * 32, SKS_FIX_MINB) fixup_kernel(ScanArgs a, int tab_len, const unsigned* off) {
  extern __shared__ __align__(16) float ivt_s[];  // fl(1/d), d = 0 .. tab_len - 1
  if (kSmemTab) {
    for (int d = threadIdx.x; d < tab_len; d += blockDim.x) ivt_s[d] = __frcp_rn(static_cast<float>(d));
    __syncthreads();
  }
  const float* ivt = kSmemTab ? ivt_s : a.ivt;
  const unsigned grp = static_cast<unsigned>(a.fix_group);
  const unsigned total = off[a.n_items];
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned w = blockIdx.x * blockDim.x + threadIdx.x; w < total; w += stride) {
    // item: the last it with off[it] <= w
    int lo = 0, hi = a.n_items;  // off[lo] <= w < off[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(off + mid) <= w) lo = mid; else hi = mid;
    }
    const int it = lo;
    const unsigned wj = w - __ldg(off + it);
    const ScanItem item = a.items[it];
    const SectorDev& sd = a.b.sectors[item.s];
    const int2 rg = a.b.ranges[sd.row_off + item.q];
    const int first = rg.x;
    const int L = rg.y - rg.x;
    const long long rowoff = sd.sdem_off + static_cast<long long>(item.q) * sd.pitch;
    const float* row = a.b.sdem + rowoff + first;
    // forward entries at the segment start, backward ones from slot L
    const unsigned nf = __ldg(a.fix_cnt + it) & 0xffffu;
    const unsigned e = wj / grp;
    const unsigned ent = a.fix_queue[a.fix_off[it] + (e < nf ? e : static_cast<unsigned>(L) + (e - nf))];
    const int dir = static_cast<int>(ent >> 31);
    const int y = static_cast<int>((ent & 0x7fffffffu) * grp + wj % grp);
    if (y >= L) continue;
    const int x = dir ? (L - 1 - y) : y;
    const int D = min(sd.max_dd, dir ? x : (L - 1 - x));
    const bool dbg = a.dbg_j0 >= 0 && item.s == 0 && item.q == 0 && first + x == a.dbg_j0;
    const double h = dbg ? a.dbg_h : __dadd_rn(static_cast<double>(row[x]), a.h0);
    uint8_t* vis = dbg ? (dir ? a.dbg_vis_bwd : a.dbg_vis_fwd) : nullptr;
    const float* wm = a.wm16 != nullptr ? a.wm16 + rowoff / 16 : nullptr;
    const int cv = exact_pov(row, wm, ivt, x, dir ? -1 : 1, D, h, a.force_exact != 0, vis);
    if (cv != 0) {
      int* dst = ((dir && a.b.cv_bwd) ? a.b.cv_bwd : a.b.cv) + rowoff + first;
      atomicAdd(dst + x, cv);
    }
  }
}

// ---------------------------------------------------------------------------
// Warp-per-POV fixup (opt-in, SKS_FIXUP=warp; measured 2-3x slower than the
// thread-per-POV kernel: config 2 fixup 3.79 vs 1.79 ms, config 4 65.9 vs
// 30.1 ms, config 5 5.88 vs 2.01 s — each 32-target step is a chain of
// shuffles plus an L2 round trip, and 32 warps per SM keep too few steps in
// flight; the thread kernel's 512 independent POVs per SM hide the latency
// better). The thread-per-POV kernel above keeps 512
// POVs in flight per SM but its lanes diverge: each POV skips its own blocks,
// so only ~11 of 32 lanes are busy in eval_block (ncu, round 1), and its cost
// grows with the row length (config 5: 32 % of the step). Here a warp takes
// one POV and walks its targets 32 at a time:
//   * skip: each lane tests one 16-target window of the next 32 (512 targets)
//     with the same exact bound as exact_pov; candidates are re-tested
//     against lo as it rises and evaluated two windows per step;
//   * step: lane i holds target i of the step (in scan order) and computes
//     the certified FP32 t; the state before lane i is R_i = max(R, t of the
//     lanes before i) (the FP32 value of the last record when every earlier
//     decision was certain: a record's t exceeds the previous hi, a hidden
//     target's t lies below lo), an exclusive warp max-scan; record if
//     t > hi(R_i), hidden if t < lo(R_i), else the first such band lane is
//     decided with the reference's FP64 operations against the exact max
//     (theta of the last record, computed lazily) and the lanes after it are
//     re-run from the resolved state.
// Every decision that reaches cv is the reference's (scan.cpp:24-34), as in
// exact_pov; POVs whose h does not split run the FP64 recurrence with an FP64
// warp max-scan.
__device__ __forceinline__ float warp_excl_max(float v, int lane) {
  float incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = fmaxf(incl, u);
  }
  const float ex = __shfl_up_sync(0xffffffffu, incl, 1);
  return lane == 0 ? -INFINITY : ex;
}

__device__ __forceinline__ double warp_excl_max_d(double v, int lane) {
  double incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = fmax(incl, u);
  }
  const double ex = __shfl_up_sync(0xffffffffu, incl, 1);
  return lane == 0 ? -INFINITY : ex;
}

struct WarpState {
  float hf, hl;
  double h;
  float R;        // FP32 t of the last record (-inf: none yet)
  int r;          // its dd (0: none)
  double M;       // exact max theta when Mvalid
  bool Mvalid;
  int cv;         // this lane's share of the ring sum
};

__device__ __forceinline__ float lo_of(float R) { return R == -INFINITY ? -FLT_MAX : __fmaf_rn(fabsf(R), -kBand, R); }

// One step: lane i holds target dd (valid: act), elevation e, certified t.
__device__ __forceinline__ void warp_step(WarpState& S, const float* row, int x, int sg, bool act, int dd, float e,
                                          float t, int lane) {
  int start = 0;
  for (;;) {
    const bool mine = act && lane >= start;
    const float Ri = fmaxf(S.R, warp_excl_max(mine ? t : -INFINITY, lane));
    bool rec, band;
    if (Ri == -INFINITY) {
      rec = mine;  // nothing seen yet: every finite target is above -inf
      band = false;
    } else {
      const float at = fabsf(Ri);
      rec = mine && t > __fmaf_rn(at, kBand, Ri);
      band = mine && !rec && t >= __fmaf_rn(at, -kBand, Ri);
    }
    const unsigned bm = __ballot_sync(0xffffffffu, band);
    const int stop = bm ? __ffs(bm) - 1 : 32;
    const bool take = rec && lane < stop;
    const unsigned rm = __ballot_sync(0xffffffffu, take);
    if (take) S.cv += 2 * dd + 1;
    if (rm) {
      const int last = 31 - __clz(rm);
      S.R = __shfl_sync(0xffffffffu, t, last);
      S.r = __shfl_sync(0xffffffffu, dd, last);
      S.Mvalid = false;
    }
    if (stop == 32) return;
    // the first band target, decided exactly (scan.cpp:24-25): theta against
    // the exact running max, theta of the last record r
    const float eb = __shfl_sync(0xffffffffu, e, stop);
    const int db = __shfl_sync(0xffffffffu, dd, stop);
    const float tb = __shfl_sync(0xffffffffu, t, stop);
    const double th = __ddiv_rn(__dsub_rn(static_cast<double>(eb), S.h), static_cast<double>(db));
    if (!S.Mvalid) {
      S.M = S.r == 0 ? -INFINITY
                     : __ddiv_rn(__dsub_rn(static_cast<double>(__ldg(row + x + sg * S.r)), S.h),
                                 static_cast<double>(S.r));
      S.Mvalid = true;
    }
    if (th > S.M) {
      if (lane == stop) S.cv += 2 * db + 1;
      S.M = th;
      S.R = tb;
      S.r = db;
    }
    start = stop + 1;
  }
}

// cv of one POV (every lane returns the same value).
__device__ int warp_pov(const float* row, const float* wm, const float* ivt, int x, int sg, int D, double h,
                        bool force_exact, int lane) {
  WarpState S;
  S.h = h;
  S.hf = __double2float_rn(h);
  const double hld = __dsub_rn(h, static_cast<double>(S.hf));
  S.hl = __double2float_rn(hld);
  S.R = -INFINITY;
  S.r = 0;
  S.M = -INFINITY;
  S.Mvalid = true;
  S.cv = 0;
  if (D < 1) return 0;
  const bool exact_all = force_exact || static_cast<double>(S.hl) != hld || !(fabsf(S.hf) < 1e30f);
  if (exact_all || wm == nullptr) {
    // the FP64 recurrence, 32 targets per step (an FP64 max-scan)
    double M = -INFINITY;
    int cv = 0;
    for (int d0 = 1; d0 <= D; d0 += 32) {
      const int dd = d0 + lane;
      const bool act = dd <= D;
      const double th = act ? __ddiv_rn(__dsub_rn(static_cast<double>(__ldg(row + x + sg * dd)), h),
                                        static_cast<double>(dd))
                            : -INFINITY;
      const double Mi = fmax(M, warp_excl_max_d(th, lane));
      if (act && th > Mi) cv += 2 * dd + 1;
      M = fmax(Mi, th);
      M = __shfl_sync(0xffffffffu, M, 31);
    }
    return __reduce_add_sync(0xffffffffu, cv);
  }
  // 16-target windows in scan order (row positions 16w .. 16w+15)
  const int pfirst = x + sg, plast = x + sg * D;
  const int w0 = pfirst >> 4, w1 = plast >> 4;
  const int nblk = (w1 - w0) * sg + 1;
  for (int b0 = 0; b0 < nblk; b0 += 32) {
    const int j = b0 + lane;
    const bool valid = j < nblk;
    float B = INFINITY;  // max slope bound of window j (+inf: not a window)
    if (valid) {
      const int w = w0 + sg * j;
      const int da = max(1, sg > 0 ? 16 * w - x : x - (16 * w + 15));
      const int db = min(D, sg > 0 ? 16 * w + 15 - x : x - 16 * w);
      const float N = __fadd_rn(__fsub_rn(__ldg(wm + w), S.hf), -S.hl);
      B = fmaxf(__fmul_rn(N, ivt[da]), __fmul_rn(N, ivt[db]));
    }
    unsigned pend = __ballot_sync(0xffffffffu, valid);
    for (;;) {
      // candidates against the current lo (it only rises: re-tested each step)
      const unsigned cand = __ballot_sync(0xffffffffu, !(B < lo_of(S.R))) & pend;
      if (cand == 0) break;
      const int ja = __ffs(cand) - 1;
      const unsigned rest = cand & (cand - 1);
      const int jb = rest ? __ffs(rest) - 1 : -1;
      pend &= ~(1u << ja);
      if (jb >= 0) pend &= ~(1u << jb);
      // lanes 0-15: window ja, 16-31: window jb (scan order within each)
      const int jj = lane < 16 ? ja : jb;
      const int w = w0 + sg * (b0 + jj);
      const int pos = sg > 0 ? 16 * w + (lane & 15) : 16 * w + 15 - (lane & 15);
      const int dd = sg * (pos - x);
      const bool act = jj >= 0 && dd >= 1 && dd <= D;
      const float e = act ? __ldg(row + pos) : 0.f;
      const float t = act ? __fmul_rn(__fadd_rn(__fsub_rn(e, S.hf), -S.hl), ivt[dd]) : -INFINITY;
      warp_step(S, row, x, sg, act, dd, e, t, lane);
    }
  }
  return __reduce_add_sync(0xffffffffu, S.cv);
}

// the sequential form for the debug POV (outlined: keeps the warp kernel's registers)
__device__ __noinline__ int exact_pov_dbg(const float* row, const float* wm, const float* ivt, int x, int sg, int D,
                                          double h, bool force_exact, uint8_t* vis) {
  return exact_pov(row, wm, ivt, x, sg, D, h, force_exact, vis);
}

#ifndef SKS_FIXW_MINB
#define SKS_FIXW_MINB 4
#endif
template <bool kSmemTab>
__global__ void __launch_bounds__(kWarps * 32, SKS_FIXW_MINB) fixup_warp_kernel(ScanArgs a, int tab_len,
                                                                              const unsigned* off) {
  extern __shared__ __align__(16) float ivt_s[];  // fl(1/d), d = 0 .. tab_len - 1
  if (kSmemTab) {
    for (int d = threadIdx.x; d < tab_len; d += blockDim.x) ivt_s[d] = __frcp_rn(static_cast<float>(d));
    __syncthreads();
  }
  const float* ivt = kSmemTab ? ivt_s : a.ivt;
  const int lane = threadIdx.x & 31;
  const unsigned grp = static_cast<unsigned>(a.fix_group);
  const unsigned total = off[a.n_items];
  const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
  for (unsigned w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total; w += nwarps) {
    // item: the last it with off[it] <= w (warp-uniform)
    int lo = 0, hi = a.n_items;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(off + mid) <= w) lo = mid; else hi = mid;
    }
    const int it = lo;
    const unsigned wj = w - __ldg(off + it);
    const ScanItem item = a.items[it];
    const SectorDev& sd = a.b.sectors[item.s];
    const int2 rg = a.b.ranges[sd.row_off + item.q];
    const int first = rg.x;
    const int L = rg.y - rg.x;
    const long long rowoff = sd.sdem_off + static_cast<long long>(item.q) * sd.pitch;
    const float* row = a.b.sdem + rowoff + first;
    const unsigned nf = __ldg(a.fix_cnt + it) & 0xffffu;
    const unsigned e = wj / grp;
    const unsigned ent = a.fix_queue[a.fix_off[it] + (e < nf ? e : static_cast<unsigned>(L) + (e - nf))];
    const int dir = static_cast<int>(ent >> 31);
    const int y = static_cast<int>((ent & 0x7fffffffu) * grp + wj % grp);
    if (y >= L) continue;
    const int x = dir ? (L - 1 - y) : y;
    const int D = min(sd.max_dd, dir ? x : (L - 1 - x));
    const bool dbg = a.dbg_j0 >= 0 && item.s == 0 && item.q == 0 && first + x == a.dbg_j0;
    const double h = dbg ? a.dbg_h : __dadd_rn(static_cast<double>(row[x]), a.h0);
    const float* wm = a.wm16 != nullptr ? a.wm16 + rowoff / 16 : nullptr;
    int cv;
    if (dbg) {
      // debug capture of the per-target decisions: the sequential form
      cv = 0;
      if (lane == 0) {
        cv = exact_pov_dbg(row, wm, ivt, x, dir ? -1 : 1, D, h, a.force_exact != 0,
                           dir ? a.dbg_vis_bwd : a.dbg_vis_fwd);
      }
      cv = __shfl_sync(0xffffffffu, cv, 0);
    } else {
      cv = warp_pov(row, wm, ivt, x, dir ? -1 : 1, D, h, a.force_exact != 0, lane);
    }
    if (lane == 0 && cv != 0) {
      int* dst = ((dir && a.b.cv_bwd) ? a.b.cv_bwd : a.b.cv) + rowoff + first;
      atomicAdd(dst + x, cv);
    }
  }
}

// Long rows (items [0, n_long)): one CTA per row writes the row's 16-cell
// window maxima (what scan2's row loader writes for the rows it scans) and
// queues every POV in both directions (forward entries y = 0 .. L-1 at the
// segment start, backward ones from slot L, as scan2 queues flagged POVs).
__global__ void __launch_bounds__(256) long_rows_kernel(ScanArgs a) {
  const int it = blockIdx.x;
  const ScanItem item = a.items[it];
  const SectorDev& sd = a.b.sectors[item.s];
  const int2 rg = a.b.ranges[sd.row_off + item.q];
  const int L = rg.y - rg.x;
  const long long rowoff = sd.sdem_off + static_cast<long long>(item.q) * sd.pitch;
  const float* row = a.b.sdem + rowoff + rg.x;
  float* wm = a.wm16 + rowoff / 16;
  for (int w = threadIdx.x; 16 * w < L; w += blockDim.x) {
    float m = -INFINITY;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (16 * w + u < L) m = fmaxf(m, __ldg(row + 16 * w + u));
    }
    wm[w] = m;
  }
  unsigned* q = a.fix_queue + a.fix_off[it];
  for (int y = threadIdx.x; y < L; y += blockDim.x) {
    q[y] = pack_fix(0u, static_cast<unsigned>(y));
    q[L + y] = pack_fix(1u, static_cast<unsigned>(y));
  }
  if (threadIdx.x == 0) {
    a.fix_cnt[it] = static_cast<unsigned>(L) | (static_cast<unsigned>(L) << 16);
    atomicAdd(a.fix_count, 2u * static_cast<unsigned>(L));
  }
}

__global__ void ivt_table_kernel(float* ivt, int n) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < n) ivt[d] = __frcp_rn(static_cast<float>(d));
}

// fl(1/d) tables up to this many entries live in shared memory (64 KB)
constexpr int kSmemTabMax = 16384;

}  // namespace

int launch_fixup(const ScanArgs& a, unsigned* off, void* stream) {
  if (a.n_items == 0) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  {
    // off[] has n_items + 1 slots plus room for the block sums after them
    const int nb = std::max(1, std::min(sms, (a.n_items + kPrefixThreads - 1) / kPrefixThreads));
    const int chunk = (a.n_items + nb - 1) / nb;
    unsigned* bsum = off + a.n_items + 1;
    fixup_prefix_sums_kernel<<<nb, kPrefixThreads, 0, static_cast<cudaStream_t>(stream)>>>(a, chunk, bsum);
    fixup_prefix_write_kernel<<<nb, kPrefixThreads, 0, static_cast<cudaStream_t>(stream)>>>(a, chunk, bsum, off);
  }
  const int tab_len = ((std::max(a.lmax_all, a.lmax) + 31) / 32) * 32;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  // SKS_FIXUP=warp selects the warp-per-POV kernel (measured slower, kept
  // for experiments)
  const char* fx = std::getenv("SKS_FIXUP");
  const bool thread_kernel = !(fx != nullptr && std::string(fx) == "warp");
  if (!thread_kernel) {
    const bool smem_tab = tab_len <= kSmemTabMax;
    if (!smem_tab && a.ivt == nullptr) return static_cast<int>(cudaErrorInvalidValue);
    const size_t smem = smem_tab ? static_cast<size_t>(tab_len) * sizeof(float) : 0;
    auto kern = smem_tab ? fixup_warp_kernel<true> : fixup_warp_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return static_cast<int>(e);
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem);
    if (e != cudaSuccess) return static_cast<int>(e);
    kern<<<sms * (per_sm > 0 ? per_sm : 1), kWarps * 32, smem, st>>>(a, tab_len, off);
    return static_cast<int>(cudaGetLastError());
  }
  if (tab_len <= kSmemTabMax) {
    const size_t smem = static_cast<size_t>(tab_len) * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(fixup_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return static_cast<int>(e);
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fixup_kernel<true>, kWarps * 32, smem);
    if (e != cudaSuccess) return static_cast<int>(e);
    fixup_kernel<true><<<sms * (per_sm > 0 ? per_sm : 1), kWarps * 32, smem, st>>>(a, tab_len, off);
  } else {
    if (a.ivt == nullptr) return static_cast<int>(cudaErrorInvalidValue);
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fixup_kernel<false>, kWarps * 32, 0);
    if (e != cudaSuccess) return static_cast<int>(e);
    fixup_kernel<false><<<sms * (per_sm > 0 ? per_sm : 1), kWarps * 32, 0, st>>>(a, tab_len, off);
  }
  return static_cast<int>(cudaGetLastError());
}

int launch_long_rows(const ScanArgs& a, int n_long, void* stream) {
  if (n_long <= 0) return 0;
  long_rows_kernel<<<n_long, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return static_cast<int>(cudaGetLastError());
}

int launch_ivt_table(float* ivt, int n, void* stream) {
  ivt_table_kernel<<<(n + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(ivt, n);
  return static_cast<int>(cudaGetLastError());
}

int fixup_smem_table_max() { return kSmemTabMax; }

#ifdef SKS_EXP_BANDHIST
extern "C" int sks_exp_bandhist(unsigned long long* out, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_bandhist, sizeof(g_bandhist));
  if (reset) {
    static const unsigned long long z[64] = {};
    cudaMemcpyToSymbol(g_bandhist, z, sizeof(z));
  }
  return static_cast<int>(e);
}
#endif

}  // namespace sks
