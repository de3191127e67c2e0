// Line-of-sight scan over PAIRS of adjacent skewed rows (sm_100a).
//
// Same decisions as scan2 (reference scan.cpp:8-85 under the certified FP32
// filter; flagged POVs go to the exact fixup), with a
// different lane mapping: a task covers 32 consecutive POV positions y of TWO
// adjacent skewed rows q, q+1 of one sector (one direction); lane l owns
// position y = 32c + l in both rows. Compared with scan2's 64 consecutive
// POVs of one row per task:
//   * the two POVs of a lane share dd = k - y, so one fl(1/dd) pair load
//     serves both (per 4 targets: 2 elevation quads + 2 table pairs instead
//     of 1 quad + 4 pairs);
//   * the warp-uniform hidden-window skip covers a 32-position span (of two
//     correlated rows) instead of 64 positions of one row, and the task
//     triangle (targets that are dead for some POVs of the task) is 32
//     targets long instead of 64;
//   * each lane still runs two independent record chains (one per row), the
//     latency cover that single-POV lanes lose.
// Offline model (fractal 2000^2, sampled long rows): 17 % fewer evaluated
// windows than scan2's mapping; on SmoothedNoise 9 % more (rows differ more
// than neighbouring positions of one row there).
//
// The window maxima of the two rows are stored interleaved as float2
// (m(row b), m(row a)) so one LDS.64 feeds the pair's skip test. The two
// fl(1/dd) table copies are offset by 18 floats mod 32 so that the pair loads
// of even lanes (copy 0) and odd lanes (copy 1) never share a bank.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdint>

#include "sks_device.cuh"
#include "sks_ptx.cuh"

namespace sks {

namespace {

constexpr int kW = 16;        // fine window (targets)
#ifndef SKS3_COARSE
#define SKS3_COARSE 128  // measured (quads, config 2): 32: 54.3 ms scan, 64: 50.2, 128: 49.7, 256: 51.4
#endif
constexpr int kH = SKS3_COARSE;  // coarse window (targets)
#ifndef SKS3_TOP
#define SKS3_TOP 0  // third level (targets, a multiple of kH; 0: two levels)
#endif
constexpr int kTop = SKS3_TOP;
constexpr int kTopN = kTop > 0 ? kTop / kH : 1;  // coarse windows per top window
constexpr int kOff = 128;  // table index offset (dd >= -kOff + 1 addressable)
#ifndef SKS3_THREADS
#define SKS3_THREADS 768
#endif
constexpr int kThreads = SKS3_THREADS;
constexpr int kMaxSlots = 8;
constexpr int kCtlInts = 32;
constexpr float kBand = 5.9604644775390625e-07f;  // 10 * 2^-24
constexpr int kSumShift = 22;
constexpr int kSumMask = (1 << kSumShift) - 1;
constexpr int kCopy1Shift = 18;  // copy 1's bank offset (floats) against copy 0

// kR rows per task group (2: row pairs, 4: row quads); a task covers
// kP = 64 / kR consecutive positions of every row of its group. Lane l owns
// position y = kP c + (l mod kP) of rows 2 ph and 2 ph + 1, ph = l / kP.
template <int kR>
struct Geo {
  static constexpr int kP = 64 / kR;
#ifdef SKS3_NEAR_EXTRA
  static constexpr int kNear = kP + SKS3_NEAR_EXTRA;
#else
  static constexpr int kNear = kP + 16;  // no skip tests in a task's first kNear targets
#endif
};

template <int kR>
struct Layout3 {
  int lb;      // row buffer (floats) per row and direction
  int nw16, nw64, nwt;  // nw64 rounded up to kTopN (padding windows are -inf)
  int T;       // table length per copy (floats, a multiple of 32)
  int wpair;   // floats of window maxima per row pair
  int slot;    // floats per slot (kR rows)
  int tables;  // offset of table copy 0
  int slots;   // offset of slot 0
  __host__ __device__ explicit Layout3(int lmax) {
    lb = ((lmax + kH + kH - 1) / kH) * kH;
    nw16 = lb / kW;
    nw64 = ((lb / kH + kTopN - 1) / kTopN) * kTopN;
    nwt = kTop > 0 ? nw64 / kTopN : 0;
    T = ((kOff + lb + 16 + 31) / 32) * 32;
    wpair = 4 * nw16 + 4 * nw64 + 4 * nwt;
    slot = 2 * kR * lb + (kR / 2) * wpair;
    tables = kMaxSlots * kCtlInts;
    slots = tables + 2 * T + kCopy1Shift + 14;  // 14: keeps the slots 16-byte aligned
  }
  __host__ __device__ int copy(int r) const { return tables + r * (T + kCopy1Shift); }
  __host__ __device__ int total(int nslots) const { return slots + nslots * slot; }
};

// control block of one slot (ints): per row r < kR: L, first, item
enum : int { kWord = 0, kRemaining, kDead, kS, kQ0, kCap, kRowL = 8, kRowFirst = 12, kRowItem = 16 };

template <int kR>
struct Slot3 {
  float* S[kR];  // forward copies
  float* R[kR];  // reversed copies
  float2* W16S[kR / 2]; float2* W16R[kR / 2];  // per row pair: (m(row 2ph+1), m(row 2ph)) per window
  float2* W64S[kR / 2]; float2* W64R[kR / 2];
  float2* WTS[kR / 2]; float2* WTR[kR / 2];  // top level (kTop > 0)
};

template <int kR>
__device__ __forceinline__ Slot3<kR> slot_ptrs(float* base, const Layout3<kR>& lay) {
  Slot3<kR> s;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    s.S[r] = base + r * lay.lb;
    s.R[r] = base + (kR + r) * lay.lb;
  }
#pragma unroll
  for (int ph = 0; ph < kR / 2; ++ph) {
    float2* w = reinterpret_cast<float2*>(base + 2 * kR * lay.lb + ph * lay.wpair);
    s.W16S[ph] = w;
    s.W16R[ph] = w + lay.nw16;
    s.W64S[ph] = w + 2 * lay.nw16;
    s.W64R[ph] = w + 2 * lay.nw16 + lay.nw64;
    s.WTS[ph] = w + 2 * lay.nw16 + 2 * lay.nw64;
    s.WTR[ph] = w + 2 * lay.nw16 + 2 * lay.nw64 + lay.nwt;
  }
  return s;
}

// Loads the next row group (longest first) into slot `base`; one warp.
template <int kR>
__device__ void load_group(const ScanArgs& a, int* ctl, float* base, const Layout3<kR>& lay, int lane) {
  int it = 0;
  if (lane == 0) it = static_cast<int>(atomicAdd(a.item_counter, 1u));
  it = __shfl_sync(0xffffffffu, it, 0);
  if (it >= a.n_pairs) {
    if (lane == 0) atomicExch(ctl + kDead, 1);
    return;
  }
  const int4 gi = a.pairs[it];  // items of rows q0 .. q0 + kR - 1 (-1: not scanned)
  const int its[4] = {gi.x, gi.y, gi.z, gi.w};
  int s = 0, q0 = 0;
#pragma unroll
  for (int r = kR - 1; r >= 0; --r) {
    if (its[r] >= 0) {
      const ScanItem item = a.items[its[r]];
      s = item.s;
      q0 = item.q - r;
    }
  }
  const SectorDev& sd = a.b.sectors[s];
  const Slot3<kR> sp = slot_ptrs<kR>(base, lay);
  const float ninf = -INFINITY;
  int Ls[kR], firsts[kR];
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    float* S = sp.S[r];
    float* R = sp.R[r];
    Ls[r] = 0;
    firsts[r] = 0;
    if (its[r] < 0) {
      for (int x = lane; x < lay.lb; x += 32) S[x] = R[x] = ninf;
      continue;
    }
    const int2 rg = a.b.ranges[sd.row_off + q0 + r];
    const int L = rg.y - rg.x;
    Ls[r] = L;
    firsts[r] = rg.x;
    const float* src = a.b.sdem + sd.sdem_off + static_cast<long long>(q0 + r) * sd.pitch + rg.x;
#pragma unroll 4
    for (int x = lane; x < lay.lb; x += 32) S[x] = x < L ? __ldg(src + x) : ninf;
    __syncwarp();
    for (int x = lane; x < lay.lb; x += 32) R[x] = x < L ? S[L - 1 - x] : ninf;
  }
  __syncwarp();
  // window maxima per row pair, interleaved (row 2ph+1, row 2ph); the 16-cell
  // forward maxima of each row also go to wm16 for the fixup's per-POV skip
#pragma unroll
  for (int ph = 0; ph < kR / 2; ++ph) {
    const unsigned sa0 = smem_u32(sp.S[2 * ph]), sa1 = smem_u32(sp.S[2 * ph + 1]);
    const unsigned ra0 = smem_u32(sp.R[2 * ph]), ra1 = smem_u32(sp.R[2 * ph + 1]);
    for (int w = lane; w < lay.nw16; w += 32) {
      float ms0 = -INFINITY, ms1 = -INFINITY, mr0 = -INFINITY, mr1 = -INFINITY;
#pragma unroll
      for (int u = 0; u < kW / 4; ++u) {
        const unsigned o = 4 * kW * w + 16 * u;
        const float4 a0 = lds128(sa0 + o), a1 = lds128(sa1 + o);
        const float4 b0 = lds128(ra0 + o), b1 = lds128(ra1 + o);
        ms0 = fmaxf(ms0, fmaxf(fmaxf(a0.x, a0.y), fmaxf(a0.z, a0.w)));
        ms1 = fmaxf(ms1, fmaxf(fmaxf(a1.x, a1.y), fmaxf(a1.z, a1.w)));
        mr0 = fmaxf(mr0, fmaxf(fmaxf(b0.x, b0.y), fmaxf(b0.z, b0.w)));
        mr1 = fmaxf(mr1, fmaxf(fmaxf(b1.x, b1.y), fmaxf(b1.z, b1.w)));
      }
      sp.W16S[ph][w] = make_float2(ms1, ms0);
      sp.W16R[ph][w] = make_float2(mr1, mr0);
      if (a.wm16 != nullptr) {
        const long long r0 = sd.sdem_off + static_cast<long long>(q0 + 2 * ph) * sd.pitch;
        if (16 * w < Ls[2 * ph]) a.wm16[r0 / 16 + w] = ms0;
        if (16 * w < Ls[2 * ph + 1]) a.wm16[(r0 + sd.pitch) / 16 + w] = ms1;
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int ph = 0; ph < kR / 2; ++ph) {
    for (int w = lane; w < lay.nw64; w += 32) {
      float2 ms = make_float2(-INFINITY, -INFINITY), mr = make_float2(-INFINITY, -INFINITY);
      if ((kH / kW) * w < lay.nw16) {
#pragma unroll
        for (int u = 0; u < kH / kW; ++u) {
          const float2 s2 = sp.W16S[ph][(kH / kW) * w + u], r2 = sp.W16R[ph][(kH / kW) * w + u];
          ms = make_float2(fmaxf(ms.x, s2.x), fmaxf(ms.y, s2.y));
          mr = make_float2(fmaxf(mr.x, r2.x), fmaxf(mr.y, r2.y));
        }
      }
      sp.W64S[ph][w] = ms;
      sp.W64R[ph][w] = mr;
    }
  }
  __syncwarp();
  if (kTop > 0) {
#pragma unroll
    for (int ph = 0; ph < kR / 2; ++ph) {
      for (int w = lane; w < lay.nwt; w += 32) {
        float2 ms = make_float2(-INFINITY, -INFINITY), mr = make_float2(-INFINITY, -INFINITY);
#pragma unroll
        for (int u = 0; u < kTopN; ++u) {
          const float2 s2 = sp.W64S[ph][kTopN * w + u], r2 = sp.W64R[ph][kTopN * w + u];
          ms = make_float2(fmaxf(ms.x, s2.x), fmaxf(ms.y, s2.y));
          mr = make_float2(fmaxf(mr.x, r2.x), fmaxf(mr.y, r2.y));
        }
        sp.WTS[ph][w] = ms;
        sp.WTR[ph][w] = mr;
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    int L = 0;
#pragma unroll
    for (int r = 0; r < kR; ++r) L = max(L, Ls[r]);
    const int ntasks = 2 * ((L + Geo<kR>::kP - 1) / Geo<kR>::kP);
    volatile int* v = ctl;
    v[kS] = s;
    v[kQ0] = q0;
    v[kCap] = sd.max_dd;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      v[kRowL + r] = Ls[r];
      v[kRowFirst + r] = firsts[r];
      v[kRowItem + r] = its[r];
    }
    __threadfence_block();
    atomicExch(ctl + kRemaining, ntasks);
    __threadfence_block();
    atomicExch(reinterpret_cast<unsigned*>(ctl + kWord), static_cast<unsigned>(ntasks) << 16);
  }
  __syncwarp();
}

// Per-lane state: POV 0 = row a at y, POV 1 = row b at y.
struct PovP {
  int y;
  bool v0, v1;
  float hf0, hf1, hl0, hl1;
  float hi0, hi1, lo0, lo1;
  int A0[4], A1[4];
  float G0, G1;
  int cv0, cv1;
  unsigned flag0, flag1;
};

__device__ __forceinline__ void flush(PovP& P) {
  int n0 = 0, n1 = 0, s0 = 0, s1 = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c0 = P.A0[i] >> kSumShift, c1 = P.A1[i] >> kSumShift;
    n0 += c0;
    n1 += c1;
    s0 += (P.A0[i] & kSumMask) + i * c0;
    s1 += (P.A1[i] & kSumMask) + i * c1;
    P.A0[i] = 0;
    P.A1[i] = 0;
  }
  if (__float2int_rn(P.G0) != n0) P.flag0 = 1u;
  if (__float2int_rn(P.G1) != n1) P.flag1 = 1u;
  P.cv0 += 2 * s0 - (2 * P.y - 1) * n0;
  P.cv1 += 2 * s1 - (2 * P.y - 1) * n1;
  P.G0 = 0.f;
  P.G1 = 0.f;
}

// one target of one POV, as scan2's step (scan.cpp:24-34 under the filter)
__device__ __forceinline__ void step(float t, float& hi, float& lo, int& A, float& G, int kb) {
  asm("{\n\t.reg .pred pa, pg;\n\t.reg .f32 at;\n\t"
      "setp.gt.f32 pa, %4, %0;\n\t"
      "setp.ge.f32 pg, %4, %1;\n\t"
      "abs.f32 at, %4;\n\t"
      "@pa fma.rn.f32 %0, at, %6, %4;\n\t"
      "@pa fma.rn.f32 %1, at, %7, %4;\n\t"
      "@pa add.s32 %2, %2, %5;\n\t"
      "@pg add.rn.f32 %3, %3, 0f3F800000;\n\t}"
      : "+f"(hi), "+f"(lo), "+r"(A), "+f"(G)
      : "f"(t), "r"(kb), "f"(kBand), "f"(-kBand));
}

__device__ __forceinline__ bool step_vis(float t, float& hi, float& lo, int& A, float& G, int kb) {
  const bool pa = t > hi;
  const bool pg = t >= lo;
  if (pa) {
    const float at = fabsf(t);
    hi = __fmaf_rn(at, kBand, t);
    lo = __fmaf_rn(at, -kBand, t);
    A += kb;
  }
  if (pg) G = __fadd_rn(G, 1.0f);
  return pa;
}

// Skip test for window [k0, k0 + w): both POVs share dl = k0 - y (clamped to
// 1 by the table's NaN for d <= 0: such a window never passes) and
// dh + 1 = k0 + w - y. em2 = (m_b, m_a). Every t of the window is <= B =
// max(fl(N fl(1/dl)), fl(N fl(1/(dh+1)))) per POV (monotone rounding, both
// signs of N).
template <bool kHl>
__device__ __forceinline__ bool window_hidden(const PovP& P, float2 em2, unsigned tb, int k0, int w) {
  float2 N = __fadd2_rn(em2, make_float2(-P.hf1, -P.hf0));
  if (kHl) N = __fadd2_rn(N, make_float2(-P.hl1, -P.hl0));
  const unsigned ra = tb + 4u * static_cast<unsigned>(k0);
  const float i1 = lds32(ra), i2 = lds32(ra + 4u * static_cast<unsigned>(w));
  const float2 b1 = __fmul2_rn(N, make_float2(i1, i1));
  const float2 b2 = __fmul2_rn(N, make_float2(i2, i2));
  const bool ok = (b1.x < P.lo1) & (b2.x < P.lo1) & (b1.y < P.lo0) & (b2.y < P.lo0);
  return __all_sync(0xffffffffu, ok);
}

// targets k0 .. k0+15 for both POVs; sa/sb: the two rows' buffers; ivb: the
// lane's table copy (dd = k - y shared by both POVs)
template <bool kHl, bool kVis>
__device__ __forceinline__ void eval16(PovP& P, unsigned sa, unsigned sb, unsigned ivb, int k0, int vis_p,
                                       uint8_t* vis, int vis_D) {
#pragma unroll
  for (int g = 0; g < kW / 4; ++g) {
    const int k = k0 + 4 * g;
    const float4 ea = lds128(sa + 4 * k);
    const float4 eb = lds128(sb + 4 * k);
    const float2 qa = lds64(ivb + 4 * k), qb = lds64(ivb + 4 * k + 8);
    float2 n0a = __fadd2_rn(make_float2(ea.x, ea.y), make_float2(-P.hf0, -P.hf0));
    float2 n0b = __fadd2_rn(make_float2(ea.z, ea.w), make_float2(-P.hf0, -P.hf0));
    float2 n1a = __fadd2_rn(make_float2(eb.x, eb.y), make_float2(-P.hf1, -P.hf1));
    float2 n1b = __fadd2_rn(make_float2(eb.z, eb.w), make_float2(-P.hf1, -P.hf1));
    if (kHl) {
      n0a = __fadd2_rn(n0a, make_float2(-P.hl0, -P.hl0));
      n0b = __fadd2_rn(n0b, make_float2(-P.hl0, -P.hl0));
      n1a = __fadd2_rn(n1a, make_float2(-P.hl1, -P.hl1));
      n1b = __fadd2_rn(n1b, make_float2(-P.hl1, -P.hl1));
    }
    const float2 t0a = __fmul2_rn(n0a, qa);
    const float2 t0b = __fmul2_rn(n0b, qb);
    const float2 t1a = __fmul2_rn(n1a, qa);
    const float2 t1b = __fmul2_rn(n1b, qb);
    const float t0[4] = {t0a.x, t0a.y, t0b.x, t0b.y};
    const float t1[4] = {t1a.x, t1a.y, t1b.x, t1b.y};
    const int kb = k + (1 << kSumShift);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (kVis) {
        const bool a0 = step_vis(t0[i], P.hi0, P.lo0, P.A0[i], P.G0, kb);
        const bool a1 = step_vis(t1[i], P.hi1, P.lo1, P.A1[i], P.G1, kb);
        if (vis_p >= 0) {
          const int d = k + i - P.y;
          if (d >= 1 && d <= vis_D) vis[d - 1] = (vis_p == 0 ? a0 : a1) ? 1 : 0;
        }
      } else {
        step(t0[i], P.hi0, P.lo0, P.A0[i], P.G0, kb);
        step(t1[i], P.hi1, P.lo1, P.A1[i], P.G1, kb);
      }
    }
  }
}

// eval16 past kmain of a capped row: target k is a no-op (NaN) for both POVs
// once dd = k - y exceeds the cap (kc = y + cap, the last target).
template <bool kHl>
__device__ __forceinline__ void eval16_capped(PovP& P, unsigned sa, unsigned sb, unsigned ivb, int k0, int kc) {
  const float qn = __int_as_float(0x7fc00000);
#pragma unroll
  for (int g = 0; g < kW / 4; ++g) {
    const int k = k0 + 4 * g;
    const float4 ea = lds128(sa + 4 * k);
    const float4 eb = lds128(sb + 4 * k);
    float2 qa = lds64(ivb + 4 * k), qb = lds64(ivb + 4 * k + 8);
    const int m = kc - k;  // last valid slot index
    qa.x = m >= 0 ? qa.x : qn;
    qa.y = m >= 1 ? qa.y : qn;
    qb.x = m >= 2 ? qb.x : qn;
    qb.y = m >= 3 ? qb.y : qn;
    float2 n0a = __fadd2_rn(make_float2(ea.x, ea.y), make_float2(-P.hf0, -P.hf0));
    float2 n0b = __fadd2_rn(make_float2(ea.z, ea.w), make_float2(-P.hf0, -P.hf0));
    float2 n1a = __fadd2_rn(make_float2(eb.x, eb.y), make_float2(-P.hf1, -P.hf1));
    float2 n1b = __fadd2_rn(make_float2(eb.z, eb.w), make_float2(-P.hf1, -P.hf1));
    if (kHl) {
      n0a = __fadd2_rn(n0a, make_float2(-P.hl0, -P.hl0));
      n0b = __fadd2_rn(n0b, make_float2(-P.hl0, -P.hl0));
      n1a = __fadd2_rn(n1a, make_float2(-P.hl1, -P.hl1));
      n1b = __fadd2_rn(n1b, make_float2(-P.hl1, -P.hl1));
    }
    const float2 t0a = __fmul2_rn(n0a, qa);
    const float2 t0b = __fmul2_rn(n0b, qb);
    const float2 t1a = __fmul2_rn(n1a, qa);
    const float2 t1b = __fmul2_rn(n1b, qb);
    const float t0[4] = {t0a.x, t0a.y, t0b.x, t0b.y};
    const float t1[4] = {t1a.x, t1a.y, t1b.x, t1b.y};
    const int kb = k + (1 << kSumShift);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      step(t0[i], P.hi0, P.lo0, P.A0[i], P.G0, kb);
      step(t1[i], P.hi1, P.lo1, P.A1[i], P.G1, kb);
    }
  }
}

template <int kR, bool kHl, bool kVis, bool kCapped>
__device__ void run_task(const Layout3<kR>& lay, const Slot3<kR>& sl, const float* IV, int dir, int chunk, int L,
                         int cap, int ph, PovP& P, int vis_p, uint8_t* vis, int vis_D,
                         unsigned long long& skipped) {
  const unsigned sa = smem_u32(dir ? sl.R[2 * ph] : sl.S[2 * ph]);
  const unsigned sb = smem_u32(dir ? sl.R[2 * ph + 1] : sl.S[2 * ph + 1]);
  const float2* W16 = dir ? sl.W16R[ph] : sl.W16S[ph];
  const float2* W64 = dir ? sl.W64R[ph] : sl.W64S[ph];
  const unsigned wta = kTop > 0 ? smem_u32(dir ? sl.WTR[ph] : sl.WTS[ph]) : 0u;
  // copy r with (k - y - r) even for k % 4 == 0: r = y & 1; the window
  // tests read copy 0 at element d + kOff
  const int r = P.y & 1;
  const unsigned ivb = smem_u32(IV + lay.copy(r)) + 4u * static_cast<unsigned>(kOff - r - P.y);
  const unsigned tb = smem_u32(IV + lay.copy(0)) + 4u * static_cast<unsigned>(kOff - P.y);
  const unsigned w16a = smem_u32(W16), w64a = smem_u32(W64);
  constexpr int kP = Geo<kR>::kP;
  const int ymin = chunk * kP;
  const bool capped = cap < L - 1;
  const int kmain = capped ? ymin + cap : INT_MAX / 2;
  const int klast = L - 1;
  int k0 = ymin;
  unsigned long long nskip = 0;
  int nev = 0;  // flush after 32 evaluated windows (A stays exact: scan2's bound)
  const int ktest = ymin + Geo<kR>::kNear;
  while (k0 <= klast) {
    // top windows (kTop > 0) and coarse windows where k0 is aligned to them;
    // fine windows up to the next coarse-aligned position
    if (kTop > 0 && !kVis && (k0 & (kTop - 1)) == 0 && k0 >= ktest && k0 + kTop - 1 <= kmain) {
      const float2 em = lds64(wta + 8u * (static_cast<unsigned>(k0) / kTop));
      if (window_hidden<kHl>(P, em, tb, k0, kTop)) {
        k0 += kTop;
        nskip += kTop;
        continue;
      }
    }
    if (!kVis && (k0 & (kH - 1)) == 0 && k0 >= ktest && k0 + kH - 1 <= kmain) {
      const float2 em = lds64(w64a + 8u * (static_cast<unsigned>(k0) / kH));
      if (window_hidden<kHl>(P, em, tb, k0, kH)) {
        k0 += kH;
        nskip += kH;
        continue;
      }
    }
    const int kc = (k0 & ~(kH - 1)) + kH;
    while (k0 < kc && k0 <= klast && k0 + kW - 1 <= kmain) {
      if (!kVis && k0 >= ktest) {
        const float2 em = lds64(w16a + 8u * (static_cast<unsigned>(k0) / kW));
        if (window_hidden<kHl>(P, em, tb, k0, kW)) {
          k0 += kW;
          nskip += kW;
          continue;
        }
      }
      eval16<kHl, kVis>(P, sa, sb, ivb, k0, vis_p, vis, vis_D);
      if (++nev == 32) {
        flush(P);
        nev = 0;
      }
      k0 += kW;
    }
    if (k0 < kc && k0 <= klast) break;  // next window crosses the cap: tail
  }
  flush(P);
  if (kCapped && capped) {
    // masked tail (both POVs share dd, so one mask)
    const int ylast = ymin + kP - 1;
    const int kt_end = min(klast, ylast + cap);
    const int kcap = P.y + cap;
    int cnt = 0;
    for (; k0 <= kt_end; k0 += kW) {
      if (!kVis && k0 >= ktest) {
        const float2 em = lds64(w16a + 8u * (static_cast<unsigned>(k0) / kW));
        if (window_hidden<kHl>(P, em, tb, k0, kW)) {
          nskip += kW;
          continue;
        }
      }
      if (kVis) {
        // debug capture: one target at a time
        const float* IVf = IV + lay.copy(0) + kOff;
        for (int k = k0; k < k0 + kW && k <= kt_end; ++k) {
          const int d = k - P.y;
          const bool m = d >= 1 && d <= cap;
          const float qn = __int_as_float(0x7fc00000);
          const float ivd = m ? IVf[d] : qn;
          const float ea = dir ? sl.R[2 * ph][k] : sl.S[2 * ph][k];
          const float eb = dir ? sl.R[2 * ph + 1][k] : sl.S[2 * ph + 1][k];
          const float t0 = __fmul_rn(__fadd_rn(__fadd_rn(ea, -P.hf0), -P.hl0), ivd);
          const float t1 = __fmul_rn(__fadd_rn(__fadd_rn(eb, -P.hf1), -P.hl1), ivd);
          const int kb = k + (1 << kSumShift);
          const bool a0 = step_vis(t0, P.hi0, P.lo0, P.A0[0], P.G0, kb);
          const bool a1 = step_vis(t1, P.hi1, P.lo1, P.A1[0], P.G1, kb);
          if (vis_p >= 0 && d >= 1 && d <= vis_D) vis[d - 1] = (vis_p == 0 ? a0 : a1) ? 1 : 0;
        }
      } else {
        eval16_capped<kHl>(P, sa, sb, ivb, k0, kcap);
      }
      if (++cnt == (kVis ? 8 : 32)) {
        flush(P);
        cnt = 0;
      }
    }
    flush(P);
  }
  skipped += nskip;
}

template <int kR, bool kCapped>
__global__ void __launch_bounds__(kThreads, 1) scan3_kernel(const __grid_constant__ ScanArgs a, int nslots, int lmax) {
  extern __shared__ __align__(16) float smem[];
  const Layout3<kR> lay(lmax);
  int* ctl_all = reinterpret_cast<int*>(smem);
  float* IV = smem;
  float* slots = smem + lay.slots;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  constexpr int kP = Geo<kR>::kP;
  const int ph = lane / kP;    // row pair of this lane
  const int yl = lane % kP;    // position within the task

  // fl(1/d) tables, 2 copies shifted by r: IV[r][i] = fl(1/(i - kOff + r)),
  // NaN for d <= 0 (a no-op target)
  const float qnan = __int_as_float(0x7fc00000);
  for (int i = tid; i < 2 * lay.T; i += blockDim.x) {
    const int r = i / lay.T, j = i - r * lay.T;
    const int d = j - kOff + r;
    smem[lay.copy(r) + j] = d >= 1 ? __frcp_rn(static_cast<float>(d)) : qnan;
  }
  for (int i = tid; i < kMaxSlots * kCtlInts; i += blockDim.x) ctl_all[i] = 0;
  __syncthreads();
  if (warp < nslots) load_group<kR>(a, ctl_all + warp * kCtlInts, slots + warp * lay.slot, lay, lane);

  unsigned long long skipped = 0;
  int cur = warp % nslots;
  for (;;) {
    int sl = -1, task = 0, alldead = 0;
    if (lane == 0) {
      for (int t = 0; t < nslots && sl < 0; ++t) {
        const int i = (cur + t) % nslots;
        unsigned* wp = reinterpret_cast<unsigned*>(ctl_all + i * kCtlInts + kWord);
        unsigned w = *reinterpret_cast<volatile unsigned*>(wp);
        while ((w & 0xffffu) < (w >> 16)) {
          const unsigned old = atomicCAS(wp, w, w + 1u);
          if (old == w) {
            sl = i;
            task = static_cast<int>(w & 0xffffu);
            break;
          }
          w = old;
        }
      }
      if (sl < 0) {
        alldead = 1;
        for (int i = 0; i < nslots; ++i) {
          if (*reinterpret_cast<volatile int*>(ctl_all + i * kCtlInts + kDead) == 0) alldead = 0;
        }
      }
    }
    sl = __shfl_sync(0xffffffffu, sl, 0);
    if (sl < 0) {
      if (__shfl_sync(0xffffffffu, alldead, 0)) break;
      __nanosleep(200);
      continue;
    }
    task = __shfl_sync(0xffffffffu, task, 0);
    cur = sl;
    __threadfence_block();
    int* ctl = ctl_all + sl * kCtlInts;
    const volatile int* vc = ctl;
    const int s = vc[kS], cap = vc[kCap], q0 = vc[kQ0];
    int L = 0;
#pragma unroll
    for (int r = 0; r < kR; ++r) L = max(L, vc[kRowL + r]);
    // this lane's two rows
    const int Lr[2] = {vc[kRowL + 2 * ph], vc[kRowL + 2 * ph + 1]};
    const int firstr[2] = {vc[kRowFirst + 2 * ph], vc[kRowFirst + 2 * ph + 1]};
    const int itr[2] = {vc[kRowItem + 2 * ph], vc[kRowItem + 2 * ph + 1]};
    const Slot3<kR> sp = slot_ptrs<kR>(slots + sl * lay.slot, lay);
    const int dir = task & 1, chunk = task >> 1;

    PovP P;
    P.y = chunk * kP + yl;
    P.v0 = P.y < Lr[0];
    P.v1 = P.y < Lr[1];
#pragma unroll
    for (int i = 0; i < 4; ++i) P.A0[i] = P.A1[i] = 0;
    P.G0 = P.G1 = 0.f;
    P.cv0 = P.cv1 = 0;
    P.flag0 = P.flag1 = a.force_exact ? 1u : 0u;
    int vis_p = -1, vis_D = 0;
    float hf[2], hl[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int y = P.y;
      hf[p] = INFINITY;  // absent POV: N = -inf in the skip test
      hl[p] = 0.f;
      if (y < Lr[p]) {
        const int x = dir ? (Lr[p] - 1 - y) : y;
        const float* B = dir ? sp.R[2 * ph + p] : sp.S[2 * ph + p];
        double h;
        if (a.dbg_j0 >= 0 && s == 0 && q0 + 2 * ph + p == 0 && firstr[p] + x == a.dbg_j0) {
          h = a.dbg_h;
          vis_p = p;
          vis_D = min(cap, Lr[p] - 1 - y);
        } else {
          h = __dadd_rn(static_cast<double>(B[y]), a.h0);
        }
        const float hff = __double2float_rn(h);
        const double hld = __dsub_rn(h, static_cast<double>(hff));
        const float hlf = __double2float_rn(hld);
        if (static_cast<double>(hlf) != hld || !(fabsf(hff) < 1e30f)) {
          if (p == 0) P.flag0 = 1u; else P.flag1 = 1u;
        }
        hf[p] = hff;
        hl[p] = hlf;
      }
    }
    P.hf0 = hf[0];
    P.hf1 = hf[1];
    P.hl0 = hl[0];
    P.hl1 = hl[1];
    P.hi0 = P.v0 ? -INFINITY : INFINITY;
    P.lo0 = P.v0 ? -FLT_MAX : INFINITY;
    P.hi1 = P.v1 ? -INFINITY : INFINITY;
    P.lo1 = P.v1 ? -FLT_MAX : INFINITY;
    uint8_t* vis = nullptr;
    if (vis_p >= 0) vis = dir ? a.dbg_vis_bwd : a.dbg_vis_fwd;
    const bool vis_mode = a.dbg_vis_fwd != nullptr || a.dbg_vis_bwd != nullptr;
    const bool any_hl = __any_sync(0xffffffffu, P.hl0 != 0.f || P.hl1 != 0.f);
    if (vis_mode) {
      if (any_hl) {
        run_task<kR, true, true, kCapped>(lay, sp, IV, dir, chunk, L, cap, ph, P, vis ? vis_p : -1, vis, vis_D,
                                          skipped);
      } else {
        run_task<kR, false, true, kCapped>(lay, sp, IV, dir, chunk, L, cap, ph, P, vis ? vis_p : -1, vis, vis_D,
                                           skipped);
      }
    } else if (any_hl) {
      run_task<kR, true, false, kCapped>(lay, sp, IV, dir, chunk, L, cap, ph, P, -1, nullptr, 0, skipped);
    } else {
      run_task<kR, false, false, kCapped>(lay, sp, IV, dir, chunk, L, cap, ph, P, -1, nullptr, 0, skipped);
    }

    {
      // per POV: exact result into its row's cv, or a fixup queue entry in
      // its row's segment
      const SectorDev& sd = a.b.sectors[s];
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const bool v = p ? P.v1 : P.v0;
        if (!v) continue;
        const unsigned fl = p ? P.flag1 : P.flag0;
        const int cvp = p ? P.cv1 : P.cv0;
        const int y = P.y;
        const int Lp = Lr[p];
        const int item = itr[p];
        if (fl) {
          atomicAdd(a.fix_count, 1u);
          const unsigned old = atomicAdd(a.fix_cnt + item, dir ? 0x10000u : 1u);
          const unsigned slot = dir ? static_cast<unsigned>(Lp) + (old >> 16) : (old & 0xffffu);
          a.fix_queue[a.fix_off[item] + slot] = pack_fix(static_cast<unsigned>(dir), static_cast<unsigned>(y));
        } else if (cvp != 0) {
          int* dst = ((dir && a.b.cv_bwd) ? a.b.cv_bwd : a.b.cv) + sd.sdem_off +
                     static_cast<long long>(q0 + 2 * ph + p) * sd.pitch + firstr[p];
          atomicAdd(dst + (dir ? Lp - 1 - y : y), cvp);
        }
      }
    }
    __syncwarp();
    int last = 0;
    if (lane == 0) last = atomicSub(ctl + kRemaining, 1) == 1;
    if (__shfl_sync(0xffffffffu, last, 0)) load_group<kR>(a, ctl, slots + sl * lay.slot, lay, lane);
  }
  if (a.skipped != nullptr && lane == 0 && skipped != 0) {
    atomicAdd(a.skipped, 64ull * skipped);
  }
}

}  // namespace

int scan3_slots(int lmax, int rows) {
  if (lmax >= 32768 - 128) return 0;
  const long long cap = 227 * 1024;
  auto fit = [&](auto lay) {
    const long long n = (cap - 4LL * lay.slots) / (4LL * lay.slot);
    return static_cast<int>(std::min<long long>(std::max<long long>(n, 0), kMaxSlots));
  };
  return rows == 4 ? fit(Layout3<4>(lmax)) : fit(Layout3<2>(lmax));
}

template <int kR>
static int launch_scan3_t(const ScanArgs& a, int nslots, int sms, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(Layout3<kR>(a.lmax).total(nslots)) * sizeof(float);
  auto kern = a.any_capped ? scan3_kernel<kR, true> : scan3_kernel<kR, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return static_cast<int>(e);
  kern<<<sms, kThreads, smem, st>>>(a, nslots, a.lmax);
  return static_cast<int>(cudaGetLastError());
}

// Sets the kernel's shared-memory attribute only (loads its module under lazy
// loading), so a timed launch that follows measures the kernel, not the load.
int prepare_scan3(int lmax, int rows, int any_capped) {
  const int nslots = scan3_slots(lmax, rows);
  if ((rows != 2 && rows != 4) || nslots < 1) return 0;
  auto set = [&](auto kern, size_t smem) {
    return static_cast<int>(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  };
  if (rows == 4) {
    const size_t smem = static_cast<size_t>(Layout3<4>(lmax).total(nslots)) * sizeof(float);
    return any_capped ? set(scan3_kernel<4, true>, smem) : set(scan3_kernel<4, false>, smem);
  }
  const size_t smem = static_cast<size_t>(Layout3<2>(lmax).total(nslots)) * sizeof(float);
  return any_capped ? set(scan3_kernel<2, true>, smem) : set(scan3_kernel<2, false>, smem);
}

int launch_scan3(const ScanArgs& a, int nslots, int rows, void* stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if ((rows != 2 && rows != 4) || nslots < 1 || nslots > scan3_slots(a.lmax, rows)) {
    return static_cast<int>(cudaErrorInvalidValue);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return rows == 4 ? launch_scan3_t<4>(a, nslots, sms, st) : launch_scan3_t<2>(a, nslots, sms, st);
}

}  // namespace sks
