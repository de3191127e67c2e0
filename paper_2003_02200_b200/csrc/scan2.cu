// Line-of-sight scan, target-lockstep mapping (sm_100a) — the production scan.
//
// Replaces sector_viewshed / linear_viewshed_row (reference scan.cpp:8-85),
// with a certified FP32 filter and an exact FP64 fixup (DESIGN.md
// §3.2): per target t = fl(fl(fl(e - hf) - hl) * fl(1/dd)), band
// [lo, hi] = t_r -+ 10u|t_r| around the last record; t > hi is a record
// (visible), t < lo hidden, anything else flags the POV for the exact
// FP64 fixup kernel.
//
// Mapping. A task is 64 consecutive POVs of one skewed row in one direction;
// lane l owns POVs y = 64c + 2l and 64c + 2l + 1. All lanes of a warp walk the
// SAME target position k (not the same distance dd): a ridge at position k is
// then one step for the whole warp, so the warp-uniform hidden-window skip
// below removes far more work than a distance-lockstep walk (offline model,
// fractal 2000^2: 27% of target slots evaluated vs 46%).
//
// Per group of 4 targets a lane loads one broadcast quad of elevations and,
// per POV, the 4 fl(1/dd) from a table copy whose shift aligns them (dd =
// k - y differs per lane): two pair loads from one of 2 shifted copies by
// default (the smaller tables leave room for one more row slot, measured
// faster), or one quad from one of 4 copies with -DSKS_PREFER_NC4. The ring
// sum cv = sum over visible targets of (2dd+1) is accumulated without a
// per-lane table: records add (k + 2^22) to an integer (one predicated IADD3;
// one accumulator per slot of a 4-target group so that the added register is
// the group's, not the target's), so after a 64-target window
// A = sum(k) + n*2^22 and cv += 2*sum(k) - (2y-1)*n. Near hits (t >= lo) are counted per POV in a float G;
// G != n means a target fell in the uncertainty band (the POV alone is queued).
//
// Hidden-window skip (exact, no inflation). For a window [k0, k0+w) and POV
// p: N = fl(fl(em - hf) - hl) with em the window's maximum elevation, and
// B = max(fl(N*fl(1/dl)), fl(N*fl(1/dh))), dl/dh the window's smallest and
// largest dd. Rounding is monotone, so every t of the window is <= B (both
// signs of N); if B < lo for every POV of the warp no target can
// be a record or a band hit and the window is skipped. Coarse windows of 64
// targets are tested first, then windows of 16.
//
// Scheduling. One persistent CTA per SM (24 warps) keeps up to 8 rows in
// shared-memory slots. Warps claim tasks from any ready slot (CAS on the
// slot's packed next/ntasks word); the warp that completes a row's last task
// loads the next row (longest first, global counter) into that slot. There is
// no CTA-wide barrier after the start-up.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdint>
#include <cstdlib>

#include "sks_device.cuh"
#include "sks_ptx.cuh"

namespace sks {

namespace {

constexpr int kTaskPovs = 64;
#ifndef SKS_FINE_W
#define SKS_FINE_W 16
#endif
constexpr int kW = SKS_FINE_W;  // fine window (targets): 8 or 16
#ifndef SKS_NEAR_NOTEST
#define SKS_NEAR_NOTEST 80  // measured: 32 60.6, 48 60.4, 64 60.2, 80 59.7, 96 59.8, 128 61.4 ms (config 2)
#endif
#ifndef SKS_COARSE_NOTEST
#define SKS_COARSE_NOTEST SKS_NEAR_NOTEST
#endif
#ifndef SKS_COARSE_W
#define SKS_COARSE_W 128  // round 2: 128 vs 64: SmoothedNoise 122.1 vs 123.1 ms, config 5 3764 vs 3878 ms (fractal config 2 59.3 vs 58.9, where scan3 runs)
#endif
constexpr int kH = SKS_COARSE_W;  // coarse window (targets)
// coarse windows longer than a task: tested only where k0 is kH-aligned
constexpr bool kCoarseAligned = kTaskPovs % kH == 0;
constexpr int kOff = 128;  // table index offset (dd >= -kOff + 1 addressable)
#ifndef SKS_SCAN_THREADS
#define SKS_SCAN_THREADS 768
#endif
constexpr int kThreads = SKS_SCAN_THREADS;  // 24 warps: 80 registers, no spills (1024 spills at 64)
#ifndef SKS_MAX_SLOTS
#define SKS_MAX_SLOTS 8
#endif
constexpr int kMaxSlots = SKS_MAX_SLOTS;
constexpr int kCtlInts = 16;  // per slot control block
constexpr float kBand = 5.9604644775390625e-07f;  // 10 * 2^-24
constexpr int kSumShift = 22;
constexpr int kSumMask = (1 << kSumShift) - 1;

struct Layout2 {
  int nc;     // fl(1/dd) table copies: 4 (quad loads), 2 (pair loads) or 1 (long rows)
  int lb;     // row buffer (floats) per direction
  int nw16, nw64;
  int T;      // table length per copy (floats, a multiple of 32)
  int slot;   // floats per slot
  int ctl;    // floats of control blocks
  int tables; // offset of the table copies
  int slots;  // offset of slot 0
  __host__ __device__ Layout2(int lmax, int ncopies) {
    nc = ncopies;
    lb = ((lmax + kH + kH - 1) / kH) * kH;
    nw16 = lb / kW;
    nw64 = lb / kH;
    T = ((kOff + lb + 16 + 31) / 32) * 32;
    slot = 2 * lb + 4 * nw16 + 4 * nw64;
    ctl = kMaxSlots * kCtlInts;
    tables = ctl;
    slots = tables + nc * T + 32;
  }
  // Copy r (IV_r[i] = fl(1/(i - kOff + r))) starts at r*T plus, with 4
  // copies, a bank offset (in quads: 0, 0, 5, 4) so that the two copies one
  // LDS.128 reads (0/2 for the first POV of even/odd lanes, 3/1 for the
  // second) hit disjoint banks in every quarter-warp. With 2 copies the
  // first POV of every lane reads copy 0 and the second copy 1.
  __host__ __device__ int copy(int r) const {
    return tables + r * T + (nc == 4 ? 4 * ((0x4500 >> (4 * r)) & 15) : 0);
  }
  __host__ __device__ int total(int nslots) const { return slots + nslots * slot; }
};

// control block of one slot (ints)
// kBar: the slot's mbarrier (8-byte aligned: slot blocks are 64 B apart) for
// the TMA bulk copy of its rows; kLoads: rows loaded into the slot so far
// (the barrier phase parity)
enum : int { kWord = 0, kRemaining, kDead, kS, kQ, kL, kFirst, kCap, kItem, kLoads, kBar = 10 };

struct Slot {
  const float* S;
  const float* R;
  const float2* WS16;
  const float2* WR16;
  const float2* WS64;
  const float2* WR64;
};

__device__ __forceinline__ Slot slot_ptrs(float* base, const Layout2& lay) {
  Slot s;
  s.S = base;
  s.R = base + lay.lb;
  const float2* w = reinterpret_cast<const float2*>(base + 2 * lay.lb);
  s.WS16 = w;
  s.WR16 = w + lay.nw16;
  s.WS64 = w + 2 * lay.nw16;
  s.WR64 = w + 2 * lay.nw16 + lay.nw64;
  return s;
}

// Loads the next row (longest first) into slot `sl`; one warp. Returns false
// and marks the slot dead when the work list is exhausted.
#ifdef SKS_EXP_LOADCLK
__device__ void load_slot_(const ScanArgs& a, int* ctl, float* base, const Layout2& lay, int lane);
__device__ void load_slot(const ScanArgs& a, int* ctl, float* base, const Layout2& lay, int lane) {
  const long long t0 = clock64();
  load_slot_(a, ctl, base, lay, lane);
  if (lane == 0 && a.skipped) atomicAdd(a.skipped, static_cast<unsigned long long>(clock64() - t0) << 20);
}
__device__ void load_slot_(const ScanArgs& a, int* ctl, float* base, const Layout2& lay, int lane) {
#else
__device__ void load_slot(const ScanArgs& a, int* ctl, float* base, const Layout2& lay, int lane) {
#endif
  int it = 0;
  if (lane == 0) it = static_cast<int>(atomicAdd(a.item_counter, 1u));
  it = __shfl_sync(0xffffffffu, it, 0);
  if (it >= a.n_items) {
    if (lane == 0) atomicExch(ctl + kDead, 1);
    return;
  }
  const ScanItem item = a.items[it];
  const SectorDev& sd = a.b.sectors[item.s];
  const int2 rg = a.b.ranges[sd.row_off + item.q];
  const int L = rg.y - rg.x;
  const long long row0 = sd.sdem_off + static_cast<long long>(item.q) * sd.pitch + rg.x;
  float* S = base;
  float* R = base + lay.lb;
  const float ninf = -INFINITY;
  if (a.b.dem != nullptr) {
    // Fused relocation: gather v(q, j) = (+0 + (1-f)*pre(i, j)) + f*pre(i+1, j),
    // i = q - base + dest[j], exactly as relocate_kernel (skew.cpp:163-183),
    // with pre(i, j) = dem(to_source(i, j)) (apply_pre_ops, skew.cpp:103-142).
    // The row also goes to sdem (the fixup reads it) and its cv range is zeroed.
    const int* m = sd.map;
    float* gdst = a.b.sdem + row0;
    int* cz = a.b.cv + row0;
    int* czb = a.b.cv_bwd ? a.b.cv_bwd + row0 : nullptr;
    const int qb = item.q - sd.base;
    const int nsr = sd.rows;
    // kU cells per lane in flight: the dest/frac loads, then the dependent
    // DEM gathers (L2 hits; strided for transposed sectors), then the stores
    constexpr int kU = 4;
    for (int xb = 0; xb < lay.lb; xb += 32 * kU) {
      int im[kU];
      float f[kU], v1[kU], v2[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        // shear_params (skew.cpp:97-101) in the same IEEE double ops: no
        // dependent load before the gathers
        const int x = xb + 32 * u + lane;
        const double y = __dmul_rn(sd.shear_tan, static_cast<double>(rg.x + x));
        const int dj = __double2int_rz(y);
        f[u] = __double2float_rn(__dsub_rn(y, static_cast<double>(dj)));
        im[u] = x < L ? qb + dj : -2;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = rg.x + xb + 32 * u + lane;
        const int i1 = im[u], i2 = im[u] + 1;
        v1[u] = (i1 >= 0 && i1 < nsr)
                    ? __ldg(a.b.dem + static_cast<long long>(m[0] * i1 + m[1] * j + m[2]) * sd.src_cols +
                            (m[3] * i1 + m[4] * j + m[5]))
                    : 0.0f;
        v2[u] = (i2 >= 0 && i2 < nsr)
                    ? __ldg(a.b.dem + static_cast<long long>(m[0] * i2 + m[1] * j + m[2]) * sd.src_cols +
                            (m[3] * i2 + m[4] * j + m[5]))
                    : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int x = xb + 32 * u + lane;
        if (x >= lay.lb) break;
        float v = ninf;
        if (x < L) {
          float acc = 0.0f;
          if (im[u] >= 0 && im[u] < nsr) acc = __fadd_rn(acc, __fmul_rn(__fsub_rn(1.0f, f[u]), v1[u]));
          if (im[u] + 1 >= 0 && im[u] + 1 < nsr) acc = __fadd_rn(acc, __fmul_rn(f[u], v2[u]));
#ifndef SKS_EXP_NOSTORE
          gdst[x] = acc;
          cz[x] = 0;
          if (czb) czb[x] = 0;
#endif
          v = acc;
        }
        S[x] = v;
      }
    }
  } else {
#ifndef SKS_SCAN_TMA
    // Default: one warp's __ldg loop. The TMA bulk-copy loader below
    // (-DSKS_SCAN_TMA) is bit-identical but measured neutral on fractal terrain
    // (58.90 vs 58.92 ms) and 1.7 % slower on SmoothedNoise (125.3 vs 123.2
    // ms): the loader is 1.4 % of the scan's warp time, and its code changes
    // the register allocation of the hot loop (variants with the loader
    // outlined or the shift copy vectorised moved either terrain by 1-3 %,
    // profiles/r02_scan_loader_ab.txt).
    const float* src = a.b.sdem + row0;
#pragma unroll 4
    for (int x = lane; x < lay.lb; x += 32) S[x] = x < L ? __ldg(src + x) : ninf;
#else
    // TMA bulk copy of the row into the R buffer (free: it is rebuilt from S
    // below). The copy starts at the 16-byte boundary below the row start
    // (sdem_off and pitch are multiples of 32 floats, so the shift is
    // rg.x & 3) and ends at the next boundary after it: within the row's
    // pitch in global memory and within lb >= lmax + 64 floats here. One
    // lane issues it on the slot's mbarrier; the warp waits on the phase.
    const int sh = rg.x & 3;
    const unsigned bytes = static_cast<unsigned>(((sh + L + 3) & ~3) * 4);
    uint64_t* bar = reinterpret_cast<uint64_t*>(ctl + kBar);
    volatile int* vl = ctl;
    const unsigned parity = static_cast<unsigned>(vl[kLoads]) & 1u;
    __syncwarp();
    if (lane == 0) {
      vl[kLoads] = vl[kLoads] + 1;
      // R was last read through the generic proxy (the previous row's tasks)
      fence_proxy_async();
      mbar_expect_tx(bar, bytes);
      tma_bulk_g2s(R, a.b.sdem + (row0 - sh), bytes, bar);
    }
    mbar_wait(bar, parity);
    for (int x = lane; x < lay.lb; x += 32) S[x] = x < L ? R[x + sh] : ninf;
#endif
  }
  __syncwarp();
  for (int x = lane; x < lay.lb; x += 32) R[x] = x < L ? S[L - 1 - x] : ninf;
  __syncwarp();
  float2* w16s = reinterpret_cast<float2*>(base + 2 * lay.lb);
  float2* w16r = w16s + lay.nw16;
  float2* w64s = w16s + 2 * lay.nw16;
  float2* w64r = w64s + lay.nw64;
  const unsigned sa = smem_u32(S), ra = smem_u32(R);
  for (int w = lane; w < lay.nw16; w += 32) {
    float ms = -INFINITY, mr = -INFINITY;
#pragma unroll
    for (int u = 0; u < kW / 4; ++u) {
      const float4 a4 = lds128(sa + 4 * kW * w + 16 * u);
      const float4 b4 = lds128(ra + 4 * kW * w + 16 * u);
      ms = fmaxf(ms, fmaxf(fmaxf(a4.x, a4.y), fmaxf(a4.z, a4.w)));
      mr = fmaxf(mr, fmaxf(fmaxf(b4.x, b4.y), fmaxf(b4.z, b4.w)));
    }
    w16s[w] = make_float2(ms, ms);
    w16r[w] = make_float2(mr, mr);
    if (kW == 16 && a.wm16 != nullptr && 16 * w < L) {
      a.wm16[(sd.sdem_off + static_cast<long long>(item.q) * sd.pitch) / 16 + w] = ms;
    }
  }
  __syncwarp();
  for (int w = lane; w < lay.nw64; w += 32) {
    float ms = -INFINITY, mr = -INFINITY;
#pragma unroll
    for (int u = 0; u < kH / kW; ++u) {
      ms = fmaxf(ms, w16s[(kH / kW) * w + u].x);
      mr = fmaxf(mr, w16r[(kH / kW) * w + u].x);
    }
    w64s[w] = make_float2(ms, ms);
    w64r[w] = make_float2(mr, mr);
  }
  __syncwarp();
  if (lane == 0) {
    const int ntasks = 2 * ((L + kTaskPovs - 1) / kTaskPovs);
    volatile int* v = ctl;
    v[kS] = item.s;
    v[kQ] = item.q;
    v[kL] = L;
    v[kFirst] = rg.x;
    v[kCap] = sd.max_dd;
    v[kItem] = it;
    __threadfence_block();
    atomicExch(ctl + kRemaining, ntasks);
    __threadfence_block();
    atomicExch(reinterpret_cast<unsigned*>(ctl + kWord), static_cast<unsigned>(ntasks) << 16);
  }
  __syncwarp();
}

// Per-lane state of one task (two POVs).
struct Pov2 {
  int y0;          // first POV (buffer coordinates); second is y0 + 1
  bool v0, v1;     // POV exists (y < L)
  float hf0, hf1, hl0, hl1;
  float hi0, hi1, lo0, lo1;
  int A0[4], A1[4];  // per target slot i of a 4-target group: sum(k - i) + n * 2^22 of records
  float G0, G1;    // near hits (t >= lo) in the current flush window, per POV
  int cv0, cv1;    // exact ring sums
  unsigned flag0, flag1;  // POV must go to the exact fixup
};

__device__ __forceinline__ void flush(Pov2& P) {
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
  P.cv0 += 2 * s0 - (2 * P.y0 - 1) * n0;
  P.cv1 += 2 * s1 - (2 * P.y0 + 1) * n1;
  P.G0 = 0.f;
  P.G1 = 0.f;
}

// One target of one POV (reference semantics scan.cpp:24-34 under the
// filter): record if t > hi (band update, A += kb), near hit if t >= lo.
// Written in PTX so every update stays a single predicated instruction
// (C++ lets ptxas turn the integer add into SEL + IADD3).
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

// Same with the decision returned (debug visibility capture).
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

// Skip test for window [k0, k0 + w): see the file header. tb addresses
// table copy 1 so that the pair at tb + 4*k0 is (fl(1/dl1), fl(1/dl0)) —
// both POVs' smallest dd, the second POV first — and the pair w floats on
// is (fl(1/(dh1 + 1)), fl(1/(dh0 + 1))), one past each POV's largest dd
// (still a bound: fl(1/d) is monotone); the N pair is ordered to match. A
// dd <= 0 reads NaN and fails the test (never skipped: conservative).
// Absent POVs have hf = +inf, so N = -inf and they never block a skip.
// With one table copy (kNC == 1, long rows) tb addresses copy 0 with the
// same element offset, where the pairs are not 8-B aligned: two scalar loads.
template <bool kHl, int kNC = 2>
__device__ __forceinline__ bool window_hidden(const Pov2& P, float2 em2, unsigned tb, int k0, int w) {
  float2 N = __fadd2_rn(em2, make_float2(-P.hf1, -P.hf0));
  if (kHl) N = __fadd2_rn(N, make_float2(-P.hl1, -P.hl0));
  const unsigned ra = tb + 4u * static_cast<unsigned>(k0);
  float2 i1, i2;
  if constexpr (kNC == 1) {
    const unsigned rb = ra + 4u * static_cast<unsigned>(w);
    i1 = make_float2(lds32(ra), lds32(ra + 4));
    i2 = make_float2(lds32(rb), lds32(rb + 4));
  } else {
    i1 = lds64(ra);
    i2 = lds64(ra + 4u * static_cast<unsigned>(w));
  }
  const float2 b1 = __fmul2_rn(N, i1);
  const float2 b2 = __fmul2_rn(N, i2);
  const bool ok = (b1.x < P.lo1) & (b2.x < P.lo1) & (b1.y < P.lo0) & (b2.y < P.lo0);
  return __all_sync(0xffffffffu, ok);
}

// Evaluates targets k0 .. k0+kW-1 for both POVs.
template <bool kHl, bool kVis, int kNC>
__device__ __forceinline__ void eval16(Pov2& P, unsigned sb, unsigned ivb0, unsigned ivb1, int k0,
                                       int vis_p, uint8_t* vis, int vis_D) {
#pragma unroll
  for (int g = 0; g < kW / 4; ++g) {
    const int k = k0 + 4 * g;
    const float4 e = lds128(sb + 4 * k);
    float4 q0, q1;
    if (kNC == 4) {
      q0 = lds128(ivb0 + 4 * k);
      q1 = lds128(ivb1 + 4 * k);
    } else if constexpr (kNC == 1) {
      // one copy: the first POV's quad is pair-aligned, the second's starts
      // one element off (a scalar, a pair, a scalar)
      const float2 a0 = lds64(ivb0 + 4 * k), b0 = lds64(ivb0 + 4 * k + 8);
      const float2 m1 = lds64(ivb1 + 4 * k + 4);
      q0 = make_float4(a0.x, a0.y, b0.x, b0.y);
      q1 = make_float4(lds32(ivb1 + 4 * k), m1.x, m1.y, lds32(ivb1 + 4 * k + 12));
    } else {
      const float2 a0 = lds64(ivb0 + 4 * k), b0 = lds64(ivb0 + 4 * k + 8);
      const float2 a1 = lds64(ivb1 + 4 * k), b1 = lds64(ivb1 + 4 * k + 8);
      q0 = make_float4(a0.x, a0.y, b0.x, b0.y);
      q1 = make_float4(a1.x, a1.y, b1.x, b1.y);
    }
    float2 n0a = __fadd2_rn(make_float2(e.x, e.y), make_float2(-P.hf0, -P.hf0));
    float2 n0b = __fadd2_rn(make_float2(e.z, e.w), make_float2(-P.hf0, -P.hf0));
    float2 n1a = __fadd2_rn(make_float2(e.x, e.y), make_float2(-P.hf1, -P.hf1));
    float2 n1b = __fadd2_rn(make_float2(e.z, e.w), make_float2(-P.hf1, -P.hf1));
    if (kHl) {
      n0a = __fadd2_rn(n0a, make_float2(-P.hl0, -P.hl0));
      n0b = __fadd2_rn(n0b, make_float2(-P.hl0, -P.hl0));
      n1a = __fadd2_rn(n1a, make_float2(-P.hl1, -P.hl1));
      n1b = __fadd2_rn(n1b, make_float2(-P.hl1, -P.hl1));
    }
    const float2 t0a = __fmul2_rn(n0a, make_float2(q0.x, q0.y));
    const float2 t0b = __fmul2_rn(n0b, make_float2(q0.z, q0.w));
    const float2 t1a = __fmul2_rn(n1a, make_float2(q1.x, q1.y));
    const float2 t1b = __fmul2_rn(n1b, make_float2(q1.z, q1.w));
    const float t0[4] = {t0a.x, t0a.y, t0b.x, t0b.y};
    const float t1[4] = {t1a.x, t1a.y, t1b.x, t1b.y};
    // every record of slot i adds the group's k + 2^22 (one register for
    // the group; the slot offset i is added back at the flush)
    const int kb = k + (1 << kSumShift);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (kVis) {
        const bool a0 = step_vis(t0[i], P.hi0, P.lo0, P.A0[i], P.G0, kb);
        const bool a1 = step_vis(t1[i], P.hi1, P.lo1, P.A1[i], P.G1, kb);
        if (vis_p >= 0) {
          const int d = k + i - (P.y0 + vis_p);
          if (d >= 1 && d <= vis_D) vis[d - 1] = (vis_p == 0 ? a0 : a1) ? 1 : 0;
        }
      } else {
        step(t0[i], P.hi0, P.lo0, P.A0[i], P.G0, kb);
        step(t1[i], P.hi1, P.lo1, P.A1[i], P.G1, kb);
      }
    }
  }
}

// eval16 for the windows past kmain of a capped row: target k of POV y is a
// no-op (fl(1/d) replaced by NaN: every comparison false) once
// d = k - y exceeds the cap. kc0 = y0 + cap, the last target of the first POV.
template <bool kHl, int kNC>
__device__ __forceinline__ void eval16_capped(Pov2& P, unsigned sb, unsigned ivb0, unsigned ivb1, int k0, int kc0) {
  const float qn = __int_as_float(0x7fc00000);
#pragma unroll
  for (int g = 0; g < kW / 4; ++g) {
    const int k = k0 + 4 * g;
    const float4 e = lds128(sb + 4 * k);
    float4 q0, q1;
    if (kNC == 4) {
      q0 = lds128(ivb0 + 4 * k);
      q1 = lds128(ivb1 + 4 * k);
    } else if constexpr (kNC == 1) {
      // one copy: the first POV's quad is pair-aligned, the second's starts
      // one element off (a scalar, a pair, a scalar)
      const float2 a0 = lds64(ivb0 + 4 * k), b0 = lds64(ivb0 + 4 * k + 8);
      const float2 m1 = lds64(ivb1 + 4 * k + 4);
      q0 = make_float4(a0.x, a0.y, b0.x, b0.y);
      q1 = make_float4(lds32(ivb1 + 4 * k), m1.x, m1.y, lds32(ivb1 + 4 * k + 12));
    } else {
      const float2 a0 = lds64(ivb0 + 4 * k), b0 = lds64(ivb0 + 4 * k + 8);
      const float2 a1 = lds64(ivb1 + 4 * k), b1 = lds64(ivb1 + 4 * k + 8);
      q0 = make_float4(a0.x, a0.y, b0.x, b0.y);
      q1 = make_float4(a1.x, a1.y, b1.x, b1.y);
    }
    const int m0 = kc0 - k, m1 = m0 + 1;  // last valid slot index per POV
    q0.x = m0 >= 0 ? q0.x : qn;
    q0.y = m0 >= 1 ? q0.y : qn;
    q0.z = m0 >= 2 ? q0.z : qn;
    q0.w = m0 >= 3 ? q0.w : qn;
    q1.x = m1 >= 0 ? q1.x : qn;
    q1.y = m1 >= 1 ? q1.y : qn;
    q1.z = m1 >= 2 ? q1.z : qn;
    q1.w = m1 >= 3 ? q1.w : qn;
    float2 n0a = __fadd2_rn(make_float2(e.x, e.y), make_float2(-P.hf0, -P.hf0));
    float2 n0b = __fadd2_rn(make_float2(e.z, e.w), make_float2(-P.hf0, -P.hf0));
    float2 n1a = __fadd2_rn(make_float2(e.x, e.y), make_float2(-P.hf1, -P.hf1));
    float2 n1b = __fadd2_rn(make_float2(e.z, e.w), make_float2(-P.hf1, -P.hf1));
    if (kHl) {
      n0a = __fadd2_rn(n0a, make_float2(-P.hl0, -P.hl0));
      n0b = __fadd2_rn(n0b, make_float2(-P.hl0, -P.hl0));
      n1a = __fadd2_rn(n1a, make_float2(-P.hl1, -P.hl1));
      n1b = __fadd2_rn(n1b, make_float2(-P.hl1, -P.hl1));
    }
    const float2 t0a = __fmul2_rn(n0a, make_float2(q0.x, q0.y));
    const float2 t0b = __fmul2_rn(n0b, make_float2(q0.z, q0.w));
    const float2 t1a = __fmul2_rn(n1a, make_float2(q1.x, q1.y));
    const float2 t1b = __fmul2_rn(n1b, make_float2(q1.z, q1.w));
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

template <bool kHl, bool kVis, int kNC, bool kCapped>
__device__ void run_task(const ScanArgs& a, const Layout2& lay, const Slot& sl, const float* IV,
                         int dir, int chunk, int L, int cap, Pov2& P, int vis_p, uint8_t* vis,
                         int vis_D, unsigned long long& skipped) {
  const float* B = dir ? sl.R : sl.S;
  const float2* W16 = dir ? sl.WR16 : sl.WS16;
  const float2* W64 = dir ? sl.WR64 : sl.WS64;
  const unsigned sb = smem_u32(B);
  // copy 1 holds fl(1/d) at element d + kOff - 1 (window tests, pair loads;
  // one copy: copy 0 at element d + kOff)
  const unsigned tb = kNC == 1 ? smem_u32(IV + lay.copy(0)) + 4u * static_cast<unsigned>(kOff - 1 - P.y0)
                               : smem_u32(IV + lay.copy(1)) + 4u * static_cast<unsigned>(kOff - 2 - P.y0);
  // per POV: the table copy r with (k - y - r) % kNC == 0 for k % 4 == 0
  // (y0 is even: with 2 copies the first POV reads copy 0, the second copy 1)
  const int y1 = P.y0 + 1;
  const int r0 = (-P.y0) & (kNC - 1), r1 = (-y1) & (kNC - 1);
  const unsigned ivb0 = smem_u32(IV + lay.copy(r0)) + 4u * static_cast<unsigned>(kOff - r0 - P.y0);
  const unsigned ivb1 = smem_u32(IV + lay.copy(r1)) + 4u * static_cast<unsigned>(kOff - r1 - y1);
  const unsigned w16a = smem_u32(W16), w64a = smem_u32(W64);
  const int ymin = chunk * kTaskPovs;
  // kCapped: the batch has distance-capped rows and gets the packed tail
  // (the uncapped kernel keeps the one-target tail only, which leaves its
  // main loop's code generation as measured fastest)
  const bool capped = cap < L - 1;
  // last target every POV of the task may still use (windows wholly inside
  // run in the main loop; the remainder is the masked tail)
  const int kmain = capped ? ymin + cap : INT_MAX / 2;
  const int klast = L - 1;
  int k0 = ymin;
  unsigned long long nskip = 0;
  // Flush after 32 evaluated windows: each of the 4 slot accumulators then
  // holds <= 128 records with sum(k) < 128 * 2^15 (k < lb < 32768) and
  // n * 2^22 <= 2^29 (A stays exact); G <= 1024.
  int nev = 0;
  // the first coarse window holds the task triangle and every POV's nearest
  // targets, where almost no window is hidden: no skip tests there
  const int ktest = ymin + SKS_NEAR_NOTEST;
  const int kctest = ymin + SKS_COARSE_NOTEST;  // coarse tests only from here
  while (k0 <= klast) {
    if (!kVis && (kCoarseAligned || (k0 & (kH - 1)) == 0) && k0 >= kctest && k0 + kH - 1 <= kmain) {
      const float2 em = lds64(w64a + 8u * (static_cast<unsigned>(k0) / kH));
      if (window_hidden<kHl, kNC>(P, em, tb, k0, kH)) {
        k0 += kH;
        nskip += kH;
        continue;
      }
    }
    const int kc = kCoarseAligned ? k0 + kH : (k0 & ~(kH - 1)) + kH;
    while (k0 < kc && k0 <= klast && k0 + kW - 1 <= kmain) {
      if (!kVis && k0 >= ktest) {
        const float2 em = lds64(w16a + 8u * (static_cast<unsigned>(k0) / kW));
        if (window_hidden<kHl, kNC>(P, em, tb, k0, kW)) {
          k0 += kW;
          nskip += kW;
          continue;
        }
      }
      eval16<kHl, kVis, kNC>(P, sb, ivb0, ivb1, k0, vis_p, vis, vis_D);
      if (++nev == 32) {
        flush(P);
        nev = 0;
      }
      k0 += kW;
    }
    if (k0 < kc && k0 <= klast) break;  // next window crosses the cap: tail
  }
  flush(P);
  if (kCapped && capped && !kVis) {
    // masked tail: targets beyond some POVs' distance cap, packed like the
    // main loop, with the same hidden-window skip
    const int ylast = min(L - 1, ymin + kTaskPovs - 1);
    const int kt_end = min(klast, ylast + cap);
    const int kc0 = P.y0 + cap;
    int cnt = 0;
    for (; k0 <= kt_end; k0 += kW) {
      if (k0 >= ktest) {  // the bound over the whole window also covers the masked targets
        const float2 em = lds64(w16a + 8u * (static_cast<unsigned>(k0) / kW));
        if (window_hidden<kHl, kNC>(P, em, tb, k0, kW)) {
          nskip += kW;
          continue;
        }
      }
      eval16_capped<kHl, kNC>(P, sb, ivb0, ivb1, k0, kc0);
      if (++cnt == 32) {
        flush(P);
        cnt = 0;
      }
    }
    flush(P);
  } else if (capped) {
    // masked tail, one target at a time (debug visibility capture)
    const int ylast = min(L - 1, ymin + kTaskPovs - 1);
    const int kt_end = min(klast, ylast + cap);
    const float* IVf = IV + lay.copy(0) + kOff;
    int cnt = 0;
    for (int k = k0; k <= kt_end; ++k) {
      const float e = B[k];
      const int d0 = k - P.y0, d1 = d0 - 1;
      const bool m0 = P.v0 && d0 >= 1 && d0 <= cap;
      const bool m1 = P.v1 && d1 >= 1 && d1 <= cap;
      const float qn = __int_as_float(0x7fc00000);
      float t0 = __fmul_rn(__fadd_rn(__fadd_rn(e, -P.hf0), -P.hl0), m0 ? IVf[d0] : qn);
      float t1 = __fmul_rn(__fadd_rn(__fadd_rn(e, -P.hf1), -P.hl1), m1 ? IVf[d1] : qn);
      const int kb = k + (1 << kSumShift);
      const bool a0 = step_vis(t0, P.hi0, P.lo0, P.A0[0], P.G0, kb);
      const bool a1 = step_vis(t1, P.hi1, P.lo1, P.A1[0], P.G1, kb);
      if (kVis && vis_p >= 0) {
        const int d = vis_p == 0 ? d0 : d1;
        if (d >= 1 && d <= vis_D) vis[d - 1] = (vis_p == 0 ? a0 : a1) ? 1 : 0;
      }
      if (++cnt == kH) {
        flush(P);
        cnt = 0;
      }
    }
    flush(P);
  }
  skipped += nskip;
}

template <int kThr, int kNC, bool kCapped>
__global__ void __launch_bounds__(kThr, 1) scan2_kernel(const __grid_constant__ ScanArgs a, int nslots, int lmax) {
  extern __shared__ __align__(16) float smem[];
  const Layout2 lay(lmax, kNC);
  int* ctl_all = reinterpret_cast<int*>(smem);
  float* IV = smem;  // table copies at lay.copy(r)
  float* slots = smem + lay.slots;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;

  // fl(1/d) tables, 4 copies shifted by r: IV[r][i] = fl(1/(i - kOff + r)),
  // NaN for d <= 0 (a no-op target: every comparison is false)
  const float qnan = __int_as_float(0x7fc00000);
  for (int i = tid; i < kNC * lay.T; i += blockDim.x) {
    const int r = i / lay.T, j = i - r * lay.T;
    const int d = j - kOff + r;
    smem[lay.copy(r) + j] = d >= 1 ? __frcp_rn(static_cast<float>(d)) : qnan;
  }
  for (int i = tid; i < kMaxSlots * kCtlInts; i += blockDim.x) ctl_all[i] = 0;
  __syncthreads();
  if (tid < nslots) mbar_init(reinterpret_cast<uint64_t*>(ctl_all + tid * kCtlInts + kBar), 1);
  __syncthreads();
  if (warp < nslots) load_slot(a, ctl_all + warp * kCtlInts, slots + warp * lay.slot, lay, lane);

  unsigned long long skipped = 0;
#ifdef SKS_EXP_TAIL
  unsigned long long t_idle = 0;   // start of the current wait for a task
  unsigned long long idle_ns = 0;  // accumulated waits
#endif
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
#ifdef SKS_EXP_TAIL
      if (t_idle == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_idle));
#endif
      if (__shfl_sync(0xffffffffu, alldead, 0)) break;
      __nanosleep(200);
      continue;
    }
    task = __shfl_sync(0xffffffffu, task, 0);
#ifdef SKS_EXP_TAIL
    if (t_idle != 0) {
      unsigned long long t_now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
      idle_ns += t_now - t_idle;
      t_idle = 0;
    }
#endif
    cur = sl;
    __threadfence_block();
    int* ctl = ctl_all + sl * kCtlInts;
    const volatile int* vc = ctl;
    const int s = vc[kS], q = vc[kQ], L = vc[kL], first = vc[kFirst], cap = vc[kCap], item = vc[kItem];
    const Slot sp = slot_ptrs(slots + sl * lay.slot, lay);
    const int dir = task & 1, chunk = task >> 1;
    const float* B = dir ? sp.R : sp.S;

    Pov2 P;
    P.y0 = chunk * kTaskPovs + 2 * lane;
    P.v0 = P.y0 < L;
    P.v1 = P.y0 + 1 < L;
#pragma unroll
    for (int i = 0; i < 4; ++i) P.A0[i] = P.A1[i] = 0;
    P.G0 = P.G1 = 0.f;
    P.cv0 = P.cv1 = 0;
    P.flag0 = P.flag1 = a.force_exact ? 1u : 0u;
    int vis_p = -1, vis_D = 0;
    float hf[2], hl[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int y = P.y0 + p;
      hf[p] = INFINITY;  // absent POV: N = -inf in the skip test
      hl[p] = 0.f;
      if (y < L) {
        const int x = dir ? (L - 1 - y) : y;
        double h;
        if (a.dbg_j0 >= 0 && s == 0 && q == 0 && first + x == a.dbg_j0) {
          h = a.dbg_h;
          vis_p = p;
          vis_D = min(cap, L - 1 - y);
        } else {
          h = __dadd_rn(static_cast<double>(B[y]), a.h0);
        }
        const float hff = __double2float_rn(h);
        const double hld = __dsub_rn(h, static_cast<double>(hff));
        const float hlf = __double2float_rn(hld);
        // filter preconditions: h = hf + hl exactly, far from overflow
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
        run_task<true, true, kNC, kCapped>(a, lay, sp, IV, dir, chunk, L, cap, P, vis ? vis_p : -1, vis, vis_D, skipped);
      } else {
        run_task<false, true, kNC, kCapped>(a, lay, sp, IV, dir, chunk, L, cap, P, vis ? vis_p : -1, vis, vis_D, skipped);
      }
    } else if (any_hl) {
      run_task<true, false, kNC, kCapped>(a, lay, sp, IV, dir, chunk, L, cap, P, -1, nullptr, 0, skipped);
    } else {
      run_task<false, false, kNC, kCapped>(a, lay, sp, IV, dir, chunk, L, cap, P, -1, nullptr, 0, skipped);
    }

    {
      // per POV: exact result, or a fixup queue entry (fix_group 1: entry = POV)
      const SectorDev& sd = a.b.sectors[s];
      int* dst = ((dir && a.b.cv_bwd) ? a.b.cv_bwd : a.b.cv) + sd.sdem_off +
                 static_cast<long long>(q) * sd.pitch + first;
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const bool v = p ? P.v1 : P.v0;
        const unsigned fl = p ? P.flag1 : P.flag0;
        const int cvp = p ? P.cv1 : P.cv0;
        const int y = P.y0 + p;
        if (!v) continue;
        if (fl) {
          atomicAdd(a.fix_count, 1u);
          // forward entries fill the segment's first L slots, backward ones
          // the next L (16-bit counts packed in one counter), so the fixup's
          // neighbouring lanes walk the same direction
          const unsigned old = atomicAdd(a.fix_cnt + item, dir ? 0x10000u : 1u);
          const unsigned slot = dir ? static_cast<unsigned>(L) + (old >> 16) : (old & 0xffffu);
          a.fix_queue[a.fix_off[item] + slot] = pack_fix(static_cast<unsigned>(dir), static_cast<unsigned>(y));
        } else if (cvp != 0) {
          atomicAdd(dst + (dir ? L - 1 - y : y), cvp);
        }
      }
    }
    __syncwarp();
    int last = 0;
    if (lane == 0) last = atomicSub(ctl + kRemaining, 1) == 1;
    if (__shfl_sync(0xffffffffu, last, 0)) load_slot(a, ctl, slots + sl * lay.slot, lay, lane);
  }
  if (a.skipped != nullptr && lane == 0 && skipped != 0) {
    atomicAdd(a.skipped, 64ull * skipped);
  }
#ifdef SKS_EXP_TAIL
  // experiment build: warp-nanoseconds spent without a task (waiting for a
  // slot's next row or for the end), added << 20 to the skipped counter
  // (tools/loader_cycles.py reads it back)
  unsigned long long t_end;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
  if (t_idle != 0) idle_ns += t_end - t_idle;
  if (a.skipped != nullptr && lane == 0) atomicAdd(a.skipped, idle_ns << 20);
#endif
}

}  // namespace

// Table copies and slots that fit the opt-in shared memory for rows up to
// lmax: 2 copies (pair loads) where >= 2 slots fit (rows up to ~8 000
// cells; 4 copies with quad loads measured slower: the freed memory holds
// more row slots, config 2 scan 59.7 -> 58.9 ms, -DSKS_PREFER_NC4 keeps
// them); beyond, one copy if that fits more slots (config 5's 10 000-cell
// rows: 2 slots instead of 1; the second POV's table quads and the window
// tests then take scalar loads), else whichever holds one slot (rows up to
// ~17 000 cells). 0 slots: the rows go through the fixup kernel whole (long
// rows, engine.cu).
static void scan2_config(int lmax, int* copies, int* slots) {
  *copies = 0;
  *slots = 0;
  if (lmax >= 32768 - 128) return;  // k < 2^15 keeps the flush sums exact
  const long long cap = 227 * 1024;
  auto fit = [&](int nc) {
    const Layout2 lay(lmax, nc);
    const long long n = (cap - 4LL * lay.slots) / (4LL * lay.slot);
    return static_cast<int>(std::min<long long>(std::max<long long>(n, 0), kMaxSlots));
  };
#ifdef SKS_PREFER_NC4
  if (fit(4) >= 2) {
    *copies = 4;
    *slots = fit(4);
    return;
  }
#endif
  const int n2 = fit(2), n1 = fit(1);
  if (n2 >= 2 || (n2 >= 1 && n1 <= n2)) {
    *copies = 2;
    *slots = n2;
  } else if (n1 >= 1) {
    *copies = 1;
    *slots = n1;
  }
}

int scan2_slots(int lmax) {
  int c = 0, n = 0;
  scan2_config(lmax, &c, &n);
  return n;
}

int scan2_max_row() {
  static const int m = [] {
    int lo = 4, hi = 32768;  // scan2_slots(lo) >= 1, scan2_slots(hi) == 0
    while (hi - lo > 1) {
      const int mid = (lo + hi) / 2;
      if (scan2_slots(mid) >= 1) lo = mid; else hi = mid;
    }
    return lo;
  }();
  return m;
}

size_t scan2_smem_bytes(int lmax, int nslots) {
  int c = 0, n = 0;
  scan2_config(lmax, &c, &n);
  return static_cast<size_t>(Layout2(lmax, c > 0 ? c : 4).total(nslots)) * sizeof(float);
}

template <int kThr, int kNC, bool kCapped>
static int launch_scan2_t(const ScanArgs& a, int nslots, int sms, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(Layout2(a.lmax, kNC).total(nslots)) * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(scan2_kernel<kThr, kNC, kCapped>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return static_cast<int>(e);
  scan2_kernel<kThr, kNC, kCapped><<<sms, kThr, smem, st>>>(a, nslots, a.lmax);
  return static_cast<int>(cudaGetLastError());
}

// Shared-memory attribute of the instance launch_scan2 would use (loads its
// module under lazy loading; the engine calls it before a timed launch).
int prepare_scan2(int lmax, int any_capped) {
  int copies = 0, fit = 0;
  scan2_config(lmax, &copies, &fit);
  if (copies == 0 || fit < 1) return 0;
  const size_t smem = static_cast<size_t>(Layout2(lmax, copies).total(fit)) * sizeof(float);
  auto set = [&](auto kern) {
    return static_cast<int>(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  };
  if (any_capped) {
    return copies == 4 ? set(scan2_kernel<kThreads, 4, true>)
           : copies == 2 ? set(scan2_kernel<kThreads, 2, true>)
                         : set(scan2_kernel<kThreads, 1, true>);
  }
  return copies == 4 ? set(scan2_kernel<kThreads, 4, false>)
         : copies == 2 ? set(scan2_kernel<kThreads, 2, false>)
                       : set(scan2_kernel<kThreads, 1, false>);
}

int launch_scan2(const ScanArgs& a, int nslots, void* stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int copies = 0, fit = 0;
  scan2_config(a.lmax, &copies, &fit);
  if (copies == 0 || nslots < 1 || nslots > fit) return static_cast<int>(cudaErrorInvalidValue);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (a.any_capped) {
    return copies == 4   ? launch_scan2_t<kThreads, 4, true>(a, nslots, sms, st)
           : copies == 2 ? launch_scan2_t<kThreads, 2, true>(a, nslots, sms, st)
                         : launch_scan2_t<kThreads, 1, true>(a, nslots, sms, st);
  }
  return copies == 4   ? launch_scan2_t<kThreads, 4, false>(a, nslots, sms, st)
         : copies == 2 ? launch_scan2_t<kThreads, 2, false>(a, nslots, sms, st)
                       : launch_scan2_t<kThreads, 1, false>(a, nslots, sms, st);
}

}  // namespace sks
