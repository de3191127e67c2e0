// Line-of-sight scan kernels for the sDEM pipeline (sm_100a).
//
// Replaces sector_viewshed / linear_viewshed_row (reference scan.cpp:8-85).
//
// Algorithm. For observer (POV) j0 with absolute height h = row[j0] + h0
// (double, scan.cpp:76) the reference visits targets k = j0 +- dd, computes
// theta = (row[k] - h) / dd in FP64 and calls a target visible when theta
// strictly exceeds the running maximum (scan.cpp:24-34). Its open/close ring
// bookkeeping telescopes to cv = sum over visible targets of (2*dd + 1)
// (SURVEY §7 hard part 2), which is what we accumulate.
//
// FP32 certified filter. Per target the kernel evaluates
//     t = ((e - hf) - hl) * fl(1/dd)           (h = hf + hl exactly)
// in FP32 (packed FADD2/FMUL2). |t - theta| <= 4.01u|theta| (u = 2^-24;
// DESIGN.md "Certified filter" gives the derivation and the preconditions,
// which the kernel checks per POV). The state is a band [lo, hi] around the
// last record r, lo/hi = t_r -+ 10u|t_r|. A target is certainly visible if
// t > hi and certainly hidden if t < lo; anything in between (near ties,
// exact ties, collinear terrain) sets a per-lane flag. A flagged POV group
// (4 POVs x one direction) is not trusted: its cv is discarded and the
// group is queued for the fixup kernel, which re-runs the reference
// recurrence in IEEE FP64 (division included) — so every decision that
// reaches the output is bit-identical to the reference's.
//
// Mapping. A CTA owns one skewed row at a time. The row is prefetched with a
// TMA bulk copy (cp.async.bulk + mbarrier) while the previous row is being
// scanned, then laid out four times in shared memory: S (forward), S1 (S
// shifted by one), R (reversed, so the backward scan is a forward scan) and
// R1, each followed by -inf sentinels so lanes past the row end need no
// bounds checks. Warps take 128-POV tasks (chunk, direction) longest first;
// a lane owns 4 consecutive POVs and walks dd in blocks of 4: per block it
// loads two 16-byte quads (S and S1, which make every packed pair register-
// aligned) plus one broadcast quad each of 1/dd and 2dd+1. Per target that is
// 1.5 packed FP32 instructions for t, then 2 FSETP (ALU) and 3 predicated
// FMA-pipe ops (band update and the ring add), i.e. ~6.6 issue slots for the
// 4 algorithmic FP32 ops the roofline counts.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "sks_device.cuh"
#include "sks_ptx.cuh"

namespace sks {

namespace {

constexpr int kChunk = 128;  // POVs per warp task
constexpr int kPad = 144;    // -inf sentinels after each row copy
constexpr float kBand = 5.9604644775390625e-07f;  // 10 * 2^-24

__host__ __device__ inline int round4(int x) { return (x + 3) & ~3; }

struct SmemLayout {
  int lp;   // round4(lmax)
  int lb;   // row buffer length (floats)
  int lt;   // dd table length (floats)
  int staging, s, s1, r, r1, inv, xt, wms, wmr, ip, total;  // float offsets / total floats
  __host__ __device__ SmemLayout(int lmax, bool shifted) {
    lp = round4(lmax);
    lb = lp + kPad;
    lt = round4(lmax + 32);
    staging = 8;  // first 32 bytes: mbarrier + control words
    s = staging + lp + 8;
    s1 = s + lb;
    r = s1 + (shifted ? lb : 0);
    r1 = r + lb;
    inv = r1 + (shifted ? lb : 0);
    xt = inv + lt;
    wms = xt + lt;          // window max of S per quad (12 positions)
    wmr = wms + lb / 4;     // same for R
    ip = wmr + lb / 4;      // (fl(1/8g), fl(1/(8g+7))) per 8-dd group
    total = ip + round4(lt / 4 + 8);
  }
};

// ---- the certified per-target step ----------------------------------------
// Reference semantics of one target (scan.cpp:24-34) under the FP32 filter.
// Returns the decision; sets flag when the decision is not certified.
__device__ __forceinline__ bool step1(float t, float X, float& hi, float& lo, float& cv,
                                      unsigned& flag) {
  const bool above = t > hi;
  if (above) {
    const float at = fabsf(t);
    hi = __fmaf_rn(at, kBand, t);
    lo = __fmaf_rn(at, -kBand, t);
    cv = __fadd_rn(cv, X);
  } else if (t >= lo) {
    flag = 1u;
  }
  return above;
}

// Same decisions as 16 x step1 (4 dd steps x 4 POVs). Per target: two
// FSETP on the ALU pipe (t > hi: record; t >= lo: not certainly hidden) and
// four predicated FP32-pipe ops (band update hi and lo, ring add, and `cvg`,
// the ring add over every target with t >= lo). Over a flush window cvg ==
// sum(cv) iff no target fell inside the uncertainty band (every band target
// adds 2dd+1 >= 3 to cvg only); both sums are exact integers below 2^24.
// (Measured on B200: FADD/FFMA issue 1/clk/SMSP, FADD2/FMUL2 hold the FP32
// pipe 2 clk. Keeping the flag in a predicate instead (FSETP+FSETP+PLOP3)
// makes ptxas spill the record predicates to GPR bits.)
__device__ __forceinline__ void block16(const float (&t)[4][4], const float4 X, float (&hi)[4],
                                        float (&lo)[4], float (&cv)[4], float& cvg) {
  const float xs[4] = {X.x, X.y, X.z, X.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const float tt = t[i][p];
      const bool pg = tt >= lo[p];
      const bool pa = tt > hi[p];
      const float at = fabsf(tt);
      if (pa) {
        hi[p] = __fmaf_rn(at, kBand, tt);
        lo[p] = __fmaf_rn(at, -kBand, tt);
        cv[p] = __fadd_rn(cv[p], xs[i]);
      }
      if (pg) cvg = __fadd_rn(cvg, xs[i]);
    }
  }
}

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// t for the two POV pairs of one dd step: e01/e23 are the (register-aligned)
// target pairs, nhf/nhl the negated splits of h, inv = fl(1/dd).
__device__ __forceinline__ void tpair(float2 e01, float2 e23, float2 nhf01, float2 nhf23,
                                      float2 nhl01, float2 nhl23, float inv, float (&t)[4]) {
  const float2 iv = f2(inv, inv);
  const float2 a = __fmul2_rn(__fadd2_rn(__fadd2_rn(e01, nhf01), nhl01), iv);
  const float2 b = __fmul2_rn(__fadd2_rn(__fadd2_rn(e23, nhf23), nhl23), iv);
  t[0] = a.x;
  t[1] = a.y;
  t[2] = b.x;
  t[3] = b.y;
}

// One 128-POV task: POVs y0..y0+3 per lane in buffer B (row copy, forward
// direction in B's own coordinates), dd = 1..Dw. Returns per-POV cv and the
// lane flag. kVis: debug path recording decisions of one POV.
template <bool kShifted, bool kVis>
__device__ __forceinline__ void scan_task(const float* __restrict__ B,
                                          const float* __restrict__ B1,
                                          const float4* __restrict__ INV4,
                                          const float4* __restrict__ X4, int y0, int L, int Dw,
                                          const float (&hf)[4], const float (&hl)[4],
                                          float (&hi)[4], float (&lo)[4], int (&cvi)[4],
                                          unsigned& flag, int vis_p, uint8_t* vis,
                                          const float* __restrict__ WM,
                                          const float2* __restrict__ IP, float hfm, float hlm,
                                          unsigned long long* skipped) {
  float cv[4] = {0.f, 0.f, 0.f, 0.f};
  const float2 nhf01 = f2(-hf[0], -hf[1]), nhf23 = f2(-hf[2], -hf[3]);
  const float2 nhl01 = f2(-hl[0], -hl[1]), nhl23 = f2(-hl[2], -hl[3]);
  const float* INV = reinterpret_cast<const float*>(INV4);
  const float* XT = reinterpret_cast<const float*>(X4);

  if (kVis || !kShifted) {
    // Straight per-dd loop (debug / no shifted copies); same arithmetic.
    for (int dd = 1; dd <= Dw; ++dd) {
      const float inv = INV[dd];
      const float X = XT[dd];
      float t[4];
      const float* e = B + y0 + dd;
      tpair(f2(e[0], e[1]), f2(e[2], e[3]), nhf01, nhf23, nhl01, nhl23, inv, t);
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const bool a = step1(t[p], X, hi[p], lo[p], cv[p], flag);
        if (kVis && p == vis_p) vis[dd - 1] = a ? 1 : 0;
      }
      if ((dd & 255) == 0) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          cvi[p] += __float2int_rn(cv[p]);
          cv[p] = 0.f;
        }
      }
    }
  } else {
    // Full blocks only: dd = 4b..4b+3 for b = 0..nb-1 (nb even, 4nb-1 >= Dw).
    // dd = 0 and dd beyond the distance cap read fl(1/dd) = NaN (every
    // comparison false: a no-op target); positions past a lane's row end
    // read -inf sentinels (t = -inf: hidden). So no partial-block code.
    const int nb = ((Dw >> 2) + 2) & ~1;
    unsigned ra = smem_u32(B + y0);   // row quad of block b
    unsigned ra1 = smem_u32(B1 + y0); // shifted-copy quad of block b
    unsigned ta = smem_u32(INV4);     // fl(1/dd) quad of block b
    const unsigned xd = smem_u32(X4) - ta;
    unsigned wa = smem_u32(WM + (y0 >> 2));  // window max of the lane's next 2 blocks
    unsigned pa = smem_u32(IP);               // inv pair of the next 2 blocks
    float4 qa = lds128(ra), qa1 = lds128(ra1);
    float cvg = 0.f;
    int backoff = 0, wait = 1;  // skip-test back-off (b = 0 reads fl(1/0) = NaN anyway)
    unsigned nskip = 0;
    for (int b = 0; b < nb; b += 2) {
      // Hidden-block skip (warp-uniform): a monotone FP32 upper bound of
      // every t of the lane's 32 targets in blocks b, b+1 — window max
      // elevation, the lane's lowest observer, fl(1/dd) at both ends —
      // inflated by 10u to cover the FP32 errors of t and of the bound
      // must lie below the lane's lowest band edge lo. Then no
      // target can be a record or fall in the band: nothing to do.
      if (wait == 0) {
        const float em = lds32(wa);
        const float2 ipv = lds64(pa);
        const float nn = __fadd_rn(__fsub_rn(em, hfm), -hlm);
        const float2 bb = __fmul2_rn(f2(nn, nn), ipv);
        const float bnd = fmaxf(bb.x, bb.y);
        const float bc = __fmaf_rn(fabsf(bnd), kBand, bnd);
        const float lom = fminf(fminf(lo[0], lo[1]), fminf(lo[2], lo[3]));
        if (__all_sync(0xffffffffu, bc < lom)) {
          backoff = 0;
          ++nskip;
          ra += 32;
          ra1 += 32;
          ta += 32;
          wa += 8;
          pa += 8;
          qa = lds128(ra);
          qa1 = lds128(ra1);
          if ((b & 31) == 30 || b + 2 >= nb) {
            if (cvg != __fadd_rn(__fadd_rn(cv[0], cv[1]), __fadd_rn(cv[2], cv[3]))) flag = 1u;
            cvg = 0.f;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              cvi[p] += __float2int_rn(cv[p]);
              cv[p] = 0.f;
            }
          }
          continue;
        }
        backoff = min(2 * backoff + 1, 15);
        wait = backoff;
      } else {
        --wait;
      }
      const float4 qb = lds128(ra + 16), qc = lds128(ra + 32);
      const float4 qb1 = lds128(ra1 + 16), qc1 = lds128(ra1 + 32);
      const float4 iv0 = lds128(ta), iv1 = lds128(ta + 16);
      const float4 xx0 = lds128(ta + xd), xx1 = lds128(ta + xd + 16);
      ra += 32;
      ra1 += 32;
      ta += 32;
      wa += 8;
      pa += 8;
      float t[4][4];
      tpair(f2(qa.x, qa.y), f2(qa.z, qa.w), nhf01, nhf23, nhl01, nhl23, iv0.x, t[0]);
      tpair(f2(qa1.x, qa1.y), f2(qa1.z, qa1.w), nhf01, nhf23, nhl01, nhl23, iv0.y, t[1]);
      tpair(f2(qa.z, qa.w), f2(qb.x, qb.y), nhf01, nhf23, nhl01, nhl23, iv0.z, t[2]);
      tpair(f2(qa1.z, qa1.w), f2(qb1.x, qb1.y), nhf01, nhf23, nhl01, nhl23, iv0.w, t[3]);
      block16(t, xx0, hi, lo, cv, cvg);
      tpair(f2(qb.x, qb.y), f2(qb.z, qb.w), nhf01, nhf23, nhl01, nhl23, iv1.x, t[0]);
      tpair(f2(qb1.x, qb1.y), f2(qb1.z, qb1.w), nhf01, nhf23, nhl01, nhl23, iv1.y, t[1]);
      tpair(f2(qb.z, qb.w), f2(qc.x, qc.y), nhf01, nhf23, nhl01, nhl23, iv1.z, t[2]);
      tpair(f2(qb1.z, qb1.w), f2(qc1.x, qc1.y), nhf01, nhf23, nhl01, nhl23, iv1.w, t[3]);
      block16(t, xx1, hi, lo, cv, cvg);
      qa = qc;
      qa1 = qc1;
      if ((b & 31) == 30 || b + 2 >= nb) {
        // band check of the window, then flush the exact float sums
        if (cvg != __fadd_rn(__fadd_rn(cv[0], cv[1]), __fadd_rn(cv[2], cv[3]))) flag = 1u;
        cvg = 0.f;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          cvi[p] += __float2int_rn(cv[p]);
          cv[p] = 0.f;
        }
      }
    }
    // 2 blocks x 4 dd x 4 POVs x 32 lanes per skipped pair
    if (skipped != nullptr && nskip != 0 && (threadIdx.x & 31) == 0) {
      atomicAdd(skipped, 1024ull * nskip);
    }
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) cvi[p] += __float2int_rn(cv[p]);
}

template <bool kShifted, bool kVis>
__global__ void __launch_bounds__(512, 2) scan_kernel(ScanArgs a) {
  extern __shared__ __align__(16) float smem[];
  const SmemLayout lay(a.lmax, kShifted);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  int* ctrl = reinterpret_cast<int*>(smem + 2);  // [0] next item, [1] task counter
  float* staging = smem + lay.staging;
  float* S = smem + lay.s;
  float* S1 = smem + lay.s1;
  float* R = smem + lay.r;
  float* R1 = smem + lay.r1;
  float* INV = smem + lay.inv;
  float* XT = smem + lay.xt;
  float* WMS = smem + lay.wms;
  float* WMR = smem + lay.wmr;
  float2* IP = reinterpret_cast<float2*>(smem + lay.ip);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int nthreads = blockDim.x;

  auto issue = [&](int it) {
    const ScanItem item = a.items[it];
    const SectorDev& sd = a.b.sectors[item.s];
    const int2 rg = a.b.ranges[sd.row_off + item.q];
    const int fa = rg.x & ~3;
    const int la = round4(rg.y);
    const float* src = a.b.sdem + sd.sdem_off + static_cast<long long>(item.q) * sd.pitch + fa;
    const unsigned bytes = static_cast<unsigned>(la - fa) * 4u;
    mbar_expect_tx(bar, bytes);
    tma_bulk_g2s(staging, src, bytes, bar);
  };

  if (tid == 0) {
    mbar_init(bar, 1);
    const int it = static_cast<int>(atomicAdd(a.item_counter, 1u));
    ctrl[0] = it;
    if (it < a.n_items) issue(it);
  }
  // fl(1/dd) and 2dd+1; dd = 0 and the table tail read NaN (no-op targets)
  const float qnan = __int_as_float(0x7fc00000);
  for (int d = tid; d < lay.lt; d += nthreads) {
    INV[d] = (d == 0 || d >= a.lmax + 8) ? qnan : __frcp_rn(static_cast<float>(d));
    XT[d] = static_cast<float>(2 * d + 1);
  }
  __syncthreads();

  unsigned phase = 0;
  int table_cap = -1;  // forces the first row to write INV and IP
  for (;;) {
    const int cur = ctrl[0];
    if (cur >= a.n_items) break;
    const ScanItem item = a.items[cur];
    const SectorDev sd = a.b.sectors[item.s];
    const int2 rg = a.b.ranges[sd.row_off + item.q];
    const int first = rg.x;
    const int L = rg.y - rg.x;
    const int off = first & 3;
    // distance cap: fl(1/dd) reads NaN for dd > max_dd (rows of one sector
    // share the cap; the table is rewritten when it changes)
    const int want_cap = min(sd.max_dd, a.lmax + 8);
    if (want_cap != table_cap) {
      for (int d = tid; d < lay.lt; d += nthreads) {
        INV[d] = (d == 0 || d > want_cap || d >= a.lmax + 8) ? qnan
                                                             : __frcp_rn(static_cast<float>(d));
      }
      // (fl(1/8g), fl(1/(8g+7))) for the skip test; NaN (= never skip) for
      // g = 0 and for groups reaching past the cap
      for (int g = tid; g < lay.lt / 8; g += nthreads) {
        const int d0 = 8 * g, d1 = 8 * g + 7;
        IP[g] = (g == 0 || d1 > want_cap || d1 >= a.lmax + 8)
                    ? make_float2(qnan, qnan)
                    : make_float2(__frcp_rn(static_cast<float>(d0)), __frcp_rn(static_cast<float>(d1)));
      }
      table_cap = want_cap;
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    const float ninf = -INFINITY;
    for (int x = tid; x < lay.lb; x += nthreads) {
      S[x] = x < L ? staging[off + x] : ninf;
      R[x] = x < L ? staging[off + L - 1 - x] : ninf;
      if (kShifted) {
        S1[x] = x + 1 < L ? staging[off + x + 1] : ninf;
        R1[x] = x + 1 < L ? staging[off + L - 2 - x] : ninf;
      }
    }
    // window maxima for the hidden-block skip: positions 4j..4j+11
    for (int j = tid; j < lay.lb / 4; j += nthreads) {
      float ms = -FLT_MAX, mr = -FLT_MAX;
      for (int u = 0; u < 12; ++u) {
        const int x = 4 * j + u;
        if (x < L) {
          ms = fmaxf(ms, staging[off + x]);
          mr = fmaxf(mr, staging[off + L - 1 - x]);
        }
      }
      WMS[j] = ms;
      WMR[j] = mr;
    }
    if (tid == 0) ctrl[1] = 0;
    __syncthreads();
    if (tid == 0) {
      fence_proxy_async();
      const int it = static_cast<int>(atomicAdd(a.item_counter, 1u));
      ctrl[0] = it;
      if (it < a.n_items) issue(it);
    }
    const int nchunks = (L + kChunk - 1) / kChunk;
    const int ntasks = 2 * nchunks;
    const int max_dd = sd.max_dd;
    int* cvrow = a.b.cv + sd.sdem_off + static_cast<long long>(item.q) * sd.pitch;
    int* cvrow_b =
        (a.b.cv_bwd ? a.b.cv_bwd : a.b.cv) + sd.sdem_off + static_cast<long long>(item.q) * sd.pitch;
    // Warps claim tasks (chunk, direction) longest first; the CTA barrier
    // after the loop closes the row.
    for (;;) {
      int task = 0;
      if (lane == 0) task = atomicAdd(&ctrl[1], 1);
      const int tsk = __shfl_sync(0xffffffffu, task, 0);
      if (tsk >= ntasks) break;
      const int dir = tsk & 1;
      const int chunk = tsk >> 1;
      const int Dw = min(max_dd, L - 1 - chunk * kChunk);
      if (Dw <= 0) continue;
      const float* B = dir ? R : S;
      const float* B1 = dir ? R1 : S1;
      const int y0 = chunk * kChunk + lane * 4;
      float hf[4], hl[4], hi[4], lo[4];
      int cvi[4] = {0, 0, 0, 0};
      unsigned flag = a.force_exact ? 1u : 0u;
      bool any_valid = false;
      int vis_p = -1;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int y = y0 + p;
        if (y < L) {
          any_valid = true;
          const int x = dir ? (L - 1 - y) : y;
          double h;
          if (a.dbg_j0 >= 0 && item.s == 0 && item.q == 0 && first + x == a.dbg_j0) {
            h = a.dbg_h;
            vis_p = p;
          } else {
            h = __dadd_rn(static_cast<double>(B[y]), a.h0);
          }
          const float hff = __double2float_rn(h);
          const double hld = __dsub_rn(h, static_cast<double>(hff));
          const float hlf = __double2float_rn(hld);
          // preconditions of the certified filter: h splits
          // exactly into two floats and stays far from overflow.
          if (static_cast<double>(hlf) != hld || !(fabsf(hff) < 1e30f)) flag = 1u;
          hf[p] = hff;
          hl[p] = hlf;
          hi[p] = -INFINITY;
          lo[p] = -FLT_MAX;
        } else {
          hf[p] = 0.f;
          hl[p] = 0.f;
          hi[p] = INFINITY;
          lo[p] = INFINITY;
        }
      }
      uint8_t* vis = nullptr;
      if (kVis && vis_p >= 0) vis = dir ? a.dbg_vis_bwd : a.dbg_vis_fwd;
      // the lane's lowest observer, split like h (for the skip bound)
      double hmin = INFINITY;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        if (y0 + p < L) hmin = fmin(hmin, __dadd_rn(static_cast<double>(hf[p]), static_cast<double>(hl[p])));
      }
      float hfm = 0.f, hlm = 0.f;
      if (hmin < INFINITY) {
        hfm = __double2float_rn(hmin);
        hlm = __double2float_rn(__dsub_rn(hmin, static_cast<double>(hfm)));
      }
      scan_task<kShifted, kVis>(B, B1, reinterpret_cast<const float4*>(INV),
                                reinterpret_cast<const float4*>(XT), y0, L, Dw, hf, hl, hi, lo,
                                cvi, flag, vis ? vis_p : -1, vis, dir ? WMR : WMS, IP, hfm, hlm,
                                a.skipped);
      if (!any_valid) continue;
      if (flag) {
        atomicAdd(a.fix_count, 1u);
        // forward groups first, backward groups from slot L (packed counts)
        const unsigned old = atomicAdd(a.fix_cnt + cur, dir ? 0x10000u : 1u);
        const unsigned slot = dir ? static_cast<unsigned>(L) + (old >> 16) : (old & 0xffffu);
        a.fix_queue[a.fix_off[cur] + slot] = pack_fix(static_cast<unsigned>(dir), static_cast<unsigned>(y0 >> 2));
      } else {
        int* dst = dir ? cvrow_b : cvrow;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int y = y0 + p;
          if (y < L && cvi[p] != 0) {
            const int x = dir ? (L - 1 - y) : y;
            atomicAdd(dst + first + x, cvi[p]);
          }
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace

size_t scan_smem_bytes(int lmax, bool shifted) {
  return static_cast<size_t>(SmemLayout(lmax, shifted).total) * sizeof(float);
}

static bool use_shifted(int lmax) { return scan_smem_bytes(lmax, true) <= 220 * 1024 && lmax <= 16000; }

int scan_block_threads(int lmax) { return use_shifted(lmax) ? 512 : 512; }

int scan_occupancy(int lmax, int* grid_out) {
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool sh = use_shifted(lmax);
  const size_t smem = scan_smem_bytes(lmax, sh);
  auto fn = sh ? scan_kernel<true, false> : scan_kernel<false, false>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return static_cast<int>(e);
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, scan_block_threads(lmax), smem);
  if (e != cudaSuccess) return static_cast<int>(e);
  *grid_out = sms * (per_sm > 0 ? per_sm : 1);
  return 0;
}

int launch_scan(const ScanArgs& a, int grid, void* stream) {
  const bool vis = a.dbg_vis_fwd != nullptr || a.dbg_vis_bwd != nullptr;
  const bool sh = use_shifted(a.lmax) && !vis;
  const size_t smem = scan_smem_bytes(a.lmax, sh);
  auto fn = vis ? scan_kernel<false, true> : (sh ? scan_kernel<true, false> : scan_kernel<false, false>);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return static_cast<int>(e);
  fn<<<grid, scan_block_threads(a.lmax), smem, static_cast<cudaStream_t>(stream)>>>(a);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace sks
