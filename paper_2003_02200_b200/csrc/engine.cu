// Engine and C ABI of the B200 sDEM total-viewshed path.
//
// Replaces the reference engine (engine.cpp:29-244): instead of a pool of
// std::threads each running relocation -> scan -> unskew on one sector, a
// per-GPU context runs whole BATCHES of sectors with one launch per phase:
//   relocate (all sectors of the batch) -> scan (one persistent launch over
//   every skewed row of the batch, longest first) -> exact fixup of flagged
//   POV groups -> unskew + accumulate (ascending k, into the FP64 map).
// Sector plans (pure geometry) and the batch metadata are cached per
// context, so repeated runs on DEMs of the same shape only move elevations.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numbers>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/skewshed_b200.h"
#include "sks_device.cuh"
#include "sks_io.hpp"
#include "sks_plan.hpp"
#include "sks_sweep.hpp"

namespace sks {

namespace {

thread_local std::string g_error;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::ostringstream os;
    os << what << ": " << cudaGetErrorString(e);
    throw CudaError(os.str());
  }
}
void cuda_check(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }

template <typename Fn>
sks_status guarded(Fn&& fn) {
  try {
    fn();
    g_error.clear();
    return SKS_OK;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return SKS_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_error = e.what();
    return SKS_OUT_OF_RANGE;
  } catch (const GridFormatError& e) {
    g_error = e.what();
    return SKS_FORMAT_ERROR;
  } catch (const CudaError& e) {
    g_error = e.what();
    return SKS_CUDA_ERROR;
  } catch (const std::exception& e) {
    g_error = e.what();
    return SKS_INTERNAL;
  }
}

// Device buffer that only grows.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int device = -1;
  void ensure(size_t n, int dev) {
    if (n <= bytes && p) return;
    release();
    cuda_check(cudaMalloc(&p, std::max<size_t>(n, 256)), "cudaMalloc");
    bytes = std::max<size_t>(n, 256);
    device = dev;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  ~DevBuf() { release(); }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

int round_up(int x, int m) { return (x + m - 1) / m * m; }

// device counters: [0] scan item, [1] flagged groups, [4] fixup item,
// [8..9] skipped target slots (u64)
constexpr size_t kCounterBytes = 64;

// One batch of sectors, fully prepared on the host and mirrored on device.
struct Batch {
  std::vector<int> slots;  // indices into Plans::plans, ascending k
  std::vector<SectorDev> sdev;
  std::vector<int> dest;
  std::vector<float> fracf;
  std::vector<double> fracd;
  std::vector<int2> ranges;
  std::vector<ScanItem> items;
  long long pool_elems = 0;  // sdem / cv pool elements
  int lmax = 0;      // longest row scan2 scans
  int lmax_all = 0;  // longest row incl. long rows
  int n_long = 0;    // items [0, n_long): rows longer than scan2's slots (fixup only)
  bool fused = false;  // relocation fused into scan2's row loader
  bool any_capped = false;  // some item row is longer than its sector's distance cap + 1
  unsigned fix_cap = 0;
  std::vector<unsigned> fix_off;  // per item: fixup queue segment offset
  int tiles_x = 0, tiles_total = 0;
  long long target_evals = 0;
  // device copies
  // scan3 row groups (pairs, quads) over the scanned items [n_long, n_items)
  // (indices relative to n_long)
  std::vector<int4> pairs, quads;
  DevBuf d_sectors, d_dest, d_fracf, d_fracd, d_ranges, d_items, d_fix_off, d_pairs, d_quads;
  // unskew TMA tensor maps (one per sector over its cv rows), encoded for the
  // cv pool at umap_cv; re-encoded when the pool moves
  mutable DevBuf d_umaps;
  mutable const int* umap_cv = nullptr;
  mutable bool umap_ok = false;
};

struct Plans {
  std::vector<SectorPlanH> plans;  // ascending k
  std::vector<std::unique_ptr<Batch>> batches;
};

// Rows longer than this go through the fixup kernel whole (every POV, both
// directions) instead of scan2: scan2's shared-memory slots hold rows up to
// scan2_max_row() cells. SKS_LONG_ROW lowers the limit (tests exercise the
// long-row path at small sizes with it); read when a batch is built.
int long_row_limit() {
  int lim = scan2_max_row();
  if (const char* s = std::getenv("SKS_LONG_ROW")) {
    const int v = std::atoi(s);
    if (v >= 2) lim = std::min(lim, v);
  }
  return lim;
}

// The ring sums are exact int32s: a POV's cv is at most L^2 - 1 (forward +
// backward over a row of L cells), and the fixup queue counts pack two 16-bit
// halves, so rows are limited to 46340 cells (a DEM side of 46340 cells:
// 8.6 GB of f32 elevations).
constexpr int kMaxRow = 46340;

// Relocation fused into scan2's row loader: opt-in with
// SKS_FUSED=1, read when a batch is built. Measured on config 2 it removes
// the 1.1 ms relocation launch but the loader warp's dependent DEM gathers
// add 1.45 ms to the scan, so the default stays the
// standalone relocation kernel.
bool fused_relocation() {
  const char* s = std::getenv("SKS_FUSED");
  return s != nullptr && std::atoi(s) != 0;
}

long long batch_budget_bytes() {
  if (const char* s = std::getenv("SKS_BATCH_GB")) {
    double gb = std::atof(s);
    if (gb > 0) return static_cast<long long>(gb * (1LL << 30));
  }
  return 24LL << 30;
}

std::unique_ptr<Batch> make_batch(const std::vector<SectorPlanH>& plans,
                                  const std::vector<int>& slots, int device) {
  auto b = std::make_unique<Batch>();
  b->slots = slots;
  long long off = 0;
  int col_off = 0, row_off = 0;
  int max_cols = 0, max_rows = 0;
  for (size_t s = 0; s < slots.size(); ++s) {
    const SectorPlanH& p = plans[slots[s]];
    SectorDev d{};
    d.k = p.k;
    d.rows = p.rows;
    d.cols = p.cols;
    d.src_rows = p.src_rows;
    d.src_cols = p.src_cols;
    d.base = p.base;
    d.skw_rows = p.skw_rows;
    d.pitch = round_up(p.cols, 32);
    d.max_dd = p.max_dd;
    d.col_off = col_off;
    d.row_off = row_off;
    d.q_lo = p.q_lo;
    d.q_hi = p.q_hi < 0 ? p.skw_rows : p.q_hi;
    std::copy(p.map, p.map + 6, d.map);
    std::copy(p.inv, p.inv + 6, d.inv);
    d.correction = p.correction;
    d.shear_tan = p.shear_tan;
    d.sdem_off = off;
    off += static_cast<long long>(p.skw_rows) * d.pitch;
    col_off += p.cols;
    row_off += p.skw_rows;
    b->dest.insert(b->dest.end(), p.dest.begin(), p.dest.end());
    b->fracf.insert(b->fracf.end(), p.fracf.begin(), p.fracf.end());
    b->fracd.insert(b->fracd.end(), p.fracd.begin(), p.fracd.end());
    for (int q = 0; q < p.skw_rows; ++q) {
      const RowRange& r = p.ranges[q];
      b->ranges.push_back(make_int2(r.first, r.last));
      const int L = r.last - r.first;
      if (L >= 2 && p.max_dd < L - 1 && q >= d.q_lo && q < d.q_hi) b->any_capped = true;
      if (L >= 1 && q >= d.q_lo && q < d.q_hi) {
        // rows with no target (L = 1 or a zero cap) only matter to the fused
        // loader, which zeroes their cv range; dropped below otherwise
        b->items.push_back(ScanItem{static_cast<int>(s), q});
        if (L >= 2 && p.max_dd > 0) {
          b->lmax_all = std::max(b->lmax_all, L);
          b->target_evals += row_target_evals(L, p.max_dd);
        }
      }
    }
    max_cols = std::max(max_cols, p.cols);
    max_rows = std::max(max_rows, p.skw_rows);
    b->sdev.push_back(d);
  }
  b->pool_elems = off;
  if (b->lmax_all > kMaxRow) {
    std::ostringstream os;
    os << "grid too large: skewed rows of " << b->lmax_all << " cells exceed the " << kMaxRow
       << "-cell limit of the exact int32 ring sums";
    throw std::invalid_argument(os.str());
  }
  const int limit = long_row_limit();
  auto item_len = [&](const ScanItem& it) {
    const int2 r = b->ranges[b->sdev[it.s].row_off + it.q];
    return r.y - r.x;
  };
  bool any_long = false;
  for (const ScanItem& it : b->items) any_long |= item_len(it) > limit;
  // the fused loader builds the rows scan2 reads; long rows are not scanned
  b->fused = fused_relocation() && !any_long;
  if (!b->fused) {
    std::erase_if(b->items, [&](const ScanItem& it) {
      const int2 r = b->ranges[b->sdev[it.s].row_off + it.q];
      return r.y - r.x < 2 || b->sdev[it.s].max_dd <= 0;
    });
  }
  // longest rows first (load balance of the persistent scan; long rows, the
  // fixup-only items, therefore come first: items [0, n_long))
  std::stable_sort(b->items.begin(), b->items.end(), [&](const ScanItem& x, const ScanItem& y) {
    const int2 rx = b->ranges[b->sdev[x.s].row_off + x.q];
    const int2 ry = b->ranges[b->sdev[y.s].row_off + y.q];
    return (rx.y - rx.x) > (ry.y - ry.x);
  });
  for (const ScanItem& it : b->items) {
    const int L = item_len(it);
    if (L > limit) ++b->n_long; else if (L >= 2 && b->sdev[it.s].max_dd > 0) b->lmax = std::max(b->lmax, L);
  }
  // scan3 row groups of kR = 2 and 4: rows q0 .. q0+kR-1 (q0 = q & ~(kR-1))
  // of a sector, each a scanned item or -1, longest group first
  for (int kR : {2, 4}) {
    std::map<std::pair<int, int>, int4> groups;  // (sector slot, q0) -> items
    std::map<std::pair<int, int>, int> glen;
    for (size_t i = b->n_long; i < b->items.size(); ++i) {
      const ScanItem& it = b->items[i];
      const int q0 = it.q & ~(kR - 1);
      auto key = std::make_pair(it.s, q0);
      auto [g, fresh] = groups.try_emplace(key, make_int4(-1, -1, -1, -1));
      int* slot = &g->second.x;
      slot[it.q - q0] = static_cast<int>(i) - b->n_long;
      glen[key] = std::max(glen[key], item_len(it));
    }
    std::vector<std::pair<int, int4>> pl;
    for (const auto& [key, g] : groups) pl.push_back({glen[key], g});
    std::stable_sort(pl.begin(), pl.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    auto& out = kR == 2 ? b->pairs : b->quads;
    for (const auto& pg : pl) out.push_back(pg.second);
  }
  // fixup queue segments, in item order: one entry per POV and direction,
  // the exact bound
  b->fix_off.resize(b->items.size());
  long long fix_total = 0;
  for (size_t i = 0; i < b->items.size(); ++i) {
    const int2 r = b->ranges[b->sdev[b->items[i].s].row_off + b->items[i].q];
    b->fix_off[i] = static_cast<unsigned>(fix_total);
    fix_total += 2LL * (r.y - r.x);
  }
  if (fix_total >= (1LL << 32)) throw std::runtime_error("fixup queue of one batch exceeds 2^32 entries");
  b->fix_cap = static_cast<unsigned>(fix_total);
  b->tiles_x = (max_cols + relocate_tile_cols() - 1) / relocate_tile_cols();
  // tile rows from each sector's first owned tile row to its last owned row
  int tq_max = 0;
  for (const SectorDev& d : b->sdev) {
    const int tr = relocate_tile_rows();
    const int hi = std::max(d.q_hi, d.q_lo + 1);
    tq_max = std::max(tq_max, (hi + tr - 1) / tr - d.q_lo / tr);
  }
  (void)max_rows;
  b->tiles_total = b->tiles_x * tq_max;
  if (b->fix_cap == 0) b->fix_cap = 1;
  // upload metadata once
  auto up = [&](DevBuf& buf, const void* src, size_t bytes) {
    buf.ensure(bytes, device);
    if (bytes) cuda_check(cudaMemcpy(buf.p, src, bytes, cudaMemcpyHostToDevice), "upload metadata");
  };
  up(b->d_sectors, b->sdev.data(), b->sdev.size() * sizeof(SectorDev));
  up(b->d_dest, b->dest.data(), b->dest.size() * sizeof(int));
  up(b->d_fracf, b->fracf.data(), b->fracf.size() * sizeof(float));
  up(b->d_fracd, b->fracd.data(), b->fracd.size() * sizeof(double));
  up(b->d_ranges, b->ranges.data(), b->ranges.size() * sizeof(int2));
  up(b->d_items, b->items.data(), b->items.size() * sizeof(ScanItem));
  up(b->d_fix_off, b->fix_off.data(), b->fix_off.size() * sizeof(unsigned));
  up(b->d_pairs, b->pairs.data(), b->pairs.size() * sizeof(int4));
  up(b->d_quads, b->quads.data(), b->quads.size() * sizeof(int4));
  return b;
}

// Device bytes one sector adds to a batch, from the formulas ensure_pools
// and make_batch size the buffers with: sdem f32 + cv i32 per pool element,
// window maxima (one f32 per 16 pool elements), the fixup queue (2 u32
// entries per covered cell: one per POV and direction) and per-row metadata
// (range, item, fix_off, fix_cnt, prefix).
long long sector_batch_bytes(const SectorPlanH& p) {
  const long long pool = static_cast<long long>(p.skw_rows) * round_up(p.cols, 32);
  const long long cells = static_cast<long long>(p.rows) * p.cols;
  return pool * 8 + (pool / 16) * 4 + cells * 8 + static_cast<long long>(p.skw_rows) * 28 +
         static_cast<long long>(p.cols) * 16;
}

// Split plans (ascending k) into batches under the memory budget (and under
// 2^31 fixup queue entries per batch: the queue offsets are 32-bit).
void make_batches(Plans& P, int device) {
  const long long budget = batch_budget_bytes();
  std::vector<int> cur;
  long long cur_bytes = 0, cur_queue = 0;
  for (int s = 0; s < static_cast<int>(P.plans.size()); ++s) {
    const SectorPlanH& p = P.plans[s];
    const long long bytes = sector_batch_bytes(p);
    const long long queue = 2LL * p.rows * p.cols;
    if (!cur.empty() && (cur_bytes + bytes > budget || cur_queue + queue >= (1LL << 31))) {
      P.batches.push_back(make_batch(P.plans, cur, device));
      cur.clear();
      cur_bytes = 0;
      cur_queue = 0;
    }
    cur.push_back(s);
    cur_bytes += bytes;
    cur_queue += queue;
  }
  if (!cur.empty()) P.batches.push_back(make_batch(P.plans, cur, device));
}

}  // namespace

}  // namespace sks

using namespace sks;

struct sks_context {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  int sms = 0;
  std::mutex mu;
  // plan cache
  std::map<std::tuple<int, int, int, double, double, std::vector<int>, int, int, std::vector<double>>,
           std::unique_ptr<Plans>>
      cache;
  // work buffers
  DevBuf sdem, cv, cvb, queue, fixcnt, fixoff, wm16, counters, dem, map, vis, check, ivt, dem_pitched;
  int ivt_len = 0;  // entries of the global fl(1/d) table computed so far
  unsigned long long* h_check = nullptr;  // pinned: device DEM scan result
  cudaEvent_t ev[8] = {};
  long long launches = 0;

  void activate() const { cuda_check(cudaSetDevice(device), "cudaSetDevice"); }

  Plans& plans_for(int dimy, int dimx, int ns, double cellsize, double max_distance,
                   const std::vector<int>& sectors, int part = 0, int nparts = 1,
                   const std::vector<double>& cuts = {}) {
    auto key = std::make_tuple(dimy, dimx, ns, cellsize, max_distance, sectors, part, nparts, cuts);
    auto it = cache.find(key);
    if (it != cache.end()) return *it->second;
    if (cache.size() > 16) cache.clear();
    auto P = std::make_unique<Plans>();
    for (int k : sectors) {
      P->plans.push_back(plan_sector(k, ns, dimy, dimx, cellsize, max_distance));
      if (nparts > 1) set_row_block(P->plans.back(), part, nparts, cuts.empty() ? nullptr : cuts.data());
    }
    make_batches(*P, device);
    Plans& ref = *P;
    cache.emplace(key, std::move(P));
    return ref;
  }

  BatchDev batch_dev(const Batch& b, bool split_bwd) {
    BatchDev d{};
    d.sectors = b.d_sectors.as<SectorDev>();
    d.n_sectors = static_cast<int>(b.sdev.size());
    d.dest = b.d_dest.as<int>();
    d.fracf = b.d_fracf.as<float>();
    d.fracd = b.d_fracd.as<double>();
    d.ranges = b.d_ranges.as<int2>();
    d.sdem = sdem.as<float>();
    d.cv = cv.as<int>();
    d.cv_bwd = split_bwd ? cvb.as<int>() : nullptr;
    for (const SectorDev& sd : b.sdev) {
      if (sd.q_lo > 0 || sd.q_hi < sd.skw_rows) d.row_blocks = 1;
    }
    d.umaps = unskew_maps(b, d);
    return d;
  }

  // Tensor maps of the TMA-staged unskew (unskew_tma_kernel), or nullptr for
  // the register-staged kernel: the fused loader, DEM sides
  // that are not a multiple of 4 (a box's first column must be 16-byte
  // aligned: tile column starts are then multiples of 4 in every pre-op
  // orientation), SKS_UNSKEW_TMA=0.
  const void* unskew_maps(const Batch& b, const BatchDev& d) {
    const char* env = std::getenv("SKS_UNSKEW_TMA");
    if ((env != nullptr && env[0] == '0') || b.fused || b.sdev.empty() || d.cv == nullptr) return nullptr;
    if (b.umap_cv == d.cv) return b.umap_ok ? b.d_umaps.p : nullptr;
    b.umap_cv = d.cv;
    b.umap_ok = false;
    std::vector<unsigned char> h(128 * b.sdev.size());
    for (size_t s = 0; s < b.sdev.size(); ++s) {
      const SectorDev& sd = b.sdev[s];
      if (sd.src_rows % 4 != 0 || sd.src_cols % 4 != 0 || sd.sdem_off % 4 != 0) return nullptr;
      // row blocks: the map covers the owned rows only (the TMA zero-fills
      // the others); a sector owning none is never published
      if (sd.q_hi <= sd.q_lo) continue;
      if (!unskew_make_map(h.data() + 128 * s, d.cv + sd.sdem_off + static_cast<long long>(sd.q_lo) * sd.pitch,
                           sd.pitch, sd.q_hi - sd.q_lo, unskew_box_rows(sd.shear_tan))) {
        return nullptr;
      }
    }
    b.d_umaps.ensure(h.size(), device);
    cuda_check(cudaMemcpy(b.d_umaps.p, h.data(), h.size(), cudaMemcpyHostToDevice), "upload tensor maps");
    b.umap_ok = true;
    return b.d_umaps.p;
  }

  void ensure_pools(const Batch& b, bool split_bwd) {
    // + slack: the fixup reads whole 16-position blocks past a row end
    sdem.ensure(static_cast<size_t>(b.pool_elems + 64) * sizeof(float), device);
    cv.ensure(static_cast<size_t>(b.pool_elems) * sizeof(int), device);
    if (split_bwd) cvb.ensure(static_cast<size_t>(b.pool_elems) * sizeof(int), device);
    queue.ensure(static_cast<size_t>(b.fix_cap) * sizeof(unsigned), device);
    fixcnt.ensure(std::max<size_t>(b.items.size(), 1) * sizeof(unsigned), device);
    fixoff.ensure((b.items.size() + 1 + 1024) * sizeof(unsigned), device);  // + prefix block sums
    wm16.ensure(static_cast<size_t>(b.pool_elems / 16 + 1) * sizeof(float), device);
    counters.ensure(kCounterBytes, device);
  }

  // Relocation of a batch from a device DEM. The kernel's TMA tensor maps
  // need a 16-byte aligned base and a row pitch of whole 16-byte units; a DEM
  // without them (dimx not a multiple of 4) is first copied into a pitched
  // buffer (one D2D copy of the DEM, microseconds).
  void relocate(const float* d_dem, int dimy, int dimx, const BatchDev& bd, const Batch& b, cudaStream_t st) {
    const int al = relocate_dem_align();
    const float* src = d_dem;
    long long pitch = dimx;
    if ((reinterpret_cast<uintptr_t>(d_dem) & 15u) != 0 || dimx % al != 0) {
      pitch = round_up(dimx, 32);
      dem_pitched.ensure(static_cast<size_t>(pitch) * dimy * sizeof(float), device);
      cuda_check(cudaMemcpy2DAsync(dem_pitched.p, pitch * sizeof(float), d_dem, dimx * sizeof(float),
                                   dimx * sizeof(float), dimy, cudaMemcpyDeviceToDevice, st),
                 "pitch DEM");
      src = dem_pitched.as<float>();
    }
    cuda_check(launch_relocate_grid(src, dimy, dimx, pitch, bd, b.tiles_x, b.tiles_total, st), "launch relocate");
    ++launches;
  }

  // Global fl(1/d) table for batches whose longest row exceeds the fixup's
  // shared-memory table (long rows); nullptr otherwise.
  const float* ivt_for(const Batch& b, cudaStream_t st) {
    const int need = round_up(std::max(b.lmax_all, b.lmax) + 1, 32);
    if (need <= fixup_smem_table_max()) return nullptr;
    if (need > ivt_len) {
      ivt.ensure(static_cast<size_t>(need) * sizeof(float), device);
      cuda_check(launch_ivt_table(ivt.as<float>(), need, st), "launch ivt table");
      ++launches;
      ivt_len = need;
    }
    return ivt.as<float>();
  }

  ScanArgs scan_args(const Batch& b, const BatchDev& bd, double h0, cudaStream_t st) {
    ScanArgs a{};
    a.b = bd;
    a.items = b.d_items.as<ScanItem>();
    a.n_items = static_cast<int>(b.items.size());
    a.lmax = std::max(b.lmax, 4);
    a.lmax_all = std::max(b.lmax_all, a.lmax);
    a.ivt = ivt_for(b, st);
    a.item_counter = counters.as<unsigned>();
    a.fix_queue = queue.as<unsigned>();
    a.fix_off = b.d_fix_off.as<unsigned>();
    a.fix_cnt = fixcnt.as<unsigned>();
    a.fix_count = counters.as<unsigned>() + 1;
    a.fix_item_counter = counters.as<unsigned>() + 4;
    a.wm16 = wm16.as<float>();
    a.skipped = reinterpret_cast<unsigned long long*>(counters.as<unsigned>() + 8);
    a.h0 = h0;
    a.dbg_j0 = -1;
    a.dbg_h = 0.0;
    a.dbg_vis_fwd = nullptr;
    a.dbg_vis_bwd = nullptr;
    a.force_exact = 0;
    a.fix_group = 1;  // one POV per fixup entry
    a.any_capped = b.any_capped ? 1 : 0;
    return a;
  }

  // scan + fixup of one batch whose sDEM is already in the pool
  // zero_cv: the cv pool must be cleared here (debug paths that upload an
  // sDEM directly); after relocate_kernel it already is (the kernel zeroes
  // the cv cells of every tile it writes).
  // Scan kernel choice per workload shape (dims, ns, max_distance, row
  // block): scan3 over groups of adjacent rows evaluates fewer windows on
  // rough terrain and more on near-flat terrain (config 2 scan: fractal
  // 58.9 ms scan2, 52.9 pairs, 50.2 quads; SmoothedNoise 123.1, 135.6,
  // 155.4), so the first call of a shape scans its first batch with scan2,
  // pairs and quads (each timed on the device, the cv pool re-zeroed in
  // between) and the fastest is kept for every later batch and call; all
  // give identical results. Tuning inside one call keeps later calls
  // uniform (the row-block rebalancers measure them). SKS_SCAN3 = 0 / 1 / 4
  // forces scan2 / pairs / quads.
  struct ScanTune {
    float t[5] = {-1.f, -1.f, -1.f, -1.f, -1.f};  // device time per mode (2, 3, 4)
    int choice = 0;  // 0: undecided, else the mode
  };
  std::map<std::tuple<int, int, int, double, int, int>, ScanTune> tune;

  void scan_batch(const Batch& b, const ScanArgs& a, cudaStream_t st, bool split_bwd, bool zero_cv,
                  int mode = 0) {
    if (zero_cv) {
      cuda_check(cudaMemsetAsync(cv.p, 0, static_cast<size_t>(b.pool_elems) * sizeof(int), st),
                 "memset cv");
    }
    if (split_bwd) {
      cuda_check(cudaMemsetAsync(cvb.p, 0, static_cast<size_t>(b.pool_elems) * sizeof(int), st),
                 "memset cvb");
    }
    cuda_check(cudaMemsetAsync(counters.p, 0, kCounterBytes, st), "memset counters");
    if (!b.items.empty()) {
      cuda_check(cudaMemsetAsync(fixcnt.p, 0, b.items.size() * sizeof(unsigned), st), "memset fix_cnt");
    }
    if (b.n_long > 0) {
      cuda_check(launch_long_rows(a, b.n_long, st), "launch long rows");
      ++launches;
    }
    if (a.n_items > b.n_long) {
      // scan2 sees only the rows that fit its slots (items [n_long, n_items))
      ScanArgs s2 = a;
      s2.items += b.n_long;
      s2.n_items -= b.n_long;
      s2.fix_off += b.n_long;
      s2.fix_cnt += b.n_long;
      const int rows = scan3_rows(b, s2.lmax, mode);
      if (rows > 0) {
        s2.pairs = rows == 4 ? b.d_quads.as<int4>() : b.d_pairs.as<int4>();
        s2.n_pairs = static_cast<int>(rows == 4 ? b.quads.size() : b.pairs.size());
        cuda_check(launch_scan3(s2, scan3_slots(s2.lmax, rows), rows, st), "launch scan3");
      } else {
        cuda_check(launch_scan2(s2, scan2_slots(s2.lmax), st), "launch scan2");
      }
      ++launches;
    }
  }

  // scan3 (row pairs) where at least 2 pair slots fit and the
  // relocation is not fused into the loader; SKS_SCAN3=0 keeps scan2 (read
  // per launch)
  // kernel modes: 2 = scan2 (64 positions of one row per task), 3 = scan3
  // over row pairs, 4 = scan3 over row quads; a group mode
  // needs >= 2 slots of its size
  static bool mode_fits(const Batch& b, int lmax, int mode) {
    if (mode == 2) return true;
    return !b.fused && scan3_slots(lmax, mode == 4 ? 4 : 2) >= 2;
  }
  static int forced_scan() {
    const char* v = std::getenv("SKS_SCAN3");  // 0: scan2, 1 / 2: pairs, 4: quads
    if (v == nullptr) return 0;
    const std::string m(v);
    return m == "0" ? 2 : m == "4" ? 4 : 3;
  }
  // rows per group of the scan3 launch for `mode` (0: scan2)
  static int scan3_rows(const Batch& b, int lmax, int mode) {
    const int f = forced_scan();
    if (f != 0) mode = f;
    if (mode == 0) mode = 3;
    if (mode == 2 || !mode_fits(b, lmax, mode)) {
      return mode == 4 && mode_fits(b, lmax, 3) ? 2 : 0;
    }
    return mode == 4 ? 4 : 2;
  }

  void fixup_batch(const ScanArgs& a, cudaStream_t st) {
    if (a.n_items == 0) return;
    cuda_check(launch_fixup(a, fixoff.as<unsigned>(), st), "launch fixup");
    launches += 3;
  }

  // Host entry point: the last batch's map pass runs in row chunks and each
  // chunk's D2H starts on copy_stream while the next chunk is computed.
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t chunk_ev[4] = {};

  void ensure_copy_stream() {
    if (copy_stream) return;
    cuda_check(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking), "copy stream");
    for (cudaEvent_t& e : chunk_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  }

  ~sks_context() {
    for (cudaEvent_t& e : ev) {
      if (e) cudaEventDestroy(e);
    }
    for (cudaEvent_t& e : chunk_ev) {
      if (e) cudaEventDestroy(e);
    }
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (own_stream) cudaStreamDestroy(own_stream);
    if (h_check) cudaFreeHost(h_check);
  }
};

namespace {

std::mutex g_ctx_mu;
std::map<int, std::unique_ptr<sks_context>> g_default;

sks_context* default_context(int device) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  auto it = g_default.find(device);
  if (it != g_default.end()) return it->second.get();
  auto ctx = std::make_unique<sks_context>();
  ctx->device = device;
  ctx->activate();
  cuda_check(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking), "stream");
  cuda_check(cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device), "attr");
  for (cudaEvent_t& e : ctx->ev) cuda_check(cudaEventCreate(&e), "event");
  sks_context* raw = ctx.get();
  g_default.emplace(device, std::move(ctx));
  return raw;
}

void require_valid(const float* dem, int dimy, int dimx, double cellsize,
                   const sks_run_config* cfg) {
  if (!cfg) throw std::invalid_argument("null run config");
  if (!dem) throw std::invalid_argument("null DEM");
  std::string err =
      validate_inputs(dem, dimy, dimx, cellsize, nullptr, cfg->ns, cfg->h0, cfg->max_distance, cfg->n_gpus);
  if (!err.empty()) throw std::invalid_argument(err);
}

// Elevation magnitudes the FP32 filter's proof covers: every
// nonzero |e| and h0 in [2^-40, 2^40]. Outside, the whole run uses the exact
// FP64 path.
bool filter_preconditions_hold(const float* dem, size_t n, double h0) {
  const double lo = std::ldexp(1.0, -40), hi = std::ldexp(1.0, 40);
  if (h0 != 0.0 && (h0 < lo || h0 > hi)) return false;
  for (size_t i = 0; i < n; ++i) {
    const double a = std::fabs(static_cast<double>(dem[i]));
    if (a != 0.0 && (a < lo || a > hi)) return false;
  }
  return true;
}

double elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cuda_check(cudaEventElapsedTime(&ms, a, b), "event time");
  return ms * 1e-3;
}

// Core: run the given sectors on device data. Accumulates into d_map.
void run_sectors(sks_context* ctx, const float* d_dem, int dimy, int dimx, double cellsize,
                 const sks_run_config* cfg, std::vector<int> sectors, double* d_map,
                 cudaStream_t st, sks_stats* stats, bool force_exact, int part = 0, int nparts = 1,
                 const std::vector<double>& cuts = {}, BatchDev* defer_last = nullptr) {
  std::sort(sectors.begin(), sectors.end());
  sectors.erase(std::unique(sectors.begin(), sectors.end()), sectors.end());
  for (int k : sectors) {
    if (k < 0 || k >= cfg->ns / 2) throw std::out_of_range("sector index out of range");
  }
  Plans& P = ctx->plans_for(dimy, dimx, cfg->ns, cellsize, cfg->max_distance, sectors, part, nparts, cuts);
  const long long launches0 = ctx->launches;
  double t_skew = 0, t_scan = 0, t_fix = 0, t_unskew = 0;
  // scan kernel choice (sks_context::ScanTune): time one call of each where
  // scan3 fits, then keep the faster
  auto& tn = ctx->tune[std::make_tuple(dimy, dimx, cfg->ns, cfg->max_distance, part, nparts)];
  const bool tune_now = tn.choice == 0 && sks_context::forced_scan() == 0;
  long long flagged = 0, evals = 0, skipped = 0;
  for (auto& bp : P.batches) {
    Batch& b = *bp;
    ctx->ensure_pools(b, false);
    BatchDev bd = ctx->batch_dev(b, false);
    const bool fused = b.fused;  // relocation inside scan2's row loader
    if (fused) bd.dem = d_dem;
    ScanArgs a = ctx->scan_args(b, bd, cfg->h0, st);
    a.force_exact = force_exact ? 1 : 0;
    if (stats) cuda_check(cudaEventRecord(ctx->ev[0], st), "event");
    if (!fused) ctx->relocate(d_dem, dimy, dimx, bd, b, st);
    if (stats) cuda_check(cudaEventRecord(ctx->ev[1], st), "event");
    if (tune_now && tn.choice == 0) {
      // first call of the shape: scan this batch with every kernel mode that
      // fits (each timed on the device, the cv pool re-zeroed in between:
      // every trial leaves the same cv, queue and window maxima), keep the
      // fastest for every later batch and call
      int best = 0;
      float best_ms = 0.f;
      int ntrial = 0;
      for (int m : {2, 3, 4}) {
        const int lm = std::max(b.lmax, 4);
        if (!sks_context::mode_fits(b, lm, m)) continue;
        if (ntrial++ > 0) {
          cuda_check(cudaMemsetAsync(ctx->cv.p, 0, static_cast<size_t>(b.pool_elems) * sizeof(int), st),
                     "memset cv");
        }
        // module loads and attribute calls stay outside the timed region
        const int rows = sks_context::scan3_rows(b, lm, m);
        cuda_check(rows > 0 ? prepare_scan3(lm, rows, b.any_capped ? 1 : 0) : prepare_scan2(lm, b.any_capped ? 1 : 0),
                   "prepare scan");
        cuda_check(cudaEventRecord(ctx->ev[5], st), "event");
        ctx->scan_batch(b, a, st, false, false, m);
        cuda_check(cudaEventRecord(ctx->ev[6], st), "event");
        cuda_check(cudaEventSynchronize(ctx->ev[6]), "sync");
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, ctx->ev[5], ctx->ev[6]), "elapsed");
        tn.t[m] = ms;
        if (best == 0 || ms < best_ms) {
          best = m;
          best_ms = ms;
        }
      }
      tn.choice = best;  // the pool holds the last trial's state (the same for every mode)
    } else {
      ctx->scan_batch(b, a, st, false, false, tn.choice);
    }
    if (stats) cuda_check(cudaEventRecord(ctx->ev[2], st), "event");
    ctx->fixup_batch(a, st);
    if (stats) cuda_check(cudaEventRecord(ctx->ev[3], st), "event");
    if (defer_last != nullptr && !stats && &bp == &P.batches.back()) {
      *defer_last = bd;  // the caller runs this batch's map pass (chunked)
      continue;
    }
    cuda_check(launch_unskew(bd, nullptr, d_map, dimy, dimx, st), "launch unskew");
    ++ctx->launches;
    if (stats) {
      cuda_check(cudaEventRecord(ctx->ev[4], st), "event");
      cuda_check(cudaEventSynchronize(ctx->ev[4]), "sync");
      t_skew += elapsed(ctx->ev[0], ctx->ev[1]);
      t_scan += elapsed(ctx->ev[1], ctx->ev[2]);
      t_fix += elapsed(ctx->ev[2], ctx->ev[3]);
      t_unskew += elapsed(ctx->ev[3], ctx->ev[4]);
      unsigned cnt[10] = {};
      cuda_check(cudaMemcpy(cnt, ctx->counters.p, sizeof(cnt), cudaMemcpyDeviceToHost), "counters");
      flagged += cnt[1];
      if (std::getenv("SKS_FIXUP_REPORT") != nullptr && !b.items.empty()) {
        // distribution of queued POV groups over rows (diagnostics)
        std::vector<unsigned> fc(b.items.size());
        cuda_check(cudaMemcpy(fc.data(), ctx->fixcnt.p, fc.size() * sizeof(unsigned), cudaMemcpyDeviceToHost),
                   "fix_cnt");
        long long rows = 0, chunks = 0, tot = 0, work = 0, maxw = 0;
        unsigned mx = 0;
        for (size_t i = 0; i < fc.size(); ++i) {
          fc[i] = (fc[i] & 0xffffu) + (fc[i] >> 16);  // forward | backward << 16
          if (fc[i] == 0) continue;
          const int2 r = b.ranges[b.sdev[b.items[i].s].row_off + b.items[i].q];
          ++rows;
          tot += fc[i];
          mx = std::max(mx, fc[i]);
          chunks += (fc[i] * a.fix_group + 31) / 32;
          const long long w = static_cast<long long>((fc[i] * a.fix_group + 31) / 32) * (r.y - r.x);
          work += w;
          maxw = std::max(maxw, w);
        }
        std::fprintf(stderr,
                     "fixup: %lld groups in %lld rows (of %zu), max %u per row, %lld warp-chunks, "
                     "chunk-work %lld (max %lld)\n",
                     tot, rows, fc.size(), mx, chunks, work, maxw);
      }
      unsigned long long sk = 0;
      std::memcpy(&sk, cnt + 8, sizeof(sk));
      skipped += static_cast<long long>(sk);
    }
    evals += b.target_evals;
  }
  if (stats) {
    stats->skew_seconds += t_skew;
    stats->scan_seconds += t_scan;
    stats->fixup_seconds += t_fix;
    stats->unskew_seconds += t_unskew;
    stats->sectors += static_cast<int>(sectors.size());
    stats->batches += static_cast<int>(P.batches.size());
    stats->kernel_launches += ctx->launches - launches0;
    stats->target_evals += evals;
    stats->flagged_groups += flagged;
    stats->skipped_target_slots += skipped;
    if (!P.batches.empty()) {
      const Batch& lb = *P.batches.back();
      const int rows = sks_context::scan3_rows(lb, std::max(lb.lmax, 4), tn.choice);
      stats->scan_kernel = rows == 4 ? 4 : rows == 2 ? 3 : 2;
    }
  }
}

// Cell scan of a device DEM (dem_check_kernel) with one small D2H: throws
// the reference's invalid_argument for the first non-finite cell, then
// validates the config (validate(Dem) before validate(RunConfig),
// engine.cpp:68-81); returns true when the FP32 filter's preconditions do
// not hold (every POV then takes the exact FP64 path).
bool device_check(sks_context* ctx, const float* d_dem, int dimy, int dimx, const sks_run_config* cfg,
                  cudaStream_t st) {
  const size_t n = static_cast<size_t>(dimy) * dimx;
  ctx->check.ensure(2 * sizeof(unsigned long long), ctx->device);
  if (ctx->h_check == nullptr) {
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_check), 2 * sizeof(unsigned long long),
                             cudaHostAllocDefault),
               "pinned check");
  }
  cuda_check(cudaMemsetAsync(ctx->check.p, 0xff, sizeof(unsigned long long), st), "memset check");
  cuda_check(cudaMemsetAsync(static_cast<char*>(ctx->check.p) + 8, 0, sizeof(unsigned long long), st),
             "memset check");
  cuda_check(launch_dem_check(d_dem, static_cast<long long>(n), ctx->check.as<unsigned long long>(), st),
             "launch dem check");
  ++ctx->launches;
  cuda_check(cudaMemcpyAsync(ctx->h_check, ctx->check.p, 2 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, st),
             "D2H check");
  cuda_check(cudaStreamSynchronize(st), "sync check");
  if (ctx->h_check[0] != ~0ull) {
    throw std::invalid_argument(nonfinite_message(static_cast<long long>(ctx->h_check[0]), dimx));
  }
  const std::string err = validate_config(cfg->ns, cfg->h0, cfg->max_distance, cfg->n_gpus);
  if (!err.empty()) throw std::invalid_argument(err);
  const double plo = std::ldexp(1.0, -40), phi = std::ldexp(1.0, 40);
  return ctx->h_check[1] != 0 || (cfg->h0 != 0.0 && (cfg->h0 < plo || cfg->h0 > phi));
}

void total_host(sks_context* ctx, const float* dem, int dimy, int dimx, double cellsize,
                const sks_run_config* cfg, int raw, double* out, sks_stats* stats) {
  auto t0 = std::chrono::steady_clock::now();
  if (!cfg) throw std::invalid_argument("null run config");
  if (!dem) throw std::invalid_argument("null DEM");
  if (!out) throw std::invalid_argument("null output");
  // validate(Dem) then validate(RunConfig) (engine.cpp:68-81), in the
  // reference's order; the O(N) cell scan runs on device after the upload
  std::string err = validate_grid_header(dimy, dimx, cellsize);
  if (!err.empty()) throw std::invalid_argument(err);
  ctx->activate();
  std::lock_guard<std::mutex> lk(ctx->mu);
  const size_t n = static_cast<size_t>(dimy) * dimx;
  cudaStream_t st = ctx->own_stream;
  ctx->dem.ensure(n * sizeof(float), ctx->device);
  ctx->map.ensure(n * sizeof(double), ctx->device);
  cuda_check(cudaMemcpyAsync(ctx->dem.p, dem, n * sizeof(float), cudaMemcpyHostToDevice, st), "H2D dem");
  const bool exact = device_check(ctx, ctx->dem.as<float>(), dimy, dimx, cfg, st);
  cuda_check(cudaMemsetAsync(ctx->map.p, 0, n * sizeof(double), st), "memset map");
  std::vector<int> all(cfg->ns / 2);
  std::iota(all.begin(), all.end(), 0);
  sks_stats local{};
  local.kernel_launches += 1;  // dem_check
  // Without stats, the last batch's unskew + scale run in row chunks and each
  // chunk's D2H overlaps the next chunk's compute (the map rows a chunk of
  // DEM tiles writes are final once that chunk's unskew and scale are done).
  BatchDev last{};
  last.n_sectors = -1;
  run_sectors(ctx, ctx->dem.as<float>(), dimy, dimx, cellsize, cfg, all, ctx->map.as<double>(), st,
              stats ? &local : nullptr, exact, 0, 1, {}, stats ? nullptr : &last);
  const double factor = area_scale_factor(cfg->ns, cellsize, cfg->units);
  double* map = ctx->map.as<double>();
  if (last.n_sectors >= 0) {
    ctx->ensure_copy_stream();
    const int tr = unskew_tile_rows();
    const int tiles = (dimy + tr - 1) / tr;
    const int nch = std::min(4, tiles);
    for (int c = 0; c < nch; ++c) {
      const int t0 = tiles * c / nch, t1 = tiles * (c + 1) / nch;
      const int y0 = t0 * tr, y1 = std::min(dimy, t1 * tr);
      const size_t off = static_cast<size_t>(y0) * dimx, cnt = static_cast<size_t>(y1 - y0) * dimx;
      cuda_check(launch_unskew(last, nullptr, map, dimy, dimx, st, t0, t1 - t0), "launch unskew");
      ++ctx->launches;
      if (!raw) {
        cuda_check(launch_scale(map + off, static_cast<long long>(cnt), factor, st), "launch scale");
        ++ctx->launches;
      }
      cuda_check(cudaEventRecord(ctx->chunk_ev[c], st), "event");
      cuda_check(cudaStreamWaitEvent(ctx->copy_stream, ctx->chunk_ev[c], 0), "wait");
      cuda_check(cudaMemcpyAsync(out + off, map + off, cnt * sizeof(double), cudaMemcpyDeviceToHost, ctx->copy_stream),
                 "D2H map");
    }
    cuda_check(cudaStreamSynchronize(ctx->copy_stream), "sync");
  } else {
    if (!raw) {
      cuda_check(launch_scale(map, static_cast<long long>(n), factor, st), "launch scale");
      ++ctx->launches;
      local.kernel_launches += 1;
    }
    cuda_check(cudaMemcpyAsync(out, ctx->map.p, n * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H map");
  }
  cuda_check(cudaStreamSynchronize(st), "sync");
  if (stats) {
    local.h2d_bytes = static_cast<long long>(n * sizeof(float));
    local.d2h_bytes = static_cast<long long>(n * sizeof(double));
    local.total_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *stats = local;
  }
}

// Single-sector debug batch from a custom plan; the sDEM is produced by the
// relocation kernel from `grid` (pre_ops applied through the plan's map).
struct DebugBatch {
  std::vector<SectorPlanH> plans;
  std::unique_ptr<Batch> batch;
};

DebugBatch debug_batch(SectorPlanH plan, int device) {
  DebugBatch d;
  d.plans.push_back(std::move(plan));
  d.batch = make_batch(d.plans, {0}, device);
  return d;
}

}  // namespace

extern "C" {

const char* sks_last_error(void) { return g_error.c_str(); }

void sks_set_last_error(const char* msg) { g_error = msg ? msg : ""; }

const char* sks_version(void) { return "skewshed_b200 0.2.0 (sm_100a)"; }

int sks_scan_row_limit(void) { return scan2_max_row(); }

int sks_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

sks_status sks_plan_sector(int k, int ns, int dimy, int dimx, sks_sector_plan* out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null output");
    SectorPlanH p = plan_sector(k, ns, dimy, dimx, 1.0, 0.0);
    out->sector_index = p.k;
    out->ns = p.ns;
    out->sector_deg = p.sector_deg;
    out->shear_deg = p.shear_deg;
    out->shear_tan = p.shear_tan;
    out->n_ops = p.n_ops;
    std::copy(p.ops, p.ops + 3, out->ops);
    out->rows = p.rows;
    out->cols = p.cols;
    out->src_rows = p.src_rows;
    out->src_cols = p.src_cols;
    std::copy(p.map, p.map + 6, out->to_source);
    out->base = p.base;
    out->skw_rows = p.skw_rows;
  });
}

void sks_shear_params(double shear_tan, int j, int* dest, double* frac) {
  shear_params(shear_tan, j, dest, frac);
}

int sks_distance_cap_cells(double max_distance, double shear_tan, double cellsize) {
  return distance_cap_cells(max_distance, shear_tan, cellsize);
}

double sks_area_scale_factor(int ns, double cellsize, int units) {
  return area_scale_factor(ns, cellsize, units);
}

sks_status sks_row_ranges(int rows, int cols, double shear_tan, int* ranges, int* skw_rows_out) {
  return guarded([&] {
    SectorPlanH p = plan_custom(rows, cols, shear_tan);
    if (skw_rows_out) *skw_rows_out = p.skw_rows;
    if (ranges) {
      for (int q = 0; q < p.skw_rows; ++q) {
        ranges[2 * q] = p.ranges[q].first;
        ranges[2 * q + 1] = p.ranges[q].last;
      }
    }
  });
}

long long sks_sector_target_evals(int k, int ns, int dimy, int dimx, double cellsize,
                                  double max_distance) {
  long long r = -1;
  guarded([&] { r = plan_sector(k, ns, dimy, dimx, cellsize, max_distance).target_evals; });
  return r;
}

sks_status sks_partition_sectors(int ns, int dimy, int dimx, double cellsize, double max_distance,
                                 int world, int* owner) {
  return guarded([&] {
    if (world < 1 || !owner) throw std::invalid_argument("world must be >= 1");
    if (ns < 2 || ns % 2) throw std::invalid_argument("ns must be an even integer >= 2");
    std::vector<long long> work(ns / 2);
    for (int k = 0; k < ns / 2; ++k) {
      work[k] = plan_sector(k, ns, dimy, dimx, cellsize, max_distance).target_evals;
    }
    std::vector<int> o = partition_lpt(work, world);
    std::copy(o.begin(), o.end(), owner);
  });
}

sks_status sks_make_synthetic(int kind, int dimy, int dimx, uint32_t seed, float* out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null output");
    make_synthetic(kind, dimy, dimx, seed, out);
  });
}

sks_status sks_validate(const float* dem, int dimy, int dimx, double cellsize, const float* nodata,
                        const sks_run_config* cfg) {
  return guarded([&] {
    if (!cfg || !dem) throw std::invalid_argument("null argument");
    std::string err =
        validate_inputs(dem, dimy, dimx, cellsize, nodata, cfg->ns, cfg->h0, cfg->max_distance, cfg->n_gpus);
    if (!err.empty()) throw std::invalid_argument(err);
  });
}

sks_status sks_context_create(int device, sks_context** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null output");
    auto ctx = std::make_unique<sks_context>();
    ctx->device = device;
    ctx->activate();
    cuda_check(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking), "stream");
    cuda_check(cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device), "attr");
    for (cudaEvent_t& e : ctx->ev) cuda_check(cudaEventCreate(&e), "event");
    *out = ctx.release();
  });
}

void sks_context_destroy(sks_context* ctx) { delete ctx; }

sks_status sks_context_run_sectors(sks_context* ctx, const float* d_dem, int dimy, int dimx,
                                   double cellsize, const sks_run_config* cfg, const int* sectors,
                                   int n_sectors, double* d_map, void* stream, sks_stats* stats) {
  return guarded([&] {
    if (!ctx || !cfg || !d_dem || !d_map) throw std::invalid_argument("null argument");
    const std::string err = validate_grid_header(dimy, dimx, cellsize);
    if (!err.empty()) throw std::invalid_argument(err);
    ctx->activate();
    std::lock_guard<std::mutex> lk(ctx->mu);
    std::vector<int> ks(sectors, sectors + n_sectors);
    sks_stats local{};
    const bool exact = device_check(ctx, d_dem, dimy, dimx, cfg, static_cast<cudaStream_t>(stream));
    local.kernel_launches += 1;  // dem_check
    run_sectors(ctx, d_dem, dimy, dimx, cellsize, cfg, ks, d_map, static_cast<cudaStream_t>(stream),
                stats ? &local : nullptr, exact);
    if (stats) *stats = local;
  });
}

sks_status sks_context_run_rows(sks_context* ctx, const float* d_dem, int dimy, int dimx,
                                double cellsize, const sks_run_config* cfg, int part, int nparts,
                                double* d_map, void* stream, sks_stats* stats) {
  return sks_context_run_rows_cuts(ctx, d_dem, dimy, dimx, cellsize, cfg, part, nparts, nullptr, d_map, stream,
                                   stats);
}

sks_status sks_context_run_rows_cuts(sks_context* ctx, const float* d_dem, int dimy, int dimx,
                                     double cellsize, const sks_run_config* cfg, int part, int nparts,
                                     const double* cuts, double* d_map, void* stream, sks_stats* stats) {
  return guarded([&] {
    if (!ctx || !cfg || !d_dem || !d_map) throw std::invalid_argument("null argument");
    if (nparts < 1 || part < 0 || part >= nparts) throw std::out_of_range("row part out of range");
    std::vector<double> cv;
    if (cuts != nullptr && nparts > 1) {
      cv.assign(cuts, cuts + nparts + 1);
      for (int b = 0; b <= nparts; ++b) {
        if (!(cv[b] >= 0.0 && cv[b] <= 1.0) || (b > 0 && cv[b] < cv[b - 1])) {
          throw std::invalid_argument("row cuts must be non-decreasing fractions in [0, 1]");
        }
      }
    }
    const std::string err = validate_grid_header(dimy, dimx, cellsize);
    if (!err.empty()) throw std::invalid_argument(err);
    ctx->activate();
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (cfg->ns < 2 || cfg->ns % 2) throw std::invalid_argument("ns must be an even integer >= 2");
    std::vector<int> all(cfg->ns / 2);
    std::iota(all.begin(), all.end(), 0);
    sks_stats local{};
    const bool exact = device_check(ctx, d_dem, dimy, dimx, cfg, static_cast<cudaStream_t>(stream));
    local.kernel_launches += 1;  // dem_check
    run_sectors(ctx, d_dem, dimy, dimx, cellsize, cfg, all, d_map, static_cast<cudaStream_t>(stream),
                stats ? &local : nullptr, exact, part, nparts, cv);
    if (stats) *stats = local;
  });
}

sks_status sks_context_scale(sks_context* ctx, double* d_map, long long n, int ns, double cellsize,
                             int units, void* stream) {
  return guarded([&] {
    if (!ctx || !d_map) throw std::invalid_argument("null argument");
    ctx->activate();
    cuda_check(launch_scale(d_map, n, area_scale_factor(ns, cellsize, units),
                            static_cast<cudaStream_t>(stream)),
               "launch scale");
    ++ctx->launches;
  });
}

sks_status sks_context_total_viewshed(sks_context* ctx, const float* dem, int dimy, int dimx,
                                      double cellsize, const sks_run_config* cfg, int raw,
                                      double* out, sks_stats* stats) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    total_host(ctx, dem, dimy, dimx, cellsize, cfg, raw, out, stats);
  });
}

// n_gpus > 1 (or SKS_ALL_GPUS with several visible): one host thread per GPU
// and one NCCL reduce (multi.cu); else the single-device path.
static sks_status total_dispatch(const float* dem, int dimy, int dimx, double cellsize, const sks_run_config* cfg, int raw,
                          double* out, sks_stats* stats) {
  std::vector<int> devs(64);
  int nd = 0;
  const sks_status s = guarded([&] {
    require_valid(dem, dimy, dimx, cellsize, cfg);  // before touching the device
    nd = sks_config_devices(cfg, devs.data(), static_cast<int>(devs.size()));
    if (nd > static_cast<int>(devs.size())) throw std::invalid_argument("too many GPUs requested");
    if (nd <= 1) total_host(default_context(cfg->device), dem, dimy, dimx, cellsize, cfg, raw, out, stats);
  });
  if (s != SKS_OK || nd <= 1) return s;
  return sks_total_viewshed_devices(dem, dimy, dimx, cellsize, cfg, devs.data(), nd, raw, out, stats);
}

sks_status sks_total_viewshed(const float* dem, int dimy, int dimx, double cellsize,
                              const sks_run_config* cfg, double* out_vs, sks_stats* stats) {
  return total_dispatch(dem, dimy, dimx, cellsize, cfg, 0, out_vs, stats);
}

sks_status sks_total_viewshed_raw(const float* dem, int dimy, int dimx, double cellsize,
                                  const sks_run_config* cfg, double* out_raw, sks_stats* stats) {
  return total_dispatch(dem, dimy, dimx, cellsize, cfg, 1, out_raw, stats);
}

sks_status sks_sector_sweep(const float* dem, int dimy, int dimx, double cellsize,
                            const sks_run_config* cfg, int k, double* out) {
  return guarded([&] {
    require_valid(dem, dimy, dimx, cellsize, cfg);
    if (k < 0 || k >= cfg->ns / 2) throw std::out_of_range("sector index out of range");
    if (!out) throw std::invalid_argument("null output");
    sks_context* ctx = default_context(cfg->device);
    ctx->activate();
    std::lock_guard<std::mutex> lk(ctx->mu);
    const size_t n = static_cast<size_t>(dimy) * dimx;
    cudaStream_t st = ctx->own_stream;
    ctx->dem.ensure(n * sizeof(float), ctx->device);
    ctx->map.ensure(n * sizeof(double), ctx->device);
    cuda_check(cudaMemcpyAsync(ctx->dem.p, dem, n * sizeof(float), cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemsetAsync(ctx->map.p, 0, n * sizeof(double), st), "memset");
    run_sectors(ctx, ctx->dem.as<float>(), dimy, dimx, cellsize, cfg, {k}, ctx->map.as<double>(), st,
                nullptr, !filter_preconditions_hold(dem, n, cfg->h0));
    cuda_check(cudaMemcpyAsync(out, ctx->map.p, n * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
  });
}

namespace {

// Relocation of one debug batch from a host grid; values copied back with
// every cell (the pool is zeroed first so empty tiles read as +0).
void debug_relocate(sks_context* ctx, Batch& b, const float* grid, size_t grid_elems,
                    float* values) {
  cudaStream_t st = ctx->own_stream;
  ctx->ensure_pools(b, false);
  ctx->dem.ensure(grid_elems * sizeof(float), ctx->device);
  cuda_check(cudaMemcpyAsync(ctx->dem.p, grid, grid_elems * sizeof(float), cudaMemcpyHostToDevice, st),
             "H2D grid");
  cuda_check(cudaMemsetAsync(ctx->sdem.p, 0, static_cast<size_t>(b.pool_elems) * sizeof(float), st),
             "memset sdem");
  BatchDev bd = ctx->batch_dev(b, false);
  const SectorDev& s0 = b.sdev[0];
  ctx->relocate(ctx->dem.as<float>(), s0.src_rows, s0.src_cols, bd, b, st);
  const SectorDev& sd = b.sdev[0];
  cuda_check(cudaMemcpy2DAsync(values, sizeof(float) * sd.cols, ctx->sdem.p, sizeof(float) * sd.pitch,
                               sizeof(float) * sd.cols, sd.skw_rows, cudaMemcpyDeviceToHost, st),
             "D2H sdem");
  cuda_check(cudaStreamSynchronize(st), "sync");
}

}  // namespace

sks_status sks_build_sector_sdem(const float* dem, int dimy, int dimx, int k, int ns, int device,
                                 float* values, int* ranges) {
  return guarded([&] {
    if (!dem || !values) throw std::invalid_argument("null argument");
    SectorPlanH p = plan_sector(k, ns, dimy, dimx, 1.0, 0.0);
    sks_context* ctx = default_context(device);
    ctx->activate();
    std::lock_guard<std::mutex> lk(ctx->mu);
    DebugBatch d = debug_batch(p, device);
    debug_relocate(ctx, *d.batch, dem, static_cast<size_t>(dimy) * dimx, values);
    if (ranges) {
      for (int q = 0; q < p.skw_rows; ++q) {
        ranges[2 * q] = p.ranges[q].first;
        ranges[2 * q + 1] = p.ranges[q].last;
      }
    }
  });
}

sks_status sks_build_skw(const float* g, int rows, int cols, double shear_tan, int device,
                         float* values, int* ranges, int* base_out) {
  return guarded([&] {
    if (!g || !values) throw std::invalid_argument("null argument");
    SectorPlanH p = plan_custom(rows, cols, shear_tan);
    sks_context* ctx = default_context(device);
    ctx->activate();
    std::lock_guard<std::mutex> lk(ctx->mu);
    DebugBatch d = debug_batch(p, device);
    debug_relocate(ctx, *d.batch, g, static_cast<size_t>(rows) * cols, values);
    if (ranges) {
      for (int q = 0; q < p.skw_rows; ++q) {
        ranges[2 * q] = p.ranges[q].first;
        ranges[2 * q + 1] = p.ranges[q].last;
      }
    }
    if (base_out) *base_out = p.base;
  });
}

namespace {

// Scan of a caller-provided sDEM (values + ranges) with split fwd/bwd output.
void debug_scan(sks_context* ctx, const float* values, const int* ranges, int skw_rows, int cols,
                double shear_tan, double h0, int max_dd, int dbg_j0, double dbg_h,
                uint8_t* vis_fwd_host, uint8_t* vis_bwd_host, int vis_len, std::vector<int>& cvf,
                std::vector<int>& cvb) {
  cudaStream_t st = ctx->own_stream;
  // A one-sector batch with the caller's geometry.
  SectorPlanH p;
  p.rows = p.src_rows = skw_rows;
  p.cols = p.src_cols = cols;
  p.base = 0;
  p.skw_rows = skw_rows;
  p.shear_tan = shear_tan;
  p.correction = 1.0 + shear_tan * shear_tan;
  p.max_dd = max_dd;
  p.dest.assign(cols, 0);
  p.fracf.assign(cols, 0.f);
  p.fracd.assign(cols, 0.0);
  p.ranges.resize(skw_rows);
  for (int q = 0; q < skw_rows; ++q) p.ranges[q] = RowRange{ranges[2 * q], ranges[2 * q + 1]};
  std::vector<SectorPlanH> plans{p};
  auto b = make_batch(plans, {0}, ctx->device);
  ctx->ensure_pools(*b, true);
  const SectorDev& sd = b->sdev[0];
  cuda_check(cudaMemcpy2DAsync(ctx->sdem.p, sizeof(float) * sd.pitch, values, sizeof(float) * cols,
                               sizeof(float) * cols, skw_rows, cudaMemcpyHostToDevice, st),
             "H2D sdem");
  BatchDev bd = ctx->batch_dev(*b, true);
  ScanArgs a = ctx->scan_args(*b, bd, h0, st);
  uint8_t* dvis = nullptr;
  if (dbg_j0 >= 0) {
    a.dbg_j0 = dbg_j0;
    a.dbg_h = dbg_h;
    if (vis_fwd_host || vis_bwd_host) {
      ctx->vis.ensure(2 * static_cast<size_t>(std::max(vis_len, 1)), ctx->device);
      dvis = ctx->vis.as<uint8_t>();
      cuda_check(cudaMemsetAsync(dvis, 0xff, 2 * static_cast<size_t>(std::max(vis_len, 1)), st), "memset vis");
      a.dbg_vis_fwd = dvis;
      a.dbg_vis_bwd = dvis + std::max(vis_len, 1);
    }
  }
  ctx->scan_batch(*b, a, st, true, true);
  ctx->fixup_batch(a, st);
  cvf.assign(static_cast<size_t>(skw_rows) * cols, 0);
  cvb.assign(static_cast<size_t>(skw_rows) * cols, 0);
  cuda_check(cudaMemcpy2DAsync(cvf.data(), sizeof(int) * cols, ctx->cv.p, sizeof(int) * sd.pitch,
                               sizeof(int) * cols, skw_rows, cudaMemcpyDeviceToHost, st),
             "D2H cvf");
  cuda_check(cudaMemcpy2DAsync(cvb.data(), sizeof(int) * cols, ctx->cvb.p, sizeof(int) * sd.pitch,
                               sizeof(int) * cols, skw_rows, cudaMemcpyDeviceToHost, st),
             "D2H cvb");
  if (dvis) {
    if (vis_fwd_host) cuda_check(cudaMemcpyAsync(vis_fwd_host, dvis, vis_len, cudaMemcpyDeviceToHost, st), "D2H vis");
    if (vis_bwd_host) cuda_check(cudaMemcpyAsync(vis_bwd_host, dvis + std::max(vis_len, 1), vis_len, cudaMemcpyDeviceToHost, st), "D2H vis");
  }
  cuda_check(cudaStreamSynchronize(st), "sync");
}

}  // namespace

sks_status sks_sector_viewshed(const float* values, const int* ranges, int skw_rows, int cols,
                               double shear_tan, double h0, int max_dd, int device, double* out,
                               int* cv_fwd, int* cv_bwd) {
  return guarded([&] {
    if (!values || !ranges || !out) throw std::invalid_argument("null argument");
    if (skw_rows < 1 || cols < 1) throw std::invalid_argument("empty sDEM");
    if (max_dd < 0) throw std::invalid_argument("max_dd must be >= 0");
    sks_context* ctx = default_context(device);
    ctx->activate();
    std::lock_guard<std::mutex> lk(ctx->mu);
    std::vector<int> cvf, cvb;
    debug_scan(ctx, values, ranges, skw_rows, cols, shear_tan, h0, max_dd, -1, 0.0, nullptr, nullptr,
               0, cvf, cvb);
    // skwVS = (fwd + bwd) * (1 + tan^2) on device (scan.cpp:67-82)
    const size_t n = static_cast<size_t>(skw_rows) * cols;
    DevBuf df, db, dout;
    df.ensure(n * sizeof(int), device);
    db.ensure(n * sizeof(int), device);
    dout.ensure(n * sizeof(double), device);
    cudaStream_t st = ctx->own_stream;
    cuda_check(cudaMemcpyAsync(df.p, cvf.data(), n * sizeof(int), cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(db.p, cvb.data(), n * sizeof(int), cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(launch_cv_to_vs(df.as<int>(), db.as<int>(), dout.as<double>(), static_cast<long long>(n),
                               1.0 + shear_tan * shear_tan, st),
               "launch cv_to_vs");
    cuda_check(cudaMemcpyAsync(out, dout.p, n * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    if (cv_fwd) std::copy(cvf.begin(), cvf.end(), cv_fwd);
    if (cv_bwd) std::copy(cvb.begin(), cvb.end(), cv_bwd);
  });
}

sks_status sks_linear_viewshed_row(const float* row, int n, int first, int last, int j0, double h,
                                   int dir, int max_dd, int device, double* cv_out,
                                   uint8_t* visible_out, int* n_visible) {
  return guarded([&] {
    if (!row || !cv_out) throw std::invalid_argument("null argument");
    if (!(0 <= first && first <= j0 && j0 < last && last <= n)) {
      throw std::invalid_argument("require 0 <= first <= j0 < last <= n");
    }
    if (max_dd < 0) throw std::invalid_argument("max_dd must be >= 0");
    const int D = std::min(max_dd, dir == 0 ? last - 1 - j0 : j0 - first);
    if (n_visible) *n_visible = D;
    if (D <= 0) {
      *cv_out = 0.0;
      return;
    }
    sks_context* ctx = default_context(device);
    ctx->activate();
    std::lock_guard<std::mutex> lk(ctx->mu);
    int rr[2] = {first, last};
    std::vector<int> cvf, cvb;
    std::vector<uint8_t> vf(D), vb(D);
    // both directions of POV j0 are scanned; each capture buffer holds a
    // whole row so the longer direction cannot overrun the other's bytes
    vf.assign(n, 0);
    vb.assign(n, 0);
    debug_scan(ctx, row, rr, 1, n, 0.0, 0.0, max_dd, j0, h, visible_out ? vf.data() : nullptr,
               visible_out ? vb.data() : nullptr, n, cvf, cvb);
    *cv_out = static_cast<double>(dir == 0 ? cvf[j0] : cvb[j0]);
    if (visible_out) std::copy_n(dir == 0 ? vf.data() : vb.data(), D, visible_out);
  });
}

sks_status sks_unskew_accumulate(const double* skw_vs, int skw_rows, int cols, int k, int ns,
                                 int dimy, int dimx, int device, double* out) {
  return guarded([&] {
    if (!skw_vs || !out) throw std::invalid_argument("null argument");
    SectorPlanH p = plan_sector(k, ns, dimy, dimx, 1.0, 0.0);
    if (skw_rows != p.skw_rows || cols != p.cols) {
      std::ostringstream os;
      os << "skewed grid shape " << skw_rows << "x" << cols << " does not match plan ("
         << p.skw_rows << "x" << p.cols << ")";
      throw std::invalid_argument(os.str());
    }
    sks_context* ctx = default_context(device);
    ctx->activate();
    std::lock_guard<std::mutex> lk(ctx->mu);
    DebugBatch d = debug_batch(p, device);
    Batch& b = *d.batch;
    // skw_vs is read with the batch's cell indexing: give it pitch = cols.
    b.sdev[0].pitch = cols;
    b.sdev[0].sdem_off = 0;
    cuda_check(cudaMemcpy(b.d_sectors.p, b.sdev.data(), sizeof(SectorDev), cudaMemcpyHostToDevice),
               "upload");
    const size_t nv = static_cast<size_t>(skw_rows) * cols;
    const size_t nm = static_cast<size_t>(dimy) * dimx;
    DevBuf dvs, dmap;
    dvs.ensure(nv * sizeof(double), device);
    dmap.ensure(nm * sizeof(double), device);
    cudaStream_t st = ctx->own_stream;
    cuda_check(cudaMemcpyAsync(dvs.p, skw_vs, nv * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(dmap.p, out, nm * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
    BatchDev bd = ctx->batch_dev(b, false);
    cuda_check(launch_unskew_from_vs(bd, dvs.as<double>(), dmap.as<double>(), dimy, dimx, st),
               "launch unskew");
    cuda_check(cudaMemcpyAsync(out, dmap.p, nm * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
  });
}

// ---- ESRI ASCII grid I/O (sks_io.cpp) ----------------------------------

struct sks_ascii_grid {
  AsciiGrid g;
};

sks_status sks_ascii_grid_read(const char* path, sks_ascii_grid** out) {
  return guarded([&] {
    if (!path || !out) throw std::invalid_argument("null argument");
    *out = nullptr;
    auto h = std::make_unique<sks_ascii_grid>();
    h->g = read_ascii_grid_file(path);
    *out = h.release();
  });
}

sks_status sks_ascii_grid_parse(const char* text, size_t len, const char* source_name,
                                sks_ascii_grid** out) {
  return guarded([&] {
    if ((!text && len) || !out) throw std::invalid_argument("null argument");
    *out = nullptr;
    auto h = std::make_unique<sks_ascii_grid>();
    h->g = parse_ascii_grid(text ? text : "", len, source_name ? source_name : "<input>");
    *out = h.release();
  });
}

sks_status sks_ascii_grid_header(const sks_ascii_grid* grid, sks_grid_header* out) {
  return guarded([&] {
    if (!grid || !out) throw std::invalid_argument("null argument");
    const AsciiGrid& g = grid->g;
    *out = sks_grid_header{g.nrows, g.ncols, g.xllcorner, g.yllcorner, g.cellsize, g.has_nodata ? 1 : 0, g.nodata};
  });
}

sks_status sks_ascii_grid_values(const sks_ascii_grid* grid, float* out) {
  return guarded([&] {
    if (!grid || !out) throw std::invalid_argument("null argument");
    std::copy(grid->g.values.begin(), grid->g.values.end(), out);
  });
}

void sks_ascii_grid_free(sks_ascii_grid* grid) { delete grid; }

sks_status sks_float_grid_read(const char* path, sks_ascii_grid** out) {
  return guarded([&] {
    if (!path || !out) throw std::invalid_argument("null argument");
    *out = nullptr;
    auto h = std::make_unique<sks_ascii_grid>();
    h->g = read_float_grid(path);
    *out = h.release();
  });
}

sks_status sks_write_float_grid(const char* path, const float* values, const sks_grid_header* hdr) {
  return guarded([&] {
    if (!path || !values || !hdr) throw std::invalid_argument("null argument");
    write_float_grid(path, values, hdr->nrows, hdr->ncols, hdr->xllcorner, hdr->yllcorner, hdr->cellsize,
                     hdr->has_nodata ? &hdr->nodata : nullptr);
  });
}

sks_status sks_write_ascii_grid_dem(const char* path, const float* values, const sks_grid_header* hdr) {
  return guarded([&] {
    if (!path || !values || !hdr) throw std::invalid_argument("null argument");
    write_ascii_grid_dem(path, values, hdr->nrows, hdr->ncols, hdr->xllcorner, hdr->yllcorner, hdr->cellsize,
                         hdr->has_nodata ? &hdr->nodata : nullptr);
  });
}

sks_status sks_write_ascii_grid_vs(const char* path, const double* values, int nrows, int ncols, int units_in,
                                   int units_out, double cellsize, double xllcorner, double yllcorner) {
  return guarded([&] {
    if (!path || !values) throw std::invalid_argument("null argument");
    // convert_units (dem.cpp:24-34)
    const double factor = units_in == units_out ? 1.0 : (units_out == SKS_UNITS_KM2 ? 1e-6 : 1e6);
    write_ascii_grid_vs(path, values, nrows, ncols, factor, xllcorner, yllcorner, cellsize);
  });
}

}  // extern "C"

// ---- rotational-sweep reference on the GPU (oracle.cpp:74-194) -----------

namespace {

void require_inside(int dimy, int dimx, int i, int j) {  // oracle.cpp:14-21
  if (i < 0 || i >= dimy || j < 0 || j >= dimx) {
    std::ostringstream os;
    os << "observer (" << i << ", " << j << ") outside grid " << dimy << "x" << dimx;
    throw std::out_of_range(os.str());
  }
}

// singular_viewshed (oracle.cpp:108-129) of npov observers — povs (i, j
// pairs) or, when null, the linear cell indices [0, npov) — times
// unit_factor, into out[npov] (host). Observers run in batches whose
// per-azimuth sums fit in ~1 GiB.
void sweep_areas(sks_context* ctx, const float* dem, int dimy, int dimx, double cellsize, const int* povs,
                 long long npov, double h0, int ns, double max_distance, double unit_factor, double* out) {
  if (npov <= 0) return;
  const double max_cells = max_distance != 0.0 ? max_distance / cellsize : INFINITY;
  const SweepTable tab = build_sweep_table(ns, dimy, dimx, max_cells);
  static_assert(sizeof(SweepStep) == sizeof(SweepStepDev), "table layout");
  ctx->activate();
  std::lock_guard<std::mutex> lk(ctx->mu);
  cudaStream_t st = ctx->own_stream;
  const size_t n = static_cast<size_t>(dimy) * dimx;
  DevBuf d_tab, d_len, d_povs, d_buf, d_out;
  ctx->dem.ensure(n * sizeof(float), ctx->device);
  d_tab.ensure(tab.steps.size() * sizeof(SweepStep), ctx->device);
  d_len.ensure(tab.len.size() * sizeof(int), ctx->device);
  d_out.ensure(static_cast<size_t>(npov) * sizeof(double), ctx->device);
  const long long batch = std::max(1LL, std::min(npov, (1LL << 27) / tab.ndir));
  d_buf.ensure(static_cast<size_t>(batch) * tab.ndir * sizeof(double), ctx->device);
  cuda_check(cudaMemcpyAsync(ctx->dem.p, dem, n * sizeof(float), cudaMemcpyHostToDevice, st), "H2D dem");
  cuda_check(cudaMemcpyAsync(d_tab.p, tab.steps.data(), tab.steps.size() * sizeof(SweepStep),
                             cudaMemcpyHostToDevice, st),
             "H2D sweep table");
  cuda_check(cudaMemcpyAsync(d_len.p, tab.len.data(), tab.len.size() * sizeof(int), cudaMemcpyHostToDevice, st),
             "H2D sweep lengths");
  // FP32 filter preconditions (elevation magnitudes)
  ctx->check.ensure(2 * sizeof(unsigned long long), ctx->device);
  cuda_check(cudaMemsetAsync(ctx->check.p, 0xff, sizeof(unsigned long long), st), "memset check");
  cuda_check(cudaMemsetAsync(static_cast<char*>(ctx->check.p) + 8, 0, sizeof(unsigned long long), st),
             "memset check");
  cuda_check(launch_dem_check(ctx->dem.as<float>(), static_cast<long long>(n), ctx->check.as<unsigned long long>(),
                              st),
             "launch dem check");
  unsigned long long chk[2] = {0, 0};
  cuda_check(cudaMemcpyAsync(chk, ctx->check.p, sizeof(chk), cudaMemcpyDeviceToHost, st), "D2H check");
  cuda_check(cudaStreamSynchronize(st), "sync check");
  const bool filter = chk[1] == 0 && !(h0 != 0.0 && (std::fabs(h0) < std::ldexp(1.0, -40) ||
                                                     std::fabs(h0) > std::ldexp(1.0, 40)));
  if (povs) {
    d_povs.ensure(static_cast<size_t>(npov) * sizeof(int2), ctx->device);
    cuda_check(cudaMemcpyAsync(d_povs.p, povs, static_cast<size_t>(npov) * sizeof(int2), cudaMemcpyHostToDevice, st),
               "H2D povs");
  }
  const double pi_over_ns = std::numbers::pi / ns;
  for (long long b0 = 0; b0 < npov; b0 += batch) {
    const int nb = static_cast<int>(std::min(batch, npov - b0));
    cuda_check(launch_sweep(ctx->dem.as<float>(), dimy, dimx, d_tab.as<SweepStepDev>(), d_len.as<int>(),
                            tab.stride, tab.ndir, povs ? d_povs.as<int2>() + b0 : nullptr, b0, nb, h0,
                            d_buf.as<double>(), filter && std::getenv("SKS_SWEEP_EXACT") == nullptr, st),
               "launch sweep");
    cuda_check(launch_sweep_sum(d_buf.as<double>(), tab.ndir, nb, pi_over_ns, cellsize, unit_factor,
                                d_out.as<double>(), b0, st),
               "launch sweep sum");
    ctx->launches += 2;
  }
  cuda_check(cudaMemcpyAsync(out, d_out.p, static_cast<size_t>(npov) * sizeof(double), cudaMemcpyDeviceToHost, st),
             "D2H areas");
  cuda_check(cudaStreamSynchronize(st), "sync sweep");
}

void require_sector_count(int ns) {  // oracle.cpp:110-112
  if (ns < 2 || ns % 2 != 0) throw std::invalid_argument("sector count must be an even integer >= 2");
}

}  // namespace

extern "C" {

sks_status sks_singular_viewshed(const float* dem, int dimy, int dimx, double cellsize, int i, int j, double h0,
                                 int ns, double max_distance, int device, double* area) {
  return guarded([&] {
    if (!dem || !area) throw std::invalid_argument("null argument");
    require_inside(dimy, dimx, i, j);
    require_sector_count(ns);
    const int p[2] = {i, j};
    sweep_areas(default_context(device), dem, dimy, dimx, cellsize, p, 1, h0, ns, max_distance, 1.0, area);
  });
}

sks_status sks_multi_viewshed(const float* dem, int dimy, int dimx, double cellsize, const int* povs, int npovs,
                              double h0, int ns, double max_distance, int device, double* pov_area,
                              double* grid, double* total_area) {
  return guarded([&] {
    if (!dem || (npovs > 0 && !povs)) throw std::invalid_argument("null argument");
    // the reference validates inside the per-observer loop (oracle.cpp:131-141):
    // the first observer's position, then ns, then the remaining observers
    for (int t = 0; t < npovs; ++t) {
      require_inside(dimy, dimx, povs[2 * t], povs[2 * t + 1]);
      if (t == 0) require_sector_count(ns);
    }
    std::vector<double> area(static_cast<size_t>(std::max(npovs, 0)));
    sweep_areas(default_context(device), dem, dimy, dimx, cellsize, povs, npovs, h0, ns, max_distance, 1.0,
                area.data());
    if (grid) std::fill(grid, grid + static_cast<size_t>(dimy) * dimx, 0.0);
    double total = 0.0;
    for (int t = 0; t < npovs; ++t) {  // list order (oracle.cpp:137-139)
      if (grid) grid[static_cast<size_t>(povs[2 * t]) * dimx + povs[2 * t + 1]] += area[t];
      total += area[t];
    }
    if (pov_area) std::copy(area.begin(), area.end(), pov_area);
    if (total_area) *total_area = total;
  });
}

sks_status sks_total_viewshed_reference(const float* dem, int dimy, int dimx, double cellsize,
                                        const float* nodata, const sks_run_config* cfg, int force,
                                        double* out) {
  return guarded([&] {
    if (!dem || !cfg || !out) throw std::invalid_argument("null argument");
    // validate(Dem), validate(RunConfig) (oracle.cpp:145-153)
    std::string err = validate_grid_header(dimy, dimx, cellsize);
    if (!err.empty()) throw std::invalid_argument(err);
    const size_t n = static_cast<size_t>(dimy) * dimx;
    for (size_t c = 0; c < n; ++c) {
      if (nodata && dem[c] == *nodata) continue;
      if (!std::isfinite(dem[c])) throw std::invalid_argument(nonfinite_message(static_cast<long long>(c), dimx));
    }
    err = validate_config(cfg->ns, cfg->h0, cfg->max_distance, cfg->n_gpus);
    if (!err.empty()) throw std::invalid_argument(err);
    const long long cells = static_cast<long long>(dimy) * dimx;
    if (cells > SKS_REFERENCE_CELL_GUARD && !force) {  // oracle.cpp:154-163
      std::ostringstream os;
      os << "reference total viewshed on " << dimy << "x" << dimx << " (" << cells
         << " cells) refused: the sweep costs on the order of ns * N^(3/2) elevation tests and grids above "
         << SKS_REFERENCE_CELL_GUARD << " cells take a long time; pass force to run anyway";
      throw std::runtime_error(os.str());
    }
    sweep_areas(default_context(cfg->device), dem, dimy, dimx, cellsize, nullptr, cells, cfg->h0, cfg->ns,
                cfg->max_distance, cfg->units == SKS_UNITS_KM2 ? 1e-6 : 1.0, out);
  });
}

sks_status sks_linear_scan(const float* dem, int dimy, int dimx, int i0, int j0, double pov_h, double azimuth_deg,
                           double max_dist_cells, int device, double* cv, double* rings, int cap, int* nrings) {
  return guarded([&] {
    if (!dem || !cv) throw std::invalid_argument("null argument");
    require_inside(dimy, dimx, i0, j0);
    const std::vector<SweepStep> tab = ray_table(dimy, dimx, azimuth_deg, max_dist_cells);
    sks_context* ctx = default_context(device);
    ctx->activate();
    std::lock_guard<std::mutex> lk(ctx->mu);
    cudaStream_t st = ctx->own_stream;
    const size_t n = static_cast<size_t>(dimy) * dimx;
    const int rcap = std::max(cap, 0);
    DevBuf d_tab, d_out;
    ctx->dem.ensure(n * sizeof(float), ctx->device);
    d_tab.ensure(std::max<size_t>(tab.size(), 1) * sizeof(SweepStep), ctx->device);
    d_out.ensure((1 + 2 * static_cast<size_t>(rcap)) * sizeof(double) + sizeof(int), ctx->device);
    cuda_check(cudaMemcpyAsync(ctx->dem.p, dem, n * sizeof(float), cudaMemcpyHostToDevice, st), "H2D dem");
    if (!tab.empty()) {
      cuda_check(cudaMemcpyAsync(d_tab.p, tab.data(), tab.size() * sizeof(SweepStep), cudaMemcpyHostToDevice, st),
                 "H2D ray");
    }
    double* dcv = d_out.as<double>();
    double* drings = dcv + 1;
    int* dn = reinterpret_cast<int*>(drings + 2 * rcap);
    cuda_check(launch_linear_scan(ctx->dem.as<float>(), dimy, dimx, i0, j0, pov_h, d_tab.as<SweepStepDev>(),
                                  static_cast<int>(tab.size()), dcv, drings, rcap, dn, st),
               "launch linear scan");
    ++ctx->launches;
    std::vector<double> host(1 + 2 * static_cast<size_t>(rcap));
    int nr = 0;
    cuda_check(cudaMemcpyAsync(host.data(), dcv, host.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(&nr, dn, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    *cv = host[0];
    if (nrings) *nrings = nr;
    if (rings) std::copy(host.begin() + 1, host.begin() + 1 + 2 * std::min(nr, rcap), rings);
  });
}

sks_status sks_axis_point_set(int dimy, int dimx, int i0, int j0, double azimuth_deg, int* ij, int cap,
                              int* count) {
  return guarded([&] {
    if (!count) throw std::invalid_argument("null argument");
    require_inside(dimy, dimx, i0, j0);
    const std::vector<SweepStep> pts = axis_points(dimy, dimx, i0, j0, azimuth_deg);
    *count = static_cast<int>(pts.size());
    for (int t = 0; t < std::min(cap, *count) && ij; ++t) {
      ij[2 * t] = pts[t].di;
      ij[2 * t + 1] = pts[t].dj;
    }
  });
}

sks_status sks_random_povs(int dimy, int dimx, int count, uint32_t seed, int* ij) {
  return guarded([&] {
    if (count > 0 && !ij) throw std::invalid_argument("null argument");
    random_povs(dimy, dimx, count, seed, ij);
  });
}

sks_status sks_fill_nodata_nearest(const float* dem, int dimy, int dimx, float nodata, float* out) {
  return guarded([&] {
    if ((!dem || !out) && static_cast<long long>(dimy) * dimx > 0) throw std::invalid_argument("null argument");
    if (dimy < 0 || dimx < 0) throw std::invalid_argument("grid dimensions must be non-negative");
    fill_nodata_nearest(dem, dimy, dimx, nodata, out);
  });
}

sks_status sks_write_heatmap(const char* path, const double* values, int rows, int cols, int palette) {
  return guarded([&] {
    if (!path || (!values && static_cast<long long>(rows) * cols > 0)) throw std::invalid_argument("null argument");
    if (palette != SKS_PALETTE_GRAY && palette != SKS_PALETTE_BLUE_RED) throw std::invalid_argument("unknown palette");
    write_heatmap(path, values, rows, cols, palette);
  });
}

}  // extern "C"
