// Device-side data layout shared by the sm_100a kernels and the engine.
//
// HBM layout for one batch of sectors:
//   * dem      : dimy x dimx float32, row-major (the caller's DEM, resident).
//   * sdem pool: for each sector slot s, skw_rows_s x pitch_s float32
//                (pitch a multiple of 32 floats = 128 B), at sdem_off_s.
//   * cv pool  : same geometry as the sdem pool, int32 per skewed cell: the
//                exact integer ring sum cv = sum over visible targets of
//                (2*dd+1), forward + backward (SURVEY §7 hard part 2).
//   * column tables (per sector, at col_off): dest int32, fracf float32,
//                fracd float64 (skew.cpp:155-158, 222-227).
//   * row ranges (per sector, at row_off): int2 [first, last).
//   * map      : dimy x dimx float64, the raw total-viewshed accumulator.
#pragma once

#include <cstdint>

namespace sks {

struct SectorDev {
  int k;
  int rows, cols;          // pre_ops space
  int src_rows, src_cols;  // DEM space
  int base, skw_rows, pitch;
  int max_dd;
  int col_off;   // into dest / fracf / fracd
  int row_off;   // into ranges
  int q_lo, q_hi;  // skewed rows this run owns (row-block sharding; all: 0, skw_rows)
  int map[6];    // pre (i, j) -> DEM (si, sj)
  int inv[6];    // DEM (si, sj) -> pre (i, j)
  double correction;  // 1 + tan^2
  double shear_tan;   // shear_params (skew.cpp:97-101) on device: the fused loader
  long long sdem_off;  // element offset of this sector in the sdem / cv pools
};

// One unit of scan work: skewed row q of sector slot s (L >= 2).
struct ScanItem {
  int s;
  int q;
};

struct BatchDev {
  const SectorDev* sectors;
  int n_sectors;
  const int* dest;
  const float* fracf;
  const double* fracd;
  const int2* ranges;
  float* sdem;
  int* cv;
  int* cv_bwd;  // debug: backward scan results kept apart (nullptr = cv)
  // Fused relocation (scan2 only): the row loader builds each sDEM row from
  // this DEM (writing it to sdem for the fixup and zeroing the row's cv
  // range), and the unskew treats cv outside the row ranges as 0. nullptr:
  // rows come from sdem written by relocate_kernel, which zeroes cv.
  const float* dem;
  int row_blocks;  // some sector owns only a block of its rows (multi-GPU run_rows)
  // Unskew TMA staging (unskew_tma_kernel): one 2-D tensor map per sector
  // over its owned cv rows (dims {pitch, q_hi - q_lo}, box {32,
  // unskew_box_rows(tan)}), CUtensorMap objects (128 B each) in global
  // memory; nullptr: the register-staged unskew_pipe_kernel (the fused
  // loader, DEM sides not a multiple of 4 — a box's column start must be
  // 16-byte aligned).
  const void* umaps;
};

// Rows of the unskew TMA box of a sector: a 32x32 DEM tile reads skewed rows
// [p_min, p_min + 33 + d_hi - d_lo), d_hi - d_lo <= floor(31 tan) + 1; one
// more for the rounding of fl(j tan). Host and device evaluate the same IEEE
// product.
__host__ __device__ inline int unskew_box_rows(double shear_tan) {
  return 35 + static_cast<int>(31.0 * shear_tan);
}

struct ScanArgs {
  BatchDev b;
  const ScanItem* items;
  int n_items;
  int lmax;               // longest row length in the batch
  unsigned* item_counter; // zero before launch
  // Fixup queue: item it owns the segment fix_queue[fix_off[it] ..) of
  // 2*L entries (the exact bound: one per POV and direction);
  // fix_cnt[it] counts its entries. Entry = dir << 31 | group index.
  unsigned* fix_queue;
  const unsigned* fix_off;
  unsigned* fix_cnt;      // n_items counters, zero before launch
  unsigned* fix_count;    // total flagged groups (stats), zero before launch
  unsigned* fix_item_counter;  // fixup kernel work counter, zero before launch
  // Window maxima of every scanned row (forward orientation, 16 positions
  // each) at (sdem_off + q * pitch) / 16 + w, written by scan2's row loader
  // for the fixup's per-POV skip; nullptr: no skip (distance-lockstep scan).
  float* wm16;
  unsigned long long* skipped;     // lane-target slots decided by the hidden-block skip
  double h0;
  // debug single-POV mode (sks_linear_viewshed_row): POV j0 of row 0 of
  // sector slot 0 uses the absolute height h_abs; its per-target decisions
  // are written to vis (one byte per target, forward or backward).
  int dbg_j0;
  double dbg_h;
  uint8_t* dbg_vis_fwd;
  uint8_t* dbg_vis_bwd;
  int force_exact;        // every POV group goes through the FP64 fixup
  int any_capped;         // some row's distance cap is shorter than the row
  int fix_group;          // POVs per fixup entry (1: an entry is one POV)
  // Rows too long for scan2's shared-memory slots ("long rows", items
  // [0, n_long) of the fixup's item list): every POV of such a row, both
  // directions, goes through the fixup kernel (long_rows_kernel fills their
  // queue segments and window maxima).
  int lmax_all;           // longest row of the batch incl. long rows (fixup table)
  const float* ivt;       // global fl(1/d) table (lmax_all + 32 entries) when the
                          // fixup's shared-memory table would not fit; else nullptr
  // scan3 (row groups of 2 or 4 adjacent skewed rows q0 .. q0+kR-1 of one
  // sector): pairs[i] = the rows' items (-1: not scanned), longest group
  // first; the items index `items`/fix_off/fix_cnt
  const int4* pairs;
  int n_pairs;
};

__host__ __device__ inline unsigned pack_fix(unsigned dir, unsigned g) { return (dir << 31) | g; }

// Kernel entry points (launch wrappers). All return the launch error.
// grid: (tiles_total, n_sectors); tile t -> (t / tiles_x, t % tiles_x)
// dem: dem_rows x dem_cols floats with a row pitch of dem_pitch floats; the
// base 16-byte aligned and dem_pitch a multiple of relocate_dem_align() (the
// TMA tensor maps' stride rule); else cudaErrorMisalignedAddress.
int launch_relocate_grid(const float* dem, int dem_rows, int dem_cols, long long dem_pitch,
                         const BatchDev& b, int tiles_x, int tiles_total, void* stream);
int relocate_dem_align();
int relocate_tile_rows();
int relocate_tile_cols();
int launch_fixup(const ScanArgs& a, unsigned* off, void* stream);  // fixup.cu (off: n_items + 1)
// Queue every POV (both directions) of items [0, n_long) for the fixup and
// write their rows' window maxima (fixup.cu).
int launch_long_rows(const ScanArgs& a, int n_long, void* stream);
int launch_ivt_table(float* ivt, int n, void* stream);  // ivt[d] = fl(1/d)
int fixup_smem_table_max();  // longest row whose fl(1/d) table the fixup keeps in shared memory
int scan2_slots(int lmax);  // 0: rows too long for the target-lockstep kernel
int scan2_max_row();        // longest row scan2 can hold (>= 1 slot)
size_t scan2_smem_bytes(int lmax, int nslots);
int launch_scan2(const ScanArgs& a, int nslots, void* stream);
int scan3_slots(int lmax, int rows);  // row-group slots that fit (rows 2 or 4; 0: rows too long)
int launch_scan3(const ScanArgs& a, int nslots, int rows, void* stream);
int prepare_scan2(int lmax, int any_capped);             // kernel attributes only (before a timed launch)
int prepare_scan3(int lmax, int rows, int any_capped);
// tile rows [tile_row0, tile_row0 + tile_rows) of the map (32 DEM rows each;
// tile_rows < 0: to the end)
int launch_unskew(const BatchDev& b, const float* unused, double* map,
                  int dimy, int dimx, void* stream, int tile_row0 = 0, int tile_rows = -1);
int unskew_tile_rows();
// Encode the unskew tensor map of one sector into tm (128 bytes, host
// memory): cv rows [0, rows) of `pitch` int32 starting at base. false: the
// driver rejected it (the caller keeps the register-staged kernel).
bool unskew_make_map(void* tm, const int* base, int pitch, int rows, int box_rows);
int launch_unskew_from_vs(const BatchDev& b, const double* skw_vs,
                          double* map, int dimy, int dimx, void* stream);
int launch_scale(double* map, long long n, double factor, void* stream);
int launch_dem_check(const float* dem, long long n, unsigned long long* res, void* stream);
int launch_cv_to_vs(const int* cvf, const int* cvb, double* out,
                    long long n, double correction, void* stream);

// rotational sweep (sweep.cu); same layout as the host SweepStep
struct SweepStepDev {
  int di, dj;
  double dist;
  float inv;
  int pad;
};
int launch_sweep(const float* dem, int rows, int cols, const SweepStepDev* tab, const int* len,
                 int stride, int ndir, const int2* povs, long long pov0, int npov, double h0,
                 double* buf, bool filter, void* stream);
int launch_linear_scan(const float* dem, int rows, int cols, int i0, int j0, double pov_h,
                       const SweepStepDev* tab, int len, double* out_cv, double* rings, int cap,
                       int* nrings, void* stream);
int launch_sweep_sum(const double* buf, int ndir, int npov, double pi_over_ns, double cellsize,
                     double unit_factor, double* out, long long out_off, void* stream);

}  // namespace sks
