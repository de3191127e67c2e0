// Host-side sector planning for the B200 sDEM pipeline.
//
// Everything here is O(rows + cols) per sector and independent of the
// elevations, so plans are built once per geometry and cached by the engine.
// The arithmetic mirrors the reference bit for bit (plan_sector's std::tan,
// shear_params' truncation, build_skw's float weights), because the device
// kernels consume these tables verbatim.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace sks {

inline constexpr int kNoCap = 2147483647;        // scan.hpp:15 kNoDistanceCap
inline constexpr float kFullWeightTol = 1e-6f;   // skew.hpp:70

struct RowRange {
  int first;
  int last;
};

// One sector, fully planned. Mirrors SectorPlan (skew.hpp:29-41) plus the
// per-column shear tables of build_skw/unskew_accumulate (skew.cpp:155-158,
// 222-227) and the row ranges of build_skw (skew.cpp:185-195).
struct SectorPlanH {
  int k = 0;
  int ns = 0;
  double sector_deg = 0.0;
  double shear_deg = 0.0;
  double shear_tan = 0.0;
  int n_ops = 0;
  int ops[3] = {0, 0, 0};  // 0 Transpose, 1 FlipCols, 2 FlipRows
  int rows = 0, cols = 0;          // pre_ops space
  int src_rows = 0, src_cols = 0;  // DEM space
  int map[6] = {1, 0, 0, 0, 1, 0};  // to_source: ii, ij, ci, ji, jj, cj
  int inv[6] = {1, 0, 0, 0, 1, 0};  // DEM (si, sj) -> pre (i, j), same layout
  int base = 0;
  int skw_rows = 0;
  int max_dd = kNoCap;
  double correction = 1.0;  // 1 + tan^2 (scan.cpp:67-69)
  std::vector<int> dest;       // floor(tan * j)
  std::vector<float> fracf;    // (float)frac, build_skw's weights
  std::vector<double> fracd;   // frac, unskew_accumulate's weights
  std::vector<RowRange> ranges;  // per skewed row, [first, last)
  long long target_evals = 0;    // exact scan work of the sector
  int q_lo = 0, q_hi = -1;       // owned skewed rows [q_lo, q_hi); q_hi < 0: all
};

// Row-block sharding: the skewed rows of a sector split into
// nparts contiguous blocks of equal exact scan work; block `part` of the
// plan's rows. Sets p.q_lo / p.q_hi.
// Row block `part` of `nparts` of the sector's skewed rows, balanced by the
// row cost model; with cuts (nparts + 1 non-decreasing fractions, 0 .. 1)
// block b holds the rows whose preceding cost lies in [cuts[b], cuts[b+1])
// of the total (measured-time rebalancing, distributed.py).
void set_row_block(SectorPlanH& p, int part, int nparts, const double* cuts = nullptr);

// skew.cpp:16-19
int base_offset(int src_rows, int cols, double shear_tan);
// skew.cpp:97-101
void shear_params(double shear_tan, int j, int* dest, double* frac);
// engine.cpp:29-36 (max_distance <= 0 means off)
int distance_cap_cells(double max_distance, double shear_tan, double cellsize);
// engine.cpp:103-107
double area_scale_factor(int ns, double cellsize, int units);

// skew.cpp:23-95 plus tables. Throws std::invalid_argument /
// std::out_of_range exactly where plan_sector does.
SectorPlanH plan_sector(int k, int ns, int dimy, int dimx, double cellsize,
                        double max_distance);
// A sector with identity pre_ops and an arbitrary shear in [0, 1]
// (build_skw on a grid already in pre_ops space, skew.cpp:144-150).
SectorPlanH plan_custom(int rows, int cols, double shear_tan);

// build_skw's row ranges (skew.cpp:185-195) from the float weights implied by
// (dest, fracf): exact for any geometry, O((rows + cols) * alpha).
std::vector<RowRange> row_ranges(int rows, int cols, int base,
                                 const std::vector<int>& dest,
                                 const std::vector<float>& fracf);

// Exact target evaluations of one skewed row of length L, capped at max_dd.
long long row_target_evals(long long L, long long max_dd);

// Longest-processing-time assignment of sectors to ranks.
std::vector<int> partition_lpt(const std::vector<long long>& work, int world);

// dem.cpp:118-173 kinds 0..3, plus kind 4 = Fractal (diamond-square).
void make_synthetic(int kind, int dimy, int dimx, uint32_t seed, float* out);

// dem.cpp:36-87 + engine.cpp:68-81; returns "" when valid, else the first
// error message with the reference's wording.
std::string validate_inputs(const float* dem, int dimy, int dimx,
                            double cellsize, const float* nodata, int ns,
                            double h0, double max_distance, int n_gpus = 1);
// The same checks in pieces, for the device-side cell scan (total_host):
// grid header (dims, cellsize), the first non-finite cell's message, config.
std::string validate_grid_header(int dimy, int dimx, double cellsize);
std::string nonfinite_message(long long idx, int dimx);
std::string validate_config(int ns, double h0, double max_distance, int n_gpus = 1);

}  // namespace sks
