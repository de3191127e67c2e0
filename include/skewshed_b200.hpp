// skewshed_b200 — C++ facade over the C ABI (skewshed_b200.h).
//
// Restores the reference's entry points (proj/include/skewshed/*.hpp) with
// the same names, argument meaning and exception types, so reference-style
// C++ callers switch by changing the namespace and linking
// libskewshed_b200.so:
//   engine.hpp:42-53  total_viewshed_raw, total_viewshed, sector_sweep,
//                     accumulate_into, reduce_ordered, area_scale_factor
//   skew.hpp:45-89    plan_sector, shear_params, build_skw, unskew_accumulate
//   scan.hpp:27-45    linear_viewshed_row, sector_viewshed, area_scale
//   dem.hpp:13-71     Dem, RunConfig, VsGrid, Units, make_synthetic, validate
// std::invalid_argument / std::out_of_range / std::runtime_error are thrown
// for SKS_INVALID_ARGUMENT / SKS_OUT_OF_RANGE / everything else.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <functional>
#include <istream>
#include <limits>
#include <iterator>
#include <numbers>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "skewshed_b200.h"

namespace skewshed_b200 {

// ascii_grid.hpp:15-18
class GridFormatError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(sks_status s) {
  if (s == SKS_OK) return;
  std::string msg = sks_last_error();
  if (s == SKS_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (s == SKS_FORMAT_ERROR) throw GridFormatError(msg);
  if (s == SKS_OUT_OF_RANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

// grid.hpp:11-63: row-major, row 0 north, col 0 west.
template <typename T>
class Grid {
 public:
  Grid() = default;
  Grid(int rows, int cols, T fill = T{}) { reset(rows, cols, fill); }
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  std::size_t size() const { return data_.size(); }
  bool empty() const { return data_.empty(); }
  T& operator()(int i, int j) { return data_[static_cast<std::size_t>(i) * cols_ + j]; }
  const T& operator()(int i, int j) const { return data_[static_cast<std::size_t>(i) * cols_ + j]; }
  T* row(int i) { return data_.data() + static_cast<std::size_t>(i) * cols_; }
  const T* row(int i) const { return data_.data() + static_cast<std::size_t>(i) * cols_; }
  std::vector<T>& data() { return data_; }
  const std::vector<T>& data() const { return data_; }
  void reset(int rows, int cols, T fill = T{}) {
    if (rows < 0 || cols < 0) throw std::invalid_argument("grid dimensions must be non-negative");
    rows_ = rows;
    cols_ = cols;
    data_.assign(static_cast<std::size_t>(rows) * cols, fill);
  }
  bool same_shape(const Grid& o) const { return rows_ == o.rows_ && cols_ == o.cols_; }
  friend bool operator==(const Grid&, const Grid&) = default;

 private:
  int rows_ = 0, cols_ = 0;
  std::vector<T> data_;
};

enum class Units { SquareMeters = SKS_UNITS_M2, SquareKilometers = SKS_UNITS_KM2 };
enum class SyntheticKind { Flat = 0, Ramp = 1, Cone = 2, SmoothedNoise = 3, Fractal = 4 };
enum class ScanDir { Forward = SKS_SCAN_FORWARD, Backward = SKS_SCAN_BACKWARD };
enum class AxisOp { Transpose = 0, FlipCols = 1, FlipRows = 2 };
inline constexpr int kNoDistanceCap = SKS_NO_DISTANCE_CAP;

// dem.hpp:13-17
struct GridOrigin {
  double easting = 0.0;
  double northing = 0.0;
  std::string zone;
};

struct Dem {
  Grid<float> values;
  double cellsize = 1.0;
  std::optional<float> nodata;
  GridOrigin origin;
  int dimy() const { return values.rows(); }
  int dimx() const { return values.cols(); }
};

// dem.hpp:40-46. `workers` (host threads sharing one call) becomes n_gpus
// (GPUs sharing one call from `device` on; SKS_ALL_GPUS = every visible one):
// total_viewshed then runs one host thread per GPU and one NCCL reduce.
struct RunConfig {
  int ns = 360;
  double h0 = 1.5;
  int device = 0;
  int n_gpus = 1;
  std::optional<double> max_distance;
  Units units = Units::SquareKilometers;
  sks_run_config to_c() const {
    return sks_run_config{ns, h0, max_distance.value_or(0.0), static_cast<int>(units), device, n_gpus};
  }
};

struct VsGrid {
  Grid<double> values;
  Units units = Units::SquareMeters;
};

struct EngineStats : sks_stats {
  EngineStats() : sks_stats{} {}
};

struct SectorResult {
  int sector_index = 0;
  Grid<double> contribution;
};

using ProgressFn = std::function<void(int sector_index, double wall_seconds)>;

struct SectorPlan : sks_sector_plan {
  std::pair<int, int> to_source_ij(int i, int j) const {
    const int* m = to_source;
    return {m[0] * i + m[1] * j + m[2], m[3] * i + m[4] * j + m[5]};
  }
};

struct ShearParams {
  int dest;
  double frac;
};

struct SkwGrid {
  int src_rows = 0;
  int cols = 0;
  int base = 0;
  double shear_tan = 0.0;
  Grid<float> values;
  std::vector<std::pair<int, int>> row_ranges;
  int skw_rows() const { return values.rows(); }
};

inline Dem make_synthetic(SyntheticKind kind, int dimy, int dimx, double cellsize,
                          std::uint32_t seed = 0) {
  if (!(cellsize > 0.0)) throw std::invalid_argument("synthetic cellsize must be positive");
  Dem d;
  d.cellsize = cellsize;
  d.values.reset(dimy, dimx);
  check(sks_make_synthetic(static_cast<int>(kind), dimy, dimx, seed, d.values.data().data()));
  return d;
}

inline SectorPlan plan_sector(int k, int ns, int dimy, int dimx) {
  SectorPlan p{};
  check(sks_plan_sector(k, ns, dimy, dimx, &p));
  return p;
}

inline ShearParams shear_params(double shear_tan, int j) {
  ShearParams sp{};
  sks_shear_params(shear_tan, j, &sp.dest, &sp.frac);
  return sp;
}

inline double area_scale_factor(const RunConfig& cfg, double cellsize) {
  return sks_area_scale_factor(cfg.ns, cellsize, static_cast<int>(cfg.units));
}

inline double area_scale(double cv_sum, int ns, double cellsize) {
  return cv_sum * (std::numbers::pi / ns) * cellsize * cellsize;
}

inline void validate_or_throw(const Dem& dem, const RunConfig& cfg) {
  sks_run_config c = cfg.to_c();
  const float* nod = dem.nodata ? &*dem.nodata : nullptr;
  check(sks_validate(dem.values.data().data(), dem.dimy(), dem.dimx(), dem.cellsize, nod, &c));
}

namespace detail {
// ProgressFn (engine.hpp:34-36): once per sector, ascending k, on the calling
// thread; sectors run batched on the GPU, so each gets the device time of the
// phases attributed by its exact scan work.
inline void report_progress(const Dem& dem, const RunConfig& cfg, const EngineStats& st, const ProgressFn& progress) {
  const double busy = st.skew_seconds + st.scan_seconds + st.fixup_seconds + st.unskew_seconds;
  std::vector<double> work(cfg.ns / 2);
  double total = 0.0;
  for (int k = 0; k < cfg.ns / 2; ++k) {
    work[k] = static_cast<double>(sks_sector_target_evals(k, cfg.ns, dem.dimy(), dem.dimx(), dem.cellsize,
                                                          cfg.max_distance.value_or(0.0)));
    total += work[k];
  }
  for (int k = 0; k < cfg.ns / 2; ++k) progress(k, total > 0.0 ? busy * work[k] / total : 0.0);
}
}  // namespace detail

inline Grid<double> total_viewshed_raw(const Dem& dem, const RunConfig& cfg,
                                       EngineStats* stats = nullptr,
                                       const ProgressFn& progress = {}) {
  if (dem.nodata) validate_or_throw(dem, cfg);
  Grid<double> out(dem.dimy(), dem.dimx());
  sks_run_config c = cfg.to_c();
  EngineStats local;
  EngineStats* st = stats ? stats : (progress ? &local : nullptr);
  check(sks_total_viewshed_raw(dem.values.data().data(), dem.dimy(), dem.dimx(), dem.cellsize, &c,
                               out.data().data(), st));
  if (progress) detail::report_progress(dem, cfg, *st, progress);
  return out;
}

inline VsGrid total_viewshed(const Dem& dem, const RunConfig& cfg, EngineStats* stats = nullptr,
                             const ProgressFn& progress = {}) {
  if (dem.nodata) validate_or_throw(dem, cfg);
  VsGrid out;
  out.units = cfg.units;
  out.values.reset(dem.dimy(), dem.dimx());
  sks_run_config c = cfg.to_c();
  EngineStats local;
  EngineStats* st = stats ? stats : (progress ? &local : nullptr);
  check(sks_total_viewshed(dem.values.data().data(), dem.dimy(), dem.dimx(), dem.cellsize, &c,
                           out.values.data().data(), st));
  if (progress) detail::report_progress(dem, cfg, *st, progress);
  return out;
}

inline SectorResult sector_sweep(const Dem& dem, const RunConfig& cfg, int k) {
  if (dem.nodata) validate_or_throw(dem, cfg);
  SectorResult r;
  r.sector_index = k;
  r.contribution.reset(dem.dimy(), dem.dimx());
  sks_run_config c = cfg.to_c();
  check(sks_sector_sweep(dem.values.data().data(), dem.dimy(), dem.dimx(), dem.cellsize, &c, k,
                         r.contribution.data().data()));
  return r;
}

inline void accumulate_into(Grid<double>& accum, const Grid<double>& contribution) {
  if (!accum.same_shape(contribution)) {
    throw std::invalid_argument("cannot accumulate grids of different shape");
  }
  for (std::size_t n = 0; n < accum.size(); ++n) accum.data()[n] += contribution.data()[n];
}

inline Grid<double> reduce_ordered(std::span<const Grid<double>> buffers) {
  if (buffers.empty()) throw std::invalid_argument("nothing to reduce");
  Grid<double> acc(buffers.front().rows(), buffers.front().cols(), 0.0);
  for (const auto& b : buffers) accumulate_into(acc, b);
  return acc;
}

inline SkwGrid build_skw(const Grid<float>& g, double shear_tan, int device = 0) {
  int skw_rows = 0;
  check(sks_row_ranges(g.rows(), g.cols(), shear_tan, nullptr, &skw_rows));
  SkwGrid s;
  s.src_rows = g.rows();
  s.cols = g.cols();
  s.shear_tan = shear_tan;
  s.values.reset(skw_rows, g.cols());
  std::vector<int> rr(2 * static_cast<std::size_t>(skw_rows));
  check(sks_build_skw(g.data().data(), g.rows(), g.cols(), shear_tan, device, s.values.data().data(),
                      rr.data(), &s.base));
  s.row_ranges.resize(skw_rows);
  for (int q = 0; q < skw_rows; ++q) s.row_ranges[q] = {rr[2 * q], rr[2 * q + 1]};
  return s;
}

inline Grid<double> sector_viewshed(const SkwGrid& skw, double h0, int max_dd = kNoDistanceCap,
                                    int device = 0) {
  std::vector<int> rr(2 * skw.row_ranges.size());
  for (std::size_t q = 0; q < skw.row_ranges.size(); ++q) {
    rr[2 * q] = skw.row_ranges[q].first;
    rr[2 * q + 1] = skw.row_ranges[q].second;
  }
  Grid<double> out(skw.skw_rows(), skw.cols);
  check(sks_sector_viewshed(skw.values.data().data(), rr.data(), skw.skw_rows(), skw.cols,
                            skw.shear_tan, h0, max_dd, device, out.data().data(), nullptr, nullptr));
  return out;
}

inline double linear_viewshed_row(std::span<const float> row, int first, int last, int j0, double h,
                                  ScanDir dir, int max_dd = kNoDistanceCap,
                                  std::vector<std::uint8_t>* visible_out = nullptr, int device = 0) {
  double cv = 0.0;
  int nv = 0;
  std::vector<std::uint8_t> vis(row.size() + 1);
  check(sks_linear_viewshed_row(row.data(), static_cast<int>(row.size()), first, last, j0, h,
                                static_cast<int>(dir), max_dd, device, &cv,
                                visible_out ? vis.data() : nullptr, &nv));
  if (visible_out) visible_out->insert(visible_out->end(), vis.begin(), vis.begin() + nv);
  return cv;
}

inline void unskew_accumulate(const Grid<double>& skw_vs, const SectorPlan& plan, Grid<double>& out,
                              int device = 0) {
  if (out.rows() != plan.src_rows || out.cols() != plan.src_cols) {
    throw std::invalid_argument("output shape does not match source grid");
  }
  check(sks_unskew_accumulate(skw_vs.data().data(), skw_vs.rows(), skw_vs.cols(), plan.sector_index,
                              plan.ns, plan.src_rows, plan.src_cols, device, out.data().data()));
}

// ---- ESRI ASCII grid I/O (ascii_grid.hpp:20-31) ----

namespace detail {
inline Dem take_ascii_grid(sks_ascii_grid* g) {
  sks_grid_header h{};
  sks_status s = sks_ascii_grid_header(g, &h);
  Dem dem;
  if (s == SKS_OK) {
    dem.values.reset(h.nrows, h.ncols);
    s = sks_ascii_grid_values(g, dem.values.data().data());
  }
  sks_ascii_grid_free(g);
  check(s);
  dem.cellsize = h.cellsize;
  dem.origin.easting = h.xllcorner;
  dem.origin.northing = h.yllcorner;
  if (h.has_nodata) dem.nodata = h.nodata;
  return dem;
}
}  // namespace detail

inline Dem read_ascii_grid(const std::filesystem::path& path) {
  sks_ascii_grid* g = nullptr;
  check(sks_ascii_grid_read(path.string().c_str(), &g));
  return detail::take_ascii_grid(g);
}

inline Dem read_ascii_grid(std::istream& in, std::string_view source_name) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  const std::string src(source_name);
  sks_ascii_grid* g = nullptr;
  check(sks_ascii_grid_parse(text.data(), text.size(), src.c_str(), &g));
  return detail::take_ascii_grid(g);
}

// dem.hpp:71 / dem.cpp:175-213 (the CLI's `fill`)
inline Dem fill_nodata_nearest(const Dem& dem) {
  Dem out = dem;
  if (!dem.nodata) return out;
  check(sks_fill_nodata_nearest(dem.values.data().data(), dem.dimy(), dem.dimx(), *dem.nodata,
                                out.values.data().data()));
  out.nodata.reset();
  return out;
}

// Binary side format (ESRI .hdr + .flt float32), the fast load of large DEMs.
inline Dem read_float_grid(const std::filesystem::path& path) {
  sks_ascii_grid* g = nullptr;
  check(sks_float_grid_read(path.string().c_str(), &g));
  return detail::take_ascii_grid(g);
}

inline void write_float_grid(const Dem& dem, const std::filesystem::path& path) {
  const sks_grid_header h{dem.dimy(), dem.dimx(), dem.origin.easting, dem.origin.northing,
                          dem.cellsize, dem.nodata ? 1 : 0, dem.nodata.value_or(0.0f)};
  check(sks_write_float_grid(path.string().c_str(), dem.values.data().data(), &h));
}

inline void write_ascii_grid(const Dem& dem, const std::filesystem::path& path) {
  const sks_grid_header h{dem.dimy(), dem.dimx(), dem.origin.easting, dem.origin.northing,
                          dem.cellsize, dem.nodata ? 1 : 0, dem.nodata.value_or(0.0f)};
  check(sks_write_ascii_grid_dem(path.string().c_str(), dem.values.data().data(), &h));
}

inline void write_ascii_grid(const VsGrid& grid, Units out_units, double cellsize,
                             const GridOrigin& origin, const std::filesystem::path& path) {
  check(sks_write_ascii_grid_vs(path.string().c_str(), grid.values.data().data(), grid.values.rows(),
                                grid.values.cols(), static_cast<int>(grid.units),
                                static_cast<int>(out_units), cellsize, origin.easting,
                                origin.northing));
}

// ---- bench report (bench.hpp:14-40) ----
// scan_seconds is the GPU scan phase (scan + exact fixup kernels); workers is
// the number of GPUs.
struct BenchReport {
  std::string dataset;
  int dimy = 0, dimx = 0, ns = 0, workers = 0;
  double skew_seconds = 0.0, scan_seconds = 0.0, unskew_seconds = 0.0, reduce_seconds = 0.0;
  double total_seconds = 0.0, povs_per_second = 0.0, speedup = 0.0;
};

inline BenchReport make_bench_report(const std::string& dataset, int dimy, int dimx, const RunConfig& cfg,
                                     const EngineStats& stats, double baseline_total_seconds = 0.0,
                                     int workers = 1) {
  BenchReport r;
  r.dataset = dataset;
  r.dimy = dimy;
  r.dimx = dimx;
  r.ns = cfg.ns;
  r.workers = workers;
  r.skew_seconds = stats.skew_seconds;
  r.scan_seconds = stats.scan_seconds + stats.fixup_seconds;
  r.unskew_seconds = stats.unskew_seconds;
  r.reduce_seconds = stats.reduce_seconds;
  r.total_seconds = stats.total_seconds;
  r.povs_per_second = static_cast<double>(dimy) * static_cast<double>(dimx) * static_cast<double>(cfg.ns / 2) /
                      r.scan_seconds;
  if (baseline_total_seconds > 0.0) r.speedup = baseline_total_seconds / r.total_seconds;
  return r;
}

inline std::string format_bench_report(const BenchReport& r) {
  auto num = [](double v) {
    char b[64];
    std::snprintf(b, sizeof(b), "%.17g", v);
    return std::string(b);
  };
  std::string s = "dataset: " + r.dataset + "\n" + "dimy: " + std::to_string(r.dimy) + "\n" +
                  "dimx: " + std::to_string(r.dimx) + "\n" + "ns: " + std::to_string(r.ns) + "\n" +
                  "workers: " + std::to_string(r.workers) + "\n" + "skew_seconds: " + num(r.skew_seconds) + "\n" +
                  "scan_seconds: " + num(r.scan_seconds) + "\n" + "unskew_seconds: " + num(r.unskew_seconds) +
                  "\n" + "reduce_seconds: " + num(r.reduce_seconds) + "\n" + "total_seconds: " +
                  num(r.total_seconds) + "\n" + "povs_per_second: " + num(r.povs_per_second) + "\n";
  if (r.speedup > 0.0) s += "speedup: " + num(r.speedup) + "\n";
  return s;
}

// ---- heatmaps (heatmap.hpp) ----
enum class Palette { Gray = SKS_PALETTE_GRAY, BlueRed = SKS_PALETTE_BLUE_RED };

inline void write_heatmap(const VsGrid& grid, const std::filesystem::path& path, Palette palette) {
  check(sks_write_heatmap(path.string().c_str(), grid.values.data().data(), grid.values.rows(), grid.values.cols(),
                          static_cast<int>(palette)));
}

// ---- the rotational-sweep oracle on the GPU (oracle.hpp) ----
namespace oracle {

struct GridPoint {
  int i = 0;
  int j = 0;
};

struct RingSector {
  double r_open = 0.0;
  double r_close = 0.0;
};

using RingSectorSet = std::vector<RingSector>;

inline constexpr int kReferenceCellGuard = SKS_REFERENCE_CELL_GUARD;

inline std::vector<GridPoint> select_axis_point_set(const Dem& dem, int i0, int j0, double azimuth_deg) {
  int n = 0;
  check(sks_axis_point_set(dem.dimy(), dem.dimx(), i0, j0, azimuth_deg, nullptr, 0, &n));
  std::vector<int> ij(2 * static_cast<size_t>(std::max(n, 1)));
  check(sks_axis_point_set(dem.dimy(), dem.dimx(), i0, j0, azimuth_deg, ij.data(), n, &n));
  std::vector<GridPoint> pts(static_cast<size_t>(n));
  for (int t = 0; t < n; ++t) pts[t] = {ij[2 * t], ij[2 * t + 1]};
  return pts;
}

inline double linear_scan(const Dem& dem, int i0, int j0, double pov_h, double azimuth_deg,
                          double max_dist_cells = std::numeric_limits<double>::infinity(),
                          RingSectorSet* rings_out = nullptr, int device = 0) {
  double cv = 0.0;
  int n = 0;
  check(sks_linear_scan(dem.values.data().data(), dem.dimy(), dem.dimx(), i0, j0, pov_h, azimuth_deg,
                        max_dist_cells, device, &cv, nullptr, 0, &n));
  if (rings_out && n > 0) {
    std::vector<double> r(2 * static_cast<size_t>(n));
    check(sks_linear_scan(dem.values.data().data(), dem.dimy(), dem.dimx(), i0, j0, pov_h, azimuth_deg,
                          max_dist_cells, device, &cv, r.data(), n, &n));
    for (int t = 0; t < n; ++t) rings_out->push_back({r[2 * t], r[2 * t + 1]});
  }
  return cv;
}

inline double singular_viewshed(const Dem& dem, int i0, int j0, double h0, int ns,
                                std::optional<double> max_distance = {}, int device = 0) {
  double area = 0.0;
  check(sks_singular_viewshed(dem.values.data().data(), dem.dimy(), dem.dimx(), dem.cellsize, i0, j0, h0, ns,
                              max_distance.value_or(0.0), device, &area));
  return area;
}

struct MultiViewshed {
  VsGrid grid;  // nonzero only at the observer cells, m^2
  double total_area = 0.0;
};

inline MultiViewshed multi_viewshed(const Dem& dem, std::span<const GridPoint> povs, double h0, int ns,
                                    std::optional<double> max_distance = {}, int device = 0) {
  std::vector<int> ij(2 * povs.size());
  for (size_t t = 0; t < povs.size(); ++t) {
    ij[2 * t] = povs[t].i;
    ij[2 * t + 1] = povs[t].j;
  }
  MultiViewshed out;
  out.grid.units = Units::SquareMeters;
  out.grid.values.reset(dem.dimy(), dem.dimx(), 0.0);
  check(sks_multi_viewshed(dem.values.data().data(), dem.dimy(), dem.dimx(), dem.cellsize, ij.data(),
                           static_cast<int>(povs.size()), h0, ns, max_distance.value_or(0.0), device, nullptr,
                           out.grid.values.data().data(), &out.total_area));
  return out;
}

inline VsGrid total_viewshed_reference(const Dem& dem, const RunConfig& cfg, bool force = false) {
  VsGrid out;
  out.units = cfg.units;
  out.values.reset(dem.dimy(), dem.dimx());
  const sks_run_config c = cfg.to_c();
  const float nod = dem.nodata.value_or(0.0f);
  check(sks_total_viewshed_reference(dem.values.data().data(), dem.dimy(), dem.dimx(), dem.cellsize,
                                     dem.nodata ? &nod : nullptr, &c, force ? 1 : 0, out.values.data().data()));
  return out;
}

}  // namespace oracle

}  // namespace skewshed_b200
