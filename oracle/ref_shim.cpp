// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (skewshed, built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets the
// Python tests, golden-fixture generator and bench.py's CPU baseline call the
// reference's own public API through ctypes with plain pointers. Every entry
// point forwards to one reference function; the citation names it.
//
// Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
// legs may load this library.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <optional>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include <sstream>

#include "skewshed/ascii_grid.hpp"
#include "skewshed/dem.hpp"
#include "skewshed/engine.hpp"
#include "skewshed/heatmap.hpp"
#include "skewshed/oracle.hpp"
#include "skewshed/scan.hpp"
#include "skewshed/skew.hpp"

using namespace skewshed;

namespace {

thread_local std::string g_err;

Dem make_dem(const float* v, int dimy, int dimx, double cellsize) {
  Dem dem;
  dem.cellsize = cellsize;
  dem.values.reset(dimy, dimx, 0.0f);
  std::memcpy(dem.values.data().data(), v,
              sizeof(float) * static_cast<size_t>(dimy) * dimx);
  return dem;
}

RunConfig make_cfg(int ns, double h0, int workers, double max_distance,
                   int units) {
  RunConfig cfg;
  cfg.ns = ns;
  cfg.h0 = h0;
  cfg.workers = workers;
  if (max_distance > 0.0) cfg.max_distance = max_distance;
  cfg.units = units == 1 ? Units::SquareKilometers : Units::SquareMeters;
  return cfg;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// dem.cpp:118-173 make_synthetic
int ref_make_synthetic(int kind, int dimy, int dimx, double cellsize,
                       uint32_t seed, float* out) {
  return guarded([&] {
    Dem d = make_synthetic(static_cast<SyntheticKind>(kind), dimy, dimx,
                           cellsize, seed);
    std::memcpy(out, d.values.data().data(),
                sizeof(float) * static_cast<size_t>(dimy) * dimx);
  });
}

// skew.cpp:23-95 plan_sector. ops_out: up to 3 AxisOp codes
// (0 Transpose, 1 FlipCols, 2 FlipRows); map_out: ii,ij,ci,ji,jj,cj.
int ref_plan_sector(int k, int ns, int dimy, int dimx, double* degs_out,
                    int* shape_out, int* map_out, int* ops_out,
                    int* n_ops_out) {
  return guarded([&] {
    SectorPlan p = plan_sector(k, ns, dimy, dimx);
    degs_out[0] = p.sector_deg;
    degs_out[1] = p.shear_deg;
    degs_out[2] = p.shear_tan;
    shape_out[0] = p.rows;
    shape_out[1] = p.cols;
    const IndexMap& m = p.to_source;
    int mm[6] = {m.ii, m.ij, m.ci, m.ji, m.jj, m.cj};
    std::memcpy(map_out, mm, sizeof(mm));
    *n_ops_out = static_cast<int>(p.pre_ops.size());
    for (size_t i = 0; i < p.pre_ops.size(); ++i) {
      ops_out[i] = static_cast<int>(p.pre_ops[i]);
    }
  });
}

// skew.cpp:97-101 shear_params
void ref_shear_params(double shear_tan, int j, int* dest, double* frac) {
  ShearParams sp = shear_params(shear_tan, j);
  *dest = sp.dest;
  *frac = sp.frac;
}

// skew.cpp:103-136 apply_pre_ops for sector k's plan
int ref_apply_pre_ops(const float* dem, int dimy, int dimx, int k, int ns,
                      float* out) {
  return guarded([&] {
    SectorPlan p = plan_sector(k, ns, dimy, dimx);
    Dem d = make_dem(dem, dimy, dimx, 1.0);
    Grid<float> pre = apply_pre_ops(d.values, p.pre_ops);
    std::memcpy(out, pre.data().data(), sizeof(float) * pre.size());
  });
}

// skew.cpp:144-196 build_skw. values/weights capacity cap_rows*cols.
// Returns skw_rows through *skw_rows_out and base through *base_out.
int ref_build_skw(const float* g, int rows, int cols, double shear_tan,
                  int cap_rows, float* values, float* weights, int* ranges,
                  int* skw_rows_out, int* base_out) {
  return guarded([&] {
    Dem d = make_dem(g, rows, cols, 1.0);
    SkwGrid skw = build_skw(d.values, shear_tan);
    *skw_rows_out = skw.skw_rows();
    *base_out = skw.base;
    if (skw.skw_rows() > cap_rows) {
      throw std::runtime_error("ref_build_skw: capacity too small");
    }
    std::memcpy(values, skw.values.data().data(),
                sizeof(float) * skw.values.size());
    if (weights) {
      std::memcpy(weights, skw.weights.data().data(),
                  sizeof(float) * skw.weights.size());
    }
    for (int q = 0; q < skw.skw_rows(); ++q) {
      ranges[2 * q] = skw.row_ranges[q].first;
      ranges[2 * q + 1] = skw.row_ranges[q].second;
    }
  });
}

// scan.cpp:8-62 linear_viewshed_row; dir 0 forward, 1 backward.
// visible_out (optional) receives one flag per scanned target; *n_vis its
// count.
double ref_linear_viewshed_row(const float* row, int n, int first, int last,
                               int j0, double h, int dir, int max_dd,
                               uint8_t* visible_out, int* n_vis) {
  std::vector<uint8_t> vis;
  double cv = linear_viewshed_row(
      std::span<const float>(row, n), first, last, j0, h,
      dir == 0 ? ScanDir::Forward : ScanDir::Backward, max_dd,
      visible_out ? &vis : nullptr);
  if (visible_out) {
    std::memcpy(visible_out, vis.data(), vis.size());
    *n_vis = static_cast<int>(vis.size());
  }
  return cv;
}

// scan.cpp:64-85 sector_viewshed over an sDEM given as values + row ranges.
int ref_sector_viewshed(const float* values, const int* ranges, int skw_rows,
                        int cols, int src_rows, int base, double shear_tan,
                        double h0, int max_dd, double* out) {
  return guarded([&] {
    SkwGrid skw;
    skw.src_rows = src_rows;
    skw.cols = cols;
    skw.base = base;
    skw.shear_tan = shear_tan;
    skw.values.reset(skw_rows, cols, 0.0f);
    std::memcpy(skw.values.data().data(), values,
                sizeof(float) * static_cast<size_t>(skw_rows) * cols);
    skw.weights.reset(skw_rows, cols, 0.0f);
    skw.row_ranges.resize(skw_rows);
    for (int q = 0; q < skw_rows; ++q) {
      skw.row_ranges[q] = {ranges[2 * q], ranges[2 * q + 1]};
    }
    Grid<double> vs;
    sector_viewshed(skw, h0, max_dd, vs);
    std::memcpy(out, vs.data().data(), sizeof(double) * vs.size());
  });
}

// skew.cpp:204-263 unskew_accumulate (out is read-modify-written).
int ref_unskew_accumulate(const double* skw_vs, int skw_rows, int cols, int k,
                          int ns, int dimy, int dimx, double* out) {
  return guarded([&] {
    SectorPlan plan = plan_sector(k, ns, dimy, dimx);
    Grid<double> vs(skw_rows, cols, 0.0);
    std::memcpy(vs.data().data(), skw_vs, sizeof(double) * vs.size());
    Grid<double> o(dimy, dimx, 0.0);
    std::memcpy(o.data().data(), out, sizeof(double) * o.size());
    unskew_accumulate(vs, plan, o);
    std::memcpy(out, o.data().data(), sizeof(double) * o.size());
  });
}

// engine.cpp:235-244 sector_sweep
int ref_sector_sweep(const float* dem, int dimy, int dimx, double cellsize,
                     int ns, double h0, double max_distance, int k,
                     double* out, double* phase_seconds) {
  return guarded([&] {
    Dem d = make_dem(dem, dimy, dimx, cellsize);
    RunConfig cfg = make_cfg(ns, h0, 1, max_distance, 0);
    SectorResult r = sector_sweep(d, cfg, k);
    std::memcpy(out, r.contribution.data().data(),
                sizeof(double) * r.contribution.size());
    if (phase_seconds) {
      phase_seconds[0] = r.skew_seconds;
      phase_seconds[1] = r.scan_seconds;
      phase_seconds[2] = r.unskew_seconds;
      phase_seconds[3] = r.wall_seconds;
    }
  });
}

// engine.cpp:109-220 total_viewshed_raw (raw=1) or engine.cpp:222-233
// total_viewshed (raw=0). stats_out: skew, scan, unskew, reduce, total secs.
int ref_total_viewshed(const float* dem, int dimy, int dimx, double cellsize,
                       int ns, double h0, int workers, double max_distance,
                       int units, int raw, double* out, double* stats_out) {
  return guarded([&] {
    Dem d = make_dem(dem, dimy, dimx, cellsize);
    RunConfig cfg = make_cfg(ns, h0, workers, max_distance, units);
    EngineStats st;
    if (raw) {
      Grid<double> g = total_viewshed_raw(d, cfg, &st);
      std::memcpy(out, g.data().data(), sizeof(double) * g.size());
    } else {
      VsGrid g = total_viewshed(d, cfg, &st);
      std::memcpy(out, g.values.data().data(),
                  sizeof(double) * g.values.size());
    }
    if (stats_out) {
      stats_out[0] = st.skew_seconds;
      stats_out[1] = st.scan_seconds;
      stats_out[2] = st.unskew_seconds;
      stats_out[3] = st.reduce_seconds;
      stats_out[4] = st.total_seconds;
    }
  });
}

// engine.cpp:103-107 area_scale_factor
double ref_area_scale_factor(int ns, double cellsize, int units) {
  RunConfig cfg = make_cfg(ns, 1.5, 1, 0.0, units);
  return area_scale_factor(cfg, cellsize);
}

// oracle.cpp:143-194 total_viewshed_reference (rotational sweep, secondary
// sanity oracle).
int ref_rotational_total_viewshed(const float* dem, int dimy, int dimx,
                                  double cellsize, int ns, double h0,
                                  double max_distance, double* out) {
  return guarded([&] {
    Dem d = make_dem(dem, dimy, dimx, cellsize);
    RunConfig cfg = make_cfg(ns, h0, 1, max_distance, 0);
    cfg.workers = std::max(1u, std::thread::hardware_concurrency());
    VsGrid g = oracle::total_viewshed_reference(d, cfg, true);
    std::memcpy(out, g.values.data().data(), sizeof(double) * g.values.size());
  });
}

// Benchmark input: the fractal terrain of BASELINE config 1-5 (DESIGN.md
// "Inputs"). The reference has no fractal generator (its kinds are Flat, Ramp,
// Cone, SmoothedNoise, dem.hpp:60-67), so this is the bench's own definition,
// restated here so that the reference arm never loads the product library:
// diamond-square midpoint displacement on the smallest (2^m+1)^2 lattice
// covering the grid, cropped top-left; raw std::mt19937(seed) words mapped to
// [-1, 1) as 2*(x/2^32)-1 (as dem.cpp:94-96 maps its draws); corners first at
// amplitude 300 m, then per level l the diamond step and the square step in
// row-major order at amplitude 300*2^(-0.8(l+1)); 500 m + lattice as float32.
// tests/test_oracle.py pins it to the product's generator bit for bit.
int ref_make_fractal(int dimy, int dimx, uint32_t seed, float* out) {
  return guarded([&] {
    if (dimy < 2 || dimx < 2) throw std::invalid_argument("synthetic grid dimensions must be >= 2");
    int m = 0;
    while ((1 << m) + 1 < std::max(dimy, dimx)) ++m;
    const int S = (1 << m) + 1;
    std::vector<double> lat(static_cast<size_t>(S) * S, 0.0);
    std::mt19937 gen(seed);
    auto unit = [&] { return 2.0 * (static_cast<double>(gen()) / 4294967296.0) - 1.0; };
    auto h = [&](int i, int j) -> double& { return lat[static_cast<size_t>(i) * S + j]; };
    for (auto [ci, cj] : {std::pair{0, 0}, std::pair{0, S - 1}, std::pair{S - 1, 0}, std::pair{S - 1, S - 1}}) {
      h(ci, cj) = 300.0 * unit();
    }
    for (int l = 0; l < m; ++l) {
      const int step = 1 << (m - l), half = step / 2;
      const double amp = 300.0 * std::pow(2.0, -0.8 * (l + 1));
      for (int i = half; i < S; i += step) {  // diamond: centre of each square
        for (int j = half; j < S; j += step) {
          const double corners = h(i - half, j - half) + h(i - half, j + half) + h(i + half, j - half) +
                                 h(i + half, j + half);
          h(i, j) = corners / 4.0 + amp * unit();
        }
      }
      for (int i = 0; i < S; i += half) {  // square: edge midpoints, row-major
        for (int j = ((i / half) % 2 == 0) ? half : 0; j < S; j += step) {
          double sum = 0.0;
          int n = 0;
          if (i >= half) sum += h(i - half, j), ++n;
          if (i + half < S) sum += h(i + half, j), ++n;
          if (j >= half) sum += h(i, j - half), ++n;
          if (j + half < S) sum += h(i, j + half), ++n;
          h(i, j) = sum / n + amp * unit();
        }
      }
    }
    for (int i = 0; i < dimy; ++i) {
      for (int j = 0; j < dimx; ++j) out[static_cast<size_t>(i) * dimx + j] = static_cast<float>(500.0 + h(i, j));
    }
  });
}

// CPU baseline sample: the reference's public per-sector entry point
// sector_sweep (engine.cpp:235-244: plan_sector -> apply_pre_ops ->
// build_skw -> sector_viewshed -> unskew_accumulate, the same
// compute_sector the engine's workers run, engine.cpp:45-66) on the listed
// sectors, claimed dynamically by `threads` host threads as the engine's
// workers claim them (engine.cpp:150-160). Returns the wall seconds.
int ref_sweep_sample(const float* dem, int dimy, int dimx, double cellsize, int ns, double h0,
                     double max_distance, const int* sectors, int n_sectors, int threads,
                     double* seconds_out) {
  return guarded([&] {
    const Dem d = make_dem(dem, dimy, dimx, cellsize);
    const RunConfig cfg = make_cfg(ns, h0, 1, max_distance, 0);
    std::atomic<int> next{0};
    std::atomic<long long> sink{0};
    std::exception_ptr failure;
    std::mutex mu;
    auto worker = [&] {
      try {
        for (;;) {
          const int i = next.fetch_add(1);
          if (i >= n_sectors) break;
          SectorResult r = sector_sweep(d, cfg, sectors[i]);
          sink += static_cast<long long>(r.contribution.data()[0]) & 1;
        }
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!failure) failure = std::current_exception();
      }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, std::min(threads, n_sectors)); ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    *seconds_out = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (failure) std::rethrow_exception(failure);
  });
}

// Exact scan work of sector k (target evaluations: for every full cell of
// every skewed row, the forward and backward scan lengths, capped by
// distance_cap_cells, engine.cpp:29-36 / scan.cpp:20-22,37-39), from the
// reference's own plan_sector and build_skw row ranges (which depend on the
// geometry only, so a zero grid of the right shape gives them).
long long ref_sector_work(int dimy, int dimx, double cellsize, int ns, int k, double max_distance) {
  long long total = -1;
  guarded([&] {
    const SectorPlan p = plan_sector(k, ns, dimy, dimx);
    int max_dd = kNoDistanceCap;
    if (max_distance > 0.0) {
      const double step = cellsize * std::sqrt(1.0 + p.shear_tan * p.shear_tan);
      const double cap = std::floor(max_distance / step);
      max_dd = cap >= static_cast<double>(kNoDistanceCap) ? kNoDistanceCap : std::max(0, static_cast<int>(cap));
    }
    Grid<float> zero;
    zero.reset(p.rows, p.cols, 0.0f);
    const SkwGrid skw = build_skw(zero, p.shear_tan);
    long long w = 0;
    for (auto [first, last] : skw.row_ranges) {
      for (int j0 = first; j0 < last; ++j0) {
        w += std::min<long long>(last - 1 - j0, max_dd) + std::min<long long>(j0 - first, max_dd);
      }
    }
    total = w;
  });
  return total;
}

// read_ascii_grid(istream, source_name) (ascii_grid.cpp:110-196). Returns 0,
// 3 for GridFormatError (message in ref_last_error) or 4 for another error.
int ref_parse_ascii_grid(const char* text, size_t len, const char* source, int* nrows, int* ncols,
                         double* hdr /* xll, yll, cellsize */, int* has_nodata, float* nodata,
                         float* values, long long cap) {
  try {
    std::istringstream in(std::string(text, len));
    Dem dem = read_ascii_grid(in, source);
    *nrows = dem.dimy();
    *ncols = dem.dimx();
    hdr[0] = dem.origin.easting;
    hdr[1] = dem.origin.northing;
    hdr[2] = dem.cellsize;
    *has_nodata = dem.nodata.has_value() ? 1 : 0;
    *nodata = dem.nodata.value_or(0.0f);
    const long long n = static_cast<long long>(dem.dimy()) * dem.dimx();
    if (values && n <= cap) std::memcpy(values, dem.values.data().data(), sizeof(float) * n);
    return 0;
  } catch (const GridFormatError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

// write_ascii_grid(Dem, path) (ascii_grid.cpp:225-245)
int ref_write_ascii_grid_dem(const char* path, const float* v, int nrows, int ncols, double xll, double yll,
                             double cellsize, int has_nodata, float nodata) {
  try {
    Dem dem = make_dem(v, nrows, ncols, cellsize);
    dem.origin.easting = xll;
    dem.origin.northing = yll;
    if (has_nodata) dem.nodata = nodata;
    write_ascii_grid(dem, path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

// write_ascii_grid(VsGrid, out_units, cellsize, origin, path) (ascii_grid.cpp:247-272)
int ref_write_ascii_grid_vs(const char* path, const double* v, int nrows, int ncols, int units_in, int units_out,
                            double cellsize, double xll, double yll) {
  try {
    VsGrid vs;
    vs.units = units_in ? Units::SquareKilometers : Units::SquareMeters;
    vs.values.reset(nrows, ncols, 0.0);
    std::memcpy(vs.values.data().data(), v, sizeof(double) * static_cast<size_t>(nrows) * ncols);
    GridOrigin o;
    o.easting = xll;
    o.northing = yll;
    write_ascii_grid(vs, units_out ? Units::SquareKilometers : Units::SquareMeters, cellsize, o, path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

// oracle.cpp:108-129 singular_viewshed (max_distance 0 = unset)
int ref_singular_viewshed(const float* dem, int dimy, int dimx, double cellsize, int i, int j, double h0,
                          int ns, double max_distance, double* area) {
  return guarded([&] {
    Dem d = make_dem(dem, dimy, dimx, cellsize);
    std::optional<double> md;
    if (max_distance != 0.0) md = max_distance;
    *area = oracle::singular_viewshed(d, i, j, h0, ns, md);
  });
}

// oracle.cpp:131-141 multi_viewshed: grid (dimy*dimx) and total
int ref_multi_viewshed(const float* dem, int dimy, int dimx, double cellsize, const int* povs, int npovs,
                       double h0, int ns, double max_distance, double* grid, double* total) {
  return guarded([&] {
    Dem d = make_dem(dem, dimy, dimx, cellsize);
    std::vector<oracle::GridPoint> p(static_cast<size_t>(npovs));
    for (int t = 0; t < npovs; ++t) p[t] = {povs[2 * t], povs[2 * t + 1]};
    std::optional<double> md;
    if (max_distance != 0.0) md = max_distance;
    oracle::MultiViewshed mv = oracle::multi_viewshed(d, p, h0, ns, md);
    std::memcpy(grid, mv.grid.values.data().data(), sizeof(double) * mv.grid.values.size());
    *total = mv.total_area;
  });
}

// oracle.cpp:143-194 total_viewshed_reference with the caller's units/force/
// nodata (error paths included)
int ref_total_viewshed_reference(const float* dem, int dimy, int dimx, double cellsize, const float* nodata,
                                 int ns, double h0, double max_distance, int units, int force, double* out) {
  return guarded([&] {
    Dem d = make_dem(dem, dimy, dimx, cellsize);
    if (nodata) d.nodata = *nodata;
    RunConfig cfg = make_cfg(ns, h0, 1, 0.0, units);
    if (max_distance != 0.0) cfg.max_distance = max_distance;
    cfg.workers = std::max(1u, std::thread::hardware_concurrency());
    VsGrid g = oracle::total_viewshed_reference(d, cfg, force != 0);
    std::memcpy(out, g.values.data().data(), sizeof(double) * g.values.size());
  });
}

// oracle.cpp:74-106 linear_scan with the ring sectors
int ref_linear_scan(const float* dem, int dimy, int dimx, int i0, int j0, double pov_h, double az, double max_cells,
                    double* cv, double* rings, int cap, int* nrings) {
  return guarded([&] {
    Dem d = make_dem(dem, dimy, dimx, 1.0);
    oracle::RingSectorSet rs;
    *cv = oracle::linear_scan(d, i0, j0, pov_h, az, max_cells, &rs);
    *nrings = static_cast<int>(rs.size());
    for (int t = 0; t < std::min(cap, *nrings); ++t) {
      rings[2 * t] = rs[t].r_open;
      rings[2 * t + 1] = rs[t].r_close;
    }
  });
}

// dem.cpp:175-213 fill_nodata_nearest
int ref_fill_nodata_nearest(const float* v, int dimy, int dimx, float nodata, float* out) {
  return guarded([&] {
    Dem d = make_dem(v, dimy, dimx, 1.0);
    d.nodata = nodata;
    Dem f = fill_nodata_nearest(d);
    std::memcpy(out, f.values.data().data(), sizeof(float) * f.values.size());
  });
}

// oracle.cpp:62-71 select_axis_point_set
int ref_axis_point_set(int dimy, int dimx, int i0, int j0, double azimuth_deg, int* ij, int cap, int* count) {
  return guarded([&] {
    Dem d;
    d.values.reset(dimy, dimx, 0.0f);
    auto pts = oracle::select_axis_point_set(d, i0, j0, azimuth_deg);
    *count = static_cast<int>(pts.size());
    for (int t = 0; t < std::min(cap, *count); ++t) {
      ij[2 * t] = pts[t].i;
      ij[2 * t + 1] = pts[t].j;
    }
  });
}

// heatmap.cpp:11-56 write_heatmap
int ref_write_heatmap(const char* path, const double* v, int rows, int cols, int palette) {
  return guarded([&] {
    VsGrid g;
    g.values.reset(rows, cols, 0.0);
    if (g.values.size()) std::memcpy(g.values.data().data(), v, sizeof(double) * g.values.size());
    write_heatmap(g, path, palette ? Palette::BlueRed : Palette::Gray);
  });
}

}  // extern "C"
