// Host-side sector planning; see sks_plan.hpp. Compiled with
// -ffp-contract=off so that no expression here is contracted into an FMA
// (the reference is built the same way).
#include "sks_plan.hpp"

#include <algorithm>
#include <cmath>
#include <numbers>
#include <numeric>
#include <random>
#include <sstream>
#include <stdexcept>

namespace sks {

int base_offset(int src_rows, int cols, double shear_tan) {
  int dest_max = static_cast<int>(shear_tan * (cols - 1));
  return std::max(src_rows, dest_max + 1);
}

void shear_params(double shear_tan, int j, int* dest, double* frac) {
  double y = shear_tan * j;
  int d = static_cast<int>(y);  // y >= 0: truncation is floor
  *dest = d;
  *frac = y - d;
}

int distance_cap_cells(double max_distance, double shear_tan,
                       double cellsize) {
  if (!(max_distance > 0.0)) return kNoCap;
  double step = cellsize * std::sqrt(1.0 + shear_tan * shear_tan);
  double cap = std::floor(max_distance / step);
  if (cap >= static_cast<double>(kNoCap)) return kNoCap;
  return std::max(0, static_cast<int>(cap));
}

double area_scale_factor(int ns, double cellsize, int units) {
  double factor = (std::numbers::pi / ns) * cellsize * cellsize;
  if (units == 1) factor *= 1e-6;
  return factor;
}

long long row_target_evals(long long L, long long max_dd) {
  if (L < 2) return 0;
  // sum_{x=0}^{L-1} min(L-1-x, c) + min(x, c) = 2 * sum_{x=0}^{L-1} min(x, c)
  long long c = std::min<long long>(max_dd, L - 1);
  long long s = c * (c + 1) / 2 + (L - 1 - c) * c;
  return 2 * s;
}

namespace {

bool full_weight(float w) {
  return w > 1.0f - kFullWeightTol && w < 1.0f + kFullWeightTol;
}

// Disjoint-set "next free row" with path halving.
int find_next(std::vector<int>& nxt, int q) {
  while (nxt[q] != q) {
    nxt[q] = nxt[nxt[q]];
    q = nxt[q];
  }
  return q;
}

void fill_tables(SectorPlanH& p) {
  p.base = base_offset(p.rows, p.cols, p.shear_tan);
  p.skw_rows = p.base + p.rows;
  p.correction = 1.0 + p.shear_tan * p.shear_tan;
  p.dest.resize(p.cols);
  p.fracf.resize(p.cols);
  p.fracd.resize(p.cols);
  for (int j = 0; j < p.cols; ++j) {
    shear_params(p.shear_tan, j, &p.dest[j], &p.fracd[j]);
    p.fracf[j] = static_cast<float>(p.fracd[j]);
  }
  p.ranges = row_ranges(p.rows, p.cols, p.base, p.dest, p.fracf);
  long long work = 0;
  for (const RowRange& r : p.ranges) {
    work += row_target_evals(r.last - r.first, p.max_dd);
  }
  p.target_evals = work;
  // inverse of the signed-permutation part of to_source: (i, j) =
  // M^T (si - ci, sj - cj)
  const int* m = p.map;
  int ii = m[0], ij = m[1], ci = m[2], ji = m[3], jj = m[4], cj = m[5];
  // i = ii*(si-ci) + ji*(sj-cj); j = ij*(si-ci) + jj*(sj-cj)
  p.inv[0] = ii;
  p.inv[1] = ji;
  p.inv[2] = -(ii * ci + ji * cj);
  p.inv[3] = ij;
  p.inv[4] = jj;
  p.inv[5] = -(ij * ci + jj * cj);
}

}  // namespace

void set_row_block(SectorPlanH& p, int part, int nparts, const double* cuts) {
  if (nparts <= 1) {
    p.q_lo = 0;
    p.q_hi = p.skw_rows;
    return;
  }
  // Row cost model: the exact scan work L(L-1) (capped) plus a constant per
  // 64-POV task, whose first 64-target window is always evaluated in full
  // (fitted from per-block times of the 2000^2 bench: ~60k target-equivalents):
  // short rows cost far more per target than the work alone says.
  constexpr long long kTaskCost = 60000;
  auto row_cost = [&](int q) {
    const long long L = p.ranges[q].last - p.ranges[q].first;
    if (L < 2 || p.max_dd <= 0) return 0LL;
    return row_target_evals(L, p.max_dd) + 2 * ((L + 63) / 64) * kTaskCost;
  };
  long long total = 0;
  for (int q = 0; q < p.skw_rows; ++q) total += row_cost(q);
  // block b starts at the first row whose preceding cost reaches b/nparts of
  // the total (exact integer comparison: cum * nparts >= b * total)
  auto start = [&](int b) {
    if (b <= 0) return 0;
    if (b >= nparts) return p.skw_rows;
    long long cum = 0;
    for (int q = 0; q < p.skw_rows; ++q) {
      if (cuts != nullptr ? static_cast<double>(cum) >= cuts[b] * static_cast<double>(total)
                          : cum * nparts >= static_cast<long long>(b) * total) {
        return q;
      }
      cum += row_cost(q);
    }
    return p.skw_rows;
  };
  p.q_lo = start(part);
  p.q_hi = start(part + 1);
}

std::vector<RowRange> row_ranges(int rows, int cols, int base,
                                 const std::vector<int>& dest,
                                 const std::vector<float>& fracf) {
  const int skw_rows = base + rows;
  // Per column j the full-weight rows form at most three pieces: the row
  // that only receives the carry (weight f), the rows receiving both (weight
  // fl(fl(1-f)+f)) and the row that only receives the main share (weight
  // 1-f), in the accumulation order of build_skw (skew.cpp:172-183).
  struct Piece {
    int lo, hi;
  };
  auto pieces = [&](int j, Piece out[3]) {
    int n = 0;
    float f = fracf[j];
    float a = 1.0f - f;
    int A = base - dest[j];  // row receiving (1-f) from source row 0
    // carry-only row A-1 (from source row 0), weight f
    bool fc = full_weight(0.0f + f);
    // rows with both shares: A .. A+rows-2
    bool fb = full_weight((0.0f + a) + f);
    // main-only row A+rows-1 (from source row rows-1), weight 1-f
    bool fm = full_weight(0.0f + a);
    if (rows >= 2) {
      if (fc && fb && fm) {
        out[n++] = {A - 1, A + rows - 1};
        return n;
      }
      if (fc) out[n++] = {A - 1, A - 1};
      if (fb) out[n++] = {A, A + rows - 2};
      if (fm) out[n++] = {A + rows - 1, A + rows - 1};
    } else {
      // rows == 1: row A gets only the main share, row A-1 only the carry.
      if (fc) out[n++] = {A - 1, A - 1};
      if (fm) out[n++] = {A, A};
    }
    return n;
  };
  std::vector<int> first(skw_rows, -1), last(skw_rows, -1);
  std::vector<int> nxt(skw_rows + 1);
  Piece pc[3];
  // first: sweep columns left to right; each row takes the first column that
  // covers it.
  std::iota(nxt.begin(), nxt.end(), 0);
  for (int j = 0; j < cols; ++j) {
    int n = pieces(j, pc);
    for (int t = 0; t < n; ++t) {
      int lo = std::max(pc[t].lo, 0), hi = std::min(pc[t].hi, skw_rows - 1);
      for (int q = lo <= hi ? find_next(nxt, lo) : skw_rows; q <= hi;
           q = find_next(nxt, q)) {
        first[q] = j;
        nxt[q] = q + 1;
      }
    }
  }
  std::iota(nxt.begin(), nxt.end(), 0);
  for (int j = cols - 1; j >= 0; --j) {
    int n = pieces(j, pc);
    for (int t = 0; t < n; ++t) {
      int lo = std::max(pc[t].lo, 0), hi = std::min(pc[t].hi, skw_rows - 1);
      for (int q = lo <= hi ? find_next(nxt, lo) : skw_rows; q <= hi;
           q = find_next(nxt, q)) {
        last[q] = j + 1;
        nxt[q] = q + 1;
      }
    }
  }
  std::vector<RowRange> out(skw_rows, RowRange{0, 0});
  for (int q = 0; q < skw_rows; ++q) {
    if (first[q] >= 0 && first[q] < last[q]) out[q] = {first[q], last[q]};
  }
  return out;
}

SectorPlanH plan_sector(int k, int ns, int dimy, int dimx, double cellsize,
                        double max_distance) {
  if (ns < 2 || ns % 2 != 0) {
    throw std::invalid_argument("sector count must be an even integer >= 2");
  }
  if (k < 0 || k >= ns / 2) {
    std::ostringstream os;
    os << "sector index " << k << " out of range [0, " << ns / 2 << ")";
    throw std::out_of_range(os.str());
  }
  if (dimy < 1 || dimx < 1) {
    throw std::invalid_argument("grid dimensions must be positive");
  }
  SectorPlanH p;
  p.k = k;
  p.ns = ns;
  p.sector_deg = k * (360.0 / ns);
  p.src_rows = dimy;
  p.src_cols = dimx;
  double s = p.sector_deg;
  // Octant fold, skew.cpp:46-58.
  if (s <= 45.0) {
    p.shear_deg = s;
  } else if (s <= 90.0) {
    p.shear_deg = 90.0 - s;
    p.n_ops = 1;
    p.ops[0] = 0;
  } else if (s < 135.0) {
    p.shear_deg = s - 90.0;
    p.n_ops = 2;
    p.ops[0] = 0;
    p.ops[1] = 1;
  } else {
    p.shear_deg = 180.0 - s;
    p.n_ops = 1;
    p.ops[0] = 1;
  }
  // Pinned corners, skew.cpp:61-67. std::tan runs on the host only.
  if (p.shear_deg == 0.0) {
    p.shear_tan = 0.0;
  } else if (p.shear_deg == 45.0) {
    p.shear_tan = 1.0;
  } else {
    p.shear_tan = std::tan(p.shear_deg * std::numbers::pi / 180.0);
  }
  // Inverse index map composition, skew.cpp:72-94.
  int rows = dimy, cols = dimx;
  int ii = 1, ij = 0, ci = 0, ji = 0, jj = 1, cj = 0;
  for (int o = 0; o < p.n_ops; ++o) {
    int a, b, c, d, e, f;
    if (p.ops[o] == 0) {
      a = ij; b = ii; c = ci; d = jj; e = ji; f = cj;
      std::swap(rows, cols);
    } else if (p.ops[o] == 1) {
      a = ii; b = -ij; c = ci + ij * (cols - 1);
      d = ji; e = -jj; f = cj + jj * (cols - 1);
    } else {
      a = -ii; b = ij; c = ci + ii * (rows - 1);
      d = -ji; e = jj; f = cj + ji * (rows - 1);
    }
    ii = a; ij = b; ci = c; ji = d; jj = e; cj = f;
  }
  p.rows = rows;
  p.cols = cols;
  int m[6] = {ii, ij, ci, ji, jj, cj};
  std::copy(m, m + 6, p.map);
  p.max_dd = distance_cap_cells(max_distance, p.shear_tan, cellsize);
  fill_tables(p);
  return p;
}

SectorPlanH plan_custom(int rows, int cols, double shear_tan) {
  if (rows < 1 || cols < 1) {
    throw std::invalid_argument("cannot shear an empty grid");
  }
  if (!(shear_tan >= 0.0 && shear_tan <= 1.0)) {
    throw std::invalid_argument("shear_tan must lie in [0, 1]");
  }
  SectorPlanH p;
  p.k = 0;
  p.ns = 2;
  p.shear_tan = shear_tan;
  p.rows = p.src_rows = rows;
  p.cols = p.src_cols = cols;
  fill_tables(p);
  return p;
}

std::vector<int> partition_lpt(const std::vector<long long>& work, int world) {
  std::vector<int> order(work.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return work[a] > work[b]; });
  std::vector<long long> load(world, 0);
  std::vector<int> owner(work.size(), 0);
  for (int s : order) {
    int best = 0;
    for (int r = 1; r < world; ++r) {
      if (load[r] < load[best]) best = r;
    }
    owner[s] = best;
    load[best] += work[s];
  }
  return owner;
}

namespace {

double next_unit(std::mt19937& rng) {  // dem.cpp:94-96
  return static_cast<double>(rng()) * (1.0 / 4294967296.0);
}

void box_blur(const std::vector<double>& g, int rows, int cols,
              std::vector<double>& out) {  // dem.cpp:98-114
  out.assign(g.size(), 0.0);
  for (int i = 0; i < rows; ++i) {
    for (int j = 0; j < cols; ++j) {
      double sum = 0.0;
      for (int di = -1; di <= 1; ++di) {
        for (int dj = -1; dj <= 1; ++dj) {
          int ii = std::clamp(i + di, 0, rows - 1);
          int jj = std::clamp(j + dj, 0, cols - 1);
          sum += g[static_cast<size_t>(ii) * cols + jj];
        }
      }
      out[static_cast<size_t>(i) * cols + j] = sum / 9.0;
    }
  }
}

// Fractal terrain: diamond-square midpoint displacement
// on the smallest (2^m+1)^2 lattice covering the grid, cropped top-left.
// Draws are raw mt19937(seed) words mapped to [-1, 1) as 2*(x/2^32)-1;
// corners first (amplitude 300 m), then per level l = 0.. the diamond step
// and the square step in row-major order with amplitude 300*2^(-0.8(l+1)).
// Values are 500 m + lattice, stored as float32.
void fractal(int dimy, int dimx, uint32_t seed, float* out) {
  int m = 0;
  while ((1 << m) + 1 < std::max(dimy, dimx)) ++m;
  const int S = (1 << m) + 1;
  std::vector<double> H(static_cast<size_t>(S) * S, 0.0);
  std::mt19937 rng(seed);
  auto draw = [&] { return 2.0 * (static_cast<double>(rng()) / 4294967296.0) - 1.0; };
  auto at = [&](int i, int j) -> double& { return H[static_cast<size_t>(i) * S + j]; };
  at(0, 0) = 300.0 * draw();
  at(0, S - 1) = 300.0 * draw();
  at(S - 1, 0) = 300.0 * draw();
  at(S - 1, S - 1) = 300.0 * draw();
  for (int l = 0; l < m; ++l) {
    const int step = 1 << (m - l);
    const int half = step / 2;
    const double amp = 300.0 * std::pow(2.0, -0.8 * (l + 1));
    for (int i = half; i < S; i += step) {
      for (int j = half; j < S; j += step) {
        double s = at(i - half, j - half) + at(i - half, j + half) +
                   at(i + half, j - half) + at(i + half, j + half);
        at(i, j) = s / 4.0 + amp * draw();
      }
    }
    for (int i = 0; i < S; i += half) {
      int j0 = ((i / half) % 2 == 0) ? half : 0;
      for (int j = j0; j < S; j += step) {
        double s = 0.0;
        int c = 0;
        if (i - half >= 0) { s += at(i - half, j); ++c; }
        if (i + half < S) { s += at(i + half, j); ++c; }
        if (j - half >= 0) { s += at(i, j - half); ++c; }
        if (j + half < S) { s += at(i, j + half); ++c; }
        at(i, j) = s / c + amp * draw();
      }
    }
  }
  for (int i = 0; i < dimy; ++i) {
    for (int j = 0; j < dimx; ++j) {
      out[static_cast<size_t>(i) * dimx + j] = static_cast<float>(500.0 + at(i, j));
    }
  }
}

}  // namespace

void make_synthetic(int kind, int dimy, int dimx, uint32_t seed, float* out) {
  if (dimy < 2 || dimx < 2) {
    throw std::invalid_argument("synthetic grid dimensions must be >= 2");
  }
  const size_t n = static_cast<size_t>(dimy) * dimx;
  std::fill(out, out + n, 0.0f);
  switch (kind) {
    case 0:
      break;
    case 1:
      for (int i = 0; i < dimy; ++i)
        for (int j = 0; j < dimx; ++j) out[static_cast<size_t>(i) * dimx + j] = static_cast<float>(j);
      break;
    case 2: {
      double cy = (dimy - 1) / 2.0, cx = (dimx - 1) / 2.0;
      double peak = 0.5 * std::min(dimy, dimx);
      for (int i = 0; i < dimy; ++i)
        for (int j = 0; j < dimx; ++j) {
          double d = std::hypot(i - cy, j - cx);
          out[static_cast<size_t>(i) * dimx + j] = static_cast<float>(std::max(0.0, peak - d));
        }
      break;
    }
    case 3: {
      std::mt19937 rng(seed);
      std::vector<double> a(n), b;
      for (size_t i = 0; i < n; ++i) a[i] = 3.0 * next_unit(rng);
      box_blur(a, dimy, dimx, b);
      box_blur(b, dimy, dimx, a);
      for (size_t i = 0; i < n; ++i) out[i] = static_cast<float>(a[i]);
      break;
    }
    case 4:
      fractal(dimy, dimx, seed, out);
      break;
    default:
      throw std::invalid_argument("unknown synthetic terrain kind");
  }
}

std::string validate_grid_header(int dimy, int dimx, double cellsize) {
  std::ostringstream os;
  if (dimy < 2 || dimx < 2) {
    os << "invalid grid: grid must be at least 2x2, got " << dimy << "x" << dimx;
    return os.str();
  }
  if (!(cellsize > 0.0) || !std::isfinite(cellsize)) {
    os << "invalid grid: cellsize must be a positive finite number, got " << cellsize;
    return os.str();
  }
  return "";
}

std::string nonfinite_message(long long idx, int dimx) {
  std::ostringstream os;
  os << "invalid grid: non-finite elevation at cell (" << idx / dimx << ", " << idx % dimx << ")";
  return os.str();
}

std::string validate_config(int ns, double h0, double max_distance, int n_gpus) {
  std::ostringstream os;
  if (ns < 2 || ns % 2 != 0) {
    os << "invalid config: ns must be an even integer >= 2, got " << ns;
    return os.str();
  }
  if (!(h0 >= 0.0) || !std::isfinite(h0)) {
    os << "invalid config: observer height must be >= 0, got " << h0;
    return os.str();
  }
  if (n_gpus < 1 && n_gpus != -1) {  // workers >= 1 (dem.cpp:74-78); -1 = every visible GPU
    os << "invalid config: GPU count must be >= 1 (or -1 for all), got " << n_gpus;
    return os.str();
  }
  if (max_distance != 0.0 && (!(max_distance > 0.0) || !std::isfinite(max_distance))) {
    os << "invalid config: max distance must be a positive finite number, got " << max_distance;
    return os.str();
  }
  return "";
}

std::string validate_inputs(const float* dem, int dimy, int dimx,
                            double cellsize, const float* nodata, int ns,
                            double h0, double max_distance, int n_gpus) {
  std::string e = validate_grid_header(dimy, dimx, cellsize);
  if (!e.empty()) return e;
  const size_t n = static_cast<size_t>(dimy) * dimx;
  for (size_t i = 0; i < n; ++i) {
    const float v = dem[i];
    if (nodata && v == *nodata) continue;
    if (!std::isfinite(v)) return nonfinite_message(static_cast<long long>(i), dimx);
  }
  if (nodata) {
    for (size_t i = 0; i < n; ++i) {
      if (dem[i] == *nodata) {
        return "grid contains nodata cells; fill them before running the engine";
      }
    }
  }
  return validate_config(ns, h0, max_distance, n_gpus);
}

}  // namespace sks
