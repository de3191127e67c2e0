// Host ray tables for the GPU rotational sweep (see sks_sweep.hpp).
// Compiled with -ffp-contract=off like the reference, and calling the same
// glibc functions in the same order as walk_ray (oracle.cpp:26-58).
#include "sks_sweep.hpp"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numbers>
#include <random>

namespace sks {

namespace {

// The ray from any observer toward azimuth_deg: steps n = 1..n_max along the
// dominant axis (oracle.cpp:31-57). fn(di, dj) per step.
template <typename Fn>
void ray_offsets(int dimy, int dimx, double azimuth_deg, Fn&& fn) {
  const double rad = azimuth_deg * std::numbers::pi / 180.0;
  const double vj = std::cos(rad);
  const double vi = std::sin(rad);
  if (std::abs(vj) >= std::abs(vi)) {
    const int sj = vj >= 0.0 ? 1 : -1;
    const double slope = vi / vj;
    for (int n = 1; n < dimx; ++n) {
      const int dj = n * sj;
      if (!fn(static_cast<int>(std::lround(slope * dj)), dj)) break;
    }
  } else {
    const int si = vi >= 0.0 ? 1 : -1;
    const double slope = vj / vi;
    for (int n = 1; n < dimy; ++n) {
      const int di = n * si;
      if (!fn(di, static_cast<int>(std::lround(slope * di)))) break;
    }
  }
}

double azimuth(int d, int ns) {
  const double s = (d / 2) * (360.0 / ns);  // oracle.cpp:123
  return d % 2 == 0 ? s : s + 180.0;        // oracle.cpp:124-125
}

}  // namespace

SweepTable build_sweep_table(int ns, int dimy, int dimx, double max_cells) {
  SweepTable t;
  t.ndir = ns;
  t.stride = std::max(1, std::max(dimy, dimx) - 1);
  t.steps.assign(static_cast<size_t>(t.ndir) * t.stride, SweepStep{0, 0, 0.0, 0.0f, 0});
  t.len.assign(t.ndir, 0);
  for (int d = 0; d < t.ndir; ++d) {
    SweepStep* row = t.steps.data() + static_cast<size_t>(d) * t.stride;
    int n = 0;
    ray_offsets(dimy, dimx, azimuth(d, ns), [&](int di, int dj) {
      // the grid bound is per observer (device); the distance cap is not
      const double dist = std::hypot(static_cast<double>(di), static_cast<double>(dj));
      if (dist > max_cells) return false;  // oracle.cpp:84
      row[n++] = SweepStep{di, dj, dist, static_cast<float>(1.0 / dist), 0};
      return true;
    });
    t.len[d] = n;
  }
  return t;
}

std::vector<SweepStep> ray_table(int dimy, int dimx, double azimuth_deg, double max_cells) {
  std::vector<SweepStep> steps;
  ray_offsets(dimy, dimx, azimuth_deg, [&](int di, int dj) {
    const double dist = std::hypot(static_cast<double>(di), static_cast<double>(dj));
    if (dist > max_cells) return false;  // oracle.cpp:84
    steps.push_back(SweepStep{di, dj, dist, static_cast<float>(1.0 / dist), 0});
    return true;
  });
  return steps;
}

std::vector<SweepStep> axis_points(int dimy, int dimx, int i0, int j0, double azimuth_deg) {
  std::vector<SweepStep> pts;
  ray_offsets(dimy, dimx, azimuth_deg, [&](int di, int dj) {
    const int i = i0 + di, j = j0 + dj;
    if (i < 0 || i >= dimy || j < 0 || j >= dimx) return false;  // oracle.cpp:40,52
    const double d = std::hypot(static_cast<double>(di), static_cast<double>(dj));
    pts.push_back(SweepStep{i, j, d, static_cast<float>(1.0 / d), 0});
    return true;
  });
  return pts;
}

void random_povs(int dimy, int dimx, int count, unsigned seed, int* ij) {
  std::mt19937 rng(seed);
  for (int n = 0; n < count; ++n) {
    // scaled raw 32-bit draws, i first (cli.cpp:212-218)
    ij[2 * n] = static_cast<int>((static_cast<std::uint64_t>(rng()) * static_cast<std::uint64_t>(dimy)) >> 32);
    ij[2 * n + 1] = static_cast<int>((static_cast<std::uint64_t>(rng()) * static_cast<std::uint64_t>(dimx)) >> 32);
  }
}

}  // namespace sks
