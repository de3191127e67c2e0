// Rotational-sweep viewshed (the reference's independent oracle,
// oracle.cpp:26-194) on the GPU: host-side ray tables.
//
// Every observer walks the same rasterised ray per azimuth: the cell offsets
// (di, dj) at step n and their Euclidean distance depend only on the
// azimuth, not on the observer (oracle.cpp:26-58). The host therefore
// evaluates the reference's own glibc cos/sin/lround/hypot once per
// (azimuth, step) and the kernel only reads the table — which is what makes
// the device results bit-identical to oracle.cpp (glibc's hypot is not the
// correctly rounded sqrt(di^2+dj^2) the device would compute: 0.6% of the
// integer pairs below 6000 differ).
#pragma once

#include <cstdint>
#include <vector>

namespace sks {

struct SweepStep {
  int di, dj;   // offset of the ray cell from the observer
  double dist;  // std::hypot(di, dj), oracle.cpp:43-44
  float inv;    // fl32(1 / dist): the device's FP32 filter
  int pad;
};

struct SweepTable {
  int ndir = 0;     // ns azimuths: k*(360/ns) then +180 (oracle.cpp:122-126)
  int stride = 0;   // steps per direction in `steps`
  std::vector<SweepStep> steps;  // ndir * stride
  std::vector<int> len;          // usable steps per direction (grid + distance cap)
};

// max_cells = max_distance / cellsize, +inf when uncapped (oracle.cpp:117-119).
SweepTable build_sweep_table(int ns, int dimy, int dimx, double max_cells);

// The ray of one azimuth (any observer), steps with dist > max_cells cut.
std::vector<SweepStep> ray_table(int dimy, int dimx, double azimuth_deg, double max_cells);

// select_axis_point_set (oracle.cpp:62-71) for one observer and azimuth.
std::vector<SweepStep> axis_points(int dimy, int dimx, int i0, int j0, double azimuth_deg);

// random_povs (cli.cpp:207-221): count (i, j) pairs from raw mt19937 draws.
void random_povs(int dimy, int dimx, int count, unsigned seed, int* ij);

}  // namespace sks
