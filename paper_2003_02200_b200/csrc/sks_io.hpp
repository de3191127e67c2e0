// ESRI ASCII grid I/O (host C++): reference ascii_grid.hpp:15-31.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

namespace sks {

// read_ascii_grid's failure type (ascii_grid.hpp:15-18): message with the
// offending source:line:col.
class GridFormatError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct AsciiGrid {
  int nrows = 0, ncols = 0;
  double xllcorner = 0.0, yllcorner = 0.0, cellsize = 1.0;
  bool has_nodata = false;
  float nodata = 0.f;
  std::vector<float> values;  // nrows * ncols, north row first
};

// read_ascii_grid(istream, source_name) / read_ascii_grid(path)
AsciiGrid parse_ascii_grid(const char* buf, size_t n, const std::string& source);
AsciiGrid read_ascii_grid_file(const std::string& path);

// write_ascii_grid(Dem, path): header "%.10g", cells "%.9g", optional NODATA_value
void write_ascii_grid_dem(const std::string& path, const float* values, int nrows, int ncols, double xll,
                          double yll, double cellsize, const float* nodata);
// write_ascii_grid(VsGrid, units, cellsize, origin, path): cells "%.10g" of
// value * factor (factor 1 when the units already match, else
// convert_units' 1e-6 / 1e6, dem.cpp:24-34)
void write_ascii_grid_vs(const std::string& path, const double* values, int nrows, int ncols, double factor,
                         double xll, double yll, double cellsize);

// Binary side format for large DEMs: the ESRI float grid,
// a `.hdr` text header (ncols, nrows, xllcorner|xllcenter,
// yllcorner|yllcenter, cellsize, optional NODATA_value, byteorder
// LSBFIRST|MSBFIRST) next to a `.flt` file of nrows*ncols IEEE float32, north
// row first. `path` may name either file (or neither extension).
AsciiGrid read_float_grid(const std::string& path);
void write_float_grid(const std::string& path, const float* values, int nrows, int ncols, double xll,
                      double yll, double cellsize, const float* nodata);

// fill_nodata_nearest (dem.cpp:175-213): every nodata cell takes the value
// of the cell the multi-source breadth-first search (seeds in row-major
// order, neighbours up/down/left/right) reaches it from. Throws
// std::runtime_error for a grid that is entirely nodata.
void fill_nodata_nearest(const float* in, int rows, int cols, float nodata, float* out);

// write_heatmap (heatmap.cpp:11-56): min-max normalised 8-bit raster, binary
// PGM (palette 0, Gray) or PPM (palette 1, BlueRed).
void write_heatmap(const std::string& path, const double* values, int rows, int cols, int palette);

}  // namespace sks
