// ESRI ASCII grid ingest and output — the "DEM load" entry point of the
// reference (ascii_grid.hpp:15-31, src/ascii_grid.cpp:110-274), host C++.
//
// Same accepted language and the same diagnostics as read_ascii_grid:
// header keys ncols, nrows, xllcorner, yllcorner, cellsize (in that order,
// case-insensitive), optional NODATA_value, then nrows*ncols cell values,
// north row first; numbers are read with std::from_chars as double and cell
// values / NODATA rounded to float (ascii_grid.cpp:85-108, 160-178); errors
// carry "source:line:col" for a token and "source:line" at end of input
// (ascii_grid.cpp:55-65), then validate(Dem) runs (dem.cpp:36-60).
//
// Unlike the reference's single istream tokenizer, the body (about 1 GB of
// text for a 10000^2 grid) is parsed by all host threads: the buffer is cut
// into chunks at whitespace, each thread converts its chunk into a private
// vector, and the chunks are concatenated in order. Line and column of a
// diagnostic are recomputed only when there is one. Writers format rows in
// parallel with the reference's "%.9g" (DEM) / "%.10g" (viewshed) and
// write the pieces in order.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "sks_io.hpp"

namespace sks {

namespace {

constexpr long long kMaxCells = 1LL << 31;  // ascii_grid.cpp:108

inline bool is_space(char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; }

// Position of byte offset o for diagnostics: 1-based line and column (the
// reference's getline/isspace tokenizer counts bytes within a line).
void line_col(const char* buf, size_t o, int* line, int* col) {
  int ln = 1;
  size_t last_nl = static_cast<size_t>(-1);
  for (size_t i = 0; i < o; ++i) {
    if (buf[i] == '\n') {
      ++ln;
      last_nl = i;
    }
  }
  *line = ln;
  *col = static_cast<int>(o - (last_nl + 1)) + 1;
}

// The line count the reference's tokenizer has reached at end of input:
// the number of getline() calls that succeeded.
int eof_line(const char* buf, size_t n) {
  int lines = 0;
  for (size_t i = 0; i < n; ++i) lines += buf[i] == '\n';
  if (n > 0 && buf[n - 1] != '\n') ++lines;
  return lines;
}

struct Cursor {
  const char* buf;
  size_t n;
  size_t pos = 0;
  // next whitespace-separated token: [b, e); false at end of input
  bool next(size_t* b, size_t* e) {
    while (pos < n && is_space(buf[pos])) ++pos;
    if (pos >= n) return false;
    *b = pos;
    while (pos < n && !is_space(buf[pos])) ++pos;
    *e = pos;
    return true;
  }
};

std::string lower(const char* b, const char* e) {
  std::string s(b, e);
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

[[noreturn]] void fail_at(const std::string& src, const char* buf, size_t o, const std::string& what) {
  int line = 0, col = 0;
  line_col(buf, o, &line, &col);
  throw GridFormatError(src + ":" + std::to_string(line) + ":" + std::to_string(col) + ": " + what);
}

[[noreturn]] void fail_eof(const std::string& src, const char* buf, size_t n, const std::string& what) {
  throw GridFormatError(src + ":" + std::to_string(eof_line(buf, n)) + ": " + what);
}

bool to_double(const char* b, const char* e, double* v) {
  auto [p, ec] = std::from_chars(b, e, *v);
  return ec == std::errc{} && p == e;
}

bool to_long(const char* b, const char* e, long* v) {
  auto [p, ec] = std::from_chars(b, e, *v);
  return ec == std::errc{} && p == e;
}

std::string fmt_g(double v) {  // operator<< on a double (default stream precision 6)
  char b[64];
  std::snprintf(b, sizeof(b), "%g", v);
  return b;
}

unsigned threads_for(size_t bytes) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t per = 1 << 20;  // at least 1 MB of text per thread
  return static_cast<unsigned>(std::min<size_t>(hw, std::max<size_t>(1, bytes / per)));
}

}  // namespace

AsciiGrid parse_ascii_grid(const char* buf, size_t n, const std::string& src) {
  Cursor cur{buf, n};
  size_t b = 0, e = 0;
  auto expect_key = [&](const char* key) {
    if (!cur.next(&b, &e)) fail_eof(src, buf, n, std::string("missing header key '") + key + "'");
    if (lower(buf + b, buf + e) != key) {
      fail_at(src, buf, b, std::string("expected header key '") + key + "', got '" + std::string(buf + b, buf + e) +
                               "'");
    }
    if (!cur.next(&b, &e)) fail_eof(src, buf, n, std::string("missing value for header key '") + key + "'");
  };
  auto need_long = [&](const char* what) {
    long v = 0;
    if (!to_long(buf + b, buf + e, &v)) {
      fail_at(src, buf, b, std::string("expected an integer for ") + what + ", got '" + std::string(buf + b, buf + e) +
                               "'");
    }
    return v;
  };
  auto need_double = [&](const char* what) {
    double v = 0;
    if (!to_double(buf + b, buf + e, &v)) {
      fail_at(src, buf, b, std::string("expected a number for ") + what + ", got '" + std::string(buf + b, buf + e) +
                               "'");
    }
    return v;
  };
  AsciiGrid g;
  expect_key("ncols");
  const long ncols = need_long("ncols");
  expect_key("nrows");
  const long nrows = need_long("nrows");
  expect_key("xllcorner");
  g.xllcorner = need_double("xllcorner");
  expect_key("yllcorner");
  g.yllcorner = need_double("yllcorner");
  expect_key("cellsize");
  g.cellsize = need_double("cellsize");
  if (ncols < 2 || nrows < 2) {
    throw GridFormatError(src + ": grid must be at least 2x2, header declares " + std::to_string(nrows) + "x" +
                          std::to_string(ncols));
  }
  if (static_cast<long long>(ncols) * nrows > kMaxCells) {
    throw GridFormatError(src + ": declared grid " + std::to_string(nrows) + "x" + std::to_string(ncols) +
                          " is too large");
  }
  if (!(g.cellsize > 0.0)) throw GridFormatError(src + ": cellsize must be positive, got " + fmt_g(g.cellsize));
  g.nrows = static_cast<int>(nrows);
  g.ncols = static_cast<int>(ncols);
  if (!cur.next(&b, &e)) fail_eof(src, buf, n, "no cell values after the header");
  if (lower(buf + b, buf + e) == "nodata_value") {
    if (!cur.next(&b, &e)) fail_eof(src, buf, n, "missing value for header key 'NODATA_value'");
    g.has_nodata = true;
    g.nodata = static_cast<float>(need_double("NODATA_value"));
    if (!cur.next(&b, &e)) fail_eof(src, buf, n, "no cell values after the header");
  }

  // Body from the first cell token on, in parallel chunks cut at whitespace.
  const size_t body = b;
  const long long total = static_cast<long long>(ncols) * nrows;
  const unsigned T = threads_for(n - body);
  std::vector<size_t> cut(T + 1);
  cut[0] = body;
  cut[T] = n;
  for (unsigned t = 1; t < T; ++t) {
    size_t c = body + (n - body) * t / T;
    while (c < n && !is_space(buf[c])) ++c;  // move to a token boundary
    cut[t] = std::max(c, cut[t - 1]);
  }
  struct Part {
    std::vector<float> v;
    size_t bad = static_cast<size_t>(-1);  // offset of the first malformed token
    long long bad_index = -1;              // its index within the part
  };
  std::vector<Part> parts(T);
  auto work = [&](unsigned t) {
    Part& p = parts[t];
    Cursor c{buf, cut[t + 1]};
    c.pos = cut[t];
    p.v.reserve(static_cast<size_t>(std::min<long long>(total, (cut[t + 1] - cut[t]) / 2 + 1)));
    size_t tb = 0, te = 0;
    while (c.next(&tb, &te)) {
      double d = 0;
      if (!to_double(buf + tb, buf + te, &d)) {
        p.bad = tb;
        p.bad_index = static_cast<long long>(p.v.size());
        return;  // later tokens of this chunk are not needed for the diagnosis
      }
      p.v.push_back(static_cast<float>(d));
    }
  };
  if (T == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
  }
  // The reference reads tokens in order: the first of (malformed token,
  // token past the last cell, end of input) decides the diagnostic.
  long long before = 0;  // tokens in earlier parts
  for (unsigned t = 0; t < T; ++t) {
    const Part& p = parts[t];
    if (p.bad_index >= 0 && before + p.bad_index < total) {
      fail_at(src, buf, p.bad, "expected a number for cell value, got '" +
                                   std::string(buf + p.bad, std::find_if(buf + p.bad, buf + n, is_space)) + "'");
    }
    const long long here = static_cast<long long>(p.v.size()) + (p.bad_index >= 0 ? 1 : 0);
    if (before + here > total) {
      // the first token past the last cell
      Cursor c{buf, cut[t + 1]};
      c.pos = cut[t];
      size_t tb = 0, te = 0;
      for (long long k = 0; k <= total - before; ++k) c.next(&tb, &te);
      fail_at(src, buf, tb, "trailing data after the last cell value");
    }
    before += here;
  }
  if (before < total) {
    fail_eof(src, buf, n, "unexpected end of data: expected " + std::to_string(total) + " cell values, got " +
                              std::to_string(before));
  }
  g.values.resize(static_cast<size_t>(total));
  size_t o = 0;
  for (const Part& p : parts) {
    std::copy(p.v.begin(), p.v.end(), g.values.begin() + static_cast<long long>(o));
    o += p.v.size();
  }
  // validate(Dem) (dem.cpp:36-60): cellsize finite, non-nodata cells finite
  if (!std::isfinite(g.cellsize)) {
    throw GridFormatError(src + ": cellsize must be a positive finite number, got " + fmt_g(g.cellsize));
  }
  for (size_t i = 0; i < g.values.size(); ++i) {
    const float v = g.values[i];
    if (g.has_nodata && v == g.nodata) continue;
    if (!std::isfinite(v)) {
      throw GridFormatError(src + ": non-finite elevation at cell (" + std::to_string(i / ncols) + ", " +
                            std::to_string(i % ncols) + ")");
    }
  }
  return g;
}

AsciiGrid read_ascii_grid_file(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw GridFormatError("cannot open '" + path + "' for reading");
  std::vector<char> buf;
  char chunk[1 << 16];
  size_t got = 0;
  while ((got = std::fread(chunk, 1, sizeof(chunk), f)) > 0) buf.insert(buf.end(), chunk, chunk + got);
  std::fclose(f);
  return parse_ascii_grid(buf.data(), buf.size(), path);
}

namespace {

std::string header_text(int ncols, int nrows, double xll, double yll, double cellsize) {
  char b[64];
  std::string s = "ncols " + std::to_string(ncols) + "\nnrows " + std::to_string(nrows) + "\n";
  std::snprintf(b, sizeof(b), "%.10g", xll);
  s += std::string("xllcorner ") + b + "\n";
  std::snprintf(b, sizeof(b), "%.10g", yll);
  s += std::string("yllcorner ") + b + "\n";
  std::snprintf(b, sizeof(b), "%.10g", cellsize);
  s += std::string("cellsize ") + b + "\n";
  return s;
}

// Rows [0, nrows) formatted by all host threads, written in order.
template <typename Fmt>
void write_rows(FILE* f, int nrows, int ncols, Fmt&& fmt_cell, const std::string& path) {
  const unsigned T = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), nrows));
  const int block = 256;  // rows per piece
  for (int r0 = 0; r0 < nrows; r0 += block * static_cast<int>(T)) {
    std::vector<std::string> piece(T);
    auto work = [&](unsigned t) {
      const int a = r0 + static_cast<int>(t) * block, z = std::min(nrows, a + block);
      std::string& s = piece[t];
      char b[64];
      for (int i = a; i < z; ++i) {
        for (int j = 0; j < ncols; ++j) {
          const int len = fmt_cell(b, sizeof(b), i, j);
          s.append(b, static_cast<size_t>(len));
          s.push_back(j + 1 == ncols ? '\n' : ' ');
        }
      }
    };
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
    for (const std::string& s : piece) {
      if (!s.empty() && std::fwrite(s.data(), 1, s.size(), f) != s.size()) {
        throw std::runtime_error("failed while writing '" + path + "'");
      }
    }
  }
}

}  // namespace

void write_ascii_grid_dem(const std::string& path, const float* values, int nrows, int ncols, double xll,
                          double yll, double cellsize, const float* nodata) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot open '" + path + "' for writing");
  std::string h = header_text(ncols, nrows, xll, yll, cellsize);
  if (nodata) {
    char b[64];
    std::snprintf(b, sizeof(b), "%.9g", static_cast<double>(*nodata));
    h += std::string("NODATA_value ") + b + "\n";
  }
  try {
    if (std::fwrite(h.data(), 1, h.size(), f) != h.size()) throw std::runtime_error("failed while writing '" + path + "'");
    write_rows(f, nrows, ncols, [&](char* b, size_t n, int i, int j) {
      // to_chars(general, p) is specified as printf("%.pg") in the C locale
      return static_cast<int>(std::to_chars(b, b + n, static_cast<double>(values[static_cast<size_t>(i) * ncols + j]),
                                            std::chars_format::general, 9).ptr - b);
    }, path);
  } catch (...) {
    std::fclose(f);
    throw;
  }
  if (std::fclose(f) != 0) throw std::runtime_error("failed while writing '" + path + "'");
}

void write_ascii_grid_vs(const std::string& path, const double* values, int nrows, int ncols, double factor,
                         double xll, double yll, double cellsize) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot open '" + path + "' for writing");
  const std::string h = header_text(ncols, nrows, xll, yll, cellsize);
  try {
    if (std::fwrite(h.data(), 1, h.size(), f) != h.size()) throw std::runtime_error("failed while writing '" + path + "'");
    write_rows(f, nrows, ncols, [&](char* b, size_t n, int i, int j) {
      const double v = values[static_cast<size_t>(i) * ncols + j];
      return static_cast<int>(
          std::to_chars(b, b + n, factor == 1.0 ? v : v * factor, std::chars_format::general, 10).ptr - b);
    }, path);
  } catch (...) {
    std::fclose(f);
    throw;
  }
  if (std::fclose(f) != 0) throw std::runtime_error("failed while writing '" + path + "'");
}

namespace {

// "dem.flt" / "dem.hdr" / "dem" -> ("dem.hdr", "dem.flt")
void float_grid_paths(const std::string& path, std::string* hdr, std::string* flt) {
  std::string base = path;
  const size_t dot = path.find_last_of('.');
  const size_t slash = path.find_last_of('/');
  if (dot != std::string::npos && (slash == std::string::npos || dot > slash)) {
    const std::string ext = lower(path.data() + dot, path.data() + path.size());
    if (ext == ".flt" || ext == ".hdr") base = path.substr(0, dot);
  }
  *hdr = base + ".hdr";
  *flt = base + ".flt";
}

std::string slurp(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw GridFormatError("cannot open '" + path + "' for reading");
  std::string s;
  char b[1 << 16];
  size_t k;
  while ((k = std::fread(b, 1, sizeof(b), f)) > 0) s.append(b, k);
  std::fclose(f);
  return s;
}

}  // namespace

AsciiGrid read_float_grid(const std::string& path) {
  std::string hp, fp;
  float_grid_paths(path, &hp, &fp);
  const std::string h = slurp(hp);
  AsciiGrid g;
  bool have[5] = {false, false, false, false, false};
  bool center[2] = {false, false};
  bool msb = false;
  Cursor cur{h.data(), h.size()};
  size_t b = 0, e = 0;
  while (cur.next(&b, &e)) {
    const std::string key = lower(h.data() + b, h.data() + e);
    const size_t kb = b, ke = e;
    if (!cur.next(&b, &e)) fail_eof(hp, h.data(), h.size(), "missing value for header key '" + key + "'");
    const char* vb = h.data() + b;
    const char* ve = h.data() + e;
    double d = 0.0;
    long l = 0;
    if (key == "ncols" || key == "nrows") {
      if (!to_long(vb, ve, &l) || l < 1 || l > INT32_MAX) {
        fail_at(hp, h.data(), b, "expected a positive integer for '" + key + "', got '" + std::string(vb, ve) + "'");
      }
      (key == "ncols" ? g.ncols : g.nrows) = static_cast<int>(l);
      have[key == "ncols" ? 0 : 1] = true;
    } else if (key == "byteorder") {
      const std::string v = lower(vb, ve);
      if (v == "msbfirst" || v == "m") {
        msb = true;
      } else if (v == "lsbfirst" || v == "i") {
        msb = false;
      } else {
        fail_at(hp, h.data(), b, "byteorder must be LSBFIRST or MSBFIRST, got '" + std::string(vb, ve) + "'");
      }
    } else if (key == "xllcorner" || key == "xllcenter" || key == "yllcorner" || key == "yllcenter" ||
               key == "cellsize" || key == "nodata_value") {
      if (!to_double(vb, ve, &d)) {
        fail_at(hp, h.data(), b, "expected a number for '" + key + "', got '" + std::string(vb, ve) + "'");
      }
      if (key[0] == 'x') {
        g.xllcorner = d, have[2] = true, center[0] = key == "xllcenter";
      } else if (key[0] == 'y') {
        g.yllcorner = d, have[3] = true, center[1] = key == "yllcenter";
      } else if (key == "cellsize") {
        g.cellsize = d, have[4] = true;
      } else {
        g.has_nodata = true;
        g.nodata = static_cast<float>(d);
      }
    } else {
      fail_at(hp, h.data(), kb, "unknown header key '" + std::string(h.data() + kb, h.data() + ke) + "'");
    }
  }
  static const char* names[5] = {"ncols", "nrows", "xllcorner", "yllcorner", "cellsize"};
  for (int k = 0; k < 5; ++k) {
    if (!have[k]) throw GridFormatError(hp + ": missing header key '" + names[k] + "'");
  }
  if (!(g.cellsize > 0.0) || !std::isfinite(g.cellsize)) {
    throw GridFormatError(hp + ": cellsize must be a positive finite number, got " + fmt_g(g.cellsize));
  }
  // cell-centre origins move to the corner (half a cell)
  if (center[0]) g.xllcorner -= 0.5 * g.cellsize;
  if (center[1]) g.yllcorner -= 0.5 * g.cellsize;
  const long long cells = static_cast<long long>(g.nrows) * g.ncols;
  if (cells > kMaxCells) throw GridFormatError(hp + ": grid of " + std::to_string(cells) + " cells is too large");
  FILE* f = std::fopen(fp.c_str(), "rb");
  if (!f) throw GridFormatError("cannot open '" + fp + "' for reading");
  g.values.resize(static_cast<size_t>(cells));
  const size_t got = std::fread(g.values.data(), sizeof(float), g.values.size(), f);
  const bool extra = std::fgetc(f) != EOF;
  std::fclose(f);
  if (got != g.values.size() || extra) {
    throw GridFormatError(fp + ": expected " + std::to_string(cells * 4) + " bytes of float32 cells for " +
                          std::to_string(g.nrows) + "x" + std::to_string(g.ncols) + (extra ? ", got more" : ", got fewer"));
  }
  if (msb) {
    for (float& v : g.values) {
      uint32_t u;
      std::memcpy(&u, &v, 4);
      u = __builtin_bswap32(u);
      std::memcpy(&v, &u, 4);
    }
  }
  return g;
}

void write_float_grid(const std::string& path, const float* values, int nrows, int ncols, double xll, double yll,
                      double cellsize, const float* nodata) {
  std::string hp, fp;
  float_grid_paths(path, &hp, &fp);
  std::string h = header_text(ncols, nrows, xll, yll, cellsize);
  if (nodata) {
    char b[64];
    std::snprintf(b, sizeof(b), "%.9g", static_cast<double>(*nodata));
    h += std::string("NODATA_value ") + b + "\n";
  }
  h += "byteorder LSBFIRST\n";
  FILE* f = std::fopen(hp.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot open '" + hp + "' for writing");
  const bool okh = std::fwrite(h.data(), 1, h.size(), f) == h.size();
  if (std::fclose(f) != 0 || !okh) throw std::runtime_error("failed while writing '" + hp + "'");
  f = std::fopen(fp.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot open '" + fp + "' for writing");
  const size_t n = static_cast<size_t>(nrows) * static_cast<size_t>(ncols);
  const bool ok = std::fwrite(values, sizeof(float), n, f) == n;
  if (std::fclose(f) != 0 || !ok) throw std::runtime_error("failed while writing '" + fp + "'");
}

void fill_nodata_nearest(const float* in, int rows, int cols, float nodata, float* out) {
  const size_t n = static_cast<size_t>(std::max(rows, 0)) * static_cast<size_t>(std::max(cols, 0));
  std::copy(in, in + n, out);
  // a ring buffer of cell indices is the reference's deque: every cell is
  // pushed exactly once, seeds first in row-major order
  std::vector<int> queue;
  queue.reserve(n);
  std::vector<unsigned char> filled(n, 0);
  for (size_t c = 0; c < n; ++c) {
    if (!(in[c] == nodata)) {  // Dem::is_nodata (dem.hpp:35)
      filled[c] = 1;
      queue.push_back(static_cast<int>(c));
    }
  }
  if (queue.empty()) throw std::runtime_error("cannot fill a grid that is entirely nodata");
  static constexpr int kDi[4] = {-1, 1, 0, 0};
  static constexpr int kDj[4] = {0, 0, -1, 1};
  for (size_t head = 0; head < queue.size(); ++head) {
    const int c = queue[head];
    const int i = c / cols, j = c % cols;
    for (int k = 0; k < 4; ++k) {
      const int ii = i + kDi[k], jj = j + kDj[k];
      if (ii < 0 || ii >= rows || jj < 0 || jj >= cols) continue;
      const int cc = ii * cols + jj;
      if (filled[cc]) continue;
      out[cc] = out[c];
      filled[cc] = 1;
      queue.push_back(cc);
    }
  }
}

void write_heatmap(const std::string& path, const double* values, int rows, int cols, int palette) {
  const size_t n = static_cast<size_t>(std::max(rows, 0)) * static_cast<size_t>(std::max(cols, 0));
  if (n == 0) throw std::invalid_argument("cannot render an empty grid");
  // min/max with the non-finite check, split over host threads; lo starts at
  // the first cell exactly as the reference's (heatmap.cpp:18-27)
  const unsigned T = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(),
                                                     static_cast<unsigned>((n + 65535) / 65536)));
  std::vector<double> los(T, values[0]), his(T, values[0]);
  std::vector<char> bad(T, 0);
  {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t) {
      th.emplace_back([&, t] {
        const size_t a = n * t / T, z = n * (t + 1) / T;
        double lo = values[0], hi = values[0];
        for (size_t c = a; c < z; ++c) {
          const double x = values[c];
          if (!std::isfinite(x)) {
            bad[t] = 1;
            return;
          }
          lo = std::min(lo, x);
          hi = std::max(hi, x);
        }
        los[t] = lo;
        his[t] = hi;
      });
    }
    for (auto& x : th) x.join();
  }
  for (unsigned t = 0; t < T; ++t) {
    if (bad[t]) throw std::invalid_argument("cannot render a grid with non-finite values");
  }
  double lo = values[0], hi = values[0];
  for (unsigned t = 0; t < T; ++t) {
    lo = std::min(lo, los[t]);
    hi = std::max(hi, his[t]);
  }
  const double range = hi - lo;
  const bool gray = palette == 0;
  std::string bytes = std::string(gray ? "P5\n" : "P6\n") + std::to_string(cols) + " " + std::to_string(rows) +
                      "\n255\n";
  const size_t head = bytes.size(), px = gray ? 1 : 3;
  bytes.resize(head + n * px);
  {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t) {
      th.emplace_back([&, t] {
        const size_t a = n * t / T, z = n * (t + 1) / T;
        for (size_t c = a; c < z; ++c) {
          const double u = range > 0.0 ? (values[c] - lo) / range : 0.0;
          const auto level = static_cast<unsigned char>(std::lround(u * 255.0));  // heatmap.cpp:35-36
          char* o = bytes.data() + head + c * px;
          if (gray) {
            o[0] = static_cast<char>(level);
          } else {
            o[0] = static_cast<char>(level);        // red
            o[1] = 0;                               // green
            o[2] = static_cast<char>(255 - level);  // blue
          }
        }
      });
    }
    for (auto& x : th) x.join();
  }
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot open '" + path + "' for writing");
  const bool ok = std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size();
  if (std::fclose(f) != 0 || !ok) throw std::runtime_error("failed while writing '" + path + "'");
}

}  // namespace sks
