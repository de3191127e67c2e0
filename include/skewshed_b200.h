/*
 * skewshed_b200 — C ABI of the B200-native sDEM total-viewshed path.
 *
 * This is the drop-in boundary. Every entry point takes plain
 * pointers and sizes, returns an sks_status, and never lets a C++ exception
 * cross the ABI; the message of the last failure on the calling thread is in
 * sks_last_error(). The C++ facade in skewshed_b200.hpp restores the
 * reference's signatures and exception types on top of this header.
 *
 * Citations are to the reference (/root/reference/proj/...) entry point each
 * function replaces.
 *
 * Memory: functions named *_host take host buffers (the library owns all
 * device memory for the call). Functions taking a `void* stream` and `d_`
 * pointers work on caller-owned device memory on that CUDA stream.
 */
#ifndef SKEWSHED_B200_H
#define SKEWSHED_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SKS_OK = 0,
  SKS_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  SKS_OUT_OF_RANGE = 2,     /* std::out_of_range */
  SKS_CUDA_ERROR = 3,
  SKS_NCCL_ERROR = 4,
  SKS_INTERNAL = 5, /* std::runtime_error */
  SKS_FORMAT_ERROR = 6 /* GridFormatError (ascii_grid.hpp:15-18) */
} sks_status;

enum { SKS_UNITS_M2 = 0, SKS_UNITS_KM2 = 1 };
enum { SKS_SCAN_FORWARD = 0, SKS_SCAN_BACKWARD = 1 };
enum { SKS_NO_DISTANCE_CAP = 2147483647 }; /* scan.hpp:15 kNoDistanceCap */

enum { SKS_ALL_GPUS = -1 }; /* sks_run_config.n_gpus: every visible device */

/* RunConfig, dem.hpp:40-46. std::optional<double> max_distance becomes a
 * double with 0 = off (the CLI's own convention, cli.cpp:82,112); Units
 * becomes an int. The reference's `workers` (host threads sharing one call,
 * engine.cpp:109-220) becomes n_gpus: GPUs sharing one call, devices
 * device .. device + n_gpus - 1 (SKS_ALL_GPUS: every visible one from
 * `device` on), one host thread per GPU and one NCCL reduce of the maps.
 * Validated like workers (>= 1, or SKS_ALL_GPUS). */
typedef struct {
  int ns;              /* sector count over 2*pi, even >= 2 */
  double h0;           /* observer height above ground, m, >= 0 */
  double max_distance; /* visibility cap in m; 0 = off */
  int units;           /* SKS_UNITS_M2 or SKS_UNITS_KM2 */
  int device;          /* first CUDA device ordinal */
  int n_gpus;          /* GPUs for total_viewshed[_raw]: >= 1 or SKS_ALL_GPUS */
} sks_run_config;

/* EngineStats, engine.hpp:25-32, plus GPU evidence. Phase seconds are
 * CUDA-event durations on the library's stream; total_seconds is host wall
 * time of the call. */
typedef struct {
  double skew_seconds;   /* relocation kernels (DEM -> sDEM) */
  double scan_seconds;   /* line-of-sight scan kernels */
  double fixup_seconds;  /* exact FP64 re-scan of guard-flagged POV groups */
  double unskew_seconds; /* unskew + ordered accumulation kernels */
  double reduce_seconds; /* scaling (+ collective when sharded) */
  double total_seconds;
  int sectors;
  int batches;
  long long kernel_launches;   /* our kernels launched during the call */
  long long target_evals;      /* exact sum of scanned targets */
  long long flagged_groups;    /* POV groups re-run by the exact fixup */
  long long h2d_bytes;
  long long d2h_bytes;
  long long skipped_target_slots; /* lane-target slots decided by the
                                     certified hidden-block skip */
  int scan_kernel;  /* scan kernel of the call's last batch: 2 = one row x 64
                       positions per task, 3 = row pairs, 4 = row quads
                       (autotuned per shape) */
  int pad_;
} sks_stats;

/* SectorPlan, skew.hpp:29-41. ops: 0 Transpose, 1 FlipCols, 2 FlipRows. */
typedef struct {
  int sector_index;
  int ns;
  double sector_deg;
  double shear_deg;
  double shear_tan;
  int n_ops;
  int ops[3];
  int rows, cols;         /* grid shape after pre_ops */
  int src_rows, src_cols; /* DEM shape */
  int to_source[6];       /* IndexMap ii, ij, ci, ji, jj, cj */
  int base;               /* sDEM row offset (skew.cpp:16-19) */
  int skw_rows;           /* base + rows */
} sks_sector_plan;

/* Message of the last failing call on this thread ("" if none). */
const char* sks_last_error(void);
/* Library version string. */
const char* sks_version(void);
/* Number of visible CUDA devices (0 on a host without a GPU). */
int sks_device_count(void);
/* Longest skewed row (cells) the shared-memory scan kernel holds; longer rows
 * are scanned POV by POV by the exact kernel (same results, slower). Rows are
 * limited to 46340 cells overall (the int32 ring sums; SKS_INVALID_ARGUMENT
 * beyond). No GPU needed. */
int sks_scan_row_limit(void);

/* ---- host planning (no GPU needed) ---------------------------------- */

/* plan_sector, skew.cpp:23-95 (also fills base/skw_rows). */
sks_status sks_plan_sector(int k, int ns, int dimy, int dimx,
                           sks_sector_plan* out);
/* shear_params, skew.cpp:97-101. */
void sks_shear_params(double shear_tan, int j, int* dest, double* frac);
/* distance_cap_cells, engine.cpp:29-36 (max_distance 0 = off). */
int sks_distance_cap_cells(double max_distance, double shear_tan,
                           double cellsize);
/* area_scale_factor, engine.cpp:103-107. */
double sks_area_scale_factor(int ns, double cellsize, int units);
/* row_ranges of build_skw (skew.cpp:185-195) computed from the plan alone
 * (the weights do not depend on elevations). ranges: 2*skw_rows ints. */
sks_status sks_row_ranges(int rows, int cols, double shear_tan, int* ranges,
                          int* skw_rows_out);
/* Exact number of target evaluations of sector k (sum over skewed rows and
 * POVs of the forward+backward scan lengths, capped by max_dd). */
long long sks_sector_target_evals(int k, int ns, int dimy, int dimx,
                                  double cellsize, double max_distance);
/* Static sector-to-rank assignment (longest-processing-time first on the
 * exact per-sector work). owner: ns/2 ints. */
sks_status sks_partition_sectors(int ns, int dimy, int dimx, double cellsize,
                                 double max_distance, int world, int* owner);
/* make_synthetic, dem.cpp:118-173 (kind 0 Flat, 1 Ramp, 2 Cone,
 * 3 SmoothedNoise) plus kind 4 Fractal (diamond-square). */
sks_status sks_make_synthetic(int kind, int dimy, int dimx, uint32_t seed,
                              float* out);
/* validate(Dem) + has_nodata_cells + validate(RunConfig), dem.cpp:16-87
 * (engine.cpp:68-81 require_valid). nodata: pointer to the nodata value or
 * NULL. */
sks_status sks_validate(const float* dem, int dimy, int dimx, double cellsize,
                        const float* nodata, const sks_run_config* cfg);

/* ---- end-to-end (host buffers) -------------------------------------- */

/* total_viewshed, engine.cpp:222-233: out_vs (dimy*dimx doubles) receives
 * the per-cell viewshed area in cfg->units. With cfg->n_gpus > 1 the call is
 * shared by that many GPUs (sks_total_viewshed_devices); stats then sum the
 * per-GPU device seconds (as the reference sums worker seconds) and
 * reduce_seconds is the NCCL reduce + scaling. */
sks_status sks_total_viewshed(const float* dem, int dimy, int dimx,
                              double cellsize, const sks_run_config* cfg,
                              double* out_vs, sks_stats* stats);
/* total_viewshed_raw, engine.cpp:109-220 (pre-scaling accumulator). */
sks_status sks_total_viewshed_raw(const float* dem, int dimy, int dimx,
                                  double cellsize, const sks_run_config* cfg,
                                  double* out_raw, sks_stats* stats);
/* In-process multi-GPU total viewshed (raw = 1: total_viewshed_raw): one
 * host thread per listed device runs its row block of every sector
 * (sks_context_run_rows_cuts) into a private FP64 map; ONE ncclReduce(sum,
 * f64) to devices[0] (NCCL loaded at run time) is the only exchange; then
 * scaling and the D2H copy. A list with repeated devices (ranks sharing a
 * GPU) reduces with peer adds instead of NCCL. The row-block cuts adapt to
 * measured per-GPU times over the first 3 calls per workload shape, then
 * stay fixed. Per-cell sums differ from one GPU only in order (<= 1e-12
 * relative; the reference bar is 1e-5). SKS_NCCL_ERROR when NCCL fails. */
sks_status sks_total_viewshed_devices(const float* dem, int dimy, int dimx, double cellsize,
                                      const sks_run_config* cfg, const int* devices, int n_devices,
                                      int raw, double* out, sks_stats* stats);
/* The device list a run config names (n_gpus, device); returns the count
 * (written up to cap). */
int sks_config_devices(const sks_run_config* cfg, int* devices, int cap);
/* One rebalancing step of the row-block cuts (nparts + 1 non-decreasing
 * fractions): given the per-part times measured with `cuts`, the cuts that
 * give every part an equal share when time is piecewise linear in the cost
 * fraction. Host only. */
void sks_row_cuts_update(const double* cuts, const double* times, int nparts, double* out);

/* sector_sweep, engine.cpp:235-244: one sector's unskewed contribution. */
sks_status sks_sector_sweep(const float* dem, int dimy, int dimx,
                            double cellsize, const sks_run_config* cfg, int k,
                            double* out_contribution);

/* ---- per-phase entry points (host buffers; parity and debugging) ---- */

/* apply_pre_ops + build_skw, skew.cpp:103-196, for sector k of ns:
 * values ((base+rows) x cols floats, every cell) and ranges (2*skw_rows). */
sks_status sks_build_sector_sdem(const float* dem, int dimy, int dimx, int k,
                                 int ns, int device, float* values,
                                 int* ranges);
/* build_skw, skew.cpp:144-196, on a grid already in pre_ops space. */
sks_status sks_build_skw(const float* g, int rows, int cols, double shear_tan,
                         int device, float* values, int* ranges,
                         int* base_out);
/* sector_viewshed, scan.cpp:64-85. out: skw_rows*cols doubles. cv_fwd and
 * cv_bwd (optional, skw_rows*cols ints) receive the per-direction ring sums.
 */
sks_status sks_sector_viewshed(const float* values, const int* ranges,
                               int skw_rows, int cols, double shear_tan,
                               double h0, int max_dd, int device, double* out,
                               int* cv_fwd, int* cv_bwd);
/* linear_viewshed_row, scan.cpp:8-62, evaluated by the GPU scan kernel for
 * one POV with absolute observer height h. visible_out (optional) receives
 * one byte per scanned target. */
sks_status sks_linear_viewshed_row(const float* row, int n, int first,
                                   int last, int j0, double h,
                                   int dir, int max_dd, int device,
                                   double* cv_out, uint8_t* visible_out,
                                   int* n_visible);
/* unskew_accumulate, skew.cpp:204-263: out (dimy*dimx) += unskewed skw_vs. */
sks_status sks_unskew_accumulate(const double* skw_vs, int skw_rows, int cols,
                                 int k, int ns, int dimy, int dimx, int device,
                                 double* out);

/* ---- device-resident context (one per GPU; sector sharding) ---------- */

typedef struct sks_context sks_context;

sks_status sks_context_create(int device, sks_context** out);
void sks_context_destroy(sks_context* ctx);
/* Runs sectors[0..n) (any order given; accumulated in ascending k) of the
 * total viewshed for the device-resident DEM d_dem and ADDS their raw
 * contributions into the device map d_map (dimy*dimx doubles), all on
 * `stream` (cudaStream_t). Asynchronous with respect to the host unless
 * stats is non-NULL (then it synchronises to read the phase events). */
sks_status sks_context_run_sectors(sks_context* ctx, const float* d_dem,
                                   int dimy, int dimx, double cellsize,
                                   const sks_run_config* cfg,
                                   const int* sectors, int n_sectors,
                                   double* d_map, void* stream,
                                   sks_stats* stats);
/* Row-block sharding: all ns/2 sectors, but only part
   `part` of `nparts` of every sector's skewed rows — contiguous blocks of
   equal exact scan work — accumulated into d_map. The nparts maps sum (e.g.
   one NCCL reduce) to the total raw map; per-cell summation order differs
   from the single-GPU order (relative differences ~1e-16). Replaces the
   sector pool of total_viewshed_raw (engine.cpp:109-220) across GPUs. */
sks_status sks_context_run_rows(sks_context* ctx, const float* d_dem, int dimy,
                                int dimx, double cellsize,
                                const sks_run_config* cfg, int part, int nparts,
                                double* d_map, void* stream, sks_stats* stats);
/* The same with the row blocks placed by cuts (nparts + 1 non-decreasing
   fractions of each sector's modelled cost, cuts[0] = 0, cuts[nparts] = 1;
   NULL = equal shares): measured-time rebalancing across GPUs
   (paper_2003_02200_b200/distributed.py RowBalancer). Every rank must pass
   the same cuts. */
sks_status sks_context_run_rows_cuts(sks_context* ctx, const float* d_dem, int dimy,
                                     int dimx, double cellsize, const sks_run_config* cfg,
                                     int part, int nparts, const double* cuts, double* d_map,
                                     void* stream, sks_stats* stats);

/* d_map[i] *= area_scale_factor(ns, cellsize, units) on `stream`. */
sks_status sks_context_scale(sks_context* ctx, double* d_map, long long n,
                             int ns, double cellsize, int units,
                             void* stream);
/* Total viewshed through the context with host buffers (the e2e path). */
sks_status sks_context_total_viewshed(sks_context* ctx, const float* dem,
                                      int dimy, int dimx, double cellsize,
                                      const sks_run_config* cfg, int raw,
                                      double* out, sks_stats* stats);

/* ---- ESRI ASCII grid I/O: the DEM load / map output entry points
   (ascii_grid.hpp:15-31). Host code; the body is parsed and written by all
   host threads. ---------------------------------------------------------- */
typedef struct {
  int nrows, ncols;
  double xllcorner, yllcorner, cellsize;
  int has_nodata; /* NODATA_value present */
  float nodata;
} sks_grid_header;

typedef struct sks_ascii_grid sks_ascii_grid;

/* read_ascii_grid(path) (ascii_grid.cpp:198-204): SKS_FORMAT_ERROR with the
   reference's "source:line:col: ..." message on bad input. */
sks_status sks_ascii_grid_read(const char* path, sks_ascii_grid** out);
/* read_ascii_grid(istream, source_name) (ascii_grid.cpp:110-196) on an
   in-memory text of len bytes. */
sks_status sks_ascii_grid_parse(const char* text, size_t len, const char* source_name,
                                sks_ascii_grid** out);
sks_status sks_ascii_grid_header(const sks_ascii_grid* grid, sks_grid_header* out);
/* copies the nrows*ncols cell values (float32, north row first) */
sks_status sks_ascii_grid_values(const sks_ascii_grid* grid, float* out);
void sks_ascii_grid_free(sks_ascii_grid* grid);

/* Binary side format for large DEMs (no reference counterpart; SURVEY §8f
   rank 3): ESRI float grid, `.hdr` text header + `.flt` float32 cells, north
   row first, LSBFIRST or MSBFIRST. path names either file. Same handle as
   the ASCII reader; SKS_FORMAT_ERROR on a bad header or a short/long file. */
sks_status sks_float_grid_read(const char* path, sks_ascii_grid** out);
sks_status sks_write_float_grid(const char* path, const float* values, const sks_grid_header* hdr);

/* write_ascii_grid(Dem, path) (ascii_grid.cpp:225-245); header fields from
   hdr (nodata written when has_nodata). */
sks_status sks_write_ascii_grid_dem(const char* path, const float* values,
                                    const sks_grid_header* hdr);
/* write_ascii_grid(VsGrid, out_units, cellsize, origin, path)
   (ascii_grid.cpp:247-272): values in units_in, written in units_out. */
sks_status sks_write_ascii_grid_vs(const char* path, const double* values, int nrows,
                                   int ncols, int units_in, int units_out,
                                   double cellsize, double xllcorner,
                                   double yllcorner);

/* ---- Rotational-sweep viewshed on the GPU: the reference's independent
   oracle (oracle.hpp:10-68) — rays rasterised per azimuth in unskewed grid
   space, Euclidean distances, no relocation. Bit-identical to oracle.cpp
   (the per-azimuth ray tables are computed on the host with the same glibc
   calls). max_distance: metres, 0 = unlimited. Areas in m^2. --------------- */
enum { SKS_REFERENCE_CELL_GUARD = 65536 }; /* kReferenceCellGuard (oracle.hpp:62) */

/* singular_viewshed(dem, i0, j0, h0, ns, max_distance) (oracle.cpp:108-129):
   SKS_OUT_OF_RANGE for an observer outside the grid, SKS_INVALID_ARGUMENT
   for a bad ns. */
sks_status sks_singular_viewshed(const float* dem, int dimy, int dimx, double cellsize, int i, int j,
                                 double h0, int ns, double max_distance, int device, double* area);

/* multi_viewshed(dem, povs, h0, ns, max_distance) (oracle.cpp:131-141):
   povs = npovs (i, j) pairs. Any of pov_area (npovs), grid (dimy*dimx,
   nonzero only at observers, summed in list order) and total_area may be
   null. */
sks_status sks_multi_viewshed(const float* dem, int dimy, int dimx, double cellsize, const int* povs,
                              int npovs, double h0, int ns, double max_distance, int device,
                              double* pov_area, double* grid, double* total_area);

/* total_viewshed_reference(dem, cfg, force) (oracle.cpp:143-194): the
   singular viewshed of every cell in cfg->units; grids above
   SKS_REFERENCE_CELL_GUARD cells are refused (SKS_INTERNAL, the reference's
   runtime_error) unless force. nodata may be null. */
sks_status sks_total_viewshed_reference(const float* dem, int dimy, int dimx, double cellsize,
                                        const float* nodata, const sks_run_config* cfg, int force,
                                        double* out);

/* linear_scan(dem, i0, j0, pov_h, azimuth, max_dist_cells, rings_out)
   (oracle.cpp:74-106) on the GPU: *cv, and the first min(cap, *nrings) ring
   sectors (r_open, r_close pairs, cell units) into rings (may be null).
   max_dist_cells: INFINITY for none. */
sks_status sks_linear_scan(const float* dem, int dimy, int dimx, int i0, int j0, double pov_h,
                           double azimuth_deg, double max_dist_cells, int device, double* cv,
                           double* rings, int cap, int* nrings);

/* select_axis_point_set (oracle.cpp:62-71): *count cells of the ray, the
   first min(cap, *count) written to ij as (i, j) pairs. Host only. */
sks_status sks_axis_point_set(int dimy, int dimx, int i0, int j0, double azimuth_deg, int* ij, int cap,
                              int* count);

/* random_povs(dem, count, seed) (cli.cpp:207-221): count (i, j) pairs. */
sks_status sks_random_povs(int dimy, int dimx, int count, uint32_t seed, int* ij);

/* fill_nodata_nearest(dem) (dem.cpp:175-213): out = dem with every nodata
   cell replaced by the value the reference's breadth-first search reaches it
   from (host). SKS_INTERNAL for a grid that is entirely nodata. */
sks_status sks_fill_nodata_nearest(const float* dem, int dimy, int dimx, float nodata, float* out);

/* write_heatmap(grid, path, palette) (heatmap.cpp:11-56): binary PGM / PPM of
   the min-max normalised map. Host code. */
enum { SKS_PALETTE_GRAY = 0, SKS_PALETTE_BLUE_RED = 1 };
sks_status sks_write_heatmap(const char* path, const double* values, int rows, int cols, int palette);

#ifdef __cplusplus
}
#endif

#endif /* SKEWSHED_B200_H */
