// In-process multi-GPU total viewshed behind the reference's entry point.
//
// The reference spreads one total_viewshed call over cfg.workers host threads
// (engine.cpp:109-220: a sector pool, per-sector contributions reduced in
// ascending k). Here one call spreads over GPUs: one host thread per GPU
// runs the row-block share `g` of every sector on its device
// (sks_context_run_rows_cuts: relocation -> scan -> fixup -> unskew into a
// private FP64 map), and ONE ncclReduce(sum, ncclFloat64) of the
// maps to the first GPU is the path's only exchange step; the first GPU then
// scales the map and copies it out. The orchestration is written against the
// library's own device-pointer C ABI.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy torch already
// mapped, else the system one), so single-GPU users never need it. Ranks
// that share a device (a device list with repeats: exercising the sharding
// on a smaller box) reduce by a peer add instead, since NCCL needs one rank
// per device.
//
// Row blocks are placed by cuts (fractions of every sector's modelled row
// cost). The first calls on a device list move the cuts from measured
// per-rank device times (time modelled as piecewise linear in the cost
// fraction, the new cuts give every rank an equal share) and then freeze
// them, so a repeated call is reproducible; sks_row_cuts_update is that step.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/skewshed_b200.h"

extern "C" void sks_set_last_error(const char* msg);  // engine.cu: the thread's sks_last_error()

namespace {

thread_local std::string g_multi_error;  // message of the last failure here

struct Failure {
  sks_status status = SKS_OK;
  std::string message;
};

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Failure{SKS_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e)};
}

// ---- NCCL, loaded on first use --------------------------------------------
struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static const Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) {
      r.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return r;
    }
    r.comm_init_all = reinterpret_cast<decltype(r.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
    r.comm_destroy = reinterpret_cast<decltype(r.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    r.reduce = reinterpret_cast<decltype(r.reduce)>(dlsym(h, "ncclReduce"));
    r.group_start = reinterpret_cast<decltype(r.group_start)>(dlsym(h, "ncclGroupStart"));
    r.group_end = reinterpret_cast<decltype(r.group_end)>(dlsym(h, "ncclGroupEnd"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(dlsym(h, "ncclGetErrorString"));
    r.ok = r.comm_init_all && r.comm_destroy && r.reduce && r.group_start && r.group_end && r.error_string;
    if (!r.ok) r.why = "libnccl.so.2 lacks a required symbol";
    return r;
  }();
  return n;
}

void nccl_ok(ncclResult_t e, const char* what) {
  if (e != ncclSuccess) throw Failure{SKS_NCCL_ERROR, std::string(what) + ": " + nccl().error_string(e)};
}

// map[i] += part[i] on `stream` (multi_add.cu)
extern "C" cudaError_t sks_launch_add_map(double* map, const double* part, long long n, cudaStream_t stream);

// ---- per-device-list state, cached across calls ------------------------------
struct Rank {
  int device = 0;
  sks_context* ctx = nullptr;
  cudaStream_t stream = nullptr;
  float* dem = nullptr;
  double* map = nullptr;
  size_t cells = 0;
};

struct Multi {
  std::mutex mu;
  std::vector<Rank> ranks;
  bool use_nccl = false;
  std::vector<ncclComm_t> comms;
  double* scratch = nullptr;  // root-device buffer for peer adds across devices
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // row-block cuts per workload shape (dimy, dimx, ns, cellsize,
  // max_distance), adapted over the first calls
  struct Cuts {
    std::vector<double> c;
    int updates = 0;
  };
  std::map<std::vector<double>, Cuts> cuts;

  ~Multi() {
    for (Rank& r : ranks) {
      cudaSetDevice(r.device);
      if (r.dem) cudaFree(r.dem);
      if (r.map) cudaFree(r.map);
      if (r.stream) cudaStreamDestroy(r.stream);
      if (r.ctx) sks_context_destroy(r.ctx);
    }
    if (!ranks.empty()) cudaSetDevice(ranks[0].device);
    if (scratch) cudaFree(scratch);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    for (ncclComm_t c : comms) nccl().comm_destroy(c);
  }
};

std::mutex g_multi_mu;
std::map<std::vector<int>, std::unique_ptr<Multi>> g_multi;

constexpr int kAdaptCalls = 3;  // calls whose measured times move the cuts

bool force_nccl() {
  const char* s = std::getenv("SKS_NCCL");
  return s != nullptr && std::atoi(s) != 0;
}

Multi& multi_for(const std::vector<int>& devices) {
  std::lock_guard<std::mutex> lk(g_multi_mu);
  auto it = g_multi.find(devices);
  if (it != g_multi.end()) return *it->second;
  auto m = std::make_unique<Multi>();
  std::vector<int> sorted = devices;
  std::sort(sorted.begin(), sorted.end());
  const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
  m->use_nccl = distinct && (devices.size() > 1 || force_nccl());
  if (m->use_nccl && !nccl().ok) {
    if (force_nccl()) throw Failure{SKS_NCCL_ERROR, nccl().why};
    m->use_nccl = false;  // peer adds instead
  }
  for (int d : devices) {
    Rank r;
    r.device = d;
    if (sks_context_create(d, &r.ctx) != SKS_OK) throw Failure{SKS_CUDA_ERROR, sks_last_error()};
    cuda_ok(cudaSetDevice(d), "cudaSetDevice");
    cuda_ok(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking), "stream");
    m->ranks.push_back(r);
  }
  cuda_ok(cudaSetDevice(devices[0]), "cudaSetDevice");
  cuda_ok(cudaEventCreate(&m->ev0), "event");
  cuda_ok(cudaEventCreate(&m->ev1), "event");
  if (m->use_nccl) {
    m->comms.resize(devices.size());
    nccl_ok(nccl().comm_init_all(m->comms.data(), static_cast<int>(devices.size()), devices.data()),
            "ncclCommInitAll");
  }
  Multi& ref = *m;
  g_multi.emplace(devices, std::move(m));
  return ref;
}

// One rank: DEM upload, map clear, its row block of every sector (async on
// the rank's stream; the stats read synchronises at the end of each batch).
void run_rank(Rank& r, const float* dem, int dimy, int dimx, double cellsize, const sks_run_config* cfg, int part,
              int nparts, const double* cuts, sks_stats* st) {
  const size_t n = static_cast<size_t>(dimy) * dimx;
  cuda_ok(cudaSetDevice(r.device), "cudaSetDevice");
  if (r.cells < n) {
    if (r.dem) cudaFree(r.dem);
    if (r.map) cudaFree(r.map);
    r.dem = nullptr;
    r.map = nullptr;
    r.cells = 0;
    cuda_ok(cudaMalloc(&r.dem, n * sizeof(float)), "cudaMalloc dem");
    cuda_ok(cudaMalloc(&r.map, n * sizeof(double)), "cudaMalloc map");
    r.cells = n;
  }
  cuda_ok(cudaMemcpyAsync(r.dem, dem, n * sizeof(float), cudaMemcpyHostToDevice, r.stream), "H2D dem");
  cuda_ok(cudaMemsetAsync(r.map, 0, n * sizeof(double), r.stream), "memset map");
  const sks_status s = sks_context_run_rows_cuts(r.ctx, r.dem, dimy, dimx, cellsize, cfg, part, nparts, cuts, r.map,
                                                 r.stream, st);
  if (s != SKS_OK) throw Failure{s, sks_last_error()};
}

void total_multi(const float* dem, int dimy, int dimx, double cellsize, const sks_run_config* cfg,
                 const std::vector<int>& devices, int raw, double* out, sks_stats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  if (!dem || !cfg || !out) throw Failure{SKS_INVALID_ARGUMENT, "null argument"};
  if (devices.empty()) throw Failure{SKS_INVALID_ARGUMENT, "empty device list"};
  int visible = 0;
  if (cudaGetDeviceCount(&visible) != cudaSuccess) {
    cudaGetLastError();
    visible = 0;
  }
  for (int d : devices) {
    if (d < 0 || d >= visible) {
      std::ostringstream os;
      os << "CUDA device " << d << " requested but " << visible << " visible";
      throw Failure{visible == 0 ? SKS_CUDA_ERROR : SKS_INVALID_ARGUMENT, os.str()};
    }
  }
  Multi& m = multi_for(devices);
  std::lock_guard<std::mutex> lk(m.mu);
  const int G = static_cast<int>(devices.size());
  const size_t n = static_cast<size_t>(dimy) * dimx;
  auto& cuts = m.cuts[std::vector<double>{static_cast<double>(dimy), static_cast<double>(dimx),
                                          static_cast<double>(cfg->ns), cellsize, cfg->max_distance}];
  if (static_cast<int>(cuts.c.size()) != G + 1) {
    cuts.c.resize(G + 1);
    for (int b = 0; b <= G; ++b) cuts.c[b] = static_cast<double>(b) / G;
    cuts.updates = 0;
  }
  const bool adapt = G > 1 && cuts.updates < kAdaptCalls;
  std::vector<sks_stats> st(G);
  std::vector<Failure> fail(G);
  {
    std::vector<std::thread> pool;
    for (int g = 0; g < G; ++g) {
      pool.emplace_back([&, g] {
        try {
          run_rank(m.ranks[g], dem, dimy, dimx, cellsize, cfg, g, G, G > 1 ? cuts.c.data() : nullptr,
                   (stats || adapt) ? &st[g] : nullptr);
        } catch (const Failure& f) {
          fail[g] = f;
        }
      });
    }
    for (std::thread& t : pool) t.join();
  }
  for (const Failure& f : fail) {  // the first failing rank's error, as the reference rethrows one
    if (f.status != SKS_OK) throw f;
  }
  Rank& root = m.ranks[0];
  cuda_ok(cudaSetDevice(root.device), "cudaSetDevice");
  cuda_ok(cudaEventRecord(m.ev0, root.stream), "event");
  if (G > 1 || m.use_nccl) {
    if (m.use_nccl) {
      // one grouped reduce: every rank's map summed into the root's, in place
      nccl_ok(nccl().group_start(), "ncclGroupStart");
      for (int g = 0; g < G; ++g) {
        const Rank& r = m.ranks[g];
        nccl_ok(nccl().reduce(r.map, r.map, n, ncclFloat64, ncclSum, 0, m.comms[g], r.stream), "ncclReduce");
      }
      nccl_ok(nccl().group_end(), "ncclGroupEnd");
    } else {
      // ranks sharing devices: peer adds on the root stream, in rank order
      for (int g = 1; g < G; ++g) {
        const Rank& r = m.ranks[g];
        const double* part = r.map;
        if (r.device != root.device) {
          if (m.scratch == nullptr) cuda_ok(cudaMalloc(&m.scratch, root.cells * sizeof(double)), "cudaMalloc");
          cuda_ok(cudaStreamSynchronize(r.stream), "sync rank");
          cuda_ok(cudaMemcpyPeerAsync(m.scratch, root.device, r.map, r.device, n * sizeof(double), root.stream),
                  "peer copy");
          part = m.scratch;
        } else {
          cudaEvent_t e;
          cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
          cuda_ok(cudaEventRecord(e, r.stream), "event");
          cuda_ok(cudaStreamWaitEvent(root.stream, e, 0), "wait");
          cudaEventDestroy(e);
        }
        cuda_ok(sks_launch_add_map(root.map, part, static_cast<long long>(n), root.stream), "launch add");
      }
    }
  }
  if (!raw) {
    const sks_status s = sks_context_scale(root.ctx, root.map, static_cast<long long>(n), cfg->ns, cellsize,
                                           cfg->units, root.stream);
    if (s != SKS_OK) throw Failure{s, sks_last_error()};
  }
  cuda_ok(cudaEventRecord(m.ev1, root.stream), "event");
  cuda_ok(cudaMemcpyAsync(out, root.map, n * sizeof(double), cudaMemcpyDeviceToHost, root.stream), "D2H map");
  cuda_ok(cudaStreamSynchronize(root.stream), "sync");
  float reduce_ms = 0.f;
  cuda_ok(cudaEventElapsedTime(&reduce_ms, m.ev0, m.ev1), "event time");
  if (adapt) {  // move the cuts from the ranks' measured device times
    std::vector<double> t(G);
    for (int g = 0; g < G; ++g) {
      t[g] = st[g].skew_seconds + st[g].scan_seconds + st[g].fixup_seconds + st[g].unskew_seconds;
    }
    std::vector<double> next(G + 1);
    sks_row_cuts_update(cuts.c.data(), t.data(), G, next.data());
    cuts.c = next;
    ++cuts.updates;
  }
  if (stats) {
    sks_stats total{};
    for (const sks_stats& s : st) {  // device seconds summed over GPUs, as the
      total.skew_seconds += s.skew_seconds;  // reference sums worker seconds
      total.scan_seconds += s.scan_seconds;
      total.fixup_seconds += s.fixup_seconds;
      total.unskew_seconds += s.unskew_seconds;
      total.kernel_launches += s.kernel_launches;
      total.target_evals += s.target_evals;
      total.flagged_groups += s.flagged_groups;
      total.skipped_target_slots += s.skipped_target_slots;
      total.scan_kernel = s.scan_kernel;
      total.batches += s.batches;
    }
    total.sectors = cfg->ns / 2;
    total.reduce_seconds = reduce_ms * 1e-3;
    total.kernel_launches += (G > 1 && !m.use_nccl ? G - 1 : 0) + (raw ? 0 : 1);
    total.h2d_bytes = static_cast<long long>(n * sizeof(float)) * G;
    total.d2h_bytes = static_cast<long long>(n * sizeof(double));
    total.total_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *stats = total;
  }
}

template <typename Fn>
sks_status multi_guarded(Fn&& fn) {
  try {
    fn();
    g_multi_error.clear();
    return SKS_OK;
  } catch (const Failure& f) {
    g_multi_error = f.message;
    return f.status;
  } catch (const std::exception& e) {
    g_multi_error = e.what();
    return SKS_INTERNAL;
  }
}

}  // namespace

extern "C" {

// The devices a run config names: n_gpus <= 1 -> {device}; n_gpus > 1 ->
// device .. device + n_gpus - 1; SKS_ALL_GPUS -> every visible device from
// `device` on (at least one).
int sks_config_devices(const sks_run_config* cfg, int* devices, int cap) {
  if (cfg == nullptr) return 0;
  int visible = 0;
  if (cudaGetDeviceCount(&visible) != cudaSuccess) {
    cudaGetLastError();
    visible = 0;
  }
  int n = cfg->n_gpus <= 1 && cfg->n_gpus != SKS_ALL_GPUS ? 1 : cfg->n_gpus;
  if (cfg->n_gpus == SKS_ALL_GPUS) n = std::max(1, visible - cfg->device);
  for (int g = 0; g < n && g < cap; ++g) devices[g] = cfg->device + g;
  return n;
}

sks_status sks_total_viewshed_devices(const float* dem, int dimy, int dimx, double cellsize,
                                      const sks_run_config* cfg, const int* devices, int n_devices, int raw,
                                      double* out, sks_stats* stats) {
  const sks_status s = multi_guarded([&] {
    if (n_devices < 1 || devices == nullptr) throw Failure{SKS_INVALID_ARGUMENT, "device list must not be empty"};
    total_multi(dem, dimy, dimx, cellsize, cfg, std::vector<int>(devices, devices + n_devices), raw, out, stats);
  });
  if (s != SKS_OK) sks_set_last_error(g_multi_error.c_str());
  return s;
}

void sks_row_cuts_update(const double* cuts, const double* times, int nparts, double* out) {
  // time is piecewise linear in the cost fraction: density t[r] / (c[r+1] -
  // c[r]) on block r; block b of the new cuts starts where the cumulative
  // time reaches b/nparts of the total
  std::vector<double> T(nparts + 1, 0.0);
  bool valid = nparts >= 1;
  for (int r = 0; r < nparts && valid; ++r) {
    valid = times[r] >= 0.0 && times[r] < 1e300;
    T[r + 1] = T[r] + times[r];
  }
  if (!valid || !(T[nparts] > 0.0)) {
    std::copy(cuts, cuts + nparts + 1, out);
    return;
  }
  out[0] = 0.0;
  for (int b = 1; b < nparts; ++b) {
    const double target = b * T[nparts] / nparts;
    int r = static_cast<int>(std::upper_bound(T.begin(), T.end(), target) - T.begin()) - 1;
    r = std::min(std::max(r, 0), nparts - 1);
    const double frac = times[r] > 0.0 ? (target - T[r]) / times[r] : 0.0;
    out[b] = cuts[r] + std::min(std::max(frac, 0.0), 1.0) * (cuts[r + 1] - cuts[r]);
  }
  out[nparts] = 1.0;
  for (int b = 0; b <= nparts; ++b) {  // clip to [0, 1], non-decreasing
    out[b] = std::min(std::max(out[b], 0.0), 1.0);
    if (b > 0) out[b] = std::max(out[b], out[b - 1]);
  }
}

}  // extern "C"
