// life_gpu.hpp -- C++ host mirror of the reference's step-loop API over the
// C-ABI of include/life_gpu.h (header only, C++20).
//
// Mirrors /root/reference/proj/core/include/life/engine.hpp:11-43:
//     RunResult run(Grid&& initial, const RunConfig&, const std::vector<int>& checkpoints);
//     Grid step_parallel(const Grid&, const Strategy&, int workers);
// and the exception hierarchy of errors.hpp:9-60.  The functions are
// templates over the grid type: any type with `width()`, `height()`,
// `data()` (uint8_t*, row-major, W*H bytes) and a `(width, height)`
// constructor works -- including the reference's own `life::Grid`
// (grid.hpp:24-70), which is what makes this a drop-in for its `run()`
// (see INTEGRATION.md).  Populations are uint64 (grid.cpp:40-46's int
// overflows above 2^31-1).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "life_gpu.h"

namespace lifegpu {

// errors.hpp:9-60
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ConfigError : public Error {
 public:
  using Error::Error;
};
class DimensionTooSmall : public ConfigError {
 public:
  using ConfigError::ConfigError;
};
class TooManyParts : public ConfigError {
 public:
  using ConfigError::ConfigError;
};
class OutOfBounds : public ConfigError {
 public:
  using ConfigError::ConfigError;
};
class CudaError : public Error {
 public:
  using Error::Error;
};

inline void check(int rc) {
  if (rc == LIFE_OK) return;
  const std::string msg = life_last_error();
  switch (rc) {
    case LIFE_ERR_CONFIG: throw ConfigError(msg);
    case LIFE_ERR_DIMENSION_TOO_SMALL: throw DimensionTooSmall(msg);
    case LIFE_ERR_TOO_MANY_PARTS: throw TooManyParts(msg);
    case LIFE_ERR_OUT_OF_BOUNDS: throw OutOfBounds(msg);
    case LIFE_ERR_CUDA:
    case LIFE_ERR_NO_DEVICE:
    case LIFE_ERR_OUT_OF_MEMORY: throw CudaError(msg);
    default: throw Error(msg);
  }
}

enum class Engine { Packed = LIFE_ENGINE_PACKED, Byte = LIFE_ENGINE_BYTE, Resident = LIFE_ENGINE_RESIDENT };

// RunConfig (engine.hpp:11-15) with the GPU strategy fields.
struct RunConfig {
  Engine engine = Engine::Packed;
  // Generations per kernel pass; 0 = auto: the cluster-resident engine for
  // small W % 32 == 0 tori (<= 2^22 cells, one GPU); tori of 2^29 cells or
  // more in the quad layout at 7 / 6 (W % 128 == 0, wide), of 2^27 or more in
  // the pair layout at 10 (W % 64 == 0) (life_interleave_auto); else 16 -- 12 for W % 32 != 0 tori
  // less than ~3 block waves deep (life_packed_auto_depth).
  int temporal_depth = 0;
  int workers = 1;  // validated like the reference (>= 1, <= rows)
  int64_t iterations = 0;
  int device = 0;
  // Row bands over several GPUs (life_ctx_create_multi, band_bounds of
  // decomposition.cpp:12-24): one band per entry, ids may repeat.  Empty =
  // the single GPU `device`.  The packed engine only.
  std::vector<int> devices;
};

// RunStats (engine.hpp:17-22) with uint64 populations.
struct RunStats {
  int64_t generations_computed = 0;
  std::vector<std::pair<int64_t, uint64_t>> population_checkpoints;
};

template <class GridT>
struct RunResult {
  GridT grid;
  RunStats stats;
};

// One C-ABI context: a grid resident on one GPU.
class Context {
 public:
  explicit Context(int device = 0) { check(life_ctx_create(device, &ctx_)); }
  // Row bands over `devices` (repeats allowed).
  explicit Context(const std::vector<int>& devices) {
    check(life_ctx_create_multi(static_cast<int32_t>(devices.size()), devices.data(), &ctx_));
  }
  ~Context() { life_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  template <class GridT>
  void upload(const GridT& g) {
    check(life_grid_upload_u8(ctx_, g.data(), g.width(), g.height(), g.width()));
  }
  void init_random(int64_t w, int64_t h, double density, uint64_t seed,
                   Engine e = Engine::Packed) {
    check(life_grid_init_random(ctx_, w, h, density, seed, static_cast<int>(e)));
  }
  template <class GridT>
  void download(GridT& g) {
    check(life_grid_download_u8(ctx_, g.data(), g.width()));
  }
  std::vector<uint64_t> run(int64_t generations, Engine e, int depth,
                            const std::vector<int64_t>& checkpoints) {
    std::vector<uint64_t> pops(checkpoints.size());
    check(life_run(ctx_, generations, static_cast<int>(e), depth,
                   checkpoints.empty() ? nullptr : checkpoints.data(),
                   static_cast<int32_t>(checkpoints.size()), pops.empty() ? nullptr : pops.data()));
    return pops;
  }
  uint64_t population() {
    uint64_t p = 0;
    check(life_population(ctx_, &p));
    return p;
  }
  // Full-grid checksum (life_grid_hash) for grids too big to download.
  uint64_t hash() {
    uint64_t h = 0;
    check(life_grid_hash(ctx_, &h));
    return h;
  }
  std::vector<uint8_t> window(int64_t x0, int64_t y0, int64_t w, int64_t h) {
    std::vector<uint8_t> out(static_cast<size_t>(w * h));
    check(life_grid_window_u8(ctx_, x0, y0, w, h, out.data()));
    return out;
  }
  std::vector<life_band_stats> band_stats() {
    int32_t n = 0;
    check(life_ctx_bands(ctx_, &n, nullptr, nullptr, nullptr));
    std::vector<life_band_stats> out(static_cast<size_t>(n));
    for (int32_t i = 0; i < n; ++i) check(life_ctx_band_stats(ctx_, i, &out[i]));
    return out;
  }
  life_ctx* handle() const { return ctx_; }

 private:
  life_ctx* ctx_ = nullptr;
};

// One cached context per host thread and device set: a drop-in run() call
// reuses its device buffers instead of creating a context and allocating
// two grid buffers every time (contexts are single-thread objects, hence
// thread_local).  release_cached_contexts() frees this thread's.
inline std::map<std::vector<int>, std::unique_ptr<Context>>& cached_contexts() {
  thread_local std::map<std::vector<int>, std::unique_ptr<Context>> cache;
  return cache;
}
inline Context& cached_context(const RunConfig& cfg) {
  const std::vector<int> key = cfg.devices.empty() ? std::vector<int>{cfg.device} : cfg.devices;
  auto& cache = cached_contexts();
  auto it = cache.find(key);
  if (it == cache.end()) {
    std::unique_ptr<Context> c = cfg.devices.empty() ? std::make_unique<Context>(cfg.device)
                                                     : std::make_unique<Context>(cfg.devices);
    it = cache.emplace(key, std::move(c)).first;
  }
  return *it->second;
}
inline void release_cached_contexts() { cached_contexts().clear(); }

// run (engine.cpp:157-214): check_run_config's rules (:127-148) and
// partition_rows' TooManyParts (decomposition.cpp:26-30) on `workers`, then
// `iterations` generations on the GPU; checkpoint 0 is the initial grid.
// Takes the grid by value: an rvalue moves in (the reference's Grid&&
// overload), an lvalue is copied (its const Grid& overload, engine.cpp:157-160).
template <class GridT>
RunResult<GridT> run(GridT initial, const RunConfig& cfg,
                     const std::vector<int64_t>& checkpoints = {}) {
  if (cfg.workers < 1)
    throw ConfigError("worker count must be at least 1, got " + std::to_string(cfg.workers));
  if (cfg.workers > initial.height())
    throw TooManyParts("cannot split " + std::to_string(initial.height()) + " rows into " +
                       std::to_string(cfg.workers) + " non-empty parts");
  if (cfg.iterations < 0)
    throw ConfigError("iteration count must be non-negative, got " +
                      std::to_string(cfg.iterations));
  int64_t prev = -1;
  for (int64_t cp : checkpoints) {
    if (cp < 0 || cp > cfg.iterations)
      throw ConfigError("checkpoint " + std::to_string(cp) + " is outside [0, iterations=" +
                        std::to_string(cfg.iterations) + "]");
    if (cp <= prev) throw ConfigError("checkpoints must be strictly ascending");
    prev = cp;
  }
  Context& ctx = cached_context(cfg);
  ctx.upload(initial);
  const std::vector<uint64_t> pops = ctx.run(cfg.iterations, cfg.engine, cfg.temporal_depth, checkpoints);
  ctx.download(initial);
  RunStats stats;
  stats.generations_computed = cfg.iterations;
  for (size_t i = 0; i < checkpoints.size(); ++i)
    stats.population_checkpoints.emplace_back(checkpoints[i], pops[i]);
  return RunResult<GridT>{std::move(initial), std::move(stats)};
}

// run() for a grid held in the packed exchange format (rows of
// words_per_row >= ceil(W/64) uint64, bit j of word k = column 64k+j): grids
// too big for host bytes (config 5 is 64 GiB as bytes, 8 GiB packed).
// One life_run_batch call with n = 1 on the cached context: the grid's upload
// and download overlap its first and last passes (row-chunk trapezoids), so a
// one-shot call on host memory runs near the device rate (config 5: 0.775 s vs
// 1.05 s for upload + run + download in sequence).  `in` and `out` may alias;
// use pinned memory for the overlap.  Packed engine, one device.
inline void run_packed(const uint64_t* in, uint64_t* out, int64_t width, int64_t height,
                       int64_t words_per_row, const RunConfig& cfg) {
  if (cfg.iterations < 0)
    throw ConfigError("iteration count must be non-negative, got " +
                      std::to_string(cfg.iterations));
  if (cfg.devices.size() > 1) throw ConfigError("run_packed runs on one device");
  RunConfig one = cfg;
  if (one.devices.size() == 1) one.device = one.devices[0];
  one.devices.clear();
  Context& ctx = cached_context(one);
  const uint64_t* ins[1] = {in};
  uint64_t* outs[1] = {out};
  check(life_run_batch(ctx.handle(), ins, outs, 1, width, height, words_per_row, cfg.iterations,
                       cfg.temporal_depth, nullptr));
}

// step_parallel (engine.cpp:152-155).
template <class GridT>
GridT step_parallel(const GridT& grid, RunConfig cfg) {
  cfg.iterations = 1;
  return run(grid, cfg).grid;
}

// random_fill (pattern.cpp:330-342), generated on the device.
template <class GridT>
GridT random_fill(int width, int height, double density, uint64_t seed, int device = 0) {
  GridT g(width, height);
  Context ctx(device);
  ctx.init_random(width, height, density, seed, Engine::Byte);
  ctx.download(g);
  return g;
}

}  // namespace lifegpu
