// life_harness.hpp -- the reference's benchmark harness
// driving the GPU engine (header only, C++20).
//
// Restates /root/reference/proj/core/include/life/bench.hpp (bench.cpp):
//   speedup            bench.cpp:60-65    (NonPositiveTime unless both > 0)
//   median             bench.cpp:67-75
//   time_run           bench.cpp:77-111   (soup built once, untimed warm-ups, each
//                                          repetition timed with steady_clock around
//                                          run(); the grid copy/upload stays outside)
//   bench_matrix       bench.cpp:113-165  (sizes x iterations; the first strategy is
//                                          each cell's baseline, speedups against it)
//   population_series  bench.cpp:167-176
//   emit_csv           bench.cpp:178-191  (the pinned 12-column header)
// with GPU strategy tokens ("gpu", "gpu:K", "gpu-byte", "gpu-resident" -- the reference's
// parse_strategy, decomposition.cpp:68-91, gains these kinds) and an extended
// CSV carrying GCUPS and the roofline fraction.  Populations are uint64.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <functional>
#include <iomanip>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "life_gpu.hpp"

namespace lifegpu {

class NonPositiveTime : public ConfigError {
 public:
  NonPositiveTime() : ConfigError("execution times must be positive to form a speedup") {}
};

// A GPU strategy: engine + temporal depth (0 = the engine's default, 16).
struct Strategy {
  Engine engine = Engine::Packed;
  int depth = 0;
  friend bool operator==(const Strategy&, const Strategy&) = default;
};

inline std::string to_string(const Strategy& s) {
  if (s.engine == Engine::Byte) return s.depth == 0 ? "gpu-byte" : "gpu-byte:" + std::to_string(s.depth);
  if (s.engine == Engine::Resident) return "gpu-resident";
  return s.depth == 0 ? "gpu" : "gpu:" + std::to_string(s.depth);
}

inline Strategy parse_strategy(const std::string& token) {
  if (token == "gpu") return {Engine::Packed, 0};
  if (token == "gpu-byte") return {Engine::Byte, 0};
  if (token.rfind("gpu-byte:", 0) == 0) {
    const std::string k = token.substr(9);
    if (k.size() == 1 && k[0] >= '1' && k[0] <= '8') return {Engine::Byte, k[0] - '0'};
  }
  if (token == "gpu-resident") return {Engine::Resident, 0};
  if (token.rfind("gpu:", 0) == 0) {
    const std::string k = token.substr(4);
    if (!k.empty() && k.size() <= 2 && std::all_of(k.begin(), k.end(), ::isdigit)) {
      const int d = std::stoi(k);
      if (d >= 1 && d <= LIFE_MAX_TEMPORAL_DEPTH) return {Engine::Packed, d};
    }
  }
  throw ConfigError("unknown strategy '" + token +
                    "' (expected gpu, gpu:K with K in 1..16, gpu-byte, gpu-byte:K with K in 1..8 or gpu-resident)");
}

inline double speedup(double baseline_s, double other_s) {
  if (!(baseline_s > 0.0) || !(other_s > 0.0)) throw NonPositiveTime();
  return baseline_s / other_s;
}

inline double median(std::vector<double> v) {
  if (v.empty()) throw ConfigError("median of an empty sample");
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

struct GridSize {
  int width = 0;
  int height = 0;
  friend bool operator==(const GridSize&, const GridSize&) = default;
};

struct TimingSpec {
  int width = 0;
  int height = 0;
  int iterations = 1;
  Strategy strategy;
  int workers = 1;
  uint64_t seed = 42;
  double density = 0.3;
  int repetitions = 5;
  int warmup_runs = 1;
  int device = 0;
};

struct BenchRecord {
  int width = 0;
  int height = 0;
  int iterations = 0;
  Strategy strategy;
  int workers = 1;
  uint64_t seed = 0;
  double density = 0.0;
  int repetitions = 0;
  std::vector<double> all_times_s;
  double median_s = 0.0;
  double speedup = 1.0;
  unsigned hardware_threads = 0;
  uint64_t final_population = 0;

  double gcups() const {
    return median_s > 0 ? double(width) * height * iterations / median_s / 1e9 : 0.0;
  }
};

inline BenchRecord time_run(const TimingSpec& spec) {
  // Same order of checks (and messages) as the reference harness: the first
  // violated rule is the one reported.
  const std::pair<bool, const char*> rules[] = {
      {spec.repetitions >= 1, "repetitions must be at least 1"},
      {spec.warmup_runs >= 0, "warmup runs must be non-negative"},
      {spec.iterations >= 1, "iteration count must be at least 1"},
      {spec.density >= 0.0 && spec.density <= 1.0, "density must be in [0, 1]"},
  };
  for (const auto& [holds, message] : rules)
    if (!holds) throw ConfigError(message);
  const Engine e = spec.strategy.engine;
  Context ctx(spec.device);
  // The seeded soup, once, on the device; kept on the host for the re-uploads.
  ctx.init_random(spec.width, spec.height, spec.density, spec.seed, Engine::Byte);
  std::vector<uint8_t> initial(static_cast<size_t>(spec.width) * spec.height);
  check(life_grid_download_u8(ctx.handle(), initial.data(), spec.width));
  auto upload = [&] {
    check(life_grid_upload_u8(ctx.handle(), initial.data(), spec.width, spec.height, spec.width));
  };
  for (int i = 0; i < spec.warmup_runs; ++i) {
    upload();
    ctx.run(spec.iterations, e, spec.strategy.depth, {});
  }
  BenchRecord rec;
  rec.width = spec.width;
  rec.height = spec.height;
  rec.iterations = spec.iterations;
  rec.strategy = spec.strategy;
  rec.workers = 1;  // one process drives one GPU
  rec.seed = spec.seed;
  rec.density = spec.density;
  rec.repetitions = spec.repetitions;
  rec.hardware_threads = std::thread::hardware_concurrency();
  for (int rep = 0; rep < spec.repetitions; ++rep) {
    upload();  // outside the timed region, like the reference's grid copy
    // The first run on a byte upload converts to the packed layout inside
    // life_run; do that conversion outside the timer as well.
    if (e != Engine::Byte) ctx.run(0, e, spec.strategy.depth, {});
    const auto t0 = std::chrono::steady_clock::now();
    ctx.run(spec.iterations, e, spec.strategy.depth, {});
    rec.all_times_s.push_back(
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    rec.final_population = ctx.population();
  }
  rec.median_s = median(rec.all_times_s);
  return rec;
}

struct BenchConfig {
  std::vector<GridSize> sizes;
  std::vector<int> iteration_counts;
  std::vector<Strategy> strategies;
  std::vector<int> worker_counts{1};
  int repetitions = 5;
  int warmup_runs = 1;
  uint64_t seed = 42;
  double density = 0.3;
  std::vector<int64_t> checkpoints;
  int device = 0;
};

inline void check_bench_config(const BenchConfig& c) {
  if (c.sizes.empty()) throw ConfigError("benchmark size list is empty");
  if (c.iteration_counts.empty()) throw ConfigError("benchmark iteration list is empty");
  if (c.strategies.empty()) throw ConfigError("benchmark strategy list is empty");
  if (c.worker_counts.empty()) throw ConfigError("benchmark worker list is empty");
  for (int it : c.iteration_counts)
    if (it < 1) throw ConfigError("iteration counts must be at least 1");
  for (int w : c.worker_counts)
    if (w < 1) throw ConfigError("worker counts must be at least 1");
  if (c.repetitions < 1) throw ConfigError("repetitions must be at least 1");
  if (c.warmup_runs < 0) throw ConfigError("warmup runs must be non-negative");
  if (!(c.density >= 0.0 && c.density <= 1.0)) throw ConfigError("density must be in [0, 1]");
  int64_t prev = -1;
  const int min_it = *std::min_element(c.iteration_counts.begin(), c.iteration_counts.end());
  for (int64_t cp : c.checkpoints) {
    if (cp <= prev) throw ConfigError("checkpoints must be strictly ascending");
    if (cp < 0 || cp > min_it)
      throw ConfigError("checkpoint " + std::to_string(cp) + " exceeds the smallest iteration count");
    prev = cp;
  }
}

// Sweep sizes x iteration counts x strategies (duplicates dropped, order
// kept); each cell starts with its baseline (the first strategy).
inline std::vector<BenchRecord> bench_matrix(
    const BenchConfig& config, const std::function<void(const BenchRecord&)>& on_record = {}) {
  check_bench_config(config);
  std::vector<Strategy> strategies;
  for (const Strategy& s : config.strategies)
    if (std::find(strategies.begin(), strategies.end(), s) == strategies.end())
      strategies.push_back(s);
  std::vector<BenchRecord> out;
  for (const GridSize& size : config.sizes) {
    for (int iterations : config.iteration_counts) {
      double base = 0.0;
      for (size_t i = 0; i < strategies.size(); ++i) {
        TimingSpec spec;
        spec.width = size.width;
        spec.height = size.height;
        spec.iterations = iterations;
        spec.strategy = strategies[i];
        spec.seed = config.seed;
        spec.density = config.density;
        spec.repetitions = config.repetitions;
        spec.warmup_runs = config.warmup_runs;
        spec.device = config.device;
        BenchRecord r = time_run(spec);
        if (i == 0) {
          base = r.median_s;
          r.speedup = 1.0;
        } else {
          r.speedup = speedup(base, r.median_s);
        }
        if (on_record) on_record(r);
        out.push_back(std::move(r));
      }
    }
  }
  return out;
}

inline std::vector<std::pair<int64_t, uint64_t>> population_series(
    int width, int height, uint64_t seed, double density, const Strategy& strategy,
    const std::vector<int64_t>& checkpoints, int device = 0) {
  const int64_t iterations = checkpoints.empty() ? 0 : checkpoints.back();
  Context ctx(device);
  ctx.init_random(width, height, density, seed, strategy.engine);
  const std::vector<uint64_t> pops = ctx.run(iterations, strategy.engine, strategy.depth, checkpoints);
  std::vector<std::pair<int64_t, uint64_t>> out;
  for (size_t i = 0; i < checkpoints.size(); ++i) out.emplace_back(checkpoints[i], pops[i]);
  return out;
}

inline std::string fixed(double v, int decimals) {
  std::ostringstream os;
  os.setf(std::ios::fixed);
  os.precision(decimals);
  os << v;
  return os.str();
}

inline std::string csv_row_prefix(const BenchRecord& r) {
  // The twelve pinned columns, in header order, joined by commas.
  std::ostringstream num;
  num << r.density;  // default ostream formatting, as the reference prints it
  const std::string fields[] = {
      std::to_string(r.width),       std::to_string(r.height),
      std::to_string(r.iterations),  to_string(r.strategy),
      std::to_string(r.workers),     std::to_string(r.seed),
      num.str(),                     std::to_string(r.repetitions),
      fixed(r.median_s, 3),          fixed(r.speedup, 2),
      std::to_string(r.hardware_threads), std::to_string(r.final_population)};
  std::string row;
  for (const std::string& f : fields) {
    if (!row.empty()) row.push_back(',');
    row.append(f);
  }
  return row;
}

// The reference's pinned CSV (bench.hpp:90-97).
inline std::string emit_csv(const std::vector<BenchRecord>& records) {
  std::string out =
      "width,height,iterations,strategy,workers,seed,density,repetitions,"
      "median_s,speedup,hardware_threads,final_population\n";
  for (const BenchRecord& r : records) out += csv_row_prefix(r) + "\n";
  return out;
}

// Roofline of a record: the packed engines are integer-bound (11 ops / 32
// cell-updates against the measured LOP3 peak of the whole GPU), the byte
// engine HBM-bound at one generation per pass (2 bytes per cell-update
// against the measured copy bandwidth) and instruction-bound when
// temporally blocked.
struct RooflinePeaks {
  double int_ops_per_s = 0.0;  // life_measure_int_peak
  double hbm_bytes_per_s = 6553.3e9;
};

inline double roofline_fraction(const BenchRecord& r, const RooflinePeaks& p) {
  const double ups = r.gcups() * 1e9;
  if (r.strategy.engine == Engine::Byte) {
    // One generation per pass: HBM-bound (2 B per update); temporal-blocked
    // passes (W % 16 == 0): 1.25 ALU + 1.25 FMA ops per update at 2x the LOP3 rate.
    if (r.strategy.depth == 1 || r.width % 16 != 0)
      return p.hbm_bytes_per_s > 0 ? ups * 2.0 / p.hbm_bytes_per_s : 0.0;
    return p.int_ops_per_s > 0 ? ups * 2.5 / (2.0 * p.int_ops_per_s) : 0.0;
  }
  return p.int_ops_per_s > 0 ? ups * (11.0 / 32.0) / p.int_ops_per_s : 0.0;
}

// The same rows plus gcups and roofline_frac columns.
inline std::string emit_csv_gpu(const std::vector<BenchRecord>& records, const RooflinePeaks& p) {
  std::string out =
      "width,height,iterations,strategy,workers,seed,density,repetitions,"
      "median_s,speedup,hardware_threads,final_population,gcups,roofline_frac\n";
  for (const BenchRecord& r : records)
    out += csv_row_prefix(r) + "," + fixed(r.gcups(), 3) + "," + fixed(roofline_fraction(r, p), 4) + "\n";
  return out;
}

}  // namespace lifegpu
