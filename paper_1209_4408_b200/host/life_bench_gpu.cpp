// life-bench-gpu: the reference's CLI (tools/life_bench.cpp) on the B200 engine.
//
//   life-bench-gpu run   --width W --height H --iterations N [--strategy gpu|gpu:K|gpu-byte[:K]|gpu-resident]
//                        [--workers 1] [--pattern FILE.rle|FILE.cells | --seed S --density P]
//                        [--render none|ascii|pbm] [--out PATH] [--checkpoints a,b,c]
//   life-bench-gpu bench [--sizes 120x60,240x120] [--iterations 500,1000,2000]
//                        [--strategies gpu,gpu-byte] [--workers 1] [--repetitions 5]
//                        [--warmup 1] [--seed 42] [--density 0.3] [--csv PATH] [--gpu-columns]
//
// Same behaviour as life_bench.cpp:100-236: patterns are placed centred on an
// empty grid (origin ((W-pw)/2, (H-ph)/2)), the checkpoint/final-population
// summary goes to stderr when a rendering goes to stdout, and exit codes are
// 0 success, 2 configuration error, 3 pattern parse error.  CLI11 is absent, so
// the options are parsed by hand.
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "life_gpu.hpp"
#include "life_harness.hpp"
#include "life_io.hpp"

namespace {

using lifegpu::ConfigError;

class ByteGrid {
 public:
  ByteGrid(int w, int h) : w_(w), h_(h), c_(static_cast<size_t>(w) * h, 0) {
    if (w < 3 || h < 3)
      throw lifegpu::DimensionTooSmall("grid dimensions must be at least 3x3, got " +
                                       std::to_string(w) + "x" + std::to_string(h));
  }
  int width() const { return w_; }
  int height() const { return h_; }
  const uint8_t* data() const { return c_.data(); }
  uint8_t* data() { return c_.data(); }

 private:
  int w_, h_;
  std::vector<uint8_t> c_;
};

// Fields of a separator-joined list; an empty input is one empty field.
std::vector<std::string> split(const std::string& text, char sep) {
  std::vector<std::string> fields(1);
  for (const char ch : text) {
    if (ch == sep) {
      fields.emplace_back();
    } else {
      fields.back().push_back(ch);
    }
  }
  return fields;
}

// Whole-token numeric conversion: trailing junk, overflow and empty tokens
// are all the same configuration error.
template <class T, class Convert>
T parse_number(const std::string& token, const std::string& what, Convert convert) {
  size_t consumed = 0;
  bool good = !token.empty();
  T v{};
  if (good) {
    try {
      v = static_cast<T>(convert(token, &consumed));
    } catch (const std::logic_error&) {  // invalid_argument / out_of_range
      good = false;
    }
  }
  if (!good || consumed != token.size()) throw ConfigError("invalid " + what + " '" + token + "'");
  return v;
}

int64_t to_int(const std::string& token, const std::string& what) {
  return parse_number<int64_t>(token, what,
                               [](const std::string& t, size_t* n) { return std::stoll(t, n); });
}

double to_double(const std::string& token, const std::string& what) {
  return parse_number<double>(token, what,
                              [](const std::string& t, size_t* n) { return std::stod(t, n); });
}

std::vector<int64_t> int_list(const std::string& arg, const std::string& what) {
  std::vector<int64_t> out;
  if (arg.empty()) return out;
  for (const std::string& t : split(arg, ',')) out.push_back(to_int(t, what));
  return out;
}

// An empty path means standard output.
void write_output(const std::string& path, const std::string& payload) {
  const bool to_file = !path.empty();
  std::ofstream file;
  if (to_file) file.open(path, std::ios::out | std::ios::binary | std::ios::trunc);
  std::ostream& sink = to_file ? static_cast<std::ostream&>(file) : std::cout;
  sink.write(payload.data(), static_cast<std::streamsize>(payload.size()));
  if (to_file && (!file.is_open() || file.fail()))
    throw ConfigError("cannot write output file '" + path + "'");
}

// --name value options of one subcommand; unknown names are configuration errors.
struct Options {
  std::map<std::string, std::string> values;
  std::set<std::string> flags;
  bool has(const std::string& k) const { return values.count(k) > 0; }
  std::string get(const std::string& k, const std::string& dflt = "") const {
    auto it = values.find(k);
    return it == values.end() ? dflt : it->second;
  }
};

Options parse_options(int argc, char** argv, int first, const std::set<std::string>& allowed,
                      const std::set<std::string>& allowed_flags) {
  Options o;
  for (int i = first; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--", 0) != 0) throw ConfigError("unexpected argument '" + a + "'");
    std::string name = a.substr(2), value;
    const size_t eq = name.find('=');
    if (eq != std::string::npos) {
      value = name.substr(eq + 1);
      name = name.substr(0, eq);
    } else if (allowed_flags.count(name)) {
      o.flags.insert(name);
      continue;
    } else {
      if (i + 1 >= argc) throw ConfigError("option --" + name + " needs a value");
      value = argv[++i];
    }
    if (!allowed.count(name)) throw ConfigError("unknown option --" + name);
    o.values[name] = value;
  }
  return o;
}

const char* kUsage =
    "life-bench-gpu: Game of Life on the B200 engine (the reference's life-bench CLI)\n"
    "  run   --width W --height H --iterations N [--strategy gpu|gpu:K|gpu-byte[:K]|gpu-resident] [--workers 1]\n"
    "        [--pattern FILE.rle|FILE.cells | --seed S --density P] [--render none|ascii|pbm]\n"
    "        [--out PATH] [--checkpoints a,b,c] [--device D]\n"
    "  bench [--sizes WxH,...] [--iterations a,b] [--strategies gpu,gpu:8,gpu-byte] [--workers 1]\n"
    "        [--repetitions 5] [--warmup 1] [--seed 42] [--density 0.3] [--csv PATH]\n"
    "        [--gpu-columns] [--device D]\n"
    "exit codes: 0 success, 2 configuration error, 3 pattern parse error\n";

int run_command(const Options& o) {
  for (const char* req : {"width", "height", "iterations"})
    if (!o.has(req)) throw ConfigError(std::string("--") + req + " is required");
  if (o.has("pattern") && (o.has("seed") || o.has("density")))
    throw ConfigError("--pattern excludes --seed and --density");
  const int width = static_cast<int>(to_int(o.get("width"), "width"));
  const int height = static_cast<int>(to_int(o.get("height"), "height"));
  const int64_t iterations = to_int(o.get("iterations"), "iteration count");
  const lifegpu::Strategy strategy = lifegpu::parse_strategy(o.get("strategy", "gpu"));
  const int workers = static_cast<int>(to_int(o.get("workers", "1"), "worker count"));
  const std::string render = o.get("render", "none");
  if (render != "none" && render != "ascii" && render != "pbm")
    throw ConfigError("--render must be none, ascii or pbm");
  const std::vector<int64_t> checkpoints = int_list(o.get("checkpoints"), "checkpoint");
  const int device = static_cast<int>(to_int(o.get("device", "0"), "device"));

  // Pattern first (parse errors win over dimension errors, life_bench.cpp:104-110).
  lifegpu::Pattern pat;
  if (o.has("pattern")) pat = lifegpu::load_pattern_file(o.get("pattern"));
  ByteGrid grid(width, height);
  if (o.has("pattern")) {
    grid = lifegpu::place_pattern(grid, pat, {(width - pat.width) / 2, (height - pat.height) / 2});
  } else {
    const uint64_t seed = static_cast<uint64_t>(to_int(o.get("seed", "42"), "seed"));
    const double density = to_double(o.get("density", "0.3"), "density");
    if (!(density >= 0.0 && density <= 1.0))
      throw ConfigError("density must be in [0, 1], got " + o.get("density"));
    grid = lifegpu::random_fill<ByteGrid>(width, height, density, seed, device);
  }
  lifegpu::RunConfig cfg;
  cfg.engine = strategy.engine;
  cfg.temporal_depth = strategy.depth;
  cfg.workers = workers;
  cfg.iterations = iterations;
  cfg.device = device;
  auto result = lifegpu::run(std::move(grid), cfg, checkpoints);

  const bool render_to_stdout = render != "none" && o.get("out").empty();
  std::ostream& info = render_to_stdout ? std::cerr : std::cout;
  for (const auto& [it, pop] : result.stats.population_checkpoints)
    info << "checkpoint " << it << " population " << pop << "\n";
  uint64_t final_pop = 0;
  for (int64_t i = 0; i < int64_t(width) * height; ++i) final_pop += result.grid.data()[i] != 0;
  info << "final population " << final_pop << " after " << result.stats.generations_computed
       << " generations\n";
  if (render == "ascii") write_output(o.get("out"), lifegpu::render_ascii(result.grid) + "\n");
  if (render == "pbm") write_output(o.get("out"), lifegpu::render_pbm(result.grid));
  return 0;
}

int bench_command(const Options& o) {
  lifegpu::BenchConfig config;
  for (const std::string& t : split(o.get("sizes", "120x60,240x120"), ',')) {
    const size_t x = t.find('x');
    if (x == std::string::npos || x == 0 || x + 1 >= t.size())
      throw ConfigError("invalid size '" + t + "' (expected WxH, e.g. 120x60)");
    config.sizes.push_back({static_cast<int>(to_int(t.substr(0, x), "width")),
                            static_cast<int>(to_int(t.substr(x + 1), "height"))});
  }
  for (int64_t v : int_list(o.get("iterations", "500,1000,2000"), "iteration count"))
    config.iteration_counts.push_back(static_cast<int>(v));
  for (const std::string& t : split(o.get("strategies", "gpu,gpu-byte"), ','))
    config.strategies.push_back(lifegpu::parse_strategy(t));
  config.worker_counts.clear();
  for (int64_t v : int_list(o.get("workers", "1"), "worker count"))
    config.worker_counts.push_back(static_cast<int>(v));
  config.repetitions = static_cast<int>(to_int(o.get("repetitions", "5"), "repetitions"));
  config.warmup_runs = static_cast<int>(to_int(o.get("warmup", "1"), "warmup"));
  config.seed = static_cast<uint64_t>(to_int(o.get("seed", "42"), "seed"));
  config.density = to_double(o.get("density", "0.3"), "density");
  config.device = static_cast<int>(to_int(o.get("device", "0"), "device"));
  const auto records = lifegpu::bench_matrix(config, [](const lifegpu::BenchRecord& r) {
    std::cerr << "timed " << r.width << "x" << r.height << " iterations=" << r.iterations
              << " strategy=" << lifegpu::to_string(r.strategy) << " workers=" << r.workers
              << " median=" << r.median_s << "s speedup=" << r.speedup
              << " gcups=" << r.gcups() << "\n";
  });
  if (o.flags.count("gpu-columns")) {
    lifegpu::RooflinePeaks peaks;
    double ops = 0, secs = 0;
    if (life_measure_int_peak(config.device, 2000, &ops, &secs) == LIFE_OK) peaks.int_ops_per_s = ops;
    write_output(o.get("csv"), lifegpu::emit_csv_gpu(records, peaks));
  } else {
    write_output(o.get("csv"), lifegpu::emit_csv(records));
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << kUsage;
    return 2;
  }
  const std::string cmd = argv[1];
  if (cmd == "--help" || cmd == "-h" || cmd == "help") {
    std::cout << kUsage;
    return 0;
  }
  try {
    for (int i = 2; i < argc; ++i) {
      const std::string a = argv[i];
      if (a == "--help" || a == "-h") {
        std::cout << kUsage;
        return 0;
      }
    }
    if (cmd == "run") {
      return run_command(parse_options(
          argc, argv, 2,
          {"width", "height", "iterations", "strategy", "workers", "pattern", "seed", "density",
           "render", "out", "checkpoints", "device"},
          {}));
    }
    if (cmd == "bench") {
      return bench_command(parse_options(
          argc, argv, 2,
          {"sizes", "iterations", "strategies", "workers", "repetitions", "warmup", "seed",
           "density", "csv", "device"},
          {"gpu-columns"}));
    }
    throw ConfigError("unknown subcommand '" + cmd + "' (expected run or bench)");
  } catch (const lifegpu::ParseError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
}
