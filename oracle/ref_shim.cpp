// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference core
// library (/root/reference/proj/core), compiled together with its sources by
// oracle/Makefile into oracle/_ref/liblife_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used to pin the oracle restatement
// (oracle/life_oracle.c), to generate tests/golden/ fixtures, and as the
// CPU baseline arm of bench.py (`cpu_baseline.kind = "reference"`).  No
// reference source is copied into this repository; this file only calls the
// reference's public API (proj/core/include/life/*.hpp).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "life/bench.hpp"
#include "life/decomposition.hpp"
#include "life/engine.hpp"
#include "life/grid.hpp"
#include "life/pattern.hpp"
#include "life/render.hpp"
#include "life/rng.hpp"

namespace {

thread_local std::string g_error;

// Maps the reference exception hierarchy (errors.hpp:9-60) to status codes
// that mirror include/life_gpu.h.
int fail(const std::exception& e) {
  g_error = e.what();
  if (dynamic_cast<const life::DimensionTooSmall*>(&e)) return 2;
  if (dynamic_cast<const life::TooManyParts*>(&e)) return 3;
  if (dynamic_cast<const life::OutOfBounds*>(&e)) return 4;
  if (dynamic_cast<const life::ConfigError*>(&e)) return 1;
  return 99;
}

life::Strategy strategy_of(int kind, int bx, int by) {
  switch (kind) {
    case 0: return life::Strategy::serial();
    case 1: return life::Strategy::rows();
    case 2: return life::Strategy::cols();
    default: return life::Strategy::blocks(bx, by);
  }
}

life::Grid grid_of(const std::uint8_t* cells, int w, int h) {
  life::Grid g(w, h);
  std::memcpy(g.data(), cells, static_cast<std::size_t>(w) * h);
  return g;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

unsigned ref_hardware_threads() { return std::thread::hardware_concurrency(); }

void ref_splitmix_stream(std::uint64_t seed, std::int64_t n, std::uint64_t* out) {
  life::SplitMix64 r(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = r.next();
}

void ref_splitmix_units(std::uint64_t seed, std::int64_t n, double* out) {
  life::SplitMix64 r(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = r.next_unit();
}

// life::random_fill (pattern.cpp:330-342).
int ref_random_fill(int w, int h, double density, std::uint64_t seed, std::uint8_t* out) {
  try {
    const life::Grid g = life::random_fill(w, h, density, seed);
    std::memcpy(out, g.data(), static_cast<std::size_t>(w) * h);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// life::step_serial (grid.cpp:30-38).
int ref_step_serial(const std::uint8_t* in, int w, int h, std::uint8_t* out) {
  try {
    const life::Grid g = life::step_serial(grid_of(in, w, h));
    std::memcpy(out, g.data(), static_cast<std::size_t>(w) * h);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// life::next_state (grid.cpp:22-28).
int ref_next_state(int alive, int n) {
  return life::next_state(alive ? life::CellState::Alive : life::CellState::Dead, n) ==
         life::CellState::Alive;
}

// life::run (engine.cpp:162-214).  Populations are the reference's `int`
// values widened to int64 (they overflow above 2^31-1: SURVEY.md fact 4).
int ref_run(const std::uint8_t* in, int w, int h, int kind, int bx, int by, int workers,
            int iterations, const int* checkpoints, int n_checkpoints, std::uint8_t* out,
            std::int64_t* pops, int* generations_computed) {
  try {
    std::vector<int> cps(checkpoints, checkpoints + n_checkpoints);
    life::RunResult r = life::run(grid_of(in, w, h),
                                  life::RunConfig{strategy_of(kind, bx, by), workers, iterations},
                                  cps);
    std::memcpy(out, r.grid.data(), static_cast<std::size_t>(w) * h);
    for (std::size_t i = 0; i < r.stats.population_checkpoints.size(); ++i) {
      pops[i] = r.stats.population_checkpoints[i].second;
    }
    if (generations_computed) *generations_computed = r.stats.generations_computed;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// In-place variant for large grids (no extra caller copy): `cells` is both
// input and output.
int ref_run_inplace(std::uint8_t* cells, int w, int h, int kind, int bx, int by, int workers,
                    int iterations) {
  try {
    life::Grid g(w, h);
    std::memcpy(g.data(), cells, static_cast<std::size_t>(w) * h);
    life::RunResult r =
        life::run(std::move(g), life::RunConfig{strategy_of(kind, bx, by), workers, iterations});
    std::memcpy(cells, r.grid.data(), static_cast<std::size_t>(w) * h);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// life::time_run (bench.cpp:77-111): random_fill, warmup runs, then timed
// run()s with a steady_clock around each; median seconds and the final
// population are returned.
int ref_time_run(int w, int h, int iterations, int kind, int bx, int by, int workers,
                 std::uint64_t seed, double density, int repetitions, int warmup,
                 double* median_s, std::int64_t* final_population, unsigned* hw_threads) {
  try {
    life::TimingSpec spec;
    spec.width = w;
    spec.height = h;
    spec.iterations = iterations;
    spec.strategy = strategy_of(kind, bx, by);
    spec.workers = workers;
    spec.seed = seed;
    spec.density = density;
    spec.repetitions = repetitions;
    spec.warmup_runs = warmup;
    const life::BenchRecord rec = life::time_run(spec);
    *median_s = rec.median_s;
    *final_population = rec.final_population;
    if (hw_threads) *hw_threads = rec.hardware_threads;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// life::partition_rows (decomposition.cpp:93-104): writes parts+1 y-cuts.
int ref_partition_rows(int w, int h, int parts, int* cuts) {
  try {
    const life::Partition p = life::partition_rows(w, h, parts);
    for (int i = 0; i < parts; ++i) cuts[i] = p.regions[i].y0;
    cuts[parts] = p.regions[parts - 1].y1;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Config-4 soup built with the reference's own SplitMix64 and place_pattern
// (pattern.cpp:309-328).  place_pattern copies the grid per call, so this is
// only usable on small fields; it pins oracle/life_oracle.c:orc_sparse_soup.
int ref_sparse_soup_small(int w, int h, double coverage, int bs, double p, std::uint64_t seed,
                          std::uint8_t* out) {
  try {
    life::Grid g(w, h);
    life::SplitMix64 r(seed);
    const long long blocks = std::llround(coverage * double(w) * double(h) / (double(bs) * bs));
    for (long long b = 0; b < blocks; ++b) {
      const int x0 = static_cast<int>(r.next() % static_cast<std::uint64_t>(w - bs + 1));
      const int y0 = static_cast<int>(r.next() % static_cast<std::uint64_t>(h - bs + 1));
      life::Pattern pat{bs, bs, {}};
      for (int j = 0; j < bs; ++j)
        for (int i = 0; i < bs; ++i)
          if (r.next_unit() < p) pat.live_cells.push_back({i, j});
      pat.normalize();
      g = life::place_pattern(g, pat, {x0, y0});
    }
    std::memcpy(out, g.data(), static_cast<std::size_t>(w) * h);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// life::place_pattern (pattern.cpp:309-328) with a Pattern built from bytes.
int ref_place_pattern(std::uint8_t* cells, int w, int h, const std::uint8_t* pat, int pw, int ph,
                      int x0, int y0) {
  try {
    life::Pattern p{pw, ph, {}};
    for (int j = 0; j < ph; ++j)
      for (int i = 0; i < pw; ++i)
        if (pat[j * pw + i]) p.live_cells.push_back({i, j});
    p.normalize();
    const life::Grid g = life::place_pattern(grid_of(cells, w, h), p, {x0, y0});
    std::memcpy(cells, g.data(), static_cast<std::size_t>(w) * h);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Pattern I/O and renderers (pattern.cpp:147-292, render.cpp:5-38), for the
// parity tests of the GPU engine's host I/O layer.
static int copy_str(const std::string& s, char* out, int cap) {
  if (static_cast<int>(s.size()) + 1 > cap) return -1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}

static int export_pattern(const life::Pattern& p, int* w, int* h, int* xs, int* ys, int cap,
                          int* n) {
  *w = p.width;
  *h = p.height;
  *n = static_cast<int>(p.live_cells.size());
  if (*n > cap) return -1;
  for (int i = 0; i < *n; ++i) {
    xs[i] = p.live_cells[i].x;
    ys[i] = p.live_cells[i].y;
  }
  return 0;
}

int ref_parse_rle(const char* text, int* w, int* h, int* xs, int* ys, int cap, int* n, int* line,
                  int* col, char* msg, int msgcap) {
  try {
    return export_pattern(life::parse_rle(text), w, h, xs, ys, cap, n);
  } catch (const life::ParseError& e) {
    *line = e.line();
    *col = e.column();
    copy_str(e.what(), msg, msgcap);
    return 3;
  }
}

int ref_parse_plaintext(const char* text, int* w, int* h, int* xs, int* ys, int cap, int* n,
                        int* line, int* col, char* msg, int msgcap) {
  try {
    return export_pattern(life::parse_plaintext(text), w, h, xs, ys, cap, n);
  } catch (const life::ParseError& e) {
    *line = e.line();
    *col = e.column();
    copy_str(e.what(), msg, msgcap);
    return 3;
  }
}

int ref_serialize_rle(int w, int h, const int* xs, const int* ys, int n, char* out, int cap) {
  life::Pattern p{w, h, {}};
  for (int i = 0; i < n; ++i) p.live_cells.push_back({xs[i], ys[i]});
  try {
    return copy_str(life::serialize_rle(p), out, cap);
  } catch (const life::ConfigError&) {
    return 1;
  }
}

int ref_render_ascii(const std::uint8_t* cells, int w, int h, char* out, int cap) {
  return copy_str(life::render_ascii(grid_of(cells, w, h)), out, cap);
}

int ref_render_pbm(const std::uint8_t* cells, int w, int h, char* out, int cap) {
  return copy_str(life::render_pbm(grid_of(cells, w, h)), out, cap);
}

// life::population (grid.cpp:40-46) -- returns the reference's int.
int ref_population(const std::uint8_t* cells, int w, int h) {
  return life::population(grid_of(cells, w, h));
}

}  // extern "C"
