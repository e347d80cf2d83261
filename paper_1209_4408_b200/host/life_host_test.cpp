// life_host_test.cpp -- C++ tests of the host mirror (life_gpu.hpp) on a GPU,
// in the style of the reference's doctest suites (tests/test_grid.cpp,
// tests/test_engine.cpp): known patterns, the B3/S23 rule against a plain
// serial step, error classes.  Prints one PASS/FAIL line per case (like
// acceptance.cpp:408-422); exit code 0 when nothing failed.
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "life_gpu.hpp"

namespace {

// A byte torus with the reference Grid's shape (grid.hpp:24-70).
class Grid {
 public:
  Grid(int w, int h) : w_(w), h_(h), cells_(static_cast<size_t>(w) * h, 0) {
    if (w < 3 || h < 3) throw lifegpu::DimensionTooSmall("grid dimensions must be at least 3x3");
  }
  int width() const { return w_; }
  int height() const { return h_; }
  const uint8_t* data() const { return cells_.data(); }
  uint8_t* data() { return cells_.data(); }
  uint8_t at(int x, int y) const { return cells_[static_cast<size_t>(y) * w_ + x]; }
  void set(int x, int y, uint8_t v) { cells_[static_cast<size_t>(y) * w_ + x] = v; }
  bool operator==(const Grid& o) const { return w_ == o.w_ && h_ == o.h_ && cells_ == o.cells_; }

 private:
  int w_, h_;
  std::vector<uint8_t> cells_;
};

// The plainest step (grid.cpp:30-38) -- the test's own checker.
Grid serial_step(const Grid& g) {
  Grid n(g.width(), g.height());
  for (int y = 0; y < g.height(); ++y)
    for (int x = 0; x < g.width(); ++x) {
      int c = 0;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx)
          if (dx || dy)
            c += g.at((x + dx + g.width()) % g.width(), (y + dy + g.height()) % g.height()) != 0;
      n.set(x, y, g.at(x, y) ? (c == 2 || c == 3) : (c == 3));
    }
  return n;
}

int failures = 0;
void check_case(const char* name, const std::function<bool()>& f) {
  bool ok = false;
  std::string why;
  try {
    ok = f();
  } catch (const std::exception& e) {
    why = e.what();
  }
  std::printf("[%s] %s%s%s\n", ok ? "PASS" : "FAIL", name, why.empty() ? "" : ": ", why.c_str());
  if (!ok) ++failures;
}

template <class E>
bool throws(const std::function<void()>& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

}  // namespace

int main() {
  using lifegpu::Engine;
  using lifegpu::RunConfig;

  check_case("blinker period 2 (test_grid.cpp:189-205)", [] {
    Grid b(5, 5);
    b.set(1, 2, 1), b.set(2, 2, 1), b.set(3, 2, 1);
    for (Engine e : {Engine::Packed, Engine::Byte}) {
      RunConfig c;
      c.engine = e;
      Grid one = lifegpu::step_parallel(b, c);
      if (one == b || !(lifegpu::step_parallel(one, c) == b)) return false;
      c.iterations = 100;
      auto r = lifegpu::run(b, c, {0, 1, 100});
      if (!(r.grid == b) || r.stats.population_checkpoints.size() != 3) return false;
      for (auto& cp : r.stats.population_checkpoints)
        if (cp.second != 3) return false;
    }
    return true;
  });

  check_case("glider lap of 64 generations on 16x16 (test_grid.cpp:207-217)", [] {
    Grid g(16, 16);
    const int cells[5][2] = {{1, 0}, {2, 1}, {0, 2}, {1, 2}, {2, 2}};
    for (auto& c : cells) g.set(6 + c[0], 6 + c[1], 1);
    RunConfig c;
    c.iterations = 64;
    c.temporal_depth = 16;
    return lifegpu::run(g, c).grid == g;
  });

  check_case("random soups equal the serial step (strategy transparency)", [] {
    for (int seed = 0; seed < 6; ++seed) {
      const int w = 3 + (seed * 17 + 5) % 46 + 40 * seed, h = 3 + (seed * 29 + 11) % 46;
      Grid g = lifegpu::random_fill<Grid>(w, h, 0.3, seed);
      Grid want = g;
      for (int i = 0; i < 20; ++i) want = serial_step(want);
      for (int depth : {1, 5, 16}) {
        RunConfig c;
        c.iterations = 20;
        c.temporal_depth = depth;
        if (!(lifegpu::run(g, c).grid == want)) return false;
      }
      RunConfig cb;
      cb.engine = Engine::Byte;
      cb.iterations = 20;
      if (!(lifegpu::run(g, cb).grid == want)) return false;
    }
    return true;
  });

  check_case("illegal configurations throw the reference's classes (test_engine.cpp:132-140)", [] {
    Grid g(8, 5);
    RunConfig c;
    c.iterations = 1;
    c.workers = 10;
    if (!throws<lifegpu::TooManyParts>([&] { lifegpu::run(g, c); })) return false;
    c.workers = 0;
    if (!throws<lifegpu::ConfigError>([&] { lifegpu::run(g, c); })) return false;
    c.workers = 1;
    c.iterations = -1;
    if (!throws<lifegpu::ConfigError>([&] { lifegpu::run(g, c); })) return false;
    c.iterations = 2;
    if (!throws<lifegpu::ConfigError>([&] { lifegpu::run(g, c, {2, 1}); })) return false;
    if (!throws<lifegpu::ConfigError>([&] { lifegpu::run(g, c, {3}); })) return false;
    if (!throws<lifegpu::DimensionTooSmall>([] { lifegpu::random_fill<Grid>(2, 5, 0.5, 1); }))
      return false;
    return true;
  });

  check_case("uint64 populations and windows on a large grid", [] {
    lifegpu::Context ctx(0);
    ctx.init_random(65536, 40000, 0.5, 42);  // ~1.31e9 live cells
    const uint64_t p = ctx.population();
    const auto win = ctx.window(-3, -3, 7, 7);
    return p > (uint64_t(1) << 30) && win.size() == 49;
  });

  check_case("resident and byte engines agree with the packed engine (grid hash)", [] {
    lifegpu::Context ctx(0);
    uint64_t h[3];
    const lifegpu::Engine engines[3] = {lifegpu::Engine::Packed, lifegpu::Engine::Resident,
                                        lifegpu::Engine::Byte};
    for (int i = 0; i < 3; ++i) {
      ctx.init_random(512, 384, 0.4, 9, engines[i]);
      ctx.run(77, engines[i], 0, {});
      h[i] = ctx.hash();
    }
    return h[0] == h[1] && h[1] == h[2];
  });

  check_case("row bands over several devices equal the serial step (run(), devices = {0,0,0})", [] {
    for (int seed = 0; seed < 3; ++seed) {
      const int w = 70 + 33 * seed, h = 41 + 10 * seed;
      Grid g = lifegpu::random_fill<Grid>(w, h, 0.35, 100 + seed);
      Grid want = g;
      for (int i = 0; i < 37; ++i) want = serial_step(want);
      for (std::vector<int> devs : {std::vector<int>{0, 0}, std::vector<int>{0, 0, 0},
                                    std::vector<int>(7, 0)}) {
        RunConfig c;
        c.iterations = 37;
        c.workers = static_cast<int>(devs.size());
        c.devices = devs;
        auto r = lifegpu::run(g, c, {0, 5, 37});
        if (!(r.grid == want)) return false;
        uint64_t pop = 0;
        for (int i = 0; i < w * h; ++i) pop += want.data()[i];
        if (r.stats.population_checkpoints.back().second != pop) return false;
      }
    }
    return true;
  });

  check_case("two host threads run concurrently (SPEC.md:112: run() is thread-safe)", [] {
    bool ok[2] = {false, false};
    auto job = [&](int t) {
      try {
        for (int rep = 0; rep < 4; ++rep) {
          const int w = 200 + 64 * t + rep, h = 150 + rep;
          Grid g = lifegpu::random_fill<Grid>(w, h, 0.4, 7 * t + rep);
          Grid want = g;
          for (int i = 0; i < 25; ++i) want = serial_step(want);
          RunConfig c;
          c.iterations = 25;
          c.temporal_depth = t == 0 ? 16 : 5;
          if (!(lifegpu::run(g, c).grid == want)) return;
        }
        ok[t] = true;
      } catch (...) {
      }
    };
    std::thread a(job, 0), b(job, 1);
    a.join();
    b.join();
    return ok[0] && ok[1];
  });

  check_case("run_packed on host packed rows equals run() on bytes", [] {
    for (int rep = 0; rep < 3; ++rep) {
      const int w = 300 + 97 * rep, h = 120 + 31 * rep;
      Grid g = lifegpu::random_fill<Grid>(w, h, 0.35, 40 + rep);
      RunConfig c;
      c.iterations = 37;
      c.temporal_depth = rep == 0 ? 0 : 7;
      const Grid want = lifegpu::run(g, c).grid;
      const int64_t wpr = (w + 63) / 64;
      std::vector<uint64_t> words(static_cast<size_t>(wpr) * h, 0);
      for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
          if (g.at(x, y)) words[static_cast<size_t>(y) * wpr + x / 64] |= uint64_t(1) << (x % 64);
      lifegpu::run_packed(words.data(), words.data(), w, h, wpr, c);  // in place
      for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
          if (((words[static_cast<size_t>(y) * wpr + x / 64] >> (x % 64)) & 1) != want.at(x, y))
            return false;
    }
    return true;
  });

  std::printf("%d failure(s)\n", failures);
  return failures == 0 ? 0 : 1;
}
