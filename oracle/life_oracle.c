/*
 * life_oracle.c -- CPU restatement of the reference's generation-step path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * engine in paper_1209_4408_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never links or calls it (it fails loudly without the CUDA
 * library instead).
 *
 * Parity is pinned two ways (see tests/test_oracle.py):
 *   - against the reference's own known-answer vectors (splitmix64 streams of
 *     proj/tests/test_rng.cpp:12-57, the B3/S23 table of
 *     proj/tests/test_grid.cpp:77-93, blinker/block/glider of
 *     proj/tests/test_grid.cpp:177-217);
 *   - against the reference library itself, compiled from
 *     /root/reference/proj/core by oracle/Makefile into oracle/_ref/ and run
 *     by tests/golden/make_golden.py, whose outputs are committed under
 *     tests/golden/.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define ORC_GAMMA 0x9E3779B97F4A7C15ULL

/* splitmix64 output function: core/include/life/rng.hpp:22-27. */
static inline uint64_t orc_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* SplitMix64::next (rng.hpp:22-27): advances *state and returns the output. */
uint64_t orc_splitmix_next(uint64_t* state) {
  *state += ORC_GAMMA;
  return orc_mix(*state);
}

/* SplitMix64::next_unit (rng.hpp:30-32). */
double orc_splitmix_unit(uint64_t* state) {
  return (double)(orc_splitmix_next(state) >> 11) * 0x1.0p-53;
}

/* Fills out[0..n) with the first n draws of SplitMix64(seed). */
void orc_splitmix_stream(uint64_t seed, int64_t n, uint64_t* out) {
  uint64_t s = seed;
  for (int64_t i = 0; i < n; ++i) out[i] = orc_splitmix_next(&s);
}

/*
 * Integer threshold equivalent of `next_unit() < density`
 * (pattern.cpp:338).  next_unit() = m * 2^-53 with m = next() >> 11 an
 * integer in [0, 2^53); m * 2^-53 and density * 2^53 are both exact, so
 * `m * 2^-53 < p`  <=>  `m < p * 2^53`  <=>  `m < ceil(p * 2^53)`.
 */
uint64_t orc_density_threshold(double density) {
  if (!(density >= 0.0 && density <= 1.0)) return UINT64_MAX;
  return (uint64_t)ceil(density * 0x1.0p53);
}

/*
 * random_fill (pattern.cpp:330-342), restated counter-style.  The reference
 * draws one value per cell in row-major order from SplitMix64(seed); draw k
 * (0-based) has state seed + (k+1)*gamma, so cell i = y*W + x is alive iff
 * (mix(seed + (i+1)*gamma) >> 11) < threshold.  Returns -1 on a bad density
 * (the reference throws ConfigError, pattern.cpp:331-333).
 */
int orc_random_fill(uint8_t* out, int64_t width, int64_t height, double density,
                    uint64_t seed) {
  if (!(density >= 0.0 && density <= 1.0)) return -1;
  const uint64_t thr = orc_density_threshold(density);
  uint64_t s = seed;
  const int64_t n = width * height;
  for (int64_t i = 0; i < n; ++i) {
    s += ORC_GAMMA;
    out[i] = (uint8_t)((orc_mix(s) >> 11) < thr);
  }
  return 0;
}

/* Random-access cell of the random_fill torus (same formula as above). */
static inline uint8_t orc_random_cell(int64_t width, int64_t x, int64_t y, uint64_t seed,
                                      uint64_t thr) {
  const uint64_t i = (uint64_t)(y * width + x);
  return (uint8_t)((orc_mix(seed + (i + 1) * ORC_GAMMA) >> 11) < thr);
}

/*
 * Window [x0, x0+w) x [y0, y0+h) of random_fill(W, H, density, seed), with
 * coordinates wrapped onto the torus (Grid::wrap, grid.hpp:48-54).  Used for
 * light-cone parity on grids too large to materialise (config 5).
 */
int orc_random_window(uint8_t* out, int64_t width, int64_t height, double density,
                      uint64_t seed, int64_t x0, int64_t y0, int64_t w, int64_t h) {
  if (!(density >= 0.0 && density <= 1.0)) return -1;
  const uint64_t thr = orc_density_threshold(density);
  for (int64_t j = 0; j < h; ++j) {
    int64_t y = (y0 + j) % height;
    if (y < 0) y += height;
    for (int64_t i = 0; i < w; ++i) {
      int64_t x = (x0 + i) % width;
      if (x < 0) x += width;
      out[j * w + i] = orc_random_cell(width, x, y, seed, thr);
    }
  }
  return 0;
}

/*
 * Config-4 sparse soup (the reference has no such
 * generator, so this definition is pinned from its own building blocks):
 *   SplitMix64 r(seed); B = llround(coverage*W*H/(bs*bs));
 *   for each block: x0 = r.next() % (W-bs+1); y0 = r.next() % (H-bs+1);
 *     then bs*bs cells row-major, alive iff r.next_unit() < p,
 *     written with place_pattern's overwrite semantics (pattern.cpp:309-328:
 *     the whole footprint is cleared, then the live cells set; no wrap).
 * `out` must hold W*H bytes and is cleared first (an empty field).
 */
int orc_sparse_soup(uint8_t* out, int64_t width, int64_t height, double coverage,
                    int32_t bs, double p, uint64_t seed) {
  if (bs < 1 || bs > width || bs > height) return -1;
  if (!(p >= 0.0 && p <= 1.0) || !(coverage >= 0.0)) return -1;
  memset(out, 0, (size_t)(width * height));
  const int64_t blocks = llround(coverage * (double)width * (double)height /
                                 ((double)bs * (double)bs));
  uint64_t s = seed;
  for (int64_t b = 0; b < blocks; ++b) {
    const int64_t bx = (int64_t)(orc_splitmix_next(&s) % (uint64_t)(width - bs + 1));
    const int64_t by = (int64_t)(orc_splitmix_next(&s) % (uint64_t)(height - bs + 1));
    for (int32_t j = 0; j < bs; ++j) {
      for (int32_t i = 0; i < bs; ++i) {
        out[(by + j) * width + bx + i] = (uint8_t)(orc_splitmix_unit(&s) < p);
      }
    }
  }
  return 0;
}

/* B3/S23 transition, next_state (grid.cpp:22-28). */
static inline uint8_t orc_next_state(int alive, int n) {
  return (uint8_t)(alive ? (n == 2 || n == 3) : (n == 3));
}

/*
 * step_serial (grid.cpp:30-38) with neighbor_count (grid.cpp:7-20) and the
 * wrap of Grid::wrap (grid.hpp:48-54): any nonzero byte is alive
 * (Grid::alive, grid.hpp:42); output bytes are 0/1.
 */
void orc_step_serial(const uint8_t* in, uint8_t* out, int64_t width, int64_t height) {
  for (int64_t y = 0; y < height; ++y) {
    for (int64_t x = 0; x < width; ++x) {
      int n = 0;
      for (int dy = -1; dy <= 1; ++dy) {
        for (int dx = -1; dx <= 1; ++dx) {
          if (dx == 0 && dy == 0) continue;
          int64_t nx = (x + dx) % width;
          if (nx < 0) nx += width;
          int64_t ny = (y + dy) % height;
          if (ny < 0) ny += height;
          n += in[ny * width + nx] != 0;
        }
      }
      out[y * width + x] = orc_next_state(in[y * width + x] != 0, n);
    }
  }
}

/*
 * compute_region (engine.cpp:17-48) over rows [y0, y1) and all columns:
 * three row pointers with vertical wrap (:24-26), torus columns 0 and W-1
 * peeled (:35-39, :44-46), `out = (n==3) | ((n==2) & mid)` on 0/1 bytes
 * (:30-32).  Inputs must be 0/1 (the reference's engine adds raw bytes).
 */
static void orc_region(const uint8_t* cells, uint8_t* out, int64_t w, int64_t h, int64_t y0,
                       int64_t y1) {
  for (int64_t y = y0; y < y1; ++y) {
    const uint8_t* up = cells + (y == 0 ? h - 1 : y - 1) * w;
    const uint8_t* mid = cells + y * w;
    const uint8_t* down = cells + (y == h - 1 ? 0 : y + 1) * w;
    uint8_t* row = out + y * w;
    for (int64_t x = 0; x < w; ++x) {
      const int64_t xl = x == 0 ? w - 1 : x - 1;
      const int64_t xr = x == w - 1 ? 0 : x + 1;
      const int n = up[xl] + up[x] + up[xr] + mid[xl] + mid[xr] + down[xl] + down[x] + down[xr];
      row[x] = (uint8_t)((n == 3) | ((n == 2) & mid[x]));
    }
  }
}

/* population (grid.cpp:40-46), widened to uint64 (the reference's int
 * overflows above 2^31-1 live cells). */
uint64_t orc_population(const uint8_t* cells, int64_t n) {
  uint64_t c = 0;
  for (int64_t i = 0; i < n; ++i) c += cells[i] != 0;
  return c;
}

/*
 * run (engine.cpp:162-214), serial team: `generations` applications of
 * compute_region into a double buffer with a swap (:207).  Populations are
 * recorded at the strictly ascending checkpoints (checkpoint 0 = the initial
 * grid, :179-186).  `grid` (W*H bytes, 0/1) is updated in place.  Returns -1
 * on the ConfigError conditions of check_run_config (engine.cpp:127-148).
 */
int orc_run(uint8_t* grid, int64_t width, int64_t height, int64_t generations,
            const int64_t* checkpoints, int32_t n_checkpoints, uint64_t* pops) {
  if (generations < 0) return -1;
  int64_t prev = -1;
  for (int32_t i = 0; i < n_checkpoints; ++i) {
    if (checkpoints[i] < 0 || checkpoints[i] > generations || checkpoints[i] <= prev) return -1;
    prev = checkpoints[i];
  }
  const int64_t n = width * height;
  uint8_t* next = (uint8_t*)malloc((size_t)n);
  if (!next) return -2;
  uint8_t* cur = grid;
  int32_t ci = 0;
  while (ci < n_checkpoints && checkpoints[ci] == 0) pops[ci++] = orc_population(cur, n);
  for (int64_t g = 1; g <= generations; ++g) {
    orc_region(cur, next, width, height, 0, height);
    uint8_t* t = cur;
    cur = next;
    next = t;
    while (ci < n_checkpoints && checkpoints[ci] == g) pops[ci++] = orc_population(cur, n);
  }
  if (cur != grid) {
    memcpy(grid, cur, (size_t)n);
    free(cur);
  } else {
    free(next);
  }
  return 0;
}

/* Repeated step_serial: the plainest oracle (grid.cpp:30-38). */
int orc_run_serial(uint8_t* grid, int64_t width, int64_t height, int64_t generations) {
  const int64_t n = width * height;
  uint8_t* tmp = (uint8_t*)malloc((size_t)n);
  if (!tmp) return -2;
  for (int64_t g = 0; g < generations; ++g) {
    orc_step_serial(grid, tmp, width, height);
    memcpy(grid, tmp, (size_t)n);
  }
  free(tmp);
  return 0;
}

/*
 * Light-cone window oracle.  Takes the (S+2T) x (S+2T)
 * window of the initial torus centred on [x0, x0+S) x [y0, y0+S), runs it as
 * its own torus for T generations, and returns its central S x S block, which
 * equals the same block of the full-torus result because influence spreads
 * at most one cell per generation.  `initial_window` is (S+2T)^2 bytes with
 * origin (x0-T, y0-T); `out` gets S*S bytes.
 */
int orc_lightcone(const uint8_t* initial_window, int64_t s, int64_t t, uint8_t* out) {
  const int64_t side = s + 2 * t;
  uint8_t* g = (uint8_t*)malloc((size_t)(side * side));
  if (!g) return -2;
  memcpy(g, initial_window, (size_t)(side * side));
  int rc = orc_run(g, side, side, t, NULL, 0, NULL);
  if (rc == 0) {
    for (int64_t j = 0; j < s; ++j) memcpy(out + j * s, g + (j + t) * side + t, (size_t)s);
  }
  free(g);
  return rc;
}

/* FNV-1a-64 over n bytes (the survey's golden hash; offset 0xcbf29ce484222325,
 * prime 0x100000001b3). `h` chains calls: pass 0 to start. */
uint64_t orc_fnv1a64(const uint8_t* bytes, int64_t n, uint64_t h) {
  if (h == 0) h = 0xcbf29ce484222325ULL;
  for (int64_t i = 0; i < n; ++i) {
    h ^= bytes[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* life_grid_hash's definition (include/life_gpu.h; not a reference function:
 * the checksum of row checksums that lets the device hash rows in
 * parallel): FNV-1a-64 over the H row hashes (8 little-endian bytes each),
 * row hash = FNV-1a-64 over the row's wpr packed uint64 words. */
uint64_t orc_grid_hash(const uint64_t* words, int64_t wpr, int64_t height) {
  uint8_t* rows = (uint8_t*)malloc((size_t)height * 8);
  if (!rows) return 0;
  for (int64_t y = 0; y < height; ++y) {
    const uint64_t r = orc_fnv1a64((const uint8_t*)(words + y * wpr), wpr * 8, 0);
    for (int i = 0; i < 8; ++i) rows[y * 8 + i] = (uint8_t)(r >> (8 * i));
  }
  const uint64_t h = orc_fnv1a64(rows, height * 8, 0);
  free(rows);
  return h;
}

/*
 * Packs a W x H byte grid into the packed exchange format of
 * include/life_gpu.h: row-major rows of ceil(W/64) little-endian uint64
 * words, bit j of word k = column 64k+j, tail bits zero, nonzero byte -> 1.
 */
void orc_pack(const uint8_t* cells, int64_t width, int64_t height, uint64_t* words) {
  const int64_t wpr = (width + 63) / 64;
  memset(words, 0, (size_t)(wpr * height) * sizeof(uint64_t));
  for (int64_t y = 0; y < height; ++y) {
    for (int64_t x = 0; x < width; ++x) {
      if (cells[y * width + x]) words[y * wpr + (x >> 6)] |= 1ULL << (x & 63);
    }
  }
}

void orc_unpack(const uint64_t* words, int64_t width, int64_t height, uint8_t* cells) {
  const int64_t wpr = (width + 63) / 64;
  for (int64_t y = 0; y < height; ++y) {
    for (int64_t x = 0; x < width; ++x) {
      cells[y * width + x] = (uint8_t)((words[y * wpr + (x >> 6)] >> (x & 63)) & 1);
    }
  }
}

/* band_bounds (decomposition.cpp:12-24): parts+1 cut points; the first
 * (extent mod parts) bands get one extra unit.  Returns -1 when
 * parts < 1 or parts > extent (TooManyParts, decomposition.cpp:26-30). */
int orc_band_bounds(int64_t extent, int32_t parts, int64_t* bounds) {
  if (parts < 1 || parts > extent) return -1;
  const int64_t base = extent / parts, extra = extent % parts;
  int64_t at = 0;
  bounds[0] = 0;
  for (int32_t i = 0; i < parts; ++i) {
    at += base + (i < extra ? 1 : 0);
    bounds[i + 1] = at;
  }
  return 0;
}

/* place_pattern (pattern.cpp:309-328): the pw x ph footprint at (x0, y0) is
 * cleared and the pattern's live (nonzero) cells set; no wrap.  Returns -1
 * when the footprint does not fit (OutOfBounds, pattern.cpp:310-316). */
int orc_place_pattern(uint8_t* grid, int64_t width, int64_t height, const uint8_t* pat,
                      int64_t pw, int64_t ph, int64_t x0, int64_t y0) {
  if (x0 < 0 || y0 < 0 || x0 + pw > width || y0 + ph > height) return -1;
  for (int64_t j = 0; j < ph; ++j)
    for (int64_t i = 0; i < pw; ++i) grid[(y0 + j) * width + x0 + i] = pat[j * pw + i] != 0;
  return 0;
}
