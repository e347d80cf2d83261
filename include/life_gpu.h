/*
 * life_gpu.h -- C-ABI of the B200-native Game of Life generation-step engine.
 *
 * This is the drop-in boundary for the reference's step loop.  The reference
 * (arxiv/paper_1209_4408, /root/reference/proj) has no FFI: its operator API
 * is the C++ function set of core/include/life/engine.hpp:11-43
 *     RunResult run(Grid&& initial, const RunConfig&, const std::vector<int>& checkpoints);
 *     Grid step_parallel(const Grid&, const Strategy&, int workers);
 * over the byte-per-cell torus `Grid` (core/include/life/grid.hpp:24-70).
 * Each entry point below names the reference interface it replaces; the C++
 * host mirror (paper_1209_4408_b200/host/life_gpu.hpp) rebuilds the
 * reference's `run()` semantics on top of it, and INTEGRATION.md shows the
 * binding a maintainer adds to the reference.
 *
 * Conventions
 *   - Plain pointers and sizes only; no exceptions cross this boundary.
 *     Every function returns a status code (LIFE_OK = 0) and leaves a
 *     message in life_last_error() (thread-local).
 *   - Cell contract: byte grids are row-major, one byte
 *     per cell; any NONZERO byte is alive (Grid::alive, grid.hpp:42, i.e.
 *     step_serial semantics) and outputs are exactly 0/1.
 *   - Packed exchange format: row-major rows of words_per_row >= ceil(W/64)
 *     little-endian uint64 words; bit j of word k is column 64k+j; bits at
 *     columns >= W are ignored on input and written as zero on output.
 *   - Dimensions: W, H >= 3 (Grid ctor, grid.hpp:29-35 -> DimensionTooSmall).
 *   - Populations are uint64 (the reference's int population overflows
 *     above 2^31-1 live cells, grid.cpp:40-46).
 *   - All device work of a context is ordered on its CUDA stream; every
 *     host-buffer entry point returns only after its results are on the host.
 */
#ifndef LIFE_GPU_H
#define LIFE_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: the reference's exception hierarchy (errors.hpp:9-60). */
#define LIFE_OK 0
#define LIFE_ERR_CONFIG 1               /* life::ConfigError (engine.cpp:127-148) */
#define LIFE_ERR_DIMENSION_TOO_SMALL 2  /* life::DimensionTooSmall (grid.hpp:31-33) */
#define LIFE_ERR_TOO_MANY_PARTS 3       /* life::TooManyParts (decomposition.cpp:26-30) */
#define LIFE_ERR_OUT_OF_BOUNDS 4        /* life::OutOfBounds (pattern.cpp:310-316) */
#define LIFE_ERR_STATE 5                /* no grid loaded in the context */
#define LIFE_ERR_CUDA 10                /* CUDA runtime failure (message has the CUDA error) */
#define LIFE_ERR_NO_DEVICE 11           /* no CUDA device / bad device ordinal */
#define LIFE_ERR_OUT_OF_MEMORY 12       /* device allocation failed */

/* Engines (the reference's Strategy::Kind dispatch, decomposition.hpp:31,
 * gains GPU kinds). */
#define LIFE_ENGINE_PACKED 0 /* 64 cells/uint64, LOP3 adder network, temporal blocking */
#define LIFE_ENGINE_BYTE 1   /* one byte per cell, SWAR sums, up to 8 generations per pass */
/* Packed layout, whole torus resident in the shared memory of one thread-block
 * cluster (<= 16 CTAs), every generation in one launch: small tori with
 * W % 32 == 0 (LIFE_ERR_CONFIG otherwise).  LIFE_ENGINE_PACKED with
 * temporal_depth 0 (auto) selects it when it is the faster engine. */
#define LIFE_ENGINE_RESIDENT 2

/* Largest temporal depth (generations per kernel pass) of the packed engine. */
#define LIFE_MAX_TEMPORAL_DEPTH 16

typedef struct life_ctx life_ctx;

/* Thread-local message of the last failing call on this thread. */
const char* life_last_error(void);
const char* life_version(void);

/* ---- context (owns device buffers and a stream on one GPU) ------------- */
/* A context is used by one host thread at a time; distinct contexts may be
 * used concurrently from different threads (the reference's run() is pure and
 * safe to call from any thread). */
int life_ctx_create(int device, life_ctx** out);
/* Multi-device context: the torus is split into `n` row bands by band_bounds
 * (decomposition.cpp:12-24 -- the paper's 1-D row decomposition, what
 * run(..., RunConfig{Strategy::rows(), workers = n}) does with threads,
 * engine.cpp:162-214), band i resident on GPU devices[i].  Repeated device
 * ids are allowed (several bands on one GPU run the same code).  Owns the
 * peer-access setup: neighbouring bands on different GPUs read each other's
 * K halo rows inside the pass kernel over NVLink (LIFE_HALO_PEER), or, when
 * peer access is unavailable, copy them into ghost rows first
 * (LIFE_HALO_COPY).  Passes are ordered across bands by events between
 * NEIGHBOURING bands only -- no global barrier.  Every grid / run entry point
 * below accepts it (packed engine only: LIFE_ENGINE_BYTE / _RESIDENT and
 * life_ctx_set_stream return LIFE_ERR_CONFIG); a loaded grid needs H >= n
 * (LIFE_ERR_TOO_MANY_PARTS otherwise, decomposition.cpp:26-30). */
int life_ctx_create_multi(int32_t n, const int* devices, life_ctx** out);
int life_ctx_destroy(life_ctx* ctx);
/* Orders the context's work on an external stream (e.g. torch's current
 * stream); NULL restores the context's own stream. */
int life_ctx_set_stream(life_ctx* ctx, void* cuda_stream);
int life_ctx_sync(life_ctx* ctx);
/* Band layout: *n bands, bounds[0..n] row cut points, devices[0..n-1], *halo
 * (LIFE_HALO_*, -1 for a single-device context).  NULL outputs are skipped;
 * bounds needs n+1 entries (call with bounds = devices = NULL first). */
int life_ctx_bands(life_ctx* ctx, int32_t* n, int64_t* bounds, int32_t* devices, int32_t* halo);

/* Context options. */
#define LIFE_OPT_PROFILE 1         /* 1: CUDA events around every pass of life_run (band stats) */
#define LIFE_OPT_BATCH_TRAPEZOID 2 /* life_run_batch first/last-grid chunk schedule: -1 auto, 0, 1 */
#define LIFE_OPT_HALO 3            /* multi-device halo scheme: LIFE_HALO_PEER / LIFE_HALO_COPY */
#define LIFE_OPT_PAIR_DEPTH 4      /* pair-layout kernel (W % 64 == 0): -1 auto, 0 off, 1..12 forced depth */
#define LIFE_OPT_QUAD_DEPTH 5      /* quad-layout kernel (W % 128 == 0): -1 auto, 0 off, 1..7 forced depth */
#define LIFE_HALO_PEER 0           /* edge-strip kernels read neighbour rows over NVLink (P2P) */
#define LIFE_HALO_COPY 1           /* neighbour rows copied into local ghost rows, then computed */
int life_ctx_set_option(life_ctx* ctx, int32_t option, int64_t value);
int life_ctx_get_option(life_ctx* ctx, int32_t option, int64_t* value);

/* Per-band statistics of the last life_run (band 0 = the whole torus of a
 * single-device context).  run_ms: CUDA-event time on the band's device from
 * the run's first launch to its last; with LIFE_OPT_PROFILE, interior_ms /
 * edge_ms are the summed per-pass times of the interior launches and of the
 * edge strips (halo copies included), and wait_ms = run_ms - interior_ms -- the
 * time the band's compute stream did not run interior rows (edges, neighbour
 * waits, pass boundaries).  For a single-device context interior_ms is the
 * whole pass. */
typedef struct life_band_stats {
  int32_t band, device;
  int64_t y0, rows;
  int64_t passes;
  double run_ms, interior_ms, edge_ms, wait_ms;
} life_band_stats;
int life_ctx_band_stats(life_ctx* ctx, int32_t band, life_band_stats* out);

/* ---- grid in / out (replaces constructing and reading life::Grid) ------ */
/* Replaces `Grid` + `Grid::data()` writes (grid.hpp:29-35, :56-57).
 * `row_stride` >= width bytes between host rows. */
int life_grid_upload_u8(life_ctx* ctx, const uint8_t* cells, int64_t width, int64_t height,
                        int64_t row_stride);
int life_grid_upload_packed(life_ctx* ctx, const uint64_t* words, int64_t width,
                            int64_t height, int64_t words_per_row);
/* Replaces random_fill (pattern.cpp:330-342): identical grid, generated on the
 * device from the counter form of the splitmix64 stream.
 * `engine` selects the resident layout. */
int life_grid_init_random(life_ctx* ctx, int64_t width, int64_t height, double density,
                          uint64_t seed, int engine);
/* Config-4 sparse soup (the reference has no generator, it is
 * pinned from SplitMix64 + place_pattern, pattern.cpp:309-328) generated on the
 * device: an empty W x H field, B = llround(coverage*W*H/bs^2) bs x bs blocks
 * of Bernoulli(density) cells at seeded positions, later blocks overwriting
 * earlier ones.  Needs 4*W*H bytes of device scratch during the call. */
int life_grid_init_soup(life_ctx* ctx, int64_t width, int64_t height, double coverage,
                        int32_t block_size, double density, uint64_t seed, int engine);
/* place_pattern (pattern.cpp:309-328) on the resident grid: the pw x ph
 * footprint at (x0, y0) is overwritten by `pattern` (row-major bytes,
 * nonzero = alive); LIFE_ERR_OUT_OF_BOUNDS if it does not fit (no wrap). */
int life_grid_place_u8(life_ctx* ctx, const uint8_t* pattern, int64_t pw, int64_t ph,
                       int64_t x0, int64_t y0);
/* Replaces reading `Grid::data()` of RunResult::grid (engine.hpp:24-27). */
int life_grid_download_u8(life_ctx* ctx, uint8_t* cells, int64_t row_stride);
int life_grid_download_packed(life_ctx* ctx, uint64_t* words, int64_t words_per_row);
/* Toroidally wrapped w x h window at (x0, y0) (Grid::wrap, grid.hpp:48-54),
 * as 0/1 bytes; for light-cone parity checks of grids too big to download. */
int life_grid_window_u8(life_ctx* ctx, int64_t x0, int64_t y0, int64_t w, int64_t h,
                        uint8_t* out);
int life_grid_dims(life_ctx* ctx, int64_t* width, int64_t* height);
/* Replaces population (grid.cpp:40-46), widened to uint64. */
int life_population(life_ctx* ctx, uint64_t* out);
/* Full-grid checksum for parity checks of grids too big to download (SURVEY
 * 8(b) `grid_hash`): FNV-1a-64 over the H row hashes (8 little-endian bytes
 * each), row hash = FNV-1a-64 over the row's ceil(W/64) packed uint64 words
 * (little-endian bytes, tail bits zero).  Rows hash in parallel on the device. */
int life_grid_hash(life_ctx* ctx, uint64_t* out);

/* ---- the step loop ------------------------------------------------------ */
/* Replaces run(Grid&&, RunConfig, checkpoints) (engine.cpp:162-214):
 *   `generations` >= 0 (ConfigError otherwise, engine.cpp:133-136);
 *   `temporal_depth`: generations per kernel pass, 0 = auto (the
 *     cluster-resident engine for small tori; the quad / pair layout kernels
 *     for W % 128 / 64 == 0 tori of 2^29 / 2^27 cells or more, life_interleave_auto;
 *     else life_packed_auto_depth); packed 1..16,
 *     byte 1..8 (W % 16 == 0 or W >= 33; narrower tori run one generation per pass);
 *   `checkpoints`: strictly ascending in [0, generations] (engine.cpp:137-147);
 *     `populations[i]` receives the population after checkpoints[i]
 *     generations (checkpoint 0 = the initial grid, engine.cpp:186).
 * The grid stays resident in the context after the call. */
int life_run(life_ctx* ctx, int64_t generations, int engine, int temporal_depth,
             const int64_t* checkpoints, int32_t n_checkpoints, uint64_t* populations);
/* Replaces step_parallel (engine.cpp:152-155): run(..., iterations = 1). */
int life_step(life_ctx* ctx, int engine);
/* Throughput form of run() for a stream of independent packed grids (same
 * W x H; the reference's time_run repetitions, bench.cpp:101-107): each of the
 * `n` host grids inputs[i] is uploaded, run for `generations` on the packed
 * engine and downloaded to outputs[i] (may alias inputs[i]).  The H2D copy of
 * grid i+1 and the D2H copy of grid i-1 overlap the compute of grid i (copy
 * engines); tall grids run their first and last grid as 32 row-chunk
 * trapezoids plus boundary triangles so those copies overlap compute too;
 * temporal_depth 0 on a small W % 32 == 0 torus runs each grid on the
 * cluster-resident engine (one launch per grid).
 * Use pinned host memory for the overlap.
 * *elapsed_ms (optional) = CUDA-event time from the first upload to the last
 * download.  The context's resident grid is not touched. */
int life_run_batch(life_ctx* ctx, const uint64_t* const* inputs, uint64_t* const* outputs,
                   int32_t n, int64_t width, int64_t height, int64_t words_per_row,
                   int64_t generations, int temporal_depth, float* elapsed_ms);

/* The depth life_run uses for temporal_depth 0 on the multi-pass packed
 * engine (16; 12 for W % 32 != 0 tori less than ~3 block waves deep). */
int life_packed_auto_depth(int64_t width, int64_t height);

/* The interleaved layout life_run / life_run_batch pick for a W x H packed
 * torus (or a row band of it), given a context's LIFE_OPT_PAIR_DEPTH and
 * LIFE_OPT_QUAD_DEPTH values (-1 = the defaults) and the call's
 * temporal_depth: returns the interleave order -- 4 = the quad layout
 * (packed_il_kernel<K, 4>: W % 128 == 0, 9.5 integer ops per 32 cell-updates,
 * K <= 7), 2 = the pair layout (packed_il_kernel<K, 2>: W % 64 == 0, 10 ops,
 * K <= 12), 0 = the plain-layout kernels (11 ops) -- and writes the pass depth
 * to *depth (0 with order 0: life_packed_auto_depth applies).  With both
 * options at -1 and temporal_depth 0, tori of 2^27 cells or more run the
 * layout that keeps most lanes per integer op busy at their width (strips of
 * 32 groups advancing by 31): quad (2^29 cells or more) at K = 7 / 6 for wide
 * tori (W >= 49152 or so), pair at K = 10 for 12288..32768 columns, the plain
 * kernels below and for narrower or smaller tori; an
 * explicit temporal_depth keeps the plain kernels unless an option forces a
 * layout. */
int life_interleave_auto(int64_t width, int64_t height, int32_t pair_option, int32_t quad_option,
                         int32_t temporal_depth, int32_t* depth);

/* Which kernel(s) one torus pass of `generations` over `out_rows` rows of a
 * W-wide packed grid launches (device-buffer layer and life_run alike):
 * LIFE_LAUNCH_STEP1 packed_step1_kernel (one generation, W % 128 == 0, 16-B
 * vectors); LIFE_LAUNCH_FAST packed_tb_fast_kernel<K> (W % 32 == 0, K >= 4);
 * LIFE_LAUNCH_ALL_PATHS packed_tb_kernel<K>; LIFE_LAUNCH_SPLIT the seam strips
 * on packed_tb_kernel<K> beside packed_tb_fast_kernel<K> for the rest (W % 32
 * != 0 tori several block waves deep); -1 for a bad argument. */
#define LIFE_LAUNCH_STEP1 0
#define LIFE_LAUNCH_FAST 1
#define LIFE_LAUNCH_ALL_PATHS 2
#define LIFE_LAUNCH_SPLIT 3
int life_packed_launch_kind(int64_t width, int64_t out_rows, int32_t generations);

/* ---- row-band decomposition (multi-GPU) --------------------------------- */
/* Mirrors band_bounds / partition_rows (decomposition.cpp:12-24, :93-104):
 * writes parts+1 cut points; LIFE_ERR_TOO_MANY_PARTS if parts > extent. */
int life_band_bounds(int64_t extent, int32_t parts, int64_t* bounds);

/* ---- device-buffer layer (plain device pointers; used by the multi-GPU
 *      band driver, which owns its buffers and streams) ------------------- */
/* Device row pitch, in uint32 words, of the packed layout for width W
 * (>= 2*ceil(W/64), a multiple of 32 words = 128 B). */
int64_t life_packed_pitch_words(int64_t width);
/* Byte layout pitch (>= W, a multiple of 128 B; W % 16 != 0 rows keep 48
 * bytes of padding after the last 16-byte vector, see life_dev_byte_pass). */
int64_t life_byte_pitch(int64_t width);
/* `generations` (1..16) packed generations in one pass (W % 32 != 0 tori
 * several block waves deep run their seam strips on a library-owned side
 * stream per host thread and device, joined back into `stream`).  Output relative row
 * r (0 <= r < out_rows) is stored at out + (out_row0 + r) * out_pitch; input
 * relative row r (-generations <= r < out_rows + generations) is read from
 * physical row (in_row0 + r) mod in_rows of `in`.  The torus is the case
 * in_rows = H, in_row0 = out_row0 = 0; a band with k ghost rows above it is
 * in_row0 = k.  `in` and `out` must not overlap. */
int life_dev_packed_step(const uint32_t* in, int64_t in_pitch, int64_t in_row0,
                         int64_t in_rows, uint32_t* out, int64_t out_pitch, int64_t out_row0,
                         int64_t width, int64_t out_rows, int32_t generations, void* stream);
/* `generations` of a W x H packed torus (rows of `pitch` words) ping-ponging
 * between buf_a (holding the input) and buf_b, `depth` (1..16) generations
 * per pass (one life_dev_packed_step launch each, then the remainder): the
 * result is in buf_b if *result_in_b = 1, else in buf_a.  (A persistent
 * single-launch form with per-tile neighbour flags between passes was
 * measured 11-23 % slower on one-wave tori and is not used.) */
int life_dev_packed_run(uint32_t* buf_a, uint32_t* buf_b, int64_t pitch, int64_t width,
                        int64_t height, int64_t generations, int32_t depth, int32_t* result_in_b,
                        void* stream);
/* The same pass for one row band of a torus split across GPUs, with the
 * halo read IN the kernel over NVLink: input rows above the band come from
 * `up` (the last rows of the band above, up_rows tall -- a peer GPU's buffer
 * opened with life_ipc_open), rows below from `down` (the first rows of the
 * band below).  Band rows [out_row0, out_row0+out_rows) are written to the
 * same rows of `out`.  All buffers use `pitch`.  The caller orders passes
 * across GPUs (a barrier per pass: the neighbours must have finished writing
 * `up`/`down` and reading the buffer this pass overwrites).  Bands must be
 * >= `generations` rows. */
int life_dev_packed_step_peer(const uint32_t* in, const uint32_t* up, int64_t up_rows,
                              const uint32_t* down, int64_t down_rows, int64_t pitch,
                              int64_t band_rows, uint32_t* out, int64_t out_row0,
                              int64_t out_rows, int64_t width, int32_t generations,
                              void* stream);
/* ---- interleaved layouts at the device-buffer layer: `order` 2 = the pair
 * layout (W % 64 == 0: each uint64 group of a packed row kept as even columns
 * | odd columns), 4 = the quad layout (W % 128 == 0: 128-column groups as
 * four words, word r bit j = column 4j + r), the layouts packed_il_kernel<K,
 * N> steps at 10 / 9.5 integer ops per 32 cell-updates.  life_dev_packed_zip
 * converts rows [row0, row0 + rows) in place (to_interleaved 1: plain ->
 * interleaved, 0: back).  The _il step / run / step_peer calls are
 * life_dev_packed_step / _run / _step_peer on buffers in that layout,
 * `generations` / `depth` in 1..12 (pair) or 1..7 (quad).  Populations
 * (popcounts) are layout-independent; everything else reads the plain layout. */
int life_dev_packed_zip(uint32_t* words, int64_t pitch, int64_t width, int64_t row0, int64_t rows,
                        int32_t order, int32_t to_interleaved, void* stream);
int life_dev_packed_step_il(int32_t order, const uint32_t* in, int64_t in_pitch, int64_t in_row0,
                            int64_t in_rows, uint32_t* out, int64_t out_pitch, int64_t out_row0,
                            int64_t width, int64_t out_rows, int32_t generations, void* stream);
int life_dev_packed_run_il(int32_t order, uint32_t* buf_a, uint32_t* buf_b, int64_t pitch,
                           int64_t width, int64_t height, int64_t generations, int32_t depth,
                           int32_t* result_in_b, void* stream);
int life_dev_packed_step_il_peer(int32_t order, const uint32_t* in, const uint32_t* up,
                                 int64_t up_rows, const uint32_t* down, int64_t down_rows,
                                 int64_t pitch, int64_t band_rows, uint32_t* out, int64_t out_row0,
                                 int64_t out_rows, int64_t width, int32_t generations,
                                 void* stream);
/* `generations` packed generations of a whole W x H torus (rows of `pitch`
 * words, in == out allowed) through the cluster-resident engine
 * (LIFE_ENGINE_RESIDENT), one launch per 2^30 generations. */
int life_dev_packed_run_resident(const uint32_t* in, uint32_t* out, int64_t pitch,
                                 int64_t width, int64_t height, int64_t generations,
                                 void* stream);
/* CTAs per cluster the resident engine would use for a W x H torus on the
 * current device; 0 if the torus does not fit it. */
int life_resident_cluster_size(int64_t width, int64_t height);
/* Device buffers shareable across processes (cudaMalloc, zeroed) and CUDA
 * IPC: a 64-byte handle per buffer, opened in the peer process. */
int life_dev_alloc(int64_t bytes, void** out);
int life_dev_free(void* dev_ptr);
int life_ipc_get_handle(void* dev_ptr, void* handle_out);
int life_ipc_open(const void* handle, void** out);
int life_ipc_close(void* dev_ptr);
/* Pass ordering between neighbouring bands without a kernel: a 32-bit flag in
 * a life_dev_alloc'd buffer (the band's own, or a neighbour's opened with
 * life_ipc_open) written / awaited by stream memory operations
 * (cuStreamWriteValue32 / cuStreamWaitValue32, >= comparison), ordered on
 * `stream` like a kernel but using no SM.  The cross-device form of the
 * reference's per-generation barrier (WorkerTeam, engine.cpp:79-96), narrowed
 * to the two bands a band touches.  LIFE_ERR_CUDA if the driver lacks them. */
int life_dev_flag_write(void* flag, uint32_t value, void* stream);
int life_dev_flag_wait_geq(void* flag, uint32_t value, void* stream);
/* One byte-engine generation with the same row addressing (pitches in bytes). */
int life_dev_byte_step(const uint8_t* in, int64_t in_pitch, int64_t in_row0, int64_t in_rows,
                       uint8_t* out, int64_t out_pitch, int64_t out_row0, int64_t width,
                       int64_t out_rows, void* stream);
/* `generations` (1..8) byte-engine generations in one pass (temporal blocking;
 * more than one needs W % 16 == 0 or W >= 33), same addressing as life_dev_byte_step;
 * for W % 16 != 0 the 48 bytes after each input row's last vector (in_pitch >=
 * life_byte_pitch(W)) are overwritten with the row's seam vectors;
 * input relative rows -generations .. out_rows + generations are read. */
int life_dev_byte_pass(const uint8_t* in, int64_t in_pitch, int64_t in_row0, int64_t in_rows,
                       uint8_t* out, int64_t out_pitch, int64_t out_row0, int64_t width,
                       int64_t out_rows, int32_t generations, void* stream);
/* Rows [y0, y0+rows) of random_fill(W, H, density, seed) into a packed buffer. */
int life_dev_packed_random(uint32_t* out, int64_t pitch, int64_t width, int64_t y0,
                           int64_t rows, double density, uint64_t seed, void* stream);
/* The same rows of the soup in the byte layout (pitch a multiple of 16). */
int life_dev_byte_random(uint8_t* out, int64_t pitch, int64_t width, int64_t y0, int64_t rows,
                         double density, uint64_t seed, void* stream);
/* Adds the population of `rows` packed rows to *dev_count (device uint64). */
int life_dev_packed_population(const uint32_t* grid, int64_t pitch, int64_t width,
                               int64_t rows, uint64_t* dev_count, void* stream);
/* Row hashes of life_grid_hash for `rows` packed rows (into device memory);
 * chain them on the host with life_fnv1a64 (bands: concatenate in row order). */
int life_dev_packed_row_hashes(const uint32_t* grid, int64_t pitch, int64_t width,
                               int64_t rows, uint64_t* dev_hashes, void* stream);
/* FNV-1a-64 (offset 0xcbf29ce484222325, prime 0x100000001b3) of n host bytes,
 * continuing from h (0 = start). */
uint64_t life_fnv1a64(const void* bytes, int64_t n, uint64_t h);
/* Packs byte rows (nonzero -> 1) into packed rows and back. */
int life_dev_pack(const uint8_t* cells, int64_t cell_pitch, uint32_t* words, int64_t pitch,
                  int64_t width, int64_t rows, void* stream);
int life_dev_unpack(const uint32_t* words, int64_t pitch, uint8_t* cells, int64_t cell_pitch,
                    int64_t width, int64_t rows, void* stream);

/* ---- measurement helpers ------------------------------------------------ */
/* Integer-pipe peak: runs a LOP3 throughput kernel for ~`iters` dependent
 * steps on every SM and returns lane-ops per second in *ops_per_s. */
int life_measure_int_peak(int device, int64_t iters, double* ops_per_s, double* seconds);
/* Number of kernel launches issued by this library in this process. */
uint64_t life_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* LIFE_GPU_H */
