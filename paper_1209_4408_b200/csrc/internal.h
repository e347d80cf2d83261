// internal.h -- internals shared by the C-ABI translation units (life_gpu.cu:
// device layer + single-device contexts; life_multi.cu: multi-device
// contexts).  Not part of the installed interface (include/life_gpu.h is).
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/life_gpu.h"

namespace lifegpu {
namespace detail {

// ---- errors (thread-local message, status code returned) -------------------
int set_error(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);
void count_launch();  // life_kernel_launches() bookkeeping

#define LIFE_CUDA(call)                                                         \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess) return ::lifegpu::detail::cuda_fail(e_, #call);      \
  } while (0)

#define LIFE_CHECK_LAUNCH(name)                                                 \
  do {                                                                          \
    ::lifegpu::detail::count_launch();                                          \
    cudaError_t e_ = cudaGetLastError();                                        \
    if (e_ != cudaSuccess) return ::lifegpu::detail::cuda_fail(e_, "launch " name); \
  } while (0)

#define LIFE_TRY(expr)              \
  do {                              \
    int rc_ = (expr);               \
    if (rc_ != LIFE_OK) return rc_; \
  } while (0)

// Measurement knobs read from the environment exist only in LIFE_DEBUG_KNOBS
// builds (tools/ sweeps); the shipped library's launch schedule never
// depends on the environment and returns `dflt`.
int64_t knob(const char* name, int64_t dflt);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t nw32(int64_t width) { return ceil_div(width, 32); }
inline uint32_t tail_mask(int64_t width) {
  const int r = static_cast<int>(width & 31);
  return r == 0 ? 0xffffffffu : ((1u << r) - 1u);
}
int check_dims(int64_t width, int64_t height);
int sm_count();
int grid_stride_blocks(int64_t n, int threads);

// First-use launch parameters per device (occupancy etc.).  Several host
// threads may race on the first call: each computes the same value, sets the
// kernel attributes it needs, and publishes with release order; readers
// acquire, so a nonzero value implies the attributes are in place.
class DeviceCache {
 public:
  int get(int dev) const { return v_[dev & 63].load(std::memory_order_acquire); }
  void put(int dev, int x) { v_[dev & 63].store(x, std::memory_order_release); }

 private:
  std::atomic<int> v_[64]{};
};

// Side stream + fork/join events for split packed launches (the seam strips
// of W % 32 != 0 tori run beside the fast-only strips).  Owned by a context
// (one per stream it launches on) and destroyed with it.
struct SplitStreams {
  int device = -1;
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
int split_streams_init(SplitStreams* ss, int device);
void split_streams_destroy(SplitStreams* ss);

// life_dev_packed_step with the caller's side stream (nullptr: a per-thread,
// per-device library stream).
int packed_step(const uint32_t* in, int64_t in_pitch, int64_t in_row0, int64_t in_rows,
                uint32_t* out, int64_t out_pitch, int64_t out_row0, int64_t width,
                int64_t out_rows, int32_t generations, cudaStream_t stream, SplitStreams* ss);
// temporal_depth 0 on the multi-pass packed engine (exported as
// life_packed_auto_depth).
int packed_auto_depth(int64_t width, int64_t height);
// `generations` of a packed torus ping-ponging between buf_a (input) and
// buf_b: whole passes of `depth`, then the remainder; *result_in_b = 1 if the result is in buf_b.
int packed_run(uint32_t* buf_a, uint32_t* buf_b, int64_t pitch, int64_t width, int64_t height,
               int64_t generations, int32_t depth, cudaStream_t stream, SplitStreams* ss,
               int* result_in_b, int il = 0);

// ---- interleaved layouts (life_pair.cu, kernels_pair.cuh) -------------------
// Order 2, the PAIR layout (W % 64 == 0): each uint64 group of a packed row
// kept as (even columns, odd columns); passes of up to 12 generations at 10
// instead of 11 integer ops per 32 cell-updates.  Order 4, the QUAD layout
// (W % 128 == 0): 128-column groups as four words of every 4th column; up to
// 6 generations per pass at 9.5 ops.  Order 0 = the plain layout.
// packed_zip converts rows in place.
constexpr int kPairMaxDepthHost = 12;
constexpr int kQuadMaxDepthHost = 7;
inline bool il_eligible(int il, int64_t width) {
  return (il == 2 || il == 4) && width >= 32 * il && width % (32 * il) == 0;
}
inline int il_max_depth(int il) {
  return il == 4 ? kQuadMaxDepthHost : il == 2 ? kPairMaxDepthHost : LIFE_MAX_TEMPORAL_DEPTH;
}
int packed_il_step(int il, const uint32_t* in, int64_t in_pitch, int64_t in_row0, int64_t in_rows,
                   uint32_t* out, int64_t out_pitch, int64_t out_row0, int64_t width,
                   int64_t out_rows, int32_t generations, cudaStream_t stream);
int packed_il_step_peer(int il, const uint32_t* in, const uint32_t* up, int64_t up_rows,
                        const uint32_t* down, int64_t down_rows, int64_t pitch,
                        int64_t band_rows, uint32_t* out, int64_t out_row0, int64_t out_rows,
                        int64_t width, int32_t generations, cudaStream_t stream);
int packed_zip(int il, uint32_t* words, int64_t pitch, int64_t width, int64_t row0, int64_t rows,
               bool unzip, cudaStream_t stream);
// The layout and depth a run uses on a W-wide torus (or band) of `height`
// rows: a forced LIFE_OPT_QUAD_DEPTH / LIFE_OPT_PAIR_DEPTH (> 0) where the
// width allows it; else, when the caller left the depth to the engine
// (temporal_depth 0), the auto rule over the layouts whose option is -1
// (exported as life_interleave_auto); else order 0 (the plain kernels at
// temporal_depth or packed_auto_depth).
struct IlChoice {
  int il = 0;
  int depth = 0;
};
IlChoice il_choose(int64_t width, int64_t height, int pair_opt, int quad_opt, int temporal_depth);

// Small kernels the multi-device context launches on band buffers.
int launch_mask_tail(uint32_t* words, int64_t pitch, int64_t width, int64_t rows,
                     cudaStream_t s);
int launch_place_packed(uint32_t* words, int64_t pitch, const uint8_t* dev_pattern, int64_t pw,
                        int64_t ph, int64_t x0, int64_t y0, cudaStream_t s);
int launch_window_packed(const uint32_t* words, int64_t pitch, int64_t width, int64_t height,
                         int64_t x0, int64_t y0, int64_t w, int64_t h, uint8_t* dev_out,
                         cudaStream_t s);

// ---- multi-device contexts (life_multi.cu) ---------------------------------
struct MultiState;
int multi_create(int32_t n, const int* devices, MultiState** out);
void multi_destroy(MultiState* m);
int multi_sync(MultiState* m);
int multi_set_option(MultiState* m, int option, int64_t value);
int multi_get_option(MultiState* m, int option, int64_t* value);
int multi_dims(MultiState* m, int64_t* w, int64_t* h);
int multi_upload_u8(MultiState* m, const uint8_t* cells, int64_t w, int64_t h, int64_t stride);
int multi_upload_packed(MultiState* m, const uint64_t* words, int64_t w, int64_t h, int64_t wpr);
int multi_init_random(MultiState* m, int64_t w, int64_t h, double density, uint64_t seed);
int multi_init_soup(MultiState* m, int64_t w, int64_t h, double coverage, int32_t bs,
                    double density, uint64_t seed);
int multi_place_u8(MultiState* m, const uint8_t* pattern, int64_t pw, int64_t ph, int64_t x0,
                   int64_t y0);
int multi_download_u8(MultiState* m, uint8_t* cells, int64_t stride);
int multi_download_packed(MultiState* m, uint64_t* words, int64_t wpr);
int multi_window_u8(MultiState* m, int64_t x0, int64_t y0, int64_t w, int64_t h, uint8_t* out);
int multi_population(MultiState* m, uint64_t* out);
int multi_hash(MultiState* m, uint64_t* out);
int multi_run(MultiState* m, int64_t generations, int engine, int temporal_depth,
              const int64_t* checkpoints, int32_t n_checkpoints, uint64_t* populations);
int multi_run_batch(MultiState* m, const uint64_t* const* inputs, uint64_t* const* outputs,
                    int32_t n, int64_t width, int64_t height, int64_t words_per_row,
                    int64_t generations, int temporal_depth, float* elapsed_ms);
int multi_bands(MultiState* m, int32_t* n, int64_t* bounds, int32_t* devices, int32_t* halo);
int multi_band_stats(MultiState* m, int32_t band, life_band_stats* out);

// Rule for checkpoints and run arguments shared by both context kinds
// (check_run_config, engine.cpp:127-148).
int check_run_args(int64_t generations, const int64_t* checkpoints, int32_t n_checkpoints,
                   const uint64_t* populations);

}  // namespace detail
}  // namespace lifegpu
