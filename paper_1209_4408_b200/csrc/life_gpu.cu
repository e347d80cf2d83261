// life_gpu.cu -- C-ABI implementation (include/life_gpu.h): contexts, the
// generation-step loop, layout conversion and the device-buffer layer.
//
// Build: paper_1209_4408_b200/build.py (nvcc -gencode arch=compute_100a,code=sm_100a).
// There is no CPU fallback anywhere in this file: every entry point that
// computes launches a kernel in kernels.cuh or fails with a status code.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/life_gpu.h"
#include "internal.h"
#include "kernels.cuh"

using namespace lifegpu;
using namespace lifegpu::detail;

namespace {
thread_local std::string g_error;
std::atomic<uint64_t> g_launches{0};
std::atomic<void*> g_trace{nullptr};  // device buffer for LIFE_TRACE builds (life_debug_set_trace)
}  // namespace

namespace lifegpu {
namespace detail {

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_error = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation)
    return set_error(LIFE_ERR_OUT_OF_MEMORY, "%s: %s", what, cudaGetErrorString(e));
  return set_error(LIFE_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int64_t knob(const char* name, int64_t dflt) {
#ifdef LIFE_DEBUG_KNOBS
  const char* e = std::getenv(name);
  return e ? std::atoll(e) : dflt;
#else
  (void)name;
  return dflt;
#endif
}

int sm_count() {
  static DeviceCache cache;
  int dev = 0;
  cudaGetDevice(&dev);
  int n = cache.get(dev);
  if (n == 0) {
    n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache.put(dev, n);
  }
  return n;
}

int grid_stride_blocks(int64_t n, int threads) {
  const int64_t want = ceil_div(std::max<int64_t>(n, 1), threads);
  return static_cast<int>(std::min<int64_t>(want, static_cast<int64_t>(sm_count()) * 16));
}

int check_dims(int64_t width, int64_t height) {
  if (width < 3 || height < 3)
    return set_error(LIFE_ERR_DIMENSION_TOO_SMALL,
                     "grid dimensions must be at least 3x3, got %lldx%lld",
                     static_cast<long long>(width), static_cast<long long>(height));
  if (width > (int64_t(1) << 40) || height > (int64_t(1) << 40))
    return set_error(LIFE_ERR_CONFIG, "grid dimensions too large");
  return LIFE_OK;
}

int check_run_args(int64_t generations, const int64_t* checkpoints, int32_t n_checkpoints,
                   const uint64_t* populations) {
  // check_run_config (engine.cpp:127-148)
  if (generations < 0)
    return set_error(LIFE_ERR_CONFIG, "iteration count must be non-negative, got %lld",
                     static_cast<long long>(generations));
  if (n_checkpoints < 0 || (n_checkpoints > 0 && (!checkpoints || !populations)))
    return set_error(LIFE_ERR_CONFIG, "bad checkpoint buffers");
  int64_t prev = -1;
  for (int32_t i = 0; i < n_checkpoints; ++i) {
    const int64_t cp = checkpoints[i];
    if (cp < 0 || cp > generations)
      return set_error(LIFE_ERR_CONFIG, "checkpoint %lld is outside [0, iterations=%lld]",
                       static_cast<long long>(cp), static_cast<long long>(generations));
    if (cp <= prev) return set_error(LIFE_ERR_CONFIG, "checkpoints must be strictly ascending");
    prev = cp;
  }
  return LIFE_OK;
}

int split_streams_init(SplitStreams* ss, int device) {
  if (ss->side && ss->device == device) return LIFE_OK;
  split_streams_destroy(ss);
  LIFE_CUDA(cudaStreamCreateWithFlags(&ss->side, cudaStreamNonBlocking));
  LIFE_CUDA(cudaEventCreateWithFlags(&ss->fork, cudaEventDisableTiming));
  LIFE_CUDA(cudaEventCreateWithFlags(&ss->join, cudaEventDisableTiming));
  ss->device = device;
  return LIFE_OK;
}

void split_streams_destroy(SplitStreams* ss) {
  if (ss->side) cudaStreamDestroy(ss->side);
  if (ss->fork) cudaEventDestroy(ss->fork);
  if (ss->join) cudaEventDestroy(ss->join);
  *ss = SplitStreams{};
}

}  // namespace detail
}  // namespace lifegpu

namespace {

uint64_t density_threshold(double density) {
  return static_cast<uint64_t>(std::ceil(density * 0x1.0p53));
}

// ---- packed temporal-blocked step: template dispatch on K ----------------
#ifndef LIFE_SYNC_TRIPS
#define LIFE_SYNC_TRIPS 48
#endif
constexpr int kSyncTrips = LIFE_SYNC_TRIPS;

// Programmatic dependent launch (PDL): consecutive passes on a stream
// overlap the next grid's launch with this one's tail; the kernels wait on
// griddepcontrol.wait before their first read (LIFE_PDL=0 in LIFE_DEBUG_KNOBS
// builds disables it).  Measured with packed_tb_kernel<16> (T/s, 320
// generations): 4096^2 9.45 -> 10.0, 8192^2 23.1 -> 23.9, 16384^2 36.1 ->
// 36.7, 65536^2 unchanged.
bool pdl_enabled() {
  static const bool pdl = knob("LIFE_PDL", 1) != 0;
  return pdl;
}

template <typename Kernel, typename Args>
int launch_pdl(Kernel kernel, unsigned blocks, unsigned threads, size_t smem, cudaStream_t s,
               const Args& args) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  LIFE_CUDA(cudaLaunchKernelEx(&cfg, kernel, args));
  return LIFE_OK;
}

// LIFE_SPLIT=0 (debug builds): W % 32 != 0 tori run every strip in the
// all-paths kernel.
bool split_disabled() {
  static const bool v = knob("LIFE_SPLIT", 1) == 0;
  return v;
}

// Block barrier interval of peer-mode (edge strip) launches (one per loop
// trip; LIFE_PEER_SYNC in debug builds, 0 = none).
int peer_sync_trips() {
  static const int v = static_cast<int>(std::max<int64_t>(knob("LIFE_PEER_SYNC", 1), 0));
  return v;
}

// Tiles up to this many rows run the fast kernel's single-loop-body variant.
constexpr int64_t kUniMaxRows = kShortTileRows;  // tiles up to this many rows: the single-loop-body variant
// One-wave fast-kernel tiles shorter than this run at half the warps per SM.
constexpr int64_t kShortTileRows = 128;

template <int K, bool FAST>
int launch_packed_kernel(PackedStepArgs a, cudaStream_t s) {
  const auto kernel = FAST ? packed_tb_fast_kernel<K> : packed_tb_kernel<K>;
  constexpr int kRing = FAST ? PackedTraits<K>::kRingBytesFast : PackedTraits<K>::kRingBytes;
  constexpr int kMaxWarps = (FAST ? PackedTraits<K>::kMaxThreadsFast : PackedTraits<K>::kMaxThreads) / 32;
  // Per device: warps per block = every warp one SM holds (register-limited),
  // one block per SM, so the block barrier keeps all of an SM's warps in
  // lockstep (LIFE_NO_LOCKSTEP builds use 4-warp blocks instead).
  static DeviceCache warps_per_block;  // per instantiation
  int dev = 0;
  cudaGetDevice(&dev);
  int wpb = warps_per_block.get(dev);
  if (wpb == 0) {
    LIFE_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kMaxWarps * kRing));
    if (FAST)
      LIFE_CUDA(cudaFuncSetAttribute(packed_tb_fast_kernel<K, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kMaxWarps * kRing));
    int nb = 0;
    LIFE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kPackedThreads, 4 * kRing));
    int w = std::min(std::max(nb, 1) * (kPackedThreads / 32), kMaxWarps);
#ifdef LIFE_NO_LOCKSTEP
    w = kPackedThreads / 32;
#else
    for (; w > 1; --w) {
      int nb2 = 0;
      LIFE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb2, kernel, 32 * w, w * kRing));
      if (nb2 >= 1) break;
    }
#endif
    // The fast-only kernel has no block barrier: LIFE_FAST_WPB (debug builds)
    // sets its warps per block (several blocks per SM), for measurement.
    const int64_t forced = knob(FAST ? "LIFE_FAST_WPB" : "LIFE_WPB", 0);
    if (forced > 0) w = std::min(static_cast<int>(forced), w);
    wpb = w;
    warps_per_block.put(dev, wpb);
  }
  int blocks_per_sm = 1;
#ifdef LIFE_NO_LOCKSTEP
  LIFE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kernel, 32 * wpb,
                                                          wpb * kRing));
#else
  if (FAST) {
    LIFE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kernel, 32 * wpb,
                                                            wpb * kRing));
    // LIFE_FAST_BPS (debug builds): blocks per SM the segment model plans for.
    static const int64_t bps = knob("LIFE_FAST_BPS", 0);
    if (bps > 0) blocks_per_sm = static_cast<int>(bps);
  }
#endif
  // Tiles of seg_rows rows x one strip; pick the segment count that
  // minimises (block waves) x (rows per tile + pipeline fill): blocks run
  // in lockstep internally, and the last wave's idle SMs are the loss.
  constexpr int kLag = PackedTraits<K>::kLag;
  constexpr int PF = FAST ? PackedTraits<K>::kPrefetchFast : PackedTraits<K>::kPrefetch;
  if (a.out_rows >= (int64_t(1) << 31) || a.in_rows >= (int64_t(1) << 31) ||
      a.in_pitch * 4 >= (int64_t(1) << 32) || a.out_pitch * 4 >= (int64_t(1) << 32))
    return set_error(LIFE_ERR_CONFIG, "grid too large for one packed pass");
  const int64_t slots = static_cast<int64_t>(blocks_per_sm) * sm_count();  // blocks per wave
  int64_t best_segs = 1;
  double best_cost = 1e300;
  // Segments down to 8 rows: small grids (less than a wave of tiles) trade
  // pipeline-fill work for parallelism -- 1024^2 1.9x, 4096^2 1.6x faster
  // than a 4K-row floor; large grids pick long segments anyway.
  constexpr int kMinSegRows = 8;
  const int64_t max_segs =
      std::max<int64_t>(1, std::min<int64_t>(a.out_rows / kMinSegRows + 1, 4096));
  for (int64_t segs = 1; segs <= max_segs; ++segs) {
    const int64_t rows = ceil_div(a.out_rows, segs);
    const int64_t blocks = ceil_div(static_cast<int64_t>(a.n_strips) * ceil_div(a.out_rows, rows), wpb);
    // Per wave: the tile's pipeline fill and block start-up, calibrated on
    // LIFE_SEGS sweeps: + 48 rows (round 1: + 64)
    // moves config 3 from one wave of 1139 tiles at 96 % occupancy to two
    // waves of 2345 (44.6 -> 45.3 T/s) and keeps config 5's 7-wave plan; a
    // lighter charge (kLag / 2 + PF + 8) also re-planned config 5's passes
    // and cost its copy-overlapped e2e 2 % (45.2 -> 44.2).
    const double cost = double(ceil_div(blocks, slots)) * double(rows + kLag + PF + 48);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best_segs = segs;
    }
  }
  static const int64_t forced_segs = knob("LIFE_SEGS", 0);  // debug builds: force the segment count
  if (forced_segs > 0) best_segs = std::min<int64_t>(forced_segs, a.out_rows);
  a.seg_rows = ceil_div(a.out_rows, best_segs);
  // Very short one-wave tiles (< kShortTileRows rows at a full SM of warps):
  // half the warps per SM, each tile twice as tall -- one warp of K
  // independent stage chains per SMSP still fills its ALU pipe, and the
  // pipeline fill is paid on twice as many rows (8192^2 at K = 16: 23.4 ->
  // 24.9 T/s; 16384^2, 238-row tiles, loses 5 % that way and keeps 8).
  if (FAST && forced_segs == 0 && wpb >= 8 && blocks_per_sm == 1 && a.seg_rows < kShortTileRows &&
      static_cast<int64_t>(a.n_strips) * ceil_div(a.out_rows, a.seg_rows) <= slots * wpb) {
    const int64_t half = wpb / 2;
    const int64_t segs2 = std::max<int64_t>(1, (slots * half) / a.n_strips);  // one wave, 1 block/SM
    const int64_t rows2 = ceil_div(a.out_rows, segs2);
    if (rows2 > a.seg_rows) {
      wpb = static_cast<int>(half);
      a.seg_rows = rows2;
    }
  }
  const int64_t tiles = static_cast<int64_t>(a.n_strips) * ceil_div(a.out_rows, a.seg_rows);
  a.steps = static_cast<int32_t>(ceil_div(a.seg_rows + kLag, PF));
  // Lockstep granularity: a block barrier every kSyncTrips trips (192 rows).
  // With the 12-op network one every 6 trips was +4 % over one per trip; the
  // 11-op network gains another ~0.8 % from going to 48 (config 5 45.33 ->
  // 45.70 T/s; 24: 45.65, none: 45.75, config 4 best at 48).  Peer-mode edge
  // strips (general fetch path, small launches) keep one per trip; the
  // fast-only kernel has no barrier.
  a.sync_every = FAST ? 0 : (a.peer ? peer_sync_trips() : kSyncTrips);
  const int64_t blocks = ceil_div(tiles, wpb);
  if (blocks > 0x7fffffff) return set_error(LIFE_ERR_CONFIG, "grid too large");
  // Short tiles of the fast kernel run the single-loop-body variant (UNI).
  const auto launch_kernel = (FAST && a.seg_rows <= kUniMaxRows) ? packed_tb_fast_kernel<K, true>
                                                                  : kernel;
  LIFE_TRY(launch_pdl(launch_kernel, static_cast<unsigned>(blocks), 32 * wpb,
                      static_cast<size_t>(wpb) * kRing, s, a));
  LIFE_CHECK_LAUNCH("packed_tb_kernel");
  return LIFE_OK;
}

// Library-owned side stream per (thread, device) for split launches of the
// device-buffer layer (life_dev_packed_step has no context to own one; see
// include/life_gpu.h).  Contexts pass their own SplitStreams instead.
int thread_split_streams(SplitStreams** out) {
  struct PerThread {
    SplitStreams s[64];
    ~PerThread() {
      for (auto& x : s) split_streams_destroy(&x);
    }
  };
  thread_local PerThread per;
  int dev = 0;
  LIFE_CUDA(cudaGetDevice(&dev));
  SplitStreams& ss = per.s[dev & 63];
  LIFE_TRY(split_streams_init(&ss, dev));
  *out = &ss;
  return LIFE_OK;
}

// W % 32 == 0 tori outside peer mode take the fast-only kernel (every warp on
// the fast fetch path, 6 rows per trip, no barrier).  Other widths split the
// strips when the grid is several block waves deep: the two or three strips
// that touch the torus seam (strip 0, which holds word -1, and the strips
// holding words nw-1 and nw) run the all-paths kernel in ONE launch on a side
// stream (strips wrap modulo the strip count), launched first (short tiles:
// one quick wave), and the strips between run the fast-only kernel beside
// and after them: 65535^2 41.5 -> 44.4 T/s, 131071 x 65536 43.3 -> 46.3;
// one-wave grids (config 4, 16383^2) keep the single all-paths launch.
template <int K>
int launch_packed_deep(PackedStepArgs a, cudaStream_t s, SplitStreams* ss) {
  #ifdef LIFE_TIMELINE
  const bool fast_ok = !a.peer && a.width >= 64;  // the fast kernel carries the phase stamps
#else
  const bool fast_ok = !a.peer && a.width >= 64 && !a.trace;
#endif
  if (fast_ok && a.width % 32 == 0) return launch_packed_kernel<K, true>(a, s);
  const int32_t total = a.n_strips;
  // Strip s holds words [31s - 1, 31s + 30]: s_last is the first strip
  // holding word nw-1 (the seam word); strips 1 .. s_last-1 hold only whole
  // words inside [0, nw-1).
  const int32_t s_last = (a.nw - 1) / kStripStride;
  // (life_packed_launch_kind restates this choice for callers.)
  const bool many_waves = static_cast<int64_t>(total) * a.out_rows >= 2000000;  // ~3 waves of 512-row tiles
  if (!fast_ok || a.strip0 != 0 || s_last < 2 || !many_waves || split_disabled())
    return launch_packed_kernel<K, false>(a, s);
  const int32_t n_end = total - s_last;  // seam strips at the end (1 or 2)
  // (Packing a one-wave grid's two launches into its single wave -- fast
  // strips at the single launch's segment length, the seam strips in the
  // blocks left over -- measured 2-10 % slower than one all-paths launch:
  // config 4 37.6 -> 36.5, 4097^2 7.8 -> 7.1.)
  if (!ss) LIFE_TRY(thread_split_streams(&ss));
  LIFE_CUDA(cudaEventRecord(ss->fork, s));
  LIFE_CUDA(cudaStreamWaitEvent(ss->side, ss->fork, 0));
  // One seam launch: strips s_last .. total-1 and (wrapping) strip 0.
  PackedStepArgs seam = a;
  seam.strips_total = total;
  seam.strip0 = s_last;
  seam.n_strips = n_end + 1;
  LIFE_TRY((launch_packed_kernel<K, false>(seam, ss->side)));
  LIFE_CUDA(cudaEventRecord(ss->join, ss->side));
  PackedStepArgs mid = a;
  mid.strip0 = 1;
  mid.n_strips = s_last - 1;
  LIFE_TRY((launch_packed_kernel<K, true>(mid, s)));
  LIFE_CUDA(cudaStreamWaitEvent(s, ss->join, 0));
  return LIFE_OK;
}

template <int K>
int launch_packed(PackedStepArgs a, cudaStream_t s, SplitStreams* ss) {
  if constexpr (K < 4) {  // shallow passes keep the all-paths kernel (no fast-only instance)
    (void)ss;
    return launch_packed_kernel<K, false>(a, s);
  } else {
    return launch_packed_deep<K>(a, s, ss);
  }
}

using PackedLauncher = int (*)(PackedStepArgs, cudaStream_t, SplitStreams*);
const PackedLauncher kPackedLaunchers[LIFE_MAX_TEMPORAL_DEPTH + 1] = {
    nullptr,           launch_packed<1>,  launch_packed<2>,  launch_packed<3>,
    launch_packed<4>,  launch_packed<5>,  launch_packed<6>,  launch_packed<7>,
    launch_packed<8>,  launch_packed<9>,  launch_packed<10>, launch_packed<11>,
    launch_packed<12>, launch_packed<13>, launch_packed<14>, launch_packed<15>,
    launch_packed<16>};

}  // namespace

// ===========================================================================
// Device-buffer layer
// ===========================================================================
extern "C" {

const char* life_last_error(void) { return g_error.c_str(); }
const char* life_version(void) { return "life-b200 0.1 (sm_100a)"; }
uint64_t life_kernel_launches(void) { return g_launches.load(); }
// Debug hook (not in the public header): LIFE_TRACE builds record per-warp
// (smid, start ns, end ns) of packed passes into this device buffer.
void life_debug_set_trace(void* dev_buf) { g_trace.store(dev_buf); }

int64_t life_packed_pitch_words(int64_t width) {
  return ceil_div(2 * ceil_div(width, 64), 32) * 32;
}

// W % 16 != 0 rows get three padding vectors after the row for the seam
// vectors of the temporal-blocked byte pass (byte_seam_prep_kernel).
int64_t life_byte_pitch(int64_t width) {
  const int64_t need = width % 16 ? ceil_div(width, 16) * 16 + 48 : width;
  return ceil_div(need, 128) * 128;
}

int life_band_bounds(int64_t extent, int32_t parts, int64_t* bounds) {
  if (parts < 1 || parts > extent)
    return set_error(LIFE_ERR_TOO_MANY_PARTS, "cannot split %lld rows into %d non-empty parts",
                     static_cast<long long>(extent), parts);
  const int64_t base = extent / parts, extra = extent % parts;
  int64_t at = 0;
  bounds[0] = 0;
  for (int32_t i = 0; i < parts; ++i) {
    at += base + (i < extra ? 1 : 0);
    bounds[i + 1] = at;
  }
  return LIFE_OK;
}

namespace {
// One generation over a W % 128 == 0 torus: packed_step1_kernel (16-byte
// vectors, HBM-bound).  Segments of >= 32 rows in ~8 waves of independent
// warps, as for the byte engine.
int launch_step1(const uint32_t* in, int64_t in_pitch, int64_t in_row0, int64_t in_rows,
                 uint32_t* out, int64_t out_pitch, int64_t out_row0, int64_t width,
                 int64_t out_rows, cudaStream_t stream) {
  // (A bulk-copy form -- one elected lane moving each 512-B strip row with
  // cp.async.bulk into an mbarrier-tracked slot -- measured 13.9 vs 21.4 T
  // cell-updates/s on 65536^2 and was dropped.)
  static DeviceCache blocks_per_sm;
  int dev = 0;
  cudaGetDevice(&dev);
  int nb = blocks_per_sm.get(dev);
  if (nb == 0) {
    LIFE_CUDA(cudaFuncSetAttribute(packed_step1_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kStep1Smem));
    LIFE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, packed_step1_kernel,
                                                            kStep1Threads, kStep1Smem));
    nb = std::max(nb, 1);
    blocks_per_sm.put(dev, nb);
  }
  Step1Args a{};
  a.in = in;
  a.in_pitch = in_pitch;
  a.in_row0 = in_row0;
  a.in_rows = in_rows;
  a.out = out;
  a.out_pitch = out_pitch;
  a.out_row0 = out_row0;
  a.out_rows = out_rows;
  a.nv = static_cast<int32_t>(width / 128);
  a.n_strips = static_cast<int32_t>(ceil_div(a.nv, kStep1Stride));
  const int64_t resident_warps =
      static_cast<int64_t>(nb) * (kStep1Threads / 32) * sm_count();
  static const int64_t waves = std::max<int64_t>(knob("LIFE_STEP1_WAVES", 8), 1);
  const int64_t segs_target = std::max<int64_t>(1, waves * resident_warps / a.n_strips);
  a.seg_rows = std::max<int64_t>(ceil_div(out_rows, segs_target), 32);
  const int64_t warps = ceil_div(out_rows, a.seg_rows) * a.n_strips;
  const int64_t blocks = ceil_div(warps, kStep1Threads / 32);
  if (blocks > 0x7fffffff) return set_error(LIFE_ERR_CONFIG, "grid too large");
  LIFE_TRY(launch_pdl(packed_step1_kernel, static_cast<unsigned>(blocks), kStep1Threads,
                      kStep1Smem, stream, a));
  LIFE_CHECK_LAUNCH("packed_step1_kernel");
  return LIFE_OK;
}
}  // namespace

}  // extern "C"

namespace lifegpu {
namespace detail {
int packed_step(const uint32_t* in, int64_t in_pitch, int64_t in_row0, int64_t in_rows,
                uint32_t* out, int64_t out_pitch, int64_t out_row0, int64_t width,
                int64_t out_rows, int32_t generations, cudaStream_t stream, SplitStreams* ss) {
  if (generations < 1 || generations > LIFE_MAX_TEMPORAL_DEPTH)
    return set_error(LIFE_ERR_CONFIG, "temporal depth must be in [1, %d], got %d",
                     LIFE_MAX_TEMPORAL_DEPTH, generations);
  if (width < 1 || in_rows < 1 || out_rows < 0 || in_pitch < 2 * ceil_div(width, 64) ||
      out_pitch < 2 * ceil_div(width, 64))
    return set_error(LIFE_ERR_CONFIG, "bad packed step geometry");
  if (out_rows == 0) return LIFE_OK;
  if (generations == 1 && width % 128 == 0 && in_pitch % 4 == 0 && out_pitch % 4 == 0 &&
      reinterpret_cast<uintptr_t>(in) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0 &&
      in_rows < (int64_t(1) << 31) && in_pitch * 4 < (int64_t(1) << 32) &&
      out_pitch * 4 < (int64_t(1) << 32) && !g_trace.load(std::memory_order_relaxed))
    return launch_step1(in, in_pitch, in_row0, in_rows, out, out_pitch, out_row0, width,
                        out_rows, stream);
  PackedStepArgs a{};
  a.in = in;
  a.in_pitch = in_pitch;
  a.in_row0 = in_row0;
  a.in_rows = in_rows;
  a.out = out;
  a.out_pitch = out_pitch;
  a.out_row0 = out_row0;
  a.width = width;
  a.out_rows = out_rows;
  a.nw = static_cast<int32_t>(nw32(width));
  a.n_strips = static_cast<int32_t>(ceil_div(a.nw + 1, kStripStride));
  a.strips_total = a.n_strips;
  a.tail_mask = tail_mask(width);
  a.trace = g_trace.load(std::memory_order_relaxed);
  return kPackedLaunchers[generations](a, stream, ss);
}

int packed_run(uint32_t* buf_a, uint32_t* buf_b, int64_t pitch, int64_t width, int64_t height,
               int64_t generations, int32_t depth, cudaStream_t stream, SplitStreams* ss,
               int* result_in_b, int il) {
  if (depth < 1 || depth > il_max_depth(il))
    return set_error(LIFE_ERR_CONFIG, "temporal depth must be in [1, %d], got %d",
                     il_max_depth(il), depth);
  if (generations < 0) return set_error(LIFE_ERR_CONFIG, "generations must be >= 0");
  if (width < 1 || height < 1 || pitch < 2 * ceil_div(width, 64) || buf_a == buf_b)
    return set_error(LIFE_ERR_CONFIG, "bad packed run geometry");
  uint32_t* cur = buf_a;
  uint32_t* nxt = buf_b;
  int flip = 0;
  const int64_t full = generations / depth;
  const int rem = static_cast<int>(generations % depth);
  auto pass = [&](int k) -> int {
    if (il != 0)  // buffers in the pair / quad layout (kernels_pair.cuh)
      return packed_il_step(il, cur, pitch, 0, height, nxt, pitch, 0, width, height, k, stream);
    return packed_step(cur, pitch, 0, height, nxt, pitch, 0, width, height, k, stream, ss);
  };
  for (int64_t i = 0; i < full; ++i) {
    LIFE_TRY(pass(depth));
    std::swap(cur, nxt);
    flip ^= 1;
  }
  if (rem > 0) {
    LIFE_TRY(pass(rem));
    flip ^= 1;
  }
  if (result_in_b) *result_in_b = flip;
  return LIFE_OK;
}
}  // namespace detail
}  // namespace lifegpu

extern "C" {

int life_dev_packed_step(const uint32_t* in, int64_t in_pitch, int64_t in_row0, int64_t in_rows,
                         uint32_t* out, int64_t out_pitch, int64_t out_row0, int64_t width,
                         int64_t out_rows, int32_t generations, void* stream) {
  return packed_step(in, in_pitch, in_row0, in_rows, out, out_pitch, out_row0, width, out_rows,
                     generations, static_cast<cudaStream_t>(stream), nullptr);
}

int life_dev_packed_run(uint32_t* buf_a, uint32_t* buf_b, int64_t pitch, int64_t width,
                        int64_t height, int64_t generations, int32_t depth, int32_t* result_in_b,
                        void* stream) {
  int flip = 0;
  LIFE_TRY(packed_run(buf_a, buf_b, pitch, width, height, generations, depth,
                      static_cast<cudaStream_t>(stream), nullptr, &flip));
  if (result_in_b) *result_in_b = flip;
  return LIFE_OK;
}

int life_dev_packed_zip(uint32_t* words, int64_t pitch, int64_t width, int64_t row0, int64_t rows,
                        int32_t order, int32_t to_interleaved, void* stream) {
  return packed_zip(order, words, pitch, width, row0, rows, /*unzip=*/to_interleaved == 0,
                    static_cast<cudaStream_t>(stream));
}

int life_dev_packed_step_il(int32_t order, const uint32_t* in, int64_t in_pitch, int64_t in_row0,
                            int64_t in_rows, uint32_t* out, int64_t out_pitch, int64_t out_row0,
                            int64_t width, int64_t out_rows, int32_t generations, void* stream) {
  return packed_il_step(order, in, in_pitch, in_row0, in_rows, out, out_pitch, out_row0, width,
                        out_rows, generations, static_cast<cudaStream_t>(stream));
}

int life_dev_packed_run_il(int32_t order, uint32_t* buf_a, uint32_t* buf_b, int64_t pitch,
                           int64_t width, int64_t height, int64_t generations, int32_t depth,
                           int32_t* result_in_b, void* stream) {
  if (!il_eligible(order, width))
    return set_error(LIFE_ERR_CONFIG, "interleave order %d needs W %% %d == 0, got %lld", order,
                     32 * order, static_cast<long long>(width));
  int flip = 0;
  LIFE_TRY(packed_run(buf_a, buf_b, pitch, width, height, generations, depth,
                      static_cast<cudaStream_t>(stream), nullptr, &flip, order));
  if (result_in_b) *result_in_b = flip;
  return LIFE_OK;
}

int life_dev_packed_step_il_peer(int32_t order, const uint32_t* in, const uint32_t* up,
                                 int64_t up_rows, const uint32_t* down, int64_t down_rows,
                                 int64_t pitch, int64_t band_rows, uint32_t* out, int64_t out_row0,
                                 int64_t out_rows, int64_t width, int32_t generations,
                                 void* stream) {
  return packed_il_step_peer(order, in, up, up_rows, down, down_rows, pitch, band_rows, out,
                             out_row0, out_rows, width, generations,
                             static_cast<cudaStream_t>(stream));
}

int life_dev_packed_step_peer(const uint32_t* in, const uint32_t* up, int64_t up_rows,
                              const uint32_t* down, int64_t down_rows, int64_t pitch,
                              int64_t band_rows, uint32_t* out, int64_t out_row0,
                              int64_t out_rows, int64_t width, int32_t generations,
                              void* stream) {
  if (generations < 1 || generations > LIFE_MAX_TEMPORAL_DEPTH)
    return set_error(LIFE_ERR_CONFIG, "temporal depth must be in [1, %d], got %d",
                     LIFE_MAX_TEMPORAL_DEPTH, generations);
  if (!in || !up || !down || !out || width < 1 || pitch < 2 * ceil_div(width, 64))
    return set_error(LIFE_ERR_CONFIG, "bad peer step geometry");
  if (band_rows < generations || up_rows < generations || down_rows < generations)
    return set_error(LIFE_ERR_TOO_MANY_PARTS, "bands must be at least %d rows", generations);
  if (out_row0 < 0 || out_rows < 0 || out_row0 + out_rows > band_rows)
    return set_error(LIFE_ERR_CONFIG, "output rows outside the band");
  if (out_rows == 0) return LIFE_OK;
  PackedStepArgs a{};
  a.in = in;
  a.in_pitch = pitch;
  a.in_row0 = out_row0;  // band coordinates: relative row 0 = band row out_row0
  a.in_rows = band_rows;
  a.out = out;
  a.out_pitch = pitch;
  a.out_row0 = out_row0;
  a.width = width;
  a.out_rows = out_rows;
  a.nw = static_cast<int32_t>(nw32(width));
  a.n_strips = static_cast<int32_t>(ceil_div(a.nw + 1, kStripStride));
  a.strips_total = a.n_strips;
  a.tail_mask = tail_mask(width);
  a.trace = g_trace.load(std::memory_order_relaxed);
  a.up = up;
  a.down = down;
  a.up_rows = up_rows;
  a.down_rows = down_rows;
  a.peer = 1;  // peer launches never split (no side stream)
  return kPackedLaunchers[generations](a, static_cast<cudaStream_t>(stream), nullptr);
}

namespace {
// Cluster-resident engine plan: the largest cluster (16, 8, 4, 2, 1 CTAs)
// whose bands (>= 2 rows each, double-buffered) fit one CTA's shared memory
// and that the device can co-schedule.
struct ResidentPlan {
  int C = 0, threads = 0, groups = 0;
  size_t smem = 0;
  ResidentArgs args{};
};

// Interior threads per CTA the resident engine aims for: enough warps to
// hide shared-memory latency, few enough that each thread's run of rows
// amortises the two rows of horizontal sums it recomputes per generation
// (measured).
// Sweep (T cell-updates/s, 800 generations): 1024^2 at 256/512/1024
// threads 1.78/1.91/1.57; 2048^2 2.48/3.00/3.04; 2048x4096 2.71/3.33/3.53.
int resident_target_threads(int nw) {
  static const int v = static_cast<int>(knob("LIFE_RESIDENT_THREADS", 0));  // debug builds
  return v > 0 ? v : (nw <= 32 ? 512 : kResidentMaxThreads);
}

int plan_resident(int64_t width, int64_t height, ResidentPlan* plan) {
  if (width < 32 || width % 32 != 0 || width / 32 > kResidentMaxThreads || height < 2)
    return LIFE_ERR_CONFIG;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  LIFE_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  static DeviceCache max_dyn;  // dynamic shared memory bytes per CTA (opt-in max - static)
  if (max_dyn.get(dev) == 0) {
    cudaFuncAttributes fa{};
    LIFE_CUDA(cudaFuncGetAttributes(&fa, packed_resident_kernel));
    const int dyn = optin - static_cast<int>(fa.sharedSizeBytes);
    LIFE_CUDA(cudaFuncSetAttribute(packed_resident_kernel,
                                   cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    LIFE_CUDA(cudaFuncSetAttribute(packed_resident_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    max_dyn.put(dev, dyn);
  }
  optin = max_dyn.get(dev);
  const int nw = static_cast<int>(width / 32);
  for (int C : {16, 8, 4, 2, 1}) {
    if (height < 2 * C) continue;
    const int64_t max_rows = ceil_div(height, C);
    const size_t smem = static_cast<size_t>(2 * (max_rows + 2) * nw) * 4;  // + 2 halo rows
    if (smem > static_cast<size_t>(optin)) continue;
    const int interior = static_cast<int>(height / C) - 2;
    // Edge warps (the two rows next to the halos) + interior warps.
    const int edge_threads = static_cast<int>(ceil_div(2 * nw, 32) * 32);
    if (edge_threads + nw > kResidentMaxThreads) continue;
    int groups = static_cast<int>(ceil_div(resident_target_threads(nw), nw));
    groups = std::max(1, std::min({groups, std::max(interior, 1),
                                   (kResidentMaxThreads - edge_threads) / nw}));
    const int threads =
        edge_threads + static_cast<int>(ceil_div(static_cast<int64_t>(groups) * nw, 32) * 32);
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, packed_resident_kernel, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (clusters < 1) continue;
    plan->C = C;
    plan->threads = threads;
    plan->groups = groups;
    plan->smem = smem;
    plan->args.nw = nw;
    plan->args.base_rows = static_cast<int32_t>(height / C);
    plan->args.extra_rows = static_cast<int32_t>(height % C);
    plan->args.max_rows = static_cast<int32_t>(max_rows);
    plan->args.groups = groups;
    return LIFE_OK;
  }
  return LIFE_ERR_CONFIG;
}
}  // namespace

int life_resident_cluster_size(int64_t width, int64_t height) {
  ResidentPlan p;
  return plan_resident(width, height, &p) == LIFE_OK ? p.C : 0;
}

int life_dev_packed_run_resident(const uint32_t* in, uint32_t* out, int64_t pitch, int64_t width,
                                 int64_t height, int64_t generations, void* stream) {
  if (generations < 0) return set_error(LIFE_ERR_CONFIG, "generations must be non-negative");
  if (!in || !out || pitch < width / 32)
    return set_error(LIFE_ERR_CONFIG, "bad resident run geometry");
  ResidentPlan p;
  const int rc = plan_resident(width, height, &p);
  if (rc != LIFE_OK) {
    if (rc == LIFE_ERR_CONFIG)
      return set_error(LIFE_ERR_CONFIG,
                       "a %lldx%lld torus does not fit the cluster-resident engine "
                       "(needs W %% 32 == 0, W <= 32768, H >= 2 and both buffers of "
                       "every band in one CTA's shared memory)",
                       static_cast<long long>(width), static_cast<long long>(height));
    return rc;
  }
  p.args.in = in;
  p.args.out = out;
  p.args.pitch = pitch;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(p.C);
  cfg.blockDim = dim3(p.threads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // One launch per 2^30 generations (the kernel counts in int32).
  int64_t left = generations;
  const uint32_t* src = in;
  do {
    const int64_t n = std::min<int64_t>(left, int64_t(1) << 30);
    p.args.in = src;
    p.args.generations = static_cast<int32_t>(n);
    LIFE_CUDA(cudaLaunchKernelEx(&cfg, packed_resident_kernel, p.args));
    LIFE_CHECK_LAUNCH("packed_resident_kernel");
    left -= n;
    src = out;
  } while (left > 0);
  return LIFE_OK;
}

int life_dev_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return set_error(LIFE_ERR_CONFIG, "bad allocation request");
  *out = nullptr;
  LIFE_CUDA(cudaMalloc(out, bytes > 0 ? bytes : 1));
  LIFE_CUDA(cudaMemset(*out, 0, bytes > 0 ? bytes : 1));
  return LIFE_OK;
}

int life_dev_free(void* p) {
  if (p) LIFE_CUDA(cudaFree(p));
  return LIFE_OK;
}

int life_ipc_get_handle(void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return set_error(LIFE_ERR_CONFIG, "null pointer");
  cudaIpcMemHandle_t h;
  LIFE_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
  std::memcpy(handle_out, &h, sizeof(h));
  return LIFE_OK;
}

int life_ipc_open(const void* handle, void** out) {
  if (!handle || !out) return set_error(LIFE_ERR_CONFIG, "null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  LIFE_CUDA(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  return LIFE_OK;
}

int life_ipc_close(void* dev_ptr) {
  if (dev_ptr) LIFE_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return LIFE_OK;
}

// Stream memory operations through the driver entry points (the library links
// cudart statically and not libcuda): cuStreamWriteValue32(stream, addr, value,
// flags) and cuStreamWaitValue32(stream, addr, value, CU_STREAM_WAIT_VALUE_GEQ).
namespace {
using StreamMemOp = int (*)(cudaStream_t, unsigned long long, uint32_t, unsigned int);
struct StreamMemOps {
  StreamMemOp write = nullptr, wait = nullptr;
  StreamMemOps() {
    void* w = nullptr;
    void* q = nullptr;
    cudaDriverEntryPointQueryResult rw, rq;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &rw) == cudaSuccess &&
        rw == cudaDriverEntryPointSuccess &&
        cudaGetDriverEntryPoint("cuStreamWaitValue32", &q, cudaEnableDefault, &rq) == cudaSuccess &&
        rq == cudaDriverEntryPointSuccess) {
      write = reinterpret_cast<StreamMemOp>(w);
      wait = reinterpret_cast<StreamMemOp>(q);
    }
  }
};
int stream_mem_op(bool wait, void* flag, uint32_t value, void* stream) {
  static const StreamMemOps ops;  // thread-safe initialisation
  if (!flag || (reinterpret_cast<uintptr_t>(flag) & 3))
    return set_error(LIFE_ERR_CONFIG, "flag must be a 4-byte aligned device pointer");
  if (!ops.write || !ops.wait)
    return set_error(LIFE_ERR_CUDA, "the driver exports no stream memory operations");
  constexpr unsigned int kGeq = 0x0;  // CU_STREAM_WAIT_VALUE_GEQ: (int32_t)(*addr - value) >= 0
  const int rc = wait ? ops.wait(static_cast<cudaStream_t>(stream),
                                 reinterpret_cast<unsigned long long>(flag), value, kGeq)
                      : ops.write(static_cast<cudaStream_t>(stream),
                                  reinterpret_cast<unsigned long long>(flag), value, 0u);
  if (rc != 0)
    return set_error(LIFE_ERR_CUDA, "%s failed (CUresult %d)",
                     wait ? "cuStreamWaitValue32" : "cuStreamWriteValue32", rc);
  return LIFE_OK;
}
}  // namespace

int life_dev_flag_write(void* flag, uint32_t value, void* stream) {
  return stream_mem_op(false, flag, value, stream);
}

int life_dev_flag_wait_geq(void* flag, uint32_t value, void* stream) {
  return stream_mem_op(true, flag, value, stream);
}

int life_dev_byte_step(const uint8_t* in, int64_t in_pitch, int64_t in_row0, int64_t in_rows,
                       uint8_t* out, int64_t out_pitch, int64_t out_row0, int64_t width,
                       int64_t out_rows, void* stream) {
  if (width < 1 || in_rows < 1 || out_rows < 0 || in_pitch < ceil_div(width, 16) * 16 ||
      out_pitch < ceil_div(width, 16) * 16 || (in_pitch & 15) || (out_pitch & 15))
    return set_error(LIFE_ERR_CONFIG, "bad byte step geometry");
  if (out_rows == 0) return LIFE_OK;
  static DeviceCache blocks_per_sm;
  int dev = 0;
  cudaGetDevice(&dev);
  int nb = blocks_per_sm.get(dev);
  if (nb == 0) {
    LIFE_CUDA(cudaFuncSetAttribute(byte_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kByteSmem));
    LIFE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, byte_step_kernel,
                                                            kByteThreads, kByteSmem));
    nb = std::max(nb, 1);
    blocks_per_sm.put(dev, nb);
  }
  ByteStepArgs a{};
  a.in = in;
  a.in_pitch = in_pitch;
  a.in_row0 = in_row0;
  a.in_rows = in_rows;
  a.out = out;
  a.out_pitch = out_pitch;
  a.out_row0 = out_row0;
  a.width = width;
  a.out_rows = out_rows;
  a.nv = static_cast<int32_t>(ceil_div(width, 16));
  a.n_strips = static_cast<int32_t>(ceil_div(a.nv, kByteStride));
  if (in_rows >= (int64_t(1) << 31) || in_pitch >= (int64_t(1) << 32) ||
      out_pitch >= (int64_t(1) << 32) || out_rows >= (int64_t(1) << 31))
    return set_error(LIFE_ERR_CONFIG, "grid too large for the byte engine");
  const int64_t resident_warps =
      static_cast<int64_t>(nb) * (kByteThreads / 32) * sm_count();
  // Many short segments (>= 32 rows; the 2 halo rows are L2 hits) so the
  // independent warps balance across SMs: 8 waves measured +3 % over 2.
#ifndef LIFE_BYTE_WAVES
#define LIFE_BYTE_WAVES 8
#endif
  const int64_t segs_target = std::max<int64_t>(1, LIFE_BYTE_WAVES * resident_warps / a.n_strips);
  a.seg_rows = std::max<int64_t>(ceil_div(out_rows, segs_target), 32);
  const int64_t warps = ceil_div(out_rows, a.seg_rows) * a.n_strips;
  const int64_t blocks = ceil_div(warps, kByteThreads / 32);
  byte_step_kernel<<<static_cast<unsigned>(blocks), kByteThreads, kByteSmem,
                     static_cast<cudaStream_t>(stream)>>>(a);
  LIFE_CHECK_LAUNCH("byte_step_kernel");
  return LIFE_OK;
}

}  // extern "C"

namespace {
template <int K>
int launch_byte_tb(ByteStepArgs a, cudaStream_t s) {
  // Two row streams per word (byte_tb2_kernel) unless LIFE_BYTE_TB2=0 (debug builds).
  // W % 16 != 0 tori need the two-stream kernel's seam path.
  static const bool two_knob = knob("LIFE_BYTE_TB2", 1) != 0;
  const bool seam = (a.width & 15) != 0;
  const bool two = two_knob || seam;
  const auto kernel = !two ? byte_tb_kernel<K>
                           : (seam ? byte_tb2_kernel<K, true> : byte_tb2_kernel<K, false>);
  const int smem = two ? kByteTb2Smem : kByteTbSmem;
  static DeviceCache blocks_per_sm[3];  // [one-stream, two-stream, two-stream seam]
  const int variant = !two ? 0 : (seam ? 2 : 1);
  int dev = 0;
  cudaGetDevice(&dev);
  int nb = blocks_per_sm[variant].get(dev);
  if (nb == 0) {
    LIFE_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    LIFE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kByteThreads, smem));
    nb = std::max(nb, 1);
    blocks_per_sm[variant].put(dev, nb);
  }
  // Segments long enough to amortise the 3K-1 step pipeline fill: one wave
  // of independent warps.
  // LIFE_BYTE_TB_WPS (debug builds): warps per SM to plan the segments for.
  static const int64_t wps = knob("LIFE_BYTE_TB_WPS", 0);
  const int64_t resident_warps =
      (wps > 0 ? wps : static_cast<int64_t>(nb) * (kByteThreads / 32)) * sm_count();
  // 1 wave: 8.41 vs 8.02 T/s (2) at 16384^2, K = 6 (LIFE_BYTE_TB_WAVES, debug builds)
  static const int64_t waves = std::max<int64_t>(knob("LIFE_BYTE_TB_WAVES", 1), 1);
  const int64_t segs_target = std::max<int64_t>(1, waves * resident_warps / a.n_strips);
  a.seg_rows = std::max<int64_t>(ceil_div(a.out_rows, segs_target), 16 * K);
  const int64_t warps = ceil_div(a.out_rows, a.seg_rows) * a.n_strips;
  const int64_t blocks = ceil_div(warps, kByteThreads / 32);
  if (blocks > 0x7fffffff) return set_error(LIFE_ERR_CONFIG, "grid too large");
  if (seam) {  // the seam vectors of every input row, into the row padding
    const SeamPrepArgs pa{const_cast<uint8_t*>(a.in), a.in_pitch, a.in_rows, a.width};
    LIFE_TRY(launch_pdl(byte_seam_prep_kernel,
                        static_cast<unsigned>(std::min<int64_t>(ceil_div(a.in_rows, 128),
                                                                4 * sm_count())),
                        128, 0, s, pa));
    LIFE_CHECK_LAUNCH("byte_seam_prep_kernel");
  }
  LIFE_TRY(launch_pdl(kernel, static_cast<unsigned>(blocks), kByteThreads, smem, s, a));
  LIFE_CHECK_LAUNCH("byte_tb_kernel");
  return LIFE_OK;
}
using ByteTbLauncher = int (*)(ByteStepArgs, cudaStream_t);
const ByteTbLauncher kByteTbLaunchers[kByteTbMaxDepth + 1] = {
    nullptr, nullptr, launch_byte_tb<2>, launch_byte_tb<3>, launch_byte_tb<4>,
    launch_byte_tb<5>, launch_byte_tb<6>, launch_byte_tb<7>, launch_byte_tb<8>};
}  // namespace

extern "C" {

int life_dev_byte_pass(const uint8_t* in, int64_t in_pitch, int64_t in_row0, int64_t in_rows,
                       uint8_t* out, int64_t out_pitch, int64_t out_row0, int64_t width,
                       int64_t out_rows, int32_t generations, void* stream) {
  if (generations < 1 || generations > kByteTbMaxDepth)
    return set_error(LIFE_ERR_CONFIG, "byte temporal depth must be in [1, %d], got %d",
                     kByteTbMaxDepth, generations);
  if (generations == 1)
    return life_dev_byte_step(in, in_pitch, in_row0, in_rows, out, out_pitch, out_row0, width,
                              out_rows, stream);
  if (width % 16 != 0 && width < kByteTbMinSeamWidth)
    return set_error(LIFE_ERR_CONFIG,
                     "byte passes of more than one generation need W %% 16 == 0 or W >= %d, "
                     "got W = %lld", kByteTbMinSeamWidth, static_cast<long long>(width));
  if (width < 1 || in_rows < 1 || out_rows < 0 || in_pitch < width || out_pitch < width ||
      (in_pitch & 15) || (out_pitch & 15))
    return set_error(LIFE_ERR_CONFIG, "bad byte pass geometry");
  if (width % 16 != 0 && in_pitch < ceil_div(width, 16) * 16 + 48)
    return set_error(LIFE_ERR_CONFIG,
                     "byte passes of W %% 16 != 0 tori need 48 bytes of row padding "
                     "(in_pitch >= life_byte_pitch(W)), got in_pitch = %lld",
                     static_cast<long long>(in_pitch));
  if (out_rows == 0) return LIFE_OK;
  if (in_rows >= (int64_t(1) << 31) || in_pitch >= (int64_t(1) << 32) ||
      out_pitch >= (int64_t(1) << 32) || out_rows >= (int64_t(1) << 31))
    return set_error(LIFE_ERR_CONFIG, "grid too large for the byte engine");
  ByteStepArgs a{};
  a.in = in;
  a.in_pitch = in_pitch;
  a.in_row0 = in_row0;
  a.in_rows = in_rows;
  a.out = out;
  a.out_pitch = out_pitch;
  a.out_row0 = out_row0;
  a.width = width;
  a.out_rows = out_rows;
  a.nv = static_cast<int32_t>(ceil_div(width, 16));
  a.n_strips = static_cast<int32_t>(ceil_div(a.nv + 1, kByteTbStride));
  a.one = 1;
  return kByteTbLaunchers[generations](a, static_cast<cudaStream_t>(stream));
}

int life_dev_packed_random(uint32_t* out, int64_t pitch, int64_t width, int64_t y0, int64_t rows,
                           double density, uint64_t seed, void* stream) {
  if (!(density >= 0.0 && density <= 1.0))
    return set_error(LIFE_ERR_CONFIG, "density must be in [0, 1], got %f", density);
  const int64_t n = rows * pitch;
  packed_random_kernel<<<grid_stride_blocks(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      out, pitch, width, y0, rows, static_cast<int32_t>(nw32(width)), seed,
      density_threshold(density));
  LIFE_CHECK_LAUNCH("packed_random_kernel");
  return LIFE_OK;
}

int life_dev_byte_random(uint8_t* out, int64_t pitch, int64_t width, int64_t y0, int64_t rows,
                         double density, uint64_t seed, void* stream) {
  if (!(density >= 0.0 && density <= 1.0))
    return set_error(LIFE_ERR_CONFIG, "density must be in [0, 1], got %f", density);
  if ((pitch & 15) || pitch < width) return set_error(LIFE_ERR_CONFIG, "bad byte pitch");
  const int64_t n = rows * (pitch / 16);
  byte_random_kernel<<<grid_stride_blocks(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      out, pitch, width, y0, rows, seed, density_threshold(density));
  LIFE_CHECK_LAUNCH("byte_random_kernel");
  return LIFE_OK;
}

int life_dev_packed_population(const uint32_t* grid, int64_t pitch, int64_t width, int64_t rows,
                               uint64_t* dev_count, void* stream) {
  const int64_t n = rows * pitch;
  packed_popcount_kernel<<<grid_stride_blocks(n / 4, 256), 256, 0,
                           static_cast<cudaStream_t>(stream)>>>(
      grid, pitch, static_cast<int32_t>(nw32(width)), rows,
      reinterpret_cast<unsigned long long*>(dev_count));
  LIFE_CHECK_LAUNCH("packed_popcount_kernel");
  return LIFE_OK;
}

int life_dev_packed_row_hashes(const uint32_t* grid, int64_t pitch, int64_t width, int64_t rows,
                               uint64_t* dev_hashes, void* stream) {
  if (!grid || !dev_hashes || width < 1 || rows < 0 || pitch < 2 * ceil_div(width, 64))
    return set_error(LIFE_ERR_CONFIG, "bad row-hash geometry");
  if (rows == 0) return LIFE_OK;
  packed_row_hash_kernel<<<grid_stride_blocks(rows, 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      grid, pitch, static_cast<int32_t>(2 * ceil_div(width, 64)), rows,
      reinterpret_cast<unsigned long long*>(dev_hashes));
  LIFE_CHECK_LAUNCH("packed_row_hash_kernel");
  return LIFE_OK;
}

uint64_t life_fnv1a64(const void* bytes, int64_t n, uint64_t h) {
  const uint8_t* p = static_cast<const uint8_t*>(bytes);
  if (h == 0) h = 0xcbf29ce484222325ULL;
  for (int64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

int life_dev_pack(const uint8_t* cells, int64_t cell_pitch, uint32_t* words, int64_t pitch,
                  int64_t width, int64_t rows, void* stream) {
  const int64_t warps = rows * ceil_div(pitch, 32);
  pack_kernel<<<grid_stride_blocks(warps * 32, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      cells, cell_pitch, words, pitch, width, rows);
  LIFE_CHECK_LAUNCH("pack_kernel");
  return LIFE_OK;
}

int life_dev_unpack(const uint32_t* words, int64_t pitch, uint8_t* cells, int64_t cell_pitch,
                    int64_t width, int64_t rows, void* stream) {
  if (cell_pitch & 15) return set_error(LIFE_ERR_CONFIG, "byte pitch must be a multiple of 16");
  const int64_t n = rows * (cell_pitch / 16);
  unpack_kernel<<<grid_stride_blocks(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      words, pitch, cells, cell_pitch, width, rows);
  LIFE_CHECK_LAUNCH("unpack_kernel");
  return LIFE_OK;
}

int life_measure_int_peak(int device, int64_t iters, double* ops_per_s, double* seconds) {
  LIFE_CUDA(cudaSetDevice(device));
  uint32_t* sink = nullptr;
  LIFE_CUDA(cudaMalloc(&sink, 4));
  cudaEvent_t e0, e1;
  LIFE_CUDA(cudaEventCreate(&e0));
  LIFE_CUDA(cudaEventCreate(&e1));
  const int blocks = sm_count() * 8, threads = 256;
  int_peak_kernel<<<blocks, threads>>>(sink, std::max<int64_t>(iters / 8, 1), 1u);  // warm-up
  LIFE_CHECK_LAUNCH("int_peak_kernel");
  LIFE_CUDA(cudaEventRecord(e0));
  int_peak_kernel<<<blocks, threads>>>(sink, iters, 2u);
  LIFE_CHECK_LAUNCH("int_peak_kernel");
  LIFE_CUDA(cudaEventRecord(e1));
  LIFE_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  LIFE_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  const double ops = double(blocks) * threads * double(iters) * 16.0 * 8.0;
  *seconds = ms * 1e-3;
  *ops_per_s = ops / (ms * 1e-3);
  return LIFE_OK;
}

}  // extern "C"

// ===========================================================================
// Contexts: one resident grid on one GPU, the reference's run() on top.
// ===========================================================================
enum Layout { kNone = -1, kPacked = LIFE_ENGINE_PACKED, kByte = LIFE_ENGINE_BYTE };

struct life_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  int64_t W = 0, H = 0;
  int layout = kNone;
  uint32_t* pk[2] = {nullptr, nullptr};
  int64_t pk_pitch = 0;  // uint32 words
  int pk_cur = 0;
  // pk[pk_cur] is in the interleaved-pair layout (kernels_pair.cuh): left so by
  // life_run between runs; every reader of the plain layout calls pk_plain().
  int pk_il = 0;  // 0 plain, 2 pair, 4 quad
  uint8_t* by[2] = {nullptr, nullptr};
  int64_t by_pitch = 0;  // bytes
  int by_cur = 0;
  unsigned long long* counts = nullptr;
  int64_t counts_cap = 0;
  uint64_t* row_hashes = nullptr;  // life_grid_hash scratch (H entries)
  int64_t row_hashes_cap = 0;
  uint8_t* window = nullptr;
  int64_t window_cap = 0;
  // life_run_batch: 2 slots x (upload/ping, pong) buffers and copy streams
  uint32_t* batch[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t batch_bytes = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaStream_t cs[4] = {};  // life_run_batch chunk streams (first / last grid)
  // Side streams of split launches: [0] for `stream`, [1..4] for cs[0..3].
  SplitStreams split[5];
  // Options (life_ctx_set_option).
  int batch_trap = -1;   // LIFE_OPT_BATCH_TRAPEZOID
  bool profile = false;  // LIFE_OPT_PROFILE
  int pair_depth = -1;   // LIFE_OPT_PAIR_DEPTH
  int quad_depth = -1;   // LIFE_OPT_QUAD_DEPTH
  // Statistics of the last life_run (life_ctx_band_stats, band 0).
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  double run_ms = 0.0, pass_ms = 0.0;
  int64_t passes = 0;
  // Multi-device contexts (life_ctx_create_multi): every grid / run entry
  // point dispatches to life_multi.cu; the fields above are unused.
  MultiState* multi = nullptr;
};

namespace {

int activate(life_ctx* c) {
  if (!c) return set_error(LIFE_ERR_STATE, "null context");
  LIFE_CUDA(cudaSetDevice(c->device));
  return LIFE_OK;
}

void free_buffers(life_ctx* c) {
  for (int i = 0; i < 2; ++i) {
    if (c->pk[i]) cudaFree(c->pk[i]);
    if (c->by[i]) cudaFree(c->by[i]);
    c->pk[i] = nullptr;
    c->by[i] = nullptr;
  }
  c->layout = kNone;
}

int set_dims(life_ctx* c, int64_t w, int64_t h) {
  LIFE_TRY(check_dims(w, h));
  c->pk_il = 0;  // callers overwrite the whole grid in the plain layout
  if (w != c->W || h != c->H) {
    LIFE_CUDA(cudaStreamSynchronize(c->stream));
    free_buffers(c);
    c->W = w;
    c->H = h;
    c->pk_pitch = life_packed_pitch_words(w);
    c->by_pitch = life_byte_pitch(w);
  }
  return LIFE_OK;
}

int ensure_packed(life_ctx* c) {
  for (int i = 0; i < 2; ++i) {
    if (!c->pk[i]) {
      const size_t bytes = static_cast<size_t>(c->pk_pitch) * c->H * 4;
      LIFE_CUDA(cudaMalloc(&c->pk[i], bytes));
      LIFE_CUDA(cudaMemsetAsync(c->pk[i], 0, bytes, c->stream));
    }
  }
  return LIFE_OK;
}

int ensure_byte(life_ctx* c) {
  for (int i = 0; i < 2; ++i) {
    if (!c->by[i]) {
      const size_t bytes = static_cast<size_t>(c->by_pitch) * c->H;
      LIFE_CUDA(cudaMalloc(&c->by[i], bytes));
      LIFE_CUDA(cudaMemsetAsync(c->by[i], 0, bytes, c->stream));
    }
  }
  return LIFE_OK;
}

int ensure_counts(life_ctx* c, int64_t n) {
  if (n > c->counts_cap) {
    if (c->counts) cudaFree(c->counts);
    c->counts = nullptr;
    LIFE_CUDA(cudaMalloc(&c->counts, sizeof(unsigned long long) * n));
    c->counts_cap = n;
  }
  return LIFE_OK;
}

// Converts the resident grid to `layout` (device-side pack / unpack).
// life_run leaves a W % 64 == 0 packed grid in the interleaved-pair layout
// (kernels_pair.cuh) so consecutive runs pay no conversion; everything that
// reads or edits the plain packed words converts it back first (in place,
// one HBM read + write of the grid).
int pk_plain(life_ctx* c) {
  if (c->layout == kPacked && c->pk_il != 0) {
    LIFE_TRY(packed_zip(c->pk_il, c->pk[c->pk_cur], c->pk_pitch, c->W, 0, c->H, /*unzip=*/true,
                        c->stream));
  }
  c->pk_il = 0;
  return LIFE_OK;
}
int pk_to_il(life_ctx* c, int il) {
  if (c->layout != kPacked || c->pk_il == il) return LIFE_OK;
  LIFE_TRY(pk_plain(c));
  LIFE_TRY(packed_zip(il, c->pk[c->pk_cur], c->pk_pitch, c->W, 0, c->H, /*unzip=*/false,
                      c->stream));
  c->pk_il = il;
  return LIFE_OK;
}

int to_layout(life_ctx* c, int layout) {
  if (c->layout == kNone) return set_error(LIFE_ERR_STATE, "no grid loaded");
  if (c->layout == layout) return LIFE_OK;
  LIFE_TRY(pk_plain(c));
  if (layout == kPacked) {
    LIFE_TRY(ensure_packed(c));
    LIFE_TRY(life_dev_pack(c->by[c->by_cur], c->by_pitch, c->pk[0], c->pk_pitch, c->W, c->H,
                           c->stream));
    c->pk_cur = 0;
  } else {
    LIFE_TRY(ensure_byte(c));
    LIFE_TRY(life_dev_unpack(c->pk[c->pk_cur], c->pk_pitch, c->by[0], c->by_pitch, c->W, c->H,
                             c->stream));
    c->by_cur = 0;
  }
  c->layout = layout;
  return LIFE_OK;
}

int population_async(life_ctx* c, unsigned long long* slot) {
  LIFE_CUDA(cudaMemsetAsync(slot, 0, sizeof(unsigned long long), c->stream));
  if (c->layout == kPacked) {
    return life_dev_packed_population(c->pk[c->pk_cur], c->pk_pitch, c->W, c->H,
                                      reinterpret_cast<uint64_t*>(slot), c->stream);
  }
  const int64_t nv = ceil_div(c->W, 16);
  byte_popcount_kernel<<<grid_stride_blocks(c->H * nv / 4, 256), 256, 0, c->stream>>>(
      c->by[c->by_cur], c->by_pitch, c->H, nv, slot);
  LIFE_CHECK_LAUNCH("byte_popcount_kernel");
  return LIFE_OK;
}

int check_engine(int engine) {
  if (engine != LIFE_ENGINE_PACKED && engine != LIFE_ENGINE_BYTE && engine != LIFE_ENGINE_RESIDENT)
    return set_error(LIFE_ERR_CONFIG, "unknown engine %d", engine);
  return LIFE_OK;
}

// The resident grid layout an engine computes on.
int engine_layout(int engine) { return engine == LIFE_ENGINE_BYTE ? kByte : kPacked; }

// temporal_depth 0 on the packed engine: the cluster-resident engine for
// small tori (W % 32 == 0, at most kResidentAutoCells cells) where it beats
// the multi-pass engine (measured), else K = 16 passes.
constexpr int64_t kResidentAutoCells = int64_t(1) << 22;
// temporal_depth 0 on the byte engine (W % 16 == 0 or W >= 33).  Two-stream kernel
// (byte_tb2_kernel), T cell-updates/s at K = 4 / 6 / 8: 16384^2 10.0 / 12.7 /
// 13.1, 32768 x 16384 10.0 / 13.8 / 13.7, 4096^2 4.6 / 4.1 / 3.6 (short grids
// pay the 3K-1 step pipeline fill).  (One stream per word, round 1: 16384^2
// 8.1 / 8.8 / 8.1.)
int byte_auto_depth(int64_t w, int64_t h) { return w * h >= (int64_t(1) << 26) ? 8 : 4; }

bool resident_auto(int64_t w, int64_t h) {
  return w % 32 == 0 && w * h <= kResidentAutoCells && life_resident_cluster_size(w, h) > 0;
}

}  // namespace

// temporal_depth 0 on the multi-pass packed engine: K = 16, except tori whose
// passes run as one all-paths launch (W % 32 != 0, less than ~3 block waves
// deep), where K = 12 fits 12 warps per SM instead of 8 (config 4: 37.5 ->
// 38.6 T/s; kbench depth sweep).
// temporal_depth 0 on tori (or row bands of them, h rows tall) of 2^27 cells
// or more (quad: 2^29): the layout with the best lanes-per-op figure -- the share of a
// strip's 32 lanes that hold cells (groups / (32 x strips), strips of 32
// groups advancing by 31) over the network's ops per word (11 plain, 10 pair,
// 9.5 quad).  Wide tori fill their strips in every layout and take quad at
// K = 7 (2^31 cells or more) or 6; narrower ones waste the last strip of the
// wider groups and keep pair (K = 10) or the plain kernels.  kbench, T
// cell-updates/s, plain K = 16 / pair K = 10 / quad K = 6 / quad K = 7:
//   262144^2      47.1 / 51.1 / 53.1 / 54.0   65536^2       44.5 / 48.1 / 52.2 / 52.8
//   131072 x 8192 39.9 / 45.3 / 48.7 / 48.1   32768^2       41.7 / 46.4 / 46.0 / 45.6
//   32768 x 65536 43.4 / 47.5 / 47.5          32768 x 16384 39.3 / 42.2 / 42.1
//   16384 x 65536 42.2 / 43.2 / 40.9          8192 x 131072 40.4 / 39.3 / 34.9
// With the phased pipeline fill (LIFE_FILL_PHASES, packed_common.cuh) the
// pair layout also pays on one-wave tori down to 2^27 cells (plain K = 16 /
// pair K = 10 / quad K = 7, tools/r5_rule.sh):
//   16384^2 (config 2) 38.8 / 40.8 / 38.2   20480^2      41.5 / 43.9 / 41.5
//   32768 x 8192       38.9 / 42.6 / 41.2   12288^2      34.8 / 36.3 / 30.1
//   16384 x 8192       34.2 / 34.5 / 29.7   8192 x 16384 32.8 / 32.2 / 26.8
//   8192^2             28.2 / 26.3 / 22.3   4096^2       14.4 / 11.5 /  8.5
// Quad stays with tori of 2^29 cells or more; smaller tori keep the plain
// kernels (their tiles are too short for the wider groups' fewer strips).
namespace {
constexpr int64_t kIlAutoCells = int64_t(1) << 27;      // pair layout from here
constexpr int64_t kIlAutoCellsQuad = int64_t(1) << 29;  // quad layout from here
double lanes_per_op(int il, int64_t w) {
  const int64_t groups = il == 0 ? nw32(w) : w / (32 * il);
  const int64_t strips = ceil_div(groups + 1, kStripStride);
  const double ops = il == 4 ? 9.5 : il == 2 ? 10.0 : 11.0;
  return static_cast<double>(groups) / static_cast<double>(32 * strips) / ops;
}
}  // namespace
lifegpu::detail::IlChoice lifegpu::detail::il_choose(int64_t w, int64_t h, int pair_opt,
                                                     int quad_opt, int temporal_depth) {
  IlChoice c;
  if (quad_opt > 0 && il_eligible(4, w)) {
    c.il = 4;
    c.depth = quad_opt;
  } else if (pair_opt > 0 && il_eligible(2, w)) {
    c.il = 2;
    c.depth = pair_opt;
  } else if (temporal_depth == 0 && w * h >= kIlAutoCells) {
    double best = lanes_per_op(0, w);
    if (pair_opt < 0 && il_eligible(2, w) && lanes_per_op(2, w) > best) {
      best = lanes_per_op(2, w);
      c.il = 2;
      c.depth = 10;
    }
    if (quad_opt < 0 && w * h >= kIlAutoCellsQuad && il_eligible(4, w) &&
        lanes_per_op(4, w) > best) {
      c.il = 4;  // K = 7 (243 registers) pays on the largest tori only
      c.depth = w * h >= (int64_t(1) << 31) ? 7 : 6;
    }
  }
  return c;
}

int lifegpu::detail::packed_auto_depth(int64_t w, int64_t h) {
  const int64_t strips = ceil_div(nw32(w) + 1, kStripStride);
  return (w % 32 != 0 && strips * h < 2000000) ? 12 : LIFE_MAX_TEMPORAL_DEPTH;
}

extern "C" {

int life_packed_auto_depth(int64_t width, int64_t height) {
  if (width < 1 || height < 1) return LIFE_MAX_TEMPORAL_DEPTH;
  return packed_auto_depth(width, height);
}

int life_interleave_auto(int64_t width, int64_t height, int32_t pair_option, int32_t quad_option,
                         int32_t temporal_depth, int32_t* depth) {
  if (depth) *depth = 0;
  if (width < 1 || height < 1) return 0;
  const IlChoice c = il_choose(width, height, pair_option, quad_option, temporal_depth);
  if (depth) *depth = c.depth;
  return c.il;
}

int life_packed_launch_kind(int64_t width, int64_t out_rows, int32_t generations) {
  if (width < 1 || out_rows < 1 || generations < 1 || generations > LIFE_MAX_TEMPORAL_DEPTH)
    return -1;
  // Mirrors packed_step (aligned buffers, no trace) -> launch_packed ->
  // launch_packed_deep for a torus pass outside peer mode.
  if (generations == 1 && width % 128 == 0) return LIFE_LAUNCH_STEP1;
  if (generations < 4 || width < 64) return LIFE_LAUNCH_ALL_PATHS;
  if (width % 32 == 0) return LIFE_LAUNCH_FAST;
  const int64_t nw = nw32(width);
  const int64_t strips = ceil_div(nw + 1, kStripStride);
  const int64_t s_last = (nw - 1) / kStripStride;
  const bool many_waves = strips * out_rows >= 2000000;
  if (s_last < 2 || !many_waves || split_disabled()) return LIFE_LAUNCH_ALL_PATHS;
  return LIFE_LAUNCH_SPLIT;
}

int life_ctx_create(int device, life_ctx** out) {
  if (!out) return set_error(LIFE_ERR_CONFIG, "null output pointer");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return set_error(LIFE_ERR_NO_DEVICE, "no CUDA device available (%s)",
                     e == cudaSuccess ? "count 0" : cudaGetErrorString(e));
  if (device < 0 || device >= n)
    return set_error(LIFE_ERR_NO_DEVICE, "device %d out of range [0, %d)", device, n);
  LIFE_CUDA(cudaSetDevice(device));
  life_ctx* c = new life_ctx();
  c->device = device;
  e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaStreamCreate");
  }
  c->stream = c->own;
  *out = c;
  return LIFE_OK;
}

int life_ctx_create_multi(int32_t n, const int* devices, life_ctx** out) {
  if (!out) return set_error(LIFE_ERR_CONFIG, "null output pointer");
  *out = nullptr;
  MultiState* m = nullptr;
  LIFE_TRY(multi_create(n, devices, &m));
  life_ctx* c = new life_ctx();
  c->device = devices[0];
  c->multi = m;
  *out = c;
  return LIFE_OK;
}

int life_ctx_destroy(life_ctx* c) {
  if (!c) return LIFE_OK;
  if (c->multi) {
    multi_destroy(c->multi);
    delete c;
    return LIFE_OK;
  }
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  free_buffers(c);
  if (c->counts) cudaFree(c->counts);
  if (c->row_hashes) cudaFree(c->row_hashes);
  if (c->window) cudaFree(c->window);
  for (auto& b : c->batch)
    if (b) cudaFree(b);
  for (auto& st : c->cs)
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  for (auto& ss : c->split) {
    if (ss.side) cudaStreamSynchronize(ss.side);
    split_streams_destroy(&ss);
  }
  if (c->t0) cudaEventDestroy(c->t0);
  if (c->t1) cudaEventDestroy(c->t1);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
  return LIFE_OK;
}

int life_ctx_set_stream(life_ctx* c, void* stream) {
  if (c && c->multi)
    return set_error(LIFE_ERR_CONFIG,
                     "a multi-device context orders its work on its own per-band streams");
  LIFE_TRY(activate(c));
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own;
  return LIFE_OK;
}

int life_ctx_sync(life_ctx* c) {
  if (c && c->multi) return multi_sync(c->multi);
  LIFE_TRY(activate(c));
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  return LIFE_OK;
}

int life_ctx_set_option(life_ctx* c, int32_t option, int64_t value) {
  if (!c) return set_error(LIFE_ERR_STATE, "null context");
  if (c->multi) return multi_set_option(c->multi, option, value);
  switch (option) {
    case LIFE_OPT_PROFILE:
      c->profile = value != 0;
      return LIFE_OK;
    case LIFE_OPT_BATCH_TRAPEZOID:
      if (value < -1 || value > 1)
        return set_error(LIFE_ERR_CONFIG, "LIFE_OPT_BATCH_TRAPEZOID must be -1, 0 or 1");
      c->batch_trap = static_cast<int>(value);
      return LIFE_OK;
    case LIFE_OPT_HALO:
      return set_error(LIFE_ERR_CONFIG, "LIFE_OPT_HALO applies to multi-device contexts");
    case LIFE_OPT_PAIR_DEPTH:
      if (value < -1 || value > kPairMaxDepthHost)
        return set_error(LIFE_ERR_CONFIG, "LIFE_OPT_PAIR_DEPTH must be in [-1, %d]",
                         kPairMaxDepthHost);
      c->pair_depth = static_cast<int>(value);
      return LIFE_OK;
    case LIFE_OPT_QUAD_DEPTH:
      if (value < -1 || value > kQuadMaxDepthHost)
        return set_error(LIFE_ERR_CONFIG, "LIFE_OPT_QUAD_DEPTH must be in [-1, %d]",
                         kQuadMaxDepthHost);
      c->quad_depth = static_cast<int>(value);
      return LIFE_OK;
    default:
      return set_error(LIFE_ERR_CONFIG, "unknown option %d", option);
  }
}

int life_ctx_get_option(life_ctx* c, int32_t option, int64_t* value) {
  if (!c || !value) return set_error(LIFE_ERR_STATE, "null context or output");
  if (c->multi) return multi_get_option(c->multi, option, value);
  switch (option) {
    case LIFE_OPT_PROFILE: *value = c->profile ? 1 : 0; return LIFE_OK;
    case LIFE_OPT_BATCH_TRAPEZOID: *value = c->batch_trap; return LIFE_OK;
    case LIFE_OPT_PAIR_DEPTH: *value = c->pair_depth; return LIFE_OK;
    case LIFE_OPT_QUAD_DEPTH: *value = c->quad_depth; return LIFE_OK;
    default: return set_error(LIFE_ERR_CONFIG, "unknown option %d", option);
  }
}

int life_ctx_bands(life_ctx* c, int32_t* n, int64_t* bounds, int32_t* devices, int32_t* halo) {
  if (!c) return set_error(LIFE_ERR_STATE, "null context");
  if (c->multi) return multi_bands(c->multi, n, bounds, devices, halo);
  if (n) *n = 1;
  if (bounds) {
    bounds[0] = 0;
    bounds[1] = c->H;
  }
  if (devices) devices[0] = c->device;
  if (halo) *halo = -1;
  return LIFE_OK;
}

int life_ctx_band_stats(life_ctx* c, int32_t band, life_band_stats* out) {
  if (!c || !out) return set_error(LIFE_ERR_STATE, "null context or output");
  if (c->multi) return multi_band_stats(c->multi, band, out);
  if (band != 0) return set_error(LIFE_ERR_CONFIG, "band %d out of range [0, 1)", band);
  *out = life_band_stats{};
  out->band = 0;
  out->device = c->device;
  out->y0 = 0;
  out->rows = c->H;
  out->passes = c->passes;
  out->run_ms = c->run_ms;
  out->interior_ms = c->pass_ms;
  out->edge_ms = 0.0;
  out->wait_ms = c->profile ? c->run_ms - c->pass_ms : 0.0;
  return LIFE_OK;
}

int life_grid_dims(life_ctx* c, int64_t* w, int64_t* h) {
  if (c && c->multi) return multi_dims(c->multi, w, h);
  if (!c) return set_error(LIFE_ERR_STATE, "null context");
  if (c->layout == kNone) return set_error(LIFE_ERR_STATE, "no grid loaded");
  *w = c->W;
  *h = c->H;
  return LIFE_OK;
}

int life_grid_upload_u8(life_ctx* c, const uint8_t* cells, int64_t width, int64_t height,
                        int64_t row_stride) {
  if (c && c->multi) return multi_upload_u8(c->multi, cells, width, height, row_stride);
  LIFE_TRY(activate(c));
  if (!cells) return set_error(LIFE_ERR_CONFIG, "null cell buffer");
  LIFE_TRY(set_dims(c, width, height));
  if (row_stride < width) return set_error(LIFE_ERR_CONFIG, "row_stride < width");
  LIFE_TRY(ensure_byte(c));
  c->by_cur = 0;
  LIFE_CUDA(cudaMemcpy2DAsync(c->by[0], c->by_pitch, cells, row_stride, width, height,
                              cudaMemcpyHostToDevice, c->stream));
  const int64_t n = c->H * c->by_pitch;
  byte_normalise_kernel<<<grid_stride_blocks(n, 256), 256, 0, c->stream>>>(c->by[0], c->by_pitch,
                                                                           width, height);
  LIFE_CHECK_LAUNCH("byte_normalise_kernel");
  c->layout = kByte;
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  return LIFE_OK;
}

int life_grid_upload_packed(life_ctx* c, const uint64_t* words, int64_t width, int64_t height,
                            int64_t words_per_row) {
  if (c && c->multi) return multi_upload_packed(c->multi, words, width, height, words_per_row);
  LIFE_TRY(activate(c));
  if (!words) return set_error(LIFE_ERR_CONFIG, "null word buffer");
  LIFE_TRY(set_dims(c, width, height));
  const int64_t wpr = ceil_div(width, 64);
  if (words_per_row < wpr) return set_error(LIFE_ERR_CONFIG, "words_per_row < ceil(W/64)");
  LIFE_TRY(ensure_packed(c));
  c->pk_cur = 0;
  LIFE_CUDA(cudaMemcpy2DAsync(c->pk[0], c->pk_pitch * 4, words, words_per_row * 8, wpr * 8,
                              height, cudaMemcpyHostToDevice, c->stream));
  const int32_t nw = static_cast<int32_t>(nw32(width));
  const int64_t n = height * (c->pk_pitch - nw + 1);
  packed_mask_tail_kernel<<<grid_stride_blocks(n, 256), 256, 0, c->stream>>>(
      c->pk[0], c->pk_pitch, nw, tail_mask(width), height);
  LIFE_CHECK_LAUNCH("packed_mask_tail_kernel");
  c->layout = kPacked;
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  return LIFE_OK;
}

int life_grid_init_random(life_ctx* c, int64_t width, int64_t height, double density,
                          uint64_t seed, int engine) {
  if (c && c->multi) {
    LIFE_TRY(check_engine(engine));
    return multi_init_random(c->multi, width, height, density, seed);
  }
  LIFE_TRY(activate(c));
  LIFE_TRY(check_engine(engine));
  if (!(density >= 0.0 && density <= 1.0))
    return set_error(LIFE_ERR_CONFIG, "density must be in [0, 1], got %f", density);
  LIFE_TRY(set_dims(c, width, height));
  if (engine != LIFE_ENGINE_BYTE) {
    LIFE_TRY(ensure_packed(c));
    c->pk_cur = 0;
    LIFE_TRY(life_dev_packed_random(c->pk[0], c->pk_pitch, width, 0, height, density, seed,
                                    c->stream));
    c->layout = kPacked;
  } else {
    LIFE_TRY(ensure_byte(c));
    c->by_cur = 0;
    LIFE_TRY(life_dev_byte_random(c->by[0], c->by_pitch, width, 0, height, density, seed,
                                  c->stream));
    c->layout = kByte;
  }
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  return LIFE_OK;
}

int life_grid_init_soup(life_ctx* c, int64_t width, int64_t height, double coverage,
                        int32_t block_size, double density, uint64_t seed, int engine) {
  if (c && c->multi) {
    LIFE_TRY(check_engine(engine));
    return multi_init_soup(c->multi, width, height, coverage, block_size, density, seed);
  }
  LIFE_TRY(activate(c));
  LIFE_TRY(check_engine(engine));
  if (!(density >= 0.0 && density <= 1.0))
    return set_error(LIFE_ERR_CONFIG, "density must be in [0, 1], got %f", density);
  if (!(coverage >= 0.0)) return set_error(LIFE_ERR_CONFIG, "coverage must be >= 0");
  LIFE_TRY(check_dims(width, height));
  if (block_size < 1 || block_size > width || block_size > height)
    return set_error(LIFE_ERR_OUT_OF_BOUNDS, "soup block %d does not fit a %lldx%lld field",
                     block_size, static_cast<long long>(width), static_cast<long long>(height));
  if (width * height >= (int64_t(1) << 40))
    return set_error(LIFE_ERR_CONFIG, "soup field too large for the owner scratch");
  LIFE_TRY(set_dims(c, width, height));
  LIFE_TRY(ensure_byte(c));
  const double bsq = double(block_size) * double(block_size);
  const int64_t blocks = std::llround(coverage * double(width) * double(height) / bsq);
  if (blocks >= (int64_t(1) << 32) - 1) return set_error(LIFE_ERR_CONFIG, "too many soup blocks");
  unsigned int* owner = nullptr;
  LIFE_CUDA(cudaMallocAsync(&owner, sizeof(unsigned int) * width * height, c->stream));
  LIFE_CUDA(cudaMemsetAsync(owner, 0, sizeof(unsigned int) * width * height, c->stream));
  LIFE_CUDA(cudaMemsetAsync(c->by[0], 0, static_cast<size_t>(c->by_pitch) * height, c->stream));
  c->by_cur = 0;
  const int64_t n = blocks * block_size * block_size;
  if (n > 0) {
    soup_claim_kernel<<<grid_stride_blocks(n, 256), 256, 0, c->stream>>>(owner, width, height,
                                                                        blocks, block_size, seed);
    LIFE_CHECK_LAUNCH("soup_claim_kernel");
    soup_write_kernel<<<grid_stride_blocks(n, 256), 256, 0, c->stream>>>(
        owner, c->by[0], c->by_pitch, width, height, blocks, block_size, seed,
        density_threshold(density));
    LIFE_CHECK_LAUNCH("soup_write_kernel");
  }
  LIFE_CUDA(cudaFreeAsync(owner, c->stream));
  c->layout = kByte;
  if (engine != LIFE_ENGINE_BYTE) LIFE_TRY(to_layout(c, kPacked));
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  return LIFE_OK;
}

int life_grid_place_u8(life_ctx* c, const uint8_t* pattern, int64_t pw, int64_t ph, int64_t x0,
                       int64_t y0) {
  if (c && c->multi) return multi_place_u8(c->multi, pattern, pw, ph, x0, y0);
  LIFE_TRY(activate(c));
  if (c->layout == kNone) return set_error(LIFE_ERR_STATE, "no grid loaded");
  if (pw < 0 || ph < 0 || (pw * ph > 0 && !pattern))
    return set_error(LIFE_ERR_CONFIG, "bad pattern buffer");
  if (x0 < 0 || y0 < 0 || x0 + pw > c->W || y0 + ph > c->H)
    return set_error(LIFE_ERR_OUT_OF_BOUNDS,
                     "pattern footprint %lldx%lld at (%lld, %lld) exceeds grid %lldx%lld",
                     static_cast<long long>(pw), static_cast<long long>(ph),
                     static_cast<long long>(x0), static_cast<long long>(y0),
                     static_cast<long long>(c->W), static_cast<long long>(c->H));
  if (pw * ph == 0) return LIFE_OK;
  LIFE_TRY(pk_plain(c));
  uint8_t* dpat = nullptr;
  LIFE_CUDA(cudaMallocAsync(&dpat, pw * ph, c->stream));
  LIFE_CUDA(cudaMemcpyAsync(dpat, pattern, pw * ph, cudaMemcpyHostToDevice, c->stream));
  if (c->layout == kByte) {
    place_byte_kernel<<<grid_stride_blocks(pw * ph, 256), 256, 0, c->stream>>>(
        c->by[c->by_cur], c->by_pitch, dpat, pw, ph, x0, y0);
  } else {
    const int64_t n = (((x0 + pw - 1) >> 5) - (x0 >> 5) + 1) * ph;
    place_packed_kernel<<<grid_stride_blocks(n, 256), 256, 0, c->stream>>>(
        c->pk[c->pk_cur], c->pk_pitch, dpat, pw, ph, x0, y0);
  }
  LIFE_CHECK_LAUNCH("place_kernel");
  LIFE_CUDA(cudaFreeAsync(dpat, c->stream));
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  return LIFE_OK;
}

int life_grid_download_u8(life_ctx* c, uint8_t* cells, int64_t row_stride) {
  if (c && c->multi) return multi_download_u8(c->multi, cells, row_stride);
  LIFE_TRY(activate(c));
  if (c->layout == kNone) return set_error(LIFE_ERR_STATE, "no grid loaded");
  if (!cells || row_stride < c->W) return set_error(LIFE_ERR_CONFIG, "bad output buffer");
  LIFE_TRY(pk_plain(c));
  const uint8_t* src;
  if (c->layout == kByte) {
    src = c->by[c->by_cur];
  } else {  // unpack into the (free) byte buffer
    LIFE_TRY(ensure_byte(c));
    LIFE_TRY(life_dev_unpack(c->pk[c->pk_cur], c->pk_pitch, c->by[0], c->by_pitch, c->W, c->H,
                             c->stream));
    src = c->by[0];
  }
  LIFE_CUDA(cudaMemcpy2DAsync(cells, row_stride, src, c->by_pitch, c->W, c->H,
                              cudaMemcpyDeviceToHost, c->stream));
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  return LIFE_OK;
}

int life_grid_download_packed(life_ctx* c, uint64_t* words, int64_t words_per_row) {
  if (c && c->multi) return multi_download_packed(c->multi, words, words_per_row);
  LIFE_TRY(activate(c));
  if (c->layout == kNone) return set_error(LIFE_ERR_STATE, "no grid loaded");
  const int64_t wpr = ceil_div(c->W, 64);
  if (!words || words_per_row < wpr) return set_error(LIFE_ERR_CONFIG, "bad output buffer");
  LIFE_TRY(pk_plain(c));
  const uint32_t* src;
  if (c->layout == kPacked) {
    src = c->pk[c->pk_cur];
  } else {  // pack into the (free) packed buffer
    LIFE_TRY(ensure_packed(c));
    LIFE_TRY(life_dev_pack(c->by[c->by_cur], c->by_pitch, c->pk[0], c->pk_pitch, c->W, c->H,
                           c->stream));
    src = c->pk[0];
  }
  LIFE_CUDA(cudaMemcpy2DAsync(words, words_per_row * 8, src, c->pk_pitch * 4, wpr * 8, c->H,
                              cudaMemcpyDeviceToHost, c->stream));
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  return LIFE_OK;
}

int life_grid_window_u8(life_ctx* c, int64_t x0, int64_t y0, int64_t w, int64_t h, uint8_t* out) {
  if (c && c->multi) return multi_window_u8(c->multi, x0, y0, w, h, out);
  LIFE_TRY(activate(c));
  if (c->layout == kNone) return set_error(LIFE_ERR_STATE, "no grid loaded");
  if (w < 0 || h < 0 || !out) return set_error(LIFE_ERR_CONFIG, "bad window");
  const int64_t n = w * h;
  if (n == 0) return LIFE_OK;
  LIFE_TRY(pk_plain(c));
  if (n > c->window_cap) {
    if (c->window) cudaFree(c->window);
    c->window = nullptr;
    LIFE_CUDA(cudaMalloc(&c->window, n));
    c->window_cap = n;
  }
  if (c->layout == kPacked) {
    packed_window_kernel<<<grid_stride_blocks(n, 256), 256, 0, c->stream>>>(
        c->pk[c->pk_cur], c->pk_pitch, c->W, c->H, x0, y0, w, h, c->window);
  } else {
    byte_window_kernel<<<grid_stride_blocks(n, 256), 256, 0, c->stream>>>(
        c->by[c->by_cur], c->by_pitch, c->W, c->H, x0, y0, w, h, c->window);
  }
  LIFE_CHECK_LAUNCH("window_kernel");
  LIFE_CUDA(cudaMemcpyAsync(out, c->window, n, cudaMemcpyDeviceToHost, c->stream));
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  return LIFE_OK;
}

int life_population(life_ctx* c, uint64_t* out) {
  if (c && c->multi) return multi_population(c->multi, out);
  LIFE_TRY(activate(c));
  if (c->layout == kNone) return set_error(LIFE_ERR_STATE, "no grid loaded");
  LIFE_TRY(ensure_counts(c, 1));
  LIFE_TRY(population_async(c, c->counts));
  LIFE_CUDA(cudaMemcpyAsync(out, c->counts, 8, cudaMemcpyDeviceToHost, c->stream));
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  return LIFE_OK;
}

int life_grid_hash(life_ctx* c, uint64_t* out) {
  if (c && c->multi) return multi_hash(c->multi, out);
  LIFE_TRY(activate(c));
  if (!out) return set_error(LIFE_ERR_CONFIG, "null output pointer");
  if (c->layout == kNone) return set_error(LIFE_ERR_STATE, "no grid loaded");
  LIFE_TRY(to_layout(c, kPacked));
  LIFE_TRY(pk_plain(c));
  if (c->H > c->row_hashes_cap) {
    if (c->row_hashes) cudaFree(c->row_hashes);
    c->row_hashes = nullptr;
    LIFE_CUDA(cudaMalloc(&c->row_hashes, sizeof(uint64_t) * c->H));
    c->row_hashes_cap = c->H;
  }
  LIFE_TRY(life_dev_packed_row_hashes(c->pk[c->pk_cur], c->pk_pitch, c->W, c->H, c->row_hashes,
                                      c->stream));
  std::vector<uint64_t> rows(static_cast<size_t>(c->H));
  LIFE_CUDA(cudaMemcpyAsync(rows.data(), c->row_hashes, sizeof(uint64_t) * c->H,
                            cudaMemcpyDeviceToHost, c->stream));
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  *out = life_fnv1a64(rows.data(), static_cast<int64_t>(rows.size() * sizeof(uint64_t)), 0);
  return LIFE_OK;
}

int life_run(life_ctx* c, int64_t generations, int engine, int temporal_depth,
             const int64_t* checkpoints, int32_t n_checkpoints, uint64_t* populations) {
  if (c && c->multi) {
    LIFE_TRY(check_engine(engine));
    return multi_run(c->multi, generations, engine, temporal_depth, checkpoints, n_checkpoints,
                     populations);
  }
  LIFE_TRY(activate(c));
  LIFE_TRY(check_engine(engine));
  LIFE_TRY(check_run_args(generations, checkpoints, n_checkpoints, populations));
  int depth = temporal_depth;
  int il = 0;  // 2 / 4: passes on the pair / quad layout
  if (engine != LIFE_ENGINE_BYTE) {
    if (depth < 0 || depth > LIFE_MAX_TEMPORAL_DEPTH)
      return set_error(LIFE_ERR_CONFIG, "temporal depth must be in [0, %d], got %d",
                       LIFE_MAX_TEMPORAL_DEPTH, temporal_depth);
    if (c->layout == kNone) return set_error(LIFE_ERR_STATE, "no grid loaded");
    if (engine == LIFE_ENGINE_PACKED && depth == 0 && resident_auto(c->W, c->H))
      engine = LIFE_ENGINE_RESIDENT;
    if (engine == LIFE_ENGINE_RESIDENT && life_resident_cluster_size(c->W, c->H) == 0)
      return set_error(LIFE_ERR_CONFIG,
                       "a %lldx%lld torus does not fit the cluster-resident engine "
                       "(needs W %% 32 == 0 and every band in one CTA's shared memory)",
                       static_cast<long long>(c->W), static_cast<long long>(c->H));
    if (depth == 0) depth = packed_auto_depth(c->W, c->H);
    // Pair / quad layout kernels: forced by LIFE_OPT_PAIR_DEPTH / _QUAD_DEPTH,
    // or the auto rule's choice when the caller left the depth to the engine.
    if (engine == LIFE_ENGINE_PACKED) {
      const IlChoice ch = il_choose(c->W, c->H, c->pair_depth, c->quad_depth, temporal_depth);
      if (ch.il != 0) {
        il = ch.il;
        depth = ch.depth;
      }
    }
  } else {
    // Byte engine: K generations per pass (byte_tb2_kernel) when W % 16 == 0 or
    // W >= 33 (the seam path);
    // other widths run one generation per pass whatever the depth asks.
    if (depth < 0 || depth > kByteTbMaxDepth)
      return set_error(LIFE_ERR_CONFIG, "byte engine temporal depth must be in [0, %d], got %d",
                       kByteTbMaxDepth, temporal_depth);
    if (depth == 0) depth = byte_auto_depth(c->W, c->H);
    if (c->W % 16 != 0 && c->W < kByteTbMinSeamWidth) depth = 1;
  }
  if (c->layout == kNone) return set_error(LIFE_ERR_STATE, "no grid loaded");
  LIFE_TRY(to_layout(c, engine_layout(engine)));
  if (il != 0 && generations > 0) {
    LIFE_TRY(pk_to_il(c, il));
  } else if (generations > 0 || engine != LIFE_ENGINE_PACKED) {
    LIFE_TRY(pk_plain(c));
  }
  if (n_checkpoints > 0) LIFE_TRY(ensure_counts(c, n_checkpoints));
  LIFE_TRY(split_streams_init(&c->split[0], c->device));
  if (!c->t0) LIFE_CUDA(cudaEventCreate(&c->t0));
  if (!c->t1) LIFE_CUDA(cudaEventCreate(&c->t1));
  // LIFE_OPT_PROFILE: CUDA events around every pass (life_ctx_band_stats).
  struct PassEvents {
    std::vector<cudaEvent_t> v;
    ~PassEvents() {
      for (cudaEvent_t e : v) cudaEventDestroy(e);
    }
  } prof;
  auto prof_mark = [&]() -> int {
    if (!c->profile) return LIFE_OK;
    cudaEvent_t e;
    LIFE_CUDA(cudaEventCreate(&e));
    prof.v.push_back(e);
    LIFE_CUDA(cudaEventRecord(e, c->stream));
    return LIFE_OK;
  };

  int32_t ci = 0;
  auto record = [&](int64_t gen) -> int {
    while (ci < n_checkpoints && checkpoints[ci] == gen) {
      LIFE_TRY(population_async(c, c->counts + ci));
      ++ci;
    }
    return LIFE_OK;
  };
  LIFE_TRY(record(0));
  c->passes = 0;
  LIFE_CUDA(cudaEventRecord(c->t0, c->stream));
  int64_t done = 0;
  while (done < generations) {
    const int64_t stop = ci < n_checkpoints ? checkpoints[ci] : generations;
    LIFE_TRY(prof_mark());
    if (engine == LIFE_ENGINE_RESIDENT) {  // every generation up to the next stop in one launch
      LIFE_TRY(life_dev_packed_run_resident(c->pk[c->pk_cur], c->pk[c->pk_cur ^ 1], c->pk_pitch,
                                            c->W, c->H, stop - done, c->stream));
      c->pk_cur ^= 1;
      done = stop;
      ++c->passes;
      LIFE_TRY(prof_mark());
      LIFE_TRY(record(done));
      continue;
    }
    if (engine == LIFE_ENGINE_PACKED && !c->profile && stop - done >= 2 * int64_t(depth)) {
      // Every generation up to the next stop (packed_run: full passes, then
      // the remainder).
      int flip = 0;
      LIFE_TRY(packed_run(c->pk[c->pk_cur], c->pk[c->pk_cur ^ 1], c->pk_pitch, c->W, c->H,
                          stop - done, depth, c->stream, &c->split[0], &flip, c->pk_il));
      c->pk_cur ^= flip;
      c->passes += ceil_div(stop - done, int64_t(depth));
      done = stop;
      LIFE_TRY(prof_mark());
      LIFE_TRY(record(done));
      continue;
    }
    const int step = static_cast<int>(std::min<int64_t>(depth, stop - done));
    if (engine == LIFE_ENGINE_PACKED) {
      const int nxt = c->pk_cur ^ 1;
      if (c->pk_il != 0) {
        LIFE_TRY(packed_il_step(c->pk_il, c->pk[c->pk_cur], c->pk_pitch, 0, c->H, c->pk[nxt],
                                c->pk_pitch, 0, c->W, c->H, step, c->stream));
      } else {
        LIFE_TRY(packed_step(c->pk[c->pk_cur], c->pk_pitch, 0, c->H, c->pk[nxt], c->pk_pitch, 0,
                             c->W, c->H, step, c->stream, &c->split[0]));
      }
      c->pk_cur = nxt;
    } else {
      const int nxt = c->by_cur ^ 1;
      LIFE_TRY(life_dev_byte_pass(c->by[c->by_cur], c->by_pitch, 0, c->H, c->by[nxt],
                                  c->by_pitch, 0, c->W, c->H, step, c->stream));
      c->by_cur = nxt;
    }
    done += step;
    ++c->passes;
    LIFE_TRY(prof_mark());
    LIFE_TRY(record(done));
  }
  LIFE_CUDA(cudaEventRecord(c->t1, c->stream));
  if (n_checkpoints > 0) {
    LIFE_CUDA(cudaMemcpyAsync(populations, c->counts, sizeof(uint64_t) * n_checkpoints,
                              cudaMemcpyDeviceToHost, c->stream));
  }
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  float ms = 0.0f;
  LIFE_CUDA(cudaEventElapsedTime(&ms, c->t0, c->t1));
  c->run_ms = ms;
  c->pass_ms = 0.0;
  for (size_t i = 0; i + 1 < prof.v.size(); i += 2) {
    LIFE_CUDA(cudaEventElapsedTime(&ms, prof.v[i], prof.v[i + 1]));
    c->pass_ms += ms;
  }
  return LIFE_OK;
}

int life_step(life_ctx* c, int engine) { return life_run(c, 1, engine, 1, nullptr, 0, nullptr); }

namespace {
// ---- life_run_batch: trapezoid / triangle schedule for the first and last grid
//
// With whole-grid passes, the first grid's upload and the last grid's
// download (8 GiB each at config 5) are exposed.  The first and last grid of
// a batch are instead cut into kTrapChunks row chunks.  Chunk c's TRAPEZOID
// runs all P passes on its own rows only, pass p producing the rows
// [start + kShrink*(p+1), end - kShrink*(p+1)) (each pass loses kShrink = K,
// the pass depth, rows per side of valid data), so it starts as soon as
// chunk c has arrived and its interior can leave as soon as it is done.  The
// TRIANGLE at the boundary row B between chunks c-1 and c then runs the P
// passes on [B - kShrink*(p+1), B + kShrink*(p+1)), reading the trapezoids'
// outputs of the previous pass.  No launch overwrites rows another still
// needs: trapezoid pass p+1 writes the buffer of pass p-1 only below
// B - kShrink*(p+2), exactly where triangle pass p stops reading; triangles
// run after both neighbouring trapezoids.  Middle grids keep whole-grid
// passes (their copies overlap the neighbouring grids' compute anyway).
//
// Chunk heights (round 2): only the chunks whose own copy is exposed need to
// be small -- the first ones of a grid no earlier grid computes behind, the
// last ones of a grid no later grid computes behind.  A chunk computes
// `growth` times longer than it takes to copy (generations x ~0.009: PCIe
// moves ~4e11 cells/s, the kernels ~4.5e13 cell-updates/s), so each chunk may
// be up to that much taller than the one before it and still find its rows
// arrived: heights grow geometrically from the exposed end(s) and the rest
// of the grid is one chunk -- 7 chunks for one config-5 grid instead of 32
// equal ones, a quarter of the launches, and most rows run in tall
// trapezoids at whole-grid speed.  (32 equal chunks, the round-1 schedule:
// e2e / value 0.967 at K = 16 but 0.936 at the quad kernel's K = 6, whose 84
// passes make 5376 small launches per chunked grid.)  Few generations per
// byte copied (growth < 1.5) keep equal chunks.
#ifndef LIFE_TRAP_CHUNKS
#define LIFE_TRAP_CHUNKS 32  // most chunks per grid (equal chunks: 8 0.945, 16 0.953, 32 0.967, 48 0.955)
#endif
constexpr int kTrapChunks = LIFE_TRAP_CHUNKS;
#ifndef LIFE_TRAP_MIN_ROWS
#define LIFE_TRAP_MIN_ROWS 8192  // equal chunks shorter than this run their passes too slowly
#endif
constexpr int64_t kTrapMinChunkRows = LIFE_TRAP_MIN_ROWS;
constexpr int kSmallFirst = 1, kSmallLast = 2;

// Cut points of a chunked grid into bounds[0..n]; returns n (0: does not fit).
// min_rows: the shortest chunk (its trapezoid must survive every pass).
int plan_chunks(int64_t height, int64_t min_rows, double growth, int profile, int64_t* bounds) {
  std::vector<int64_t> head, tail;
  int64_t rem = height, cur = min_rows;
  while (true) {
    const int64_t last = head.empty() ? (tail.empty() ? 0 : tail.back()) : head.back();
    const int64_t need = ((profile & kSmallFirst) ? cur : 0) + ((profile & kSmallLast) ? cur : 0);
    if (last > 0 && static_cast<double>(rem) <= growth * static_cast<double>(last)) break;
    if (rem - need < min_rows || static_cast<int>(head.size() + tail.size()) + 3 > kTrapChunks) break;
    if (profile & kSmallFirst) head.push_back(cur);
    if (profile & kSmallLast) tail.push_back(cur);
    rem -= need;
    cur = static_cast<int64_t>(std::min(static_cast<double>(cur) * growth, 4e18));
  }
  if (head.empty() && tail.empty()) return 0;
  int n = 0;
  bounds[0] = 0;
  for (int64_t v : head) {
    bounds[n + 1] = bounds[n] + v;
    ++n;
  }
  bounds[n + 1] = bounds[n] + rem;  // the rest of the grid: one chunk
  ++n;
  for (auto it = tail.rbegin(); it != tail.rend(); ++it) {
    bounds[n + 1] = bounds[n] + *it;
    ++n;
  }
  return n;
}

struct BatchGeom {
  int64_t width, height, wpr, words_per_row, pitch, generations;
  int depth, passes;
  int il;  // 2 / 4: passes on the pair / quad layout (zip after upload, unzip before download)
  int nchunks;  // chunks of the grid being scheduled
  int64_t bounds[kTrapChunks + 1];
};

// out rows [r0, r0 + rows) (mod H) of pass p: one launch per contiguous piece.
int pass_rows(const BatchGeom& g, uint32_t* const* buf, int p, int64_t r0, int64_t rows,
              cudaStream_t s, SplitStreams* ss) {
  const int k = static_cast<int>(std::min<int64_t>(g.depth, g.generations - int64_t(p) * g.depth));
  r0 %= g.height;
  if (r0 < 0) r0 += g.height;
  while (rows > 0) {
    const int64_t piece = std::min(rows, g.height - r0);
    if (g.il != 0) {
      LIFE_TRY(packed_il_step(g.il, buf[p & 1], g.pitch, r0, g.height, buf[(p & 1) ^ 1], g.pitch,
                              r0, g.width, piece, k, s));
    } else {
      LIFE_TRY(packed_step(buf[p & 1], g.pitch, r0, g.height, buf[(p & 1) ^ 1], g.pitch, r0,
                           g.width, piece, k, s, ss));
    }
    rows -= piece;
    r0 = 0;
  }
  return LIFE_OK;
}

// Layout conversion of rows [r0, r0 + rows) (mod H) of a batch buffer.
int zip_rows(const BatchGeom& g, uint32_t* buf, int64_t r0, int64_t rows, bool unzip,
             cudaStream_t s) {
  r0 %= g.height;
  if (r0 < 0) r0 += g.height;
  while (rows > 0) {
    const int64_t piece = std::min(rows, g.height - r0);
    LIFE_TRY(packed_zip(g.il, buf, g.pitch, g.width, r0, piece, unzip, s));
    rows -= piece;
    r0 = 0;
  }
  return LIFE_OK;
}

int copy_rows(const BatchGeom& g, void* host, const uint32_t* dev, int64_t r0, int64_t rows,
              bool h2d, cudaStream_t s) {
  r0 %= g.height;
  if (r0 < 0) r0 += g.height;
  while (rows > 0) {
    const int64_t piece = std::min(rows, g.height - r0);
    uint64_t* hrow = static_cast<uint64_t*>(host) + r0 * g.words_per_row;
    uint32_t* drow = const_cast<uint32_t*>(dev) + r0 * g.pitch;
    if (h2d) {
      LIFE_CUDA(cudaMemcpy2DAsync(drow, g.pitch * 4, hrow, g.words_per_row * 8, g.wpr * 8, piece,
                                  cudaMemcpyHostToDevice, s));
    } else {
      LIFE_CUDA(cudaMemcpy2DAsync(hrow, g.words_per_row * 8, drow, g.pitch * 4, g.wpr * 8, piece,
                                  cudaMemcpyDeviceToHost, s));
    }
    rows -= piece;
    r0 = 0;
  }
  return LIFE_OK;
}
}  // namespace

int life_run_batch(life_ctx* c, const uint64_t* const* inputs, uint64_t* const* outputs, int32_t n,
                   int64_t width, int64_t height, int64_t words_per_row, int64_t generations,
                   int temporal_depth, float* elapsed_ms) {
  if (c && c->multi)
    return multi_run_batch(c->multi, inputs, outputs, n, width, height, words_per_row,
                           generations, temporal_depth, elapsed_ms);
  LIFE_TRY(activate(c));
  LIFE_TRY(check_dims(width, height));
  if (n < 0 || (n > 0 && (!inputs || !outputs)))
    return set_error(LIFE_ERR_CONFIG, "bad batch buffers");
  if (generations < 0)
    return set_error(LIFE_ERR_CONFIG, "iteration count must be non-negative, got %lld",
                     static_cast<long long>(generations));
  int depth = temporal_depth == 0 ? packed_auto_depth(width, height) : temporal_depth;
  if (depth < 1 || depth > LIFE_MAX_TEMPORAL_DEPTH)
    return set_error(LIFE_ERR_CONFIG, "temporal depth must be in [0, %d], got %d",
                     LIFE_MAX_TEMPORAL_DEPTH, temporal_depth);
  // temporal_depth 0 on a small W % 32 == 0 torus: the cluster-resident engine
  // (as life_run's auto mode), one launch per grid.
  const bool resident = temporal_depth == 0 && resident_auto(width, height);
  // Pair / quad layout kernels, chosen as in life_run: the grids are converted
  // on the device after their upload and before their download.
  int il = 0;
  if (!resident && generations > 0) {
    const IlChoice ch = il_choose(width, height, c->pair_depth, c->quad_depth, temporal_depth);
    if (ch.il != 0) {
      il = ch.il;
      depth = ch.depth;
    }
  }
  const int64_t wpr = ceil_div(width, 64);
  if (words_per_row < wpr) return set_error(LIFE_ERR_CONFIG, "words_per_row < ceil(W/64)");
  if (n == 0) return LIFE_OK;
  const int64_t pitch = life_packed_pitch_words(width);
  const size_t bytes = static_cast<size_t>(pitch) * height * 4;
  if (c->batch_bytes != bytes) {
    for (auto& b : c->batch) {
      if (b) cudaFree(b);
      b = nullptr;
    }
    c->batch_bytes = 0;
    for (auto& b : c->batch) {
      LIFE_CUDA(cudaMalloc(&b, bytes));
      LIFE_CUDA(cudaMemsetAsync(b, 0, bytes, c->stream));
    }
    c->batch_bytes = bytes;
    LIFE_CUDA(cudaStreamSynchronize(c->stream));
  }
  for (auto& ss : c->split) LIFE_TRY(split_streams_init(&ss, c->device));
  if (!c->h2d) LIFE_CUDA(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
  if (!c->d2h) LIFE_CUDA(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
  BatchGeom g{};
  g.width = width;
  g.height = height;
  g.wpr = wpr;
  g.words_per_row = words_per_row;
  g.pitch = pitch;
  g.generations = generations;
  g.depth = depth;
  g.il = il;
  g.passes = static_cast<int>(ceil_div(generations, depth));
  // Chunked first/last grid when every chunk outlives its shrinking
  // trapezoid with room to spare.  LIFE_OPT_BATCH_TRAPEZOID 0 / 1 forces it
  // off / on (when it fits); auto: grids of 32768 rows or more.
  const int64_t kShrink = depth;  // rows per side a pass gives up
  const int trap_env = c->batch_trap;
  const int64_t min_chunk = std::max<int64_t>(2 * kShrink * g.passes + 1024, 2048);
  const double growth = std::min(std::max(double(generations) * 0.007, 1.0), 6.0);
  const bool geometric = growth >= 1.5;
  // Plans for a grid that is first, last, or both: the chunk count of the
  // most demanding one decides whether the schedule fits.
  auto plan = [&](int profile, int64_t* bounds) -> int {
    if (geometric) return plan_chunks(height, min_chunk, growth, profile, bounds);
    if (height / kTrapChunks < min_chunk) return 0;
    return life_band_bounds(height, kTrapChunks, bounds) == LIFE_OK ? kTrapChunks : 0;
  };
  const bool fits = n >= 1 && generations > 0 && !resident &&
                    plan(n == 1 ? (kSmallFirst | kSmallLast) : kSmallFirst, g.bounds) >= 2;
  const bool tall = geometric ? height >= 32768 : height / kTrapChunks >= kTrapMinChunkRows;
  const bool trap = fits && (trap_env == 1 || (trap_env != 0 && tall));
  if (trap) {
    for (auto& st : c->cs)
      if (!st) LIFE_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  }
  // Every event is destroyed on every exit path (errors included).
  struct Events {
    std::vector<cudaEvent_t> v;
    ~Events() {
      for (cudaEvent_t e : v) cudaEventDestroy(e);
    }
  } evs;
  auto mk = [&](cudaEvent_t* e, unsigned flags = cudaEventDisableTiming) -> int {
    LIFE_CUDA(cudaEventCreateWithFlags(e, flags));
    evs.v.push_back(*e);
    return LIFE_OK;
  };
  std::vector<cudaEvent_t> up(n), comp(n), down(n);
  for (int32_t i = 0; i < n; ++i) {
    LIFE_TRY(mk(&up[i]));
    LIFE_TRY(mk(&comp[i]));
    LIFE_TRY(mk(&down[i]));
  }
  // LIFE_BATCH_TRACE (debug builds): timed chunk events of the last chunked grid on stderr.
  static const bool trace_chunks = knob("LIFE_BATCH_TRACE", 0) != 0;
  const unsigned chunk_flags = trace_chunks ? cudaEventDefault : cudaEventDisableTiming;
  cudaEvent_t chunk_up[kTrapChunks], trap_done[kTrapChunks], tri_done[kTrapChunks],
      chunk_down[kTrapChunks], strip_down[kTrapChunks];
  if (trap) {
    for (int i = 0; i < kTrapChunks; ++i) {
      LIFE_TRY(mk(&chunk_up[i], chunk_flags));
      LIFE_TRY(mk(&trap_done[i], chunk_flags));
      LIFE_TRY(mk(&tri_done[i], chunk_flags));
      if (trace_chunks) {
        LIFE_TRY(mk(&chunk_down[i], chunk_flags));
        LIFE_TRY(mk(&strip_down[i], chunk_flags));
      }
    }
  }
  int traced_nc = 0;
  int64_t traced_bounds[kTrapChunks + 1] = {0};
  cudaEvent_t t0, t1;
  LIFE_TRY(mk(&t0, cudaEventDefault));
  LIFE_TRY(mk(&t1, cudaEventDefault));
  const int32_t nw = static_cast<int32_t>(nw32(width));
  const int P = g.passes;
  LIFE_CUDA(cudaEventRecord(t0, c->h2d));
  int rc = LIFE_OK;
  // The passes of consecutive grids run one grid after another: each grid
  // fills the GPU by itself, and passes of two grids launched side by side
  // (programmatic dependent launch) park early blocks of the one on the SMs
  // the other could be using (config 5, 3 grids: 2.17 s side by side, against
  // 1.94 s of passes).  main_done: the previous grid's whole-grid passes, or
  // its trapezoids and triangles, are complete.  (Triangles left running
  // beside the next grid's passes get an SM only at its block-wave
  // boundaries: their 84 small launches then outlast it, and the grid after
  // it, which reuses the chunked grid's buffers, uploads late.)
  cudaEvent_t main_done = nullptr;
  cudaEvent_t tri_join[2] = {nullptr, nullptr};
  if (trap)
    for (auto& e : tri_join) LIFE_TRY(mk(&e));
  for (int32_t i = 0; i < n && rc == LIFE_OK; ++i) {
    uint32_t* buf[2] = {c->batch[2 * (i & 1)], c->batch[2 * (i & 1) + 1]};
    // Upload grid i into its slot once grid i-2 has left it.
    if (i >= 2) LIFE_CUDA(cudaStreamWaitEvent(c->h2d, down[i - 2], 0));
    // Chunk plan of a first / last grid (small chunks where its own copy is exposed).
    const int nc = trap && (i == 0 || i == n - 1)
                       ? plan((i == 0 ? kSmallFirst : 0) | (i == n - 1 ? kSmallLast : 0), g.bounds)
                       : 0;
    const bool chunked = nc >= 2;
    if (!chunked) {
      LIFE_CUDA(cudaMemcpy2DAsync(buf[0], pitch * 4, inputs[i], words_per_row * 8, wpr * 8, height,
                                  cudaMemcpyHostToDevice, c->h2d));
      LIFE_CUDA(cudaEventRecord(up[i], c->h2d));
      // Compute on the context stream.
      LIFE_CUDA(cudaStreamWaitEvent(c->stream, up[i], 0));
      if (main_done) LIFE_CUDA(cudaStreamWaitEvent(c->stream, main_done, 0));
      const int64_t mask_n = height * (pitch - nw + 1);
      packed_mask_tail_kernel<<<grid_stride_blocks(mask_n, 256), 256, 0, c->stream>>>(
          buf[0], pitch, nw, tail_mask(width), height);
      LIFE_CHECK_LAUNCH("packed_mask_tail_kernel");
      if (resident) {  // small torus: every generation in one cluster-resident launch
        rc = life_dev_packed_run_resident(buf[0], buf[1], pitch, width, height, generations,
                                          c->stream);
      } else {
        if (g.il != 0) LIFE_TRY(zip_rows(g, buf[0], 0, height, /*unzip=*/false, c->stream));
        for (int p = 0; p < P && rc == LIFE_OK; ++p) rc = pass_rows(g, buf, p, 0, height, c->stream, &c->split[0]);
        if (g.il != 0 && rc == LIFE_OK) rc = zip_rows(g, buf[P & 1], 0, height, /*unzip=*/true, c->stream);
      }
      LIFE_CUDA(cudaEventRecord(comp[i], c->stream));
      main_done = comp[i];
      // Download on the D2H stream.
      LIFE_CUDA(cudaStreamWaitEvent(c->d2h, comp[i], 0));
      LIFE_CUDA(cudaMemcpy2DAsync(outputs[i], words_per_row * 8, buf[resident ? 1 : (P & 1)],
                                  pitch * 4, wpr * 8, height, cudaMemcpyDeviceToHost, c->d2h));
      LIFE_CUDA(cudaEventRecord(down[i], c->d2h));
      continue;
    }
    g.nchunks = nc;
    const int64_t shrink = kShrink * P;  // rows per side the trapezoid gives up
    for (int ch = 0; ch < nc; ++ch) {
      const int64_t y0 = g.bounds[ch], rows = g.bounds[ch + 1] - y0;
      LIFE_TRY(copy_rows(g, const_cast<uint64_t*>(inputs[i]), buf[0], y0, rows, true, c->h2d));
      LIFE_CUDA(cudaEventRecord(chunk_up[ch], c->h2d));
    }
    // Trapezoids in chunk order on one stream (so they finish one after
    // another and their interiors leave early), each as soon as its chunk has
    // arrived; triangles on two other streams, each as soon as its two
    // trapezoids are done.
    if (main_done) LIFE_CUDA(cudaStreamWaitEvent(c->cs[0], main_done, 0));
    for (int ch = 0; ch < nc && rc == LIFE_OK; ++ch) {
      cudaStream_t st = c->cs[0];  // one after another: a chunk's rows leave as early as possible
      const int64_t y0 = g.bounds[ch], rows = g.bounds[ch + 1] - y0;
      LIFE_CUDA(cudaStreamWaitEvent(st, chunk_up[ch], 0));
      const int64_t mask_n = rows * (pitch - nw + 1);
      packed_mask_tail_kernel<<<grid_stride_blocks(mask_n, 256), 256, 0, st>>>(
          buf[0] + y0 * pitch, pitch, nw, tail_mask(width), rows);
      LIFE_CHECK_LAUNCH("packed_mask_tail_kernel");
      if (g.il != 0) LIFE_TRY(zip_rows(g, buf[0], y0, rows, /*unzip=*/false, st));
      for (int p = 0; p < P && rc == LIFE_OK; ++p)
        rc = pass_rows(g, buf, p, y0 + kShrink * (p + 1), rows - 2 * kShrink * (p + 1), st,
                       &c->split[1]);
      // The interior leaves in the plain layout; the triangles never read
      // these rows of the final buffer (their last read of it, pass P-2,
      // stays within kShrink * P rows of the boundary).
      if (g.il != 0 && rc == LIFE_OK)
        rc = zip_rows(g, buf[P & 1], y0 + shrink, rows - 2 * shrink, /*unzip=*/true, st);
      LIFE_CUDA(cudaEventRecord(trap_done[ch], st));
    }
    // Triangles at boundary b (row bounds[b]) between chunks b-1 and b.
    for (int bi = 1; bi <= nc && rc == LIFE_OK; ++bi) {
      const int b = bi % nc;  // boundary 0 (the torus seam) needs the last chunk: last
      cudaStream_t st = c->cs[2 + bi % 2];
      LIFE_CUDA(cudaStreamWaitEvent(st, trap_done[(b + nc - 1) % nc], 0));
      LIFE_CUDA(cudaStreamWaitEvent(st, trap_done[b], 0));
      for (int p = 0; p < P && rc == LIFE_OK; ++p)
        rc = pass_rows(g, buf, p, g.bounds[b] - kShrink * (p + 1), 2 * kShrink * (p + 1), st,
                       &c->split[3 + bi % 2]);
      if (g.il != 0 && rc == LIFE_OK)
        rc = zip_rows(g, buf[P & 1], g.bounds[b] - shrink, 2 * shrink, /*unzip=*/true, st);
      LIFE_CUDA(cudaEventRecord(tri_done[b], st));
    }
    // The next grid's passes start when this grid's launches are all done:
    // join the triangle streams into the trapezoid stream.
    for (int k = 0; k < 2; ++k) {
      LIFE_CUDA(cudaEventRecord(tri_join[k], c->cs[2 + k]));
      LIFE_CUDA(cudaStreamWaitEvent(c->cs[0], tri_join[k], 0));
    }
    LIFE_CUDA(cudaEventRecord(comp[i], c->cs[0]));
    main_done = comp[i];
    // Downloads: each chunk's interior as soon as its trapezoid is done, on
    // the D2H stream; the boundary strips on a second copy stream (cs[1]), so
    // a triangle still running -- its small launches wait for the trapezoid
    // passes to free SM slots -- never holds up the interiors behind it.
    cudaStream_t strips = c->cs[1];
    for (int ch = 0; ch < nc; ++ch) {
      const int64_t y0 = g.bounds[ch], rows = g.bounds[ch + 1] - y0;
      LIFE_CUDA(cudaStreamWaitEvent(c->d2h, trap_done[ch], 0));
      LIFE_TRY(copy_rows(g, outputs[i], buf[P & 1], y0 + shrink, rows - 2 * shrink, false, c->d2h));
      if (trace_chunks) LIFE_CUDA(cudaEventRecord(chunk_down[ch], c->d2h));
    }
    for (int bi = 1; bi <= nc; ++bi) {  // the order the triangles were launched in
      const int b = bi % nc;
      LIFE_CUDA(cudaStreamWaitEvent(strips, tri_done[b], 0));
      LIFE_TRY(copy_rows(g, outputs[i], buf[P & 1], g.bounds[b] - shrink, 2 * shrink, false,
                         strips));
      if (trace_chunks) LIFE_CUDA(cudaEventRecord(strip_down[b], strips));
    }
    cudaEvent_t strips_done;
    LIFE_TRY(mk(&strips_done));
    LIFE_CUDA(cudaEventRecord(strips_done, strips));
    LIFE_CUDA(cudaStreamWaitEvent(c->d2h, strips_done, 0));
    traced_nc = nc;
    for (int ch = 0; ch <= nc; ++ch) traced_bounds[ch] = g.bounds[ch];
    LIFE_CUDA(cudaEventRecord(down[i], c->d2h));
  }
  LIFE_CUDA(cudaEventRecord(t1, c->d2h));
  LIFE_CUDA(cudaEventSynchronize(t1));
  LIFE_CUDA(cudaStreamSynchronize(c->stream));
  if (trap)
    for (auto& st : c->cs) LIFE_CUDA(cudaStreamSynchronize(st));
  float ms = 0;
  LIFE_CUDA(cudaEventElapsedTime(&ms, t0, t1));
  if (elapsed_ms) *elapsed_ms = ms;
  if (trace_chunks && traced_nc > 0 && rc == LIFE_OK) {
    std::fprintf(stderr, "life_run_batch trace (n = %d, total %.1f ms): chunk rows  up  trap  down | boundary tri  strip-down\n", n, ms);
    for (int ch = 0; ch < traced_nc; ++ch) {
      float a = 0, b = 0, d = 0, e = 0, f = 0;
      cudaEventElapsedTime(&a, t0, chunk_up[ch]);
      cudaEventElapsedTime(&b, t0, trap_done[ch]);
      cudaEventElapsedTime(&d, t0, chunk_down[ch]);
      cudaEventElapsedTime(&e, t0, tri_done[ch]);
      cudaEventElapsedTime(&f, t0, strip_down[ch]);
      std::fprintf(stderr, "  %2d %7lld  %7.1f %7.1f %7.1f | %7.1f %7.1f\n", ch,
                   static_cast<long long>(traced_bounds[ch + 1] - traced_bounds[ch]), a, b, d, e, f);
    }
  }
  return rc;
}

}  // extern "C"

// ---- small launchers shared with life_multi.cu ------------------------------
namespace lifegpu {
namespace detail {

int launch_mask_tail(uint32_t* words, int64_t pitch, int64_t width, int64_t rows,
                     cudaStream_t s) {
  const int32_t nw = static_cast<int32_t>(nw32(width));
  const int64_t n = rows * (pitch - nw + 1);
  if (n <= 0) return LIFE_OK;
  packed_mask_tail_kernel<<<grid_stride_blocks(n, 256), 256, 0, s>>>(words, pitch, nw,
                                                                      tail_mask(width), rows);
  LIFE_CHECK_LAUNCH("packed_mask_tail_kernel");
  return LIFE_OK;
}

int launch_place_packed(uint32_t* words, int64_t pitch, const uint8_t* dev_pattern, int64_t pw,
                        int64_t ph, int64_t x0, int64_t y0, cudaStream_t s) {
  if (pw * ph == 0) return LIFE_OK;
  const int64_t n = (((x0 + pw - 1) >> 5) - (x0 >> 5) + 1) * ph;
  place_packed_kernel<<<grid_stride_blocks(n, 256), 256, 0, s>>>(words, pitch, dev_pattern, pw,
                                                                  ph, x0, y0);
  LIFE_CHECK_LAUNCH("place_packed_kernel");
  return LIFE_OK;
}

int launch_window_packed(const uint32_t* words, int64_t pitch, int64_t width, int64_t height,
                         int64_t x0, int64_t y0, int64_t w, int64_t h, uint8_t* dev_out,
                         cudaStream_t s) {
  const int64_t n = w * h;
  if (n == 0) return LIFE_OK;
  packed_window_kernel<<<grid_stride_blocks(n, 256), 256, 0, s>>>(words, pitch, width, height,
                                                                   x0, y0, w, h, dev_out);
  LIFE_CHECK_LAUNCH("packed_window_kernel");
  return LIFE_OK;
}

}  // namespace detail
}  // namespace lifegpu
