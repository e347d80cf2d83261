// life_pair.cu -- launchers of the interleaved-layout packed kernels
// (kernels_pair.cuh): packed_il_kernel<K, N> passes (N = 2 pair, 4 quad), the peer-mode edge strips
// of multi-GPU row bands, and the in-place layout conversion.  Its own
// translation unit so the K instantiations compile beside life_gpu.cu.
#include <algorithm>
#include <cstdint>

#include "../../include/life_gpu.h"
#include "internal.h"
#include "kernels_pair.cuh"

using namespace lifegpu;
using namespace lifegpu::detail;

static_assert(kPairMaxDepth == kPairMaxDepthHost && kQuadMaxDepth == kQuadMaxDepthHost,
              "internal.h and kernels_pair.cuh disagree");

namespace {

constexpr int64_t kUniMaxRows = kShortTileRows;  // tiles up to this many rows: the single-loop-body variant

template <typename Kernel>
int launch_pdl_pair(Kernel kernel, unsigned blocks, unsigned threads, size_t smem, cudaStream_t s,
                    const PackedStepArgs& args) {
  static const bool pdl = knob("LIFE_PDL", 1) != 0;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  LIFE_CUDA(cudaLaunchKernelEx(&cfg, kernel, args));
  return LIFE_OK;
}

// One pass of K generations.  Tiles of seg_rows rows x one strip, one per
// warp, kWarps warps per block, one block per SM; the segment count minimises
// (block waves) x (rows per tile + pipeline fill), the cost model of
// launch_packed_kernel (life_gpu.cu).
template <int K, int N, bool PEER>
int launch_pair(PackedStepArgs a, cudaStream_t s) {
  using T = PairTraits<K, N>;
  // Peer-mode edge strips are 2K rows: always the single-loop-body variant.
  const auto kernel = packed_il_kernel<K, N, PEER, PEER>;
  const auto kernel_uni = packed_il_kernel<K, N, true, PEER>;
  static DeviceCache ready;  // per instantiation
  int dev = 0;
  cudaGetDevice(&dev);
  int bps = ready.get(dev);
  if (bps == 0) {
    LIFE_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   T::kWarps * T::kRingBytes));
    LIFE_CUDA(cudaFuncSetAttribute(kernel_uni, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   T::kWarps * T::kRingBytes));
    LIFE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kernel, 32 * T::kWarps,
                                                            T::kWarps * T::kRingBytes));
    if (bps < 1) return set_error(LIFE_ERR_CUDA, "packed_il_kernel<%d, %d> does not fit an SM", K, N);
    ready.put(dev, bps);
  }
  int wpb = static_cast<int>(std::min<int64_t>(knob("LIFE_PAIR_WPB", T::kWarps), T::kWarps));
  if (wpb < 1) wpb = T::kWarps;
  if (wpb != T::kWarps)
    LIFE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kernel, 32 * wpb,
                                                            wpb * T::kRingBytes));
  static const int64_t forced_bps = knob("LIFE_PAIR_BPS", 0);  // debug builds: blocks per SM the plan assumes
  if (forced_bps > 0) bps = static_cast<int>(forced_bps);
  if (a.out_rows >= (int64_t(1) << 31) || a.in_rows >= (int64_t(1) << 31) ||
      a.in_pitch * 4 >= (int64_t(1) << 32) || a.out_pitch * 4 >= (int64_t(1) << 32))
    return set_error(LIFE_ERR_CONFIG, "grid too large for one packed pass");
  constexpr int kLag = T::kLag;
  constexpr int PF = T::kPrefetch;
  const int64_t slots = static_cast<int64_t>(bps) * sm_count();  // blocks per wave
  int64_t best_segs = 1;
  double best_cost = 1e300;
  constexpr int kMinSegRows = 8;
  const int64_t max_segs =
      std::max<int64_t>(1, std::min<int64_t>(a.out_rows / kMinSegRows + 1, 4096));
  for (int64_t segs = 1; segs <= max_segs; ++segs) {
    const int64_t rows = ceil_div(a.out_rows, segs);
    const int64_t blocks =
        ceil_div(static_cast<int64_t>(a.n_strips) * ceil_div(a.out_rows, rows), wpb);
    const double cost = double(ceil_div(blocks, slots)) * double(rows + kLag + PF + 48);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best_segs = segs;
    }
  }
  static const int64_t forced_segs = knob("LIFE_SEGS", 0);  // debug builds
  if (forced_segs > 0) best_segs = std::min<int64_t>(forced_segs, a.out_rows);
  a.seg_rows = ceil_div(a.out_rows, best_segs);
  const int64_t tiles = static_cast<int64_t>(a.n_strips) * ceil_div(a.out_rows, a.seg_rows);
  a.steps = static_cast<int32_t>(ceil_div(a.seg_rows + kLag, PF));
  const int64_t blocks = ceil_div(tiles, wpb);
  if (blocks > 0x7fffffff) return set_error(LIFE_ERR_CONFIG, "grid too large");
  LIFE_TRY(launch_pdl_pair(a.seg_rows <= kUniMaxRows ? kernel_uni : kernel,
                           static_cast<unsigned>(blocks), 32 * wpb,
                           static_cast<size_t>(wpb) * T::kRingBytes, s, a));
  LIFE_CHECK_LAUNCH("packed_il_kernel");
  return LIFE_OK;
}

using PairLauncher = int (*)(PackedStepArgs, cudaStream_t);
template <bool PEER>
struct PairTable {
  static constexpr PairLauncher v[kPairMaxDepth + 1] = {
      nullptr,                 launch_pair<1, 2, PEER>,  launch_pair<2, 2, PEER>,
      launch_pair<3, 2, PEER>, launch_pair<4, 2, PEER>,  launch_pair<5, 2, PEER>,
      launch_pair<6, 2, PEER>, launch_pair<7, 2, PEER>,  launch_pair<8, 2, PEER>,
      launch_pair<9, 2, PEER>, launch_pair<10, 2, PEER>, launch_pair<11, 2, PEER>,
      launch_pair<12, 2, PEER>};
};
template <bool PEER>
struct QuadTable {
  static constexpr PairLauncher v[kQuadMaxDepth + 1] = {
      nullptr,                 launch_pair<1, 4, PEER>, launch_pair<2, 4, PEER>,
      launch_pair<3, 4, PEER>, launch_pair<4, 4, PEER>, launch_pair<5, 4, PEER>,
      launch_pair<6, 4, PEER>, launch_pair<7, 4, PEER>};
};

int fill_args(int il, PackedStepArgs* a, const uint32_t* in, int64_t in_pitch, int64_t in_row0,
              int64_t in_rows, uint32_t* out, int64_t out_pitch, int64_t out_row0, int64_t width,
              int64_t out_rows, int32_t generations) {
  if (il != 2 && il != 4)
    return set_error(LIFE_ERR_CONFIG, "interleave order must be 2 (pair) or 4 (quad), got %d", il);
  if (generations < 1 || generations > il_max_depth(il))
    return set_error(LIFE_ERR_CONFIG, "%s-layout temporal depth must be in [1, %d], got %d",
                     il == 4 ? "quad" : "pair", il_max_depth(il), generations);
  if (!il_eligible(il, width))
    return set_error(LIFE_ERR_CONFIG, "the %s layout needs W %% %d == 0, got %lld",
                     il == 4 ? "quad" : "pair", 32 * il, static_cast<long long>(width));
  if (in_rows < 1 || out_rows < 0 || in_pitch < width / 32 || out_pitch < width / 32 ||
      in_pitch % il != 0 || out_pitch % il != 0 || reinterpret_cast<uintptr_t>(in) % (4 * il) != 0 ||
      reinterpret_cast<uintptr_t>(out) % (4 * il) != 0)
    return set_error(LIFE_ERR_CONFIG, "bad interleaved step geometry");
  *a = PackedStepArgs{};
  a->in = in;
  a->in_pitch = in_pitch;
  a->in_row0 = in_row0;
  a->in_rows = in_rows;
  a->out = out;
  a->out_pitch = out_pitch;
  a->out_row0 = out_row0;
  a->width = width;
  a->out_rows = out_rows;
  a->nw = static_cast<int32_t>(width / (32 * il));  // groups
  a->n_strips = static_cast<int32_t>(ceil_div(a->nw + 1, kStripStride));
  a->strips_total = a->n_strips;
  a->tail_mask = 0xffffffffu;
  return LIFE_OK;
}

}  // namespace

namespace lifegpu {
namespace detail {

int packed_il_step(int il, const uint32_t* in, int64_t in_pitch, int64_t in_row0, int64_t in_rows,
                   uint32_t* out, int64_t out_pitch, int64_t out_row0, int64_t width,
                   int64_t out_rows, int32_t generations, cudaStream_t stream) {
  PackedStepArgs a;
  LIFE_TRY(fill_args(il, &a, in, in_pitch, in_row0, in_rows, out, out_pitch, out_row0, width,
                     out_rows, generations));
  if (out_rows == 0) return LIFE_OK;
  return il == 4 ? QuadTable<false>::v[generations](a, stream)
                 : PairTable<false>::v[generations](a, stream);
}

int packed_il_step_peer(int il, const uint32_t* in, const uint32_t* up, int64_t up_rows,
                        const uint32_t* down, int64_t down_rows, int64_t pitch,
                        int64_t band_rows, uint32_t* out, int64_t out_row0, int64_t out_rows,
                        int64_t width, int32_t generations, cudaStream_t stream) {
  if (!up || !down) return set_error(LIFE_ERR_CONFIG, "bad peer step geometry");
  if (band_rows < generations || up_rows < generations || down_rows < generations)
    return set_error(LIFE_ERR_TOO_MANY_PARTS, "bands must be at least %d rows", generations);
  if (out_row0 < 0 || out_rows < 0 || out_row0 + out_rows > band_rows)
    return set_error(LIFE_ERR_CONFIG, "output rows outside the band");
  PackedStepArgs a;
  LIFE_TRY(fill_args(il, &a, in, pitch, out_row0, band_rows, out, pitch, out_row0, width,
                     out_rows, generations));
  if (out_rows == 0) return LIFE_OK;
  a.up = up;
  a.down = down;
  a.up_rows = up_rows;
  a.down_rows = down_rows;
  a.peer = 1;
  return il == 4 ? QuadTable<true>::v[generations](a, stream)
                 : PairTable<true>::v[generations](a, stream);
}

int packed_zip(int il, uint32_t* words, int64_t pitch, int64_t width, int64_t row0, int64_t rows,
               bool unzip, cudaStream_t stream) {
  if (!il_eligible(il, width) || pitch < width / 32 || pitch % il != 0 ||
      reinterpret_cast<uintptr_t>(words) % (4 * il) != 0 || rows < 0 || row0 < 0)
    return set_error(LIFE_ERR_CONFIG, "bad layout conversion geometry");
  if (rows == 0) return LIFE_OK;
  const int64_t groups = width / (32 * il);
  const int64_t bx = ceil_div(groups, 256);
  const int64_t by = std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t(sm_count()) * 64) / bx));
  const dim3 grid(static_cast<unsigned>(bx), static_cast<unsigned>(std::min<int64_t>(by, 65535)));
  if (il == 4) {
    if (unzip)
      packed_zip_kernel<true, 4><<<grid, 256, 0, stream>>>(words, pitch, groups, row0, rows);
    else
      packed_zip_kernel<false, 4><<<grid, 256, 0, stream>>>(words, pitch, groups, row0, rows);
  } else if (unzip) {
    packed_zip_kernel<true, 2><<<grid, 256, 0, stream>>>(words, pitch, groups, row0, rows);
  } else {
    packed_zip_kernel<false, 2><<<grid, 256, 0, stream>>>(words, pitch, groups, row0, rows);
  }
  LIFE_CHECK_LAUNCH("packed_zip_kernel");
  return LIFE_OK;
}

}  // namespace detail
}  // namespace lifegpu
