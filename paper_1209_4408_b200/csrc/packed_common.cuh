// packed_common.cuh -- pieces shared by the packed-engine kernels of
// kernels.cuh (plain layout) and kernels_pair.cuh (interleaved-pair layout):
// the bit-sliced rule network's row-combining half, the pass arguments and the
// cp.async / addressing helpers.  Templates and inline functions only, so
// several translation units may include it.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

// Pipeline fill of the temporal-blocked kernels as compile-time phases (one
// straight-line trip body per number of active stage groups) instead of one
// fill body with a warp-uniform branch per group: 0 = off, 1 = the short-tile
// (UNI) variant of the fast kernel and the all-paths kernel, 2 = the long-tile
// fast kernel too.  Timeline of a config-2 tile (tools/r5_timeline.py): fill
// 12.6 -> 6.7 us of a 114 us tile.
#ifndef LIFE_FILL_PHASES
#define LIFE_FILL_PHASES 1
#endif
// The interleaved kernels take the phased fill in every variant: their long
// tiles gain too (config 5 53.95 -> 54.26 T/s, 131072^2 52.0 -> 52.3, one of
// config 5's 8 bands 51.15 -> 51.46; tools/r5_il2.sh, three runs each).
#ifndef LIFE_FILL_PHASES_IL
#define LIFE_FILL_PHASES_IL 2
#endif
// Byte engine (byte_tb2_kernel): two coarse compile-time fill phases; 0 = off.
#ifndef LIFE_BYTE_FILL_PHASES
#define LIFE_BYTE_FILL_PHASES 0
#endif
// Drain of short tiles as specialised last trips (kernels_pair.cuh): 0 = off.
#ifndef LIFE_DRAIN_PHASES
#define LIFE_DRAIN_PHASES 0
#endif
// Tiles up to this many rows are "short": they run the single-loop-body (UNI)
// kernel variants.
constexpr long long kShortTileRows = 1024;

namespace lifegpu {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) {
  return (a & b) | (a & c) | (b & c);
}

struct HSum {
  uint32_t h0, h1;
};


template <uint32_t LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return d;
}

__device__ __forceinline__ uint32_t rule(HSum a, HSum b, HSum c, uint32_t self) {
  const uint32_t t0 = a.h0 ^ b.h0 ^ c.h0;
  const uint32_t k0 = maj3(a.h0, b.h0, c.h0);
  const uint32_t p = a.h1 ^ b.h1 ^ c.h1;
  const uint32_t q = maj3(a.h1, b.h1, c.h1);
  // lop3 immediates: bit (x<<2 | y<<1 | z) of the LUT is f(x, y, z).
  const uint32_t g1 = lop3<0x53>(t0, self, q);  // (~t0 & ~self) | (t0 & ~q)
  const uint32_t g2 = lop3<0x43>(p, k0, q);     // (~p & ~k0) | (p & k0 & ~q)
  return lop3<0x42>(t0, g1, g2);                // t0 ? (g1 & ~g2) : (~g1 & g2)
}

// Physical row index (base + r) mod m for possibly negative r.
__device__ __forceinline__ int64_t wrap_row(int64_t base, int64_t r, int64_t m) {
  int64_t p = (base + r) % m;
  return p < 0 ? p + m : p;
}


struct PackedStepArgs {
  const uint32_t* in;
  int64_t in_pitch;   // uint32 words
  int64_t in_row0;    // physical row of relative row 0
  int64_t in_rows;    // rows of `in` (row index wraps modulo this)
  uint32_t* out;
  int64_t out_pitch;
  int64_t out_row0;
  int64_t width;      // cells
  int64_t out_rows;
  int64_t seg_rows;   // output rows per tile (strip x segment)
  int32_t steps;      // loop trips every warp runs (lockstep)
  int32_t sync_every; // loop trips per block barrier
  int32_t nw;         // ceil(width / 32): words holding cells
  int32_t n_strips;   // strips this launch covers (all: ceil((nw + 1) / 31))
  int32_t strip0;     // first strip of this launch (strips wrap modulo strips_total)
  int32_t strips_total;  // ceil((nw + 1) / 31)
  uint32_t tail_mask; // valid bits of word nw-1
  void* trace;        // LIFE_TRACE builds: per-warp (smid, start, end)
  // Peer mode (multi-GPU row bands over NVLink): input relative row r < 0 is
  // row up_rows + r of `up` (the band above, a peer GPU's buffer), r >=
  // in_rows is row r - in_rows of `down` (the band below); in_row0 = 0 and
  // no modular wrap.  The halo never leaves the kernel: edge tiles cp.async
  // their ghost rows straight from the neighbours' HBM.
  const uint32_t* up;
  const uint32_t* down;
  int64_t up_rows;
  int64_t down_rows;
  int32_t peer;
};

// A warp covers 32 consecutive words; strips advance by 31 words, so
// neighbouring strips share one word: lane 31 of strip s and lane 0 of strip
// s+1.  After K <= 16 generations the shuffle edges have corrupted at most K
// bits at each end of the warp, so lane 31 still holds valid bits 0..15 and
// lane 0 valid bits 16..31: they store those halves (16-bit stores), and
// lanes 1..30 store whole words.  Ghost overhead is 1 word in 32.
constexpr int kStripStride = 31;

__device__ __forceinline__ const char* row_addr(const char* base, uint32_t idx, uint32_t stride) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(idx), "r"(stride), "l"(base));
  return reinterpret_cast<const char*>(r);
}


__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// cp.async.wait_group (MAX - u) for a loop index u the unroller has made a
// constant (the operand must be an immediate).
template <int MAX>
__device__ __forceinline__ void cp_async_wait_dyn(int u) {
  switch (u) {
    case 0: cp_async_wait<MAX>(); break;
    case 1: cp_async_wait<(MAX > 1 ? MAX - 1 : 0)>(); break;
    case 2: cp_async_wait<(MAX > 2 ? MAX - 2 : 0)>(); break;
    case 3: cp_async_wait<(MAX > 3 ? MAX - 3 : 0)>(); break;
    case 4: cp_async_wait<(MAX > 4 ? MAX - 4 : 0)>(); break;
    case 5: cp_async_wait<(MAX > 5 ? MAX - 5 : 0)>(); break;
    case 6: cp_async_wait<(MAX > 6 ? MAX - 6 : 0)>(); break;
    case 7: cp_async_wait<(MAX > 7 ? MAX - 7 : 0)>(); break;
    default: cp_async_wait<0>(); break;
  }
}


}  // namespace lifegpu
