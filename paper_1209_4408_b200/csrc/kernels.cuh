// kernels.cuh -- sm_100a device code of the generation-step engine.
//
// Layouts in HBM:
//   packed: rows of `pitch` uint32 words (pitch a multiple of 32 words, 128 B);
//           bit j of word k = column 32k+j (this is the little-endian view of
//           the uint64 exchange format of include/life_gpu.h); words
//           k >= ceil(W/32) and bits at columns >= W are kept zero.
//   byte:   rows of `pitch` bytes (a multiple of 16), one 0/1 byte per cell,
//           bytes at columns >= W kept zero.
//
// Rule: B3/S23 (next_state, grid.cpp:22-28).  With S the 9-cell sum
// (cell + 8 neighbours), next = (S == 3) | (S == 4 & self), which equals
// compute_region's `(n==3)|((n==2)&mid)` (engine.cpp:30-32) with n = S - self.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "packed_common.cuh"

namespace lifegpu {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

// ---------------------------------------------------------------------------
// Bit-sliced rule network (packed engine).
//
// A row word x (32 cells) with its left/right neighbour words gives the
// horizontal 3-cell sums h = L + x + R as two bit planes (h0, h1):
//   L = x<<1 | xl>>31,  R = x>>1 | xr<<31   (2 SHF.W funnel shifts)
//   h0 = L^x^R,  h1 = maj(L,x,R)            (2 LOP3)
// Three rows' planes a (above), b (the cell's row), c (below) give
//   S = a + b + c = t0 + 2*(k0 + p + 2q) with
//   t0 = a0^b0^c0, k0 = maj(a0,b0,c0), p = a1^b1^c1, q = maj(a1,b1,c1)
//                                           (4 LOP3)
// and next = (S==3) | (S==4 & self) in three more LOP3 (found by an
// exhaustive search over 3-gate LUT3 circuits, tools/rule_search.c):
//   g1 = (~t0 & ~self) | (t0 & ~q)
//   g2 = (~p & ~k0) | (p & k0 & ~q)        [k0 + p + 2q in {0, 2}, q = 0 for 2]
//   next = t0 ? (g1 & ~g2) : (~g1 & g2)    = t0 ? (~q & ~g2) : (self & g2)
// t0 = 1: S == 3 <=> k0 + p + 2q == 1 <=> ~q & ~g2.  t0 = 0: S == 4 <=>
// k0 + p + 2q == 2, i.e. g2 except k0 = p = q = 0 -- but then S = 0, and
// S >= self because b = L + self + R, so self = 0 there: the don't-care
// makes the 4-valued case split fit one gate.  11 integer ops per 32
// cell-updates (2 SHF + 9 LOP3); verified against next_state over all 512
// 3x3 neighbourhoods in tests/test_rule_network.py.
// ---------------------------------------------------------------------------
__device__ __forceinline__ HSum hsum(uint32_t xl, uint32_t x, uint32_t xr) {
  const uint32_t L = __funnelshift_l(xl, x, 1);  // (x << 1) | (xl >> 31)
  const uint32_t R = __funnelshift_r(x, xr, 1);  // (x >> 1) | (xr << 31)
  return HSum{L ^ x ^ R, maj3(L, x, R)};
}

// (Building L and R on the FMA pipe -- IMAD / IMAD.HI by 2 and 2^31 -- to
// offload the ALU pipe was measured 2-19 % slower for 1-4 of every 4 stages.)

// 32 cells starting at column 32*wi of the infinitely repeated row (period
// W): the toroidal wrap of Grid::wrap (grid.hpp:48-54) applied to a word.
// Slow path for words that straddle the row end or lie outside [0, W).
__device__ __noinline__ uint32_t load_word_wrapped(const uint32_t* __restrict__ row,
                                                   int64_t wi, int64_t width, int32_t nw) {
  int64_t c = (32 * wi) % width;
  if (c < 0) c += width;
  uint32_t v = 0;
  int filled = 0;
  while (filled < 32) {
    const int64_t avail = width - c;
    const int n = avail < (32 - filled) ? static_cast<int>(avail) : 32 - filled;
    const int64_t w0 = c >> 5;
    const uint32_t lo = row[w0];
    const uint32_t hi = (w0 + 1 < nw) ? row[w0 + 1] : 0u;
    uint32_t bits = __funnelshift_r(lo, hi, static_cast<uint32_t>(c & 31));
    if (n < 32) bits &= (1u << n) - 1u;
    v |= bits << filled;
    filled += n;
    c += n;
    if (c >= width) c = 0;
  }
  return v;
}

constexpr int kPackedThreads = 128;

// kMaxThreads: the warps of one SM that fit the pipeline's registers
// (16K registers per SM sub-partition / (warps per sub-partition x 32 x
// regs)); one such block per SM.
template <int K>
struct PackedTraits {
#ifdef LIFE_PF_HI
  static constexpr int kPrefetch = K <= 3 ? 6 : LIFE_PF_HI;
#else
  static constexpr int kPrefetch = K <= 3 ? 6 : 4;
#endif
#ifdef LIFE_WARPS16
  static constexpr int kWarps[17] = {0, 28, 24, 24, 20, 16, 16, 16, 16, 12, 12, 12, 12, 12, LIFE_WARPS16, LIFE_WARPS16, LIFE_WARPS16};
#else
  static constexpr int kWarps[17] = {0, 28, 24, 24, 20, 16, 16, 16, 16, 12, 12, 12, 12, 12, 8, 8, 8};
#endif
  static constexpr int kMaxThreads = 32 * kWarps[K];
  static constexpr int kRingBytes = 2 * kPrefetch * 96 * 4;  // per warp
  // packed_tb_fast_kernel (W % 32 == 0 tori, no peer tiles): 6 rows per trip.
#ifndef LIFE_PF_FAST
#define LIFE_PF_FAST 6
#endif
  static constexpr int kPrefetchFast = K >= 8 ? LIFE_PF_FAST : 6;
  static constexpr int kRingBytesFast = 2 * kPrefetchFast * 96 * 4;
#ifdef LIFE_FAST_WARPS_HI
  static constexpr int kWarpsFast = K >= 14 ? LIFE_FAST_WARPS_HI : kWarps[K];
#else
  static constexpr int kWarpsFast = kWarps[K];
#endif
  static constexpr int kMaxThreadsFast = 32 * kWarpsFast;
  static constexpr int kLag = 3 * K - 1;  // output row j leaves the pipeline at step j + 3K - 1
};

#ifndef LIFE_GROUP
#define LIFE_GROUP 4
#endif

constexpr int kGroup = LIFE_GROUP;  // stages issued level by level together

// How a lane fetches its 32-cell word of a row.  The column is the same for
// every row, so the plan is computed once per strip:
//   mode 0: one aligned load of word `src` -- the word lies inside [0, W),
//           or W is a multiple of 32 and the torus wrap (Grid::wrap,
//           grid.hpp:48-54) is just an index wrap;
//   mode 1: W % 32 != 0 and the word straddles the seam or lies outside
//           [0, W): n1 cells from column c (two words, funnel-shifted) then
//           32-n1 cells from column 0;
//   mode 2: W < 32 (the row wraps several times inside one word): loop.
struct WordPlan {
  int mode;
  int32_t src;      // mode 0
  int32_t p0, p1;   // words holding columns c.. (mode 1)
  uint32_t sh;      // c & 31
  uint32_t m1, m2;  // masks of the two segments
  uint32_t s2;      // shift of the second segment (n1 & 31)
};

__device__ __forceinline__ WordPlan make_plan(int64_t wi, int64_t width, int32_t nw) {
  WordPlan p{};
  if (wi >= 0 && (wi + 1) * 32 <= width) {
    p.mode = 0;
    p.src = static_cast<int32_t>(wi);
    return p;
  }
  if (width < 32) {
    p.mode = 2;
    return p;
  }
  if ((width & 31) == 0) {
    p.mode = 0;
    int64_t w = wi % nw;
    p.src = static_cast<int32_t>(w < 0 ? w + nw : w);
    return p;
  }
  int64_t c = (32 * wi) % width;
  if (c < 0) c += width;
  const int64_t n1 = width - c < 32 ? width - c : 32;
  p.mode = 1;
  p.p0 = static_cast<int32_t>(c >> 5);
  p.p1 = p.p0 + 1 < nw ? p.p0 + 1 : p.p0;
  p.sh = static_cast<uint32_t>(c & 31);
  p.m1 = n1 == 32 ? 0xffffffffu : ((1u << n1) - 1u);
  p.m2 = n1 == 32 ? 0u : ~p.m1;  // the low 32-n1 bits of word 0, shifted up by n1
  p.s2 = static_cast<uint32_t>(n1 & 31);
  return p;
}

// Seam path (W % 32 != 0, W >= 64): every lane builds its word from two
// aligned words A = row[p0], B = row[p1] of the same row as
//   ((A >> sh) & m1) | ((B << s2) & ~m1).
// Only three words straddle the torus seam (Grid::wrap, grid.hpp:48-54),
// with r = W % 32 and d = 32 - r:
//   wi = nw-1 (r cells, then columns 0..d-1):   A = nw-1, B = 0, sh = 0, s2 = r
//   wi = nw   (columns d..d+31):                A = 0,    B = 1, sh = d, s2 = r
//   wi = -1   (columns W-32..W-1):              A = nw-2, B = nw-1, sh = r, s2 = d
// Aligned words use A = B = wi, sh = s2 = 0, m1 = ~0.  Words right of nw
// and left of -1 are never needed: after K <= 16 generations their garbage
// has reached at most 16 bits into the neighbouring ghost word.
__device__ __forceinline__ WordPlan make_seam_plan(int64_t wi, int64_t width, int32_t nw) {
  WordPlan p{};
  p.mode = 1;
  p.m1 = kFull;
  const uint32_t r = static_cast<uint32_t>(width & 31), d = 32u - r;
  if (wi >= 0 && (wi + 1) * 32 <= width) {
    p.p0 = p.p1 = static_cast<int32_t>(wi);
  } else if (r == 0) {  // (LIFE_FORCE_SEAM builds) W % 32 == 0: index wrap
    const int64_t w = wi % nw;
    p.p0 = p.p1 = static_cast<int32_t>(w < 0 ? w + nw : w);
  } else if (wi == nw - 1) {
    p.p0 = nw - 1;
    p.p1 = 0;
    p.s2 = r;
    p.m1 = (1u << r) - 1u;
  } else if (wi == nw) {
    p.p0 = 0;
    p.p1 = 1;
    p.sh = d;
    p.s2 = r;
    p.m1 = (1u << r) - 1u;
  } else if (wi == -1) {
    p.p0 = nw - 2;
    p.p1 = nw - 1;
    p.sh = r;
    p.s2 = d;
    p.m1 = (1u << d) - 1u;
  }  // else: p0 = p1 = 0, don't-care word
  return p;
}

// base + idx * stride as one IMAD.WIDE (FMA pipe) with the 64-bit base as
// addend, so no IADD3 pair lands on the ALU pipe that the rule network fills.
// cp.async (LDGSTS) of one 32-bit word into this lane's ring slot.
__device__ __forceinline__ void cp_async4(uint32_t* smem_dst, const uint32_t* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
// The two 16-bit halves of a lane's output word, each stored only if the
// output row j is inside the segment (j < n as unsigned: negative j fails)
// and the lane owns that half -- predicates, no branch.
__device__ __forceinline__ void st_halves_if(char* p, uint32_t v, uint32_t j, uint32_t n,
                                             bool lo, bool hi) {
  asm volatile(
      "{\n .reg .pred q, a, b;\n setp.lt.u32 q, %3, %4;\n"
      " setp.ne.and.u32 a, %5, 0, q;\n setp.ne.and.u32 b, %6, 0, q;\n"
      " @a st.global.u16 [%0], %1;\n @b st.global.u16 [%0+2], %2;\n}\n" ::"l"(p),
      "h"(static_cast<uint16_t>(v)), "h"(static_cast<uint16_t>(v >> 16)), "r"(j), "r"(n),
      "r"(static_cast<uint32_t>(lo)), "r"(static_cast<uint32_t>(hi))
      : "memory");
}

// A warp's work is one tile (strip, y, n): a fresh pipeline of n + kLag
// steps (tile indices are int64; rows and trips are int32 -- the host
// rejects passes with in_rows or out_rows >= 2^31).

// One pipeline segment of a warp: strip `strip`, output rows [y, y+n).
// Runs ceil((n + kLag) / PF) loop trips (a block barrier after every
// sync_every-th) and returns that count.  Three fetch paths, chosen per warp (warp-uniform):
//   kPathFast:  every lane's word is one aligned word of the row (W % 32 == 0
//               or the strip does not touch the seam): one cp.async per row;
//   kPathSeam:  W % 32 != 0 and some lane's word straddles the seam: every
//               lane fetches three words and funnel-combines them (lanes whose
//               word is aligned use a plan that reduces to their own word), so
//               the loop stays branch-free;
//   kPathGeneral: W < 32 (the row wraps several times inside one word) or a
//               peer-mode tile whose rows reach into a neighbour band.
constexpr int kPathFast = 0, kPathSeam = 1, kPathGeneral = 2;

// UNI: one loop body for every output trip (first / last trips included, the
// row test as a store predicate): short tiles no longer run the cold check-
// trip copies (16384^2 +1.4 %, 8192^2 +3.8 %; 65536^2 -0.5 %, so long tiles
// keep the steady/check split).
// TRIP: the PF rows of a loop trip are requested together at its start (one
// row-wrap test and one address per trip) instead of one per step.  The
// all-paths kernel uses it (config 4 38.7 -> 39.3 T/s); the fast-only kernel
// keeps the per-step requests (short tiles lose to the larger loop body:
// 16384^2 37.3 -> 36.7, 8192^2 24.9 -> 22.4; long tiles unchanged).
// LIFE_TIMELINE builds (tools/r5_timeline.py): lane 0 of every warp of the
// fast-only kernel stamps %clock64 at the phases of its tile.
#ifdef LIFE_TIMELINE
#define LIFE_TL(i)                                                   \
  do {                                                               \
    if (tl != nullptr && lane == 0) {                                \
      unsigned long long c_;                                         \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_)::"memory");   \
      tl[i] = c_;                                                    \
    }                                                                \
  } while (0)
#else
#define LIFE_TL(i) \
  do {             \
  } while (0)
#endif

template <int K, int PATH, int PF = PackedTraits<K>::kPrefetch, bool UNI = false,
          bool TRIP = false>
__device__ __forceinline__ int packed_segment(const PackedStepArgs& a, const int lane,
                                              const int strip, const int y, const int n,
                                              uint32_t* ring, unsigned long long* tl = nullptr) {
  (void)tl;
  constexpr int kLag = PackedTraits<K>::kLag;
  constexpr bool EDGE = PATH == kPathGeneral;
  const bool tiny = a.width < 32;  // warp-uniform (general path only)
  const int in_rows = static_cast<int>(a.in_rows);
  const int64_t wi = static_cast<int64_t>(strip) * kStripStride + lane - 1;
  WordPlan plan = make_plan(wi, a.width, a.nw);
  if (PATH == kPathSeam) plan = make_seam_plan(wi, a.width, a.nw);

  // Input rows y-K, y-K+1, ... stream through a ring of 2*PF slots; step i
  // lives in slot i mod 2PF and is fetched PF steps ahead.  Row addresses
  // are one IMAD.WIDE (FMA pipe) from a 32-bit row index and byte pitch.
  int lrow = static_cast<int>(wrap_row(a.in_row0, static_cast<int64_t>(y) - K, a.in_rows));
  const uint32_t in_pitch_b = static_cast<uint32_t>(a.in_pitch * 4);
  const char* const in_lane = reinterpret_cast<const char*>(
      a.in + (PATH == kPathSeam ? plan.p0 : plan.src));
  const char* const in_lane1 = reinterpret_cast<const char*>(a.in + plan.p1);
  if (EDGE && a.peer) lrow = static_cast<int>(a.in_row0) + y - K;  // band row, resolved across bands
  auto issue = [&](int slot) {
    uint32_t* s = ring + slot * 96;
    if (!EDGE) {
      cp_async4(s, reinterpret_cast<const uint32_t*>(
                       row_addr(in_lane, static_cast<uint32_t>(lrow), in_pitch_b)));
      if (PATH == kPathSeam)
        cp_async4(s + 32, reinterpret_cast<const uint32_t*>(
                              row_addr(in_lane1, static_cast<uint32_t>(lrow), in_pitch_b)));
      cp_async_commit();
      lrow = (lrow + 1 == in_rows) ? 0 : lrow + 1;
      return;
    }
    const uint32_t* row;
    bool peer_row = false;
    if (a.peer) {
      const int64_t r = lrow;
      if (r < 0) {
        row = a.up + (a.up_rows + r) * a.in_pitch;
        peer_row = true;
      } else if (r < in_rows) {
        row = a.in + r * a.in_pitch;
      } else {
        const int64_t d = r - in_rows;  // rows past the light cone are over-reads: clamp
        row = a.down + (d < a.down_rows ? d : a.down_rows - 1) * a.in_pitch;
        peer_row = true;
      }
    } else {
      row = a.in + static_cast<int64_t>(lrow) * a.in_pitch;
    }
    if (peer_row) {
      // A neighbour GPU's row over NVLink: plain loads (peer UVA addresses)
      // staged into the ring; only the 2K ghost rows of edge tiles take this.
      if (tiny) {
        s[0] = load_word_wrapped(row, wi, a.width, a.nw);
      } else if (plan.mode == 0) {
        s[0] = row[plan.src];
      } else {
        s[0] = row[plan.p0];
        s[32] = row[plan.p1];
        s[64] = row[0];
      }
    } else if (tiny) {
      s[0] = load_word_wrapped(row, wi, a.width, a.nw);
    } else if (plan.mode == 0) {
      cp_async4(s, row + plan.src);
    } else {
      cp_async4(s, row + plan.p0);
      cp_async4(s + 32, row + plan.p1);
      cp_async4(s + 64, row);
    }
    cp_async_commit();
    if (a.peer) {
      ++lrow;
    } else {
      lrow = (lrow + 1 == in_rows) ? 0 : lrow + 1;
    }
  };
  // The PF rows of one loop trip, one commit group each, into ring slots
  // slot0 .. slot0 + PF - 1.  On the fast and seam paths the torus row wrap
  // is tested once per trip (warp-uniform): a trip that does not cross it
  // takes its rows at constant offsets from one address.
  auto issue_trip = [&](int slot0) {
    if (!EDGE && lrow + PF <= in_rows) {
      const char* p0 = row_addr(in_lane, static_cast<uint32_t>(lrow), in_pitch_b);
      const char* p1 = PATH == kPathSeam
                           ? row_addr(in_lane1, static_cast<uint32_t>(lrow), in_pitch_b)
                           : nullptr;
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        uint32_t* s = ring + (slot0 + u) * 96;
        cp_async4(s, reinterpret_cast<const uint32_t*>(p0 + static_cast<size_t>(u) * in_pitch_b));
        if (PATH == kPathSeam)
          cp_async4(s + 32,
                    reinterpret_cast<const uint32_t*>(p1 + static_cast<size_t>(u) * in_pitch_b));
        cp_async_commit();
      }
      lrow = (lrow + PF == in_rows) ? 0 : lrow + PF;
      return;
    }
#pragma unroll
    for (int u = 0; u < PF; ++u) issue(slot0 + u);
  };
  auto consume = [&](int slot) -> uint32_t {
    const uint32_t* s = ring + slot * 96;
    if (PATH == kPathFast || (EDGE && (tiny || plan.mode == 0))) return s[0];
    if (PATH == kPathSeam) {  // (A >> sh) on the m1 bits, (B << s2) on the others: 3 ALU ops
      const uint32_t lo = s[0] >> plan.sh, hi = s[32] << plan.s2;
      return (lo & plan.m1) | (hi & ~plan.m1);
    }
    return (__funnelshift_r(s[0], s[32], plan.sh) & plan.m1) | ((s[64] << plan.s2) & plan.m2);
  };

  // Stores, as two predicated 16-bit halves (no divergent branches): lanes
  // 1..30 write both, lane 0 only bits 16..31 and lane 31 only bits 0..15 of
  // the words they share with the neighbouring strips.
  const bool in_grid = wi >= 0 && wi < a.nw;
  const bool st_lo = in_grid && lane >= 1;
  const bool st_hi = in_grid && lane <= 30;
  const uint32_t st_mask = wi == a.nw - 1 ? a.tail_mask : kFull;
  char* const out_seg = reinterpret_cast<char*>(a.out + (a.out_row0 + y) * a.out_pitch + wi);
  const uint32_t out_pitch_b = static_cast<uint32_t>(a.out_pitch * 4);

  if constexpr (TRIP) {
    issue_trip(0);
  } else {
#pragma unroll
    for (int u = 0; u < PF; ++u) issue(u);
  }

  HSum sa[K], sb[K];
  uint32_t sself[K], xin[K];
#pragma unroll
  for (int g = 0; g < K; ++g) {
    sa[g] = HSum{0u, 0u};
    sb[g] = HSum{0u, 0u};
    sself[g] = 0u;
    xin[g] = 0u;
  }

  // One loop trip (PF steps).  FILL trips cover the pipeline fill: stage g
  // only sees valid input from step 3g on (stage g-1's first valid output),
  // so a group of stages whose lowest stage is g0 is skipped (warp-uniform
  // branch) while step < 3*g0 -- its window is overwritten by valid rows
  // before its first valid output at step 3g0+2.
  int half = 0;
  int sync_left = a.sync_every;  // barrier after trips t with (t + 1) % sync_every == 0
  // Trip kinds: kFill (no output yet; lower stage groups skipped), kCheck
  // (per-step test whether the output row is inside the segment), kSteady
  // (every step stores: no per-step test, no branch).
  constexpr int kFill = 0, kCheck = 1, kSteady = 2, kFillPhase = 16;
  auto trip = [&](const int t, auto kind_tag) {
    constexpr int KIND = decltype(kind_tag)::value;
    // KIND >= kFillPhase: a fill trip whose active stage groups are known at
    // compile time (groups below (KIND - kFillPhase) * kGroup), no branch.
    constexpr bool FILL = KIND == kFill || KIND >= kFillPhase;
    constexpr int kActive = KIND >= kFillPhase ? (KIND - kFillPhase) * kGroup : K;
    if constexpr (TRIP) issue_trip(half ^ PF);  // the next trip's rows
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      if constexpr (TRIP) {
        // row u of this trip: issued one trip ago; PF - 1 - u rows of that
        // trip and the PF just issued may still be in flight
        cp_async_wait_dyn<2 * PF - 1>(u);
      } else {
        issue((half ^ PF) + u);
        cp_async_wait<PF>();
      }
      xin[0] = consume(half + u);
      const int step = t * PF + u;
      // The K stages of a step are independent (skewed pipeline); they are
      // issued in groups of kGroup, level by level (all shuffles, then all
      // funnels, ...), so consecutive instructions do not depend on each
      // other and the ALU pipe sees several independent chains per warp.
      // Groups run top stage first: stage g reads xin[g] and then writes its
      // output into xin[g+1], which stage g+1 has already consumed this step,
      // so no second array of K outputs is live (saves ~K registers).
      uint32_t y_last = 0;
#pragma unroll
      for (int g0 = ((K - 1) / kGroup) * kGroup; g0 >= 0; g0 -= kGroup) {
        if constexpr (KIND >= kFillPhase) {
          if (g0 >= kActive) continue;  // compile time
        } else {
          if (FILL && step < 3 * g0) continue;
        }
        uint32_t xl[kGroup], xr[kGroup];
        HSum c[kGroup];
#pragma unroll
        for (int j = 0; j < kGroup; ++j) {
          if (g0 + j < K) {
            xl[j] = __shfl_up_sync(kFull, xin[g0 + j], 1);
            xr[j] = __shfl_down_sync(kFull, xin[g0 + j], 1);
          }
        }
#pragma unroll
        for (int j = 0; j < kGroup; ++j) {
          if (g0 + j < K) {
            c[j] = hsum(xl[j], xin[g0 + j], xr[j]);
          }
        }
#pragma unroll
        for (int j = kGroup - 1; j >= 0; --j) {
          if (g0 + j < K) {
            const int g = g0 + j;
            const uint32_t yg = rule(sa[g], sb[g], c[j], sself[g]);
            sa[g] = sb[g];
            sb[g] = c[j];
            sself[g] = xin[g];
            if (g + 1 < K) {
              xin[g + 1] = yg;
            } else {
              y_last = yg;
            }
          }
        }
      }
      // Output row j of the segment leaves the pipeline at step j + kLag.
      const int j = step - kLag;
      if (!FILL) {  // no output leaves the pipeline during the fill trips
        if (UNI && KIND == kCheck) {
          // Branch-free: the row test and the lane halves as store predicates.
          char* p = const_cast<char*>(row_addr(out_seg, static_cast<uint32_t>(j), out_pitch_b));
          const uint32_t v = PATH == kPathFast ? y_last : y_last & st_mask;
          st_halves_if(p, v, static_cast<uint32_t>(j), static_cast<uint32_t>(n), st_lo, st_hi);
        } else if (KIND == kSteady || static_cast<unsigned>(j) < static_cast<unsigned>(n)) {
          char* p = const_cast<char*>(row_addr(out_seg, static_cast<uint32_t>(j), out_pitch_b));
          // Only the seam strip holds word nw-1 (the tail): fast-path strips skip the mask.
          const uint32_t v = PATH == kPathFast ? y_last : y_last & st_mask;
          if (st_lo) *reinterpret_cast<uint16_t*>(p) = static_cast<uint16_t>(v);
          if (st_hi) *reinterpret_cast<uint16_t*>(p + 2) = static_cast<uint16_t>(v >> 16);
        }
      }
    }
    half ^= PF;
#ifndef LIFE_NO_LOCKSTEP
    if (a.sync_every > 0 && --sync_left == 0) {
      sync_left = a.sync_every;
      __syncthreads();
    }
#endif
  };

  const int trips = (n + kLag + PF - 1) / PF;
  // Trips with a skippable group: while step < 3*(top group's lowest stage).
  constexpr int kTopG0 = ((K - 1) / kGroup) * kGroup;
  constexpr int kFillTrips = (3 * kTopG0 + PF - 1) / PF;
  static_assert(PF * kFillTrips <= kLag, "fill trips must end before the first output");
  const int fill_trips = trips < kFillTrips ? trips : kFillTrips;
  // Steady trips: every step's output row j = t*PF + u - kLag is in [0, n).
  const int steady_begin = (kLag + PF - 1) / PF;
  const int steady_end = (n + kLag) / PF;
  int t = 0;
  LIFE_TL(2);  // prologue done, first PF rows requested
  // Fill as phases of 3 * kGroup steps: phase p runs groups 0..p-1 from a
  // straight-line body with no per-group branch (LIFE_FILL_PHASES 1: the
  // short-tile UNI variant only, 2: every variant, 0: the branchy fill body).
  // The all-paths kernel (TRIP) carries both fills and takes the phased one
  // on short tiles (config 4: +1 %, 16383^2: +3 %; long tiles and the split
  // launch's seam strips lose 1 % to the extra hot code, so they keep the
  // branchy body, as does the long-tile fast kernel).
  constexpr bool kPhased =
      (LIFE_FILL_PHASES == 2 || (LIFE_FILL_PHASES == 1 && (UNI || TRIP))) &&
      (3 * kGroup) % PF == 0 && kTopG0 > 0;
  const bool phased_now = true;  // (a run-time choice by tile length gave the gain back: both bodies hot)
  if constexpr (kPhased) {
    constexpr int kTripsPerPhase = 3 * kGroup / PF;
    constexpr int kPhases = kTopG0 / kGroup;
    static_assert(kPhases * kTripsPerPhase == kFillTrips, "phases cover the fill trips");
    auto phases = [&](auto self, auto p_tag) {
      constexpr int P = decltype(p_tag)::value;  // groups active in this phase
      if constexpr (P <= kPhases) {
#pragma unroll 1
        for (int r = 0; r < kTripsPerPhase; ++r, ++t) {
          trip(t, std::integral_constant<int, kFillPhase + P>{});
          if (t == 0) LIFE_TL(3);
        }
        self(self, std::integral_constant<int, P + 1>{});
      }
    };
    if (phased_now) phases(phases, std::integral_constant<int, 1>{});
  }
  (void)phased_now;
  if constexpr (!kPhased) {
    for (; t < fill_trips; ++t) {  // not phased: one body, a warp-uniform branch per group
      trip(t, std::integral_constant<int, kFill>{});
      if (t == 0) LIFE_TL(3);  // first trip: first rows have arrived
    }
  }
  LIFE_TL(4);  // fill trips done
  if constexpr (UNI) {
    (void)steady_begin;
    (void)steady_end;
#pragma unroll 1
    for (; t < trips; ++t) trip(t, std::integral_constant<int, kCheck>{});
  } else {
    for (; t < trips && (t < steady_begin || t >= steady_end); ++t)
      trip(t, std::integral_constant<int, kCheck>{});
    for (; t < steady_end; ++t) trip(t, std::integral_constant<int, kSteady>{});
    for (; t < trips; ++t) trip(t, std::integral_constant<int, kCheck>{});
  }
  cp_async_wait<0>();
  LIFE_TL(5);  // last row stored
  return trips;
}

// ---------------------------------------------------------------------------
// Temporal-blocked packed step: K generations per pass, no block-level
// data sharing.  Each warp streams input rows of a 32-word strip through a
// K-stage register pipeline: stage g turns the row stream of generation g
// into generation g+1, keeping the 3-row (h0,h1,self) window of its input in
// registers.  Horizontal neighbour words come from __shfl_up/down_sync.
// Input rows arrive through a per-warp shared-memory ring filled by
// cp.async PF rows ahead, so no load latency sits on the compute chain.
//
// The pipeline is SKEWED: stage g consumes what stage g-1 emitted on the
// previous step, so the K stages of one step are independent and their
// instruction chains (shuffle -> funnel -> 6 LOP3 levels) interleave.
// Stage g (0-based) emits at step i generation g+1 of input row i-1-2g;
// the last stage emits generation K of output row i-3K+1.
//
// Work: tiles of one strip x seg_rows rows, one per warp, strip fastest; a
// block is all the warps one SM holds, stepped in lockstep (a barrier every
// sync_every loop trips) because the warp arbiter otherwise starves some
// warps and the SM ends the pass with too few warps to fill the ALU pipe.  The host picks
// seg_rows so the number of block waves is nearly an integer.
//
// Every input row is read once per pass and every output row written once,
// so the HBM traffic per cell-update is (1 bit read + 1 bit write)/K plus the
// ghost overlap (32/31 on reads, (seg_rows+2K)/seg_rows vertically).
//
// Replaces compute_region (engine.cpp:17-48) x K generations with the
// per-generation barrier of WorkerTeam (engine.cpp:79-96) removed inside a
// pass: the dependency is carried by the pipeline order instead.
// ---------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(PackedTraits<K>::kMaxThreads)
packed_tb_kernel(const PackedStepArgs a) {
  const int lane = threadIdx.x & 31;
  // Tile = (strip, segment), strip fastest: the warps of a block are
  // neighbouring strips of the same rows, so the words they share (ghost
  // lanes, half-word stores) meet in L1/L2 at the same time.
  const int64_t tile = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int strip = (a.strip0 + static_cast<int>(tile % a.n_strips)) %
                    (a.strips_total > 0 ? a.strips_total : a.n_strips);
  const int64_t seg = tile / a.n_strips;
  const int64_t y0 = seg * a.seg_rows;
  const int64_t left = a.out_rows - y0;
  const int n = static_cast<int>(left <= 0 ? 0 : (left < a.seg_rows ? left : a.seg_rows));
#ifdef LIFE_NO_LOCKSTEP
  if (n == 0) return;  // warp-uniform
#endif
#ifdef LIFE_TRACE
  uint64_t t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
  extern __shared__ uint32_t ring_smem[];
  uint32_t* ring = ring_smem + (threadIdx.x >> 5) * (2 * PackedTraits<K>::kPrefetch * 96) + lane;
  // Programmatic dependent launch: the previous pass's grid must be complete
  // (and its writes visible) before the first read of our input rows; the
  // next pass may be scheduled as soon as we start (it waits the same way).
  // Both are no-ops for launches without the PDL attribute.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  int trips = 0;
  if (n > 0) {
    // General path for W < 32 and (peer mode) tiles whose rows reach past
    // the band into a neighbour GPU's band; seam path if a lane's word
    // straddles the torus seam (W % 32 != 0); otherwise the fast path.
    const int64_t wi = static_cast<int64_t>(strip) * kStripStride + lane - 1;
    constexpr int PF = PackedTraits<K>::kPrefetch;
    const int64_t yb = a.in_row0 + y0;  // band row of the tile's first output row
    const int64_t last_row = yb - K + (static_cast<int64_t>(a.steps) + 1) * PF;  // last row issued
    const bool near_band_edge = a.peer && (yb < K || last_row >= a.in_rows);
#if defined(LIFE_FORCE_SEAM)  // test/measurement builds: every warp on the seam path
    const int path = (a.width < 64 || near_band_edge) ? kPathGeneral : kPathSeam;
#else
    const int path = (a.width < 64 || near_band_edge) ? kPathGeneral
                     : __any_sync(kFull, make_plan(wi, a.width, a.nw).mode != 0) ? kPathSeam
                                                                                  : kPathFast;
#endif
    if (path == kPathFast) {
      trips = packed_segment<K, kPathFast, PackedTraits<K>::kPrefetch, false, true>(
          a, lane, strip, static_cast<int>(y0), n, ring);
    } else if (path == kPathSeam) {
      trips = packed_segment<K, kPathSeam, PackedTraits<K>::kPrefetch, false, true>(
          a, lane, strip, static_cast<int>(y0), n, ring);
    } else {
      trips = packed_segment<K, kPathGeneral, PackedTraits<K>::kPrefetch, false, true>(
          a, lane, strip, static_cast<int>(y0), n, ring);
    }
  }
#ifndef LIFE_NO_LOCKSTEP
  // Shorter (last) segments and spare warps pad to the block's trip count.
  if (a.sync_every > 0)
    for (; trips < a.steps; ++trips)
      if ((trips + 1) % a.sync_every == 0) __syncthreads();
#endif
#ifdef LIFE_TRACE
  if (lane == 0) {
    uint64_t t_end;
    uint32_t smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned long long* tr = reinterpret_cast<unsigned long long*>(a.trace) + 3 * tile;
    tr[0] = smid;
    tr[1] = t_start;
    tr[2] = t_end;
  }
#endif
}

// ---------------------------------------------------------------------------
// packed_tb_kernel for tori with W % 32 == 0 outside peer mode: every warp
// takes the fast fetch path (the torus column wrap is an index remap), so
// this instantiation has only that loop, runs 6 rows per loop trip instead
// of 4 and no block barrier (config 5: 45.70 -> 46.3 T/s; the deeper trip in
// the all-paths kernel cost config 4 3-11 % -- two large loop bodies hot per
// SM -- hence a separate kernel).
// ---------------------------------------------------------------------------
template <int K, bool UNI = false>
__global__ void __launch_bounds__(PackedTraits<K>::kMaxThreadsFast)
packed_tb_fast_kernel(const PackedStepArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t tile = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int strip = (a.strip0 + static_cast<int>(tile % a.n_strips)) %
                    (a.strips_total > 0 ? a.strips_total : a.n_strips);
  const int64_t seg = tile / a.n_strips;
  const int64_t y0 = seg * a.seg_rows;
  const int64_t left = a.out_rows - y0;
  const int n = static_cast<int>(left <= 0 ? 0 : (left < a.seg_rows ? left : a.seg_rows));
  if (n == 0) return;  // warp-uniform; no block barrier in this kernel
  extern __shared__ uint32_t ring_fast_smem[];
  uint32_t* ring =
      ring_fast_smem + (threadIdx.x >> 5) * (2 * PackedTraits<K>::kPrefetchFast * 96) + lane;
#ifdef LIFE_TIMELINE
  unsigned long long* tl =
      a.trace ? reinterpret_cast<unsigned long long*>(a.trace) + 8 * tile : nullptr;
  LIFE_TL(0);  // block resident
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: previous pass complete
  asm volatile("griddepcontrol.launch_dependents;");
#ifdef LIFE_TIMELINE
  LIFE_TL(1);  // previous pass complete
  if (tl != nullptr && lane == 0) {
    unsigned long long g_;
    uint32_t smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tl[6] = g_;
    tl[7] = smid;
  }
  packed_segment<K, kPathFast, PackedTraits<K>::kPrefetchFast, UNI>(
      a, lane, strip, static_cast<int>(y0), n, ring, tl);
#else
  packed_segment<K, kPathFast, PackedTraits<K>::kPrefetchFast, UNI>(a, lane, strip,
                                                                   static_cast<int>(y0), n, ring);
#endif
}

// ---------------------------------------------------------------------------
// Byte engine: one generation per pass over the byte layout.  Each lane owns
// 16 cells (one uint4) of a row and walks down a segment of rows, keeping
// the 3-row window of horizontal byte sums in registers, so each input row
// is read once (plus 2 halo rows per segment) and each output row written
// once: 2 B of HBM traffic per cell-update.  Neighbour bytes across lanes
// come from shuffles; across warps and across the torus seam from single
// byte loads.  SWAR: bytes hold 0..9, so uint32 adds never carry between
// cells.  Restates compute_region (engine.cpp:17-48) incl. the peeled wrap
// columns (:35-39, :44-46).
// ---------------------------------------------------------------------------
struct ByteStepArgs {
  const uint8_t* in;
  int64_t in_pitch;
  int64_t in_row0;
  int64_t in_rows;
  uint8_t* out;
  int64_t out_pitch;
  int64_t out_row0;
  int64_t width;
  int64_t out_rows;
  int64_t seg_rows;
  int32_t nv;        // ceil(width / 16) vectors per row
  int32_t n_strips;  // ceil(nv / 30)
  uint32_t one;      // 1 (byte_tb_kernel's adds: a * one + b issues on the FMA pipe)
};

constexpr int kByteThreads = 128;
#ifndef LIFE_BYTE_PF
#define LIFE_BYTE_PF 6
#endif
constexpr int kBytePF = LIFE_BYTE_PF;              // rows fetched ahead
constexpr int kByteSlotWords = 32 * 4 + 4;         // 16-B vector per lane + the 2 seam words
constexpr int kByteSmem = (kByteThreads / 32) * 2 * kBytePF * kByteSlotWords * 4;  // per block
constexpr int kByteStride = 30;                    // vectors stored per warp (lanes 1..30)

struct ByteRow {
  uint32_t h[4];   // L + x + R per byte
  uint32_t hn[4];  // L + R per byte (neighbours only)
  uint32_t x[4];
};

__device__ __forceinline__ ByteRow byte_row(const uint4 v, uint32_t left_byte,
                                            uint32_t right_byte, int seam_pos, uint32_t col0) {
  uint32_t x[4] = {v.x, v.y, v.z, v.w};
  // Right-neighbour vector with the torus seam: the byte right of column W-1
  // (position seam_pos of this vector) must be column 0.
  uint32_t r[4];
  r[0] = __funnelshift_r(x[0], x[1], 8);
  r[1] = __funnelshift_r(x[1], x[2], 8);
  r[2] = __funnelshift_r(x[2], x[3], 8);
  r[3] = __funnelshift_r(x[3], right_byte, 8);
  if (seam_pos >= 0) {
    const int wsel = seam_pos >> 2, sh = (seam_pos & 3) * 8;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i == wsel) r[i] = (r[i] & ~(0xffu << sh)) | (col0 << sh);
  }
  uint32_t l[4];
  l[0] = __funnelshift_l(left_byte << 24, x[0], 8);
  l[1] = __funnelshift_l(x[0], x[1], 8);
  l[2] = __funnelshift_l(x[1], x[2], 8);
  l[3] = __funnelshift_l(x[2], x[3], 8);
  ByteRow row;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    row.x[i] = x[i];
    row.hn[i] = l[i] + r[i];
    row.h[i] = row.hn[i] + x[i];
  }
  return row;
}

__device__ __forceinline__ void st_global_v4_if(void* p, const uint32_t (&o)[4], bool pred) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %5, 0;\n"
      " @q st.global.v4.u32 [%0], {%1, %2, %3, %4};\n}\n" ::"l"(p),
      "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(static_cast<uint32_t>(pred))
      : "memory");
}

__device__ __forceinline__ void st_global_v2_if(void* p, uint32_t a, uint32_t b, bool pred) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n"
      " @q st.global.v2.u32 [%0], {%1, %2};\n}\n" ::"l"(p),
      "r"(a), "r"(b), "r"(static_cast<uint32_t>(pred))
      : "memory");
}

__device__ __forceinline__ void cp_async16(uint32_t* smem_dst, const void* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}

// One warp, one strip x segment of the byte engine.  Lanes 0 and 31 hold
// the neighbouring strips' edge vectors (ghosts; their neighbour bytes come
// from the shuffles of the lanes inside), lanes 1..30 store.  When W % 16 ==
// 0 the torus seam is an index wrap and every warp takes the plain path;
// otherwise EDGE warps fetch, per row, the byte left of column 0 and column 0
// itself for the seam lanes (compute_region's peeled columns,
// engine.cpp:35-39, :44-46).
template <bool EDGE>
__device__ __forceinline__ void byte_pass(const ByteStepArgs& a, const int lane, const int64_t vi,
                                          const int64_t y0, const int rows, uint32_t* ring) {
  constexpr int PF = kBytePF;
  const int64_t nv = a.nv;
  int64_t src = vi % nv;
  if (src < 0) src += nv;
  const bool store = lane >= 1 && lane <= kByteStride && vi >= 0 && vi < nv;
  const bool need_left = EDGE && store && vi == 0;  // byte left of column 0 = column W-1
  const int seam_pos =
      (EDGE && store && vi == nv - 1) ? static_cast<int>(a.width - 1 - vi * 16) : -1;
  const int64_t left_word = ((a.width - 1) & ~3LL);
  const uint32_t left_shift = static_cast<uint32_t>(((a.width - 1) & 3) * 8);

  const int in_rows = static_cast<int>(a.in_rows);
  int lrow = static_cast<int>(wrap_row(a.in_row0, y0 - 1, a.in_rows));
  const uint32_t in_pitch_b = static_cast<uint32_t>(a.in_pitch);
  const uint8_t* const in_lane = a.in + src * 16;
  auto issue = [&](int slot) {
    uint32_t* s = ring + slot * kByteSlotWords;
    const uint64_t off = static_cast<uint64_t>(static_cast<uint32_t>(lrow)) * in_pitch_b;
    cp_async16(s + lane * 4, in_lane + off);
    if (EDGE) {
      // At most one lane of a warp needs each seam word.
      if (need_left) cp_async4(s + 128, reinterpret_cast<const uint32_t*>(a.in + off + left_word));
      if (seam_pos >= 0) cp_async4(s + 129, reinterpret_cast<const uint32_t*>(a.in + off));
    }
    cp_async_commit();
    lrow = (lrow + 1 == in_rows) ? 0 : lrow + 1;
  };
  auto consume = [&](int slot) -> ByteRow {
    const uint32_t* s = ring + slot * kByteSlotWords;
    const uint4 v = *reinterpret_cast<const uint4*>(s + lane * 4);
    uint32_t lb = __shfl_up_sync(kFull, v.w >> 24, 1);
    const uint32_t rb = __shfl_down_sync(kFull, v.x & 0xffu, 1);
    uint32_t col0 = 0;
    if (EDGE) {
      if (need_left) lb = (s[128] >> left_shift) & 0xffu;
      if (seam_pos >= 0) col0 = s[129] & 0xffu;
    }
    return byte_row(v, lb, rb, seam_pos, col0);
  };

  const uint32_t out_pitch_b = static_cast<uint32_t>(a.out_pitch);
  uint8_t* const out_lane = a.out + (a.out_row0 + y0) * a.out_pitch + vi * 16;
#pragma unroll
  for (int u = 0; u < PF; ++u) issue(u);
  ByteRow up{}, mid{};
  // Step t consumes input row y0-1+t; output row t-2 leaves at step t >= 2.
  // Steady trips (every step's output row inside the segment) store without
  // a per-step bounds branch, so each trip is one basic block.
  const int trips = (rows + 2 + PF - 1) / PF;
  int half = 0;
  auto trip = [&](const int tr, auto steady_tag) {
    constexpr bool STEADY = decltype(steady_tag)::value;
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      issue((half ^ PF) + u);
      cp_async_wait<PF>();
      const ByteRow dn = consume(half + u);
      const int j = tr * PF + u - 2;
      uint32_t o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t n = up.h[i] + dn.h[i] + mid.hn[i];  // 8-neighbour count per byte
        // (n | self) == 3  <=>  next alive (engine.cpp:32 on 0/1 bytes);
        // t = (n|self)^3 is 0..15 per byte; zero-test via the byte's bit 7.
        const uint32_t t = (n | mid.x[i]) ^ 0x03030303u;
        o[i] = (~(t + 0x7f7f7f7fu) & 0x80808080u) >> 7;
      }
      if (EDGE && seam_pos >= 0) {  // zero the padding bytes past column W-1
        const int keep = seam_pos + 1;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int lo = i * 4;
          if (keep <= lo) o[i] = 0;
          else if (keep < lo + 4) o[i] &= (1u << ((keep - lo) * 8)) - 1u;
        }
      }
      // Predicated store (no branch: a divergent branch here would make every
      // following shuffle re-check convergence and split the trip into blocks).
      const bool st = store && (STEADY || static_cast<unsigned>(j) < static_cast<unsigned>(rows));
      st_global_v4_if(out_lane + static_cast<uint64_t>(static_cast<uint32_t>(j)) * out_pitch_b,
                      o, st);
      up = mid;
      mid = dn;
    }
    half ^= PF;
  };
  const int steady_begin = (2 + PF - 1) / PF;  // first trip with j >= 0 at u = 0
  const int steady_end = (rows + 2) / PF;      // trips below this have j < rows throughout
  int tr = 0;
  for (; tr < trips && (tr < steady_begin || tr >= steady_end); ++tr) trip(tr, std::false_type{});
  for (; tr < steady_end; ++tr) trip(tr, std::true_type{});
  for (; tr < trips; ++tr) trip(tr, std::false_type{});
  cp_async_wait<0>();
}

// Byte engine: one generation per pass over the byte layout.  Each lane owns
// 16 cells (one uint4) of a row and walks down a segment of rows, keeping
// the 3-row window of horizontal byte sums in registers; rows arrive through
// a per-warp cp.async ring kBytePF rows ahead, so each input row is read once
// (plus 2 halo rows per segment) and each output row written once: 2 B of HBM
// traffic per cell-update.  SWAR: bytes hold 0..9, so uint32 adds never carry
// between cells.  Restates compute_region (engine.cpp:17-48).
__global__ void __launch_bounds__(kByteThreads) byte_step_kernel(const ByteStepArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * kByteThreads + threadIdx.x) >> 5;
  const int strip = static_cast<int>(gwarp % a.n_strips);
  const int64_t seg = gwarp / a.n_strips;
  const int64_t y0 = seg * a.seg_rows;
  if (y0 >= a.out_rows) return;  // warp-uniform
  const int rows = static_cast<int>(min(a.seg_rows, a.out_rows - y0));
  const int64_t vi = static_cast<int64_t>(strip) * kByteStride + lane - 1;
  extern __shared__ uint32_t byte_ring[];
  uint32_t* ring = byte_ring + (threadIdx.x >> 5) * (2 * kBytePF * kByteSlotWords);
  // EDGE: W % 16 != 0 and this warp stores column 0 or column W-1.
  const bool edge = (a.width & 15) != 0 &&
                    __any_sync(kFull, lane >= 1 && lane <= kByteStride &&
                                          (vi == 0 || vi == a.nv - 1));
  if (edge) {
    byte_pass<true>(a, lane, vi, y0, rows, ring);
  } else {
    byte_pass<false>(a, lane, vi, y0, rows, ring);
  }
}

// ---------------------------------------------------------------------------
// Temporal-blocked byte engine: K generations per pass over the byte layout
// (W % 16 == 0, so the torus column wrap is an index wrap of 16-byte
// vectors).  The register pipeline of packed_tb_kernel with SWAR bytes: each
// lane owns 16 cells (one uint4) of a row; stage g keeps the (h, hn, x) byte
// sums of its 3-row window and turns the generation-g row stream into
// generation g+1; stage g eats what stage g-1 emitted on the previous step
// (skewed), so the K stages of a step are independent instruction chains.
// Lanes 0 and 31 are ghosts: K <= 8 generations corrupt at most K bytes at
// the outer end of their vectors, so lane 0 still holds 8 valid high bytes
// and lane 31 8 valid low bytes; strips advance by 31 vectors and the shared
// vector is stored as two 8-byte halves.  HBM traffic per cell-update: 2/K B.  Restates
// compute_region (engine.cpp:17-48) x K generations.
// ---------------------------------------------------------------------------
constexpr int kByteTbMaxDepth = 8;
// Narrowest W % 16 != 0 torus the temporal-blocked byte pass takes (three
// vectors per row, byte_seam_plan); narrower ones run one generation per pass.
constexpr int kByteTbMinSeamWidth = 33;
constexpr int kByteTbStride = 31;  // vectors per strip: 30 whole + 2 shared halves
#ifndef LIFE_BYTE_TB_PF
#define LIFE_BYTE_TB_PF 4
#endif
constexpr int kByteTbPF = LIFE_BYTE_TB_PF;
constexpr int kByteTbSmem = (kByteThreads / 32) * 2 * kByteTbPF * 32 * 16;  // per block

// a + b as a * one + b: `one` is a runtime 1 (kernel argument) the compiler
// cannot fold, so the add issues as IMAD on the FMA pipe and leaves the ALU
// pipe -- the bound of byte_tb_kernel -- to the shifts and logic ops.
__device__ __forceinline__ uint32_t add_fma(uint32_t a, uint32_t b, uint32_t one) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(one), "r"(b));
  return d;
}

// Horizontal byte sums of one 16-cell vector (byte_row with the adds on the
// FMA pipe): per word 2 funnel shifts (ALU) + 2 IMAD.  `lw` / `rw` are the
// whole neighbouring words (left lane's x[3], right lane's x[0]): the funnel
// shifts take the byte they need.
__device__ __forceinline__ void byte_row_fma(const uint32_t (&x)[4], uint32_t lw, uint32_t rw,
                                             uint32_t one, uint32_t (&h)[4], uint32_t (&hn)[4]) {
  uint32_t r[4], l[4];
  r[0] = __funnelshift_r(x[0], x[1], 8);
  r[1] = __funnelshift_r(x[1], x[2], 8);
  r[2] = __funnelshift_r(x[2], x[3], 8);
  r[3] = __funnelshift_r(x[3], rw, 8);
  l[0] = __funnelshift_l(lw, x[0], 8);
  l[1] = __funnelshift_l(x[0], x[1], 8);
  l[2] = __funnelshift_l(x[1], x[2], 8);
  l[3] = __funnelshift_l(x[2], x[3], 8);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    hn[i] = add_fma(l[i], r[i], one);
    h[i] = add_fma(hn[i], x[i], one);
  }
}

// (n | self) == 3 per byte (engine.cpp:32 on 0/1 bytes, n = 8-neighbour count):
// t = (n | self) ^ 3 is 0..15 per byte; alive iff t == 0, via bit 7 of t + 0x7f.
// 3 ALU ops (LOP3, SHF, LOP3) + 3 IMAD per 4 cells.
__device__ __forceinline__ uint32_t byte_rule(uint32_t up_h, uint32_t dn_h, uint32_t mid_hn,
                                              uint32_t mid_x, uint32_t one) {
  const uint32_t t = (add_fma(add_fma(up_h, dn_h, one), mid_hn, one) | mid_x) ^ 0x03030303u;
  return (~add_fma(t, 0x7f7f7f7fu, one) & 0x80808080u) >> 7;  // one LOP3 (~y & m) + SHF
}

template <int K>
__global__ void __launch_bounds__(kByteThreads) byte_tb_kernel(const ByteStepArgs a) {
  constexpr int PF = kByteTbPF;
  constexpr int kLag = 3 * K - 1;  // output row j leaves the pipeline at step j + kLag
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * kByteThreads + threadIdx.x) >> 5;
  const int strip = static_cast<int>(gwarp % a.n_strips);
  const int64_t seg = gwarp / a.n_strips;
  const int64_t y0 = seg * a.seg_rows;
  if (y0 >= a.out_rows) return;  // warp-uniform
  const int n = static_cast<int>(min(a.seg_rows, a.out_rows - y0));
  const int64_t vi = static_cast<int64_t>(strip) * kByteTbStride + lane - 1;
  int64_t src = vi % a.nv;
  if (src < 0) src += a.nv;
  // Lanes 1..30 store whole vectors; lane 31 the low 8 bytes and lane 0 the
  // high 8 bytes of the vectors shared with the neighbouring strips (K <= 8
  // generations corrupt at most 8 bytes at each end of the warp).
  const bool in_grid = vi >= 0 && vi < a.nv;
  const bool store_mid = in_grid && lane >= 1 && lane <= 30;
  const bool store_lo = in_grid && lane == 31;
  const bool store_hi = in_grid && lane == 0;
  const uint32_t one = a.one;
  extern __shared__ uint4 byte_tb_ring[];
  uint4* ring = byte_tb_ring + (threadIdx.x >> 5) * (2 * PF * 32) + lane;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: previous pass complete
  asm volatile("griddepcontrol.launch_dependents;");

  const int in_rows = static_cast<int>(a.in_rows);
  int lrow = static_cast<int>(wrap_row(a.in_row0, y0 - K, a.in_rows));
  const uint32_t in_pitch_b = static_cast<uint32_t>(a.in_pitch);
  const char* const in_lane = reinterpret_cast<const char*>(a.in + src * 16);
  auto issue = [&](int slot) {
    cp_async16(reinterpret_cast<uint32_t*>(ring + slot * 32),
               row_addr(in_lane, static_cast<uint32_t>(lrow), in_pitch_b));
    cp_async_commit();
    lrow = (lrow + 1 == in_rows) ? 0 : lrow + 1;
  };
  const uint32_t out_pitch_b = static_cast<uint32_t>(a.out_pitch);
  char* const out_lane = reinterpret_cast<char*>(a.out + (a.out_row0 + y0) * a.out_pitch + vi * 16);

#pragma unroll
  for (int u = 0; u < PF; ++u) issue(u);
  // Stage state: up.h, mid.h, mid.hn, mid.x (4 words each); xin[g] = stage g's input row.
  uint32_t uh[K][4], mh[K][4], mhn[K][4], mx[K][4], xin[K][4];
#pragma unroll
  for (int g = 0; g < K; ++g)
#pragma unroll
    for (int i = 0; i < 4; ++i) uh[g][i] = mh[g][i] = mhn[g][i] = mx[g][i] = xin[g][i] = 0u;

  const int trips = (n + kLag + PF - 1) / PF;
  int half = 0;
  auto trip = [&](const int t, auto steady_tag) {
    constexpr bool STEADY = decltype(steady_tag)::value;
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      issue((half ^ PF) + u);
      cp_async_wait<PF>();
      {
        const uint4 v = ring[(half + u) * 32];
        xin[0][0] = v.x;
        xin[0][1] = v.y;
        xin[0][2] = v.z;
        xin[0][3] = v.w;
      }
      uint32_t y_last[4];
      // Top stage first: stage g reads xin[g] and writes xin[g+1], which
      // stage g+1 has already consumed this step.
#pragma unroll
      for (int g = K - 1; g >= 0; --g) {
        const uint32_t lw = __shfl_up_sync(kFull, xin[g][3], 1);
        const uint32_t rw = __shfl_down_sync(kFull, xin[g][0], 1);
        uint32_t h[4], hn[4];
        byte_row_fma(xin[g], lw, rw, one, h, hn);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t o = byte_rule(uh[g][i], h[i], mhn[g][i], mx[g][i], one);
          uh[g][i] = mh[g][i];
          mh[g][i] = h[i];
          mhn[g][i] = hn[i];
          mx[g][i] = xin[g][i];
          if (g + 1 < K) {
            xin[g + 1][i] = o;
          } else {
            y_last[i] = o;
          }
        }
      }
      const int j = t * PF + u - kLag;
      const bool in_seg = STEADY || static_cast<unsigned>(j) < static_cast<unsigned>(n);
      char* const p = const_cast<char*>(row_addr(out_lane, static_cast<uint32_t>(j), out_pitch_b));
      st_global_v4_if(p, y_last, in_seg && store_mid);
      st_global_v2_if(p, y_last[0], y_last[1], in_seg && store_lo);
      st_global_v2_if(p + 8, y_last[2], y_last[3], in_seg && store_hi);
    }
    half ^= PF;
  };
  const int steady_begin = (kLag + PF - 1) / PF;
  const int steady_end = (n + kLag) / PF;
  int t = 0;
  for (; t < trips && (t < steady_begin || t >= steady_end); ++t) trip(t, std::false_type{});
  for (; t < steady_end; ++t) trip(t, std::true_type{});
  for (; t < trips; ++t) trip(t, std::false_type{});
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// byte_tb_kernel with TWO row streams per register word (nibble SWAR).  A
// warp's tile of n rows is split into two halves that run through the same
// K-stage pipeline side by side: stream A (rows [y, y+nA)) in the low nibble
// of every byte, stream B (rows [y+nA, y+n)) in the high nibble.  Counts stay
// <= 9 < 16, so no add carries between nibbles, and the horizontal neighbour
// is still one byte away, so the funnel shifts serve both streams at once:
// one instruction sequence updates 8 cells per 32-bit word instead of 4.
// HBM layout and traffic are unchanged (one byte per cell; stage 0 packs A |
// B << 4 from the two rows it loads, the last stage unpacks and stores both).
// Rule per nibble: n' = n & 7 (n = 8 -> 0: dead either way, and it keeps t <=
// 7 so t + 7 cannot carry), t = (n' | self) ^ 3, alive iff t == 0, i.e. bit 3
// of t + 7 clear.  Per word and stage: ALU 2 SHF (neighbours) + 2 LOP3 + 1
// LOP3 + 1 SHF, FMA 5 IMAD (hn, h, two vertical adds, t + 7) -- 11
// instructions per 8 cell-updates vs 10 per 4 in byte_tb_kernel.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t nib_rule(uint32_t up_h, uint32_t dn_h, uint32_t mid_hn,
                                             uint32_t mid_x, uint32_t one) {
  const uint32_t n = add_fma(add_fma(up_h, dn_h, one), mid_hn, one) & 0x77777777u;
  const uint32_t t = (n | mid_x) ^ 0x33333333u;
  return (~add_fma(t, 0x77777777u, one) & 0x88888888u) >> 3;
}

constexpr int kByteTb2PF = 4;
constexpr int kByteTb2Smem = (kByteThreads / 32) * 2 * kByteTb2PF * 64 * 16;  // per block

// W % 16 != 0 byte tori (r = W % 16, nv = ceil(W/16) >= 3 vectors per row,
// the bytes of vector nv-1 past column W zero): the lanes next to the column
// seam need vectors of the infinitely repeated row that are not aligned
// vectors of the stored row.  byte_seam_prep_kernel writes them, per row,
// into three padding vectors after the row (life_byte_pitch reserves them)
// before every pass, so the pass kernel only maps those lanes' loads there:
//   vector nv   : columns 16nv .. 16nv+15 of the next period  = bytes 16-r.. of [v0, v1]
//   vector nv+1 : columns W-16 .. W-1 (lane vi = -1)           = bytes r.. of [v(nv-2), v(nv-1)]
//   vector nv+2 : vi = nv-1 with the row start after column W  = v(nv-1) | bytes 16-r.. of [0, v0]
// Lanes further out only ever feed the ghost bytes K <= 8 generations
// corrupt, so they may load anything.
__device__ __forceinline__ int64_t byte_seam_src(int64_t vi, int64_t nv) {
  if (vi >= 0 && vi <= nv - 2) return vi;
  if (vi == nv - 1) return nv + 2;
  if (vi == -1) return nv + 1;
  return nv;
}
// Bytes o .. o+15 (o in 0..16) of the 32-byte concatenation [p, q].
__device__ __forceinline__ uint4 byte_extract(const uint4 p, const uint4 q, int o) {
  const uint32_t c[9] = {p.x, p.y, p.z, p.w, q.x, q.y, q.z, q.w, 0u};
  const int wo = o >> 2;
  const uint32_t sh = static_cast<uint32_t>(o & 3) * 8u;
  uint32_t w[5];
#pragma unroll
  for (int i = 0; i < 5; ++i)
    w[i] = wo == 0 ? c[i] : wo == 1 ? c[i + 1] : wo == 2 ? c[i + 2] : wo == 3 ? c[i + 3] : c[i + 4];
  return make_uint4(__funnelshift_r(w[0], w[1], sh), __funnelshift_r(w[1], w[2], sh),
                    __funnelshift_r(w[2], w[3], sh), __funnelshift_r(w[3], w[4], sh));
}
__device__ __forceinline__ void byte_tail_mask(int r, uint32_t (&m)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int valid = r - 4 * i;  // bytes of word i inside the row
    m[i] = valid >= 4 ? ~0u : (valid <= 0 ? 0u : (1u << (8 * valid)) - 1u);
  }
}

struct SeamPrepArgs {
  uint8_t* rows;
  int64_t pitch, n_rows, width;
};
__global__ void __launch_bounds__(128) byte_seam_prep_kernel(const SeamPrepArgs a) {
  uint8_t* const rows = a.rows;
  const int64_t pitch = a.pitch, n_rows = a.n_rows, width = a.width;
  const int64_t nv = (width + 15) / 16;
  const int r = static_cast<int>(width & 15);
  uint32_t m[4];
  byte_tail_mask(r, m);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: previous pass complete
  for (int64_t y = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; y < n_rows;
       y += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint4* row = reinterpret_cast<uint4*>(rows + y * pitch);
    const uint4 v0 = row[0], v1 = row[1], vm2 = row[nv - 2];
    uint4 vm1 = row[nv - 1];
    vm1 = make_uint4(vm1.x & m[0], vm1.y & m[1], vm1.z & m[2], vm1.w & m[3]);
    const uint4 zero = make_uint4(0u, 0u, 0u, 0u);
    const uint4 s = byte_extract(zero, v0, 16 - r);
    row[nv] = byte_extract(v0, v1, 16 - r);
    row[nv + 1] = byte_extract(vm2, vm1, r);
    row[nv + 2] = make_uint4(vm1.x | s.x, vm1.y | s.y, vm1.z | s.z, vm1.w | s.w);
  }
  asm volatile("griddepcontrol.launch_dependents;");
}

// One warp's tile of the two-stream kernel.  SEAMW: a W % 16 != 0 torus (the
// lanes next to the column seam load the padding vectors byte_seam_prep_kernel
// wrote, and the partial last vector is stored with its tail bytes zero).
template <int K, bool SEAMW>
__device__ __forceinline__ void byte_tb2_body(const ByteStepArgs& a, const int lane,
                                              const int64_t vi, const int64_t y0, const int n,
                                              uint4* ring) {
  constexpr int PF = kByteTb2PF;
  constexpr int kLag = 3 * K - 1;  // output row j leaves the pipeline at step j + kLag
  const int nA = (n + 1) >> 1, nB = n - nA;
  const int64_t nv = a.nv;
  int64_t src = vi % nv;
  if (src < 0) src += nv;
  if (SEAMW) src = byte_seam_src(vi, nv);
  const bool in_grid = vi >= 0 && vi < nv;
  const bool store_mid = in_grid && lane >= 1 && lane <= 30;
  const bool store_lo = in_grid && lane == 31;
  const bool store_hi = in_grid && lane == 0;
  // The partial last vector keeps its bytes past column W zero.
  uint32_t tail_mask[4] = {~0u, ~0u, ~0u, ~0u};
  if (SEAMW && vi == nv - 1) byte_tail_mask(static_cast<int>(a.width & 15), tail_mask);
  const uint32_t one = a.one;

  const int in_rows = static_cast<int>(a.in_rows);
  int rowA = static_cast<int>(wrap_row(a.in_row0, y0 - K, a.in_rows));
  int rowB = static_cast<int>(wrap_row(a.in_row0, y0 + nA - K, a.in_rows));
  const uint32_t in_pitch_b = static_cast<uint32_t>(a.in_pitch);
  const char* const in_lane = reinterpret_cast<const char*>(a.in) + src * 16;
  auto issue = [&](int slot) {
    uint4* sl = ring + slot * 64;
    cp_async16(reinterpret_cast<uint32_t*>(sl),
               row_addr(in_lane, static_cast<uint32_t>(rowA), in_pitch_b));
    cp_async16(reinterpret_cast<uint32_t*>(sl + 32),
               row_addr(in_lane, static_cast<uint32_t>(rowB), in_pitch_b));
    cp_async_commit();
    rowA = (rowA + 1 == in_rows) ? 0 : rowA + 1;
    rowB = (rowB + 1 == in_rows) ? 0 : rowB + 1;
  };
  const uint32_t out_pitch_b = static_cast<uint32_t>(a.out_pitch);
  char* const out_A = reinterpret_cast<char*>(a.out + (a.out_row0 + y0) * a.out_pitch + vi * 16);
  char* const out_B =
      reinterpret_cast<char*>(a.out + (a.out_row0 + y0 + nA) * a.out_pitch + vi * 16);

#pragma unroll
  for (int u = 0; u < PF; ++u) issue(u);
  uint32_t uh[K][4], mh[K][4], mhn[K][4], mx[K][4], xin[K][4];
#pragma unroll
  for (int g = 0; g < K; ++g)
#pragma unroll
    for (int i = 0; i < 4; ++i) uh[g][i] = mh[g][i] = mhn[g][i] = mx[g][i] = xin[g][i] = 0u;

  const int trips = (nA + kLag + PF - 1) / PF;
  int half = 0;
  // ACTIVE < K: a fill trip that runs stages 0..ACTIVE-1 only and stores
  // nothing (stage g sees valid input from step 3g on; LIFE_BYTE_FILL_PHASES).
  auto trip = [&](const int t, auto steady_tag, auto active_tag) {
    constexpr bool STEADY = decltype(steady_tag)::value;
    constexpr int ACTIVE = decltype(active_tag)::value;
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      issue((half ^ PF) + u);
      cp_async_wait<PF>();
      {
        const uint4 va = ring[(half + u) * 64];
        const uint4 vb = ring[(half + u) * 64 + 32];
        // Both streams in one word: A | B << 4 (bytes are 0/1), on the FMA pipe.
        xin[0][0] = vb.x * 16u + va.x;
        xin[0][1] = vb.y * 16u + va.y;
        xin[0][2] = vb.z * 16u + va.z;
        xin[0][3] = vb.w * 16u + va.w;
      }
      uint32_t y_last[4];
#pragma unroll
      for (int g = K - 1; g >= 0; --g) {
        if (g >= ACTIVE) continue;  // compile time
        const uint32_t lw = __shfl_up_sync(kFull, xin[g][3], 1);
        const uint32_t rw = __shfl_down_sync(kFull, xin[g][0], 1);
        uint32_t h[4], hn[4];
        byte_row_fma(xin[g], lw, rw, one, h, hn);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t o = nib_rule(uh[g][i], h[i], mhn[g][i], mx[g][i], one);
          uh[g][i] = mh[g][i];
          mh[g][i] = h[i];
          mhn[g][i] = hn[i];
          mx[g][i] = xin[g][i];
          if (g + 1 < K) {
            xin[g + 1][i] = o;
          } else {
            y_last[i] = o;
          }
        }
      }
      if constexpr (ACTIVE < K) continue;  // fill phase: no output row yet
      const int j = t * PF + u - kLag;
      uint32_t ya[4], yb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ya[i] = y_last[i] & 0x0f0f0f0fu;
        yb[i] = (y_last[i] >> 4) & 0x0f0f0f0fu;
        if (SEAMW) {
          ya[i] &= tail_mask[i];
          yb[i] &= tail_mask[i];
        }
      }
      const bool segA = STEADY || static_cast<unsigned>(j) < static_cast<unsigned>(nA);
      const bool segB = static_cast<unsigned>(j) < static_cast<unsigned>(nB);
      char* const pa = const_cast<char*>(row_addr(out_A, static_cast<uint32_t>(j), out_pitch_b));
      char* const pb = const_cast<char*>(row_addr(out_B, static_cast<uint32_t>(j), out_pitch_b));
      st_global_v4_if(pa, ya, segA && store_mid);
      st_global_v2_if(pa, ya[0], ya[1], segA && store_lo);
      st_global_v2_if(pa + 8, ya[2], ya[3], segA && store_hi);
      st_global_v4_if(pb, yb, segB && store_mid);
      st_global_v2_if(pb, yb[0], yb[1], segB && store_lo);
      st_global_v2_if(pb + 8, yb[2], yb[3], segB && store_hi);
    }
    half ^= PF;
  };
  const int steady_begin = (kLag + PF - 1) / PF;
  const int steady_end = (nA + kLag) / PF;
  using AllStages = std::integral_constant<int, K>;
  int t = 0;
#if LIFE_BYTE_FILL_PHASES
  // Two coarse fill phases of 8 steps (PF = 4): steps 0..7 need stages 0..2,
  // steps 8..15 stages 0..5; both end before the first output (step 3K - 1).
  static_assert(PF == 4, "fill phases assume 4 rows per trip");
  if constexpr (K > 3) {
    for (int r = 0; r < 2; ++r, ++t) trip(t, std::false_type{}, std::integral_constant<int, 3>{});
  }
  if constexpr (K > 6) {
    for (int r = 0; r < 2; ++r, ++t) trip(t, std::false_type{}, std::integral_constant<int, 6>{});
  }
#endif
  for (; t < trips && (t < steady_begin || t >= steady_end); ++t)
    trip(t, std::false_type{}, AllStages{});
  for (; t < steady_end; ++t) trip(t, std::true_type{}, AllStages{});
  for (; t < trips; ++t) trip(t, std::false_type{}, AllStages{});
  cp_async_wait<0>();
}

template <int K, bool SEAMW>
__global__ void __launch_bounds__(kByteThreads) byte_tb2_kernel(const ByteStepArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * kByteThreads + threadIdx.x) >> 5;
  const int strip = static_cast<int>(gwarp % a.n_strips);
  const int64_t seg = gwarp / a.n_strips;
  const int64_t y0 = seg * a.seg_rows;
  if (y0 >= a.out_rows) return;  // warp-uniform
  const int n = static_cast<int>(min(a.seg_rows, a.out_rows - y0));
  const int64_t vi = static_cast<int64_t>(strip) * kByteTbStride + lane - 1;
  extern __shared__ uint4 byte_tb2_ring[];
  uint4* ring = byte_tb2_ring + (threadIdx.x >> 5) * (2 * kByteTb2PF * 64) + lane;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: previous pass complete
  asm volatile("griddepcontrol.launch_dependents;");
  byte_tb2_body<K, SEAMW>(a, lane, vi, y0, n, ring);
}

// ---------------------------------------------------------------------------
// Packed single-generation step (K = 1, W % 128 == 0): the HBM-bound end of
// the temporal-depth range.  Each lane owns one 16-byte vector (4 words =
// 128 cells) of a row and walks a segment of rows with the 3-row window of
// (h0, h1, self) in registers; rows arrive through a cp.async ring kStep1PF
// rows ahead.  Lanes 0 and 31 are ghosts (loaded, not stored): after one
// generation only the strip's outermost bit is wrong.  Memory per
// cell-update: 1 bit read + 1 bit written (plus 2 halo rows per segment and
// the ghost vectors, both L2 hits).  Same rule network as packed_tb_kernel;
// replaces compute_region (engine.cpp:17-48) for one generation.
// ---------------------------------------------------------------------------
struct Step1Args {
  const uint32_t* in;
  int64_t in_pitch;  // words (multiple of 4)
  int64_t in_row0;
  int64_t in_rows;
  uint32_t* out;
  int64_t out_pitch;
  int64_t out_row0;
  int64_t out_rows;
  int64_t seg_rows;
  int32_t nv;        // vectors per row = W / 128
  int32_t n_strips;  // ceil(nv / 30)
};

constexpr int kStep1Threads = 128;
constexpr int kStep1PF = 8;
constexpr int kStep1Stride = 30;  // vectors stored per warp (lanes 1..30)
constexpr int kStep1Smem = (kStep1Threads / 32) * 2 * kStep1PF * 32 * 16;  // per block

struct Row4 {
  HSum h[4];
  uint32_t x[4];
};

__device__ __forceinline__ Row4 step1_row(const uint4 v) {
  const uint32_t x[4] = {v.x, v.y, v.z, v.w};
  const uint32_t left = __shfl_up_sync(kFull, x[3], 1);    // lane 0: own (ghost)
  const uint32_t right = __shfl_down_sync(kFull, x[0], 1); // lane 31: own (ghost)
  Row4 r;
  r.h[0] = hsum(left, x[0], x[1]);
  r.h[1] = hsum(x[0], x[1], x[2]);
  r.h[2] = hsum(x[1], x[2], x[3]);
  r.h[3] = hsum(x[2], x[3], right);
#pragma unroll
  for (int i = 0; i < 4; ++i) r.x[i] = x[i];
  return r;
}

__global__ void __launch_bounds__(kStep1Threads) packed_step1_kernel(const Step1Args a) {
  constexpr int PF = kStep1PF;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * kStep1Threads + threadIdx.x) >> 5;
  const int strip = static_cast<int>(gwarp % a.n_strips);
  const int64_t seg = gwarp / a.n_strips;
  const int64_t y0 = seg * a.seg_rows;
  if (y0 >= a.out_rows) return;  // warp-uniform
  const int rows = static_cast<int>(min(a.seg_rows, a.out_rows - y0));
  const int64_t vi = static_cast<int64_t>(strip) * kStep1Stride + lane - 1;
  int64_t src = vi % a.nv;  // W % 128 == 0: the torus wrap is an index remap
  if (src < 0) src += a.nv;
  const bool store = lane >= 1 && lane <= kStep1Stride && vi < a.nv;
  extern __shared__ uint4 step1_ring[];
  uint4* ring = step1_ring + (threadIdx.x >> 5) * (2 * PF * 32) + lane;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: previous pass complete
  asm volatile("griddepcontrol.launch_dependents;");

  const int in_rows = static_cast<int>(a.in_rows);
  int lrow = static_cast<int>(wrap_row(a.in_row0, y0 - 1, a.in_rows));
  const uint32_t in_pitch_b = static_cast<uint32_t>(a.in_pitch * 4);
  const char* const in_lane = reinterpret_cast<const char*>(a.in + src * 4);
  auto issue = [&](int slot) {
    cp_async16(reinterpret_cast<uint32_t*>(ring + slot * 32),
               row_addr(in_lane, static_cast<uint32_t>(lrow), in_pitch_b));
    cp_async_commit();
    lrow = (lrow + 1 == in_rows) ? 0 : lrow + 1;
  };
  const uint32_t out_pitch_b = static_cast<uint32_t>(a.out_pitch * 4);
  char* const out_lane = reinterpret_cast<char*>(a.out + (a.out_row0 + y0) * a.out_pitch + vi * 4);

#pragma unroll
  for (int u = 0; u < PF; ++u) issue(u);
  Row4 up{}, mid{};
  const int trips = (rows + 2 + PF - 1) / PF;
  int half = 0;
  auto trip = [&](const int tr, auto steady_tag) {
    constexpr bool STEADY = decltype(steady_tag)::value;
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      issue((half ^ PF) + u);
      cp_async_wait<PF>();
      const Row4 dn = step1_row(ring[(half + u) * 32]);
      const int j = tr * PF + u - 2;  // output row j leaves at step j + 2
      uint32_t o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) o[i] = rule(up.h[i], mid.h[i], dn.h[i], mid.x[i]);
      const bool st = store && (STEADY || static_cast<unsigned>(j) < static_cast<unsigned>(rows));
      st_global_v4_if(const_cast<char*>(row_addr(out_lane, static_cast<uint32_t>(j), out_pitch_b)),
                      o, st);
      up = mid;
      mid = dn;
    }
    half ^= PF;
  };
  const int steady_begin = (2 + PF - 1) / PF;
  const int steady_end = (rows + 2) / PF;
  int tr = 0;
  for (; tr < trips && (tr < steady_begin || tr >= steady_end); ++tr) trip(tr, std::false_type{});
  for (; tr < steady_end; ++tr) trip(tr, std::true_type{});
  for (; tr < trips; ++tr) trip(tr, std::false_type{});
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// Cluster-resident packed engine (small tori, W % 32 == 0): the whole torus
// lives in the distributed shared memory of ONE thread-block cluster (up to
// 16 CTAs, one per SM) and a single launch runs every generation.  CTA k of
// the cluster owns the row band band_bounds(H, C)[k] (decomposition.cpp:12-24,
// the paper's 1-D row decomposition) plus one halo row above and below,
// double-buffered in its shared memory.  Warp roles: edge warps compute band
// rows 0 and B-1, interior warps rows 1..B-2.  Per generation g:
//   __syncthreads            (this CTA's generation-g band rows are complete)
//   interior warps: rows 1..B-2 from own rows only
//   edge warps: mbarrier wait for the generation-g halo rows the neighbours
//     pushed, then rows 0 and B-1; each result is also pushed into the
//     neighbour's halo row of the next buffer with
//     st.async.shared::cluster.mbarrier::complete_tx (a DSMEM store that
//     completes the receiver's mbarrier transaction count)
// Each mbarrier phase is armed two generations ahead, before the push that
// lets the neighbours produce it; no CTA reads another's shared memory, so
// the only cross-SM latency on the critical path is the push.  One cluster
// barrier at the start (every CTA running before any push).  This replaces
// the per-generation WorkerTeam barrier (engine.cpp:79-96) with point-to-point
// DSMEM signalling, and the HBM round trip of every pass with shared memory:
// small grids (config 1) are latency-bound in the multi-pass engine (a launch
// and a grid-wide dependency per K generations); here the push chain and the
// ALU work of 16 SMs bound them.  Same rule network as packed_tb_kernel; the
// torus column wrap is an index wrap (W % 32 == 0).
// ---------------------------------------------------------------------------
struct ResidentArgs {
  const uint32_t* in;
  uint32_t* out;
  int64_t pitch;        // words per HBM row
  int32_t nw;           // W / 32
  int32_t base_rows;    // H / C
  int32_t extra_rows;   // H % C: the first extra_rows bands hold one more row
  int32_t max_rows;     // rows of the largest band (smem slab = (max_rows + 2) * nw words)
  int32_t groups;       // row groups per CTA: thread t works column t % nw, group t / nw
  int32_t generations;
};

constexpr int kResidentMaxThreads = 1024;

__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_ctas() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
// Shared-window address of the same variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t map_rank(const void* smem_ptr, uint32_t rank) {
  const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(smem_ptr));
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
  return remote;
}
// Remote store into CTA-rank memory of the cluster that also completes
// 4 bytes of the transaction count of the receiver's mbarrier.
__device__ __forceinline__ void st_async_u32(uint32_t remote_addr, uint32_t v, uint32_t remote_mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];"
               ::"r"(remote_addr), "r"(v), "r"(remote_mbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n .reg .pred done;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 done, [%0], %1;\n"
      " @!done bra WAIT_%=;\n}\n" ::"r"(a), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(kResidentMaxThreads)
packed_resident_kernel(const ResidentArgs a) {
  extern __shared__ __align__(16) uint32_t res_smem[];
  __shared__ uint64_t halo_bar[2];  // halo rows of buffer b have landed
  const int C = static_cast<int>(cluster_ctas());
  const int k = static_cast<int>(cluster_rank());
  const int nw = a.nw;
  // Per buffer: slab row 0 = halo row above the band, rows 1..B = the band,
  // row B+1 = halo row below.
  const int slab = (a.max_rows + 2) * nw;
  uint32_t* const buf0 = res_smem;
  const int B = a.base_rows + (k < a.extra_rows ? 1 : 0);
  const int64_t H = static_cast<int64_t>(a.base_rows) * C + a.extra_rows;
  const int64_t y0 = static_cast<int64_t>(k) * a.base_rows + (k < a.extra_rows ? k : a.extra_rows);
  const int up = k == 0 ? C - 1 : k - 1;
  const int dn = k == C - 1 ? 0 : k + 1;
  const int B_up = a.base_rows + (up < a.extra_rows ? 1 : 0);
  // Where our edge rows go: our row 0 is the halo below the band above
  // (its slab row B_up + 1), our row B-1 the halo above the band below.
  const uint32_t push_up = map_rank(buf0 + (B_up + 1) * nw, static_cast<uint32_t>(up));
  const uint32_t push_dn = map_rank(buf0, static_cast<uint32_t>(dn));
  const uint32_t bar_up = map_rank(halo_bar, static_cast<uint32_t>(up));
  const uint32_t bar_dn = map_rank(halo_bar, static_cast<uint32_t>(dn));
  const uint32_t halo_bytes = static_cast<uint32_t>(2 * nw * 4);

  // Band rows plus both halo rows of generation 0 straight from HBM.
  for (int i = threadIdx.x; i < (B + 2) * nw; i += blockDim.x) {
    const int r = i / nw;
    int64_t y = y0 + r - 1;
    y = y < 0 ? y + H : (y >= H ? y - H : y);
    buf0[i] = __ldg(a.in + y * a.pitch + (i - r * nw));
  }
  // Halo generation g >= 1 lands in buffer g & 1; its mbarrier phase is
  // armed two generations ahead (before we push the rows that let the
  // neighbours compute it), so no complete_tx ever precedes its expect_tx.
  if (threadIdx.x == 0) {
    mbar_init(&halo_bar[0], 1);
    mbar_init(&halo_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (a.generations >= 1) mbar_expect_tx(&halo_bar[1], halo_bytes);
    if (a.generations >= 2) mbar_expect_tx(&halo_bar[0], halo_bytes);
  }
  // Every CTA of the cluster is running (and its mbarriers initialised)
  // before anyone stores into its shared memory.
  cluster_arrive_release();
  cluster_wait_acquire();

  // Warp roles: the first ceil(2 nw / 32) warps compute the two edge rows
  // (and push them); the others the interior rows, column t % nw, a run of
  // rows per group.
  const int edge_threads = static_cast<int>((2 * nw + 31) / 32 * 32);
  const bool is_edge = static_cast<int>(threadIdx.x) < edge_threads;
  const int t = static_cast<int>(threadIdx.x) - (is_edge ? 0 : edge_threads);
  const int interior = B - 2;
  int w = t % nw, grp = t / nw;
  const bool worker = !is_edge && grp < a.groups && interior > 0;
  const int r_begin = 1 + (worker ? interior * grp / a.groups : 0);
  const int r_end = 1 + (worker ? interior * (grp + 1) / a.groups : 0);
  if (is_edge) w = t % nw;
  const int wl = w == 0 ? nw - 1 : w - 1, wr = w == nw - 1 ? 0 : w + 1;
  const bool edge_bottom = t >= nw;
  const bool edge_active = is_edge && t < 2 * nw;
  const int edge_r = edge_bottom ? B - 1 : 0;
  const uint32_t edge_push = (edge_bottom ? push_dn : push_up) + static_cast<uint32_t>(w * 4);
  const uint32_t edge_bar = edge_bottom ? bar_dn : bar_up;

  for (int g = 0; g < a.generations; ++g) {
    const int cur = g & 1;
    const uint32_t* src = buf0 + cur * slab + nw;  // band row 0
    uint32_t* dst = buf0 + (cur ^ 1) * slab + nw;
    __syncthreads();  // this CTA's generation-g band rows are in place
    if (!is_edge) {
      if (r_begin < r_end) {
        const uint32_t* p = src + (r_begin - 1) * nw;
        HSum ha = hsum(p[wl], p[w], p[wr]);
        p += nw;
        uint32_t self = p[w];
        HSum hb = hsum(p[wl], self, p[wr]);
        uint32_t* q = dst + r_begin * nw + w;
#pragma unroll 4
        for (int r = r_begin; r < r_end; ++r) {
          p += nw;
          const uint32_t x = p[w];
          const HSum hc = hsum(p[wl], x, p[wr]);
          *q = rule(ha, hb, hc, self);
          q += nw;
          ha = hb;
          hb = hc;
          self = x;
        }
      }
    } else {
      if (g >= 1) {
        const uint32_t use = static_cast<uint32_t>(cur ? (g - 1) / 2 : g / 2 - 1);
        mbar_wait(&halo_bar[cur], use & 1);  // the neighbours' pushes of our generation-g halos
        __syncwarp();
        if (threadIdx.x == 0 && g + 2 <= a.generations) mbar_expect_tx(&halo_bar[cur], halo_bytes);
      }
      if (edge_active) {
        // Edge rows 0 and B-1 (B >= 2) from local rows (the halos are
        // local copies); each result also goes to a neighbour's halo row
        // of the next buffer.
        const uint32_t* p = src + (edge_r - 1) * nw;
        const HSum ha = hsum(p[wl], p[w], p[wr]);
        p += nw;
        const uint32_t self = p[w];
        const HSum hb = hsum(p[wl], self, p[wr]);
        p += nw;
        const uint32_t v = rule(ha, hb, hsum(p[wl], p[w], p[wr]), self);
        dst[edge_r * nw + w] = v;
        st_async_u32(edge_push + static_cast<uint32_t>((cur ^ 1) * slab * 4), v,
                     edge_bar + static_cast<uint32_t>((cur ^ 1) * 8));
      }
    }
  }
  // The last pushes into our shared memory (generation G's halos) must land
  // before the CTA exits.
  const int G = a.generations;
  if (G >= 1 && is_edge) {
    const int b = G & 1;
    mbar_wait(&halo_bar[b], static_cast<uint32_t>(b ? (G - 1) / 2 : G / 2 - 1) & 1);
  }
  __syncthreads();
  const uint32_t* fin = buf0 + (G & 1) * slab + nw;
  for (int i = threadIdx.x; i < B * nw; i += blockDim.x) {
    const int r = i / nw;
    a.out[(y0 + r) * a.pitch + (i - r * nw)] = fin[i];
  }
}

// ---------------------------------------------------------------------------
// Layout conversion, seeded soup, population, windows.
// ---------------------------------------------------------------------------

// splitmix64 output (rng.hpp:22-27).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// random_fill (pattern.cpp:330-342) in counter form: cell i = y*W + x is the
// (i+1)-th draw of SplitMix64(seed), alive iff (draw >> 11) < thr where
// thr = ceil(density * 2^53) (exactly `next_unit() < density`).
// One thread per packed word; rows [y0, y0+rows) of the torus.
__global__ void packed_random_kernel(uint32_t* __restrict__ out, int64_t pitch, int64_t width,
                                     int64_t y0, int64_t rows, int32_t nw, uint64_t seed,
                                     uint64_t thr) {
  const int64_t n = rows * pitch;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / pitch;
    const int32_t w = static_cast<int32_t>(t - r * pitch);
    uint32_t word = 0;
    if (w < nw) {
      const int64_t col = static_cast<int64_t>(w) * 32;
      const int nbits = width - col < 32 ? static_cast<int>(width - col) : 32;
      uint64_t s = seed + (static_cast<uint64_t>((y0 + r) * width + col) + 1ULL) * kGamma;
      for (int j = 0; j < nbits; ++j) {
        word |= static_cast<uint32_t>((mix64(s) >> 11) < thr) << j;
        s += kGamma;
      }
    }
    out[t] = word;
  }
}

// Same soup in the byte layout (one thread per 16-byte vector).
__global__ void byte_random_kernel(uint8_t* __restrict__ out, int64_t pitch, int64_t width,
                                   int64_t y0, int64_t rows, uint64_t seed, uint64_t thr) {
  const int64_t nvec = pitch / 16;
  const int64_t n = rows * nvec;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / nvec;
    const int64_t c0 = (t - r * nvec) * 16;
    uint32_t o[4] = {0, 0, 0, 0};
    uint64_t s = seed + (static_cast<uint64_t>((y0 + r) * width + c0) + 1ULL) * kGamma;
    for (int j = 0; j < 16; ++j) {
      if (c0 + j < width) o[j >> 2] |= static_cast<uint32_t>((mix64(s) >> 11) < thr) << ((j & 3) * 8);
      s += kGamma;
    }
    *reinterpret_cast<uint4*>(out + r * pitch + c0) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// Config-4 sparse soup in counter form: block b of
// the SplitMix64(seed) stream uses draws [b*(2+bs^2), (b+1)*(2+bs^2)):
// x0 = draw % (W-bs+1), y0 = draw % (H-bs+1), then bs^2 cell draws,
// alive iff (draw >> 11) < thr.  place_pattern's overwrite order
// (pattern.cpp:309-328, later blocks win) is resolved with a per-cell
// atomicMax of (block+1): pass 1 claims, pass 2 writes the winners' cells.
__device__ __forceinline__ uint64_t draw_at(uint64_t seed, uint64_t k) {
  return mix64(seed + (k + 1) * kGamma);
}

__global__ void soup_claim_kernel(unsigned int* __restrict__ owner, int64_t width, int64_t height,
                                  int64_t blocks, int32_t bs, uint64_t seed) {
  const int64_t per = static_cast<int64_t>(bs) * bs;
  const int64_t n = blocks * per;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = t / per;
    const int j = static_cast<int>(t - b * per);
    const uint64_t k0 = static_cast<uint64_t>(b) * static_cast<uint64_t>(2 + per);
    const int64_t x0 = static_cast<int64_t>(draw_at(seed, k0) % static_cast<uint64_t>(width - bs + 1));
    const int64_t y0 = static_cast<int64_t>(draw_at(seed, k0 + 1) % static_cast<uint64_t>(height - bs + 1));
    const int64_t cell = (y0 + j / bs) * width + x0 + j % bs;
    atomicMax(owner + cell, static_cast<unsigned int>(b + 1));
  }
}

__global__ void soup_write_kernel(const unsigned int* __restrict__ owner, uint8_t* __restrict__ cells,
                                  int64_t pitch, int64_t width, int64_t height, int64_t blocks,
                                  int32_t bs, uint64_t seed, uint64_t thr) {
  const int64_t per = static_cast<int64_t>(bs) * bs;
  const int64_t n = blocks * per;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = t / per;
    const int j = static_cast<int>(t - b * per);
    const uint64_t k0 = static_cast<uint64_t>(b) * static_cast<uint64_t>(2 + per);
    const int64_t x0 = static_cast<int64_t>(draw_at(seed, k0) % static_cast<uint64_t>(width - bs + 1));
    const int64_t y0 = static_cast<int64_t>(draw_at(seed, k0 + 1) % static_cast<uint64_t>(height - bs + 1));
    const int64_t x = x0 + j % bs, y = y0 + j / bs;
    if (owner[y * width + x] == static_cast<unsigned int>(b + 1)) {
      cells[y * pitch + x] = static_cast<uint8_t>((draw_at(seed, k0 + 2 + j) >> 11) < thr);
    }
  }
}

// place_pattern (pattern.cpp:309-328) on a resident grid: the pw x ph
// footprint at (x0, y0) becomes the pattern (0/1; dead pattern cells clear).
__global__ void place_byte_kernel(uint8_t* __restrict__ cells, int64_t pitch,
                                  const uint8_t* __restrict__ pat, int64_t pw, int64_t ph,
                                  int64_t x0, int64_t y0) {
  const int64_t n = pw * ph;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = t / pw, i = t - j * pw;
    cells[(y0 + j) * pitch + x0 + i] = pat[t] != 0;
  }
}

// Packed layout: one thread per (pattern row, grid word) read-modify-write.
__global__ void place_packed_kernel(uint32_t* __restrict__ words, int64_t pitch,
                                    const uint8_t* __restrict__ pat, int64_t pw, int64_t ph,
                                    int64_t x0, int64_t y0) {
  const int64_t w_first = x0 >> 5, w_last = (x0 + pw - 1) >> 5;
  const int64_t nwords = w_last - w_first + 1;
  const int64_t n = nwords * ph;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = t / nwords;
    const int64_t w = w_first + (t - j * nwords);
    uint32_t mask = 0, bits = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t i = w * 32 + b - x0;  // pattern column
      if (i >= 0 && i < pw) {
        mask |= 1u << b;
        if (pat[j * pw + i]) bits |= 1u << b;
      }
    }
    uint32_t* p = words + (y0 + j) * pitch + w;
    *p = (*p & ~mask) | bits;
  }
}

// Byte rows -> packed rows: lane j of a warp reads column 32w+j and a warp
// ballot forms word w (coalesced byte reads, nonzero -> alive).
__global__ void pack_kernel(const uint8_t* __restrict__ cells, int64_t cell_pitch,
                            uint32_t* __restrict__ words, int64_t pitch, int64_t width,
                            int64_t rows) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t groups = (pitch + 31) / 32;  // 32-word groups per row
  for (int64_t g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
       g < rows * groups; g += nwarps) {
    const int64_t r = g / groups;
    const int64_t w0 = (g - r * groups) * 32;
    const uint8_t* row = cells + r * cell_pitch;
    uint32_t mine = 0;
    for (int j = 0; j < 32; ++j) {
      const int64_t col = (w0 + j) * 32 + lane;
      const bool alive = col < width && row[col] != 0;
      const uint32_t word = __ballot_sync(kFull, alive);
      if (j == lane) mine = word;
    }
    if (w0 + lane < pitch) words[r * pitch + w0 + lane] = mine;
  }
}

// Packed rows -> byte rows (one thread per 16 output bytes).
__global__ void unpack_kernel(const uint32_t* __restrict__ words, int64_t pitch,
                              uint8_t* __restrict__ cells, int64_t cell_pitch, int64_t width,
                              int64_t rows) {
  const int64_t nvec = cell_pitch / 16;
  const int64_t n = rows * nvec;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / nvec;
    const int64_t c0 = (t - r * nvec) * 16;
    uint32_t bits = 0;
    if (c0 < width) bits = (words[r * pitch + (c0 >> 5)] >> (c0 & 31)) & 0xffffu;
    if (width - c0 < 16 && c0 < width) bits &= (1u << (width - c0)) - 1u;
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = (((bits >> (4 * i)) & 0xfu) * 0x00204081u) & 0x01010101u;
    *reinterpret_cast<uint4*>(cells + r * cell_pitch + c0) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__device__ __forceinline__ void block_add_u64(uint64_t v, unsigned long long* dst) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  __shared__ uint64_t part[32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) part[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    if (threadIdx.x == 0 && v) atomicAdd(dst, static_cast<unsigned long long>(v));
  }
}

// population (grid.cpp:40-46) of packed rows; padding bits are zero.
__global__ void packed_popcount_kernel(const uint32_t* __restrict__ words, int64_t pitch,
                                       int32_t nw, int64_t rows, unsigned long long* count) {
  uint64_t acc = 0;
  const int64_t n = rows * pitch;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    acc += __popc(__ldg(words + t));
  }
  (void)nw;
  block_add_u64(acc, count);
}

// Live cells of the W columns of `rows` byte rows: the first nv = ceil(W/16)
// vectors of every row (bytes past column W inside vector nv-1 are zero; the
// row padding after it is scratch, see byte_seam_prep_kernel).
__global__ void byte_popcount_kernel(const uint8_t* __restrict__ cells, int64_t pitch,
                                     int64_t rows, int64_t nv, unsigned long long* count) {
  uint64_t acc = 0;
  const int64_t per_row = pitch / 16;
  const int64_t n = rows * nv;
  const uint4* v = reinterpret_cast<const uint4*>(cells);
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / nv;
    const uint4 q = __ldg(v + r * per_row + (t - r * nv));
    acc += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);  // bytes are 0/1
  }
  block_add_u64(acc, count);
}

// FNV-1a-64 of every packed row's bytes (2*ceil(W/64) little-endian uint32
// words of the device layout = the ceil(W/64) uint64 words of the exchange
// format, tail bits zero): the per-row half of life_grid_hash, a checksum of
// row checksums -- FNV itself is sequential, so rows hash in parallel and the
// host chains the H row hashes.  One thread per row.
__global__ void packed_row_hash_kernel(const uint32_t* __restrict__ words, int64_t pitch,
                                       int32_t nwords, int64_t rows,
                                       unsigned long long* __restrict__ out) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t* row = words + r * pitch;
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int32_t k = 0; k < nwords; ++k) {
      uint32_t v = __ldg(row + k);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        h ^= (v & 0xffu);
        h *= 0x100000001b3ULL;
        v >>= 8;
      }
    }
    out[r] = h;
  }
}

// Wrapped window of a packed grid as 0/1 bytes.
__global__ void packed_window_kernel(const uint32_t* __restrict__ words, int64_t pitch,
                                     int64_t width, int64_t height, int64_t x0, int64_t y0,
                                     int64_t w, int64_t h, uint8_t* __restrict__ out) {
  const int64_t n = w * h;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = t / w, i = t - j * w;
    int64_t y = (y0 + j) % height;
    if (y < 0) y += height;
    int64_t x = (x0 + i) % width;
    if (x < 0) x += width;
    out[t] = static_cast<uint8_t>((words[y * pitch + (x >> 5)] >> (x & 31)) & 1u);
  }
}

__global__ void byte_window_kernel(const uint8_t* __restrict__ cells, int64_t pitch,
                                   int64_t width, int64_t height, int64_t x0, int64_t y0,
                                   int64_t w, int64_t h, uint8_t* __restrict__ out) {
  const int64_t n = w * h;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = t / w, i = t - j * w;
    int64_t y = (y0 + j) % height;
    if (y < 0) y += height;
    int64_t x = (x0 + i) % width;
    if (x < 0) x += width;
    out[t] = cells[y * pitch + x];
  }
}

// Clears bits at columns >= W of packed rows (applied after uploads so the
// zero-padding invariant holds whatever the host sent).
__global__ void packed_mask_tail_kernel(uint32_t* __restrict__ words, int64_t pitch, int32_t nw,
                                        uint32_t tail_mask, int64_t rows) {
  const int64_t pad = pitch - nw + 1;  // word nw-1 plus the padding words
  const int64_t n = rows * pad;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / pad;
    const int64_t k = t - r * pad;
    uint32_t* p = words + r * pitch + (nw - 1) + k;
    *p = k == 0 ? (*p & tail_mask) : 0u;
  }
}

// Byte upload normalisation: nonzero -> 1 (the 0/1 contract), padding -> 0.
__global__ void byte_normalise_kernel(uint8_t* __restrict__ cells, int64_t pitch, int64_t width,
                                      int64_t rows) {
  const int64_t n = rows * pitch;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / pitch;
    const int64_t c = t - r * pitch;
    cells[t] = (c < width && cells[t] != 0) ? 1 : 0;
  }
}

// Integer-pipe peak: 8 independent LOP3 chains per thread.
__global__ void int_peak_kernel(uint32_t* sink, int64_t iters, uint32_t seed) {
  uint32_t a = seed ^ threadIdx.x, b = a * 3u, c = a * 5u, d = a * 7u;
  uint32_t e = a * 11u, f = a * 13u, g = a * 17u, h = a * 19u;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a = (a ^ b) ^ c;  b = (b & c) | d;  c = (c ^ d) ^ e;  d = (d & e) | f;
      e = (e ^ f) ^ g;  f = (f & g) | h;  g = (g ^ h) ^ a;  h = (h & a) | b;
    }
  }
  if ((a ^ b ^ c ^ d ^ e ^ f ^ g ^ h) == 0x12345678u) sink[0] = a;
}

}  // namespace lifegpu
