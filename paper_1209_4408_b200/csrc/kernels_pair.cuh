// kernels_pair.cuh -- the temporal-blocked packed step on the INTERLEAVED-PAIR
// layout (round 2): 10 integer ops per 32 cell-updates instead of 11.
//
// In the plain packed layout (kernels.cuh) every word needs two funnel shifts
// to line its left and right neighbour columns up with itself: 2 SHF of the
// 11 ops.  Here each 64-column group (one uint64 of the exchange format) is
// kept as a pair of words E / O holding its even / odd columns:
//     E bit j = column 64g + 2j,      O bit j = column 64g + 2j + 1.
// The left and right neighbours of an even column are odd columns and vice
// versa, and three of the four neighbour words are already aligned:
//     even columns:  left  = (O << 1) | (O of the group to the left  >> 31)
//                    self  = E,   right = O
//     odd columns:   left  = E,   self = O
//                    right = (E >> 1) | (E of the group to the right << 31)
// so a PAIR of words costs 2 SHF + 2 SHFL (one funnel and one shuffle per
// word instead of two each) and the rest of the network (kernels.cuh: h0/h1
// per row, t0/k0/p/q and the 3-gate rule tail, 9 LOP3 per word) is unchanged:
// 20 ops per 64 cell-updates = 0.3125 per cell-update.  Restates
// compute_region (engine.cpp:17-48) x K generations like packed_tb_kernel.
//
// A lane owns one group (8 bytes of a row, one cp.async / one vector store);
// strips are 32 groups advancing by 31, the two groups shared with the
// neighbouring strips are stored as 16-bit halves of E and O (columns 0..31
// of a group are bits 0..15 of both words).  W % 64 == 0 only (the torus
// column wrap is then an index remap, as in packed_tb_fast_kernel); the
// layout is engine-internal: grids are converted in place by
// packed_zip_kernel on their way in and out (life_gpu.cu, `pk_pair`).
#pragma once

#include "packed_common.cuh"

namespace lifegpu {

constexpr int kPairMaxDepth = 12;
constexpr int kQuadMaxDepth = 7;

// N = words per lane: 2 = the pair layout above; 4 = the QUAD layout, the same
// idea one level further: a group is 128 columns (two uint64 of the exchange
// format) kept as four words Q0..Q3, Qr bit j = column 128g + 4j + r.  Words
// Q1 and Q2 find both neighbours aligned in Q0/Q2 and Q1/Q3; only Q0's left
// and Q3's right neighbour need a funnel shift and a shuffle, so a group
// costs 2 SHF + 2 SHFL + 36 LOP3 per 128 cell-updates: 9.5 integer ops per
// 32.  Four words per stage halve the depth the registers allow (K <= 7).
#ifndef LIFE_IL_PF
#define LIFE_IL_PF 6
#endif
template <int K, int N>
struct PairTraits {
  static_assert(N == 2 || N == 4, "two or four words per lane");
  static constexpr int kPrefetch = LIFE_IL_PF;  // rows per loop trip (fetched that far ahead)
  // Warps per SM the registers allow (N words x K stages x 6 registers of
  // state per lane: N x K = 16 156 registers, 20 194, 24 234, no spills).
  static constexpr int kWarps = N * K <= 16 ? 12 : 8;
  static constexpr int kRingWords = 2 * kPrefetch * 32 * N;  // per warp: 2 PF slots x 32 lanes x N words
  static constexpr int kRingBytes = kRingWords * 4;
  static constexpr int kLag = 3 * K - 1;
};

#ifndef LIFE_PAIR_GROUP
#define LIFE_PAIR_GROUP 2
#endif
#ifndef LIFE_QUAD_GROUP
#define LIFE_QUAD_GROUP 2
#endif
// stages issued level by level together (N words each)
template <int N>
constexpr int kIlGroup = N == 2 ? LIFE_PAIR_GROUP : LIFE_QUAD_GROUP;

template <int N>
__device__ __forceinline__ void cp_async_lane(uint32_t* smem_dst, const void* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  if constexpr (N == 2) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gmem_src) : "memory");
  } else {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
  }
}

// The pair store of one output row: lanes 1..30 one 8-byte vector, the two
// shared lanes the 16-bit halves they own -- predicates, no branch.
__device__ __forceinline__ void st_pair_if(char* p, uint32_t e, uint32_t o, bool mid, bool edge,
                                           uint32_t esh) {
  char* q = p;  // edge lanes: p already points at the half they own
  asm volatile(
      "{\n .reg .pred a, b;\n setp.ne.u32 a, %3, 0;\n setp.ne.u32 b, %4, 0;\n"
      " @a st.global.v2.u32 [%0], {%1, %2};\n"
      " @b st.global.u16 [%5], %6;\n @b st.global.u16 [%5+4], %7;\n}\n" ::"l"(p),
      "r"(e), "r"(o), "r"(static_cast<uint32_t>(mid)), "r"(static_cast<uint32_t>(edge)), "l"(q),
      "h"(static_cast<uint16_t>(e >> esh)), "h"(static_cast<uint16_t>(o >> esh))
      : "memory");
}

__device__ __forceinline__ void st_quad_if(char* p, const uint32_t (&w)[4], bool mid, bool edge,
                                           uint32_t esh) {
  char* q = p;  // edge lanes: p already points at the half they own
  asm volatile(
      "{\n .reg .pred a, b;\n setp.ne.u32 a, %5, 0;\n setp.ne.u32 b, %6, 0;\n"
      " @a st.global.v4.u32 [%0], {%1, %2, %3, %4};\n"
      " @b st.global.u16 [%7], %8;\n @b st.global.u16 [%7+4], %9;\n"
      " @b st.global.u16 [%7+8], %10;\n @b st.global.u16 [%7+12], %11;\n}\n" ::"l"(p),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(static_cast<uint32_t>(mid)),
      "r"(static_cast<uint32_t>(edge)), "l"(q), "h"(static_cast<uint16_t>(w[0] >> esh)),
      "h"(static_cast<uint16_t>(w[1] >> esh)), "h"(static_cast<uint16_t>(w[2] >> esh)),
      "h"(static_cast<uint16_t>(w[3] >> esh))
      : "memory");
}

// One pipeline segment of a warp on the pair (N = 2) or quad (N = 4) layout:
// strip `strip` (32 groups from group 31*strip - 1), output rows [y, y+n).
// Same skewed K-stage register pipeline, fill-trip skipping and trip kinds as
// packed_segment's fast path.  PEER: rows outside the band come from the
// neighbour bands' buffers (multi-GPU edge strips; in_row0 is then the band
// row of y = 0).
template <int K, int N, bool UNI, bool PEER>
__device__ __forceinline__ void pair_segment(const PackedStepArgs& a, const int lane,
                                             const int strip, const int y, const int n,
                                             uint32_t* ring) {
  using T = PairTraits<K, N>;
  constexpr int kLag = T::kLag;
  constexpr int PF = T::kPrefetch;
  constexpr int LW = 32 * N;  // ring words per prefetch slot
  constexpr int G = kIlGroup<N>;
  const int in_rows = static_cast<int>(a.in_rows);
  const int64_t gi = static_cast<int64_t>(strip) * kStripStride + lane - 1;
  int64_t gs = gi % a.nw;  // a.nw = W / (32 N) groups; the torus wrap is an index remap
  if (gs < 0) gs += a.nw;

  int lrow = PEER ? static_cast<int>(a.in_row0) + y - K
                  : static_cast<int>(wrap_row(a.in_row0, static_cast<int64_t>(y) - K, a.in_rows));
  const uint32_t in_pitch_b = static_cast<uint32_t>(a.in_pitch * 4);
  const char* const in_lane = reinterpret_cast<const char*>(a.in + N * gs);
  auto issue = [&](int slot) {
    uint32_t* s = ring + slot * LW;
    if (!PEER) {
      cp_async_lane<N>(s, row_addr(in_lane, static_cast<uint32_t>(lrow), in_pitch_b));
      cp_async_commit();
      lrow = (lrow + 1 == in_rows) ? 0 : lrow + 1;
      return;
    }
    const int64_t r = lrow;
    if (r >= 0 && r < in_rows) {
      cp_async_lane<N>(s, row_addr(in_lane, static_cast<uint32_t>(lrow), in_pitch_b));
    } else {
      // A neighbour GPU's row over NVLink: a plain load (peer UVA address)
      // staged into the ring; only the 2K ghost rows of edge tiles take this.
      const uint32_t* row;
      if (r < 0) {
        row = a.up + (a.up_rows + r) * a.in_pitch;
      } else {
        const int64_t d = r - in_rows;  // rows past the light cone are over-reads: clamp
        row = a.down + (d < a.down_rows ? d : a.down_rows - 1) * a.in_pitch;
      }
      if constexpr (N == 2) {
        *reinterpret_cast<uint2*>(s) = *reinterpret_cast<const uint2*>(row + N * gs);
      } else {
        *reinterpret_cast<uint4*>(s) = *reinterpret_cast<const uint4*>(row + N * gs);
      }
    }
    cp_async_commit();
    ++lrow;
  };

  // The PF rows of one loop trip, one commit group each, into ring slots
  // slot0 .. slot0 + PF - 1.  The torus row wrap is tested once per trip
  // (warp-uniform): a trip that does not cross it takes its rows at constant
  // offsets from one address.
  auto issue_trip = [&](int slot0) {
    if (!PEER && lrow + PF <= in_rows) {
      const char* p0 = row_addr(in_lane, static_cast<uint32_t>(lrow), in_pitch_b);
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        cp_async_lane<N>(ring + (slot0 + u) * LW, p0 + static_cast<size_t>(u) * in_pitch_b);
        cp_async_commit();
      }
      lrow = (lrow + PF == in_rows) ? 0 : lrow + PF;
      return;
    }
#pragma unroll
    for (int u = 0; u < PF; ++u) issue(slot0 + u);
  };

  const bool in_grid = gi >= 0 && gi < a.nw;
  const bool st_mid = in_grid && lane >= 1 && lane <= 30;
  const bool st_edge = in_grid && (lane == 0 || lane == 31);
  // lane 0 owns the group's upper half: the high halves of its words, two
  // bytes into each -- folded into the lane's output base once
  const uint32_t esh = lane == 0 ? 16u : 0u;
  char* const out_seg =
      reinterpret_cast<char*>(a.out + (a.out_row0 + y) * a.out_pitch + N * (in_grid ? gi : 0)) +
      (lane == 0 ? 2 : 0);
  const uint32_t out_pitch_b = static_cast<uint32_t>(a.out_pitch * 4);

  issue_trip(0);

  HSum sa[K][N], sb[K][N];
  uint32_t self[K][N], x[K][N];
#pragma unroll
  for (int g = 0; g < K; ++g) {
#pragma unroll
    for (int r = 0; r < N; ++r) {
      sa[g][r] = sb[g][r] = HSum{0u, 0u};
      self[g][r] = x[g][r] = 0u;
    }
  }

  int half = 0;
  constexpr int kFill = 0, kCheck = 1, kSteady = 2, kFillPhase = 16, kDrainPhase = 32;
  auto trip = [&](const int t, auto kind_tag) {
    constexpr int KIND = decltype(kind_tag)::value;
    // kFillPhase <= KIND < kDrainPhase: a fill trip with (KIND - kFillPhase)
    // stage groups active, known at compile time (no per-group branch).
    // KIND >= kDrainPhase: one of a tile's last trips, the (KIND -
    // kDrainPhase) lowest groups skipped -- stage g's output is last needed at
    // step n + 2K - 1 + g -- otherwise a check trip.
    constexpr bool DRAIN = KIND >= kDrainPhase;
    constexpr bool FILL = KIND == kFill || (KIND >= kFillPhase && !DRAIN);
    constexpr int kActive = (KIND >= kFillPhase && !DRAIN) ? (KIND - kFillPhase) * G : K;
    constexpr int kSkipLow = DRAIN ? (KIND - kDrainPhase) * G : 0;
    issue_trip(half ^ PF);  // the next trip's rows
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      // row u of this trip: issued one trip ago, PF - 1 - u rows of that trip
      // and the PF just issued may still be in flight
      cp_async_wait_dyn<2 * PF - 1>(u);
      if constexpr (N == 2) {
        const uint2 v = *reinterpret_cast<const uint2*>(ring + (half + u) * LW);
        x[0][0] = v.x;
        x[0][1] = v.y;
      } else {
        const uint4 v = *reinterpret_cast<const uint4*>(ring + (half + u) * LW);
        x[0][0] = v.x;
        x[0][1] = v.y;
        x[0][2] = v.z;
        x[0][3] = v.w;
      }
      const int step = t * PF + u;
      uint32_t y_last[N];
#pragma unroll
      for (int r = 0; r < N; ++r) y_last[r] = 0;
#pragma unroll
      for (int g0 = ((K - 1) / G) * G; g0 >= 0; g0 -= G) {
        if constexpr (DRAIN) {
          if (g0 < kSkipLow) continue;  // compile time
        } else if constexpr (KIND >= kFillPhase) {
          if (g0 >= kActive) continue;  // compile time
        } else {
          if (FILL && step < 3 * g0) continue;
        }
        uint32_t lu[G], rd[G];
        HSum c[G][N];
#pragma unroll
        for (int j = 0; j < G; ++j) {
          if (g0 + j < K) {
            lu[j] = __shfl_up_sync(kFull, x[g0 + j][N - 1], 1);  // last word of the group to the left
            rd[j] = __shfl_down_sync(kFull, x[g0 + j][0], 1);    // first word of the group to the right
          }
        }
#pragma unroll
        for (int j = 0; j < G; ++j) {
          if (g0 + j < K) {
            const uint32_t(&w)[N] = x[g0 + j];
            // column 32N g + N j + r: the left neighbour of word r is word r-1
            // (word 0: word N-1 one bit up), the right neighbour word r+1
            // (word N-1: word 0 one bit down).
            const uint32_t lf = __funnelshift_l(lu[j], w[N - 1], 1);  // (w[N-1] << 1) | (lu >> 31)
            const uint32_t rl = __funnelshift_r(w[0], rd[j], 1);      // (w[0] >> 1) | (rd << 31)
#pragma unroll
            for (int r = 0; r < N; ++r) {
              const uint32_t l = r == 0 ? lf : w[r - 1];
              const uint32_t rr = r == N - 1 ? rl : w[r + 1];
              c[j][r] = HSum{l ^ w[r] ^ rr, maj3(l, w[r], rr)};
            }
          }
        }
#pragma unroll
        for (int j = G - 1; j >= 0; --j) {
          if (g0 + j < K) {
            const int g = g0 + j;
#pragma unroll
            for (int r = 0; r < N; ++r) {
              const uint32_t yr = rule(sa[g][r], sb[g][r], c[j][r], self[g][r]);
              sa[g][r] = sb[g][r];
              sb[g][r] = c[j][r];
              self[g][r] = x[g][r];
              if (g + 1 < K) {
                x[g + 1][r] = yr;
              } else {
                y_last[r] = yr;
              }
            }
          }
        }
      }
      const int j = step - kLag;  // output row j of the segment leaves the pipeline at step j + kLag
      if (!FILL) {
        if (UNI && (KIND == kCheck || DRAIN)) {
          const bool ok = static_cast<unsigned>(j) < static_cast<unsigned>(n);
          char* p = const_cast<char*>(row_addr(out_seg, static_cast<uint32_t>(j), out_pitch_b));
          if constexpr (N == 2) {
            st_pair_if(p, y_last[0], y_last[1], st_mid && ok, st_edge && ok, esh);
          } else {
            st_quad_if(p, y_last, st_mid && ok, st_edge && ok, esh);
          }
        } else if (KIND == kSteady || static_cast<unsigned>(j) < static_cast<unsigned>(n)) {
          char* p = const_cast<char*>(row_addr(out_seg, static_cast<uint32_t>(j), out_pitch_b));
          if constexpr (N == 2) {
            if (st_mid) *reinterpret_cast<uint2*>(p) = make_uint2(y_last[0], y_last[1]);
          } else {
            if (st_mid)
              *reinterpret_cast<uint4*>(p) = make_uint4(y_last[0], y_last[1], y_last[2], y_last[3]);
          }
          if (st_edge) {
#pragma unroll
            for (int r = 0; r < N; ++r)
              *reinterpret_cast<uint16_t*>(p + 4 * r) = static_cast<uint16_t>(y_last[r] >> esh);
          }
        }
      }
    }
    half ^= PF;
  };

  const int trips = (n + kLag + PF - 1) / PF;
  constexpr int kTopG0 = ((K - 1) / G) * G;
  // Trips that store nothing (every step before the first output, step kLag)
  // and skip the stages the input has not reached yet.
  constexpr int kFillTrips = (3 * kTopG0 + PF - 1) / PF < kLag / PF ? (3 * kTopG0 + PF - 1) / PF : kLag / PF;
  static_assert(PF * kFillTrips <= kLag, "fill trips must end before the first output");
  const int fill_trips = trips < kFillTrips ? trips : kFillTrips;
  const int steady_begin = (kLag + PF - 1) / PF;
  const int steady_end = (n + kLag) / PF;
  int t = 0;
  // Fill as phases of 3 * G steps with groups 0..p-1 active (kernels.cuh,
  // LIFE_FILL_PHASES); a fill cut short by kLag ends in the branchy body.
  constexpr bool kPhased = (LIFE_FILL_PHASES_IL == 2 || (LIFE_FILL_PHASES_IL == 1 && UNI)) &&
                           (3 * G) % PF == 0 && kTopG0 > 0;
  if constexpr (kPhased) {
    constexpr int kTripsPerPhase = 3 * G / PF;
    constexpr int kPhases = (kFillTrips / kTripsPerPhase) < (kTopG0 / G) ? (kFillTrips / kTripsPerPhase)
                                                                         : (kTopG0 / G);
    auto phases = [&](auto self, auto p_tag) {
      constexpr int P = decltype(p_tag)::value;  // groups active in this phase
      if constexpr (P <= kPhases) {
#pragma unroll 1
        for (int r = 0; r < kTripsPerPhase; ++r, ++t) trip(t, std::integral_constant<int, kFillPhase + P>{});
        self(self, std::integral_constant<int, P + 1>{});
      }
    };
    phases(phases, std::integral_constant<int, 1>{});
  }
  for (; t < fill_trips; ++t) trip(t, std::integral_constant<int, kFill>{});
  if constexpr (UNI) {
    (void)steady_begin;
    (void)steady_end;
#if LIFE_DRAIN_PHASES
    // The last two trips skip the stage groups whose outputs nothing needs
    // any more (a trip starting at step s skips group g0 if s >= n + 2K + g0
    // + G - 1), from bodies specialised on the number of skipped groups.
    constexpr int kMaxD = (kTopG0 / G) < 3 ? (kTopG0 / G) : 3;
    auto drain_trip = [&](const int tt) {
      const int x = tt * PF - (n + 2 * K + G - 1);
      const int d = x < 0 ? 0 : (x / G + 1 < kMaxD ? x / G + 1 : kMaxD);
      if constexpr (kMaxD >= 3) {
        if (d == 3) return trip(tt, std::integral_constant<int, kDrainPhase + 3>{});
      }
      if constexpr (kMaxD >= 2) {
        if (d == 2) return trip(tt, std::integral_constant<int, kDrainPhase + 2>{});
      }
      if constexpr (kMaxD >= 1) {
        if (d == 1) return trip(tt, std::integral_constant<int, kDrainPhase + 1>{});
      }
      return trip(tt, std::integral_constant<int, kCheck>{});
    };
#pragma unroll 1
    for (; t < trips - 2; ++t) trip(t, std::integral_constant<int, kCheck>{});
#pragma unroll 1
    for (; t < trips; ++t) drain_trip(t);
#else
#pragma unroll 1
    for (; t < trips; ++t) trip(t, std::integral_constant<int, kCheck>{});
#endif
  } else {
    for (; t < trips && (t < steady_begin || t >= steady_end); ++t)
      trip(t, std::integral_constant<int, kCheck>{});
    for (; t < steady_end; ++t) trip(t, std::integral_constant<int, kSteady>{});
    for (; t < trips; ++t) trip(t, std::integral_constant<int, kCheck>{});
  }
  cp_async_wait<0>();
}

// Tiles = (strip, segment), strip fastest, one per warp; no block barrier.
template <int K, int N, bool UNI, bool PEER>
__global__ void __launch_bounds__(32 * PairTraits<K, N>::kWarps)
packed_il_kernel(const PackedStepArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t tile = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int strip = static_cast<int>(tile % a.n_strips);
  const int64_t seg = tile / a.n_strips;
  const int64_t y0 = seg * a.seg_rows;
  const int64_t left = a.out_rows - y0;
  const int n = static_cast<int>(left <= 0 ? 0 : (left < a.seg_rows ? left : a.seg_rows));
  if (n == 0) return;  // warp-uniform
  extern __shared__ __align__(16) uint32_t ring_pair_smem[];
  uint32_t* ring = ring_pair_smem + (threadIdx.x >> 5) * PairTraits<K, N>::kRingWords + N * lane;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: previous pass complete
  asm volatile("griddepcontrol.launch_dependents;");
  pair_segment<K, N, UNI, PEER>(a, lane, strip, static_cast<int>(y0), n, ring);
}

// ---------------------------------------------------------------------------
// Layout conversion, in place, rows [row0, row0 + rows) of a packed buffer:
// plain packed (bit j of uint64 group g = column 64g + j) <-> interleaved
// pair (E = even columns, O = odd columns).  Grid: x over groups, y strides rows.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t compress_even(uint32_t x) {  // bits 0,2,4,.. -> bits 0..15
  x &= 0x55555555u;
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0f0f0f0fu;
  x = (x | (x >> 4)) & 0x00ff00ffu;
  x = (x | (x >> 8)) & 0x0000ffffu;
  return x;
}
__device__ __forceinline__ uint32_t spread_even(uint32_t x) {  // bits 0..15 -> bits 0,2,4,..
  x &= 0x0000ffffu;
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

__device__ __forceinline__ uint32_t compress_4th(uint32_t x) {  // bits 0,4,8,.. -> bits 0..7
  x &= 0x11111111u;
  x = (x | (x >> 3)) & 0x03030303u;
  x = (x | (x >> 6)) & 0x000f000fu;
  x = (x | (x >> 12)) & 0x000000ffu;
  return x;
}
__device__ __forceinline__ uint32_t spread_4th(uint32_t x) {  // bits 0..7 -> bits 0,4,8,..
  x &= 0x000000ffu;
  x = (x | (x << 12)) & 0x000f000fu;
  x = (x | (x << 6)) & 0x03030303u;
  x = (x | (x << 3)) & 0x11111111u;
  return x;
}

template <bool UNZIP, int N>
__global__ void __launch_bounds__(256)
packed_zip_kernel(uint32_t* __restrict__ words, int64_t pitch, int64_t groups, int64_t row0,
                  int64_t rows) {
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    if constexpr (N == 2) {
      uint2* p = reinterpret_cast<uint2*>(words + (row0 + r) * pitch) + g;
      const uint2 v = *p;
      uint2 w;
      if (UNZIP) {  // v = (E, O) -> (columns 0..31, columns 32..63)
        w.x = spread_even(v.x) | (spread_even(v.y) << 1);
        w.y = spread_even(v.x >> 16) | (spread_even(v.y >> 16) << 1);
      } else {
        w.x = compress_even(v.x) | (compress_even(v.y) << 16);
        w.y = compress_even(v.x >> 1) | (compress_even(v.y >> 1) << 16);
      }
      *p = w;
    } else {
      uint4* p = reinterpret_cast<uint4*>(words + (row0 + r) * pitch) + g;
      const uint4 v4 = *p;
      const uint32_t v[4] = {v4.x, v4.y, v4.z, v4.w};
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        w[i] = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (UNZIP)  // plain word i = columns 32i..32i+31: bit 4m + k from Qk bit 8i + m
            w[i] |= spread_4th(v[k] >> (8 * i)) << k;
          else        // Qi byte k = plain word k's bits i, i+4, ..
            w[i] |= compress_4th(v[k] >> i) << (8 * k);
        }
      }
      *p = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

}  // namespace lifegpu
