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

template <int K>
struct PairTraits {
  static constexpr int kPrefetch = 6;  // rows per loop trip (fetched that far ahead)
  // Warps per SM the registers allow (2 words x K stages x 6 registers of
  // state per lane: K = 8 156 registers, K = 10 194, K = 12 234, no spills).
  static constexpr int kWarps = K <= 8 ? 12 : 8;
  static constexpr int kRingWords = 2 * kPrefetch * 64;  // per warp: 2 PF slots x 32 lanes x 2 words
  static constexpr int kRingBytes = kRingWords * 4;
  static constexpr int kLag = 3 * K - 1;
};

#ifndef LIFE_PAIR_GROUP
#define LIFE_PAIR_GROUP 2
#endif
constexpr int kPairGroup = LIFE_PAIR_GROUP;  // stages issued level by level together (2 words each)

__device__ __forceinline__ void cp_async8(uint32_t* smem_dst, const void* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gmem_src) : "memory");
}

// The pair store of one output row: lanes 1..30 one 8-byte vector, the two
// shared lanes the 16-bit halves they own -- predicates, no branch.
__device__ __forceinline__ void st_pair_if(char* p, uint32_t e, uint32_t o, bool mid, bool edge,
                                           uint32_t eoff, uint32_t esh) {
  char* q = p + eoff;
  asm volatile(
      "{\n .reg .pred a, b;\n setp.ne.u32 a, %3, 0;\n setp.ne.u32 b, %4, 0;\n"
      " @a st.global.v2.u32 [%0], {%1, %2};\n"
      " @b st.global.u16 [%5], %6;\n @b st.global.u16 [%5+4], %7;\n}\n" ::"l"(p),
      "r"(e), "r"(o), "r"(static_cast<uint32_t>(mid)), "r"(static_cast<uint32_t>(edge)), "l"(q),
      "h"(static_cast<uint16_t>(e >> esh)), "h"(static_cast<uint16_t>(o >> esh))
      : "memory");
}

// One pipeline segment of a warp on the pair layout: strip `strip` (32 groups
// from group 31*strip - 1), output rows [y, y+n).  Same skewed K-stage
// register pipeline, fill-trip skipping and trip kinds as packed_segment's
// fast path.  PEER: rows outside the band come from the neighbour bands'
// buffers (multi-GPU edge strips; in_row0 is then the band row of y = 0).
template <int K, bool UNI, bool PEER>
__device__ __forceinline__ void pair_segment(const PackedStepArgs& a, const int lane,
                                             const int strip, const int y, const int n,
                                             uint32_t* ring) {
  constexpr int kLag = PairTraits<K>::kLag;
  constexpr int PF = PairTraits<K>::kPrefetch;
  const int in_rows = static_cast<int>(a.in_rows);
  const int64_t gi = static_cast<int64_t>(strip) * kStripStride + lane - 1;
  int64_t gs = gi % a.nw;  // a.nw = W / 64 groups; the torus wrap is an index remap
  if (gs < 0) gs += a.nw;

  int lrow = PEER ? static_cast<int>(a.in_row0) + y - K
                  : static_cast<int>(wrap_row(a.in_row0, static_cast<int64_t>(y) - K, a.in_rows));
  const uint32_t in_pitch_b = static_cast<uint32_t>(a.in_pitch * 4);
  const char* const in_lane = reinterpret_cast<const char*>(a.in + 2 * gs);
  auto issue = [&](int slot) {
    uint32_t* s = ring + slot * 64;
    if (!PEER) {
      cp_async8(s, row_addr(in_lane, static_cast<uint32_t>(lrow), in_pitch_b));
      cp_async_commit();
      lrow = (lrow + 1 == in_rows) ? 0 : lrow + 1;
      return;
    }
    const int64_t r = lrow;
    if (r >= 0 && r < in_rows) {
      cp_async8(s, row_addr(in_lane, static_cast<uint32_t>(lrow), in_pitch_b));
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
      *reinterpret_cast<uint2*>(s) = *reinterpret_cast<const uint2*>(row + 2 * gs);
    }
    cp_async_commit();
    ++lrow;
  };

  const bool in_grid = gi >= 0 && gi < a.nw;
  const bool st_mid = in_grid && lane >= 1 && lane <= 30;
  const bool st_edge = in_grid && (lane == 0 || lane == 31);
  const uint32_t eoff = lane == 0 ? 2u : 0u;   // lane 0 owns columns 32..63: the high halves
  const uint32_t esh = lane == 0 ? 16u : 0u;
  char* const out_seg =
      reinterpret_cast<char*>(a.out + (a.out_row0 + y) * a.out_pitch + 2 * (in_grid ? gi : 0));
  const uint32_t out_pitch_b = static_cast<uint32_t>(a.out_pitch * 4);

#pragma unroll
  for (int u = 0; u < PF; ++u) issue(u);

  HSum saE[K], saO[K], sbE[K], sbO[K];
  uint32_t selfE[K], selfO[K], xE[K], xO[K];
#pragma unroll
  for (int g = 0; g < K; ++g) {
    saE[g] = saO[g] = sbE[g] = sbO[g] = HSum{0u, 0u};
    selfE[g] = selfO[g] = xE[g] = xO[g] = 0u;
  }

  int half = 0;
  constexpr int kFill = 0, kCheck = 1, kSteady = 2;
  auto trip = [&](const int t, auto kind_tag) {
    constexpr int KIND = decltype(kind_tag)::value;
    constexpr bool FILL = KIND == kFill;
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      issue((half ^ PF) + u);
      cp_async_wait<PF>();
      {
        const uint2 v = *reinterpret_cast<const uint2*>(ring + (half + u) * 64);
        xE[0] = v.x;
        xO[0] = v.y;
      }
      const int step = t * PF + u;
      uint32_t yE_last = 0, yO_last = 0;
#pragma unroll
      for (int g0 = ((K - 1) / kPairGroup) * kPairGroup; g0 >= 0; g0 -= kPairGroup) {
        if (FILL && step < 3 * g0) continue;
        uint32_t ou[kPairGroup], ed[kPairGroup];
        HSum cE[kPairGroup], cO[kPairGroup];
#pragma unroll
        for (int j = 0; j < kPairGroup; ++j) {
          if (g0 + j < K) {
            ou[j] = __shfl_up_sync(kFull, xO[g0 + j], 1);    // odd columns of the group to the left
            ed[j] = __shfl_down_sync(kFull, xE[g0 + j], 1);  // even columns of the group to the right
          }
        }
#pragma unroll
        for (int j = 0; j < kPairGroup; ++j) {
          if (g0 + j < K) {
            const uint32_t e = xE[g0 + j], o = xO[g0 + j];
            const uint32_t le = __funnelshift_l(ou[j], o, 1);  // (o << 1) | (ou >> 31)
            const uint32_t ro = __funnelshift_r(e, ed[j], 1);  // (e >> 1) | (ed << 31)
            cE[j] = HSum{le ^ e ^ o, maj3(le, e, o)};
            cO[j] = HSum{e ^ o ^ ro, maj3(e, o, ro)};
          }
        }
#pragma unroll
        for (int j = kPairGroup - 1; j >= 0; --j) {
          if (g0 + j < K) {
            const int g = g0 + j;
            const uint32_t ye = rule(saE[g], sbE[g], cE[j], selfE[g]);
            const uint32_t yo = rule(saO[g], sbO[g], cO[j], selfO[g]);
            saE[g] = sbE[g];
            saO[g] = sbO[g];
            sbE[g] = cE[j];
            sbO[g] = cO[j];
            selfE[g] = xE[g];
            selfO[g] = xO[g];
            if (g + 1 < K) {
              xE[g + 1] = ye;
              xO[g + 1] = yo;
            } else {
              yE_last = ye;
              yO_last = yo;
            }
          }
        }
      }
      const int j = step - kLag;  // output row j of the segment leaves the pipeline at step j + kLag
      if (!FILL) {
        if (UNI && KIND == kCheck) {
          const bool ok = static_cast<unsigned>(j) < static_cast<unsigned>(n);
          char* p = const_cast<char*>(row_addr(out_seg, static_cast<uint32_t>(j), out_pitch_b));
          st_pair_if(p, yE_last, yO_last, st_mid && ok, st_edge && ok, eoff, esh);
        } else if (KIND == kSteady || static_cast<unsigned>(j) < static_cast<unsigned>(n)) {
          char* p = const_cast<char*>(row_addr(out_seg, static_cast<uint32_t>(j), out_pitch_b));
          if (st_mid) *reinterpret_cast<uint2*>(p) = make_uint2(yE_last, yO_last);
          if (st_edge) {
            *reinterpret_cast<uint16_t*>(p + eoff) = static_cast<uint16_t>(yE_last >> esh);
            *reinterpret_cast<uint16_t*>(p + eoff + 4) = static_cast<uint16_t>(yO_last >> esh);
          }
        }
      }
    }
    half ^= PF;
  };

  const int trips = (n + kLag + PF - 1) / PF;
  constexpr int kTopG0 = ((K - 1) / kPairGroup) * kPairGroup;
  constexpr int kFillTrips = (3 * kTopG0 + PF - 1) / PF;
  static_assert(PF * kFillTrips <= kLag || kFillTrips == 0, "fill trips must end before the first output");
  const int fill_trips = trips < kFillTrips ? trips : kFillTrips;
  const int steady_begin = (kLag + PF - 1) / PF;
  const int steady_end = (n + kLag) / PF;
  int t = 0;
  for (; t < fill_trips; ++t) trip(t, std::integral_constant<int, kFill>{});
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
}

// Tiles = (strip, segment), strip fastest, one per warp; no block barrier.
template <int K, bool UNI, bool PEER>
__global__ void __launch_bounds__(32 * PairTraits<K>::kWarps)
packed_pair_kernel(const PackedStepArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t tile = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int strip = static_cast<int>(tile % a.n_strips);
  const int64_t seg = tile / a.n_strips;
  const int64_t y0 = seg * a.seg_rows;
  const int64_t left = a.out_rows - y0;
  const int n = static_cast<int>(left <= 0 ? 0 : (left < a.seg_rows ? left : a.seg_rows));
  if (n == 0) return;  // warp-uniform
  extern __shared__ uint32_t ring_pair_smem[];
  uint32_t* ring = ring_pair_smem + (threadIdx.x >> 5) * PairTraits<K>::kRingWords + 2 * lane;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: previous pass complete
  asm volatile("griddepcontrol.launch_dependents;");
  pair_segment<K, UNI, PEER>(a, lane, strip, static_cast<int>(y0), n, ring);
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

template <bool UNZIP>
__global__ void __launch_bounds__(256)
packed_zip_kernel(uint32_t* __restrict__ words, int64_t pitch, int64_t groups, int64_t row0,
                  int64_t rows) {
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
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
  }
}

}  // namespace lifegpu
