// life_multi.cu -- multi-device contexts (life_ctx_create_multi): the torus
// split into row bands across GPUs inside ONE call of the step loop.
//
// Reference: run(Grid&&, RunConfig{Strategy::rows(), workers}) (engine.cpp:
// 162-214) cuts the rows into `workers` bands with band_bounds
// (decomposition.cpp:12-24, partition_rows :93-104) and steps every band on
// its own thread, with a full barrier per generation (WorkerTeam,
// engine.cpp:60-125).  Here a band lives on a GPU and one pass advances it K
// generations; the per-generation barrier becomes per-pass CUDA-event edges
// between NEIGHBOURING bands only:
//
//   pass p of band b, reading buffer src = buf[p & 1], writing dst:
//     interior (compute stream): output rows [K, rows-K) from the band's own
//       rows -- the packed temporal-blocked kernel, no halo at all;
//     edges (edge stream): output rows [0, K) and [rows-K, rows), reading
//       the K last rows of band b-1 and the K first rows of band b+1 straight
//       from the neighbours' HBM inside the kernel (LIFE_HALO_PEER, NVLink
//       P2P loads), or from local ghost rows copied first (LIFE_HALO_COPY).
//   dependencies (events recorded per pass, two slots by pass parity):
//     interior(b,p) after edges(b,p-1)      -- it reads rows [0,K) they wrote;
//     edges(b,p)   after interior(b,p-1)    -- it reads rows [K,2K) it wrote,
//                                              and overwrites rows it read;
//     edges(b,p)   after edges(b+-1,p-1)    -- the neighbours' rows it reads
//                                              were written by those, and
//                                              those read the rows it writes.
//   (A pass shallower than the last one -- a checkpoint split -- also makes
//   interior(b,p) wait for the neighbours' edges; a deeper one makes edges(b,p)
//   wait for the neighbours' interiors, since the rows they read grew.)
//
// Interior and edges of one pass run concurrently; nothing waits on a band
// that is not a neighbour.  Bands may repeat a device: the same events and
// kernels, several bands per GPU.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/life_gpu.h"
#include "internal.h"

namespace lifegpu {
namespace detail {

namespace {

struct Band {
  int device = 0;
  int64_t y0 = 0, rows = 0;
  uint32_t* buf[2] = {nullptr, nullptr};
  uint32_t* ghost[2] = {nullptr, nullptr};  // LIFE_HALO_COPY: K rows above / below
  cudaStream_t main = nullptr, edge = nullptr, h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_int[2] = {nullptr, nullptr}, ev_edge[2] = {nullptr, nullptr};
  cudaEvent_t ev_up = nullptr, ev_comp = nullptr, ev_down = nullptr;  // life_run_batch
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  SplitStreams split;
  unsigned long long* counts = nullptr;
  int64_t counts_cap = 0;
  uint64_t* row_hashes = nullptr;
  int64_t row_hashes_cap = 0;
  uint8_t* scratch = nullptr;
  int64_t scratch_cap = 0;
  uint32_t* batch[4] = {nullptr, nullptr, nullptr, nullptr};  // 2 slots x (ping, pong)
  size_t batch_bytes = 0;
  std::vector<cudaEvent_t> prof_int, prof_edge;  // LIFE_OPT_PROFILE: pairs per pass
  int64_t passes = 0;
  double run_ms = 0.0, interior_ms = 0.0, edge_ms = 0.0;
};

constexpr int kMaxGhostRows = LIFE_MAX_TEMPORAL_DEPTH;
constexpr int64_t kScratchBytes = int64_t(64) << 20;  // byte-row staging per chunk

}  // namespace

struct MultiState {
  std::vector<Band> bands;
  int halo = LIFE_HALO_PEER;
  bool peer_ok = true;  // every pair of neighbouring bands can use P2P loads
  bool profile = false;
  bool loaded = false;
  int64_t W = 0, H = 0, pitch = 0;
  int cur = 0;
  // Layout of the resident bands buf[cur]: 0 plain, 2 pair, 4 quad
  // (kernels_pair.cuh); left interleaved by multi_run between runs; every
  // reader of the plain layout calls to_plain() first.
  int il = 0;
  int pair_depth = -1;  // LIFE_OPT_PAIR_DEPTH
  int quad_depth = -1;  // LIFE_OPT_QUAD_DEPTH
  int64_t batch_bytes_total = 0;
};

namespace {

int nbands(const MultiState* m) { return static_cast<int>(m->bands.size()); }
int up_of(const MultiState* m, int b) { return (b + nbands(m) - 1) % nbands(m); }
int down_of(const MultiState* m, int b) { return (b + 1) % nbands(m); }

int use(const Band& b) {
  LIFE_CUDA(cudaSetDevice(b.device));
  return LIFE_OK;
}

void free_band_buffers(Band& b) {
  cudaSetDevice(b.device);
  for (auto& p : b.buf) {
    if (p) cudaFree(p);
    p = nullptr;
  }
  for (auto& p : b.ghost) {
    if (p) cudaFree(p);
    p = nullptr;
  }
}

int ensure_scratch(Band& b, int64_t bytes) {
  if (bytes <= b.scratch_cap) return LIFE_OK;
  if (b.scratch) cudaFree(b.scratch);
  b.scratch = nullptr;
  b.scratch_cap = 0;
  LIFE_CUDA(cudaMalloc(&b.scratch, bytes));
  b.scratch_cap = bytes;
  return LIFE_OK;
}

int sync_all(MultiState* m) {
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    for (cudaStream_t s : {b.main, b.edge, b.h2d, b.d2h, b.split.side})
      if (s) LIFE_CUDA(cudaStreamSynchronize(s));
  }
  return LIFE_OK;
}

// Band layout for an H-row torus; reallocates when the dimensions change.
int set_dims(MultiState* m, int64_t w, int64_t h) {
  LIFE_TRY(check_dims(w, h));
  const int n = nbands(m);
  std::vector<int64_t> bounds(n + 1);
  LIFE_TRY(life_band_bounds(h, n, bounds.data()));  // TooManyParts when n > H
  if (w == m->W && h == m->H && m->loaded) return LIFE_OK;
  LIFE_TRY(sync_all(m));
  m->W = w;
  m->H = h;
  m->pitch = life_packed_pitch_words(w);
  m->loaded = false;
  for (int i = 0; i < n; ++i) {
    Band& b = m->bands[i];
    free_band_buffers(b);
    b.y0 = bounds[i];
    b.rows = bounds[i + 1] - bounds[i];
    LIFE_TRY(use(b));
    const size_t bytes = static_cast<size_t>(b.rows) * m->pitch * 4;
    for (auto& p : b.buf) {
      LIFE_CUDA(cudaMalloc(&p, bytes));
      LIFE_CUDA(cudaMemsetAsync(p, 0, bytes, b.main));
    }
  }
  m->cur = 0;
  m->il = 0;
  return LIFE_OK;
}

int ensure_ghosts(MultiState* m) {
  for (Band& b : m->bands) {
    if (b.ghost[0]) continue;
    LIFE_TRY(use(b));
    const size_t bytes = static_cast<size_t>(kMaxGhostRows) * m->pitch * 4;
    for (auto& p : b.ghost) {
      LIFE_CUDA(cudaMalloc(&p, bytes));
      LIFE_CUDA(cudaMemsetAsync(p, 0, bytes, b.main));
    }
  }
  return LIFE_OK;
}

int ensure_counts(Band& b, int64_t n) {
  if (n <= b.counts_cap) return LIFE_OK;
  if (b.counts) cudaFree(b.counts);
  b.counts = nullptr;
  b.counts_cap = 0;
  LIFE_CUDA(cudaMalloc(&b.counts, sizeof(unsigned long long) * n));
  b.counts_cap = n;
  return LIFE_OK;
}

int check_loaded(const MultiState* m) {
  if (!m->loaded) return set_error(LIFE_ERR_STATE, "no grid loaded");
  return LIFE_OK;
}

// Rows [r0, r0 + rows) of a packed host grid (uint64 rows of wpr words)
// <-> the same rows of band buffer `dev` (pitch words), on stream s.
// Layout conversion of the resident bands, in place on each band's stream.
int to_plain(MultiState* m) {
  if (m->il == 0) return LIFE_OK;
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    LIFE_TRY(packed_zip(m->il, b.buf[m->cur], m->pitch, m->W, 0, b.rows, /*unzip=*/true, b.main));
  }
  m->il = 0;
  return LIFE_OK;
}
int to_il(MultiState* m, int il) {
  if (m->il == il) return LIFE_OK;
  LIFE_TRY(to_plain(m));
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    LIFE_TRY(packed_zip(il, b.buf[m->cur], m->pitch, m->W, 0, b.rows, /*unzip=*/false, b.main));
  }
  m->il = il;
  return LIFE_OK;
}

int copy_band_rows(const MultiState* m, void* host, int64_t words_per_row, uint32_t* dev,
                   int64_t rows, bool h2d, cudaStream_t s) {
  const int64_t wpr = ceil_div(m->W, 64);
  if (rows == 0) return LIFE_OK;
  if (h2d) {
    LIFE_CUDA(cudaMemcpy2DAsync(dev, m->pitch * 4, host, words_per_row * 8, wpr * 8, rows,
                                cudaMemcpyHostToDevice, s));
  } else {
    LIFE_CUDA(cudaMemcpy2DAsync(host, words_per_row * 8, dev, m->pitch * 4, wpr * 8, rows,
                                cudaMemcpyDeviceToHost, s));
  }
  return LIFE_OK;
}

// One pass of depth k (the previous pass had depth kprev; 0 = none) over every
// band: src[b] -> dst[b].  Pass index p selects the event slots.
int issue_pass(MultiState* m, uint32_t* const* src, uint32_t* const* dst, int64_t p, int k,
               int kprev, int il) {
  // One torus / interior launch and one edge-strip launch on either layout.
  auto step = [&](const uint32_t* in, int64_t in_row0, int64_t in_rows, uint32_t* out,
                  int64_t out_rows, cudaStream_t s, SplitStreams* ss) -> int {
    if (il != 0)
      return packed_il_step(il, in, m->pitch, in_row0, in_rows, out, m->pitch, in_row0, m->W,
                            out_rows, k, s);
    return packed_step(in, m->pitch, in_row0, in_rows, out, m->pitch, in_row0, m->W, out_rows, k,
                       s, ss);
  };
  auto step_peer = [&](const uint32_t* in, const uint32_t* up, int64_t up_rows,
                       const uint32_t* down, int64_t down_rows, int64_t band_rows, uint32_t* out,
                       int64_t out_row0, int64_t out_rows, cudaStream_t s) -> int {
    if (il != 0)
      return packed_il_step_peer(il, in, up, up_rows, down, down_rows, m->pitch, band_rows, out,
                                 out_row0, out_rows, m->W, k, s);
    return life_dev_packed_step_peer(in, up, up_rows, down, down_rows, m->pitch, band_rows, out,
                                     out_row0, out_rows, m->W, k, static_cast<void*>(s));
  };
  const int n = nbands(m);
  const int now = static_cast<int>(p & 1), prev = now ^ 1;
  auto prof_event = [&](std::vector<cudaEvent_t>& v, cudaStream_t s) -> int {
    cudaEvent_t e;
    LIFE_CUDA(cudaEventCreate(&e));
    v.push_back(e);
    LIFE_CUDA(cudaEventRecord(e, s));
    return LIFE_OK;
  };
  if (n == 1) {  // the whole torus: the kernel wraps rows itself
    Band& b = m->bands[0];
    LIFE_TRY(use(b));
    if (m->profile) LIFE_TRY(prof_event(b.prof_int, b.main));
    LIFE_TRY(step(src[0], 0, b.rows, dst[0], b.rows, b.main, &b.split));
    if (m->profile) LIFE_TRY(prof_event(b.prof_int, b.main));
    LIFE_CUDA(cudaEventRecord(b.ev_int[now], b.main));
    LIFE_CUDA(cudaEventRecord(b.ev_edge[now], b.main));
    ++b.passes;
    return LIFE_OK;
  }
  // Interiors first (the long launches), then the edge strips.
  for (int i = 0; i < n; ++i) {
    Band& b = m->bands[i];
    LIFE_TRY(use(b));
    LIFE_CUDA(cudaStreamWaitEvent(b.main, b.ev_edge[prev], 0));
    if (k < kprev) {  // rows [k, kprev) were read by the neighbours' last edges
      LIFE_CUDA(cudaStreamWaitEvent(b.main, m->bands[up_of(m, i)].ev_edge[prev], 0));
      LIFE_CUDA(cudaStreamWaitEvent(b.main, m->bands[down_of(m, i)].ev_edge[prev], 0));
    }
    if (b.rows > 2 * k) {
      if (m->profile) LIFE_TRY(prof_event(b.prof_int, b.main));
      LIFE_TRY(step(src[i], k, b.rows, dst[i], b.rows - 2 * k, b.main, &b.split));
      if (m->profile) LIFE_TRY(prof_event(b.prof_int, b.main));
    }
    LIFE_CUDA(cudaEventRecord(b.ev_int[now], b.main));
  }
  for (int i = 0; i < n; ++i) {
    Band& b = m->bands[i];
    const int iu = up_of(m, i), id = down_of(m, i);
    Band& u = m->bands[iu];
    Band& d = m->bands[id];
    LIFE_TRY(use(b));
    LIFE_CUDA(cudaStreamWaitEvent(b.edge, b.ev_int[prev], 0));
    LIFE_CUDA(cudaStreamWaitEvent(b.edge, u.ev_edge[prev], 0));
    LIFE_CUDA(cudaStreamWaitEvent(b.edge, d.ev_edge[prev], 0));
    if (k > kprev) {  // the neighbour rows read now were partly written by their interiors
      LIFE_CUDA(cudaStreamWaitEvent(b.edge, u.ev_int[prev], 0));
      LIFE_CUDA(cudaStreamWaitEvent(b.edge, d.ev_int[prev], 0));
    }
    if (m->profile) LIFE_TRY(prof_event(b.prof_edge, b.edge));
    const uint32_t* up = src[iu];
    const uint32_t* down = src[id];
    int64_t up_rows = u.rows, down_rows = d.rows;
    if (m->halo == LIFE_HALO_COPY) {
      const size_t bytes = static_cast<size_t>(k) * m->pitch * 4;
      LIFE_CUDA(cudaMemcpyPeerAsync(b.ghost[0], b.device, src[iu] + (u.rows - k) * m->pitch,
                                    u.device, bytes, b.edge));
      LIFE_CUDA(cudaMemcpyPeerAsync(b.ghost[1], b.device, src[id], d.device, bytes, b.edge));
      up = b.ghost[0];
      down = b.ghost[1];
      up_rows = down_rows = k;
    }
    if (b.rows > 2 * k) {
      LIFE_TRY(step_peer(src[i], up, up_rows, down, down_rows, b.rows, dst[i], 0, k, b.edge));
      LIFE_TRY(step_peer(src[i], up, up_rows, down, down_rows, b.rows, dst[i], b.rows - k, k,
                         b.edge));
    } else {
      LIFE_TRY(step_peer(src[i], up, up_rows, down, down_rows, b.rows, dst[i], 0, b.rows, b.edge));
    }
    if (m->profile) LIFE_TRY(prof_event(b.prof_edge, b.edge));
    LIFE_CUDA(cudaEventRecord(b.ev_edge[now], b.edge));
    ++b.passes;
  }
  return LIFE_OK;
}

// Marks the start of a pass sequence: the "previous pass" events of every
// band complete when its compute stream reaches this point.
int mark_start(MultiState* m) {
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    LIFE_CUDA(cudaEventRecord(b.ev_int[1], b.main));
    LIFE_CUDA(cudaEventRecord(b.ev_edge[1], b.main));
  }
  return LIFE_OK;
}

// The band's compute stream waits for everything of pass p.
int join_pass(MultiState* m, int64_t p) {
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    LIFE_CUDA(cudaStreamWaitEvent(b.main, b.ev_edge[p & 1], 0));
  }
  return LIFE_OK;
}

void clear_prof(Band& b) {
  for (cudaEvent_t e : b.prof_int) cudaEventDestroy(e);
  for (cudaEvent_t e : b.prof_edge) cudaEventDestroy(e);
  b.prof_int.clear();
  b.prof_edge.clear();
}

int sum_pairs(const std::vector<cudaEvent_t>& v, double* out) {
  *out = 0.0;
  for (size_t i = 0; i + 1 < v.size(); i += 2) {
    float ms = 0.0f;
    LIFE_CUDA(cudaEventElapsedTime(&ms, v[i], v[i + 1]));
    *out += ms;
  }
  return LIFE_OK;
}

int check_packed_engine(int engine) {
  if (engine != LIFE_ENGINE_PACKED)
    return set_error(LIFE_ERR_CONFIG,
                     "multi-device contexts run the packed engine (LIFE_ENGINE_PACKED), got %d",
                     engine);
  return LIFE_OK;
}

// Depth of a run: the auto rule on the tallest band, capped by the thinnest
// band (a band feeds its neighbours K rows per pass).
int run_depth(const MultiState* m, int temporal_depth, int* depth, int* il) {
  if (temporal_depth < 0 || temporal_depth > LIFE_MAX_TEMPORAL_DEPTH)
    return set_error(LIFE_ERR_CONFIG, "temporal depth must be in [0, %d], got %d",
                     LIFE_MAX_TEMPORAL_DEPTH, temporal_depth);
  int64_t min_rows = m->H, max_rows = 0;
  for (const Band& b : m->bands) {
    min_rows = std::min(min_rows, b.rows);
    max_rows = std::max(max_rows, b.rows);
  }
  int k = temporal_depth == 0 ? packed_auto_depth(m->W, max_rows) : temporal_depth;
  // Pair / quad layout kernels, chosen as in life_run: forced by
  // LIFE_OPT_PAIR_DEPTH / _QUAD_DEPTH, or the auto rule on the tallest band.
  const IlChoice ch = il_choose(m->W, max_rows, m->pair_depth, m->quad_depth, temporal_depth);
  if (ch.il != 0) k = ch.depth;
  if (nbands(m) > 1) k = static_cast<int>(std::min<int64_t>(k, min_rows));
  *depth = std::max(k, 1);
  *il = ch.il;
  return LIFE_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
int multi_create(int32_t n, const int* devices, MultiState** out) {
  if (n < 1 || !devices) return set_error(LIFE_ERR_CONFIG, "need n >= 1 device ids, got %d", n);
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return set_error(LIFE_ERR_NO_DEVICE, "no CUDA device available (%s)",
                     e == cudaSuccess ? "count 0" : cudaGetErrorString(e));
  for (int i = 0; i < n; ++i)
    if (devices[i] < 0 || devices[i] >= count)
      return set_error(LIFE_ERR_NO_DEVICE, "device %d out of range [0, %d)", devices[i], count);
  MultiState* m = new MultiState();
  m->bands.resize(n);
  auto fail = [&](int rc) {
    multi_destroy(m);
    return rc;
  };
  for (int i = 0; i < n; ++i) {
    Band& b = m->bands[i];
    b.device = devices[i];
    if (cudaSetDevice(b.device) != cudaSuccess) return fail(cuda_fail(cudaGetLastError(), "cudaSetDevice"));
    for (cudaStream_t* s : {&b.main, &b.edge, &b.h2d, &b.d2h}) {
      e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
      if (e != cudaSuccess) return fail(cuda_fail(e, "cudaStreamCreate"));
    }
    for (cudaEvent_t* ev : {&b.ev_int[0], &b.ev_int[1], &b.ev_edge[0], &b.ev_edge[1], &b.ev_up,
                            &b.ev_comp, &b.ev_down}) {
      e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
      if (e != cudaSuccess) return fail(cuda_fail(e, "cudaEventCreate"));
    }
    for (cudaEvent_t* ev : {&b.t0, &b.t1}) {
      e = cudaEventCreate(ev);
      if (e != cudaSuccess) return fail(cuda_fail(e, "cudaEventCreate"));
    }
    const int rc = split_streams_init(&b.split, b.device);
    if (rc != LIFE_OK) return fail(rc);
  }
  // Peer access between neighbouring bands on different GPUs (the edge
  // kernels read the neighbours' rows over NVLink).
  for (int i = 0; i < n && n > 1; ++i) {
    for (int j : {up_of(m, i), down_of(m, i)}) {
      const int a = m->bands[i].device, b = m->bands[j].device;
      if (a == b) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a, b);
      if (can) {
        cudaSetDevice(a);
        e = cudaDeviceEnablePeerAccess(b, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
        } else if (e != cudaSuccess) {
          cudaGetLastError();
          can = 0;
        }
      }
      if (!can) m->peer_ok = false;
    }
  }
  m->halo = m->peer_ok ? LIFE_HALO_PEER : LIFE_HALO_COPY;
  *out = m;
  return LIFE_OK;
}

void multi_destroy(MultiState* m) {
  if (!m) return;
  sync_all(m);
  for (Band& b : m->bands) {
    cudaSetDevice(b.device);
    free_band_buffers(b);
    clear_prof(b);
    for (auto* p : b.batch)
      if (p) cudaFree(p);
    if (b.counts) cudaFree(b.counts);
    if (b.row_hashes) cudaFree(b.row_hashes);
    if (b.scratch) cudaFree(b.scratch);
    for (cudaEvent_t ev : {b.ev_int[0], b.ev_int[1], b.ev_edge[0], b.ev_edge[1], b.ev_up,
                           b.ev_comp, b.ev_down, b.t0, b.t1})
      if (ev) cudaEventDestroy(ev);
    split_streams_destroy(&b.split);
    for (cudaStream_t s : {b.main, b.edge, b.h2d, b.d2h})
      if (s) cudaStreamDestroy(s);
  }
  delete m;
}

int multi_sync(MultiState* m) { return sync_all(m); }

int multi_set_option(MultiState* m, int option, int64_t value) {
  switch (option) {
    case LIFE_OPT_PROFILE:
      m->profile = value != 0;
      return LIFE_OK;
    case LIFE_OPT_HALO:
      if (value != LIFE_HALO_PEER && value != LIFE_HALO_COPY)
        return set_error(LIFE_ERR_CONFIG, "LIFE_OPT_HALO must be LIFE_HALO_PEER or LIFE_HALO_COPY");
      if (value == LIFE_HALO_PEER && !m->peer_ok)
        return set_error(LIFE_ERR_CONFIG, "peer access is unavailable between neighbouring bands");
      LIFE_TRY(sync_all(m));
      m->halo = static_cast<int>(value);
      return LIFE_OK;
    case LIFE_OPT_BATCH_TRAPEZOID:
      return LIFE_OK;  // the multi-device batch has no chunk schedule
    case LIFE_OPT_PAIR_DEPTH:
      if (value < -1 || value > kPairMaxDepthHost)
        return set_error(LIFE_ERR_CONFIG, "LIFE_OPT_PAIR_DEPTH must be in [-1, %d]",
                         kPairMaxDepthHost);
      m->pair_depth = static_cast<int>(value);
      return LIFE_OK;
    case LIFE_OPT_QUAD_DEPTH:
      if (value < -1 || value > kQuadMaxDepthHost)
        return set_error(LIFE_ERR_CONFIG, "LIFE_OPT_QUAD_DEPTH must be in [-1, %d]",
                         kQuadMaxDepthHost);
      m->quad_depth = static_cast<int>(value);
      return LIFE_OK;
    default:
      return set_error(LIFE_ERR_CONFIG, "unknown option %d", option);
  }
}

int multi_get_option(MultiState* m, int option, int64_t* value) {
  switch (option) {
    case LIFE_OPT_PROFILE: *value = m->profile ? 1 : 0; return LIFE_OK;
    case LIFE_OPT_HALO: *value = m->halo; return LIFE_OK;
    case LIFE_OPT_BATCH_TRAPEZOID: *value = 0; return LIFE_OK;
    case LIFE_OPT_PAIR_DEPTH: *value = m->pair_depth; return LIFE_OK;
    case LIFE_OPT_QUAD_DEPTH: *value = m->quad_depth; return LIFE_OK;
    default: return set_error(LIFE_ERR_CONFIG, "unknown option %d", option);
  }
}

int multi_dims(MultiState* m, int64_t* w, int64_t* h) {
  LIFE_TRY(check_loaded(m));
  *w = m->W;
  *h = m->H;
  return LIFE_OK;
}

int multi_bands(MultiState* m, int32_t* n, int64_t* bounds, int32_t* devices, int32_t* halo) {
  const int nb = nbands(m);
  if (n) *n = nb;
  if (bounds) {
    if (m->loaded) {
      for (int i = 0; i < nb; ++i) bounds[i] = m->bands[i].y0;
      bounds[nb] = m->H;
    } else {
      for (int i = 0; i <= nb; ++i) bounds[i] = 0;
    }
  }
  if (devices)
    for (int i = 0; i < nb; ++i) devices[i] = m->bands[i].device;
  if (halo) *halo = m->halo;
  return LIFE_OK;
}

int multi_band_stats(MultiState* m, int32_t band, life_band_stats* out) {
  if (band < 0 || band >= nbands(m))
    return set_error(LIFE_ERR_CONFIG, "band %d out of range [0, %d)", band, nbands(m));
  const Band& b = m->bands[band];
  *out = life_band_stats{};
  out->band = band;
  out->device = b.device;
  out->y0 = b.y0;
  out->rows = b.rows;
  out->passes = b.passes;
  out->run_ms = b.run_ms;
  out->interior_ms = b.interior_ms;
  out->edge_ms = b.edge_ms;
  out->wait_ms = m->profile ? b.run_ms - b.interior_ms : 0.0;
  return LIFE_OK;
}

// ---- grid in / out ---------------------------------------------------------
int multi_upload_packed(MultiState* m, const uint64_t* words, int64_t w, int64_t h, int64_t wpr) {
  if (!words) return set_error(LIFE_ERR_CONFIG, "null word buffer");
  LIFE_TRY(set_dims(m, w, h));
  if (wpr < ceil_div(w, 64)) return set_error(LIFE_ERR_CONFIG, "words_per_row < ceil(W/64)");
  m->cur = 0;
  m->il = 0;
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    LIFE_TRY(copy_band_rows(m, const_cast<uint64_t*>(words) + b.y0 * wpr, wpr, b.buf[0], b.rows,
                            true, b.main));
    LIFE_TRY(launch_mask_tail(b.buf[0], m->pitch, w, b.rows, b.main));
  }
  LIFE_TRY(sync_all(m));
  m->loaded = true;
  return LIFE_OK;
}

int multi_upload_u8(MultiState* m, const uint8_t* cells, int64_t w, int64_t h, int64_t stride) {
  if (!cells) return set_error(LIFE_ERR_CONFIG, "null cell buffer");
  LIFE_TRY(set_dims(m, w, h));
  if (stride < w) return set_error(LIFE_ERR_CONFIG, "row_stride < width");
  const int64_t bp = life_byte_pitch(w);
  const int64_t chunk = std::max<int64_t>(1, kScratchBytes / bp);
  m->cur = 0;
  m->il = 0;
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    LIFE_TRY(ensure_scratch(b, std::min(chunk, b.rows) * bp));
    for (int64_t r = 0; r < b.rows; r += chunk) {
      const int64_t n = std::min(chunk, b.rows - r);
      LIFE_CUDA(cudaMemcpy2DAsync(b.scratch, bp, cells + (b.y0 + r) * stride, stride, w, n,
                                  cudaMemcpyHostToDevice, b.main));
      // pack: any nonzero byte is alive, columns >= W zero
      LIFE_TRY(life_dev_pack(b.scratch, bp, b.buf[0] + r * m->pitch, m->pitch, w, n, b.main));
    }
  }
  LIFE_TRY(sync_all(m));
  m->loaded = true;
  return LIFE_OK;
}

int multi_init_random(MultiState* m, int64_t w, int64_t h, double density, uint64_t seed) {
  if (!(density >= 0.0 && density <= 1.0))
    return set_error(LIFE_ERR_CONFIG, "density must be in [0, 1], got %f", density);
  LIFE_TRY(set_dims(m, w, h));
  m->cur = 0;
  m->il = 0;
  for (Band& b : m->bands) {  // band rows y0.. of random_fill's row-major stream
    LIFE_TRY(use(b));
    LIFE_TRY(life_dev_packed_random(b.buf[0], m->pitch, w, b.y0, b.rows, density, seed, b.main));
  }
  LIFE_TRY(sync_all(m));
  m->loaded = true;
  return LIFE_OK;
}

int multi_init_soup(MultiState* m, int64_t w, int64_t h, double coverage, int32_t bs,
                    double density, uint64_t seed) {
  // The soup's overwrite order is global: generate it whole on the first
  // band's GPU (one context), then distribute the packed rows.
  LIFE_TRY(check_dims(w, h));
  std::vector<int64_t> bounds(m->bands.size() + 1);
  LIFE_TRY(life_band_bounds(h, nbands(m), bounds.data()));
  life_ctx* tmp = nullptr;
  LIFE_TRY(life_ctx_create(m->bands[0].device, &tmp));
  const int64_t wpr = ceil_div(w, 64);
  std::vector<uint64_t> host;
  int rc = life_grid_init_soup(tmp, w, h, coverage, bs, density, seed, LIFE_ENGINE_PACKED);
  if (rc == LIFE_OK) {
    host.resize(static_cast<size_t>(h * wpr));
    rc = life_grid_download_packed(tmp, host.data(), wpr);
  }
  life_ctx_destroy(tmp);
  if (rc != LIFE_OK) return rc;
  return multi_upload_packed(m, host.data(), w, h, wpr);
}

int multi_place_u8(MultiState* m, const uint8_t* pattern, int64_t pw, int64_t ph, int64_t x0,
                   int64_t y0) {
  LIFE_TRY(check_loaded(m));
  LIFE_TRY(to_plain(m));
  if (pw < 0 || ph < 0 || (pw * ph > 0 && !pattern))
    return set_error(LIFE_ERR_CONFIG, "bad pattern buffer");
  if (x0 < 0 || y0 < 0 || x0 + pw > m->W || y0 + ph > m->H)
    return set_error(LIFE_ERR_OUT_OF_BOUNDS,
                     "pattern footprint %lldx%lld at (%lld, %lld) exceeds grid %lldx%lld",
                     static_cast<long long>(pw), static_cast<long long>(ph),
                     static_cast<long long>(x0), static_cast<long long>(y0),
                     static_cast<long long>(m->W), static_cast<long long>(m->H));
  if (pw * ph == 0) return LIFE_OK;
  for (Band& b : m->bands) {  // the pattern rows inside this band
    const int64_t r0 = std::max(y0, b.y0), r1 = std::min(y0 + ph, b.y0 + b.rows);
    if (r0 >= r1) continue;
    LIFE_TRY(use(b));
    const int64_t bytes = (r1 - r0) * pw;
    LIFE_TRY(ensure_scratch(b, bytes));
    LIFE_CUDA(cudaMemcpyAsync(b.scratch, pattern + (r0 - y0) * pw, bytes, cudaMemcpyHostToDevice,
                              b.main));
    LIFE_TRY(launch_place_packed(b.buf[m->cur], m->pitch, b.scratch, pw, r1 - r0, x0, r0 - b.y0,
                                 b.main));
    LIFE_CUDA(cudaStreamSynchronize(b.main));
  }
  return LIFE_OK;
}

int multi_download_packed(MultiState* m, uint64_t* words, int64_t wpr) {
  LIFE_TRY(check_loaded(m));
  LIFE_TRY(to_plain(m));
  if (!words || wpr < ceil_div(m->W, 64)) return set_error(LIFE_ERR_CONFIG, "bad output buffer");
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    LIFE_TRY(copy_band_rows(m, words + b.y0 * wpr, wpr, b.buf[m->cur], b.rows, false, b.main));
  }
  return sync_all(m);
}

int multi_download_u8(MultiState* m, uint8_t* cells, int64_t stride) {
  LIFE_TRY(check_loaded(m));
  LIFE_TRY(to_plain(m));
  if (!cells || stride < m->W) return set_error(LIFE_ERR_CONFIG, "bad output buffer");
  const int64_t bp = life_byte_pitch(m->W);
  const int64_t chunk = std::max<int64_t>(1, kScratchBytes / bp);
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    LIFE_TRY(ensure_scratch(b, std::min(chunk, b.rows) * bp));
    for (int64_t r = 0; r < b.rows; r += chunk) {
      const int64_t n = std::min(chunk, b.rows - r);
      LIFE_TRY(life_dev_unpack(b.buf[m->cur] + r * m->pitch, m->pitch, b.scratch, bp, m->W, n,
                               b.main));
      LIFE_CUDA(cudaMemcpy2DAsync(cells + (b.y0 + r) * stride, stride, b.scratch, bp, m->W, n,
                                  cudaMemcpyDeviceToHost, b.main));
    }
  }
  return sync_all(m);
}

int multi_window_u8(MultiState* m, int64_t x0, int64_t y0, int64_t w, int64_t h, uint8_t* out) {
  LIFE_TRY(check_loaded(m));
  LIFE_TRY(to_plain(m));
  if (w < 0 || h < 0 || !out) return set_error(LIFE_ERR_CONFIG, "bad window");
  if (w * h == 0) return LIFE_OK;
  // Window rows j map to torus row (y0 + j) mod H; cut them into runs that
  // stay inside one band (no wrap inside a run).
  int64_t j = 0;
  while (j < h) {
    int64_t y = (y0 + j) % m->H;
    if (y < 0) y += m->H;
    int bi = 0;
    while (bi + 1 < nbands(m) && m->bands[bi + 1].y0 <= y) ++bi;
    Band& b = m->bands[bi];
    const int64_t run = std::min(h - j, b.y0 + b.rows - y);
    LIFE_TRY(use(b));
    LIFE_TRY(ensure_scratch(b, run * w));
    LIFE_TRY(launch_window_packed(b.buf[m->cur], m->pitch, m->W, b.rows, x0, y - b.y0, w, run,
                                  b.scratch, b.main));
    LIFE_CUDA(cudaMemcpyAsync(out + j * w, b.scratch, run * w, cudaMemcpyDeviceToHost, b.main));
    LIFE_CUDA(cudaStreamSynchronize(b.main));
    j += run;
  }
  return LIFE_OK;
}

int multi_population(MultiState* m, uint64_t* out) {
  LIFE_TRY(check_loaded(m));
  if (!out) return set_error(LIFE_ERR_CONFIG, "null output pointer");
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    LIFE_TRY(ensure_counts(b, 1));
    LIFE_CUDA(cudaMemsetAsync(b.counts, 0, sizeof(unsigned long long), b.main));
    LIFE_TRY(life_dev_packed_population(b.buf[m->cur], m->pitch, m->W, b.rows,
                                        reinterpret_cast<uint64_t*>(b.counts), b.main));
  }
  uint64_t total = 0;
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    uint64_t v = 0;
    LIFE_CUDA(cudaMemcpyAsync(&v, b.counts, 8, cudaMemcpyDeviceToHost, b.main));
    LIFE_CUDA(cudaStreamSynchronize(b.main));
    total += v;
  }
  *out = total;
  return LIFE_OK;
}

int multi_hash(MultiState* m, uint64_t* out) {
  LIFE_TRY(check_loaded(m));
  LIFE_TRY(to_plain(m));
  if (!out) return set_error(LIFE_ERR_CONFIG, "null output pointer");
  std::vector<uint64_t> rows(static_cast<size_t>(m->H));
  for (Band& b : m->bands) {  // row hashes of the bands, concatenated in row order
    LIFE_TRY(use(b));
    if (b.rows > b.row_hashes_cap) {
      if (b.row_hashes) cudaFree(b.row_hashes);
      b.row_hashes = nullptr;
      LIFE_CUDA(cudaMalloc(&b.row_hashes, sizeof(uint64_t) * b.rows));
      b.row_hashes_cap = b.rows;
    }
    LIFE_TRY(life_dev_packed_row_hashes(b.buf[m->cur], m->pitch, m->W, b.rows, b.row_hashes,
                                        b.main));
    LIFE_CUDA(cudaMemcpyAsync(rows.data() + b.y0, b.row_hashes, sizeof(uint64_t) * b.rows,
                              cudaMemcpyDeviceToHost, b.main));
  }
  LIFE_TRY(sync_all(m));
  *out = life_fnv1a64(rows.data(), static_cast<int64_t>(rows.size() * sizeof(uint64_t)), 0);
  return LIFE_OK;
}

// ---- the step loop ---------------------------------------------------------
int multi_run(MultiState* m, int64_t generations, int engine, int temporal_depth,
              const int64_t* checkpoints, int32_t n_checkpoints, uint64_t* populations) {
  LIFE_TRY(check_packed_engine(engine));
  LIFE_TRY(check_run_args(generations, checkpoints, n_checkpoints, populations));
  LIFE_TRY(check_loaded(m));
  int depth = 0;
  int il = 0;
  LIFE_TRY(run_depth(m, temporal_depth, &depth, &il));
  if (generations > 0) LIFE_TRY(il != 0 ? to_il(m, il) : to_plain(m));
  if (m->halo == LIFE_HALO_COPY) LIFE_TRY(ensure_ghosts(m));
  const int n = nbands(m);
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    if (n_checkpoints > 0) {
      LIFE_TRY(ensure_counts(b, n_checkpoints));
      LIFE_CUDA(cudaMemsetAsync(b.counts, 0, sizeof(unsigned long long) * n_checkpoints, b.main));
    }
    clear_prof(b);
    b.passes = 0;
  }
  int32_t ci = 0;
  auto record = [&](int64_t gen) -> int {
    while (ci < n_checkpoints && checkpoints[ci] == gen) {
      for (Band& b : m->bands) {  // band populations, summed on the host (engine.cpp:179-186)
        LIFE_TRY(use(b));
        LIFE_TRY(life_dev_packed_population(b.buf[m->cur], m->pitch, m->W, b.rows,
                                            reinterpret_cast<uint64_t*>(b.counts + ci), b.main));
      }
      ++ci;
    }
    return LIFE_OK;
  };
  LIFE_TRY(record(0));
  LIFE_TRY(mark_start(m));
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    LIFE_CUDA(cudaEventRecord(b.t0, b.main));
  }
  std::vector<uint32_t*> src(n), dst(n);
  int64_t done = 0, p = 0;
  int kprev = 0;
  while (done < generations) {
    const int64_t stop = ci < n_checkpoints ? checkpoints[ci] : generations;
    const int k = static_cast<int>(std::min<int64_t>(depth, stop - done));
    for (int i = 0; i < n; ++i) {
      src[i] = m->bands[i].buf[m->cur];
      dst[i] = m->bands[i].buf[m->cur ^ 1];
    }
    LIFE_TRY(issue_pass(m, src.data(), dst.data(), p, k, kprev, m->il));
    m->cur ^= 1;
    done += k;
    kprev = k;
    if (ci < n_checkpoints && checkpoints[ci] == done) {
      LIFE_TRY(join_pass(m, p));
      LIFE_TRY(record(done));
    }
    ++p;
  }
  if (p > 0) LIFE_TRY(join_pass(m, p - 1));
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    LIFE_CUDA(cudaEventRecord(b.t1, b.main));
  }
  LIFE_TRY(sync_all(m));
  std::vector<uint64_t> total(static_cast<size_t>(n_checkpoints), 0);
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    float ms = 0.0f;
    LIFE_CUDA(cudaEventElapsedTime(&ms, b.t0, b.t1));
    b.run_ms = ms;
    LIFE_TRY(sum_pairs(b.prof_int, &b.interior_ms));
    LIFE_TRY(sum_pairs(b.prof_edge, &b.edge_ms));
    if (n_checkpoints > 0) {
      std::vector<uint64_t> v(static_cast<size_t>(n_checkpoints));
      LIFE_CUDA(cudaMemcpy(v.data(), b.counts, sizeof(uint64_t) * n_checkpoints,
                           cudaMemcpyDeviceToHost));
      for (int32_t i = 0; i < n_checkpoints; ++i) total[i] += v[i];
    }
  }
  for (int32_t i = 0; i < n_checkpoints; ++i) populations[i] = total[i];
  return LIFE_OK;
}

// Throughput form over a stream of packed host grids: each band uploads its
// rows of grid i into one of two slots on its own copy stream while grid i-1
// computes, and downloads them while grid i+1 computes.  Grid i+2's upload
// into a slot waits for the band's download of grid i AND for the
// neighbouring bands' last pass of grid i (whose edges read this band's rows).
int multi_run_batch(MultiState* m, const uint64_t* const* inputs, uint64_t* const* outputs,
                    int32_t n, int64_t width, int64_t height, int64_t words_per_row,
                    int64_t generations, int temporal_depth, float* elapsed_ms) {
  if (n < 0 || (n > 0 && (!inputs || !outputs)))
    return set_error(LIFE_ERR_CONFIG, "bad batch buffers");
  if (generations < 0)
    return set_error(LIFE_ERR_CONFIG, "iteration count must be non-negative, got %lld",
                     static_cast<long long>(generations));
  if (words_per_row < ceil_div(width, 64))
    return set_error(LIFE_ERR_CONFIG, "words_per_row < ceil(W/64)");
  LIFE_TRY(set_dims(m, width, height));  // band layout (the resident grid is not used)
  int depth = 0;
  int il = 0;
  LIFE_TRY(run_depth(m, temporal_depth, &depth, &il));
  if (generations == 0) il = 0;
  if (n == 0) return LIFE_OK;
  if (m->halo == LIFE_HALO_COPY) LIFE_TRY(ensure_ghosts(m));
  const int nb = nbands(m);
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    const size_t bytes = static_cast<size_t>(b.rows) * m->pitch * 4;
    if (b.batch_bytes != bytes) {
      for (auto& p : b.batch) {
        if (p) cudaFree(p);
        p = nullptr;
      }
      b.batch_bytes = 0;
      for (auto& p : b.batch) {
        LIFE_CUDA(cudaMalloc(&p, bytes));
        LIFE_CUDA(cudaMemsetAsync(p, 0, bytes, b.main));
      }
      b.batch_bytes = bytes;
    }
    clear_prof(b);
    b.passes = 0;
  }
  LIFE_TRY(sync_all(m));
  // Per band and grid: upload / compute / download events.
  struct Events {
    std::vector<cudaEvent_t> v;
    ~Events() {
      for (cudaEvent_t e : v) cudaEventDestroy(e);
    }
  } evs;
  auto mk = [&](int dev) -> cudaEvent_t {
    cudaEvent_t e = nullptr;
    cudaSetDevice(dev);
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    evs.v.push_back(e);
    return e;
  };
  std::vector<std::vector<cudaEvent_t>> up(nb), comp(nb), down(nb);
  for (int b = 0; b < nb; ++b) {
    for (int32_t i = 0; i < n; ++i) {
      up[b].push_back(mk(m->bands[b].device));
      comp[b].push_back(mk(m->bands[b].device));
      down[b].push_back(mk(m->bands[b].device));
      if (!up[b].back() || !comp[b].back() || !down[b].back())
        return cuda_fail(cudaGetLastError(), "cudaEventCreate");
    }
  }
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    LIFE_CUDA(cudaEventRecord(b.t0, b.h2d));
  }
  const int passes = static_cast<int>(ceil_div(generations, depth));
  std::vector<uint32_t*> src(nb), dst(nb);
  int64_t p_global = 0;
  for (int32_t i = 0; i < n; ++i) {
    const int slot = i & 1;
    for (int b = 0; b < nb; ++b) {
      Band& bd = m->bands[b];
      LIFE_TRY(use(bd));
      if (i >= 2) {
        LIFE_CUDA(cudaStreamWaitEvent(bd.h2d, down[b][i - 2], 0));
        LIFE_CUDA(cudaStreamWaitEvent(bd.h2d, comp[up_of(m, b)][i - 2], 0));
        LIFE_CUDA(cudaStreamWaitEvent(bd.h2d, comp[down_of(m, b)][i - 2], 0));
      }
      LIFE_TRY(copy_band_rows(m, const_cast<uint64_t*>(inputs[i]) + bd.y0 * words_per_row,
                              words_per_row, bd.batch[2 * slot], bd.rows, true, bd.h2d));
      LIFE_TRY(launch_mask_tail(bd.batch[2 * slot], m->pitch, width, bd.rows, bd.h2d));
      if (il != 0)  // the band's rows into the pair / quad layout, behind their copy
        LIFE_TRY(packed_zip(il, bd.batch[2 * slot], m->pitch, width, 0, bd.rows, /*unzip=*/false,
                            bd.h2d));
      LIFE_CUDA(cudaEventRecord(up[b][i], bd.h2d));
    }
    // Every band's compute and edge streams start grid i once the band and
    // its neighbours have their rows.
    for (int b = 0; b < nb; ++b) {
      Band& bd = m->bands[b];
      LIFE_TRY(use(bd));
      for (int j : {b, up_of(m, b), down_of(m, b)}) {
        LIFE_CUDA(cudaStreamWaitEvent(bd.main, up[j][i], 0));
        LIFE_CUDA(cudaStreamWaitEvent(bd.edge, up[j][i], 0));
      }
    }
    LIFE_TRY(mark_start(m));
    p_global = 0;
    int kprev = 0;
    for (int p = 0; p < passes; ++p) {
      const int k = static_cast<int>(std::min<int64_t>(depth, generations - int64_t(p) * depth));
      for (int b = 0; b < nb; ++b) {
        src[b] = m->bands[b].batch[2 * slot + (p & 1)];
        dst[b] = m->bands[b].batch[2 * slot + ((p & 1) ^ 1)];
      }
      LIFE_TRY(issue_pass(m, src.data(), dst.data(), p_global, k, kprev, il));
      kprev = k;
      ++p_global;
    }
    if (passes > 0) LIFE_TRY(join_pass(m, p_global - 1));
    for (int b = 0; b < nb; ++b) {
      Band& bd = m->bands[b];
      LIFE_TRY(use(bd));
      LIFE_CUDA(cudaEventRecord(comp[b][i], bd.main));
      LIFE_CUDA(cudaStreamWaitEvent(bd.d2h, comp[b][i], 0));
      if (il != 0)  // back to the plain layout (only this band's kernels wrote the result buffer)
        LIFE_TRY(packed_zip(il, bd.batch[2 * slot + (passes & 1)], m->pitch, width, 0, bd.rows,
                            /*unzip=*/true, bd.d2h));
      LIFE_TRY(copy_band_rows(m, outputs[i] + bd.y0 * words_per_row, words_per_row,
                              bd.batch[2 * slot + (passes & 1)], bd.rows, false, bd.d2h));
      LIFE_CUDA(cudaEventRecord(down[b][i], bd.d2h));
    }
  }
  float worst = 0.0f;
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    LIFE_CUDA(cudaEventRecord(b.t1, b.d2h));
  }
  LIFE_TRY(sync_all(m));
  for (Band& b : m->bands) {
    LIFE_TRY(use(b));
    float ms = 0.0f;
    LIFE_CUDA(cudaEventElapsedTime(&ms, b.t0, b.t1));
    worst = std::max(worst, ms);
  }
  if (elapsed_ms) *elapsed_ms = worst;  // max over bands (devices)
  return LIFE_OK;
}

}  // namespace detail
}  // namespace lifegpu
