"""Row-band decomposition of the torus across GPUs (one process per GPU).

Mirrors the reference's preferred 1-D row decomposition: Strategy::rows()
-> partition_rows -> band_bounds (decomposition.cpp:12-24, :93-104; the
paper's conclusion).  Rank r owns rows
[bounds[r], bounds[r+1]) and keeps `depth` ghost rows above and below its
band.  One temporal-blocked pass of k <= depth generations is

    1. post the halo exchange (NCCL send/recv over NVLink via
       torch.distributed): my top k rows -> the rank above (its bottom
       ghosts), my bottom k rows -> the rank below (its top ghosts);
    2. compute the interior output rows [k, band-k), which depend only on
       local rows, while the halos are in flight;
    3. wait for the halos;
    4. compute the two k-row edge strips.

This replaces the reference's per-generation shared-memory barrier
(WorkerTeam, engine.cpp:60-125) with one exchange per k generations.  With a
single rank the band is the whole torus and the kernel wraps rows itself
(no ghosts, no exchange).

The compute and the buffers are injectable so the same driver runs
(a) on GPUs with the CUDA kernels of the C-ABI and NCCL, and (b) in the
world-size-2 gloo tests on CPU with a test-only stepper.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import torch
import torch.distributed as dist

from . import capi
from .life import ConfigError, TooManyParts, band_bounds, check


def run_schedule(drv, generations: int, checkpoints: Sequence[int] = (),
                 on_pass: Optional[Callable[[int], None]] = None) -> list[int]:
    """The pass loop of run() (engine.cpp:162-214) for a band driver: passes
    of up to `depth` generations, split at the checkpoints, whose uint64
    populations (summed over every rank's band, engine.cpp:179-186; checkpoint
    0 = the initial grid) are returned in order.  check_run_config's rules
    (engine.cpp:127-148) on generations and checkpoints."""
    if generations < 0:
        raise ConfigError(f"iteration count must be non-negative, got {generations}")
    cps = [int(c) for c in checkpoints]
    prev = -1
    for c in cps:
        if c < 0 or c > generations:
            raise ConfigError(f"checkpoint {c} is outside [0, iterations={generations}]")
        if c <= prev:
            raise ConfigError("checkpoints must be strictly ascending")
        prev = c
    pops: list[int] = []
    ci = 0

    def record(gen: int) -> None:
        nonlocal ci
        while ci < len(cps) and cps[ci] == gen:
            pops.append(drv.population())
            ci += 1
    record(0)
    depth = drv.geo.depth
    done = 0
    while done < generations:
        stop = cps[ci] if ci < len(cps) else generations
        k = min(depth, stop - done)
        drv.pass_(k)
        done += k
        if on_pass:
            on_pass(k)
        record(done)
    return pops


@dataclass
class BandGeometry:
    width: int
    height: int
    rank: int
    world: int
    depth: int
    y0: int
    y1: int
    pitch: int  # uint32 words per row
    # Interleave order of the passes' layout (kernels_pair.cuh): 0 = plain,
    # 2 = pair (W % 64 == 0, depth <= 12), 4 = quad (W % 128 == 0, depth <= 6).
    # The drivers convert their band in place before the first pass and back
    # before anything reads the plain words.
    il: int = 0
    # world == 1 only: run the halo exchange anyway, the rank being its own
    # neighbour above and below (the torus wrap as a self send / receive).
    # This is how the NCCL halo path runs on a single GPU (tests).
    self_exchange: bool = False

    @property
    def band_rows(self) -> int:
        return self.y1 - self.y0

    @property
    def exchanges(self) -> bool:
        return self.world > 1 or self.self_exchange

    @property
    def ghost(self) -> int:
        return self.depth if self.exchanges else 0

    @property
    def buf_rows(self) -> int:
        return self.band_rows + 2 * self.ghost


def il_max_depth(il: int) -> int:
    return {0: capi.MAX_TEMPORAL_DEPTH, 2: capi.PAIR_MAX_DEPTH, 4: capi.QUAD_MAX_DEPTH}[il]


def make_geometry(width: int, height: int, rank: int, world: int, depth: int,
                  il: int = 0, self_exchange: bool = False) -> BandGeometry:
    if width < 3 or height < 3:
        raise ConfigError(f"grid dimensions must be at least 3x3, got {width}x{height}")
    if not 1 <= depth <= capi.MAX_TEMPORAL_DEPTH:
        raise ConfigError(f"temporal depth must be in [1, {capi.MAX_TEMPORAL_DEPTH}]")
    if il not in (0, 2, 4):
        raise ConfigError(f"interleave order must be 0 (plain), 2 (pair) or 4 (quad), got {il}")
    if il and (width % (32 * il) != 0 or depth > il_max_depth(il)):
        raise ConfigError(f"interleave order {il} needs W % {32 * il} == 0 and depth <= "
                          f"{il_max_depth(il)}, got W = {width}, depth {depth}")
    bounds = band_bounds(height, world)  # TooManyParts like partition_rows
    y0, y1 = bounds[rank], bounds[rank + 1]
    if (world > 1 or self_exchange) and (y1 - y0) < depth:
        raise TooManyParts(f"band of {y1 - y0} rows is thinner than the temporal depth {depth}")
    if self_exchange and world != 1:
        raise ConfigError("self_exchange is the one-rank form of the halo exchange")
    return BandGeometry(width, height, rank, world, depth, y0, y1,
                        int(capi.lib().life_packed_pitch_words(width)), il, self_exchange)


class PairLayout:
    """Mixin of the band drivers: which layout the current band is in.  A
    driver names its band rows with _band_raw() (a view of `band_rows` rows of
    `pitch` words); passes call _to_pair() first when the geometry asks for
    the pair / quad kernel (geo.il), readers of the plain layout call
    _to_plain()."""

    in_pair = False  # the band is in the geometry's interleaved layout

    def _zip(self, to_pair: bool) -> None:
        g = self.geo
        raw = self._band_raw()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        check(capi.lib().life_dev_packed_zip(raw.data_ptr(), g.pitch, g.width, 0, g.band_rows,
                                             g.il, 1 if to_pair else 0, stream))

    def set_band(self, rows: torch.Tensor) -> None:
        """Overwrites the band with `rows` (plain packed layout)."""
        self.in_pair = False
        self._band_raw().copy_(rows)

    def _to_pair(self) -> None:
        if self.geo.il and not self.in_pair:
            self._zip(True)
            self.in_pair = True

    def _to_plain(self) -> None:
        if self.in_pair:
            self._zip(False)
            self.in_pair = False


# Stepper(in, in_row0, in_rows, out, out_row0, out_rows, k): one k-generation
# pass with the addressing of life_dev_packed_step.
Stepper = Callable[[torch.Tensor, int, int, torch.Tensor, int, int, int], None]


def cuda_stepper(width: int, il: int = 0) -> Stepper:
    L = capi.lib()

    def step(inp, in_row0, in_rows, out, out_row0, out_rows, k):
        pitch = inp.shape[1]
        stream = torch.cuda.current_stream(inp.device).cuda_stream
        args = (inp.data_ptr(), pitch, in_row0, in_rows, out.data_ptr(), out.shape[1], out_row0,
                width, out_rows, k, stream)
        check(L.life_dev_packed_step_il(il, *args) if il else L.life_dev_packed_step(*args))
    return step


class BandDriver(PairLayout):
    """One rank's band, ping-pong buffers and pass loop."""

    def __init__(self, geo: BandGeometry, device: torch.device, stepper: Optional[Stepper] = None,
                 group=None, overlap: bool = True,
                 counter: Optional[Callable[[torch.Tensor], int]] = None):
        self.geo = geo
        self.device = device
        self.group = group
        self.overlap = overlap
        if geo.il and stepper is not None:
            raise ConfigError("the interleaved layouts run on the CUDA stepper")
        self.stepper = stepper or cuda_stepper(geo.width, geo.il)
        self.counter = counter  # test hook: band rows -> live cells (default: CUDA popcount)
        shape = (geo.buf_rows, geo.pitch)
        self.buf = [torch.zeros(shape, dtype=torch.int32, device=device) for _ in range(2)]
        # CUDA: the k-row edge strips run on a side stream as soon as the
        # halos land, filling SMs between the interior kernel's block waves.
        self.edge_stream = torch.cuda.Stream(device) if device.type == "cuda" else None
        self.cur = 0
        self.generations = 0
        self.exchange_bytes = 0  # per pass, both directions, this rank

    # -- views ---------------------------------------------------------
    def _band_raw(self) -> torch.Tensor:
        return self.buf[self.cur][self.geo.ghost:self.geo.ghost + self.geo.band_rows]

    def band(self, which: Optional[int] = None) -> torch.Tensor:
        """This rank's band rows in the plain packed layout."""
        if which is None or which == self.cur:
            self._to_plain()
        b = self.buf[self.cur if which is None else which]
        return b[self.geo.ghost:self.geo.ghost + self.geo.band_rows]

    # -- halo exchange -------------------------------------------------
    def _peers(self) -> tuple[int, int]:
        r, p = self.geo.rank, self.geo.world
        return (r - 1) % p, (r + 1) % p  # above, below (torus ring)

    def halo_views(self, k: int):
        """(top rows, bottom rows, top ghost rows, bottom ghost rows) of the
        current buffer for a depth-k pass."""
        g = self.geo
        a = self.buf[self.cur]
        top = a[g.ghost:g.ghost + k]
        bottom = a[g.ghost + g.band_rows - k:g.ghost + g.band_rows]
        ghost_top = a[g.ghost - k:g.ghost]
        ghost_bottom = a[g.ghost + g.band_rows:g.ghost + g.band_rows + k]
        return top, bottom, ghost_top, ghost_bottom

    def post_exchange(self, k: int):
        """Sends my top/bottom k rows, receives k ghost rows on each side."""
        g = self.geo
        if not g.exchanges:
            return None
        up, down = self._peers()
        top, bottom, ghost_top, ghost_bottom = self.halo_views(k)
        # Same issue order on every rank: per peer pair, the i-th send
        # matches the i-th receive (needed when up == down, world == 2).
        ops = [dist.P2POp(dist.isend, top, up, self.group),
               dist.P2POp(dist.isend, bottom, down, self.group),
               dist.P2POp(dist.irecv, ghost_bottom, down, self.group),
               dist.P2POp(dist.irecv, ghost_top, up, self.group)]
        self.exchange_bytes = 2 * top.numel() * 4
        return dist.batch_isend_irecv(ops)

    @staticmethod
    def wait(works) -> None:
        if works:
            for w in works:
                w.wait()

    # -- one pass ------------------------------------------------------
    def compute_interior(self, k: int) -> bool:
        """Output rows [k, band-k): local rows only.  Returns False when the
        band is too thin to split (compute_all must then run after the halos)."""
        g = self.geo
        n = g.band_rows
        if not (self.overlap and n > 2 * k):
            return False
        a, b = self.buf[self.cur], self.buf[self.cur ^ 1]
        self.stepper(a, g.ghost + k, g.buf_rows, b, g.ghost + k, n - 2 * k, k)
        return True

    def compute_edges(self, k: int, interior_done: bool) -> None:
        """The two k-row edge strips (or the whole band), after the halos."""
        g = self.geo
        n = g.band_rows
        a, b = self.buf[self.cur], self.buf[self.cur ^ 1]
        if interior_done:
            self.stepper(a, g.ghost, g.buf_rows, b, g.ghost, k, k)
            self.stepper(a, g.ghost + n - k, g.buf_rows, b, g.ghost + n - k, k, k)
        else:
            self.stepper(a, g.ghost, g.buf_rows, b, g.ghost, n, k)

    def finish_pass(self, k: int) -> None:
        self.cur ^= 1
        self.generations += k

    def pass_(self, k: int) -> None:
        g = self.geo
        if not 1 <= k <= g.depth:
            raise ConfigError(f"pass depth {k} outside [1, {g.depth}]")
        self._to_pair()
        if not g.exchanges:
            a, b = self.buf[self.cur], self.buf[self.cur ^ 1]
            self.stepper(a, 0, g.height, b, 0, g.height, k)
        elif self.edge_stream is None:
            works = self.post_exchange(k)
            interior = self.compute_interior(k)
            self.wait(works)
            self.compute_edges(k, interior)
        else:
            main = torch.cuda.current_stream(self.device)
            start = torch.cuda.Event()
            start.record(main)
            works = self.post_exchange(k)  # NCCL waits for `main` (last pass done)
            interior = self.compute_interior(k)
            with torch.cuda.stream(self.edge_stream):
                self.edge_stream.wait_event(start)
                self.wait(works)  # edge stream waits for the halos
                self.compute_edges(k, interior)
                done = torch.cuda.Event()
                done.record(self.edge_stream)
            main.wait_event(done)
        self.finish_pass(k)

    def run(self, generations: int, on_pass: Optional[Callable[[int], None]] = None,
            checkpoints: Sequence[int] = ()) -> list[int]:
        """`generations` in passes of up to `depth`; populations at the
        checkpoints (summed over ranks), see run_schedule."""
        return run_schedule(self, generations, checkpoints, on_pass)

    # -- init / reductions (CUDA) ----------------------------------------
    def init_random(self, density: float, seed: int) -> None:
        g = self.geo
        self.in_pair = False  # overwritten whole, in the plain layout
        band = self.band()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        check(capi.lib().life_dev_packed_random(band.data_ptr(), g.pitch, g.width, g.y0,
                                                g.band_rows, density, seed, stream))
        self.generations = 0

    def load_rows(self, words) -> None:
        """Loads this band's rows [y0, y1) from a host packed grid (numpy
        uint64 rows of ceil(W/64) words, the include/life_gpu.h exchange format)."""
        g = self.geo
        rows = words[g.y0:g.y1]
        src = torch.from_numpy(rows.view("int32").copy())
        self.in_pair = False
        self.band()[:, :src.shape[1]].copy_(src)
        self.generations = 0

    def population(self) -> int:
        """Band population (CUDA popcount, or the injected `counter`), summed
        over ranks when distributed (uint64 semantics; grid.cpp:40-46)."""
        g = self.geo
        if self.counter is not None:
            acc = torch.tensor([int(self.counter(self.band()))], dtype=torch.int64)
        else:  # a popcount: the same in either layout
            acc = torch.zeros(1, dtype=torch.int64, device=self.device)
            stream = torch.cuda.current_stream(self.device).cuda_stream
            check(capi.lib().life_dev_packed_population(self._band_raw().data_ptr(), g.pitch,
                                                        g.width, g.band_rows, acc.data_ptr(),
                                                        stream))
        if g.world > 1:
            dist.all_reduce(acc, group=self.group)
        return int(acc.item())


class TorusDriver(PairLayout):
    """The single-GPU case of the band drivers (one band = the whole torus,
    no halo): run() is ONE life_dev_packed_run call (the full-depth passes,
    then the remainder).  `on_launch(kind, generations, fn)` (optional)
    splits it into the full-pass call and the remainder call and wraps each,
    so a profiler can put events around them."""

    def __init__(self, geo: BandGeometry, device: torch.device):
        if geo.world != 1:
            raise ConfigError("TorusDriver is the one-band case")
        self.geo = geo
        self.device = device
        shape = (geo.height, geo.pitch)
        self.buf = [torch.zeros(shape, dtype=torch.int32, device=device) for _ in range(2)]
        self.cur = 0
        self.generations = 0
        self.on_launch = None

    def _band_raw(self) -> torch.Tensor:
        return self.buf[self.cur]

    def band(self) -> torch.Tensor:
        """The torus in the plain packed layout."""
        self._to_plain()
        return self.buf[self.cur]

    def _call(self, gens: int) -> None:
        import ctypes as C
        g = self.geo
        self._to_pair()
        a, b = self.buf[self.cur], self.buf[self.cur ^ 1]
        flip = C.c_int32(0)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        L = capi.lib()
        args = (a.data_ptr(), b.data_ptr(), g.pitch, g.width, g.height, gens, g.depth,
                C.byref(flip), stream)
        check(L.life_dev_packed_run_il(g.il, *args) if g.il else L.life_dev_packed_run(*args))
        self.cur ^= flip.value
        self.generations += gens

    def pass_(self, k: int) -> None:
        g = self.geo
        self._to_pair()
        a, b = self.buf[self.cur], self.buf[self.cur ^ 1]
        stream = torch.cuda.current_stream(self.device).cuda_stream
        L = capi.lib()
        args = (a.data_ptr(), g.pitch, 0, g.height, b.data_ptr(), g.pitch, 0, g.width, g.height,
                k, stream)
        check(L.life_dev_packed_step_il(g.il, *args) if g.il else L.life_dev_packed_step(*args))
        self.cur ^= 1
        self.generations += k

    def run(self, generations: int, checkpoints: Sequence[int] = ()) -> list[int]:
        if checkpoints:
            return run_schedule(self, generations, checkpoints)
        if generations < 0:
            raise ConfigError(f"iteration count must be non-negative, got {generations}")
        k = self.geo.depth
        if self.on_launch is None:
            self._call(generations)
            return []
        full = generations // k * k
        if full:
            self.on_launch("full", full, lambda: self._call(full))
        if generations - full:
            self.on_launch("rem", generations - full, lambda: self._call(generations - full))
        return []

    def init_random(self, density: float, seed: int) -> None:
        g = self.geo
        self.in_pair = False
        stream = torch.cuda.current_stream(self.device).cuda_stream
        check(capi.lib().life_dev_packed_random(self.band().data_ptr(), g.pitch, g.width, 0,
                                                g.height, density, seed, stream))
        self.generations = 0

    def load_rows(self, words) -> None:
        src = torch.from_numpy(words.view("int32").copy())
        self.in_pair = False
        self.band()[:, :src.shape[1]].copy_(src)
        self.generations = 0

    def population(self) -> int:
        g = self.geo
        acc = torch.zeros(1, dtype=torch.int64, device=self.device)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        check(capi.lib().life_dev_packed_population(self._band_raw().data_ptr(), g.pitch, g.width,
                                                    g.height, acc.data_ptr(), stream))
        return int(acc.item())


class LocalBands:
    """P row bands of one torus on ONE device, halos exchanged by device
    copies instead of NCCL: exercises the band seams, ghost addressing and
    interior/edge split of BandDriver with the real kernels on a single GPU
    (no rank ever waits on another)."""

    def __init__(self, width: int, height: int, parts: int, depth: int, device: torch.device,
                 overlap: bool = True, il: int = 0):
        self.drivers = [BandDriver(make_geometry(width, height, r, parts, depth, il), device,
                                   overlap=overlap) for r in range(parts)]

    def init_random(self, density: float, seed: int) -> None:
        for d in self.drivers:
            d.init_random(density, seed)

    def pass_(self, k: int) -> None:
        ds = self.drivers
        p = len(ds)
        if p == 1:
            ds[0].pass_(k)
            return
        for d in ds:
            d._to_pair()
        views = [d.halo_views(k) for d in ds]
        done = [d.compute_interior(k) for d in ds]
        for r in range(p):
            up, down = (r - 1) % p, (r + 1) % p
            views[r][2].copy_(views[up][1])    # my top ghosts <- bottom rows of the band above
            views[r][3].copy_(views[down][0])  # my bottom ghosts <- top rows of the band below
        for d, i in zip(ds, done):
            d.compute_edges(k, i)
        for d in ds:
            d.finish_pass(k)

    def run(self, generations: int) -> None:
        depth = self.drivers[0].geo.depth
        done = 0
        while done < generations:
            k = min(depth, generations - done)
            self.pass_(k)
            done += k

    def gather(self) -> torch.Tensor:
        """The whole torus as packed uint32 rows (device)."""
        return torch.cat([d.band() for d in self.drivers], dim=0)


# ---------------------------------------------------------------------------
# Fused halo over NVLink: the pass kernel reads the neighbour bands' rows
# straight from their HBM (CUDA IPC peer mappings), so a pass is ONE launch
# per GPU and there is no separate exchange step.  Between passes a band only
# has to wait for its two NEIGHBOURS (the rows it reads next pass are theirs,
# and the buffer it overwrites next pass is the one they read this pass):
# a stream-ordered NCCL send/recv of a 4-byte token with the band above and
# the band below, no global collective.
# ---------------------------------------------------------------------------
class DeviceBuffer:
    """cudaMalloc'd packed rows (IPC-shareable), exposed to torch zero-copy."""

    def __init__(self, rows: int, pitch: int, device: torch.device):
        import ctypes as C
        self.rows, self.pitch, self.device = rows, pitch, device
        self.ptr = C.c_void_p()
        with torch.cuda.device(device):
            check(capi.lib().life_dev_alloc(rows * pitch * 4, C.byref(self.ptr)))
        self.tensor = torch.as_tensor(_CudaArray(self.ptr.value, (rows, pitch), device),
                                      device=device)

    def handle(self) -> bytes:
        import ctypes as C
        h = (C.c_ubyte * 64)()
        check(capi.lib().life_ipc_get_handle(self.ptr, h))
        return bytes(h)

    def free(self) -> None:
        if self.ptr:
            capi.lib().life_dev_free(self.ptr)
            self.ptr = None


class _CudaArray:
    """Minimal __cuda_array_interface__ view so torch can wrap a raw pointer."""

    def __init__(self, ptr: int, shape, device: torch.device):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<i4",
                                         "data": (ptr, False), "version": 3, "strides": None}


def open_peer(handle: bytes) -> int:
    import ctypes as C
    buf = (C.c_ubyte * 64).from_buffer_copy(handle)
    out = C.c_void_p()
    check(capi.lib().life_ipc_open(buf, C.byref(out)))
    return out.value


def peer_pass(width: int, src: int, up: int, up_rows: int, down: int, down_rows: int,
              pitch: int, band_rows: int, dst: int, k: int, device: torch.device,
              edge_stream: Optional["torch.cuda.Stream"] = None,
              interior_done: Optional["torch.cuda.Event"] = None, il: int = 0,
              before_edges: Optional[Callable[[], None]] = None) -> None:
    """One depth-k pass of a band with in-kernel NVLink halos: the interior
    rows [k, band-k) read only the band's own rows (the branch-free kernel
    path); the two k-row edge strips read the neighbours' rows through peer
    pointers and run on `edge_stream` (if given) beside the interior.
    `il` 2 / 4: every buffer is in the pair / quad layout (packed_il_kernel).
    `before_edges` (needs `edge_stream`, band taller than 2k): called with the
    edge stream current, after it has joined the compute stream and before the
    edge strips -- where the overlapped pass sync waits for the neighbours."""
    L = capi.lib()

    def step(*args):
        return L.life_dev_packed_step_il(il, *args) if il else L.life_dev_packed_step(*args)

    def step_peer(*args):
        return (L.life_dev_packed_step_il_peer(il, *args) if il
                else L.life_dev_packed_step_peer(*args))
    main = torch.cuda.current_stream(device)
    if band_rows <= 2 * k:
        check(step_peer(src, up, up_rows, down, down_rows, pitch, band_rows, dst, 0, band_rows,
                        width, k, main.cuda_stream))
        if interior_done is not None:
            interior_done.record(main)
        return
    if edge_stream is not None:
        edge_stream.wait_stream(main)
    check(step(src, pitch, k, band_rows, dst, pitch, k, width, band_rows - 2 * k, k,
               main.cuda_stream))
    if interior_done is not None:
        interior_done.record(main)
    es = edge_stream.cuda_stream if edge_stream is not None else main.cuda_stream
    if before_edges is not None:
        with torch.cuda.stream(edge_stream):
            before_edges()
    for r0 in (0, band_rows - k):
        check(step_peer(src, up, up_rows, down, down_rows, pitch, band_rows, dst, r0, k, width,
                        k, es))
    if edge_stream is not None:
        main.wait_stream(edge_stream)


def neighbour_token(token: torch.Tensor, inbox: torch.Tensor, rank: int, world: int,
                    group=None) -> None:
    """Pass ordering with the two neighbouring ranks only: send `token` (one
    element) to the rank above and the rank below, receive theirs into
    inbox[0] (from above) and inbox[1] (from below).  Same issue order on every
    rank (send up, send down, recv down, recv up) so the i-th send to a peer
    matches its i-th receive, also when up == down (two ranks).  With NCCL,
    wait() orders the current stream after the transfers (the host does not
    block); with gloo it blocks the host."""
    up, down = (rank - 1) % world, (rank + 1) % world
    ops = [dist.P2POp(dist.isend, token, up, group),
           dist.P2POp(dist.isend, token, down, group),
           dist.P2POp(dist.irecv, inbox[1:2], down, group),
           dist.P2POp(dist.irecv, inbox[0:1], up, group)]
    for w in dist.batch_isend_irecv(ops):
        w.wait()


class PeerBandDriver(PairLayout):
    """One rank's band for the fused NVLink halo (see above).

    `sync` orders passes across ranks: "neighbour" (default with NCCL) -- a
    4-byte token sent to and received from the bands above and below,
    stream-ordered on the compute stream (the reference's per-generation
    barrier, engine.cpp:79-96, narrowed to the two ranks whose rows a band
    touches); "neighbour_overlap" (opt-in, NCCL only) -- the same token, but
    exchanged on the EDGE stream before a pass's edge strips instead of on the
    compute stream after the pass: the token of pass p-1 only guards pass p's
    edge strips (they read the neighbours' rows and overwrite the rows the
    neighbours read), while pass p's interior reads the band's own rows and
    writes rows no neighbour reads, so it starts without waiting and hides the
    exchange; "flag" / "flag_overlap" (opt-in) -- the same two orders with no
    kernel at all: each rank owns two 32-bit flags in a CUDA-IPC buffer, the
    neighbours bump them with stream memory operations
    (life_dev_flag_write) and the rank waits for both on its stream
    (life_dev_flag_wait_geq): no SM slot, no NCCL launch;
    "allreduce" -- a 1-element NCCL all-reduce over every rank;
    "host" (forced with non-NCCL groups) -- synchronize + dist.barrier.
    With `profile` on, CUDA events around each pass's interior launch and
    barrier give per-rank interior / barrier times (stats())."""

    def __init__(self, geo: BandGeometry, device: torch.device, group=None,
                 sync: str = "neighbour", profile: bool = False):
        if geo.world < 2 and not geo.self_exchange:
            raise ConfigError("PeerBandDriver needs at least two ranks")
        self.geo = geo
        self.device = device
        self.group = group
        self.buf = [DeviceBuffer(geo.band_rows, geo.pitch, device) for _ in range(2)]
        # Pass-ordering flags (sync "flag"): word 0 is bumped by the band above,
        # word 1 by the band below (zeroed by life_dev_alloc).
        self.flags = DeviceBuffer(1, 32, device)
        self._epoch = 0
        torch.cuda.synchronize(device)
        self.cur = 0
        self.generations = 0
        # Exchange IPC handles and band heights with every rank.
        mine = (geo.band_rows, [b.handle() for b in self.buf] + [self.flags.handle()])
        allinfo = [None] * geo.world
        dist.all_gather_object(allinfo, mine, group=group)
        up, down = (geo.rank - 1) % geo.world, (geo.rank + 1) % geo.world
        self._opened = []

        def peer_ptrs(r):
            rows, handles = allinfo[r]
            ptrs = []
            for i, h in enumerate(handles):
                if r == geo.rank:
                    ptrs.append((self.buf + [self.flags])[i].ptr.value)
                else:
                    p = open_peer(h)
                    self._opened.append(p)
                    ptrs.append(p)
            return rows, ptrs

        with torch.cuda.device(device):
            self.up_rows, self.up_ptrs = peer_ptrs(up)
            self.down_rows, self.down_ptrs = (self.up_rows, self.up_ptrs) if down == up \
                else peer_ptrs(down)
        self._flag = torch.zeros(1, dtype=torch.int32, device=device)
        self._tok_in = torch.zeros(2, dtype=torch.int32, device=device)
        self._nccl = dist.get_backend(group) == "nccl"
        if sync not in ("neighbour", "neighbour_overlap", "flag", "flag_overlap", "allreduce",
                        "host"):
            raise ConfigError(f"unknown pass sync {sync!r}")
        # flags need no collective backend; the NCCL orders fall back to host barriers
        self.sync = sync if (self._nccl or sync.startswith("flag")) else "host"
        self.edge_stream = torch.cuda.Stream(device)
        self.profile = profile
        self._events = []  # (start, interior done, pass done, barrier done) per pass
        self._passes_since_sync = 0  # neighbour_overlap: passes whose token is still owed
        self._last_k = 0             # ... and the depth of the previous pass

    def _band_raw(self) -> torch.Tensor:
        return self.buf[self.cur].tensor

    def band(self) -> torch.Tensor:
        """This rank's band in the plain packed layout (converted in place
        after the last pass's barrier, so no neighbour still reads it)."""
        self._to_plain()
        return self.buf[self.cur].tensor

    def barrier(self) -> None:
        if self.sync in ("flag", "flag_overlap"):
            # "I am past this point" into the neighbours' flags, then wait for
            # theirs: up's word 1 (I am its band below), down's word 0.
            L = capi.lib()
            s = torch.cuda.current_stream(self.device).cuda_stream
            self._epoch += 1
            check(L.life_dev_flag_write(self.up_ptrs[2] + 4, self._epoch, s))
            check(L.life_dev_flag_write(self.down_ptrs[2], self._epoch, s))
            check(L.life_dev_flag_wait_geq(self.flags.ptr.value, self._epoch, s))
            check(L.life_dev_flag_wait_geq(self.flags.ptr.value + 4, self._epoch, s))
        elif self.sync in ("neighbour", "neighbour_overlap"):
            neighbour_token(self._flag, self._tok_in, self.geo.rank, self.geo.world, self.group)
        elif self.sync == "allreduce":
            dist.all_reduce(self._flag, group=self.group)  # ordered on the current stream
        else:
            torch.cuda.synchronize(self.device)
            dist.barrier(group=self.group)

    def compute(self, k: int, interior_done=None, before_edges=None) -> None:
        """The pass's kernels (interior + peer edge strips), no barrier."""
        g = self.geo
        c = self.cur
        peer_pass(g.width, self.buf[c].ptr.value, self.up_ptrs[c], self.up_rows,
                  self.down_ptrs[c], self.down_rows, g.pitch, g.band_rows,
                  self.buf[c ^ 1].ptr.value, k, self.device, self.edge_stream,
                  interior_done=interior_done, il=g.il, before_edges=before_edges)

    def pass_(self, k: int) -> None:
        g = self.geo
        if not 1 <= k <= g.depth:
            raise ConfigError(f"pass depth {k} outside [1, {g.depth}]")
        if g.il and not self.in_pair:
            raise ConfigError("band in the plain layout: interleaved passes start through run() "
                              "(conversion, then a barrier with the neighbours)")
        if self.sync in ("neighbour_overlap", "flag_overlap"):
            # run() has exchanged the "initial band in place" token; from then
            # on each pass waits for "previous pass done" on its edge stream.
            # The interior writes rows [k, band - k) of the buffer the previous
            # pass read; the neighbours read that buffer's outer k_prev rows, so
            # the interior may run ahead of the token only if k >= k_prev (a
            # shallower remainder pass after a full one waits like the rest).
            owed = self._passes_since_sync > 0
            if g.band_rows > 2 * k and k >= self._last_k:
                self.compute(k, before_edges=self.barrier if owed else None)
            else:  # thin band (one peer-mode launch) or a shallower pass: token first
                if owed:
                    self.barrier()
                self.compute(k)
            self._passes_since_sync += 1
            self._last_k = k
        elif self.profile:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record()
            self.compute(k, interior_done=ev[1])
            ev[2].record()
            self.barrier()
            ev[3].record()
            self._events.append((k, ev))
        else:
            self.compute(k)
            self.barrier()
        self.cur ^= 1
        self.generations += k

    def stats(self, reset: bool = True) -> dict:
        """Summed per-pass times (ms) of the profiled passes on this rank:
        interior launch, pass (interior + edge strips joined) and barrier."""
        torch.cuda.synchronize(self.device)
        out = {"passes": len(self._events), "interior_ms": 0.0, "pass_ms": 0.0,
               "barrier_ms": 0.0, "interior_full_ms": 0.0,
               "ks": [k for k, _ in self._events]}
        for k, ev in self._events:
            t = ev[0].elapsed_time(ev[1])
            out["interior_ms"] += t
            if k == self.geo.depth:
                out["interior_full_ms"] += t
            out["pass_ms"] += ev[0].elapsed_time(ev[2])
            out["barrier_ms"] += ev[2].elapsed_time(ev[3])
        if reset:
            self._events = []
        return out

    def run(self, generations: int, on_pass: Optional[Callable[[int], None]] = None,
            checkpoints: Sequence[int] = ()) -> list[int]:
        self._to_pair()  # before the barrier: the neighbours read this band in that layout
        self.barrier()  # every rank's initial band is in place
        self._passes_since_sync = 0
        self._last_k = 0
        pops = run_schedule(self, generations, checkpoints, on_pass)
        if self.sync in ("neighbour_overlap", "flag_overlap") and self._passes_since_sync:
            self.barrier()  # the last pass's token: nobody reads this band's old rows any more
            self._passes_since_sync = 0
        return pops

    def init_random(self, density: float, seed: int) -> None:
        g = self.geo
        self.in_pair = False
        stream = torch.cuda.current_stream(self.device).cuda_stream
        check(capi.lib().life_dev_packed_random(self.band().data_ptr(), g.pitch, g.width, g.y0,
                                                g.band_rows, density, seed, stream))
        self.generations = 0

    def load_rows(self, words) -> None:
        g = self.geo
        src = torch.from_numpy(words[g.y0:g.y1].view("int32").copy())
        self.in_pair = False
        self.band()[:, :src.shape[1]].copy_(src)
        self.generations = 0

    def population(self) -> int:
        g = self.geo
        acc = torch.zeros(1, dtype=torch.int64, device=self.device)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        check(capi.lib().life_dev_packed_population(self._band_raw().data_ptr(), g.pitch, g.width,
                                                    g.band_rows, acc.data_ptr(), stream))
        dist.all_reduce(acc, group=self.group)
        return int(acc.item())

    def close(self) -> None:
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            capi.lib().life_ipc_close(p)
        self._opened = []
        for b in self.buf + [self.flags]:
            b.free()


class LocalPeerBands:
    """P bands of one torus on ONE device through the fused-halo kernel
    (life_dev_packed_step_peer with the neighbours' local buffers as the
    peers): exercises the in-kernel cross-band row addressing with no
    cross-GPU waits."""

    def __init__(self, width: int, height: int, parts: int, depth: int, device: torch.device,
                 il: int = 0):
        if parts < 2:
            raise ConfigError("LocalPeerBands needs at least two bands")
        self.geos = [make_geometry(width, height, r, parts, depth, il) for r in range(parts)]
        self.il = il
        self.in_pair = False
        self.device = device
        self.bufs = [[torch.zeros((g.band_rows, g.pitch), dtype=torch.int32, device=device)
                      for _ in range(2)] for g in self.geos]
        self.cur = 0
        self.edge_stream = torch.cuda.Stream(device)

    def init_random(self, density: float, seed: int) -> None:
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self.in_pair = False
        for g, b in zip(self.geos, self.bufs):
            check(capi.lib().life_dev_packed_random(b[self.cur].data_ptr(), g.pitch, g.width, g.y0,
                                                    g.band_rows, density, seed, stream))

    def _zip(self, to_pair: bool) -> None:
        stream = torch.cuda.current_stream(self.device).cuda_stream
        for g, b in zip(self.geos, self.bufs):
            check(capi.lib().life_dev_packed_zip(b[self.cur].data_ptr(), g.pitch, g.width, 0,
                                                 g.band_rows, self.il, 1 if to_pair else 0,
                                                 stream))
        self.in_pair = to_pair

    def pass_(self, k: int) -> None:
        p = len(self.geos)
        if self.il and not self.in_pair:
            self._zip(True)
        c = self.cur
        for r, g in enumerate(self.geos):
            up, down = (r - 1) % p, (r + 1) % p
            peer_pass(g.width, self.bufs[r][c].data_ptr(), self.bufs[up][c].data_ptr(),
                      self.geos[up].band_rows, self.bufs[down][c].data_ptr(),
                      self.geos[down].band_rows, g.pitch, g.band_rows,
                      self.bufs[r][c ^ 1].data_ptr(), k, self.device, self.edge_stream,
                      il=self.il)
        self.cur ^= 1

    def run(self, generations: int) -> None:
        depth = self.geos[0].depth
        done = 0
        while done < generations:
            k = min(depth, generations - done)
            self.pass_(k)
            done += k

    def gather(self) -> torch.Tensor:
        """The whole torus as packed uint32 rows (device), plain layout."""
        if self.in_pair:
            self._zip(False)
        return torch.cat([b[self.cur] for b in self.bufs], dim=0)
