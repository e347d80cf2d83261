"""Python mirror of the reference's operator API for the step loop, running on
the B200 engine through the C-ABI (include/life_gpu.h).

Reference interface mirrored (paths under /root/reference/proj):
  - errors:  Error > ConfigError > {DimensionTooSmall, TooManyParts, OutOfBounds}
             (core/include/life/errors.hpp:9-60)
  - Grid:    byte-per-cell torus, >= 3x3, row-major (core/include/life/grid.hpp:24-70)
  - Strategy / RunConfig / RunStats / RunResult (decomposition.hpp:30-49,
             engine.hpp:11-27), with GPU strategy kinds added
  - run(initial, config, checkpoints) (engine.hpp:40-43, engine.cpp:157-214)
  - step_parallel(grid, strategy, workers) (engine.hpp:33, engine.cpp:152-155)
  - random_fill(width, height, density, seed) (pattern.hpp:55, pattern.cpp:330-342)
  - population(grid) (grid.hpp:84, grid.cpp:40-46) -- returns a Python int (no overflow)

`Engine` is the resident-grid handle (one C-ABI context): upload once, run
many generations, read windows/populations without downloading.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import capi


class Error(RuntimeError):
    """life::Error (errors.hpp:9-13)."""


class ConfigError(Error):
    """life::ConfigError (errors.hpp:17-20)."""


class DimensionTooSmall(ConfigError):
    """life::DimensionTooSmall (errors.hpp:22-27)."""


class TooManyParts(ConfigError):
    """life::TooManyParts (errors.hpp:29-35)."""


class OutOfBounds(ConfigError):
    """life::OutOfBounds (errors.hpp:37-40)."""


class CudaError(Error):
    """CUDA runtime failure inside the engine (no reference equivalent)."""


class NoDevice(CudaError):
    pass


_ERRORS = {
    capi.ERR_CONFIG: ConfigError,
    capi.ERR_DIMENSION_TOO_SMALL: DimensionTooSmall,
    capi.ERR_TOO_MANY_PARTS: TooManyParts,
    capi.ERR_OUT_OF_BOUNDS: OutOfBounds,
    capi.ERR_STATE: Error,
    capi.ERR_CUDA: CudaError,
    capi.ERR_NO_DEVICE: NoDevice,
    capi.ERR_OUT_OF_MEMORY: CudaError,
}


def check(rc: int) -> None:
    if rc != capi.OK:
        raise _ERRORS.get(rc, Error)(capi.last_error())


MIN_DIMENSION = 3


class Grid:
    """Byte-per-cell toroidal grid (grid.hpp:24-70); cells are 0/1 uint8."""

    def __init__(self, width: int, height: int, cells: np.ndarray | None = None):
        if width < MIN_DIMENSION or height < MIN_DIMENSION:
            raise DimensionTooSmall(
                f"grid dimensions must be at least 3x3, got {width}x{height}")
        self._w = int(width)
        self._h = int(height)
        if cells is None:
            self.cells = np.zeros((height, width), np.uint8)
        else:
            cells = np.asarray(cells, dtype=np.uint8)
            if cells.shape != (height, width):
                raise ConfigError(f"cell array shape {cells.shape} != {(height, width)}")
            self.cells = np.ascontiguousarray(cells)

    @classmethod
    def from_array(cls, cells: np.ndarray) -> "Grid":
        cells = np.asarray(cells)
        return cls(cells.shape[1], cells.shape[0], cells)

    def width(self) -> int:
        return self._w

    def height(self) -> int:
        return self._h

    def at(self, x: int, y: int) -> int:
        return int(self.cells[y, x])

    def alive(self, x: int, y: int) -> bool:
        return self.cells[y, x] != 0

    def set(self, x: int, y: int, state: int) -> None:
        self.cells[y, x] = state

    def wrap(self, x: int, y: int) -> tuple[int, int]:
        """Grid::wrap (grid.hpp:48-54)."""
        return x % self._w, y % self._h

    def data(self) -> np.ndarray:
        return self.cells

    def copy(self) -> "Grid":
        return Grid(self._w, self._h, self.cells.copy())

    def __eq__(self, other) -> bool:
        return (isinstance(other, Grid) and self._w == other._w and self._h == other._h
                and np.array_equal(self.cells, other.cells))

    def __repr__(self) -> str:
        return f"Grid({self._w}x{self._h}, population={population(self)})"


def population(grid: Grid) -> int:
    """population (grid.cpp:40-46) over 0/1 cells, as an unbounded int."""
    return int(np.count_nonzero(grid.cells))


@dataclass(frozen=True)
class Strategy:
    """Strategy (decomposition.hpp:30-49) plus the GPU kinds this engine adds.

    `gpu_packed` runs the bit-packed temporal-blocked engine with `depth`
    generations per kernel pass (0 = auto: the cluster-resident engine for
    small tori with W % 32 == 0, else 16); `gpu_resident` keeps the whole
    torus in one thread-block cluster's shared memory and runs every
    generation in one launch; `gpu_byte` runs the byte-per-cell engine,
    `depth` (1..8, 0 = auto: 4) generations per pass when W % 16 == 0, else one."""

    kind: str = "gpu_packed"
    blocks_x: int = 1
    blocks_y: int = 1
    depth: int = 0

    @staticmethod
    def gpu_packed(depth: int = 0) -> "Strategy":
        return Strategy("gpu_packed", 1, 1, depth)

    @staticmethod
    def gpu_byte(depth: int = 0) -> "Strategy":
        return Strategy("gpu_byte", 1, 1, depth)

    @staticmethod
    def gpu_resident() -> "Strategy":
        return Strategy("gpu_resident", 1, 1, 0)

    def engine(self) -> int:
        if self.kind == "gpu_packed":
            return capi.ENGINE_PACKED
        if self.kind == "gpu_byte":
            return capi.ENGINE_BYTE
        if self.kind == "gpu_resident":
            return capi.ENGINE_RESIDENT
        raise ConfigError(f"strategy '{self.kind}' is not a GPU strategy")


def to_string(strategy: Strategy) -> str:
    """Strategy token (decomposition.cpp:51-66 style): gpu, gpu:K, gpu-byte,
    gpu-resident."""
    if strategy.kind == "gpu_byte":
        return "gpu-byte" if strategy.depth == 0 else f"gpu-byte:{strategy.depth}"
    if strategy.kind == "gpu_resident":
        return "gpu-resident"
    return "gpu" if strategy.depth == 0 else f"gpu:{strategy.depth}"


def parse_strategy(token: str) -> Strategy:
    """parse_strategy (decomposition.cpp:68-91) for the GPU tokens."""
    if token == "gpu":
        return Strategy.gpu_packed()
    if token == "gpu-byte":
        return Strategy.gpu_byte()
    if token == "gpu-resident":
        return Strategy.gpu_resident()
    for prefix, limit, make in (("gpu:", capi.MAX_TEMPORAL_DEPTH, Strategy.gpu_packed),
                                ("gpu-byte:", capi.MAX_BYTE_DEPTH, Strategy.gpu_byte)):
        if token.startswith(prefix):
            try:
                k = int(token[len(prefix):])
            except ValueError:
                k = -1
            if 1 <= k <= limit:
                return make(k)
    raise ConfigError(f"unknown strategy '{token}' (expected gpu, gpu:K (1..16), gpu-byte, "
                      "gpu-byte:K (1..8) or gpu-resident)")


@dataclass
class RunConfig:
    """RunConfig (engine.hpp:11-15)."""

    strategy: Strategy = field(default_factory=Strategy.gpu_packed)
    workers: int = 1
    iterations: int = 0
    device: int = 0
    # Row bands over several GPUs (life_ctx_create_multi): one band per entry,
    # ids may repeat.  Empty = one GPU (`device`).
    devices: tuple = ()


@dataclass
class RunStats:
    """RunStats (engine.hpp:17-22); populations are unbounded ints."""

    generations_computed: int = 0
    population_checkpoints: list = field(default_factory=list)


@dataclass
class RunResult:
    grid: Grid
    stats: RunStats


class Engine:
    """One C-ABI context: a grid resident on one GPU, or -- with `devices` --
    split into row bands over several GPUs (life_ctx_create_multi; repeated
    device ids put several bands on one GPU)."""

    def __init__(self, device: int = 0, devices: Sequence[int] | None = None):
        self._lib = capi.lib()
        self._ctx = C.c_void_p()
        if devices is not None:
            devs = (C.c_int * len(devices))(*[int(d) for d in devices])
            check(self._lib.life_ctx_create_multi(len(devices), devs, C.byref(self._ctx)))
            self.device = int(devices[0]) if len(devices) else device
            self.devices = [int(d) for d in devices]
        else:
            check(self._lib.life_ctx_create(device, C.byref(self._ctx)))
            self.device = device
            self.devices = [device]

    def close(self) -> None:
        if self._ctx:
            self._lib.life_ctx_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._ctx

    def set_stream(self, stream_ptr: int | None) -> None:
        check(self._lib.life_ctx_set_stream(self._ctx, stream_ptr))

    def sync(self) -> None:
        check(self._lib.life_ctx_sync(self._ctx))

    def set_option(self, option: int, value: int) -> None:
        check(self._lib.life_ctx_set_option(self._ctx, option, value))

    def get_option(self, option: int) -> int:
        v = C.c_int64()
        check(self._lib.life_ctx_get_option(self._ctx, option, C.byref(v)))
        return int(v.value)

    def bands(self) -> dict:
        """Band layout: {'bounds': [...n+1 row cuts], 'devices': [...], 'halo': int}."""
        n, halo = C.c_int32(), C.c_int32()
        check(self._lib.life_ctx_bands(self._ctx, C.byref(n), None, None, C.byref(halo)))
        bounds = np.zeros(n.value + 1, np.int64)
        devs = np.zeros(n.value, np.int32)
        check(self._lib.life_ctx_bands(self._ctx, None, bounds.ctypes.data, devs.ctypes.data, None))
        return {"bounds": [int(x) for x in bounds], "devices": [int(x) for x in devs],
                "halo": int(halo.value)}

    def band_stats(self) -> list[dict]:
        """life_band_stats of every band for the last run()."""
        n = C.c_int32()
        check(self._lib.life_ctx_bands(self._ctx, C.byref(n), None, None, None))
        out = []
        for i in range(n.value):
            s = capi.BandStats()
            check(self._lib.life_ctx_band_stats(self._ctx, i, C.byref(s)))
            out.append(s.as_dict())
        return out

    # -- grid in / out ----------------------------------------------------
    def upload(self, cells: np.ndarray) -> None:
        cells = np.asarray(cells)
        if cells.dtype != np.uint8:
            cells = cells.astype(np.uint8)
        if cells.ndim != 2 or cells.strides[1] != 1:
            cells = np.ascontiguousarray(cells)
        h, w = cells.shape
        check(self._lib.life_grid_upload_u8(self._ctx, cells.ctypes.data, w, h, cells.strides[0]))

    def upload_packed(self, words: np.ndarray, width: int) -> None:
        words = np.ascontiguousarray(words, dtype=np.uint64)
        h, wpr = words.shape
        check(self._lib.life_grid_upload_packed(self._ctx, words.ctypes.data, width, h, wpr))

    def init_random(self, width: int, height: int, density: float, seed: int,
                    engine: int = capi.ENGINE_PACKED) -> None:
        check(self._lib.life_grid_init_random(self._ctx, width, height, density, seed, engine))

    def init_soup(self, width: int, height: int, coverage: float = 0.02, block: int = 5,
                  density: float = 0.5, seed: int = 42, engine: int = capi.ENGINE_PACKED) -> None:
        """Config-4 sparse soup generated on the device (life_grid_init_soup)."""
        check(self._lib.life_grid_init_soup(self._ctx, width, height, coverage, block, density,
                                            seed, engine))

    def place(self, pattern: np.ndarray, x0: int, y0: int) -> None:
        """place_pattern (pattern.cpp:309-328) on the resident grid."""
        pat = np.ascontiguousarray(pattern, dtype=np.uint8)
        ph, pw = pat.shape
        check(self._lib.life_grid_place_u8(self._ctx, pat.ctypes.data, pw, ph, x0, y0))

    def dims(self) -> tuple[int, int]:
        w, h = C.c_int64(), C.c_int64()
        check(self._lib.life_grid_dims(self._ctx, C.byref(w), C.byref(h)))
        return w.value, h.value

    def download(self, out: np.ndarray | None = None) -> np.ndarray:
        w, h = self.dims()
        if out is None:
            out = np.empty((h, w), np.uint8)
        check(self._lib.life_grid_download_u8(self._ctx, out.ctypes.data, out.strides[0]))
        return out

    def download_packed(self, out: np.ndarray | None = None) -> np.ndarray:
        w, h = self.dims()
        if out is None:
            out = np.empty((h, (w + 63) // 64), np.uint64)
        check(self._lib.life_grid_download_packed(self._ctx, out.ctypes.data, out.shape[1]))
        return out

    def window(self, x0: int, y0: int, w: int, h: int) -> np.ndarray:
        out = np.empty((h, w), np.uint8)
        check(self._lib.life_grid_window_u8(self._ctx, x0, y0, w, h, out.ctypes.data))
        return out

    def population(self) -> int:
        v = C.c_uint64()
        check(self._lib.life_population(self._ctx, C.byref(v)))
        return int(v.value)

    def hash(self) -> int:
        """life_grid_hash: FNV-1a-64 of the packed rows' FNV-1a-64 hashes."""
        v = C.c_uint64()
        check(self._lib.life_grid_hash(self._ctx, C.byref(v)))
        return int(v.value)

    # -- the step loop ----------------------------------------------------
    def run(self, generations: int, engine: int = capi.ENGINE_PACKED, depth: int = 0,
            checkpoints: Sequence[int] = ()) -> list[int]:
        cps = np.asarray(list(checkpoints), dtype=np.int64)
        pops = np.zeros(max(len(cps), 1), np.uint64)
        check(self._lib.life_run(self._ctx, generations, engine, depth,
                                 cps.ctypes.data if len(cps) else None, len(cps),
                                 pops.ctypes.data))
        return [int(p) for p in pops[:len(cps)]]

    def step(self, engine: int = capi.ENGINE_PACKED) -> None:
        check(self._lib.life_step(self._ctx, engine))

    def run_batch(self, inputs: Sequence[np.ndarray], outputs: Sequence[np.ndarray], width: int,
                  generations: int, depth: int = 0) -> float:
        """life_run_batch: packed host grids (uint64 rows) in, results out,
        copies overlapped with compute.  Returns the CUDA-event time in ms."""
        n = len(inputs)
        if len(outputs) != n:
            raise ConfigError("inputs and outputs differ in length")
        if n == 0:
            return 0.0
        h, wpr = inputs[0].shape
        for a in list(inputs) + list(outputs):
            if a.shape != (h, wpr) or a.dtype != np.uint64 or not a.flags.c_contiguous:
                raise ConfigError("batch buffers must be C-contiguous uint64 (H, words_per_row)")
        ins = (C.c_void_p * n)(*[a.ctypes.data for a in inputs])
        outs = (C.c_void_p * n)(*[a.ctypes.data for a in outputs])
        ms = C.c_float()
        check(self._lib.life_run_batch(self._ctx, ins, outs, n, width, h, wpr, generations, depth,
                                       C.byref(ms)))
        return float(ms.value)


def _check_workers(config: RunConfig, height: int) -> None:
    if config.workers < 1:
        raise ConfigError(f"worker count must be at least 1, got {config.workers}")
    if config.workers > height:
        raise TooManyParts(
            f"cannot split {height} rows into {config.workers} non-empty parts")


def run(initial: Grid, config: RunConfig, checkpoints: Iterable[int] = ()) -> RunResult:
    """run (engine.cpp:157-214) on the GPU: `config.iterations` generations,
    populations at the strictly ascending checkpoints (0 = initial grid).
    `workers` is validated like the reference's row bands (engine.cpp:127-131,
    decomposition.cpp:26-30); `config.devices` spreads the torus over row
    bands on several GPUs (band_bounds, decomposition.cpp:12-24) in this one
    call, as the reference's Strategy::rows() does over threads."""
    checkpoints = list(checkpoints)
    _check_workers(config, initial.height())
    engine = config.strategy.engine()
    with (Engine(devices=list(config.devices)) if config.devices else Engine(config.device)) as e:
        e.upload(initial.cells)
        pops = e.run(config.iterations, engine, config.strategy.depth, checkpoints)
        out = e.download()
    stats = RunStats(config.iterations, list(zip(checkpoints, pops)))
    return RunResult(Grid(initial.width(), initial.height(), out), stats)


def step_parallel(grid: Grid, strategy: Strategy, workers: int = 1) -> Grid:
    """step_parallel (engine.cpp:152-155): one generation."""
    return run(grid, RunConfig(strategy, workers, 1)).grid


def random_fill(width: int, height: int, density: float, seed: int, device: int = 0) -> Grid:
    """random_fill (pattern.cpp:330-342), generated on the device."""
    if not (0.0 <= density <= 1.0):
        raise ConfigError(f"density must be in [0, 1], got {density}")
    with Engine(device) as e:
        e.init_random(width, height, density, seed, capi.ENGINE_BYTE)
        return Grid(width, height, e.download())


def band_bounds(extent: int, parts: int) -> list[int]:
    """band_bounds (decomposition.cpp:12-24) through the C-ABI."""
    b = np.zeros(max(parts, 0) + 1, np.int64)
    check(capi.lib().life_band_bounds(extent, parts, b.ctypes.data))
    return [int(x) for x in b]
