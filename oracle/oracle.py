"""ctypes front-end for the parity checkers -- TEST INFRASTRUCTURE ONLY.

`Oracle` wraps oracle/liboracle.so (the C restatement, oracle/life_oracle.c);
`Reference` wraps oracle/_ref/liblife_ref.so (the unmodified reference core,
built by `make -C oracle ref` from /root/reference/proj/core).  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs may import this
module; the product package (paper_1209_4408_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblife_ref.so")

_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def build_oracle() -> None:
    """Compiles oracle/liboracle.so (and oracle/_ref when the reference tree is present)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if os.path.isdir("/root/reference/proj/core"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


class Oracle:
    """The C restatement of the reference path (oracle/life_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
        L = C.CDLL(path)
        self.lib = L
        L.orc_splitmix_stream.argtypes = [C.c_uint64, C.c_int64, _u64p]
        L.orc_density_threshold.argtypes = [C.c_double]
        L.orc_density_threshold.restype = C.c_uint64
        L.orc_random_fill.argtypes = [_u8p, C.c_int64, C.c_int64, C.c_double, C.c_uint64]
        L.orc_random_window.argtypes = [_u8p, C.c_int64, C.c_int64, C.c_double, C.c_uint64,
                                        C.c_int64, C.c_int64, C.c_int64, C.c_int64]
        L.orc_sparse_soup.argtypes = [_u8p, C.c_int64, C.c_int64, C.c_double, C.c_int32,
                                      C.c_double, C.c_uint64]
        L.orc_step_serial.argtypes = [_u8p, _u8p, C.c_int64, C.c_int64]
        L.orc_population.argtypes = [_u8p, C.c_int64]
        L.orc_population.restype = C.c_uint64
        L.orc_run.argtypes = [_u8p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int32,
                              C.c_void_p]
        L.orc_run_serial.argtypes = [_u8p, C.c_int64, C.c_int64, C.c_int64]
        L.orc_lightcone.argtypes = [_u8p, C.c_int64, C.c_int64, _u8p]
        L.orc_fnv1a64.argtypes = [C.c_void_p, C.c_int64, C.c_uint64]
        L.orc_fnv1a64.restype = C.c_uint64
        L.orc_grid_hash.argtypes = [_u64p, C.c_int64, C.c_int64]
        L.orc_grid_hash.restype = C.c_uint64
        L.orc_pack.argtypes = [_u8p, C.c_int64, C.c_int64, _u64p]
        L.orc_unpack.argtypes = [_u64p, C.c_int64, C.c_int64, _u8p]
        L.orc_band_bounds.argtypes = [C.c_int64, C.c_int32, _i64p]
        L.orc_place_pattern.argtypes = [_u8p, C.c_int64, C.c_int64, _u8p, C.c_int64, C.c_int64,
                                        C.c_int64, C.c_int64]

    def splitmix(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self.lib.orc_splitmix_stream(seed, n, out)
        return out

    def threshold(self, density: float) -> int:
        return int(self.lib.orc_density_threshold(density))

    def random_fill(self, w: int, h: int, density: float, seed: int) -> np.ndarray:
        g = np.empty((h, w), np.uint8)
        if self.lib.orc_random_fill(g, w, h, density, seed) != 0:
            raise ValueError(f"density must be in [0, 1], got {density}")
        return g

    def random_window(self, W: int, H: int, density: float, seed: int, x0: int, y0: int,
                      w: int, h: int) -> np.ndarray:
        g = np.empty((h, w), np.uint8)
        if self.lib.orc_random_window(g, W, H, density, seed, x0, y0, w, h) != 0:
            raise ValueError("bad density")
        return g

    def sparse_soup(self, w: int, h: int, seed: int = 42, coverage: float = 0.02,
                    block: int = 5, p: float = 0.5) -> np.ndarray:
        g = np.empty((h, w), np.uint8)
        if self.lib.orc_sparse_soup(g, w, h, coverage, block, p, seed) != 0:
            raise ValueError("bad soup parameters")
        return g

    def step_serial(self, g: np.ndarray) -> np.ndarray:
        g = np.ascontiguousarray(g, dtype=np.uint8)
        out = np.empty_like(g)
        self.lib.orc_step_serial(g, out, g.shape[1], g.shape[0])
        return out

    def run_serial(self, g: np.ndarray, generations: int) -> np.ndarray:
        g = np.array(g, dtype=np.uint8, order="C", copy=True)
        self.lib.orc_run_serial(g, g.shape[1], g.shape[0], generations)
        return g

    def run(self, g: np.ndarray, generations: int, checkpoints=()):
        """compute_region-style run (engine.cpp:162-214); returns (grid, pops)."""
        g = np.array(g, dtype=np.uint8, order="C", copy=True)
        cps = np.asarray(list(checkpoints), dtype=np.int64)
        pops = np.zeros(max(len(cps), 1), np.uint64)
        rc = self.lib.orc_run(g, g.shape[1], g.shape[0], generations,
                              cps.ctypes.data if len(cps) else None, len(cps),
                              pops.ctypes.data)
        if rc != 0:
            raise ValueError("illegal run configuration")
        return g, [int(p) for p in pops[:len(cps)]]

    def lightcone(self, initial_window: np.ndarray, s: int, t: int) -> np.ndarray:
        w = np.ascontiguousarray(initial_window, dtype=np.uint8)
        assert w.shape == (s + 2 * t, s + 2 * t)
        out = np.empty((s, s), np.uint8)
        if self.lib.orc_lightcone(w, s, t, out) != 0:
            raise MemoryError("light-cone window allocation failed")
        return out

    def population(self, g: np.ndarray) -> int:
        g = np.ascontiguousarray(g, dtype=np.uint8)
        return int(self.lib.orc_population(g, g.size))

    def fnv1a64(self, data: np.ndarray) -> int:
        data = np.ascontiguousarray(data)
        return int(self.lib.orc_fnv1a64(data.ctypes.data, data.nbytes, 0))

    def grid_hash(self, g: np.ndarray) -> int:
        """life_grid_hash's definition on a byte grid (packs it first)."""
        p = self.pack(g)
        return int(self.lib.orc_grid_hash(p, p.shape[1], p.shape[0]))

    def packed_hash(self, words: np.ndarray) -> int:
        """The same on packed rows (uint64, ceil(W/64) words per row)."""
        words = np.ascontiguousarray(words, dtype=np.uint64)
        return int(self.lib.orc_grid_hash(words, words.shape[1], words.shape[0]))

    def pack(self, g: np.ndarray) -> np.ndarray:
        g = np.ascontiguousarray(g, dtype=np.uint8)
        h, w = g.shape
        out = np.empty((h, (w + 63) // 64), np.uint64)
        self.lib.orc_pack(g, w, h, out)
        return out

    def unpack(self, words: np.ndarray, w: int) -> np.ndarray:
        words = np.ascontiguousarray(words, dtype=np.uint64)
        h = words.shape[0]
        out = np.empty((h, w), np.uint8)
        self.lib.orc_unpack(words, w, h, out)
        return out

    def place_pattern(self, grid: np.ndarray, pattern: np.ndarray, x0: int, y0: int) -> np.ndarray:
        g = np.array(grid, dtype=np.uint8, order="C", copy=True)
        p = np.ascontiguousarray(pattern, dtype=np.uint8)
        if self.lib.orc_place_pattern(g, g.shape[1], g.shape[0], p, p.shape[1], p.shape[0],
                                      x0, y0) != 0:
            raise IndexError("pattern footprint exceeds the grid")
        return g

    def band_bounds(self, extent: int, parts: int) -> list[int]:
        b = np.zeros(max(parts, 0) + 1, np.int64)
        if self.lib.orc_band_bounds(extent, parts, b) != 0:
            raise ValueError(f"cannot split {extent} rows into {parts} non-empty parts")
        return [int(x) for x in b]


class Reference:
    """The unmodified reference core (oracle/_ref/liblife_ref.so)."""

    KIND = {"serial": 0, "rows": 1, "cols": 2, "blocks": 3}

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle ref)")
        L = C.CDLL(path)
        self.lib = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_hardware_threads.restype = C.c_uint
        L.ref_splitmix_stream.argtypes = [C.c_uint64, C.c_int64, _u64p]
        L.ref_splitmix_units.argtypes = [C.c_uint64, C.c_int64, _f64p]
        L.ref_random_fill.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, _u8p]
        L.ref_step_serial.argtypes = [_u8p, C.c_int, C.c_int, _u8p]
        L.ref_next_state.argtypes = [C.c_int, C.c_int]
        L.ref_run.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                              C.c_int, C.c_void_p, C.c_int, _u8p, C.c_void_p, C.c_void_p]
        L.ref_run_inplace.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.c_int, C.c_int]
        L.ref_time_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_int, C.c_uint64, C.c_double, C.c_int, C.c_int,
                                   C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                   C.POINTER(C.c_uint)]
        L.ref_partition_rows.argtypes = [C.c_int, C.c_int, C.c_int, _i32p]
        L.ref_sparse_soup_small.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_double,
                                            C.c_uint64, _u8p]
        L.ref_population.argtypes = [_u8p, C.c_int, C.c_int]
        L.ref_place_pattern.argtypes = [_u8p, C.c_int, C.c_int, _u8p, C.c_int, C.c_int, C.c_int,
                                        C.c_int]

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    def hardware_threads(self) -> int:
        return int(self.lib.ref_hardware_threads())

    def splitmix(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self.lib.ref_splitmix_stream(seed, n, out)
        return out

    def splitmix_units(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.ref_splitmix_units(seed, n, out)
        return out

    def random_fill(self, w: int, h: int, density: float, seed: int) -> np.ndarray:
        g = np.empty((h, w), np.uint8)
        self._check(self.lib.ref_random_fill(w, h, density, seed, g))
        return g

    def step_serial(self, g: np.ndarray) -> np.ndarray:
        g = np.ascontiguousarray(g, dtype=np.uint8)
        out = np.empty_like(g)
        self._check(self.lib.ref_step_serial(g, g.shape[1], g.shape[0], out))
        return out

    def next_state(self, alive: bool, n: int) -> bool:
        return bool(self.lib.ref_next_state(int(alive), n))

    def run(self, g: np.ndarray, iterations: int, strategy: str = "serial", workers: int = 1,
            blocks=(1, 1), checkpoints=()):
        g = np.ascontiguousarray(g, dtype=np.uint8)
        out = np.empty_like(g)
        cps = np.asarray(list(checkpoints), dtype=np.int32)
        pops = np.zeros(max(len(cps), 1), np.int64)
        gens = C.c_int(0)
        self._check(self.lib.ref_run(g, g.shape[1], g.shape[0], self.KIND[strategy], blocks[0],
                                     blocks[1], workers, iterations,
                                     cps.ctypes.data if len(cps) else None, len(cps), out,
                                     pops.ctypes.data, C.byref(gens)))
        return out, [int(p) for p in pops[:len(cps)]], gens.value

    def run_inplace(self, g: np.ndarray, iterations: int, strategy: str = "blocks",
                    workers: int = 8, blocks=(4, 2)) -> None:
        assert g.flags.c_contiguous and g.dtype == np.uint8
        self._check(self.lib.ref_run_inplace(g, g.shape[1], g.shape[0], self.KIND[strategy],
                                             blocks[0], blocks[1], workers, iterations))

    def time_run(self, w: int, h: int, iterations: int, strategy: str = "serial",
                 workers: int = 1, blocks=(1, 1), seed: int = 42, density: float = 0.3,
                 repetitions: int = 1, warmup: int = 0):
        med = C.c_double(0)
        pop = C.c_int64(0)
        hw = C.c_uint(0)
        self._check(self.lib.ref_time_run(w, h, iterations, self.KIND[strategy], blocks[0],
                                          blocks[1], workers, seed, density, repetitions,
                                          warmup, C.byref(med), C.byref(pop), C.byref(hw)))
        return med.value, pop.value, hw.value

    def partition_rows(self, w: int, h: int, parts: int) -> list[int]:
        cuts = np.zeros(parts + 1, np.int32)
        self._check(self.lib.ref_partition_rows(w, h, parts, cuts))
        return [int(c) for c in cuts]

    def sparse_soup_small(self, w: int, h: int, seed: int = 42, coverage: float = 0.02,
                          block: int = 5, p: float = 0.5) -> np.ndarray:
        g = np.empty((h, w), np.uint8)
        self._check(self.lib.ref_sparse_soup_small(w, h, coverage, block, p, seed, g))
        return g

    def population(self, g: np.ndarray) -> int:
        g = np.ascontiguousarray(g, dtype=np.uint8)
        return int(self.lib.ref_population(g, g.shape[1], g.shape[0]))

    def place_pattern(self, grid: np.ndarray, pattern: np.ndarray, x0: int, y0: int) -> np.ndarray:
        g = np.array(grid, dtype=np.uint8, order="C", copy=True)
        p = np.ascontiguousarray(pattern, dtype=np.uint8)
        self._check(self.lib.ref_place_pattern(g, g.shape[1], g.shape[0], p, p.shape[1],
                                               p.shape[0], x0, y0))
        return g


class PatternIO:
    """Pattern I/O + renderers through an extern-C library with the lio_/ref_
    signatures: the reference (oracle/_ref/liblife_ref.so, prefix "ref_") or
    the engine's host layer (paper_1209_4408_b200/host/liblife_io.so,
    prefix "lio_")."""

    def __init__(self, path: str, prefix: str):
        L = C.CDLL(path)
        self.p = prefix
        self.L = L
        ip = C.POINTER(C.c_int)
        for name in ("parse_rle", "parse_plaintext"):
            f = getattr(L, prefix + name)
            f.argtypes = [C.c_char_p, ip, ip, ip, ip, C.c_int, ip, ip, ip, C.c_char_p, C.c_int]
        f = getattr(L, prefix + "serialize_rle")
        f.argtypes = [C.c_int, C.c_int, ip, ip, C.c_int, C.c_char_p, C.c_int]
        for name in ("render_ascii", "render_pbm"):
            getattr(L, prefix + name).argtypes = [_u8p, C.c_int, C.c_int, C.c_char_p, C.c_int]

    def _parse(self, name: str, text: str):
        cap = max(16, len(text) * 64 + 1024)
        w, h, n, line, col = (C.c_int(0) for _ in range(5))
        xs = (C.c_int * cap)()
        ys = (C.c_int * cap)()
        msg = C.create_string_buffer(512)
        rc = getattr(self.L, self.p + name)(text.encode(), C.byref(w), C.byref(h), xs, ys, cap,
                                            C.byref(n), C.byref(line), C.byref(col), msg, 512)
        if rc == 3:
            return {"error": "parse", "line": line.value, "column": col.value}
        if rc != 0:
            return {"error": f"rc{rc}"}
        return {"w": w.value, "h": h.value, "cells": [[xs[i], ys[i]] for i in range(n.value)]}

    def parse_rle(self, text: str):
        return self._parse("parse_rle", text)

    def parse_plaintext(self, text: str):
        return self._parse("parse_plaintext", text)

    def serialize_rle(self, w: int, h: int, cells):
        n = len(cells)
        xs = (C.c_int * max(n, 1))(*[c[0] for c in cells])
        ys = (C.c_int * max(n, 1))(*[c[1] for c in cells])
        out = C.create_string_buffer(64 + 16 * (n + w * h))
        rc = getattr(self.L, self.p + "serialize_rle")(w, h, xs, ys, n, out, len(out))
        return out.value.decode() if rc == 0 else {"error": f"rc{rc}"}

    def render(self, kind: str, grid: np.ndarray) -> str:
        g = np.ascontiguousarray(grid, dtype=np.uint8)
        out = C.create_string_buffer(4 * g.size + 64)
        rc = getattr(self.L, self.p + "render_" + kind)(g, g.shape[1], g.shape[0], out, len(out))
        assert rc == 0
        return out.value.decode()
