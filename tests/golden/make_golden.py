"""Generates the committed golden fixtures under tests/golden/ by running the
UNMODIFIED reference core (oracle/_ref/liblife_ref.so, built from
/root/reference/proj/core by `make -C oracle ref`).  Run in the CPU container:

    python tests/golden/make_golden.py small      # seconds
    python tests/golden/make_golden.py cfg2       # ~1-2 min  (16384^2 x 1000)
    python tests/golden/make_golden.py cfg4       # ~10 min   (12289 x 40961 x 5000)
    python tests/golden/make_golden.py cfg3       # ~20 min   (65536^2 x 1000, 12 GiB RAM)
    python tests/golden/make_golden.py cfg5       # light-cone windows of 262144^2 x 500
    python tests/golden/make_golden.py split      # windows of split-launch W % 32 != 0 tori

Hash conventions (tests/golden/README.md):
  fnv_bytes  = FNV-1a-64 over the row-major W*H bytes (0/1);
  fnv_packed = FNV-1a-64 over the packed exchange format of include/life_gpu.h
               (rows of ceil(W/64) little-endian uint64, bit j = column 64k+j,
               tail bits zero).
The reference generates every grid and runs every generation; the oracle
restatement (oracle/life_oracle.c) is used only for packing/hashing and for
the config-4 soup and giant-grid windows, both of which are themselves pinned
against the reference in tests/test_oracle.py.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
O = Oracle()
R = Reference()
THREADS = os.cpu_count() or 8


def blocks_shape(n: int) -> tuple[int, int]:
    m = int(np.sqrt(n))
    while n % m:
        m -= 1
    return n // m, m


def hashes(g: np.ndarray) -> dict:
    return {"fnv_bytes": f"{O.fnv1a64(g):016x}", "fnv_packed": f"{O.fnv1a64(O.pack(g)):016x}",
            "population": O.population(g)}


def dump(name: str, obj) -> None:
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(obj, f, indent=1, sort_keys=True)
    print("wrote", name, flush=True)


def run_schedule(g: np.ndarray, schedule: list[int]) -> dict:
    """Runs the reference in place through ascending generation counts and
    records the hashes at each (g is modified)."""
    bx, by = blocks_shape(THREADS)
    out = {}
    done = 0
    for gen in schedule:
        t = time.time()
        if gen > done:
            R.run_inplace(g, gen - done, "blocks", THREADS, (bx, by))
        done = gen
        out[str(gen)] = hashes(g)
        print(f"  gen {gen}: {out[str(gen)]} ({time.time() - t:.1f}s)", flush=True)
    return out


def small() -> None:
    res = {}
    res["splitmix"] = {str(s): [f"{v:016x}" for v in R.splitmix(s, 8)]
                       for s in (0, 1, 42, 0xDEADBEEF)}
    res["next_unit_42"] = [repr(float(v)) for v in R.splitmix_units(42, 6)]
    res["truth_table"] = {"alive": [R.next_state(True, n) for n in range(9)],
                          "dead": [R.next_state(False, n) for n in range(9)]}
    # Config 1 (full grid): populations via the reference's checkpoints.
    g = R.random_fill(1024, 1024, 0.5, 42)
    cfg1 = {"0": hashes(g)}
    for gens in (1, 10, 100):
        out, pops, _ = R.run(g, gens, "rows", 8, checkpoints=[gens])
        cfg1[str(gens)] = hashes(out)
        cfg1[str(gens)]["ref_population"] = pops[0]
    res["cfg1"] = cfg1
    # Strategy-transparency dims (test_engine.cpp:49-83) and acceptance
    # criterion 1 dims (acceptance.cpp:55-60), run through the reference.
    cases = []
    for seed in range(8):
        w = 3 + (seed * 17 + 5) % 46
        h = 3 + (seed * 29 + 11) % 46
        cases.append((w, h, 0.3, seed, 20))
    for seed in range(200):
        d = R.splitmix(seed, 2)
        cases.append((3 + int(d[0] % 62), 3 + int(d[1] % 62), 0.3, seed, 50))
    # Non-multiple-of-32/64 widths and tiny tori around word boundaries.
    for (w, h) in [(3, 3), (4, 7), (31, 5), (32, 9), (33, 17), (63, 4), (64, 64), (65, 3),
                   (95, 40), (127, 33), (128, 128), (129, 77), (200, 150), (257, 131),
                   (1000, 37), (2049, 19)]:
        cases.append((w, h, 0.4, w * 1000 + h, 37))
    small_cases = []
    for (w, h, p, seed, gens) in cases:
        g0 = R.random_fill(w, h, p, seed)
        out, pops, _ = R.run(g0, gens, "serial", 1, checkpoints=[0, gens] if gens else [0])
        ref_serial = g0
        for _ in range(gens):
            ref_serial = R.step_serial(ref_serial)
        assert (ref_serial == out).all()
        small_cases.append({"w": w, "h": h, "density": p, "seed": seed, "gens": gens,
                            "initial": hashes(g0), "final": hashes(out)})
    res["small_cases"] = small_cases
    # Known patterns (test_grid.cpp:177-217; acceptance.cpp:107-136).
    glider = np.zeros((16, 16), np.uint8)
    for (x, y) in [(1, 0), (2, 1), (0, 2), (1, 2), (2, 2)]:  # "bo$2bo$3o!" at (6,6)
        glider[6 + y, 6 + x] = 1
    gl = glider.copy()
    lap = []
    for cycle in range(1, 17):
        for _ in range(4):
            gl = R.step_serial(gl)
        lap.append(bool((gl == np.roll(np.roll(glider, cycle, 0), cycle, 1)).all()))
    res["glider_lap"] = {"translated_each_cycle": lap, "home_after_64": bool((gl == glider).all())}
    # Config-4-style sparse soup on a small field via place_pattern itself.
    res["soup_small"] = [{"w": w, "h": h, "seed": s, **hashes(R.sparse_soup_small(w, h, seed=s))}
                         for (w, h, s) in [(200, 150, 3), (409, 121, 42), (97, 61, 7)]]
    # partition_rows cuts (decomposition.cpp:93-104) for the multi-GPU bands.
    res["partition_rows"] = {f"{h}/{p}": R.partition_rows(64, h, p)
                             for h in (12289, 262144, 65536, 16384, 1024, 37, 9)
                             for p in (1, 2, 3, 4, 8) if p <= h}
    dump("golden_small.json", res)


def cfg2() -> None:
    g = R.random_fill(16384, 16384, 0.3, 42)
    res = {"w": 16384, "h": 16384, "density": 0.3, "seed": 42,
           "gens": run_schedule(g, [0, 1, 10, 100, 1000])}
    dump("golden_cfg2.json", res)


def cfg3() -> None:
    g = R.random_fill(65536, 65536, 0.5, 42)
    res = {"w": 65536, "h": 65536, "density": 0.5, "seed": 42,
           "gens": run_schedule(g, [0, 1, 16, 100, 1000])}
    dump("golden_cfg3.json", res)


def cfg4() -> None:
    W, H = 40961, 12289
    g = O.sparse_soup(W, H, seed=42)
    res = {"w": W, "h": H, "soup": {"seed": 42, "coverage": 0.02, "block": 5, "p": 0.5},
           "gens": run_schedule(g, [0, 1, 100, 1000, 5000])}
    dump("golden_cfg4.json", res)


def windows(W: int, H: int, density: float, seed: int, T: int, S: int, spots) -> list:
    out = []
    bx, by = blocks_shape(THREADS)
    for (x0, y0) in spots:
        init = O.random_window(W, H, density, seed, x0 - T, y0 - T, S + 2 * T, S + 2 * T)
        g = init.copy()
        t = time.time()
        R.run_inplace(g, T, "blocks", THREADS, (bx, by))
        centre = np.ascontiguousarray(g[T:T + S, T:T + S])
        out.append({"x0": x0, "y0": y0, "S": S, "T": T, "fnv_bytes": f"{O.fnv1a64(centre):016x}",
                    "population": O.population(centre)})
        print(f"  window ({x0},{y0}) {out[-1]['fnv_bytes']} ({time.time() - t:.1f}s)", flush=True)
    return out


def cfg5() -> None:
    W = H = 262144
    S = 512
    spots = [(0, 0), (W - S // 2, H - S // 2), (W - 100, 7), (123457, 200001)]
    for p in (2, 4, 8):  # band seams of band_bounds(H, p)
        for j in range(1, p):
            y = j * (H // p)
            spots.append(((j * 77777) % W, y - S // 2))
    spots = sorted(set(spots))
    res = {"w": W, "h": H, "density": 0.4, "seed": 42,
           "windows_500": windows(W, H, 0.4, 42, 500, S, spots),
           "windows_16": windows(W, H, 0.4, 42, 16, 256, spots[:6])}
    dump("golden_cfg5_windows.json", res)


def split() -> None:
    """Light-cone windows of W % 32 != 0 tori deep enough for the split launch
    (seam strips on the all-paths kernel beside the fast-only kernel,
    life_packed_launch_kind == LIFE_LAUNCH_SPLIT): windows straddle the column
    seam and both wrap corners, the boundary between the last fast strip and
    the first seam strip (column 32*(31*s_last - 1)) and the strip-0 / strip-1
    boundary (column 960); shapes with nw % 31 == 0 (three seam strips) and
    W % 32 == 1 as well as 65535^2 and 131071 x 65536."""
    S = 256
    res = {}
    for (W, H, T, p, seed) in [(65535, 65535, 64, 0.5, 42), (131071, 65536, 48, 0.4, 7),
                               (2975, 700000, 32, 0.4, 2026), (2049, 700000, 32, 0.4, 11)]:
        nw = -(-W // 32)
        s_last = (nw - 1) // 31
        seam_col = 32 * (31 * s_last - 1)
        spots = [(W - S // 2, H - S // 2), (W - 100, 7), (0, H // 3), (seam_col - S // 2, H // 2),
                 (960 - S // 2, 2 * H // 3), (W // 2, 12345)]
        res[f"{W}x{H}"] = {"w": W, "h": H, "density": p, "seed": seed, "T": T,
                           "windows": windows(W, H, p, seed, T, S, spots)}
    dump("golden_split_windows.json", res)


def cfg3w() -> None:
    """Light-cone windows of config 3 (quick GPU checks without the full hash)."""
    W = H = 65536
    spots = [(0, 0), (W - 128, H - 128), (40000, 12345), (W - 64, 30000)]
    res = {"w": W, "h": H, "density": 0.5, "seed": 42,
           "windows_100": windows(W, H, 0.5, 42, 100, 256, spots)}
    dump("golden_cfg3_windows.json", res)


def io_cases():
    """Inputs for the pattern I/O parity cases (reference tests + fuzz)."""
    rng = np.random.default_rng(1234)
    rle = ["x = 3, y = 1\n3o!", "x = 3, y = 3\nbo$2bo$3o!",
           "#N Glider\n#C the classic\nx = 3, y = 3, rule = B3/S23\nbo$2bo$3o!\n",
           "x = 2, y = 1\nBO!", "x = 3, y = 1, rule = 23/3\n3o!", "x = 3, y = 1, rule = B36/S23\n3o!",
           "x = 3, y = 5\no3$o$o!", "x = 3, y = 3\no!", "x = 2, y = 1\n5o!", "x = 3, y = 1\no$o!",
           "x = 3, y = 1\n2b2b!", "", "y = 1, x = 3\n3o!", "x = 3, y = 1\n3o", "x = 3, y = 1\n3!",
           "x = 3, y = 1\n0o!", "x = 3, y = 1\noqo!", "x = 3, y = 1\n3o! trailing notes\nmore",
           "x = 3, y = 1\n2o1o!", "x = 3, y = 2\nooo$!", "x = 3, y = 1\n1o1b1o!",
           "x=3,y=1\n3o!", "x = 3 , y = 1 , rule = b3/s23 \n3o!", "x = 3, y = 1, foo = 1\n3o!",
           "x = 3, y = 1 junk\n3o!", "   \n\n#c\nx = 4, y = 2\n 2o\n b $ o !", "x = , y = 1\n!",
           "x = 99999999999, y = 1\n!", "x = 3, y = 1\n1!", "x = 3, y = 1\n12", "#only comment",
           "x = 10, y = 3\n10o$10b$10o!", "x = 3, y = 1\nb\n\no\n\nb!", "x = 1, y = 1\n!"]
    for _ in range(80):  # mutate canonical forms
        w, h = int(rng.integers(1, 20)), int(rng.integers(1, 12))
        cells = [[x, y] for y in range(h) for x in range(w) if rng.random() < 0.35]
        text = R_IO.serialize_rle(w, h, cells)
        if rng.random() < 0.5:
            i = int(rng.integers(0, len(text)))
            text = text[:i] + str(rng.choice(list("ob$!2 \n#xq0"))) + text[i:]
        rle.append(text)
    plain = [".O.\n..O\nOOO", "OOO", "!block\nOO\nOO", ".O\nO\n\n..O", "OXO", "", "\n", "O\n",
             "!c\n!d", " O . O \t\n..", "..\r\nO.\r\n", "O.O\n!x\nO"]
    for _ in range(40):
        rows = ["".join(rng.choice(list("..O O\t"), int(rng.integers(0, 9)))) for _ in range(int(rng.integers(0, 6)))]
        t = "\n".join(rows)
        if rng.random() < 0.2:
            t += str(rng.choice(list("X*o#")))
        plain.append(t)
    ser = [(3, 1, [[0, 0], [1, 0], [2, 0]]), (1, 1, []), (3, 4, [[0, 0], [1, 0], [2, 0]]),
           (1, 4, [[0, 0], [0, 3]]), (2, 2, [[5, 0]]), (4, 4, [[3, 3], [0, 0], [0, 0], [1, 0]])]
    for _ in range(40):
        w, h = int(rng.integers(1, 32)), int(rng.integers(1, 32))
        ser.append((w, h, [[x, y] for y in range(h) for x in range(w) if rng.random() < 0.35]))
    grids = [(int(rng.integers(3, 80)), int(rng.integers(3, 12)), int(s)) for s in range(12)] + \
            [(35, 3, 99), (36, 4, 98), (70, 3, 97), (71, 3, 96)]
    return rle, plain, ser, grids


def io() -> None:
    global R_IO
    from oracle.oracle import REF_SO, PatternIO
    R_IO = PatternIO(REF_SO, "ref_")
    rle, plain, ser, grids = io_cases()
    res = {"rle": [{"text": t, "ref": R_IO.parse_rle(t)} for t in rle],
           "plaintext": [{"text": t, "ref": R_IO.parse_plaintext(t)} for t in plain],
           "serialize": [{"w": w, "h": h, "cells": c, "ref": R_IO.serialize_rle(w, h, c)}
                         for (w, h, c) in ser],
           "render": []}
    for (w, h, seed) in grids:
        g = O.random_fill(w, h, 0.4, seed)
        res["render"].append({"w": w, "h": h, "seed": seed, "ascii": R_IO.render("ascii", g),
                              "pbm": R_IO.render("pbm", g)})
    dump("golden_io.json", res)


if __name__ == "__main__":
    for stage in sys.argv[1:] or ["small"]:
        print("stage", stage, flush=True)
        t0 = time.time()
        globals()[stage]()
        print(f"stage {stage} done in {time.time() - t0:.0f}s", flush=True)
