"""GPU parity: the CUDA engine through the C-ABI vs the oracle and the
reference-generated golden fixtures.  Bit-exact (integer work).

Run on a B200:  python -m pytest tests -m gpu -x -q
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden
from paper_1209_4408_b200 import capi

pytestmark = pytest.mark.gpu

PACKED, BYTE = 0, 1


def fnv(oracle, a) -> str:
    return f"{oracle.fnv1a64(np.ascontiguousarray(a)):016x}"


def test_random_fill_on_device_matches_oracle(engine, oracle):
    for (w, h, p, s) in [(3, 3, 0.5, 1), (31, 7, 0.3, 2), (64, 5, 0.5, 3), (65, 9, 0.7, 4),
                         (1000, 37, 0.3, 5), (40961, 3, 0.02, 6), (97, 61, 0.0, 7),
                         (97, 61, 1.0, 8)]:
        want = oracle.random_fill(w, h, p, s)
        for eng in (PACKED, BYTE):
            engine.init_random(w, h, p, s, eng)
            assert np.array_equal(engine.download(), want), (w, h, p, s, eng)
            assert engine.population() == int(want.sum())


def test_upload_download_roundtrip_and_nonbinary_contract(engine, oracle):
    rng = np.random.default_rng(3)
    for (w, h) in [(3, 3), (17, 5), (33, 40), (129, 7), (1000, 13)]:
        g = rng.integers(0, 4, (h, w), dtype=np.uint8)  # nonzero bytes count as alive
        engine.upload(g)
        assert np.array_equal(engine.download(), (g != 0).astype(np.uint8))
        packed = engine.download_packed()
        assert np.array_equal(packed, oracle.pack(g != 0))
        engine.upload_packed(packed, w)
        assert np.array_equal(engine.download(), (g != 0).astype(np.uint8))
        # one step from a non-0/1 upload = step_serial semantics
        engine.upload(g)
        engine.step(BYTE)
        assert np.array_equal(engine.download(), oracle.step_serial(g))


def test_packed_upload_ignores_tail_bits(engine, oracle):
    g = oracle.random_fill(70, 9, 0.5, 1)
    p = oracle.pack(g)
    p[:, -1] |= np.uint64(0xFFFFFFFF) << np.uint64(32)  # garbage past column 70
    engine.upload_packed(p, 70)
    assert np.array_equal(engine.download(), g)
    engine.run(5, PACKED, 3)
    want, _ = oracle.run(g, 5)
    assert np.array_equal(engine.download(), want)


@pytest.mark.parametrize("eng,depth", [(PACKED, 1), (PACKED, 4), (PACKED, 7), (PACKED, 16),
                                       (BYTE, 1), (BYTE, 3), (BYTE, 8), (BYTE, 0)])
def test_small_golden_cases(engine, oracle, golden_small, eng, depth):
    for case in golden_small["small_cases"]:
        engine.init_random(case["w"], case["h"], case["density"], case["seed"], eng)
        pops = engine.run(case["gens"], eng, depth, [0, case["gens"]] if case["gens"] else [0])
        got = engine.download()
        assert fnv(oracle, got) == case["final"]["fnv_bytes"], (case, eng, depth)
        assert pops[-1] == case["final"]["population"]
        assert pops[0] == case["initial"]["population"]


def test_cfg1_full_grid_at_1_10_100(engine, oracle, golden_small):
    cfg1 = golden_small["cfg1"]
    for eng, depth in [(PACKED, 16), (PACKED, 5), (BYTE, 1), (BYTE, 4), (BYTE, 7)]:
        engine.init_random(1024, 1024, 0.5, 42, eng)
        pops = engine.run(100, eng, depth, [0, 1, 10, 100])
        assert pops == [524027, 286720, 211733, 98161]
        assert fnv(oracle, engine.download()) == "37b6d88ff40a4f22"
        for g in (1, 10, 100):
            engine.init_random(1024, 1024, 0.5, 42, eng)
            engine.run(g, eng, depth)
            out = engine.download()
            assert fnv(oracle, out) == cfg1[str(g)]["fnv_bytes"]
            assert fnv(oracle, engine.download_packed()) == cfg1[str(g)]["fnv_packed"]


def test_known_patterns(engine):
    from paper_1209_4408_b200 import life
    blinker = np.zeros((5, 5), np.uint8)
    blinker[2, 1:4] = 1
    block = np.zeros((6, 6), np.uint8)
    block[2:4, 2:4] = 1
    glider = np.zeros((16, 16), np.uint8)
    for (x, y) in [(1, 0), (2, 1), (0, 2), (1, 2), (2, 2)]:
        glider[6 + y, 6 + x] = 1
    for strat in (life.Strategy.gpu_packed(), life.Strategy.gpu_packed(3), life.Strategy.gpu_byte()):
        g = life.Grid.from_array(blinker)
        one = life.step_parallel(g, strat)
        assert one != g and life.step_parallel(one, strat) == g
        r = life.run(g, life.RunConfig(strat, 1, 100), [1, 2, 100])
        assert r.stats.population_checkpoints == [(1, 3), (2, 3), (100, 3)]
        assert r.grid == g
        b = life.Grid.from_array(block)
        assert life.run(b, life.RunConfig(strat, 1, 100)).grid == b
        gl = life.Grid.from_array(glider)
        for cycle in (1, 5, 16):
            got = life.run(gl, life.RunConfig(strat, 1, 4 * cycle)).grid
            assert np.array_equal(got.cells, np.roll(np.roll(glider, cycle, 0), cycle, 1))


def test_translation_commutes(engine, oracle):
    for seed in range(3):
        g = oracle.random_fill(133, 71, 0.3, seed)
        for (dx, dy) in [(1, 0), (0, 1), (3, 5), (-2, 4), (11, -7), (64, 33)]:
            t = np.roll(np.roll(g, dy, 0), dx, 1)
            engine.upload(t)
            engine.run(7, PACKED, 7)
            a = engine.download()
            engine.upload(g)
            engine.run(7, PACKED, 7)
            b = np.roll(np.roll(engine.download(), dy, 0), dx, 1)
            assert np.array_equal(a, b)


def test_depth_transparency_sweep(engine, oracle):
    # "strategy transparency" (test_engine.cpp:49-83) -> every temporal depth
    # and both engines give the same grid.
    for seed in range(4):
        w = 3 + (seed * 17 + 5) % 46 + seed * 37
        h = 3 + (seed * 29 + 11) % 46
        g = oracle.random_fill(w, h, 0.3, seed)
        want, _ = oracle.run(g, 41)
        for depth in range(1, 17):
            engine.upload(g)
            engine.run(41, PACKED, depth)
            assert np.array_equal(engine.download(), want), (seed, depth)
        for depth in range(1, 9):
            engine.upload(g)
            engine.run(41, BYTE, depth)
            assert np.array_equal(engine.download(), want), (seed, "byte", depth)


@pytest.mark.parametrize("w,h", [(128, 3), (128, 5), (256, 31), (1024, 97), (3968, 40),
                                 (4096, 300), (640, 1000)])
def test_single_generation_vector_path(engine, oracle, w, h):
    """Depth 1 with W % 128 == 0 takes packed_step1_kernel (16-byte vectors, ghost
    lanes, index-remap torus wrap): every generation bit-exact, incl. 3-row tori
    and more strips than one warp covers."""
    g = oracle.random_fill(w, h, 0.35, w + h)
    for gens in (1, 2, 7, 33):
        want, _ = oracle.run(g, gens)
        engine.upload(g)
        engine.run(gens, PACKED, 1)
        assert np.array_equal(engine.download(), want), (w, h, gens)


def test_checkpoints_split_passes(engine, oracle):
    g = oracle.random_fill(200, 150, 0.4, 9)
    cps = [0, 1, 3, 17, 18, 40, 64]
    _, want = oracle.run(g, 64, cps)
    for depth in (1, 4, 16):
        engine.upload(g)
        assert engine.run(64, PACKED, depth, cps) == want


def test_run_config_errors(engine):
    from paper_1209_4408_b200 import life
    g = life.Grid(8, 5)
    with pytest.raises(life.TooManyParts):
        life.run(g, life.RunConfig(life.Strategy.gpu_packed(), 10, 1))
    with pytest.raises(life.ConfigError):
        life.run(g, life.RunConfig(life.Strategy.gpu_packed(), 0, 1))
    with pytest.raises(life.ConfigError):
        life.run(g, life.RunConfig(life.Strategy.gpu_packed(), 1, -1))
    with pytest.raises(life.ConfigError):
        life.run(g, life.RunConfig(life.Strategy.gpu_packed(), 1, 2), [2, 1])
    with pytest.raises(life.ConfigError):
        life.run(g, life.RunConfig(life.Strategy.gpu_packed(), 1, 2), [3])
    with pytest.raises(life.DimensionTooSmall):
        engine.init_random(2, 5, 0.5, 1)
    with pytest.raises(life.ConfigError):
        engine.init_random(5, 5, 1.5, 1)
    engine.init_random(5, 5, 0.5, 1)
    with pytest.raises(life.ConfigError):
        engine.run(3, BYTE, 9)
    with pytest.raises(life.ConfigError):
        engine.run(3, PACKED, 17)
    r = life.run(g, life.RunConfig(life.Strategy.gpu_packed(), 1, 0), [0])
    assert r.grid == g and r.stats.generations_computed == 0


def test_windows_wrap(engine, oracle):
    g = oracle.random_fill(300, 200, 0.5, 4)
    for eng in (PACKED, BYTE):
        engine.upload(g)
        if eng == PACKED:
            engine.run(0, PACKED)
        for (x0, y0, w, h) in [(0, 0, 300, 200), (-7, -9, 40, 30), (290, 195, 33, 17),
                               (-1000, 1000, 5, 5)]:
            ys = (np.arange(h) + y0) % 200
            xs = (np.arange(w) + x0) % 300
            assert np.array_equal(engine.window(x0, y0, w, h), g[np.ix_(ys, xs)])


# ---- BASELINE.json configs ----------------------------------------------

def _check_schedule(engine, oracle, gold, eng, depth, init):
    init()
    done = 0
    for gen in sorted(int(k) for k in gold["gens"]):
        engine.run(gen - done, eng, depth)
        done = gen
        want = gold["gens"][str(gen)]
        assert fnv(oracle, engine.download_packed()) == want["fnv_packed"], (eng, depth, gen)
        assert engine.population() == want["population"]


@pytest.mark.slow
def test_cfg2_16384_1000_generations(engine, oracle):
    gold = load_golden("golden_cfg2.json")
    # depth 0 = what life_run / bench.py run: byte auto K=8, packed auto = the
    # pair layout at K=10 (2^27 cells or more; plain K=16 with an explicit depth)
    import ctypes as C
    d = C.c_int32(0)
    assert capi.lib().life_interleave_auto(16384, 16384, -1, -1, 0, C.byref(d)) == 2 and d.value == 10
    assert capi.lib().life_packed_auto_depth(16384, 16384) == 16
    for eng, depth in [(BYTE, 1), (BYTE, 4), (BYTE, 0), (BYTE, 6), (PACKED, 16), (PACKED, 8),
                       (PACKED, 0)]:
        _check_schedule(engine, oracle, gold, eng, depth,
                        lambda: engine.init_random(16384, 16384, 0.3, 42, eng))


@pytest.mark.slow
@pytest.mark.parametrize("depth", [1, 4, 8, 16])
def test_cfg3_65536_packed_depths(engine, oracle, depth):
    gold = load_golden("golden_cfg3.json")
    _check_schedule(engine, oracle, gold, PACKED, depth,
                    lambda: engine.init_random(65536, 65536, 0.5, 42, PACKED))


@pytest.mark.slow
def test_cfg3_windows(engine, oracle):
    gold = load_golden("golden_cfg3_windows.json")
    engine.init_random(65536, 65536, 0.5, 42, PACKED)
    engine.run(100, PACKED, 16)
    for w in gold["windows_100"]:
        got = engine.window(w["x0"], w["y0"], w["S"], w["S"])
        assert fnv(oracle, got) == w["fnv_bytes"], w


@pytest.mark.slow
def test_cfg4_nonpow2_sparse_soup(engine, oracle):
    gold = load_golden("golden_cfg4.json")
    soup = oracle.sparse_soup(40961, 12289, seed=42)
    # depth 0 = the engine's auto rule: K = 12 on this one-wave W % 32 != 0 torus
    assert capi.lib().life_packed_auto_depth(40961, 12289) == 12
    assert capi.lib().life_packed_launch_kind(40961, 12289, 12) == capi.LAUNCH_ALL_PATHS
    # BYTE 0 / 8: the two-stream byte kernel's seam path (W % 16 == 1)
    for eng, depth in [(BYTE, 1), (BYTE, 0), (BYTE, 8), (PACKED, 16), (PACKED, 0), (PACKED, 12)]:
        _check_schedule(engine, oracle, gold, eng, depth, lambda: engine.upload(soup))


@pytest.mark.parametrize("W", [33, 40, 47, 50, 100, 127, 1000, 1001, 2047, 2049])
def test_byte_passes_on_widths_not_multiple_of_16(engine, oracle, W):
    """Temporal-blocked byte passes on W % 16 != 0 tori: the seam lanes build
    their 16 columns from two or three vectors of the row (byte_seam_plan),
    the partial last vector keeps its bytes past W zero; equal to the oracle
    for depths 2..8, remainders and checkpoint splits."""
    rng = np.random.default_rng(W)
    H = int(rng.integers(20, 90))
    g = oracle.random_fill(W, H, 0.35, int(rng.integers(1 << 30)))
    gens = 29
    want, pops = oracle.run(g, gens, [0, 11, gens])
    for depth in (2, 3, 5, 8, 0):
        engine.upload(g)
        got_pops = engine.run(gens, BYTE, depth, [0, 11, gens])
        assert np.array_equal(engine.download(), want), (W, H, depth)
        assert got_pops == pops


@pytest.mark.slow
@pytest.mark.parametrize("shape", ["65535x65535", "131071x65536", "2975x700000", "2049x700000"])
def test_split_launch_reference_windows(engine, oracle, shape):
    """W % 32 != 0 tori that take the split launch (seam strips on the
    all-paths kernel beside the fast-only kernel) against light-cone windows
    the REFERENCE computed (make_golden.py split): column seam, both wrap
    corners, the fast/seam strip boundary, nw % 31 == 0 (three seam strips)
    and W % 32 == 1."""
    gold = load_golden("golden_split_windows.json")[shape]
    W, H, T = gold["w"], gold["h"], gold["T"]
    for depth in (0, 16, 11):
        k = depth or capi.lib().life_packed_auto_depth(W, H)
        assert capi.lib().life_packed_launch_kind(W, H, k) == capi.LAUNCH_SPLIT, (shape, k)
        engine.init_random(W, H, gold["density"], gold["seed"], PACKED)
        engine.run(T, PACKED, depth)
        for w in gold["windows"]:
            got = engine.window(w["x0"], w["y0"], w["S"], w["S"])
            assert fnv(oracle, got) == w["fnv_bytes"], (shape, depth, w)
            assert int(got.sum()) == w["population"]


@pytest.mark.slow
def test_cfg5_lightcone_windows(engine, oracle):
    gold = load_golden("golden_cfg5_windows.json")
    W = H = 262144
    engine.init_random(W, H, 0.4, 42, PACKED)
    engine.run(16, PACKED, 16)
    for w in gold["windows_16"]:
        assert fnv(oracle, engine.window(w["x0"], w["y0"], w["S"], w["S"])) == w["fnv_bytes"]
    engine.run(500 - 16, PACKED, 16)
    for w in gold["windows_500"]:
        assert fnv(oracle, engine.window(w["x0"], w["y0"], w["S"], w["S"])) == w["fnv_bytes"], w


def test_run_batch_pipelined(engine, oracle):
    """life_run_batch: every grid of the stream equals the oracle run; outputs may alias inputs."""
    W, H, G = 1000, 77, 37
    grids = [oracle.random_fill(W, H, 0.3 + 0.1 * i, i) for i in range(5)]
    ins = [oracle.pack(g) for g in grids]
    outs = [np.zeros_like(p) for p in ins]
    ms = engine.run_batch(ins, outs, W, G, 8)
    assert ms > 0
    for g, out in zip(grids, outs):
        want, _ = oracle.run(g, G)
        assert np.array_equal(oracle.unpack(out, W), want)
    engine.run_batch(ins, ins, W, G, 16)  # in-place
    for g, out in zip(grids, ins):
        want, _ = oracle.run(g, G)
        assert np.array_equal(oracle.unpack(out, W), want)


@pytest.mark.parametrize("W,H,G,depth", [(1000, 2100, 37, 8), (333, 2051, 41, 16),
                                         (2048, 600, 16, 16), (96, 4099, 0, 16), (640, 1030, 5, 3),
                                         (96, 33001, 37, 8), (100, 40000, 20, 16),
                                         (64, 32768, 48, 16), (200, 36000, 1, 1),
                                         (1024, 33000, 5, 1), (64, 80000, 48, 16),
                                         (96, 66000, 37, 8)])
def test_run_batch_banded(engine, oracle, W, H, G, depth):
    """life_run_batch on taller grids: several waves of row tiles per pass, W % 32 != 0,
    G not a multiple of the depth, G = 0, more grids than buffer slots; H >= 32768 runs
    the first and last grid as 32 chunk trapezoids + boundary triangles (forced with
    LIFE_OPT_BATCH_TRAPEZOID=1: by default only chunks of >= 8192 rows take it)."""
    if H >= 32768:
        engine.set_option(capi.OPT_BATCH_TRAPEZOID, 1)
    try:
        _run_batch_banded(engine, oracle, W, H, G, depth)
    finally:
        engine.set_option(capi.OPT_BATCH_TRAPEZOID, -1)


def _run_batch_banded(engine, oracle, W, H, G, depth):
    grids = [oracle.random_fill(W, H, 0.35, 100 + i) for i in range(3)]
    ins = [oracle.pack(g) for g in grids]
    outs = [np.zeros_like(p) for p in ins]
    engine.run_batch(ins, outs, W, G, depth)
    for g, out in zip(grids, outs):
        want, _ = oracle.run(g, G)
        assert np.array_equal(oracle.unpack(out, W), want)
    if H >= 32768:  # trapezoid schedule in place: outputs alias inputs
        engine.run_batch(ins, ins, W, G, depth)
        for g, out in zip(grids, ins):
            want, _ = oracle.run(g, G)
            assert np.array_equal(oracle.unpack(out, W), want)


def test_device_soup_matches_oracle(engine, oracle):
    for (w, h, cov, bs, p, seed) in [(200, 150, 0.02, 5, 0.5, 3), (409, 121, 0.02, 5, 0.5, 42),
                                     (97, 61, 0.3, 5, 0.5, 7), (64, 64, 0.5, 3, 0.7, 1),
                                     (33, 40, 1.0, 7, 0.5, 9), (10, 10, 0.0, 5, 0.5, 1)]:
        want = oracle.sparse_soup(w, h, seed=seed, coverage=cov, block=bs, p=p)
        for eng in (PACKED, BYTE):
            engine.init_soup(w, h, cov, bs, p, seed, eng)
            assert np.array_equal(engine.download(), want), (w, h, cov, bs, p, seed, eng)


@pytest.mark.slow
def test_device_soup_cfg4_golden(engine, oracle):
    gold = load_golden("golden_cfg4.json")
    engine.init_soup(40961, 12289, 0.02, 5, 0.5, 42, PACKED)
    assert fnv(oracle, engine.download_packed()) == gold["gens"]["0"]["fnv_packed"]
    engine.run(100, PACKED, 16)
    assert fnv(oracle, engine.download_packed()) == gold["gens"]["100"]["fnv_packed"]


def test_device_place_pattern(engine, oracle):
    from paper_1209_4408_b200 import life
    rng = np.random.default_rng(11)
    for trial in range(12):
        w, h = int(rng.integers(3, 300)), int(rng.integers(3, 60))
        g = (rng.random((h, w)) < 0.5).astype(np.uint8)
        pw, ph = int(rng.integers(0, min(w, 70) + 1)), int(rng.integers(0, h + 1))
        pat = rng.integers(0, 3, (ph, pw)).astype(np.uint8)
        x0, y0 = int(rng.integers(0, w - pw + 1)), int(rng.integers(0, h - ph + 1))
        want = oracle.place_pattern(g, pat, x0, y0)
        for eng in (PACKED, BYTE):
            engine.upload(g)
            if eng == PACKED:
                engine.run(0, PACKED)  # resident layout -> packed
            engine.place(pat, x0, y0)
            assert np.array_equal(engine.download(), want), (trial, eng)
    engine.upload(np.zeros((5, 5), np.uint8))
    with pytest.raises(life.OutOfBounds):
        engine.place(np.ones((3, 3), np.uint8), 3, 0)


def test_grid_hash_matches_oracle(engine, oracle):
    for (w, h, p, s) in [(3, 3, 0.5, 1), (64, 9, 0.4, 2), (1000, 37, 0.3, 3), (4096, 64, 0.5, 4)]:
        g = oracle.random_fill(w, h, p, s)
        for eng in (PACKED, BYTE):
            engine.upload(g)
            engine.run(3, eng, 0)
            want, _ = oracle.run(g, 3)
            assert engine.hash() == oracle.grid_hash(want), (w, h, eng)


def test_random_shape_fuzz_all_engines(engine, oracle):
    """Seeded fuzz over shapes, engines and depths (packed K = 0..16, byte
    K = 0..8, resident where it fits), including word-boundary widths and
    3-row tori: every case bit-exact against the oracle."""
    from paper_1209_4408_b200 import capi
    rng = np.random.default_rng(20261020)
    RES = 2
    widths = [3, 5, 31, 32, 33, 63, 64, 65, 95, 96, 127, 128, 129, 160, 255, 256, 257, 1000, 1024]
    for case in range(160):
        w = int(rng.choice(widths)) if case % 2 else int(rng.integers(3, 400))
        h = int(rng.integers(3, 90))
        gens = int(rng.integers(0, 60))
        g = oracle.random_fill(w, h, float(rng.uniform(0.1, 0.7)), case)
        want, _ = oracle.run(g, gens)
        kind = case % 3
        if kind == 0:
            eng, depth = PACKED, int(rng.integers(0, 17))
        elif kind == 1:
            eng, depth = BYTE, int(rng.integers(0, 9))
        else:
            eng, depth = (RES, 0) if capi.lib().life_resident_cluster_size(w, h) else (PACKED, 0)
        engine.upload(g)
        engine.run(gens, eng, depth)
        assert np.array_equal(engine.download(), want), (case, w, h, gens, eng, depth)


@pytest.mark.slow
def test_split_launch_seam_strips(engine):
    """W % 32 != 0 tori several block waves deep run the seam strips on the
    all-paths kernel beside the fast-only kernel (launch_packed's split):
    its grid hash equals depth 2 (no split, no fast kernel) and the byte
    engine (an independent implementation)."""
    W, H, G = 2001, 700000, 32  # 3 strips x 700000 rows: over the split threshold
    hashes = []
    for eng, depth in [(PACKED, 16), (PACKED, 2), (BYTE, 1)]:
        engine.init_random(W, H, 0.4, 2026, eng)
        engine.run(G, eng, depth)
        hashes.append(engine.hash())
    assert hashes[0] == hashes[1] == hashes[2]
