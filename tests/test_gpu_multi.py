"""Multi-device contexts (life_ctx_create_multi): the torus in row bands over
several GPUs inside one run() call, the reference's Strategy::rows() over
workers (engine.cpp:162-214, band_bounds decomposition.cpp:12-24).

Every test puts all bands on cuda:0 (repeated device ids): the same events,
peer-mode edge kernels and copy halos run, but no kernel ever waits on
another GPU.  Bit-exact against the oracle and the reference-generated
golden fixtures.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden
from paper_1209_4408_b200 import capi, life

pytestmark = pytest.mark.gpu

PACKED, BYTE, RES = capi.ENGINE_PACKED, capi.ENGINE_BYTE, capi.ENGINE_RESIDENT


def fnv(oracle, a) -> str:
    return f"{oracle.fnv1a64(np.ascontiguousarray(a)):016x}"


@pytest.fixture(params=[capi.HALO_PEER, capi.HALO_COPY], ids=["peer", "copy"])
def halo(request):
    return request.param


def multi(n: int, halo_mode: int = capi.HALO_PEER) -> life.Engine:
    e = life.Engine(devices=[0] * n)
    e.set_option(capi.OPT_HALO, halo_mode)
    return e


@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_bands_match_oracle_small(oracle, halo, n):
    """Random shapes, depths 1..16 and checkpoint splits (deeper pass after a
    shallower one and back): grid and uint64 populations equal the oracle."""
    rng = np.random.default_rng(100 + n)
    with multi(n, halo) as e:
        for case in range(6):
            w = int(rng.integers(3, 300))
            h = int(rng.integers(max(3, n), 200))
            g = oracle.random_fill(w, h, 0.35, int(rng.integers(1 << 30)))
            gens = int(rng.integers(0, 60))
            depth = int(rng.integers(0, 17))
            cps = sorted({0, gens, *[int(x) for x in rng.integers(0, gens + 1, 3)]})
            want, pops = oracle.run(g, gens, cps)
            e.upload(g)
            got_pops = e.run(gens, PACKED, depth, cps)
            assert np.array_equal(e.download(), want), (w, h, gens, depth, n)
            assert got_pops == pops


def test_band_layout_and_errors():
    with multi(3) as e:
        e.init_random(100, 12289 // 8 * 8 + 1, 0.5, 1)
        b = e.bands()
        assert b["devices"] == [0, 0, 0]
        assert b["bounds"] == life.band_bounds(12289 // 8 * 8 + 1, 3)
        with pytest.raises(life.ConfigError):
            e.run(1, BYTE, 1)
        with pytest.raises(life.ConfigError):
            e.run(1, RES, 0)
        with pytest.raises(life.ConfigError):
            e.set_stream(None)
        with pytest.raises(life.ConfigError):
            e.run(-1)
    with multi(5) as e:
        with pytest.raises(life.TooManyParts):  # partition_rows: 5 bands of a 4-row torus
            e.upload(np.zeros((4, 10), np.uint8))
    with pytest.raises(life.NoDevice):
        life.Engine(devices=[0, 999])


def test_thin_bands_cap_the_depth(oracle):
    """Bands thinner than the requested depth (band_bounds(20, 8): 3 and 2 rows)."""
    g = oracle.random_fill(64, 20, 0.4, 5)
    want, _ = oracle.run(g, 50)
    for halo_mode in (capi.HALO_PEER, capi.HALO_COPY):
        with multi(8, halo_mode) as e:
            e.upload(g)
            e.run(50, PACKED, 16)
            assert np.array_equal(e.download(), want)


def test_io_across_bands(oracle):
    """upload/download (bytes and packed), windows crossing band seams and the
    torus wrap, place_pattern across a seam, population and grid hash equal a
    single-device context."""
    W, H = 333, 101
    g = oracle.random_fill(W, H, 0.45, 77)
    g[3, 5] = 7  # nonzero = alive
    with life.Engine(0) as one, multi(4) as four:
        for e in (one, four):
            e.upload(g)
            e.run(13, PACKED, 5)
            e.place(np.ones((9, 4), np.uint8), 100, 21)  # rows 21..29 cross the seam at 26
        assert np.array_equal(one.download(), four.download())
        assert np.array_equal(one.download_packed(), four.download_packed())
        assert one.population() == four.population()
        assert one.hash() == four.hash()
        for (x0, y0, w, h) in [(0, 0, W, H), (-7, -9, 40, 60), (300, 90, 50, 30),
                               (10, 20, 5, 250)]:
            assert np.array_equal(one.window(x0, y0, w, h), four.window(x0, y0, w, h))
        words = one.download_packed()
        four.upload_packed(words, W)
        assert np.array_equal(four.download(), one.download())


def test_band_stats_profile(oracle):
    with multi(3) as e:
        e.set_option(capi.OPT_PROFILE, 1)
        e.init_random(4096, 3000, 0.4, 3)
        e.run(64, PACKED, 16)
        st = e.band_stats()
        assert [s["rows"] for s in st] == [1000, 1000, 1000]
        for s in st:
            assert s["passes"] == 4
            assert s["run_ms"] > 0 and s["interior_ms"] > 0 and s["edge_ms"] > 0
            assert s["interior_ms"] <= s["run_ms"] * 1.01


def test_run_batch_multi(oracle, halo):
    W, H, G = 1000, 777, 37
    grids = [oracle.random_fill(W, H, 0.3 + 0.1 * i, i) for i in range(5)]
    ins = [oracle.pack(g) for g in grids]
    outs = [np.zeros_like(p) for p in ins]
    with multi(3, halo) as e:
        ms = e.run_batch(ins, outs, W, G, 8)
        assert ms > 0
        for g, out in zip(grids, outs):
            want, _ = oracle.run(g, G)
            assert np.array_equal(oracle.unpack(out, W), want)
        e.run_batch(ins, ins, W, G, 16)  # in place
        for g, out in zip(grids, ins):
            want, _ = oracle.run(g, G)
            assert np.array_equal(oracle.unpack(out, W), want)


@pytest.mark.slow
@pytest.mark.parametrize("n", [2, 3, 8])
def test_cfg4_bands_golden(oracle, n):
    """Config 4 (12289 x 40961, 1537 + 7 x 1536 rows at n = 8) at the engine's auto
    depth against the reference's hashes at 0/1/100/1000/5000."""
    gold = load_golden("golden_cfg4.json")
    soup = oracle.sparse_soup(40961, 12289, seed=42)
    with multi(n) as e:
        e.upload(soup)
        if n == 8:
            assert np.diff(e.bands()["bounds"]).tolist() == [1537] + [1536] * 7
        done = 0
        for gen in sorted(int(k) for k in gold["gens"]):
            e.run(gen - done, PACKED, 0)
            done = gen
            want = gold["gens"][str(gen)]
            assert fnv(oracle, e.download_packed()) == want["fnv_packed"], (n, gen)
            assert e.population() == want["population"]


@pytest.mark.slow
@pytest.mark.parametrize("n,halo_mode", [(2, capi.HALO_PEER), (3, capi.HALO_PEER),
                                         (8, capi.HALO_PEER), (8, capi.HALO_COPY)])
def test_cfg5_band_seam_windows(oracle, n, halo_mode):
    """Config 5 (262144^2, p = 0.4, 500 generations) as n bands: the reference's
    light-cone windows, including every P = 2/4/8 band seam and both wrap corners."""
    gold = load_golden("golden_cfg5_windows.json")
    with multi(n, halo_mode) as e:
        e.init_random(262144, 262144, 0.4, 42)
        e.run(16, PACKED, 16)
        for w in gold["windows_16"]:
            assert fnv(oracle, e.window(w["x0"], w["y0"], w["S"], w["S"])) == w["fnv_bytes"]
        e.run(500 - 16, PACKED, 16)
        for w in gold["windows_500"]:
            assert fnv(oracle, e.window(w["x0"], w["y0"], w["S"], w["S"])) == w["fnv_bytes"], w


def test_cfg1_checkpoint_populations_multi():
    """Config 1 populations at 0/1/10/100 through 4 bands (RunStats parity at N > 1);
    SURVEY 8(c)'s values, computed with the reference."""
    with multi(4) as e:
        e.init_random(1024, 1024, 0.5, 42)
        assert e.run(100, PACKED, 0, [0, 1, 10, 100]) == [524027, 286720, 211733, 98161]
