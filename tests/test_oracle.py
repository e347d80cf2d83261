"""Pins the oracle restatement (oracle/life_oracle.c) before it is trusted:
against the reference's own known-answer vectors, against the committed
golden fixtures generated from the reference (tests/golden/make_golden.py),
and -- when oracle/_ref is built -- against the reference library directly."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden

# proj/tests/test_rng.cpp:15-30
SPLITMIX_VECTORS = {
    0: [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC],
    1: [0x910A2DEC89025CC1, 0xBEEB8DA1658EEC67, 0xF893A2EEFB32555E, 0x71C18690EE42C90B],
    42: [0xBDD732262FEB6E95, 0x28EFE333B266F103, 0x47526757130F9F52, 0x581CE1FF0E4AE394],
    0xDEADBEEF: [0x4ADFB90F68C9EB9B, 0xDE586A3141A10922, 0x021FBC2F8E1CFC1D, 0x7466CE737BE16790],
}
# proj/tests/test_rng.cpp:43-45
NEXT_UNIT_42 = [0.74156487877182331, 0.1599103928769201, 0.27860113025513866,
                0.34419071652363753, 0.038030168540246212, 0.86822807654653233]


def test_splitmix_vectors(oracle):
    for seed, expected in SPLITMIX_VECTORS.items():
        assert [int(v) for v in oracle.splitmix(seed, 4)] == expected


def test_next_unit_threshold_form(oracle):
    # random_fill's `next_unit() < p` is restated as `(next() >> 11) < ceil(p*2^53)`.
    draws = oracle.splitmix(42, 6)
    units = [float(int(d) >> 11) * 2.0 ** -53 for d in draws]
    assert units == NEXT_UNIT_42
    rng = np.random.default_rng(0)
    ds = np.concatenate([rng.random(200), [0.0, 1.0, 0.5, 0.3, 0.4, 2.0 ** -53, 1 - 2.0 ** -53]])
    for p in ds:
        thr = oracle.threshold(float(p))
        for d in oracle.splitmix(int(p * 1e9), 64):
            m = int(d) >> 11
            assert (m * 2.0 ** -53 < p) == (m < thr)


def test_golden_small_fixture_matches_known_answers(golden_small):
    assert [int(v, 16) for v in golden_small["splitmix"]["0"][:4]] == SPLITMIX_VECTORS[0]
    assert [float(v) for v in golden_small["next_unit_42"]] == NEXT_UNIT_42
    # B3/S23 truth table (test_grid.cpp:77-93)
    assert golden_small["truth_table"]["alive"] == [n in (2, 3) for n in range(9)]
    assert golden_small["truth_table"]["dead"] == [n == 3 for n in range(9)]
    assert all(golden_small["glider_lap"]["translated_each_cycle"])
    assert golden_small["glider_lap"]["home_after_64"]


def test_cfg1_goldens(oracle, golden_small):
    # populations 524027/286720/211733/98161 and FNV-1a-64.
    g = oracle.random_fill(1024, 1024, 0.5, 42)
    assert oracle.fnv1a64(g) == 0xE8E151C80A332F86
    out, pops = oracle.run(g, 100, [0, 1, 10, 100])
    assert pops == [524027, 286720, 211733, 98161]
    assert oracle.fnv1a64(out) == 0x37B6D88FF40A4F22
    cfg1 = golden_small["cfg1"]
    for gen, pop in zip([0, 1, 10, 100], pops):
        assert cfg1[str(gen)]["population"] == pop
    assert cfg1["100"]["fnv_bytes"] == "37b6d88ff40a4f22"
    assert int(cfg1["100"]["fnv_packed"], 16) == oracle.fnv1a64(oracle.pack(out))


def test_small_cases_against_reference_goldens(oracle, golden_small):
    for case in golden_small["small_cases"]:
        g = oracle.random_fill(case["w"], case["h"], case["density"], case["seed"])
        assert f"{oracle.fnv1a64(g):016x}" == case["initial"]["fnv_bytes"]
        out, pops = oracle.run(g, case["gens"], [0, case["gens"]] if case["gens"] else [0])
        assert f"{oracle.fnv1a64(out):016x}" == case["final"]["fnv_bytes"], case
        assert f"{oracle.fnv1a64(oracle.pack(out)):016x}" == case["final"]["fnv_packed"]
        assert pops[-1] == case["final"]["population"]


def test_step_serial_equals_region_engine(oracle):
    for seed in range(6):
        g = oracle.random_fill(3 + seed * 7, 3 + seed * 5, 0.35, seed)
        a = oracle.run_serial(g, 9)
        b, _ = oracle.run(g, 9)
        assert np.array_equal(a, b)


def test_glider_lap(oracle):
    # test_grid.cpp:207-217: glider `bo$2bo$3o!` at (6,6) on 16x16
    g = np.zeros((16, 16), np.uint8)
    for (x, y) in [(1, 0), (2, 1), (0, 2), (1, 2), (2, 2)]:
        g[6 + y, 6 + x] = 1
    cur = g
    for cycle in range(1, 17):
        cur, _ = oracle.run(cur, 4)
        assert np.array_equal(cur, np.roll(np.roll(g, cycle, 0), cycle, 1))
    assert np.array_equal(cur, g)


def test_pack_roundtrip(oracle):
    rng = np.random.default_rng(1)
    for w in (3, 31, 32, 33, 63, 64, 65, 127, 129, 1000):
        g = (rng.random((7, w)) < 0.5).astype(np.uint8)
        p = oracle.pack(g)
        assert p.shape == (7, (w + 63) // 64)
        assert np.array_equal(oracle.unpack(p, w), g)
        tail = w % 64
        if tail:
            assert not np.any(p[:, -1] >> np.uint64(tail))


def test_random_window_matches_fill(oracle):
    g = oracle.random_fill(97, 61, 0.4, 5)
    for (x0, y0, w, h) in [(0, 0, 97, 61), (-5, -7, 20, 30), (90, 55, 30, 20), (-200, 300, 11, 9)]:
        win = oracle.random_window(97, 61, 0.4, 5, x0, y0, w, h)
        ys = (np.arange(h) + y0) % 61
        xs = (np.arange(w) + x0) % 97
        assert np.array_equal(win, g[np.ix_(ys, xs)])


def test_lightcone_window(oracle):
    # the central S x S of an (S+2T)^2 window run as its own
    # torus for T generations equals the full-torus result.
    W, H, S, T = 300, 260, 40, 25
    g = oracle.random_fill(W, H, 0.4, 11)
    full, _ = oracle.run(g, T)
    for (x0, y0) in [(0, 0), (280, 250), (150, 3), (17, 130)]:
        init = oracle.random_window(W, H, 0.4, 11, x0 - T, y0 - T, S + 2 * T, S + 2 * T)
        centre = oracle.lightcone(init, S, T)
        ys = (np.arange(S) + y0) % H
        xs = (np.arange(S) + x0) % W
        assert np.array_equal(centre, full[np.ix_(ys, xs)])


def test_band_bounds_golden(oracle, golden_small):
    for key, cuts in golden_small["partition_rows"].items():
        h, p = map(int, key.split("/"))
        assert oracle.band_bounds(h, p) == cuts
    with pytest.raises(ValueError):
        oracle.band_bounds(5, 6)


def test_sparse_soup_golden(oracle, golden_small):
    for case in golden_small["soup_small"]:
        g = oracle.sparse_soup(case["w"], case["h"], seed=case["seed"])
        assert f"{oracle.fnv1a64(g):016x}" == case["fnv_bytes"]


# ---- direct cross-checks against the reference library (CPU container) ----

def test_oracle_vs_reference_random(oracle, reference):
    for (w, h, p, s) in [(1000, 37, 0.3, 1), (64, 64, 0.5, 42), (33, 17, 0.0, 3), (33, 17, 1.0, 3)]:
        assert np.array_equal(oracle.random_fill(w, h, p, s), reference.random_fill(w, h, p, s))


def test_oracle_vs_reference_run(oracle, reference):
    for seed in range(5):
        w, h = 3 + seed * 13, 4 + seed * 9
        g = oracle.random_fill(w, h, 0.4, seed)
        a, pa = oracle.run(g, 23, [0, 5, 23])
        b, pb, gens = reference.run(g, 23, "rows", 3 if h >= 3 else 1, checkpoints=[0, 5, 23])
        assert np.array_equal(a, b) and pa == pb and gens == 23


def test_reference_nonbinary_bytes_divergence_is_pinned(oracle, reference):
    # step_serial treats any nonzero byte as alive; the
    # engine's contract normalises nonzero -> 1 (step_serial semantics).
    g = oracle.random_fill(20, 20, 0.4, 9)
    g2 = g.copy()
    g2[3, 3] = 2
    g2[10, 11] = 255
    assert np.array_equal(reference.step_serial(g2), oracle.step_serial((g2 != 0).astype(np.uint8)))


def test_place_pattern_vs_reference(oracle, reference):
    rng = np.random.default_rng(5)
    for _ in range(30):
        w, h = int(rng.integers(3, 40)), int(rng.integers(3, 40))
        g = (rng.random((h, w)) < 0.5).astype(np.uint8)
        pw, ph = int(rng.integers(0, w + 1)), int(rng.integers(0, h + 1))
        pat = (rng.random((ph, pw)) < 0.4).astype(np.uint8)
        x0, y0 = int(rng.integers(0, w - pw + 1)), int(rng.integers(0, h - ph + 1))
        assert np.array_equal(oracle.place_pattern(g, pat, x0, y0),
                              reference.place_pattern(g, pat, x0, y0))
    with pytest.raises(IndexError):
        oracle.place_pattern(np.zeros((5, 5), np.uint8), np.ones((3, 3), np.uint8), 3, 0)
    with pytest.raises(RuntimeError):
        reference.place_pattern(np.zeros((5, 5), np.uint8), np.ones((3, 3), np.uint8), 3, 0)


def test_grid_hash_definition(oracle):
    """life_grid_hash's definition (checksum of packed-row FNV-1a-64 checksums)
    restated in pure Python on small grids, including a tail word."""
    import numpy as np

    def fnv(bs, h=0xcbf29ce484222325):
        for b in bs:
            h = ((h ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
        return h
    for (w, h, seed) in [(3, 3, 1), (64, 5, 2), (65, 7, 3), (130, 4, 4)]:
        g = oracle.random_fill(w, h, 0.5, seed)
        words = oracle.pack(g)
        rows = b"".join(fnv(words[y].tobytes()).to_bytes(8, "little") for y in range(h))
        assert oracle.grid_hash(g) == fnv(rows) == oracle.packed_hash(words)
    # any single-cell change changes it
    g = oracle.random_fill(100, 9, 0.5, 5)
    g2 = g.copy()
    g2[4, 77] ^= 1
    assert oracle.grid_hash(g) != oracle.grid_hash(g2)
