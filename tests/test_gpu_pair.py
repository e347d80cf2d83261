"""GPU parity of the interleaved-layout packed kernels (kernels_pair.cuh: the
pair layout, W % 64 == 0 tori, LIFE_OPT_PAIR_DEPTH; the quad layout, W % 128
== 0, LIFE_OPT_QUAD_DEPTH) against the oracle and the reference goldens, and
of the lazy layout conversion around them.  Bit-exact (integer work).

Run on a B200:  python -m pytest tests/test_gpu_pair.py -m gpu -x -q
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden
from paper_1209_4408_b200 import capi, life

pytestmark = pytest.mark.gpu

PACKED, BYTE = 0, 1

# (interleave order, option, deepest pass): widths below are given in pair
# groups (64 columns) and scaled to the layout's group width.
PAIR = (2, capi.OPT_PAIR_DEPTH, capi.PAIR_MAX_DEPTH)
QUAD = (4, capi.OPT_QUAD_DEPTH, capi.QUAD_MAX_DEPTH)


@pytest.fixture()
def pair_engine():
    e = life.Engine(0)
    yield e
    e.close()


def fnv(oracle, a) -> str:
    return f"{oracle.fnv1a64(np.ascontiguousarray(a)):016x}"


# ng = W / 64 groups: 1 (every lane the same group), 2, 3, 30/31/32 (the strip
# boundary: 31 groups per strip), 33, 62/63 (two strips), 100.
SHAPES = [(64, 3), (64, 40), (128, 33), (192, 100), (1920, 50), (1984, 77), (2048, 64),
          (2112, 9), (3968, 41), (4032, 130), (6400, 23)]


@pytest.mark.parametrize("layout,depth", [(PAIR, d) for d in (1, 2, 3, 5, 8, 10, 12)] +
                         [(QUAD, d) for d in (1, 2, 3, 4, 5, 6, 7)],
                         ids=lambda v: v if isinstance(v, int) else f"order{v[0]}")
def test_pair_depths_match_oracle(pair_engine, oracle, layout, depth):
    e = pair_engine
    il, opt, _ = layout
    e.set_option(opt, depth)
    for i, (w, h) in enumerate(SHAPES):
        w = w * il // 2
        g = oracle.random_fill(w, h, 0.37, 100 + i)
        gens = 2 * depth + 3  # two full passes and a remainder pass
        e.upload(g)
        pops = e.run(gens, PACKED, 0, [0, depth, gens])
        want, wpops = oracle.run(g, gens, [0, depth, gens])
        assert np.array_equal(e.download(), want), (w, h, depth)
        assert list(pops) == list(wpops), (w, h, depth)


@pytest.mark.parametrize("layout", [PAIR, QUAD], ids=["pair", "quad"])
def test_pair_layout_is_transparent_between_calls(pair_engine, oracle, layout):
    """life_run leaves the grid in the pair / quad layout; every reader of the
    plain layout (download, window, hash, place, population, the other
    engines) converts it back first."""
    e = pair_engine
    il, opt, max_depth = layout
    e.set_option(opt, 7 if il == 2 else 5)
    w, h = 2048, 300
    g = oracle.random_fill(w, h, 0.4, 9)
    e.upload(g)
    e.run(20, PACKED, 0)
    want, _ = oracle.run(g, 20)
    assert e.population() == int(want.sum())            # popcount is layout-invariant
    e.run(8, PACKED, 0)                                  # stays in the pair layout
    want, _ = oracle.run(want, 8)
    assert np.array_equal(e.window(2040, 295, 20, 12),
                          np.take(np.take(want, np.arange(295, 307) % h, axis=0),
                                  np.arange(2040, 2060) % w, axis=1))
    e.run(5, PACKED, 0)
    want, _ = oracle.run(want, 5)
    assert e.hash() == oracle.grid_hash(want)
    e.run(3, PACKED, 0)
    want, _ = oracle.run(want, 3)
    pat = np.ones((3, 5), dtype=np.uint8)
    e.place(pat, 100, 7)
    want[7:10, 100:105] = 1
    e.run(9, PACKED, 0)
    want, _ = oracle.run(want, 9)
    assert np.array_equal(e.download_packed(), oracle.pack(want))
    e.run(6, PACKED, 0)
    want, _ = oracle.run(want, 6)
    e.run(4, BYTE, 2)                                    # byte engine after a pair run
    want, _ = oracle.run(want, 4)
    e.run(11, PACKED, 0)
    want, _ = oracle.run(want, 11)
    e.run(5, PACKED, 4)                                  # explicit depth: still the forced layout
    want, _ = oracle.run(want, 5)
    if il == 4:                                          # quad -> pair without a download between
        e.set_option(capi.OPT_QUAD_DEPTH, 0)
        e.set_option(capi.OPT_PAIR_DEPTH, 9)
        e.run(10, PACKED, 0)
        want, _ = oracle.run(want, 10)
        e.set_option(capi.OPT_QUAD_DEPTH, 3)             # and back: quad wins when both are forced
        e.run(7, PACKED, 0)
        want, _ = oracle.run(want, 7)
        e.set_option(capi.OPT_PAIR_DEPTH, 0)
    e.set_option(opt, 0)                                 # layout off: the plain kernels
    e.run(6, PACKED, 0)
    want, _ = oracle.run(want, 6)
    assert np.array_equal(e.download(), want)
    e.set_option(opt, max_depth)
    e.run(0, PACKED, 0)
    assert np.array_equal(e.download(), want)


def test_pair_option_validation(pair_engine):
    e = pair_engine
    assert e.get_option(capi.OPT_PAIR_DEPTH) == -1
    assert e.get_option(capi.OPT_QUAD_DEPTH) == -1
    with pytest.raises(life.ConfigError):
        e.set_option(capi.OPT_PAIR_DEPTH, 13)
    with pytest.raises(life.ConfigError):
        e.set_option(capi.OPT_PAIR_DEPTH, -2)
    with pytest.raises(life.ConfigError):
        e.set_option(capi.OPT_QUAD_DEPTH, 8)
    # W % 128 != 0 with both forced: the quad option is skipped, pair runs
    e.set_option(capi.OPT_QUAD_DEPTH, 4)
    e.set_option(capi.OPT_PAIR_DEPTH, 8)
    e.init_random(192, 50, 0.3, 5)
    e.run(10)
    e.set_option(capi.OPT_QUAD_DEPTH, -1)
    # W % 64 != 0: the option is ignored, the plain kernels run
    e.set_option(capi.OPT_PAIR_DEPTH, 8)
    e.init_random(100, 50, 0.3, 5)
    e.run(10)
    assert e.population() > 0


def _check_schedule(e, oracle, gold):
    done = 0
    for gen in sorted(int(k) for k in gold["gens"]):
        e.run(gen - done, PACKED, 0)
        done = gen
        want = gold["gens"][str(gen)]
        assert e.population() == want["population"], gen  # on the pair layout
        assert fnv(oracle, e.download_packed()) == want["fnv_packed"], gen


@pytest.mark.slow
@pytest.mark.parametrize("layout,depth", [(PAIR, 8), (PAIR, 10), (QUAD, 5), (QUAD, 6), (QUAD, 7)],
                         ids=lambda v: v if isinstance(v, int) else f"order{v[0]}")
def test_pair_cfg2_golden(pair_engine, oracle, layout, depth):
    """Config 2 (16384^2, 1000 generations) on the pair / quad kernel against
    the reference's full-grid hashes at 0/1/10/100/1000."""
    gold = load_golden("golden_cfg2.json")
    e = pair_engine
    e.set_option(layout[1], depth)
    e.init_random(gold["w"], gold["h"], gold["density"], gold["seed"], PACKED)
    _check_schedule(e, oracle, gold)


@pytest.mark.slow
def test_pair_cfg3_golden(pair_engine, oracle):
    """Config 3 (65536^2) at the auto rule's choice (temporal_depth 0: quad, K = 7),
    then with the quad layout off (pair, K = 10)."""
    import ctypes as C
    d = C.c_int32(0)
    assert capi.lib().life_interleave_auto(65536, 65536, -1, -1, 0, C.byref(d)) == 4 and d.value == 7
    assert capi.lib().life_interleave_auto(65536, 65536, -1, 0, 0, C.byref(d)) == 2 and d.value == 10
    assert capi.lib().life_interleave_auto(65536, 65536, -1, -1, 16, C.byref(d)) == 0
    assert capi.lib().life_interleave_auto(16384, 16384, -1, -1, 0, C.byref(d)) == 2 and d.value == 10
    assert capi.lib().life_interleave_auto(8192, 8192, -1, -1, 0, C.byref(d)) == 0
    gold = load_golden("golden_cfg3.json")
    e = pair_engine
    e.init_random(gold["w"], gold["h"], gold["density"], gold["seed"], PACKED)
    _check_schedule(e, oracle, gold)
    e.set_option(capi.OPT_QUAD_DEPTH, 0)
    e.init_random(gold["w"], gold["h"], gold["density"], gold["seed"], PACKED)
    _check_schedule(e, oracle, gold)
