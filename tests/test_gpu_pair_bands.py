"""The interleaved-pair kernel (kernels_pair.cuh, W % 64 == 0) behind every
caller of the packed step besides life_run: life_run_batch (whole-grid and
trapezoid schedules), the multi-device context (row bands, peer and copy
halos, run and run_batch) and the device-buffer band drivers of
paper_1209_4408_b200.bands (torus, ghost-row bands, in-kernel peer halos).
Bit-exact against the oracle and the reference goldens.

Run on a B200:  python -m pytest tests/test_gpu_pair_bands.py -m gpu -x -q
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden
from paper_1209_4408_b200 import capi, life

pytestmark = pytest.mark.gpu

PACKED = capi.ENGINE_PACKED


def fnv(oracle, a) -> str:
    return f"{oracle.fnv1a64(np.ascontiguousarray(a)):016x}"


def words_to_cells(words: np.ndarray, width: int) -> np.ndarray:
    u = np.ascontiguousarray(words).view(np.uint32)
    bits = np.unpackbits(u.view(np.uint8), axis=1, bitorder="little")
    return bits[:, :width].astype(np.uint8)


# ---- life_run_batch ---------------------------------------------------------
@pytest.mark.parametrize("W,H,G,pair", [(64, 50, 7, 3), (2048, 600, 25, 10), (1984, 333, 24, 12),
                                        (128, 4099, 0, 8), (640, 1030, 5, 5),
                                        (64, 33280, 8, 4),      # trapezoids + triangles
                                        (128, 70000, 30, 10),   # ... 3 passes of 10
                                        (192, 40000, 17, 7)])   # ... with a remainder pass
def test_run_batch_pair(oracle, W, H, G, pair):
    """life_run_batch with LIFE_OPT_PAIR_DEPTH forced: grids zipped after the
    upload and unzipped before the download, also chunk by chunk on the
    trapezoid schedule (forced on for the tall shapes) and in place."""
    with life.Engine(0) as e:
        e.set_option(capi.OPT_PAIR_DEPTH, pair)
        if H >= 32768:
            e.set_option(capi.OPT_BATCH_TRAPEZOID, 1)
        grids = [oracle.random_fill(W, H, 0.35, 300 + i) for i in range(3)]
        ins = [oracle.pack(g) for g in grids]
        outs = [np.zeros_like(p) for p in ins]
        e.run_batch(ins, outs, W, G, 0)
        wants = [oracle.run(g, G)[0] for g in grids]
        for want, out in zip(wants, outs):
            assert np.array_equal(oracle.unpack(out, W), want)
        e.run_batch(ins, ins, W, G, 16)  # in place; the forced pair depth wins over 16
        for want, out in zip(wants, ins):
            assert np.array_equal(oracle.unpack(out, W), want)


# ---- multi-device context ---------------------------------------------------
def multi(n: int, halo_mode: int, pair: int) -> life.Engine:
    e = life.Engine(devices=[0] * n)
    e.set_option(capi.OPT_HALO, halo_mode)
    e.set_option(capi.OPT_PAIR_DEPTH, pair)
    return e


@pytest.mark.parametrize("halo_mode", [capi.HALO_PEER, capi.HALO_COPY], ids=["peer", "copy"])
@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_multi_pair_matches_oracle(oracle, halo_mode, n):
    """Row bands on the pair layout: random W % 64 == 0 shapes, pair depths
    1..12, checkpoint splits; grid, uint64 populations, windows across band
    seams, hash and place on a grid left in the pair layout."""
    rng = np.random.default_rng(500 + n)
    for case in range(5):
        w = 64 * int(rng.integers(1, 70))
        h = int(rng.integers(max(3, n), 220))
        pair = int(rng.integers(1, 13))
        gens = int(rng.integers(1, 50))
        g = oracle.random_fill(w, h, 0.35, int(rng.integers(1 << 30)))
        cps = sorted({0, gens, *[int(x) for x in rng.integers(0, gens + 1, 2)]})
        want, pops = oracle.run(g, gens, cps)
        with multi(n, halo_mode, pair) as e, life.Engine(0) as one:
            e.upload(g)
            assert e.run(gens, PACKED, 0, cps) == pops, (w, h, gens, pair, n)
            assert e.population() == int(want.sum())
            one.upload(want)
            assert e.hash() == one.hash()
            e.run(3, PACKED, 0)  # plain again after the hash; back to pair
            want2, _ = oracle.run(want, 3)
            win = e.window(w - 5, h - 4, 11, 9)
            assert np.array_equal(win, np.take(np.take(want2, np.arange(h - 4, h + 5) % h, axis=0),
                                               np.arange(w - 5, w + 6) % w, axis=1))
            e.run(2, PACKED, 0)
            want2, _ = oracle.run(want2, 2)
            if h >= 8 and w >= 64:
                e.place(np.ones((3, 5), np.uint8), 7, h // 2 - 1)
                want2[h // 2 - 1:h // 2 + 2, 7:12] = 1
            e.run(4, PACKED, 0)
            want2, _ = oracle.run(want2, 4)
            assert np.array_equal(e.download(), want2), (w, h, gens, pair, n)


def test_multi_pair_run_batch(oracle):
    W, H, G = 1024, 777, 37
    grids = [oracle.random_fill(W, H, 0.3 + 0.1 * i, i) for i in range(5)]
    ins = [oracle.pack(g) for g in grids]
    outs = [np.zeros_like(p) for p in ins]
    wants = [oracle.run(g, G)[0] for g in grids]
    for halo_mode in (capi.HALO_PEER, capi.HALO_COPY):
        with multi(3, halo_mode, 9) as e:
            assert e.run_batch(ins, outs, W, G, 0) > 0
            for want, out in zip(wants, outs):
                assert np.array_equal(oracle.unpack(out, W), want)
            for o in outs:
                o[:] = 0


def test_multi_pair_option(oracle):
    with multi(2, capi.HALO_PEER, 5) as e:
        assert e.get_option(capi.OPT_PAIR_DEPTH) == 5
        with pytest.raises(life.ConfigError):
            e.set_option(capi.OPT_PAIR_DEPTH, 13)
        # W % 64 != 0: ignored, the plain kernels run
        g = oracle.random_fill(100, 40, 0.4, 3)
        e.upload(g)
        e.run(9, PACKED, 0)
        assert np.array_equal(e.download(), oracle.run(g, 9)[0])


@pytest.mark.slow
@pytest.mark.parametrize("n", [2, 8])
def test_cfg5_pair_band_seam_windows(oracle, n):
    """Config 5 as n bands at the engine's own choice (temporal_depth 0: the
    pair kernel at K = 10): the reference's light-cone windows at T = 500,
    including every band seam and both wrap corners."""
    gold = load_golden("golden_cfg5_windows.json")
    assert capi.lib().life_pair_auto_depth(262144, 262144 // n) == 10
    with life.Engine(devices=[0] * n) as e:
        e.init_random(262144, 262144, 0.4, 42)
        e.run(500, PACKED, 0)
        for w in gold["windows_500"]:
            assert fnv(oracle, e.window(w["x0"], w["y0"], w["S"], w["S"])) == w["fnv_bytes"], w


# ---- device-buffer band drivers (bands.py) ----------------------------------
@pytest.mark.parametrize("W,H,depth,gens", [(64, 37, 4, 13), (1984, 97, 12, 50),
                                            (4096, 1025, 10, 100), (2112, 300, 1, 9)])
def test_torus_driver_pair(oracle, W, H, depth, gens):
    import torch
    from paper_1209_4408_b200.bands import TorusDriver, make_geometry
    dev = torch.device("cuda", 0)
    drv = TorusDriver(make_geometry(W, H, 0, 1, depth, pair=True), dev)
    drv.init_random(0.4, 9)
    g0 = oracle.random_fill(W, H, 0.4, 9)
    pops = drv.run(gens, checkpoints=[0, gens // 2, gens])
    want, wpops = oracle.run(g0, gens, [0, gens // 2, gens])
    assert pops == wpops
    assert drv.in_pair
    assert np.array_equal(words_to_cells(drv.band().cpu().numpy(), W), want)
    drv.run(gens)  # one life_dev_packed_run_pair call, from the plain layout again
    want, _ = oracle.run(want, gens)
    assert drv.population() == int(want.sum())
    assert np.array_equal(words_to_cells(drv.band().cpu().numpy(), W), want)


@pytest.mark.parametrize("W,H,P,depth,gens,overlap", [
    (64, 37, 2, 4, 13, True), (1984, 97, 3, 12, 50, True), (1984, 97, 3, 12, 50, False),
    (4096, 1025, 8, 10, 100, True), (40960, 12289 // 16, 8, 7, 30, True)])
def test_local_bands_pair(oracle, W, H, P, depth, gens, overlap):
    """Ghost-row bands (the NCCL scheme's addressing) on the pair layout."""
    import torch
    from paper_1209_4408_b200.bands import LocalBands
    lb = LocalBands(W, H, P, depth, torch.device("cuda", 0), overlap=overlap, pair=True)
    lb.init_random(0.4, 9)
    lb.run(gens)
    torch.cuda.synchronize()
    got = words_to_cells(lb.gather().cpu().numpy(), W)
    want, _ = oracle.run(oracle.random_fill(W, H, 0.4, 9), gens)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("W,H,P,depth,gens", [
    (64, 37, 2, 4, 13), (1984, 97, 3, 12, 50), (4096, 1025, 8, 10, 100),
    (40960, 12289 // 16, 8, 7, 30), (128, 40, 2, 12, 48), (2048, 300, 3, 1, 9)])
def test_local_peer_bands_pair(oracle, W, H, P, depth, gens):
    """In-kernel peer halos on the pair layout (life_dev_packed_step_pair_peer)."""
    import torch
    from paper_1209_4408_b200.bands import LocalPeerBands
    lb = LocalPeerBands(W, H, P, depth, torch.device("cuda", 0), pair=True)
    lb.init_random(0.4, 9)
    lb.run(gens)
    torch.cuda.synchronize()
    got = words_to_cells(lb.gather().cpu().numpy(), W)
    want, _ = oracle.run(oracle.random_fill(W, H, 0.4, 9), gens)
    assert np.array_equal(got, want)


def test_pair_geometry_errors():
    from paper_1209_4408_b200.bands import make_geometry
    with pytest.raises(life.ConfigError):
        make_geometry(100, 50, 0, 1, 8, pair=True)   # W % 64 != 0
    with pytest.raises(life.ConfigError):
        make_geometry(128, 50, 0, 1, 13, pair=True)  # deeper than the pair kernel goes
