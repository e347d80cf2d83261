"""The pair- and quad-layout kernels (kernels_pair.cuh; interleave order 2: W %
64 == 0, order 4: W % 128 == 0) behind every
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
OPT = {2: capi.OPT_PAIR_DEPTH, 4: capi.OPT_QUAD_DEPTH}
MAXK = {2: capi.PAIR_MAX_DEPTH, 4: capi.QUAD_MAX_DEPTH}


def fnv(oracle, a) -> str:
    return f"{oracle.fnv1a64(np.ascontiguousarray(a)):016x}"


def words_to_cells(words: np.ndarray, width: int) -> np.ndarray:
    u = np.ascontiguousarray(words).view(np.uint32)
    bits = np.unpackbits(u.view(np.uint8), axis=1, bitorder="little")
    return bits[:, :width].astype(np.uint8)


# ---- life_run_batch ---------------------------------------------------------
@pytest.mark.parametrize("il,W,H,G,depth", [
    (2, 64, 50, 7, 3), (2, 2048, 600, 25, 10), (2, 1984, 333, 24, 12), (2, 128, 4099, 0, 8),
    (2, 640, 1030, 5, 5),
    (2, 64, 33280, 8, 4),      # trapezoids + triangles
    (2, 128, 70000, 30, 10),   # ... 3 passes of 10
    (2, 192, 40000, 17, 7),    # ... with a remainder pass
    (4, 128, 50, 7, 3), (4, 2048, 600, 25, 6), (4, 3968, 333, 24, 5), (4, 1280, 1030, 5, 4),
    (4, 128, 33280, 8, 4), (4, 256, 70000, 30, 6), (4, 384, 40000, 17, 5)])
def test_run_batch_pair(oracle, il, W, H, G, depth):
    """life_run_batch with LIFE_OPT_PAIR_DEPTH / _QUAD_DEPTH forced: grids
    zipped after the upload and unzipped before the download, also chunk by
    chunk on the trapezoid schedule (forced on for the tall shapes) and in place."""
    with life.Engine(0) as e:
        e.set_option(OPT[il], depth)
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
def multi(n: int, halo_mode: int, il: int, depth: int) -> life.Engine:
    e = life.Engine(devices=[0] * n)
    e.set_option(capi.OPT_HALO, halo_mode)
    e.set_option(OPT[il], depth)
    return e


@pytest.mark.parametrize("il", [2, 4], ids=["pair", "quad"])
@pytest.mark.parametrize("halo_mode", [capi.HALO_PEER, capi.HALO_COPY], ids=["peer", "copy"])
@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_multi_pair_matches_oracle(oracle, halo_mode, n, il):
    """Row bands on the pair / quad layout: random shapes, every pass depth,
    checkpoint splits; grid, uint64 populations, windows across band seams,
    hash and place on a grid left in the interleaved layout."""
    rng = np.random.default_rng(500 + n + il)
    for case in range(5):
        w = 32 * il * int(rng.integers(1, 70))
        h = int(rng.integers(max(3, n), 220))
        pair = int(rng.integers(1, MAXK[il] + 1))
        gens = int(rng.integers(1, 50))
        g = oracle.random_fill(w, h, 0.35, int(rng.integers(1 << 30)))
        cps = sorted({0, gens, *[int(x) for x in rng.integers(0, gens + 1, 2)]})
        want, pops = oracle.run(g, gens, cps)
        with multi(n, halo_mode, il, pair) as e, life.Engine(0) as one:
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
    for halo_mode, il, depth in ((capi.HALO_PEER, 2, 9), (capi.HALO_COPY, 2, 9),
                                 (capi.HALO_PEER, 4, 5), (capi.HALO_COPY, 4, 6)):
        with multi(3, halo_mode, il, depth) as e:
            assert e.run_batch(ins, outs, W, G, 0) > 0
            for want, out in zip(wants, outs):
                assert np.array_equal(oracle.unpack(out, W), want)
            for o in outs:
                o[:] = 0


def test_multi_pair_option(oracle):
    with multi(2, capi.HALO_PEER, 2, 5) as e:
        assert e.get_option(capi.OPT_PAIR_DEPTH) == 5
        assert e.get_option(capi.OPT_QUAD_DEPTH) == -1
        with pytest.raises(life.ConfigError):
            e.set_option(capi.OPT_PAIR_DEPTH, 13)
        with pytest.raises(life.ConfigError):
            e.set_option(capi.OPT_QUAD_DEPTH, 8)
        # W % 64 != 0: ignored, the plain kernels run
        g = oracle.random_fill(100, 40, 0.4, 3)
        e.upload(g)
        e.run(9, PACKED, 0)
        assert np.array_equal(e.download(), oracle.run(g, 9)[0])


@pytest.mark.slow
@pytest.mark.parametrize("n,quad", [(2, -1), (8, -1), (8, 0)])
def test_cfg5_pair_band_seam_windows(oracle, n, quad):
    """Config 5 as n bands at the engine's own choice (temporal_depth 0: the
    quad kernel at K = 7; with the quad layout off, the pair kernel at K =
    10): the reference's light-cone windows at T = 500, including every band
    seam and both wrap corners."""
    import ctypes as C
    gold = load_golden("golden_cfg5_windows.json")
    d = C.c_int32(0)
    il = capi.lib().life_interleave_auto(262144, 262144 // n, -1, quad, 0, C.byref(d))
    assert (il, d.value) == ((4, 7) if quad < 0 else (2, 10))
    with life.Engine(devices=[0] * n) as e:
        e.set_option(capi.OPT_QUAD_DEPTH, quad)
        e.init_random(262144, 262144, 0.4, 42)
        e.run(500, PACKED, 0)
        for w in gold["windows_500"]:
            assert fnv(oracle, e.window(w["x0"], w["y0"], w["S"], w["S"])) == w["fnv_bytes"], w


# ---- device-buffer band drivers (bands.py) ----------------------------------
@pytest.mark.parametrize("il,W,H,depth,gens", [
    (2, 64, 37, 4, 13), (2, 1984, 97, 12, 50), (2, 4096, 1025, 10, 100), (2, 2112, 300, 1, 9),
    (4, 128, 37, 4, 13), (4, 3968, 97, 6, 50), (4, 4096, 1025, 5, 100), (4, 4224, 300, 1, 9)])
def test_torus_driver_pair(oracle, il, W, H, depth, gens):
    import torch
    from paper_1209_4408_b200.bands import TorusDriver, make_geometry
    dev = torch.device("cuda", 0)
    drv = TorusDriver(make_geometry(W, H, 0, 1, depth, il), dev)
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


@pytest.mark.parametrize("il,W,H,P,depth,gens,overlap", [
    (2, 64, 37, 2, 4, 13, True), (2, 1984, 97, 3, 12, 50, True), (2, 1984, 97, 3, 12, 50, False),
    (2, 4096, 1025, 8, 10, 100, True), (2, 40960, 12289 // 16, 8, 7, 30, True),
    (4, 128, 37, 2, 4, 13, True), (4, 3968, 97, 3, 6, 50, True), (4, 3968, 97, 3, 6, 50, False),
    (4, 4096, 1025, 8, 5, 100, True), (4, 40960, 12289 // 16, 8, 3, 30, True)])
def test_local_bands_pair(oracle, il, W, H, P, depth, gens, overlap):
    """Ghost-row bands (the NCCL scheme's addressing) on the pair / quad layout."""
    import torch
    from paper_1209_4408_b200.bands import LocalBands
    lb = LocalBands(W, H, P, depth, torch.device("cuda", 0), overlap=overlap, il=il)
    lb.init_random(0.4, 9)
    lb.run(gens)
    torch.cuda.synchronize()
    got = words_to_cells(lb.gather().cpu().numpy(), W)
    want, _ = oracle.run(oracle.random_fill(W, H, 0.4, 9), gens)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("il,W,H,P,depth,gens", [
    (2, 64, 37, 2, 4, 13), (2, 1984, 97, 3, 12, 50), (2, 4096, 1025, 8, 10, 100),
    (2, 40960, 12289 // 16, 8, 7, 30), (2, 128, 40, 2, 12, 48), (2, 2048, 300, 3, 1, 9),
    (4, 128, 37, 2, 4, 13), (4, 3968, 97, 3, 6, 50), (4, 4096, 1025, 8, 5, 100),
    (4, 40960, 12289 // 16, 8, 3, 30), (4, 256, 40, 2, 6, 48), (4, 2048, 300, 3, 1, 9)])
def test_local_peer_bands_pair(oracle, il, W, H, P, depth, gens):
    """In-kernel peer halos on the pair / quad layout (life_dev_packed_step_il_peer)."""
    import torch
    from paper_1209_4408_b200.bands import LocalPeerBands
    lb = LocalPeerBands(W, H, P, depth, torch.device("cuda", 0), il=il)
    lb.init_random(0.4, 9)
    lb.run(gens)
    torch.cuda.synchronize()
    got = words_to_cells(lb.gather().cpu().numpy(), W)
    want, _ = oracle.run(oracle.random_fill(W, H, 0.4, 9), gens)
    assert np.array_equal(got, want)


def test_pair_geometry_errors():
    from paper_1209_4408_b200.bands import make_geometry
    with pytest.raises(life.ConfigError):
        make_geometry(100, 50, 0, 1, 8, il=2)    # W % 64 != 0
    with pytest.raises(life.ConfigError):
        make_geometry(128, 50, 0, 1, 13, il=2)   # deeper than the pair kernel goes
    with pytest.raises(life.ConfigError):
        make_geometry(192, 50, 0, 1, 4, il=4)    # W % 128 != 0
    with pytest.raises(life.ConfigError):
        make_geometry(256, 50, 0, 1, 8, il=4)    # deeper than the quad kernel goes
    with pytest.raises(life.ConfigError):
        make_geometry(256, 50, 0, 1, 4, il=3)


@pytest.mark.parametrize("il,W,H,G,depth", [(0, 96, 60000, 260, 16), (2, 64, 50000, 240, 10),
                                            (4, 128, 60000, 300, 6), (4, 128, 40000, 215, 5)])
def test_run_batch_geometric_chunks(oracle, il, W, H, G, depth):
    """Enough generations per byte copied for the geometric chunk plan of the
    trapezoid schedule (growth >= 1.5): small chunks first in the first grid,
    last in the last grid, at both ends of a single grid; in place too."""
    with life.Engine(0) as e:
        if il:
            e.set_option(OPT[il], depth)
        e.set_option(capi.OPT_BATCH_TRAPEZOID, 1)
        grids = [oracle.random_fill(W, H, 0.35, 700 + i) for i in range(3)]
        wants = [oracle.run(g, G)[0] for g in grids]
        for n in (1, 2, 3):
            ins = [oracle.pack(g) for g in grids[:n]]
            outs = [np.zeros_like(p) for p in ins]
            e.run_batch(ins, outs, W, G, 0 if il else depth)
            for want, out in zip(wants, outs):
                assert np.array_equal(oracle.unpack(out, W), want), (n,)
        ins = [oracle.pack(g) for g in grids]
        e.run_batch(ins, ins, W, G, 0 if il else depth)
        for want, out in zip(wants, ins):
            assert np.array_equal(oracle.unpack(out, W), want)
