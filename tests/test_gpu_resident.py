"""GPU parity of the cluster-resident engine (LIFE_ENGINE_RESIDENT): the whole
torus in one thread-block cluster's shared memory, every generation in one
launch, neighbour bands' edge rows over DSMEM.  Bit-exact vs the oracle
(step_serial / run, grid.cpp:30-38, engine.cpp:162-214) and the reference's
config-1 goldens.

Run on a B200:  python -m pytest tests -m gpu -x -q
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PACKED, BYTE, RESIDENT = 0, 1, 2


def fnv(oracle, a) -> str:
    return f"{oracle.fnv1a64(np.ascontiguousarray(a)):016x}"


# Shapes: one CTA (H < 4), uneven bands (H % C != 0), two-row bands (no
# interior rows), one-word rows (the column wrap is a rotation of the word),
# a wide torus (many words per row), and clusters of 1/2/4/8/16 CTAs.
SHAPES = [(32, 3), (32, 4), (32, 5), (64, 7), (96, 33), (128, 64), (256, 97), (512, 31),
          (1024, 96), (2048, 40), (160, 1000), (4096, 64)]


@pytest.mark.parametrize("w,h", SHAPES)
def test_resident_matches_oracle(engine, oracle, w, h):
    from paper_1209_4408_b200 import capi
    assert capi.lib().life_resident_cluster_size(w, h) >= 1
    g = oracle.random_fill(w, h, 0.4, w * 7 + h)
    for gens in (1, 2, 5, 38):
        want, _ = oracle.run(g, gens)
        engine.upload(g)
        engine.run(gens, RESIDENT)
        assert np.array_equal(engine.download(), want), (w, h, gens)


def test_resident_cluster_sizes(engine):
    from paper_1209_4408_b200 import capi
    L = capi.lib()
    assert L.life_resident_cluster_size(1024, 1024) == 16
    assert L.life_resident_cluster_size(32, 3) == 1   # H >= 2 rows per CTA
    assert L.life_resident_cluster_size(32, 7) == 2
    assert L.life_resident_cluster_size(64, 35) == 16
    assert L.life_resident_cluster_size(33, 64) == 0  # W % 32 != 0
    assert L.life_resident_cluster_size(65536, 65536) == 0  # does not fit


def test_resident_cfg1_goldens(engine, oracle, golden_small):
    cfg1 = golden_small["cfg1"]
    engine.init_random(1024, 1024, 0.5, 42, PACKED)
    pops = engine.run(100, RESIDENT, 0, [0, 1, 10, 100])
    assert pops == [524027, 286720, 211733, 98161]
    assert fnv(oracle, engine.download()) == "37b6d88ff40a4f22"
    for g in (1, 10):
        engine.init_random(1024, 1024, 0.5, 42, PACKED)
        engine.run(g, RESIDENT)
        assert fnv(oracle, engine.download()) == cfg1[str(g)]["fnv_bytes"]
        assert fnv(oracle, engine.download_packed()) == cfg1[str(g)]["fnv_packed"]


def test_resident_auto_selection_and_checkpoints(engine, oracle):
    # depth 0 (auto) on a small W % 32 == 0 torus takes the resident engine;
    # checkpoints split the run into one launch per interval.
    g = oracle.random_fill(256, 200, 0.35, 11)
    cps = [0, 1, 3, 17, 18, 40, 64, 200]
    _, want = oracle.run(g, 200, cps)
    from paper_1209_4408_b200 import capi
    before = capi.lib().life_kernel_launches()
    engine.upload(g)
    assert engine.run(200, PACKED, 0, cps) == want
    launched = capi.lib().life_kernel_launches() - before
    assert launched <= 3 * len(cps) + 4  # one resident launch per interval (+ popcounts)
    engine.upload(g)
    assert engine.run(200, RESIDENT, 0, cps) == want


def test_resident_long_run_and_byte_layout_in(engine, oracle):
    # A grid resident in the byte layout is packed at the boundary first.
    g = oracle.random_fill(320, 48, 0.5, 5)
    want, _ = oracle.run(g, 1000)
    engine.upload(g)
    engine.run(1, BYTE)
    engine.run(999, RESIDENT)
    assert np.array_equal(engine.download(), want)


def test_resident_rejects_unfit_tori(engine):
    from paper_1209_4408_b200 import life
    engine.init_random(33, 64, 0.5, 1)
    with pytest.raises(life.ConfigError):
        engine.run(3, RESIDENT)
    # the packed engine's auto mode falls back to multi-pass K = 16
    engine.run(3, PACKED, 0)
    with pytest.raises(life.ConfigError):
        engine.run(3, RESIDENT, 17)


def test_device_layer_entry_points(oracle):
    """The device-buffer entry points of the two new engines: the resident run
    in place (in == out), and byte passes of depth > 1 (W % 16 == 0 only)."""
    import torch

    from paper_1209_4408_b200 import capi, life
    L = capi.lib()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev).cuda_stream
    W, H, G = 256, 48, 21
    g = oracle.random_fill(W, H, 0.4, 3)
    want, _ = oracle.run(g, G)
    pitch = int(L.life_packed_pitch_words(W))
    host = np.zeros((H, pitch), np.uint32)
    host[:, : W // 32] = oracle.pack(g).view(np.uint32)[:, : W // 32]
    buf = torch.from_numpy(host.view(np.int32)).to(dev)
    life.check(L.life_dev_packed_run_resident(buf.data_ptr(), buf.data_ptr(), pitch, W, H, G,
                                              stream))
    torch.cuda.synchronize()
    got = buf.cpu().numpy().view(np.uint32)[:, : W // 32].copy()
    assert np.array_equal(got, oracle.pack(want).view(np.uint32)[:, : W // 32])
    # byte passes: K = 5 in one launch == 5 oracle generations; W % 16 != 0 -> ConfigError
    bp = int(L.life_byte_pitch(W))
    hb = np.zeros((H, bp), np.uint8)
    hb[:, :W] = g
    a = torch.from_numpy(hb).to(dev)
    b = torch.zeros_like(a)
    life.check(L.life_dev_byte_pass(a.data_ptr(), bp, 0, H, b.data_ptr(), bp, 0, W, H, 5, stream))
    torch.cuda.synchronize()
    want5, _ = oracle.run(g, 5)
    assert np.array_equal(b.cpu().numpy()[:, :W], want5)
    assert L.life_dev_byte_pass(a.data_ptr(), bp, 0, H, b.data_ptr(), bp, 0, W - 8, H, 2,
                                stream) == capi.ERR_CONFIG
    assert L.life_dev_byte_pass(a.data_ptr(), bp, 0, H, b.data_ptr(), bp, 0, W, H, 9,
                                stream) == capi.ERR_CONFIG


def test_run_batch_small_tori_take_the_resident_engine(engine, oracle):
    """life_run_batch with temporal_depth 0 on small W % 32 == 0 tori: one
    resident launch per grid, copies overlapped; every grid equals the oracle
    (also G = 0 and in place)."""
    from paper_1209_4408_b200 import capi
    W, H = 1024, 96
    grids = [oracle.random_fill(W, H, 0.3 + 0.1 * i, 50 + i) for i in range(4)]
    ins = [oracle.pack(g) for g in grids]
    for G in (0, 1, 45):
        outs = [np.zeros_like(p) for p in ins]
        before = capi.lib().life_kernel_launches()
        engine.run_batch(ins, outs, W, G, 0)
        assert capi.lib().life_kernel_launches() - before <= 2 * len(grids)  # mask + 1 launch per grid
        for g, out in zip(grids, outs):
            want, _ = oracle.run(g, G)
            assert np.array_equal(oracle.unpack(out, W), want), G
    engine.run_batch(ins, ins, W, 7, 0)
    for g, out in zip(grids, ins):
        want, _ = oracle.run(g, 7)
        assert np.array_equal(oracle.unpack(out, W), want)
