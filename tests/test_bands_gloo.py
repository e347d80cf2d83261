"""Multi-rank row-band driver (paper_1209_4408_b200/bands.py) on CPU with the
gloo backend: world sizes 2 and 3, the real halo-exchange/overlap logic, and a
test-only stepper that computes each pass with the oracle.  The assembled
bands must equal the oracle's full-torus run bit for bit."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def to_words(cells: np.ndarray, pitch: int) -> np.ndarray:
    """0/1 rows -> int32 rows of the packed layout (bit j of word k = column 32k+j)."""
    h, w = cells.shape
    out = np.zeros((h, pitch), np.uint32)
    for x in range(w):
        out[:, x // 32] |= cells[:, x].astype(np.uint32) << np.uint32(x % 32)
    return out.view(np.int32)


def from_words(words: np.ndarray, w: int) -> np.ndarray:
    u = np.ascontiguousarray(words).view(np.uint32)
    return np.stack([((u[:, x // 32] >> np.uint32(x % 32)) & 1).astype(np.uint8)
                     for x in range(w)], axis=1)


def oracle_stepper(width: int):
    from oracle.oracle import Oracle
    O = Oracle()

    def step(inp, in_row0, in_rows, out, out_row0, out_rows, k):
        src = inp.numpy()
        rows = [(in_row0 + r) % in_rows for r in range(-k, out_rows + k)]
        window = from_words(src[rows], width)
        res, _ = O.run(window, k)  # vertical wrap only touches the k discarded rows
        out.numpy()[out_row0:out_row0 + out_rows] = to_words(res[k:k + out_rows], out.shape[1])
    return step


def _worker(rank, world, port, W, H, depth, gens, overlap, result_q, checkpoints=()):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_1209_4408_b200.bands import BandDriver, make_geometry
        O = Oracle()
        geo = make_geometry(W, H, rank, world, depth)
        drv = BandDriver(geo, torch.device("cpu"), stepper=oracle_stepper(W), overlap=overlap,
                         counter=lambda b: int(np.unpackbits(b.numpy().view(np.uint8)).sum()))
        init = O.random_window(W, H, 0.4, 7, 0, geo.y0, W, geo.band_rows)
        drv.band().copy_(torch.from_numpy(to_words(init, geo.pitch)))
        pops = drv.run(gens, checkpoints=checkpoints)
        band = from_words(drv.band().numpy(), W)
        parts = [None] * world
        dist.all_gather_object(parts, (geo.y0, band))
        if rank == 0:
            result_q.put((parts, pops))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,W,H,depth,gens,overlap", [
    (2, 70, 37, 4, 13, True),
    (2, 33, 16, 8, 24, False),
    (3, 64, 29, 3, 10, True),
    (2, 100, 12, 6, 6, True),
])
def test_band_driver_matches_full_torus(oracle, world, W, H, depth, gens, overlap):
    parts, _ = _run_world(world, W, H, depth, gens, overlap)
    got = np.concatenate([b for _, b in sorted(parts, key=lambda t: t[0])], axis=0)
    want, _ = oracle.run(oracle.random_fill(W, H, 0.4, 7), gens)
    assert np.array_equal(got, want)


def _run_world(world, W, H, depth, gens, overlap, checkpoints=()):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, W, H, depth, gens, overlap, q,
                                               tuple(checkpoints)))
             for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,depth,cps", [(2, 4, (0, 3, 9, 13)), (3, 3, (1, 2, 13))])
def test_band_driver_checkpoint_populations(oracle, world, depth, cps):
    """run(..., checkpoints) on N ranks: passes split at the checkpoints, the
    populations summed over every rank's band (engine.cpp:179-186) equal the
    oracle's at every checkpoint, and the final torus is unchanged."""
    W, H, gens = 70, 37, 13
    parts, pops = _run_world(world, W, H, depth, gens, True, cps)
    want, want_pops = oracle.run(oracle.random_fill(W, H, 0.4, 7), gens, list(cps))
    assert pops == want_pops
    got = np.concatenate([b for _, b in sorted(parts, key=lambda t: t[0])], axis=0)
    assert np.array_equal(got, want)


def test_run_schedule_rejects_bad_checkpoints():
    from paper_1209_4408_b200.bands import run_schedule
    from paper_1209_4408_b200.life import ConfigError

    class Dummy:
        class geo:
            depth = 4
    for gens, cps in [(-1, ()), (5, (6,)), (5, (2, 2)), (5, (3, 1))]:
        with pytest.raises(ConfigError):
            run_schedule(Dummy(), gens, cps)


def test_geometry_follows_partition_rows(golden_small):
    from paper_1209_4408_b200.bands import make_geometry
    from paper_1209_4408_b200.life import ConfigError, TooManyParts
    cuts = golden_small["partition_rows"]["12289/8"]
    for r in range(8):
        g = make_geometry(40961, 12289, r, 8, 16)
        assert (g.y0, g.y1) == (cuts[r], cuts[r + 1])
        assert g.buf_rows == g.band_rows + 32 and g.pitch % 32 == 0
    with pytest.raises(TooManyParts):
        make_geometry(64, 9, 0, 10, 1)
    with pytest.raises(TooManyParts):
        make_geometry(64, 20, 0, 4, 8)  # 5-row bands < depth 8
    with pytest.raises(ConfigError):
        make_geometry(64, 64, 0, 2, 17)


def _token_worker(rank, world, port, rounds, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1209_4408_b200.bands import neighbour_token
        got = []
        for p in range(rounds):
            tok = torch.tensor([1000 * p + rank], dtype=torch.int32)
            inbox = torch.full((2,), -1, dtype=torch.int32)
            neighbour_token(tok, inbox, rank, world)
            got.append([int(inbox[0]), int(inbox[1])])
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_neighbour_token_pairs_with_both_neighbours(world):
    """The peer band driver's pass ordering (neighbour_token): every rank
    receives, each pass, the token of the rank above and of the rank below --
    no deadlock in the up == down case (two ranks) or around the ring."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    rounds = 5
    procs = [ctx.Process(target=_token_worker, args=(r, world, port, rounds, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        up, down = (r - 1) % world, (r + 1) % world
        assert res[r] == [[1000 * p + up, 1000 * p + down] for p in range(rounds)]
