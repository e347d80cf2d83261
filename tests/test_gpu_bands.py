"""Row-band decomposition with the real CUDA kernels on ONE GPU: P emulated
bands (paper_1209_4408_b200.bands.LocalBands) with device-copy halos must give
the same torus as the single-band engine and the oracle -- band seams, ghost
addressing, interior/edge split, band_bounds remainders."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def words_to_cells(words: np.ndarray, width: int) -> np.ndarray:
    u = np.ascontiguousarray(words).view(np.uint32)
    bits = np.unpackbits(u.view(np.uint8), axis=1, bitorder="little")
    return bits[:, :width].astype(np.uint8)


@pytest.mark.parametrize("W,H,P,depth,gens,overlap", [
    (70, 37, 2, 4, 13, True),
    (1000, 97, 3, 16, 50, True),
    (1000, 97, 3, 16, 50, False),
    (4096, 1025, 8, 16, 100, True),
    (40961, 12289 // 16, 8, 7, 30, True),
    (333, 64, 4, 16, 33, True),
    (1024, 300, 3, 1, 9, True),       # depth 1, W % 128 == 0: the vector kernel per band
    (1024, 300, 3, 1, 9, False),
])
def test_local_bands_match_oracle(oracle, W, H, P, depth, gens, overlap):
    import torch
    from paper_1209_4408_b200.bands import LocalBands
    lb = LocalBands(W, H, P, depth, torch.device("cuda", 0), overlap=overlap)
    lb.init_random(0.4, 9)
    lb.run(gens)
    torch.cuda.synchronize()
    got = words_to_cells(lb.gather().cpu().numpy(), W)
    want, _ = oracle.run(oracle.random_fill(W, H, 0.4, 9), gens)
    assert np.array_equal(got, want)


@pytest.mark.slow
def test_cfg5_bands_equal_single_gpu_windows(oracle):
    """Config 5 split into 8 emulated bands: windows at every band seam equal
    the reference-generated light-cone goldens."""
    import torch
    from conftest import load_golden
    from paper_1209_4408_b200.bands import LocalBands
    gold = load_golden("golden_cfg5_windows.json")
    W = H = 262144
    lb = LocalBands(W, H, 8, 16, torch.device("cuda", 0))
    lb.init_random(0.4, 42)
    lb.run(16)
    full = lb.gather()
    for w in gold["windows_16"]:
        ys = (np.arange(w["S"]) + w["y0"]) % H
        rows = full[torch.as_tensor(ys, device=full.device)].cpu().numpy()
        cells = words_to_cells(rows, W)
        xs = (np.arange(w["S"]) + w["x0"]) % W
        win = np.ascontiguousarray(cells[:, xs])
        assert f"{oracle.fnv1a64(win):016x}" == w["fnv_bytes"], w


@pytest.mark.parametrize("W,H,P,depth,gens", [
    (70, 37, 2, 4, 13), (1000, 97, 3, 16, 50), (4096, 1025, 8, 16, 100),
    (40961, 12289 // 16, 8, 7, 30), (333, 64, 4, 16, 33), (96, 40, 2, 16, 48),
    (1024, 300, 3, 1, 9),
])
def test_local_peer_bands_match_oracle(oracle, W, H, P, depth, gens):
    """The fused-halo kernel (ghost rows read from the neighbour bands'
    buffers inside the pass) over P bands on one device."""
    import torch
    from paper_1209_4408_b200.bands import LocalPeerBands
    lb = LocalPeerBands(W, H, P, depth, torch.device("cuda", 0))
    lb.init_random(0.4, 9)
    lb.run(gens)
    torch.cuda.synchronize()
    got = words_to_cells(lb.gather().cpu().numpy(), W)
    want, _ = oracle.run(oracle.random_fill(W, H, 0.4, 9), gens)
    assert np.array_equal(got, want)


def _ipc_worker(rank, world, port, W, H, depth, gens, q, il=0, sync="neighbour"):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1209_4408_b200.bands import PeerBandDriver, make_geometry
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        drv = PeerBandDriver(make_geometry(W, H, rank, world, depth, il), dev, sync=sync)
        drv.init_random(0.4, 5)
        # gloo => host barrier per pass (sync "neighbour"), or stream-memory-operation
        # flags in the other process's IPC buffer: either way no kernel waits on another
        cps = drv.run(gens, checkpoints=[0, 5, 11, gens])  # passes split at 5 and 11
        band = drv.band().cpu().numpy()
        pop = drv.population()
        parts = [None] * world
        dist.all_gather_object(parts, (drv.geo.y0, band, pop, cps))
        drv.close()
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("W,depth,il,sync", [(500, 8, 0, "neighbour"), (576, 8, 2, "neighbour"),
                                             (512, 6, 4, "neighbour"), (500, 8, 0, "flag"),
                                             (512, 6, 4, "flag_overlap")],
                         ids=["plain", "pair", "quad", "plain-flag", "quad-flag-overlap"])
def test_peer_driver_ipc_two_processes_one_gpu(oracle, W, depth, il, sync):
    """PeerBandDriver across two processes sharing cuda:0 through CUDA IPC
    handles (host barrier between passes, so no kernel waits on another); also
    on the pair and quad layouts (bands converted before the first barrier),
    and with the passes ordered by flags each process bumps in the OTHER
    process's IPC-mapped buffer with stream memory operations (a waiting
    stream holds no SM, so two processes time-sliced on one GPU cannot
    starve each other)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    H, gens = 90, 27
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, W, H, depth, gens, q, il, sync),
                         daemon=True)
             for r in range(2)]
    for p in procs:
        p.start()
    try:
        parts = q.get(timeout=120)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
    parts.sort(key=lambda t: t[0])
    got = words_to_cells(np.concatenate([b for _, b, _, _ in parts], axis=0), W)
    want, pops = oracle.run(oracle.random_fill(W, H, 0.4, 5), gens, [0, 5, 11, gens])
    assert np.array_equal(got, want)
    assert parts[0][2] == pops[-1]
    assert parts[0][3] == parts[1][3] == pops  # checkpoint populations summed over ranks


def test_torus_driver_checkpoints(oracle):
    """TorusDriver (the one-GPU band driver bench.py uses): whole run and
    checkpointed run equal the oracle."""
    import torch
    from paper_1209_4408_b200.bands import TorusDriver, make_geometry
    W, H, gens = 1000, 301, 45
    want, pops = oracle.run(oracle.random_fill(W, H, 0.4, 21), gens, [0, 7, 30, gens])
    for cps in ([], [0, 7, 30, gens]):
        drv = TorusDriver(make_geometry(W, H, 0, 1, 16), torch.device("cuda", 0))
        drv.init_random(0.4, 21)
        got_pops = drv.run(gens, checkpoints=cps)
        torch.cuda.synchronize()
        assert np.array_equal(words_to_cells(drv.band().cpu().numpy(), W), want)
        assert got_pops == (pops if cps else [])


@pytest.mark.slow
def test_cfg5_full_grid_hash_across_band_decompositions():
    """the full 262144^2 grid hash after 32 generations
    is the same for the whole torus (one context) and for 2 / 8 row bands
    with in-kernel peer halos (emulated on one GPU), via life_grid_hash's row
    hashes (life_dev_packed_row_hashes + life_fnv1a64)."""
    import ctypes as C

    import torch

    from paper_1209_4408_b200 import capi, life
    from paper_1209_4408_b200.bands import LocalPeerBands
    W = H = 262144
    G = 32
    L = capi.lib()
    with life.Engine(0) as e:
        e.init_random(W, H, 0.4, 42)
        e.run(G, capi.ENGINE_PACKED, 16)
        want = e.hash()
    torch.cuda.empty_cache()
    dev = torch.device("cuda", 0)
    for P in (2, 8):
        lb = LocalPeerBands(W, H, P, 16, dev)
        lb.init_random(0.4, 42)
        lb.run(G)
        rows = torch.empty(H, dtype=torch.int64, device=dev)
        at = 0
        stream = torch.cuda.current_stream(dev).cuda_stream
        for bb in lb.bufs:
            band = bb[lb.cur]
            n = band.shape[0]
            life.check(L.life_dev_packed_row_hashes(band.data_ptr(), band.shape[1], W, n,
                                                    rows[at:].data_ptr(), stream))
            at += n
        host = rows.cpu().numpy()
        got = L.life_fnv1a64(host.ctypes.data, host.nbytes, 0)
        assert got == want, P
        del lb
        torch.cuda.empty_cache()


@pytest.mark.slow
def test_band_interiors_take_the_split_launch():
    """Band interiors of a W % 32 != 0 torus deep enough for launch_packed's
    split (seam strips on the all-paths kernel beside the fast-only kernel):
    2 bands (ghost-copy and peer schemes) give the single context's
    grid hash."""
    import torch

    from paper_1209_4408_b200 import capi, life
    from paper_1209_4408_b200.bands import LocalBands, LocalPeerBands
    W, H, G = 2001, 1_400_000, 32
    L = capi.lib()
    with life.Engine(0) as e:
        e.init_random(W, H, 0.35, 77)
        e.run(G, capi.ENGINE_PACKED, 16)
        want = e.hash()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev).cuda_stream
    for make in (lambda: LocalBands(W, H, 2, 16, dev), lambda: LocalPeerBands(W, H, 2, 16, dev)):
        lb = make()
        lb.init_random(0.35, 77)
        lb.run(G)
        grid = lb.gather()
        rows = torch.empty(H, dtype=torch.int64, device=dev)
        life.check(L.life_dev_packed_row_hashes(grid.data_ptr(), grid.shape[1], W, H,
                                                rows.data_ptr(), stream))
        host = rows.cpu().numpy()
        assert L.life_fnv1a64(host.ctypes.data, host.nbytes, 0) == want
        del lb, grid
        torch.cuda.empty_cache()


@pytest.mark.parametrize("W,H,depth,gens", [
    (2048, 6400, 16, 16 * 3 + 5),   # odd passes + remainder
    (2048, 6400, 16, 16 * 4),       # even passes, no remainder
    (4096, 3800, 8, 8 * 5 + 3),
    (8192, 1536, 12, 12 * 2 + 1),
    (2047, 6400, 16, 40),           # W % 32 != 0
    (2048, 100, 16, 7),             # remainder only
])
def test_dev_packed_run_matches_oracle(oracle, W, H, depth, gens):
    """life_dev_packed_run (full passes then the remainder, ping-pong) equals
    the oracle, result buffer as reported."""
    import ctypes as C

    import torch
    from paper_1209_4408_b200 import capi
    from paper_1209_4408_b200.life import check
    L = capi.lib()
    pitch = int(L.life_packed_pitch_words(W))
    dev = torch.device("cuda", 0)
    a = torch.zeros((H, pitch), dtype=torch.int32, device=dev)
    b = torch.zeros_like(a)
    s = torch.cuda.current_stream(dev).cuda_stream
    check(L.life_dev_packed_random(a.data_ptr(), pitch, W, 0, H, 0.4, 77, s))
    flip = C.c_int32(-1)
    check(L.life_dev_packed_run(a.data_ptr(), b.data_ptr(), pitch, W, H, gens, depth,
                                C.byref(flip), s))
    torch.cuda.synchronize()
    passes = gens // depth + (1 if gens % depth else 0)
    assert flip.value == passes % 2
    got = words_to_cells((b if flip.value else a).cpu().numpy(), W)
    want, _ = oracle.run(oracle.random_fill(W, H, 0.4, 77), gens)
    assert np.array_equal(got, want)
