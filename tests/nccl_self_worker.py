"""Worker of tests/test_gpu_nccl_self.py: ONE rank on cuda:0 with the real NCCL
backend.  The rank is its own neighbour above and below (self send / receive),
so the NCCL halo exchange of bands.BandDriver and the neighbour token of the
peer band driver run under NCCL's stream semantics on a single GPU -- no kernel
waits on another process.  Prints one JSON line."""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.oracle import Oracle  # noqa: E402  (the checker)
from paper_1209_4408_b200.bands import (BandDriver, PeerBandDriver, make_geometry,  # noqa: E402
                                        neighbour_token)


def words_to_cells(words: np.ndarray, width: int) -> np.ndarray:
    u = np.ascontiguousarray(words).view(np.uint32)
    bits = np.unpackbits(u.view(np.uint8), axis=1, bitorder="little")
    return bits[:, :width].astype(np.uint8)


def main() -> None:
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    out = {"backend": dist.get_backend(), "world": dist.get_world_size(), "cases": []}
    O = Oracle()
    # (W, H, depth, interleave order, generations, checkpoints)
    cases = [(333, 257, 7, 0, 40, [0, 13, 40]),      # W % 32 != 0: seam path in the edge strips
             (1024, 300, 16, 0, 50, [0, 50]),
             (1024, 300, 10, 2, 33, [0, 7, 33]),     # pair layout: ghosts travel interleaved
             (1024, 300, 6, 4, 20, [0, 20]),         # quad layout
             (70, 37, 4, 0, 13, [0, 13])]
    for (W, H, depth, il, gens, cps) in cases:
        geo = make_geometry(W, H, 0, 1, depth, il, self_exchange=True)
        drv = BandDriver(geo, dev)
        drv.init_random(0.4, 9)
        pops = drv.run(gens, checkpoints=cps)
        torch.cuda.synchronize()
        got = words_to_cells(drv.band().cpu().numpy(), W)
        want, want_pops = O.run(O.random_fill(W, H, 0.4, 9), gens, cps)
        out["cases"].append({"case": [W, H, depth, il, gens], "grid": bool(np.array_equal(got, want)),
                             "pops": [int(p) for p in pops] == [int(p) for p in want_pops],
                             "exchange_bytes": drv.exchange_bytes})
    # The fused-halo driver: the band's own buffers stand in for the neighbours'
    # (peer-mode edge kernels), passes ordered by the NCCL neighbour token / the
    # all-rank all-reduce on the compute stream.
    out["peer_cases"] = []
    for (W, H, depth, il, gens, cps, sync) in [(333, 257, 7, 0, 40, [0, 13, 40], "neighbour"),
                                               (1024, 300, 16, 0, 50, [0, 50], "allreduce"),
                                               (1024, 300, 7, 4, 30, [0, 9, 30], "neighbour"),
                                               (1024, 300, 10, 2, 33, [0, 33], "neighbour"),
                                               (333, 257, 7, 0, 40, [0, 13, 40], "neighbour_overlap"),
                                               (1024, 300, 7, 4, 30, [0, 9, 30], "neighbour_overlap"),
                                               (1024, 21, 10, 2, 33, [0, 33], "neighbour_overlap"),
                                               (333, 257, 7, 0, 40, [0, 13, 40], "flag"),
                                               (1024, 300, 7, 4, 30, [0, 9, 30], "flag_overlap"),
                                               (1024, 21, 10, 2, 33, [0, 33], "flag_overlap")]:
        geo = make_geometry(W, H, 0, 1, depth, il, self_exchange=True)
        drv = PeerBandDriver(geo, dev, sync=sync, profile=True)
        drv.init_random(0.4, 9)
        pops = drv.run(gens, checkpoints=cps)
        st = drv.stats()
        got = words_to_cells(drv.band().cpu().numpy(), W)
        want, want_pops = O.run(O.random_fill(W, H, 0.4, 9), gens, cps)
        out["peer_cases"].append({"case": [W, H, depth, il, gens, sync], "sync": drv.sync,
                                  "grid": bool(np.array_equal(got, want)),
                                  "pops": [int(p) for p in pops] == [int(p) for p in want_pops],
                                  "passes": st["passes"], "barrier_ms": st["barrier_ms"]})
        drv.close()
    # Neighbour token: stream-ordered after the work queued before it, and the
    # work queued after wait() sees the received value (the host never blocks).
    token = torch.zeros(1, dtype=torch.int32, device=dev)
    inbox = torch.full((2,), -1, dtype=torch.int32, device=dev)
    big = torch.empty(1 << 28, dtype=torch.int32, device=dev)
    seen = []
    for i in range(1, 4):
        big.fill_(i)          # ~1 GiB of stores queued ahead of the token write
        token.fill_(i)
        neighbour_token(token, inbox, 0, 1)
        seen.append(inbox.clone())  # queued right after wait(): must hold both tokens
    torch.cuda.synchronize()
    out["tokens"] = [t.cpu().tolist() for t in seen]
    dist.destroy_process_group()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
