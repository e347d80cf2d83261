"""Cost of the multi-rank band drivers' pass machinery under the REAL NCCL backend on one GPU:
one rank that is its own neighbour above and below (BandGeometry.self_exchange), so the
interior / edge-strip launches, the peer-mode edge kernels, the NCCL neighbour token (or
all-reduce) between passes and the NCCL send/recv halos all run with NCCL's stream semantics,
timed against the plain one-band torus driver on the same grid.  What it cannot see: NVLink
latency of remote rows and the skew between ranks.
usage: python tools/nccl_self_bench.py W H GENS [REPS]   -> one JSON line"""
import ctypes as C
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1209_4408_b200 import capi  # noqa: E402
from paper_1209_4408_b200.bands import (BandDriver, PeerBandDriver, TorusDriver,  # noqa: E402
                                        make_geometry)

W, H, GENS = (int(v) for v in sys.argv[1:4])
REPS = int(sys.argv[4]) if len(sys.argv) > 4 else 2
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29517")
os.environ.setdefault("RANK", "0")
os.environ.setdefault("WORLD_SIZE", "1")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
L = capi.lib()
d = C.c_int32(0)
il = int(L.life_interleave_auto(W, H, -1, -1, 0, C.byref(d)))
depth = d.value if il else int(L.life_packed_auto_depth(W, H))


def timed(drv):
    drv.init_random(0.4, 42)
    drv.run(depth * 2)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(REPS):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        drv.run(GENS)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


out = {"w": W, "h": H, "gens": GENS, "depth": depth, "il": il, "backend": dist.get_backend(),
       "passes": -(-GENS // depth)}
drv = TorusDriver(make_geometry(W, H, 0, 1, depth, il), dev)
ms = timed(drv)
pop = drv.population()
out["torus"] = {"ms": ms, "gcups": W * H * GENS / ms / 1e6}
del drv
torch.cuda.empty_cache()
geo = make_geometry(W, H, 0, 1, depth, il, self_exchange=True)
for name, make in [("peer_neighbour_token", lambda: PeerBandDriver(geo, dev, sync="neighbour")),
                   ("peer_neighbour_token_overlapped",
                    lambda: PeerBandDriver(geo, dev, sync="neighbour_overlap")),
                   ("peer_flag", lambda: PeerBandDriver(geo, dev, sync="flag")),
                   ("peer_flag_overlapped", lambda: PeerBandDriver(geo, dev, sync="flag_overlap")),
                   ("peer_allreduce", lambda: PeerBandDriver(geo, dev, sync="allreduce")),
                   ("nccl_sendrecv_halo", lambda: BandDriver(geo, dev))]:
    drv = make()
    ms = timed(drv)
    ok = drv.population() == pop  # same soup, same generation count
    rec = {"ms": ms, "gcups": W * H * GENS / ms / 1e6, "vs_torus": out["torus"]["ms"] / ms,
           "population_equal": bool(ok),
           "extra_us_per_pass": (ms - out["torus"]["ms"]) * 1e3 / out["passes"]}
    if isinstance(drv, PeerBandDriver):
        drv.profile = True
        drv.init_random(0.4, 42)
        drv.run(GENS)
        st = drv.stats()
        rec["barrier_us_per_pass"] = st["barrier_ms"] * 1e3 / max(st["passes"], 1)
        drv.close()
    out[name] = rec
    del drv
    torch.cuda.empty_cache()
dist.destroy_process_group()
print(json.dumps(out))
