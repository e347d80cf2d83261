"""life_run_batch(n = 1 and 3) on config 5 with the chunk-schedule trace (debug library,
LIFE_BATCH_TRACE=1): where the time of a chunked grid goes."""
import os
import sys
import time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1209_4408_b200 import capi, life  # noqa: E402

W = H = int(os.environ.get("TR_N", "262144"))
gens = int(os.environ.get("TR_GENS", "500"))
e = life.Engine(0)
wpr = W // 64
hin = torch.empty((H, wpr), dtype=torch.int64, pin_memory=True).numpy().view("uint64")
hout = torch.empty((H, wpr), dtype=torch.int64, pin_memory=True).numpy().view("uint64")
e.init_random(W, H, 0.4, 42, capi.ENGINE_PACKED)
e.download_packed(hin)
e.run_batch([hin], [hout], W, gens, 0)
for n in (1, 3):
    t = time.perf_counter()
    ms = e.run_batch([hin] * n, [hout] * n, W, gens, 0)
    print(f"n = {n}: event ms {ms:.1f}, host ms {1e3 * (time.perf_counter() - t):.1f}", flush=True)
