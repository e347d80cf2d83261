"""life_run_batch timing probe: ms for n = 1..3 grids of W x H (pinned host buffers)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1209_4408_b200 import capi, life  # noqa: E402

W = H = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
G = int(sys.argv[2]) if len(sys.argv) > 2 else 500
wpr = -(-W // 64)
eng = life.Engine(0)
eng.init_random(W, H, 0.4, 42)
host = torch.empty((H, wpr), dtype=torch.int64, pin_memory=True)
hin = host.numpy().view("uint64")
hin[:] = eng.download_packed().reshape(H, wpr)
out = torch.empty((H, wpr), dtype=torch.int64, pin_memory=True).numpy().view("uint64")
eng.run_batch([hin], [out], W, 16, 16)  # warm-up / allocation
t_run = None
for n in (1, 2, 3):
    ms = eng.run_batch([hin] * n, [out] * n, W, G, 16)
    print(json.dumps({"n": n, "ms": round(ms, 1), "gcups": round(W * H * G * n / ms / 1e6, 1)}))
