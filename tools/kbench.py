"""Quick packed-engine timing over arbitrary shapes (kernel-variant sweeps under gpurun).
usage: LIFE_GPU_LIB=... python tools/kbench.py WxH[,WxH...] GENS DEPTH [ENGINE]  -> one JSON line per shape
(ENGINE: 0 packed multi-pass (default), 2 cluster-resident)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1209_4408_b200 import capi, life  # noqa: E402

shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1].split(",")]
gens, depth = int(sys.argv[2]), int(sys.argv[3])
engine = int(sys.argv[4]) if len(sys.argv) > 4 else capi.ENGINE_PACKED
eng = life.Engine(0)
if os.environ.get("KB_PAIR") is not None:  # LIFE_OPT_PAIR_DEPTH: -1 auto, 0 off, 1..12 forced
    eng.set_option(capi.OPT_PAIR_DEPTH, int(os.environ["KB_PAIR"]))
if os.environ.get("KB_QUAD") is not None:  # LIFE_OPT_QUAD_DEPTH: -1 auto, 0 off, 1..7 forced
    eng.set_option(capi.OPT_QUAD_DEPTH, int(os.environ["KB_QUAD"]))
for (w, h) in shapes:
    eng.init_random(w, h, 0.4, 42)
    eng.run(max(depth, 1), engine, depth)
    eng.sync()
    best = 1e30
    for _ in range(3):
        t = time.perf_counter()
        eng.run(gens, engine, depth)
        eng.sync()
        best = min(best, time.perf_counter() - t)
    print(json.dumps({"lib": os.path.basename(os.environ.get("LIFE_GPU_LIB", "default")), "w": w, "h": h,
                      "depth": depth, "pair": os.environ.get("KB_PAIR"), "quad": os.environ.get("KB_QUAD"), "engine": engine, "gcups": round(w * h * gens / best / 1e9, 1)}))
