"""Prototype check of the quad layout (debug library, LIFE_QUAD=1: every pair-layout call
runs four words per lane): parity against the oracle on W % 128 == 0 tori, then timing."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1209_4408_b200 import capi, life  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
oracle = Oracle()

e = life.Engine(0)
bad = 0
for depth in (1, 2, 3, 4, 5, 6):
    e.set_option(capi.OPT_PAIR_DEPTH, depth)
    for i, (w, h) in enumerate([(128, 3), (128, 40), (256, 33), (384, 100), (3840, 50), (3968, 77),
                                (4096, 64), (4224, 9), (7936, 41), (8064, 130), (12800, 23)]):
        g = oracle.random_fill(w, h, 0.37, 100 + i)
        gens = 2 * depth + 3
        e.upload(g)
        pops = e.run(gens, 0, 0, [0, depth, gens])
        want, wpops = oracle.run(g, gens, [0, depth, gens])
        ok = np.array_equal(e.download(), want) and list(pops) == list(wpops)
        if not ok:
            bad += 1
            print("MISMATCH", w, h, depth)
print("quad parity:", "ok" if bad == 0 else f"{bad} mismatches")
