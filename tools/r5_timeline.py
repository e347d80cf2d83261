"""Phase timeline of the fast-only kernel's tiles (LIFE_TIMELINE build): per warp, %clock64 at
block-resident / previous-pass-complete / prologue done / first trip done / fill done / end.
usage: python tools/r5_timeline.py W H K PASSES"""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("LIFE_GPU_LIB", os.path.abspath("paper_1209_4408_b200/liblife_gpu_tl.so"))
from paper_1209_4408_b200 import capi, life
W, H, K, P = (int(v) for v in sys.argv[1:5])
L = capi.lib()
L.life_debug_set_trace.argtypes = [C.c_void_p]
L.life_debug_set_trace.restype = None
tr = torch.zeros(8 * 400000, dtype=torch.int64, device="cuda")
eng = life.Engine(0)
eng.set_option(capi.OPT_PAIR_DEPTH, 0)
eng.set_option(capi.OPT_QUAD_DEPTH, 0)
eng.init_random(W, H, 0.4, 42)
eng.run(K * 4, capi.ENGINE_PACKED, K)
eng.sync()
L.life_debug_set_trace(tr.data_ptr())
eng.run(K * P, capi.ENGINE_PACKED, K)
eng.sync()
L.life_debug_set_trace(None)
t = tr.view(-1, 8).cpu().numpy()
t = t[t[:, 5] > 0]
mhz = 1965.0
names = ["resident->prev pass complete", "griddep wait->prologue done (first rows requested)",
         "prologue->first trip done", "first trip->fill done", "fill done->end"]
print(f"{W}x{H} K={K}: {len(t)} tiles stamped (last pass)")
for i, nm in enumerate(names):
    d = (t[:, i + 1] - t[:, i]) / mhz
    print(f"  {nm:55s} us: p10 {np.percentile(d,10):7.2f} p50 {np.median(d):7.2f} p90 {np.percentile(d,90):7.2f}")
tot = (t[:, 5] - t[:, 1]) / mhz
print(f"  tile total after the wait: p50 {np.median(tot):.2f} us, max {tot.max():.2f}")
g = t[:, 6]
print(f"  globaltimer spread of 'previous pass complete' across warps: {(g.max() - g.min()) / 1e3:.2f} us")
sm = t[:, 7]
end_sm = {}
