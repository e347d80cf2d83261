"""Per-warp SM placement and timing of one packed pass (LIFE_TRACE build)."""
import ctypes as C, os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LIFE_GPU_LIB"] = os.path.abspath("paper_1209_4408_b200/liblife_gpu_trace.so")
from paper_1209_4408_b200 import capi
from paper_1209_4408_b200.bands import BandDriver, make_geometry
W = H = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
K = int(sys.argv[2]) if len(sys.argv) > 2 else 8
L = capi.lib()
L.life_debug_set_trace.argtypes = [C.c_void_p]
tr = torch.zeros(3 * 200000, dtype=torch.int64, device="cuda")
L.life_debug_set_trace(tr.data_ptr())
drv = BandDriver(make_geometry(W, H, 0, 1, K), torch.device("cuda"))
drv.init_random(0.5, 42)
drv.run(K); torch.cuda.synchronize()
tr.zero_(); drv.run(K); torch.cuda.synchronize()
t = tr.view(-1, 3).cpu().numpy()
t = t[t[:, 2] > 0]
t0 = t[:, 1].min()
st, en, sm = (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, t[:, 0]
print("warps", len(t), "kernel span us", en.max())
print("start us: min %.1f p50 %.1f max %.1f" % (st.min(), np.median(st), st.max()))
print("end   us: min %.1f p50 %.1f p90 %.1f max %.1f" % (en.min(), np.median(en), np.percentile(en, 90), en.max()))
dur = en - st
print("dur   us: min %.1f p50 %.1f max %.1f" % (dur.min(), np.median(dur), dur.max()))
cnt = np.bincount(sm, minlength=148)
print("warps per SM: min %d max %d hist %s" % (cnt.min(), cnt.max(), np.bincount(cnt).tolist()))
smend = np.array([en[sm == i].max() if (sm == i).any() else 0 for i in range(148)])
print("SM finish us: min %.1f p50 %.1f max %.1f" % (smend.min(), np.median(smend), smend.max()))
# per-SM warps vs duration
for c in sorted(set(cnt.tolist())):
    sel = np.isin(sm, np.where(cnt == c)[0])
    print(f"  SMs with {c} warps: n={int((cnt==c).sum())} mean warp dur {dur[sel].mean():.1f} us")
idx = np.nonzero(tr.view(-1, 3).cpu().numpy()[:, 2] > 0)[0]
nw = -(-W // 32); ns = -(-nw // 30)
strip = idx % ns
per_strip = np.array([dur[strip == s].mean() for s in range(ns)])
print("per-strip mean dur: min %.1f max %.1f; strips slowest:" % (per_strip.min(), per_strip.max()),
      np.argsort(per_strip)[-5:].tolist(), "fastest:", np.argsort(per_strip)[:5].tolist())
order = np.argsort(dur)
print("slowest warps (gwarp, strip, seg, sm, dur):", [(int(idx[i]), int(strip[i]), int(idx[i] // ns), int(sm[i]), round(float(dur[i]))) for i in order[-8:]])
print("fastest warps:", [(int(idx[i]), int(strip[i]), int(idx[i] // ns), int(sm[i]), round(float(dur[i]))) for i in order[:8]])
# within-SM spread
spread = [dur[sm == i].max() / dur[sm == i].min() for i in range(148) if (sm == i).any()]
print("within-SM max/min dur: p50 %.2f max %.2f" % (np.median(spread), max(spread)))
# warp slot (gwarp % 4 = warp within block)
for wslot in range(4):
    print("  warp-in-block", wslot, "mean dur %.1f" % dur[idx % 4 == wslot].mean())
print("per-strip mean dur:", [int(x) for x in per_strip])
seg = idx // ns
nseg = seg.max() + 1
print("per-seg mean dur:", [int(dur[seg == s].mean()) for s in range(nseg)])
edge_sms = set(sm[(strip == 0) | (strip == ns - 1)].tolist())
print("SM finish, SMs hosting edge warps: %.1f ; others: %.1f (max %.1f)" % (
    np.mean([smend[i] for i in edge_sms]), np.mean([smend[i] for i in range(148) if i not in edge_sms]),
    max(smend[i] for i in range(148) if i not in edge_sms)))
