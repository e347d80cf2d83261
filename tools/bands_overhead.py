"""One-GPU cost of the multi-GPU band decompositions: the torus as 1 band vs
P emulated bands (NCCL-style ghost rows + device copies, and the fused
peer-mode kernel), same total work.  Prints T cell-updates/s."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1209_4408_b200.bands import BandDriver, LocalBands, LocalPeerBands, make_geometry

W = H = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
G = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dev = torch.device("cuda", 0)

def timeit(obj, label):
    obj.run(16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); obj.run(G); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{label:28s} {W*H*G/(ms*1e-3)/1e12:7.2f} T/s ({ms:.1f} ms)", flush=True)

d = BandDriver(make_geometry(W, H, 0, 1, 16), dev); d.init_random(0.5, 1); timeit(d, "torus 1 band"); del d
for P in (2, 4, 8):
    lb = LocalPeerBands(W, H, P, 16, dev); lb.init_random(0.5, 1); timeit(lb, f"peer-kernel {P} bands"); del lb
    lb = LocalBands(W, H, P, 16, dev); lb.init_random(0.5, 1); timeit(lb, f"ghost+copy {P} bands"); del lb
    torch.cuda.empty_cache()
