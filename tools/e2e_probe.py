"""Where does the end-to-end time go?  Times H2D / forward / D2H pieces."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2412_16481_b200.backbone import Backbone  # noqa: E402

coords, feats = bench.workload(0)
C_h = torch.tensor(coords).pin_memory()
X_h = torch.tensor(feats, dtype=torch.bfloat16).pin_memory()
print("pinned:", C_h.is_pinned(), X_h.is_pinned())
dev = torch.device("cuda")
bb = Backbone()


def ev_time(fn, n=10):
    ts = []
    for _ in range(n):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


print("H2D coords ms", ev_time(lambda: C_h.to(dev, non_blocking=True)))
print("H2D feats ms", ev_time(lambda: X_h.to(dev, non_blocking=True)))
Cd = C_h.to(dev)
Xd = X_h.to(dev)
for _ in range(3):
    bb.forward(Cd, Xd)
print("forward(dev) ms", ev_time(lambda: bb.forward(Cd, Xd)))
out = [None]


def fh():
    out[0], _ = bb.forward_host(C_h, X_h, out[0])


for _ in range(3):
    fh()
print("forward_host ms", ev_time(fh))
f, c = bb.forward(Cd, Xd)
fb = f.to(torch.bfloat16)
oh = torch.empty(fb.shape, dtype=fb.dtype).pin_memory()
print("D2H out ms", ev_time(lambda: oh.copy_(fb, non_blocking=True)))
t0 = time.perf_counter()
for _ in range(10):
    fh()
torch.cuda.synchronize()
print("forward_host wall ms", (time.perf_counter() - t0) / 10 * 1e3)
