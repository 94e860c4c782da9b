"""Kernel busy time vs step span of the replayed config-B graphs (torch
profiler / CUPTI activity records): how much of a step is launch gaps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2412_16481_b200.backbone import Backbone  # noqa: E402

coords, feats = bench.workload(0)
bb = Backbone()
bb.capture(len(coords), torch.bfloat16)
bb.graph_coords.copy_(torch.tensor(coords, device="cuda"))
bb.graph_feats.copy_(torch.tensor(feats, dtype=torch.bfloat16, device="cuda"))
for _ in range(5):
    bb.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        bb.replay()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
# split into steps by the largest gaps: take the last step (3 replays)
n = len(ev) // 3
last = ev[-n:]
span = last[-1].time_range.end - last[0].time_range.start
busy = sum(e.time_range.end - e.time_range.start for e in last)
gaps = []
for a, b in zip(last, last[1:]):
    gaps.append((b.time_range.start - a.time_range.end, a.name[:40], b.name[:40]))
gaps.sort(reverse=True)
print(f"kernels/step {n}  span {span:.1f} us  busy {busy:.1f} us  gaps {span - busy:.1f} us")
for g in gaps[:12]:
    print(f"  gap {g[0]:6.1f} us  {g[1]} -> {g[2]}")
agg = {}
for e in last:
    k = e.name.split("(")[0][:60]
    d, c = agg.get(k, (0.0, 0))
    agg[k] = (d + e.time_range.end - e.time_range.start, c + 1)
print("warm kernel time per step:")
for k, (d, c) in sorted(agg.items(), key=lambda t: -t[1][0]):
    print(f"  {d:8.1f} us {c:3d}x {100 * d / busy:5.1f}%  {k}")
