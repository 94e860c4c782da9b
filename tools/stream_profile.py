"""Timeline of Backbone.stream_host (torch profiler / CUPTI): compute-stream
busy time vs span, and the copies, to see what separates the pipelined e2e
step from the device-resident step."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2412_16481_b200.backbone import Backbone  # noqa: E402

coords, feats = bench.workload(0)
C_h = torch.tensor(coords).pin_memory()
X_h = torch.tensor(feats, dtype=torch.bfloat16).pin_memory()
bb = Backbone()
bb.stream_host([(C_h, X_h)] * 4)
torch.cuda.synchronize()
K = 8
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    bb.stream_host([(C_h, X_h)] * K)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
span = ev[-1].time_range.end - ev[0].time_range.start
kern = [e for e in ev if "Memcpy" not in e.name and "Memset" not in e.name]
cp = [e for e in ev if "Memcpy" in e.name]
busy = sum(e.time_range.end - e.time_range.start for e in kern)
print(f"span {span:.0f} us for {K} steps = {span / K:.0f} us/step; kernel busy {busy / K:.0f} us/step")
for e in cp[:8]:
    print(f"  {e.name[:30]:30s} start {e.time_range.start - ev[0].time_range.start:9.0f} dur {e.time_range.end - e.time_range.start:7.0f}")
# idle gaps on the compute timeline
kern.sort(key=lambda e: e.time_range.start)
gaps = sorted(((b.time_range.start - a.time_range.end), a.name[:30], b.name[:30],
               a.time_range.end - ev[0].time_range.start) for a, b in zip(kern, kern[1:]))[::-1]
for g in gaps[:10]:
    print(f"  gap {g[0]:7.1f} at {g[3]:8.0f}: {g[1]} -> {g[2]}")
