"""torch.profiler view of one config-B forward: CPU-side time per Python
region vs GPU kernel time (finds host gaps between launches)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile, record_function  # noqa: E402

import bench  # noqa: E402
from paper_2412_16481_b200.backbone import Backbone  # noqa: E402

coords, feats = bench.workload(0)
C = torch.tensor(coords, device="cuda")
X = torch.tensor(feats, dtype=torch.float32, device="cuda")
bb = Backbone()
for _ in range(5):
    bb.forward(C, X)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    bb.forward(C, X)
torch.cuda.synchronize()
print("wall ms/step", (time.perf_counter() - t0) / 10 * 1e3)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], record_shapes=False) as prof:
    with record_function("forward"):
        bb.forward(C, X)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=40, max_name_column_width=60))
prof.export_chrome_trace(os.path.join(ROOT, "gpurun_out", "host_trace.json"))
