"""One profiled backbone forward (config B) for ncu:
    ncu --profile-from-start off ... python tools/prof_step.py
Warm-up steps run outside the cudaProfilerStart/Stop window."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2412_16481_b200.backbone import Backbone  # noqa: E402

steps = int(os.environ.get("PROF_STEPS", "1"))
coords, feats = bench.workload(0)
C = torch.tensor(coords, device="cuda")
X = torch.tensor(feats, dtype=torch.float32, device="cuda")
bb = Backbone()
for _ in range(3):
    bb.forward(C, X)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(steps):
    bb.forward(C, X)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled", steps, "step(s)")
