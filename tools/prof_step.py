"""One profiled config-B backbone step for ncu, replayed from the captured
CUDA graphs exactly as bench.py times it:
    ncu --profile-from-start off ... python tools/prof_step.py
Capture and warm-up run outside the cudaProfilerStart/Stop window."""
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
X = torch.tensor(feats, dtype=torch.float32, device="cuda")     # as bench.py
bb = Backbone()
bb.capture(C.shape[0], torch.float32)
bb.graph_coords.copy_(C)
bb.graph_feats.copy_(X)
for _ in range(3):
    bb.replay()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(steps):
    bb.replay()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled", steps, "step(s); rows out", bb.check_graph())
