"""A/B: fused tcgen05 MLP vs cuBLAS + bias_gelu + row_ln on one backbone forward."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2412_16481_b200 import stage as ST  # noqa: E402
from paper_2412_16481_b200.backbone import Backbone  # noqa: E402

coords, feats = bench.workload(0)
C = torch.tensor(coords, device="cuda")
X = torch.tensor(feats, dtype=torch.float32, device="cuda")
bb = Backbone()
ST.FUSED_MLP = True
f1, c1 = bb.forward(C, X)
ST.FUSED_MLP = False
f0, c0 = bb.forward(C, X)
print("coords equal", torch.equal(c0, c1), "rows", f0.shape[0], f1.shape[0])
rel = ((f1.double() - f0.double()).norm() / f0.double().norm()).item()
print("fused vs unfused rel-Frobenius", rel)
